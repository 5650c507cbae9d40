// qfs_runtime.cu — context, device memory plan, sweep driver, host controller
// and the C ABI of libqfs.so (include/qfs.h).
//
// The sweep driver issues, per sweep:
//   forward (B cache)  -> K fused backward launches (chi update + E_i + polar)
//   -> final cost launch -> validation forward (when requested)
// on one CUDA stream, captured once into a CUDA graph per launch shape.  The
// host controller reads the S
// costs per sweep (a few bytes) and decides convergence, plateau, overtrain
// double-and-restart, max_iter, stop_on_first.  No CPU fallback exists: every
// arithmetic step of the sweep runs in qfs_kernels.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/qfs.h"
#include "qfs_internal.h"

using namespace qfs;

namespace {

enum KClass { K_FWD_ROW = 0, K_FWD_GATE, K_BWD, K_POLAR, K_FINAL, K_VAL_ROW, K_DIST, K_REDUCE,
              K_NCCL, K_OP, K_RES, K_NCLASS };
// profiling classes: fwd_gate / bwd / final / validation are PHASES (one event
// pair around the whole run of launches of that step of the sweep)
const char *kClassName[K_NCLASS] = {"unused", "fwd_gate", "bwd", "polar", "final",
                                    "validation", "dist", "row_reduce", "nccl_allreduce", "unit_op",
                                    "resident"};

struct ProfRec {
  int cls;
  cudaEvent_t e0, e1;
  double bytes, flops;
  long long n;  // kernel launches covered by the event pair
};
struct PhaseScope;

}  // namespace

struct qfs_ctx {
  int n = 0, K = 0, device = 0;
  long long N = 0;
  std::vector<int32_t> pairs;
  int2 *d_pairs = nullptr;
  std::vector<int32_t> kinds;  // gate kinds (qfs_set_gate_kinds), default all QFS_GATE_VAR2
  // multi-qubit blocks (qfs_create_blocks with at least one 3-qubit block):
  // packed d x d gates, gsz complex entries per start (16 K for pair circuits)
  bool blocks = false;
  long long gsz = 0;
  std::vector<BlkGate> bgh;
  BlkGate *d_bg = nullptr;
  double *d_bpart = nullptr;  // [S][kBlkMaxCtas][128] environment partials of the block path
  int *d_kinds = nullptr;
  cudaStream_t st = nullptr;
  cudaStream_t cur_st = nullptr;       // stream of the launches being issued
  // distribution
  ncclComm_t comm = nullptr;
  bool owns_comm = false;
  int rank = 0, world = 1, mode = 0;
  int *d_flag = nullptr;
  // samples
  int m_pool = 0, V = 0;
  bool have_samples = false;
  double2 *d_x = nullptr, *d_y = nullptr;    // pools, TRANSPOSED: [2^n][m_pool] (sample-minor)
  double2 *d_xv = nullptr, *d_yv = nullptr;  // validation, row-major [V][2^n]
  // work buffers
  int G_cap = 0, S_cap = 0, M_cap = 0, V_cap = 0, nb_cap = 0;
  int K_alloc = 0;  // gates d_pairs / d_kinds were sized for (qfs_set_structure)
  int K_g = 0;      // gates d_gates / d_vprev were sized for (ensure_gates)
  int K_s = 0;      // gates d_B / d_sig were sized for (ensure_state)
  bool force_unfused = false;  // QFS_UNFUSED_POLAR=1: separate polar launch (sample-mode code path at world 1)
  // QFS_BWD_BULK=1: perm mode — bulk-copy backward (bwdt_kernel) on per-gate
  // permuted layouts; measured 1.3x slower than the LDGSTS kernel at C4 / C5
  // (profiles/r2_bulk_summary.md), so off by default
  bool bwd_bulk = false;
  int bulk_min_m = 16;         // QFS_BULK_MIN_M: smallest M_max that takes the bulk-copy backward
  int V_glob = 0;   // validation rows over all ranks (sample mode: sum of the ranks' V)
  // sample mode, device-initiated exchange of E (qfs_set_exchange / NEXT-2)
  bool x_basis = false;  // qfs_set_samples_basis: x_m = e_m implicit (QFactor's full basis, NEXT-1); d_x unused
  int vr = 1;       // emulated ranks on this device (qfs_create_emulated); 1 otherwise
  int xchg = 0;     // 0: host-enqueued NCCL all-reduce + polar launch per gate; 1: device exchange
  int xS = 0;       // starts the mailboxes were sized for
  unsigned long long *d_xmbox = nullptr;  // own mailbox (emulated: every rank's)
  unsigned long long *d_xepoch = nullptr;
  unsigned long long **d_xmbox_tab = nullptr;  // [world] rank q's mailbox (IPC-mapped peers)
  std::vector<void *> x_mapped;           // IPC-opened peer blocks
  double2 *d_vprev = nullptr;  // [S][K][16] right singular vectors of the last polar step (warm start)
  double2 *d_gates = nullptr, *d_chi = nullptr, *d_B = nullptr, *d_vb0 = nullptr, *d_vb1 = nullptr;
  double2 *d_chi2 = nullptr;   // perm mode: chi ping-pongs between d_chi / d_chi2 (its layout changes per gate)
  double *d_partials = nullptr, *d_ered = nullptr, *d_sig = nullptr, *d_csum = nullptr,
         *d_rowout = nullptr, *d_cval = nullptr;
  unsigned *d_counters = nullptr;
  unsigned *d_counters1 = nullptr;   // [S][40] group tickets of the two-level backward reduction
  double *d_gpart = nullptr;         // [S][40][32] group sums
  Slot *d_slots = nullptr;
  double *h_csum = nullptr, *h_cval = nullptr;  // pinned
  double2 *d_env_trace = nullptr;
  size_t env_trace_cap = 0;
  double2 *d_stage = nullptr;  // row-major staging of the pools for the transpose
  int fwd_cache_mode = 0;   // QFS_FWD_CACHE: L2 hints of the forward kernel (diagnostic)
  bool fwd_pairs = true;    // QFS_FWD_PAIRS=0: one forward pass per gate
  bool val_block = true;    // QFS_VAL_BLOCK=0: one-row-per-CTA validation kernel
  int res_per_sm = 1;       // QFS_RES_PER_SM: resident CTAs per SM the cluster plan targets
  int res_cmax = 16;        // QFS_RES_CMAX: largest cluster the plan widens to
  bool sample_check_pending = false;
  bool host_read_pending = false;     // a kernel may still read a caller's pinned buffer (upload_gates)  // a consumed queued sample set's finite check, read back after the first sweep
  int res_pair = 0;         // QFS_RES_PAIR: two starts per cluster, staggered (0 off (default: measured slower), 1 auto, 2 wherever it fits)
  int path = 0;             // 0 auto, 1 streamed (B cache in HBM), 2 cluster-resident (qfs_set_path / QFS_PATH)
  size_t stage_bytes = 0;
  // qfs_set_samples_async: up to two sample sets queued in device staging
  // buffers (H2D on a copy stream, overlapping the running instantiation); the
  // next instantiate / trace / bench call consumes the oldest one
  struct Staged {
    double2 *x = nullptr, *y = nullptr, *xv = nullptr, *yv = nullptr;
    size_t cap_xy = 0, cap_v = 0;  // bytes per array
    int m_pool = 0, v = 0;
    cudaEvent_t ev = nullptr;
    const void *hx = nullptr, *hy = nullptr, *hxv = nullptr, *hyv = nullptr;  // caller's host buffers
    bool issued = false;           // H2D copies enqueued on st_copy
  } stg[2];
  int stg_head = 0, stg_count = 0;
  // QFS_COPY_DEFER=1: a queued set's H2D copies start only after the forward
  // phase of the next sweep (event recorded inside the sweep graph), i.e.
  // during the latency-bound backward instead of the write-bound forward
  bool copy_defer = true;
  bool pub_off = false;     // QFS_PUBLISH=0: results by D2H copy + stream synchronisation (A/B)
  cudaEvent_t ev_fwd = nullptr;
  // pinned host staging of the gates (upload / download through page-locked
  // memory, so the small copies do not queue behind a pageable staging path)
  double2 *h_gates = nullptr;
  size_t h_gates_cap = 0;
  Slot *h_slots = nullptr;  // mapped pinned slot table
  unsigned *h_check = nullptr;  // pinned read-back of the gate-check flag
  unsigned *d_check = nullptr;
  bool check_pending = false;
  bool check_fetched = false;   // h_check already read back with the last sweep's costs
  size_t h_slots_cap = 0;
  int slots_on_dev = 0;
  unsigned long long *h_pubflag = nullptr;  // mapped pinned: sequence number of the last published sweep
  unsigned long long pub_seq = 0;     // d_slots holds h_slots[0, slots_on_dev) (skip the upload when unchanged)
  cudaStream_t st_copy = nullptr;
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  long long gkey[8] = {0};
  long long glaunches = 0;
  // profiling
  bool prof = false, capturing = false;
  PhaseScope *phase = nullptr;  // open profiling phase (event pair around a run of launches)
  std::vector<ProfRec> prec;   // eager launches (events released after collection)
  std::vector<ProfRec> gprec;  // event nodes of the cached graph (kept with the graph)
  std::vector<cudaEvent_t> ev_pool;
  double p_ms[K_NCLASS] = {0}, p_bytes[K_NCLASS] = {0}, p_flops[K_NCLASS] = {0};
  long long p_cnt[K_NCLASS] = {0};
  long long launches = 0;
  std::string err;
  // diagnostics (env QFS_TAIL_TIMING=1): per-gate globaltimer stamps of bwd
  unsigned long long *d_dbg = nullptr;
  std::vector<double> dbg_acc;  // [3]: main phase, partial reduce, polar (ns, summed)
  unsigned long long *d_res_dbg = nullptr;  // [8] resident-kernel phase sums (ns), QFS_TAIL_TIMING
  long long res_sweeps = 0;
  long long dbg_n = 0;
};

qfs_status issue_deferred(qfs_ctx *c);  // queued sample sets' copies (defined with the ABI below)

namespace {

qfs_status fail(qfs_ctx *c, qfs_status s, const std::string &msg) {
  if (c) {
    c->err = msg;
    // an error return must not leave a kernel reading the caller's pinned gate
    // buffer after the call (the caller may free or overwrite it)
    if (c->host_read_pending && c->st) cudaStreamSynchronize(c->st);
    c->host_read_pending = false;
  }
  return s;
}

#define CUDA_TRY(c, expr)                                                                   \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(c, QFS_ERR_DEVICE, std::string(#expr " failed: ") + cudaGetErrorString(e_)); \
  } while (0)

#define NCCL_TRY(c, expr)                                                                   \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return fail(c, QFS_ERR_DEVICE, std::string(#expr " failed: ") + ncclGetErrorString(r_)); \
  } while (0)

template <typename T>
void dfree(T *&p) {
  if (p) cudaFree(p);
  p = nullptr;
}

// ---- profiling helpers: bracket a launch with events on the library stream
cudaEvent_t take_event(qfs_ctx *c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
void record_event(qfs_ctx *c, cudaEvent_t e) {
  // inside stream capture the record becomes an event node of the graph
  if (c->capturing) cudaEventRecordWithFlags(e, c->cur_st, cudaEventRecordExternal);
  else cudaEventRecord(e, c->cur_st);
}
// A run of launches of one kernel class timed by ONE event pair on the
// launching stream (forward phase, backward phase, ...): per-launch event
// pairs would serialise the graph and inflate every kernel's duration.
struct PhaseScope {
  qfs_ctx *c;
  int cls;
  cudaEvent_t e0 = nullptr;
  double bytes = 0, flops = 0;
  long long n = 0;
  PhaseScope(qfs_ctx *c_, int cls_) : c(c_), cls(cls_) {
    c->phase = this;
    if (c->prof) {
      e0 = take_event(c);
      record_event(c, e0);
    }
  }
  ~PhaseScope() {
    c->phase = nullptr;
    if (c->prof) {
      cudaEvent_t e1 = take_event(c);
      record_event(c, e1);
      (c->capturing ? c->gprec : c->prec).push_back({cls, e0, e1, bytes, flops, n});
    }
  }
};
// One kernel launch: counted, and attributed to the open phase (or, for the
// unit ops outside any phase, timed by its own event pair).
struct LaunchScope {
  qfs_ctx *c;
  int cls;
  double bytes, flops;
  cudaEvent_t e0 = nullptr;
  LaunchScope(qfs_ctx *c_, int cls_, double b, double f) : c(c_), cls(cls_), bytes(b), flops(f) {
    c->launches++;
    if (c->phase) {
      // a phase's launch count is its own kernel class (sample mode: the
      // all-reduce and polar launches inside the backward phase add time, not launches)
      c->phase->bytes += b;
      c->phase->flops += f;
      if (cls != K_NCCL && cls != K_POLAR) c->phase->n += 1;
    } else if (c->prof) {
      e0 = take_event(c);
      record_event(c, e0);
    }
  }
  ~LaunchScope() {
    if (!c->phase && c->prof) {
      cudaEvent_t e1 = take_event(c);
      record_event(c, e1);
      (c->capturing ? c->gprec : c->prec).push_back({cls, e0, e1, bytes, flops, 1});
    }
  }
};

// accumulate the event pairs of one replay of the cached graph (after a sync)
void prof_collect_graph(qfs_ctx *c) {
  for (auto &r : c->gprec) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    c->p_ms[r.cls] += ms;
    c->p_cnt[r.cls] += r.n;
    c->p_bytes[r.cls] += r.bytes;
    c->p_flops[r.cls] += r.flops;
  }
}

void drop_graph(qfs_ctx *c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
  for (auto &r : c->gprec) { c->ev_pool.push_back(r.e0); c->ev_pool.push_back(r.e1); }
  c->gprec.clear();
}

void prof_collect(qfs_ctx *c) {
  if (c->prec.empty()) return;
  cudaStreamSynchronize(c->st);
  for (auto &r : c->prec) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    c->p_ms[r.cls] += ms;
    c->p_cnt[r.cls] += r.n;
    c->p_bytes[r.cls] += r.bytes;
    c->p_flops[r.cls] += r.flops;
    c->ev_pool.push_back(r.e0);
    c->ev_pool.push_back(r.e1);
  }
  c->prec.clear();
}


// CTAs per start: one full wave over the 148 SMs (resident CTAs per SM = bpsm),
// never more CTAs than 256-item chunks.
constexpr int kMaxBlocksPerStart = 148 * 4;
int blocks_per_start(long long items, int n_slots, int bpsm = 4) {
  const int target = 148 * std::min(bpsm, 4);
  long long nb = target / n_slots;
  long long maxnb = (items + 255) / 256;
  if (nb > maxnb) nb = maxnb;
  if (nb < 1) nb = 1;
  return (int)nb;
}

// 32-bit addressing limit of the streamed kernels (bwd / fwd2 byte and element
// offsets inside one start's [2^n][rows] block, FastDiv numerators < 2^31):
// 2^n * rows * 16 B must stay below 4 GiB.
bool offsets_fit(const qfs_ctx *c, long long rows) { return ((long long)c->N * rows) < (1LL << 28); }

// memory plan (bytes) for S starts, M_cap rows per start, V validation rows
size_t plan_bytes(const qfs_ctx *c, int S, int M, int V, int nb) {
  size_t N = (size_t)c->N;
  size_t b = 0;
  b += (size_t)S * M * N * 16 * (c->K > 1 && c->bwd_bulk ? 2 : 1);  // chi (two buffers in perm mode)
  if (c->K > 1) b += (size_t)(c->K - 1) * S * M * N * 16;  // B cache
  if ((c->n > val_row_max_n() || c->blocks) && V > 0) b += 2 * (size_t)S * V * N * 16;
  if (c->blocks) b += (size_t)S * kBlkMaxCtas * 128 * 8;
  b += (size_t)S * nb * 32 * 8 + (size_t)S * 64 * 8 + (size_t)S * c->K * 8 + (size_t)S * (V + 4) * 8;
  return b;
}

qfs_status ensure_gates(qfs_ctx *c, int S) {
  // sized for G_cap starts of K_g gates: a structure with more gates
  // (qfs_set_structure) must reallocate even when S fits
  if (S <= c->G_cap && c->K <= c->K_g) return QFS_OK;
  S = std::max(S, c->G_cap);
  const int K = std::max(c->K, c->K_g);
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  dfree(c->d_gates);
  dfree(c->d_vprev);
  c->G_cap = 0;
  c->K_g = 0;
  drop_graph(c);
  // gsz = 16 K for pair circuits; block circuits never change structure
  const long long gsz = c->blocks ? c->gsz : 16LL * K;
  CUDA_TRY(c, cudaMalloc(&c->d_gates, (size_t)S * gsz * sizeof(double2)));
  CUDA_TRY(c, cudaMalloc(&c->d_vprev, (size_t)S * K * 16 * sizeof(double2)));
  c->G_cap = S;
  c->K_g = K;
  drop_graph(c);
  return QFS_OK;
}

// Per-sweep state (chi, B cache, validation buffers, reduction scratch) for S
// starts of up to M local rows.  Contents are rebuilt every sweep, so growing
// (on a double-and-restart) may discard them; the gates live elsewhere.
qfs_status ensure_state(qfs_ctx *c, int S, int M, int V) {
  const int nb = kMaxBlocksPerStart;  // any launch: nb <= 148 * 4 (blocks_per_start)
  if (S <= c->S_cap && M <= c->M_cap && V <= c->V_cap && nb <= c->nb_cap && c->K <= c->K_s) return QFS_OK;
  // the streamed kernels address one start's [2^n][rows] block with 32-bit
  // element / byte offsets and 32-bit FastDiv numerators: refuse shapes
  // where 2^n * rows * 16 B reaches 4 GiB instead of wrapping silently
  if (!offsets_fit(c, std::max(M, c->M_cap)))
    return fail(c, QFS_ERR_CAPACITY, "2^n * M * 16 B >= 4 GiB: beyond the 32-bit offsets of the streamed kernels");
  S = std::max(S, c->S_cap);
  M = std::max(M, c->M_cap);
  // perm mode's sample blocks (16 or 32 samples) must tile M_cap exactly
  if (c->bwd_bulk) {
    if (M > 16) M = (M + 31) / 32 * 32;
    else if (M > 8) M = 16;
  }
  V = std::max(V, c->V_cap);
  const int nbc = std::max(nb, c->nb_cap);
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  dfree(c->d_chi); dfree(c->d_chi2); dfree(c->d_B); dfree(c->d_vb0); dfree(c->d_vb1); dfree(c->d_bpart);
  dfree(c->d_partials); dfree(c->d_ered); dfree(c->d_sig); dfree(c->d_csum); dfree(c->d_rowout);
  c->d_cval = nullptr; dfree(c->d_counters); dfree(c->d_slots);
  dfree(c->d_counters1); dfree(c->d_gpart);
  if (c->h_csum) cudaFreeHost(c->h_csum);
  c->h_csum = c->h_cval = nullptr;
  c->S_cap = c->M_cap = c->V_cap = c->nb_cap = 0;
  c->K_s = 0;
  drop_graph(c);
  size_t need = plan_bytes(c, S, M, V, nbc);
  size_t fr = 0, tot = 0;
  CUDA_TRY(c, cudaMemGetInfo(&fr, &tot));
  if (need + (256ull << 20) > fr) {
    char buf[256];
    snprintf(buf, sizeof buf, "memory plan %.2f GB exceeds free device memory %.2f GB (S=%d M=%d)",
             need / 1e9, fr / 1e9, S, M);
    return fail(c, QFS_ERR_CAPACITY, buf);
  }
  const size_t N = (size_t)c->N;
  CUDA_TRY(c, cudaMalloc(&c->d_chi, (size_t)S * M * N * sizeof(double2)));
  if (c->K > 1 && c->bwd_bulk) CUDA_TRY(c, cudaMalloc(&c->d_chi2, (size_t)S * M * N * sizeof(double2)));
  if (c->K > 1) CUDA_TRY(c, cudaMalloc(&c->d_B, (size_t)(c->K - 1) * S * M * N * sizeof(double2)));
  if ((c->n > val_row_max_n() || c->blocks) && V > 0) {
    CUDA_TRY(c, cudaMalloc(&c->d_vb0, (size_t)S * V * N * sizeof(double2)));
    CUDA_TRY(c, cudaMalloc(&c->d_vb1, (size_t)S * V * N * sizeof(double2)));
  }
  if (c->blocks) CUDA_TRY(c, cudaMalloc(&c->d_bpart, (size_t)S * kBlkMaxCtas * 128 * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&c->d_partials, (size_t)S * nbc * 32 * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&c->d_ered, (size_t)S * 32 * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&c->d_sig, (size_t)S * c->K * sizeof(double)));
  // per-start cost sums: csum [S] then cval [S] in ONE buffer (device and
  // pinned host), so a sweep's results come back in one copy
  CUDA_TRY(c, cudaMalloc(&c->d_csum, (size_t)2 * S * sizeof(double)));
  c->d_cval = c->d_csum + S;
  CUDA_TRY(c, cudaMalloc(&c->d_rowout, (size_t)S * std::max(V, 1) * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&c->d_counters, (size_t)S * 2 * sizeof(unsigned)));
  CUDA_TRY(c, cudaMemset(c->d_counters, 0, (size_t)S * 2 * sizeof(unsigned)));
  CUDA_TRY(c, cudaMalloc(&c->d_slots, (size_t)S * sizeof(Slot)));
  CUDA_TRY(c, cudaMalloc(&c->d_counters1, (size_t)S * 40 * sizeof(unsigned)));
  CUDA_TRY(c, cudaMemset(c->d_counters1, 0, (size_t)S * 40 * sizeof(unsigned)));
  CUDA_TRY(c, cudaMalloc(&c->d_gpart, (size_t)S * 40 * 32 * sizeof(double)));
  CUDA_TRY(c, cudaHostAlloc((void **)&c->h_csum, (size_t)2 * S * sizeof(double), cudaHostAllocMapped));
  c->h_cval = c->h_csum + S;
  c->slots_on_dev = 0;  // d_slots is new
  c->S_cap = S; c->M_cap = M; c->V_cap = V; c->nb_cap = nbc;
  c->K_s = c->K;
  return QFS_OK;
}

void xchg_release(qfs_ctx *c) {
  for (void *p : c->x_mapped) cudaIpcCloseMemHandle(p);
  c->x_mapped.clear();
  dfree(c->d_xmbox); dfree(c->d_xepoch); dfree(c->d_xmbox_tab);
  c->xS = 0;
}

// Mailboxes of the device-initiated exchange (sample mode, qfs_set_exchange):
// per rank a block [2 parity][world src][S][64] self-validating words, zeroed; emulated ranks: all blocks in one local allocation;
// real ranks: each rank's own block, CUDA-IPC handles all-gathered over the
// context's NCCL communicator and the peers' blocks mapped (peer stores over
// NVLink).  Collective over the ranks (called in the same order by all).
qfs_status ensure_xchg(qfs_ctx *c, int S) {
  if (!(c->mode == 1 && c->world > 1 && c->xchg == 1) || S <= c->xS) return QFS_OK;
  const int g = c->world;
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  if (c->comm && c->xS > 0) {  // every rank is done with the old mailboxes before they go
    NCCL_TRY(c, ncclAllReduce(c->d_flag + 2, c->d_flag + 2, 1, ncclInt32, ncclMax, c->comm, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  }
  xchg_release(c);
  drop_graph(c);
  const size_t blk = ((size_t)2 * g * S * 64 * sizeof(unsigned long long) + 255) / 256 * 256;
  const int nblk = c->vr > 1 ? g : 1;
  char *base = nullptr;
  CUDA_TRY(c, cudaMalloc(&base, blk * nblk));
  CUDA_TRY(c, cudaMemsetAsync(base, 0, blk * nblk, c->st));  // epoch 0: no valid word
  c->d_xmbox = (unsigned long long *)base;
  CUDA_TRY(c, cudaMalloc(&c->d_xepoch, (size_t)nblk * S * sizeof(unsigned long long)));
  CUDA_TRY(c, cudaMemsetAsync(c->d_xepoch, 0, (size_t)nblk * S * sizeof(unsigned long long), c->st));
  std::vector<unsigned long long *> mt(g);
  if (c->vr > 1) {
    for (int q = 0; q < g; ++q) mt[q] = (unsigned long long *)(base + q * blk);
  } else {
    if (!c->comm) return fail(c, QFS_ERR_STATE, "device exchange needs the NCCL communicator of the ranks");
    cudaIpcMemHandle_t h;
    CUDA_TRY(c, cudaIpcGetMemHandle(&h, base));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    char *d_h = nullptr;
    CUDA_TRY(c, cudaMalloc(&d_h, (size_t)64 * g));
    CUDA_TRY(c, cudaMemcpyAsync(d_h + 64 * c->rank, &h, 64, cudaMemcpyHostToDevice, c->st));
    NCCL_TRY(c, ncclAllGather(d_h + 64 * c->rank, d_h, 64, ncclChar, c->comm, c->st));
    std::vector<cudaIpcMemHandle_t> all(g);
    CUDA_TRY(c, cudaMemcpyAsync(all.data(), d_h, (size_t)64 * g, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    cudaFree(d_h);
    for (int q = 0; q < g; ++q) {
      char *pq = base;
      if (q != c->rank) {
        void *mp = nullptr;
        CUDA_TRY(c, cudaIpcOpenMemHandle(&mp, all[q], cudaIpcMemLazyEnablePeerAccess));
        c->x_mapped.push_back(mp);
        pq = (char *)mp;
      }
      mt[q] = (unsigned long long *)pq;
    }
  }
  CUDA_TRY(c, cudaMalloc(&c->d_xmbox_tab, g * sizeof(unsigned long long *)));
  CUDA_TRY(c, cudaMemcpyAsync(c->d_xmbox_tab, mt.data(), g * sizeof(unsigned long long *), cudaMemcpyHostToDevice,
                              c->st));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));
  if (c->comm) {  // every rank's zeroed mailbox exists before anyone writes into it
    NCCL_TRY(c, ncclAllReduce(c->d_flag + 2, c->d_flag + 2, 1, ncclInt32, ncclMax, c->comm, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  }
  c->xS = S;
  return QFS_OK;
}

// ---------------------------------------------------------------- sweep ----
struct SweepSpec {
  std::vector<Slot> slots;   // active starts (local rows per start)
  int M_max = 0;
  bool want_val = false;
  bool want_sig = false;         // write sum sigma per gate (sigma traces only)
  double beta = 0.0;
  double2 *env_trace = nullptr;  // device [K][S][16] or nullptr
  int S = 0;                     // total starts (trace layout / strides)
};

// Descriptor of the fused backward step for gate i (union of gate i's pair
// with gate i+1's; local order: Q pair first, then gate i's other bits).
// The transposed pools [2^n][m_pool]; with emulated ranks one such block per
// rank (rank r = slot start r, qfs_create_emulated: one start only).
View pool_view(const qfs_ctx *c, const double2 *base) {
  if (base == c->d_x && c->x_basis) return View{nullptr, 0, 0, 0, 1};  // implicit x_m = e_m
  return View{base, c->vr > 1 ? c->N * c->m_pool : 0, c->m_pool, 1};
}

GateDesc make_desc(const qfs_ctx *c, int i) {
  const int K = c->K;
  const long long N = c->N, Mc = c->M_cap, sS = N * Mc;
  const View xpool = pool_view(c, c->d_x), ypool = pool_view(c, c->d_y);
  GateDesc d{};
  const bool upd = i < K - 1;
  d.upd = upd ? 1 : 0;
  d.upd_gate = upd ? i + 1 : -1;
  d.env_gate = i;
  d.pre = upd ? 1 : 0;  // phi = B_i (i < K-1) was written by the forward pass, not the previous launch
  const int p0 = c->pairs[2 * i], p1 = c->pairs[2 * i + 1];
  int loc[4], nu;
  if (!upd) {
    loc[0] = p0; loc[1] = p1; nu = 2;
  } else {
    loc[0] = c->pairs[2 * (i + 1)]; loc[1] = c->pairs[2 * (i + 1) + 1]; nu = 2;
    int ex[2], ne = 0;
    for (int q : {p0, p1})
      if (q != loc[0] && q != loc[1]) ex[ne++] = q;
    if (ne == 2 && ex[0] > ex[1]) std::swap(ex[0], ex[1]);
    for (int t = 0; t < ne; ++t) loc[nu++] = ex[t];
  }
  d.tp0 = d.tp1 = -1;
  for (int t = 0; t < nu; ++t) {
    if (loc[t] == p0) d.tp0 = t;
    if (loc[t] == p1) d.tp1 = t;
  }
  d.nu = nu;
  int srt[4];
  for (int t = 0; t < nu; ++t) srt[t] = loc[t];
  std::sort(srt, srt + nu);
  for (int t = 0; t < 4; ++t) d.ins[t] = t < nu ? srt[t] : 0;
  for (int v = 0; v < 16; ++v) {
    long long o = 0;
    for (int t = 0; t < nu; ++t)
      if ((v >> t) & 1) o |= 1LL << loc[t];
    d.off[v] = v < (1 << nu) ? o : 0;
  }
  auto Bk = [&](int k) -> double2 * { return c->d_B + (long long)(k - 1) * c->S_cap * sS; };
  d.chi_src = (i >= K - 2) ? ypool : View{c->d_chi, sS, Mc, 1};
  d.chi_dst = upd ? ViewW{c->d_chi, sS, Mc, 1} : ViewW{nullptr, 0, 0, 0};
  d.phi = i == 0 ? xpool : View{Bk(i), sS, Mc, 1};
  return d;
}


// ---- perm mode layouts (qfs_internal.h Scatter) ----------------
// L_i (0 <= i < K): the rows of gate i's environment group lowest, in the
// backward kernel's local order (make_desc: gate i+1's pair, then gate i's
// other qubits ascending; gate K-1: its own pair), the other qubits ascending
// above them.  L_{-1}: natural order.
struct Lay {
  int nu = 0;
  int loc[4] = {0, 0, 0, 0};
  int pos[kMaxQubits];  // natural qubit -> physical row bit
  int oth[kMaxQubits];  // the other qubits, ascending (the group index bits)
};
Lay layout_of(const qfs_ctx *c, int i) {
  Lay L;
  const int n = c->n, K = c->K;
  if (i < 0) {
    for (int b = 0; b < n; ++b) L.pos[b] = L.oth[b] = b;
    return L;
  }
  const int p0 = c->pairs[2 * i], p1 = c->pairs[2 * i + 1];
  if (i == K - 1) {
    L.loc[0] = p0; L.loc[1] = p1; L.nu = 2;
  } else {
    L.loc[0] = c->pairs[2 * (i + 1)]; L.loc[1] = c->pairs[2 * (i + 1) + 1]; L.nu = 2;
    int ex[2], ne = 0;
    for (int q : {p0, p1})
      if (q != L.loc[0] && q != L.loc[1]) ex[ne++] = q;
    if (ne == 2 && ex[0] > ex[1]) std::swap(ex[0], ex[1]);
    for (int t = 0; t < ne; ++t) L.loc[L.nu++] = ex[t];
  }
  bool in_u[kMaxQubits] = {false};
  for (int t = 0; t < L.nu; ++t) {
    in_u[L.loc[t]] = true;
    L.pos[L.loc[t]] = t;
  }
  int j = 0;
  for (int b = 0; b < n; ++b)
    if (!in_u[b]) { L.pos[b] = L.nu + j; L.oth[j++] = b; }
  return L;
}
// rows of (group G of src, local v over the qubits lloc[0..nl-1]) in layout dst
Scatter make_scatter(const Lay &src, const int *lloc, int nl, const Lay &dst, int n) {
  Scatter X{};
  for (int v = 0; v < 16; ++v) {
    int r = 0;
    if (v < (1 << nl))
      for (int t = 0; t < nl; ++t)
        if ((v >> t) & 1) r |= 1 << dst.pos[lloc[t]];
    X.dv[v] = r;
  }
  for (int j = 0; j < n - src.nu; ++j) X.dpos[j] = (unsigned char)dst.pos[src.oth[j]];
  return X;
}

// Plan of the cluster-resident sweep (qfs_resident.cu) for ns starts of up to
// M_max rows: the smallest power-of-two cluster whose CTAs hold their slice of
// phi and chi (2 * 2^n * ceil(M/C) complex128) plus the gate table in shared
// memory, widened while the starts still leave SMs idle and each CTA keeps >= 2
// rows.  False when no cluster size up to 16 fits (or in sample-sharded mode:
// the per-gate environment all-reduce crosses GPUs).
struct ResPlan {
  int C = 0, ld = 0, clusters = 0;
  size_t smem = 0;
  bool pair = false;  // res_pair_kernel: clusters of start pairs
};
bool res_plan(const qfs_ctx *c, int M_max, int ns, ResPlan &pl) {
  if (c->path == 1 || (c->mode == 1 && c->world > 1) || c->force_unfused || c->x_basis || c->n > 13 || M_max < 1)
    return false;
  // auto: resident only up to n = 10 — measured crossover (profiles/r1_sweep_map.jsonl:
  // n <= 10 resident 1.3-1.9x faster, n = 11 / 12 streamed 1.14x / 1.40x faster)
  if (c->path == 0 && c->n > 10) return false;
  // two starts per cluster (res_pair_kernel, one start's polar overlapped with
  // the other's passes) when there are at least two starts with enough work
  // per start for the passes to matter (auto: M 2^n >= 2^12); the smallest
  // power-of-two cluster that holds both starts' slices, widened like below
  if (c->res_pair && ns >= 2 && (c->res_pair == 2 || (((long long)M_max << c->n) >= 4096 && !c->d_res_dbg))) {
    int C2 = 1;
    for (; C2 <= 16; C2 *= 2)
      if (res2_smem_bytes(c->n, c->K, (M_max + C2 - 1) / C2) <= res_smem_limit(1)) break;
    if (C2 <= 16) {
      const int np = (ns + 1) / 2;
      while (C2 < c->res_cmax && (long long)np * 2 * C2 <= 148LL && (M_max + 2 * C2 - 1) / (2 * C2) >= 2) C2 *= 2;
      const int ld2 = (M_max + C2 - 1) / C2;
      const size_t sm2 = res2_smem_bytes(c->n, c->K, ld2);
      const int mx2 = resident2_max_clusters(C2, sm2);
      if (mx2 >= 1) {
        pl.pair = true;
        pl.C = C2;
        pl.ld = ld2;
        pl.smem = sm2;
        pl.clusters = std::min(np, mx2);
        return true;
      }
    }
  }
  // one CTA per SM (QFS_RES_PER_SM=2: two, <= 113 KB and <= 128 registers
  // each — measured slower: the per-gate chain is latency-bound, not
  // throughput-bound); then widen the cluster while the CTAs of all starts
  // still fit on the GPU at once and each keeps >= 2 rows
  int C = 1, per_sm = c->res_per_sm;
  if (per_sm == 2)
    for (; C <= 16; C *= 2)
      if (res_smem_bytes(c->n, c->K, (M_max + C - 1) / C) <= res_smem_limit(2)) break;
  if (per_sm != 2 || C > 16) {
    per_sm = 1;
    for (C = 1; C <= 16; C *= 2)
      if (res_smem_bytes(c->n, c->K, (M_max + C - 1) / C) <= res_smem_limit(1)) break;
    if (C > 16) return false;
  }
  while (C < c->res_cmax && (long long)ns * 2 * C <= 148LL * per_sm && (M_max + 2 * C - 1) / (2 * C) >= 2) C *= 2;
  pl.C = C;
  pl.ld = (M_max + C - 1) / C;
  pl.smem = res_smem_bytes(c->n, c->K, pl.ld);
  const int mx = resident_max_clusters(C, pl.smem);
  if (mx < 1) return false;
  pl.clusters = std::min(ns, mx);
  return true;
}

// Issue the launches of one sweep for the slots [j0, j1) on stream st (no host
// synchronisation).  Scratch arrays indexed by slot are offset by j0.

// One sweep of a multi-qubit block circuit for slots [j0, j1) (qfs_blocks.cu):
// the same steps as the streamed pair sweep below, one plain launch per step
// (P:112 right to left; P:127 / P:165 B cache; P:172 environments).
qfs_status issue_blocks(qfs_ctx *c, const SweepSpec &sp, int j0, int j1, cudaStream_t st) {
  const int ns = j1 - j0, K = c->K, n = c->n;
  int M_max = 0;
  for (int j = j0; j < j1; ++j) M_max = std::max(M_max, sp.slots[j].m);
  const Slot *slots = c->d_slots + j0;
  unsigned *cnt_b = c->d_counters + j0, *cnt_f = c->d_counters + c->S_cap + j0;
  double *csum = c->d_csum + j0, *cval = c->d_cval + j0;
  double *bpart = c->d_bpart + (long long)j0 * kBlkMaxCtas * 128;
  double *dpart = c->d_partials + (long long)j0 * c->nb_cap * 32;
  const long long N = c->N, Mc = c->M_cap, sS = N * Mc;
  const View xpool = pool_view(c, c->d_x), ypool = pool_view(c, c->d_y);
  auto Bk = [&](int k) -> double2 * { return c->d_B + (long long)(k - 1) * c->S_cap * sS; };
  double units = 0;
  for (int j = j0; j < j1; ++j) units += (double)sp.slots[j].m * (double)N;
  auto apply = [&](int k, int dagger, const View &src, const ViewW &dst, int rows_fixed, long long rows) -> qfs_status {
    BlkApplyParams a{};
    a.n = n; a.k = k; a.dagger = dagger; a.rows_fixed = rows_fixed; a.slots = slots; a.bg = c->d_bg;
    a.gates = c->d_gates; a.gsz = c->gsz; a.src = src; a.dst = dst;
    const int ar = c->bgh[k].a;
    CUDA_TRY(c, launch_blk_apply(a, ar, blk_ctas((N >> ar) * rows, ns), ns, st));
    c->launches++;
    return QFS_OK;
  };
  qfs_status r;
  // (a) forward: B_{k+1} = G_k B_k
  {
    PhaseScope phase(c, K_FWD_GATE);
    LaunchScope ls(c, K_FWD_GATE, units * 32.0 * (K - 1), 0.0);
    for (int k = 0; k + 1 < K; ++k)
      if ((r = apply(k, 0, k == 0 ? xpool : View{Bk(k), sS, Mc, 1}, ViewW{Bk(k + 1), sS, Mc, 1}, 0, M_max)) != QFS_OK)
        return r;
  }
  // (b, c) backward: chi <- G_{i+1}^dag chi, then E_i and the update of gate i
  {
    PhaseScope phase(c, K_BWD);
    LaunchScope ls(c, K_BWD, units * 48.0 * K, 0.0);
    for (int i = K - 1; i >= 0; --i) {
      if (i < K - 1)
        if ((r = apply(i + 1, 1, i == K - 2 ? ypool : View{c->d_chi, sS, Mc, 1}, ViewW{c->d_chi, sS, Mc, 1}, 0, M_max)) !=
            QFS_OK)
          return r;
      BlkEnvParams e{};
      e.n = n; e.i = i; e.K = K; e.S = sp.S; e.slots = slots; e.bg = c->d_bg; e.gates = c->d_gates; e.gsz = c->gsz;
      e.phi = i == 0 ? xpool : View{Bk(i), sS, Mc, 1};
      e.chi = i == K - 1 ? ypool : View{c->d_chi, sS, Mc, 1};
      e.partials = bpart; e.counters = cnt_b; e.beta = sp.beta; e.sig = sp.want_sig ? c->d_sig : nullptr;
      e.env_trace = sp.env_trace; e.err = c->d_check;
      const int ar = c->bgh[i].a;
      CUDA_TRY(c, launch_blk_env(e, ar, blk_ctas((N >> ar) * M_max, ns), ns, st));
      c->launches++;
    }
  }
  // (d) c_train: chi' = G_0^dag chi, sum ||chi' - x||^2 (P:116-120 direct form)
  {
    PhaseScope phase(c, K_FINAL);
    LaunchScope ls(c, K_FINAL, units * 32.0, 0.0);
    if ((r = apply(0, 1, K == 1 ? ypool : View{c->d_chi, sS, Mc, 1}, ViewW{c->d_chi, sS, Mc, 1}, 0, M_max)) != QFS_OK)
      return r;
    BlkDistParams d{};
    d.n = n; d.rows_fixed = 0; d.slots = slots; d.a = View{c->d_chi, sS, Mc, 1}; d.b = xpool;
    d.partials = dpart; d.counters = cnt_f; d.out = csum;
    CUDA_TRY(c, launch_blk_dist(d, blk_ctas(N * M_max, ns), ns, st));
    c->launches++;
  }
  // validation cost: V rows through the post-sweep gates
  if (sp.want_val && c->V > 0) {
    PhaseScope phase(c, K_VAL_ROW);
    LaunchScope ls(c, K_VAL_ROW, (double)ns * c->V * N * 32.0 * K, 0.0);
    const long long VN = (long long)c->V * N;
    for (int k = 0; k < K; ++k) {
      double2 *dst = (k & 1) ? c->d_vb1 : c->d_vb0;
      const View src = k == 0 ? View{c->d_xv, 0, 1, N} : View{(k & 1) ? c->d_vb0 : c->d_vb1, VN, 1, N};
      if ((r = apply(k, 0, src, ViewW{dst, VN, 1, N}, c->V, c->V)) != QFS_OK) return r;
    }
    BlkDistParams d{};
    d.n = n; d.rows_fixed = c->V; d.slots = slots;
    d.a = View{((K - 1) & 1) ? c->d_vb1 : c->d_vb0, VN, 1, N};
    d.b = View{c->d_yv, 0, 1, N};
    d.partials = dpart; d.counters = cnt_f; d.out = cval;
    CUDA_TRY(c, launch_blk_dist(d, blk_ctas(VN, ns), ns, st));
    c->launches++;
  }
  return QFS_OK;
}

qfs_status issue_group(qfs_ctx *c, const SweepSpec &sp, int j0, int j1, cudaStream_t st) {
  if (c->blocks) return issue_blocks(c, sp, j0, j1, st);
  const int ns = j1 - j0;
  const int K = c->K, n = c->n;
  c->cur_st = st;
  int M_max = 0;
  for (int j = j0; j < j1; ++j) M_max = std::max(M_max, sp.slots[j].m);
  ResPlan pl;
  if (res_plan(c, M_max, ns, pl)) {
    // whole sweep + costs + validation in one cluster-resident launch
    ResParams r{};
    r.n = n; r.K = K; r.S = sp.S; r.C = pl.C; r.ld = pl.ld; r.n_slots = ns; r.kinds = c->d_kinds;
    r.slots = c->d_slots + j0; r.pairs = c->d_pairs; r.gates = c->d_gates;
    r.x = c->d_x; r.y = c->d_y; r.m_pool = c->m_pool; r.xv = c->d_xv; r.yv = c->d_yv;
    r.V = c->V; r.want_val = sp.want_val ? 1 : 0; r.beta = sp.beta;
    r.csum = c->d_csum + j0; r.cval = c->d_cval + j0; r.sig = sp.want_sig ? c->d_sig : nullptr; r.env_trace = sp.env_trace;
    r.dbg = c->d_res_dbg;
    double units = 0;
    for (int j = j0; j < j1; ++j) units += (double)sp.slots[j].m * (double)c->N;
    const double vunits = (sp.want_val && c->V > 0) ? (double)ns * c->V * (double)c->N : 0.0;
    PhaseScope phase(c, K_RES);
    // algorithmic flops of the sweep only (96 per amp-gate;
    // the uncompute's extra 32 and the fused validation are not counted)
    (void)vunits;
    LaunchScope ls(c, K_RES, 0.0, units * 96.0 * K);
    CUDA_TRY(c, pl.pair ? launch_resident_pair(r, pl.clusters, st) : launch_resident(r, pl.clusters, st));
    return QFS_OK;
  }
  if (c->path == 2) return fail(c, QFS_ERR_CAPACITY, "resident path requested but the state does not fit");
  const Slot *slots = c->d_slots + j0;
  double *partials = c->d_partials + (long long)j0 * c->nb_cap * 32;
  unsigned *cnt_b = c->d_counters + j0, *cnt_f = c->d_counters + c->S_cap + j0;
  double *ered = c->d_ered + (long long)j0 * 32, *csum = c->d_csum + j0, *cval = c->d_cval + j0;
  double *rowout = c->d_rowout + (long long)j0 * std::max(c->V, 1);
  const long long N = c->N;
  const long long Mc = c->M_cap;
  const View xpool = pool_view(c, c->d_x), ypool = pool_view(c, c->d_y);
  const long long sS = N * Mc;                      // per-start stride of chi / B
  auto Bk = [&](int k) -> double2 * { return c->d_B + (long long)(k - 1) * c->S_cap * sS; };
  double units = 0;  // amplitudes of all active training rows
  for (int j = j0; j < j1; ++j) units += (double)sp.slots[j].m * (double)N;
  // perm mode (bulk-copy backward): B cache and chi in the per-gate permuted
  // sample-blocked layouts L_i (qfs_internal.h); else natural sample-minor
  const bool perm = c->bwd_bulk && M_max >= c->bulk_min_m && M_max >= 16 && !c->x_basis && c->d_chi2 &&
                    c->M_cap % (c->M_cap >= 32 ? 32 : 16) == 0;
  const int psb = c->M_cap >= 32 ? 32 : 16;
  const long long pblk = N * psb;
  std::vector<Lay> lays;
  if (perm) {
    lays.reserve(K + 1);
    for (int i = -1; i < K; ++i) lays.push_back(layout_of(c, i));
  }
  auto LY = [&](int i) -> const Lay & { return lays[i + 1]; };
  auto chibuf = [&](int i) -> double2 * { return (i & 1) ? c->d_chi2 : c->d_chi; };
  // (a) forward: B_1 .. B_{K-1}: two gates per coalesced pass
  // (a single-gate pass for an odd tail)
  if (K > 1 && perm) {
    PhaseScope phase_fwd(c, K_FWD_GATE);
    for (int k = 0; k + 1 < K; k += 2) {
      FwdpParams f{};
      f.n = n; f.k = k; f.K = K; f.slots = slots; f.gates = c->d_gates; f.sb = psb; f.blk = pblk;
      int loc[4] = {c->pairs[2 * k], c->pairs[2 * k + 1], 0, 0}, nu = 2;
      const int q0 = c->pairs[2 * (k + 1)], q1 = c->pairs[2 * (k + 1) + 1];
      int ex[2], ne = 0;
      for (int q : {q0, q1})
        if (q != loc[0] && q != loc[1]) ex[ne++] = q;
      if (ne == 2 && ex[0] > ex[1]) std::swap(ex[0], ex[1]);
      for (int t = 0; t < ne; ++t) loc[nu++] = ex[t];
      f.nu = nu;
      for (int t = 0; t < nu; ++t) {
        if (loc[t] == q0) f.tp0 = t;
        if (loc[t] == q1) f.tp1 = t;
      }
      const Lay &Lk = LY(k);  // the group's qubit set = gates k, k+1 (L_k's low bits)
      f.n_oth = n - Lk.nu;
      f.src_nat = k == 0 ? 1 : 0;
      int srt[4];
      for (int t = 0; t < nu; ++t) srt[t] = loc[t];
      std::sort(srt, srt + nu);
      for (int t = 0; t < 4; ++t) f.ins[t] = t < nu ? srt[t] : 0;
      for (int v = 0; v < 16; ++v) {
        long long o = 0;
        int r = 0;
        for (int t = 0; t < nu && v < (1 << nu); ++t)
          if ((v >> t) & 1) { o |= 1LL << loc[t]; r |= 1 << Lk.pos[loc[t]]; }
        f.off[v] = o;
        f.tau[v] = r;
      }
      f.src = k == 0 ? xpool : View{Bk(k), sS, Mc, 1};
      f.dst1 = ViewW{Bk(k + 1), sS, Mc, 1};
      f.s1 = make_scatter(Lk, loc, nu, LY(k + 1), n);
      if (k + 2 < K) {
        f.dst2 = ViewW{Bk(k + 2), sS, Mc, 1};
        f.s2 = make_scatter(Lk, loc, nu, LY(k + 2), n);
      }
      f.nb = blocks_per_start(((long long)M_max * N) >> nu, ns, 1);  // fwdp_kernel: 256 threads, one CTA per SM
      const double fb = k + 2 < K ? 48.0 : 32.0;
      LaunchScope ls(c, K_FWD_GATE, units * fb, units * (k + 2 < K ? 64.0 : 32.0));
      CUDA_TRY(c, launch_fwdp(f, ns, st));
    }
  }
  if (K > 1 && !perm) {
  PhaseScope phase_fwd(c, K_FWD_GATE);
  for (int k = 0; k + 1 < K;) {
    const View src = k == 0 ? xpool : View{Bk(k), sS, Mc, 1};
    if (k + 2 < K && c->fwd_pairs) {
      Fwd2Params f{};
      f.n = n; f.k = k; f.K = K; f.slots = slots; f.gates = c->d_gates;
      int loc[4] = {c->pairs[2 * k], c->pairs[2 * k + 1], 0, 0}, nu = 2;
      const int q0 = c->pairs[2 * (k + 1)], q1 = c->pairs[2 * (k + 1) + 1];
      int ex[2], ne = 0;
      for (int q : {q0, q1})
        if (q != loc[0] && q != loc[1]) ex[ne++] = q;
      if (ne == 2 && ex[0] > ex[1]) std::swap(ex[0], ex[1]);
      for (int t = 0; t < ne; ++t) loc[nu++] = ex[t];
      f.nu = nu;
      for (int t = 0; t < nu; ++t) {
        if (loc[t] == q0) f.tp0 = t;
        if (loc[t] == q1) f.tp1 = t;
      }
      int srt[4];
      for (int t = 0; t < nu; ++t) srt[t] = loc[t];
      std::sort(srt, srt + nu);
      for (int t = 0; t < 4; ++t) f.ins[t] = t < nu ? srt[t] : 0;
      for (int v = 0; v < 16; ++v) {
        long long o = 0;
        for (int t = 0; t < nu; ++t)
          if ((v >> t) & 1) o |= 1LL << loc[t];
        f.off[v] = v < (1 << nu) ? o : 0;
      }
      f.nb = blocks_per_start(((long long)M_max * N) >> nu, ns, fwd2_min_blocks());
      f.src = src;
      f.dst1 = ViewW{Bk(k + 1), sS, Mc, 1};
      f.dst2 = ViewW{Bk(k + 2), sS, Mc, 1};
      LaunchScope ls(c, K_FWD_GATE, units * 48.0, units * 64.0);
      CUDA_TRY(c, launch_fwd2(f, ns, st));
      k += 2;
    } else {
      FwdGateParams f{};
      f.n = n; f.k = k; f.K = K; f.rows_fixed = 0; f.slots = slots;
      f.p0 = c->pairs[2 * k]; f.p1 = c->pairs[2 * k + 1]; f.gates = c->d_gates;
      f.nb = blocks_per_start(((long long)M_max * N) >> 2, ns, 3);
      f.src = src;
      f.dst = ViewW{Bk(k + 1), sS, Mc, 1};
      f.cache_mode = c->fwd_cache_mode;
      LaunchScope ls(c, K_FWD_GATE, units * 32.0, units * 32.0);
      CUDA_TRY(c, launch_fwd_gate(f, ns, st));
      k += 1;
    }
  }
  }
  if (c->copy_defer && c->ev_fwd) {  // queued sample sets start copying from here (QFS_COPY_DEFER)
    if (c->capturing) CUDA_TRY(c, cudaEventRecordWithFlags(c->ev_fwd, st, cudaEventRecordExternal));
    else CUDA_TRY(c, cudaEventRecord(c->ev_fwd, st));
  }
  // (b, c) backward: gate i = K-1 .. 0 (P:112 right to left; Fig. env_calc)
  BwdParams b{};
  b.n = n; b.K = K; b.S = sp.S; b.slots = slots; b.gates = c->d_gates; b.gates_w = c->d_gates;
  b.kinds = c->d_kinds;
  b.partials = partials; b.counters = cnt_b; b.e_red = ered;
  b.counters1 = c->d_counters1 + (long long)j0 * 40; b.gpartials = c->d_gpart + (long long)j0 * 40 * 32;
  const bool sample_ar = c->mode == 1 && c->world > 1;  // per-gate exchange of E
  const bool dev_x = sample_ar && c->xchg == 1;         // ... device-initiated (NEXT-2)
  b.fuse_polar = ((sample_ar && !dev_x) || c->force_unfused) ? 0 : 1;
  if (dev_x) {
    b.xg = c->world; b.xrank = c->vr > 1 ? -1 : c->rank; b.xS = c->xS;
    b.xmbox = c->d_xmbox_tab; b.xepoch = c->d_xepoch;
  }
  b.beta = sp.beta; b.sig = sp.want_sig ? c->d_sig : nullptr; b.env_trace = sp.env_trace;
  b.vprev = c->d_vprev;
  b.dbg = c->d_dbg;
  double bwd_bytes = 0, bwd_flops = 0;
  for (int i = K - 1; i >= 0; --i) {
    bwd_bytes += units * (i < K - 1 ? 48.0 : 32.0);
    bwd_flops += units * (i < K - 1 ? 64.0 : 32.0);
  }
  {
  PhaseScope phase_bwd(c, K_BWD);
  for (int i = K - 1; i >= 0; --i) {
    b.g = make_desc(c, i);
    const bool upd = b.g.upd != 0;
    const int nu = b.g.nu;
    b.bulk = perm ? 1 : 0;
    if (perm) {
      GateDesc &d = b.g;
      d.perm = 1; d.sb = psb; d.blk = pblk; d.n_oth = n - nu;
      d.chi_nat = i >= K - 2 ? 1 : 0;   // chi = the y pool
      d.phi_nat = i == 0 ? 1 : 0;       // phi = the x pool
      // chi changes layout every gate, so it cannot be updated in place (a
      // group's rows in L_{i-1} belong to other groups of L_i): launch i
      // reads buffer i & 1 and writes buffer (i - 1) & 1
      if (!d.chi_nat) d.chi_src = View{chibuf(i), sS, Mc, 1};
      if (upd) d.chi_dst = ViewW{chibuf(i - 1), sS, Mc, 1};
      if (upd) d.xs = make_scatter(LY(i), LY(i).loc, nu, LY(i - 1), n);
    }
    if (b.bulk) {
      // one CTA per SM over all starts (the ring of stages fills the SM's shared memory)
      const long long un = (N >> nu) * ((M_max + 31) / 32);
      long long nb = std::max(1, 148 / ns);
      nb = std::min(nb, std::max(1LL, un / bwdt_units_per_cta_min()));
      b.nb = (int)nb;
    } else {
      const long long lpt = 32 >> (nu - 2);
      const long long un = (N >> nu) * ((M_max + lpt - 1) / lpt);
      b.nt = bwd_threads(ns);
      b.nb = blocks_per_start(un * 32, ns, blocks_per_sm(b.nt));
    }
    {
      LaunchScope ls(c, K_BWD, units * (upd ? 48.0 : 32.0), units * (upd ? 64.0 : 32.0));
      CUDA_TRY(c, launch_bwd(b, ns, st));
    }
    if (!b.fuse_polar) {
      if (c->mode == 1 && c->comm) {  // (a one-rank communicator too, with QFS_UNFUSED_POLAR)
        LaunchScope ls(c, K_NCCL, 0, 0);
        NCCL_TRY(c, ncclAllReduce(ered, ered, (size_t)ns * 32, ncclFloat64, ncclSum,
                                  c->comm, st));
      }
      PolarParams pp{};
      pp.K = K; pp.gate = i; pp.S = sp.S; pp.n_slots = ns; pp.slots = slots; pp.kinds = c->d_kinds;
      pp.e_red = ered; pp.gates = c->d_gates; pp.beta = sp.beta; pp.sig = sp.want_sig ? c->d_sig : nullptr;
      pp.env_trace = sp.env_trace; pp.vprev = c->d_vprev;
      LaunchScope ls(c, K_POLAR, 0, 0);
      CUDA_TRY(c, launch_polar(pp, ns, st));
    }
  }
  }
  // (d) c_train = (1/M) sum ||G_0^dag chi - x||^2   (direct form R6)
  {
    PhaseScope phase_final(c, K_FINAL);
    FinalParams fp{};
    fp.n = n; fp.slots = slots;
    fp.chi = K == 1 ? ypool : View{c->d_chi, sS, Mc, 1};
    fp.x = xpool; fp.p0 = c->pairs[0]; fp.p1 = c->pairs[1]; fp.gates = c->d_gates; fp.K = K;
    fp.sb = (perm && K > 1) ? psb : 0;  // chi after gate 0: layout L_{-1}, sample-blocked
    fp.blk = pblk;
    if (perm && K > 1) fp.chi = View{chibuf(-1), sS, Mc, 1};
    fp.partials = partials; fp.counters = cnt_f; fp.out_sum = csum;
    fp.nb = blocks_per_start(((long long)M_max * N) >> 2, ns);
    LaunchScope ls(c, K_FINAL, units * 32.0, units * 35.0);
    CUDA_TRY(c, launch_final(fp, ns, st));
  }
  if (c->mode == 1 && c->comm && (sample_ar || c->force_unfused)) {
    LaunchScope ls(c, K_NCCL, 0, 0);
    NCCL_TRY(c, ncclAllReduce(csum, csum, ns, ncclFloat64, ncclSum, c->comm, st));
  }
  // validation cost with the post-sweep gates
  if (sp.want_val && c->V > 0) {
    PhaseScope phase_val(c, K_VAL_ROW);
    const double vunits = (double)ns * c->V * (double)N;
    if (n <= val_row_max_n()) {
      ValRowParams f{};
      f.n = n; f.K = K; f.rows = c->V; f.slots = slots; f.pairs = c->d_pairs;
      f.gates = c->d_gates; f.xv = c->d_xv; f.yv = c->d_yv; f.row_out = rowout;
      LaunchScope ls(c, K_VAL_ROW, vunits * 32.0, vunits * 32.0 * K);
      if (c->val_block && val_blk_smem(n, K, 1) + 256 <= res_smem_limit(1)) CUDA_TRY(c, launch_val_block(f, ns, st));
      else CUDA_TRY(c, launch_val_row(f, ns, st));
    } else if (c->val_block && val_cl_smem(n, K, 3) + 256 <= res_smem_limit(1)) {
      // one row per cluster of 2-8 CTAs (n >= 14 rows exceed one CTA's shared memory)
      ValRowParams f{};
      f.n = n; f.K = K; f.rows = c->V; f.slots = slots; f.pairs = c->d_pairs;
      f.gates = c->d_gates; f.xv = c->d_xv; f.yv = c->d_yv; f.row_out = rowout;
      LaunchScope ls(c, K_VAL_ROW, vunits * 32.0, vunits * 32.0 * K);
      CUDA_TRY(c, launch_val_cluster(f, ns, st));
    } else {
      const long long VN = (long long)c->V * N;
      for (int k = 0; k < K; ++k) {
        FwdGateParams f{};
        f.n = n; f.k = k; f.K = K; f.rows_fixed = c->V; f.slots = slots;
        f.p0 = c->pairs[2 * k]; f.p1 = c->pairs[2 * k + 1]; f.gates = c->d_gates;
        f.nb = blocks_per_start(((long long)c->V * N) >> 2, ns);
        double2 *dst = (k & 1) ? c->d_vb1 : c->d_vb0;
        const double2 *src = k == 0 ? c->d_xv : ((k & 1) ? c->d_vb0 : c->d_vb1);
        f.src = View{src, k == 0 ? 0 : VN, 1, N};
        f.dst = ViewW{dst, VN, 1, N};
        LaunchScope ls(c, K_FWD_GATE, vunits * 32.0, vunits * 32.0);
        CUDA_TRY(c, launch_fwd_gate(f, ns, st));
      }
      DistParams d{};
      d.n = n; d.rows = c->V; d.slots = slots;
      d.a = View{((K - 1) & 1) ? c->d_vb1 : c->d_vb0, VN, 1, N};
      d.b = View{c->d_yv, 0, 1, N}; d.row_out = rowout;
      LaunchScope ls(c, K_DIST, vunits * 32.0, vunits * 3.0);
      CUDA_TRY(c, launch_dist(d, ns, st));
    }
    {
      LaunchScope ls(c, K_REDUCE, 0, 0);
      CUDA_TRY(c, launch_row_reduce(rowout, c->V, cval, ns, st));
    }
    if (c->mode == 1 && c->comm && (sample_ar || c->force_unfused)) {
      // sample mode: every rank holds its own validation shard; the sums are
      // all-reduced so all ranks take identical controller decisions
      LaunchScope ls(c, K_NCCL, 0, 0);
      NCCL_TRY(c, ncclAllReduce(cval, cval, ns, ncclFloat64, ncclSum, c->comm, st));
    }
  }
  return QFS_OK;
}

// Issue one sweep on the context stream (all active starts in lockstep).
qfs_status issue_sweep(qfs_ctx *c, const SweepSpec &sp) {
  return issue_group(c, sp, 0, (int)sp.slots.size(), c->st);
}

// Spin until the publish kernel of sweep `seq` has written its results (see
// publish_kernel); every 256 polls the stream is queried, so a failed launch
// or a sticky device error is reported instead of spinning forever.
qfs_status wait_published(qfs_ctx *c, unsigned long long seq) {
  for (unsigned it = 1;; ++it) {
    if (__atomic_load_n(c->h_pubflag, __ATOMIC_ACQUIRE) == seq) return QFS_OK;
    if ((it & 255u) == 0) {
      const cudaError_t e = cudaStreamQuery(c->st);
      if (e == cudaSuccess) {
        if (__atomic_load_n(c->h_pubflag, __ATOMIC_ACQUIRE) == seq) return QFS_OK;
        return fail(c, QFS_ERR_DEVICE, "sweep finished without publishing its results");
      }
      if (e != cudaErrorNotReady) return fail(c, QFS_ERR_DEVICE, cudaGetErrorString(e));
    }
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  }
}

// Run one sweep: upload the slot table, issue (graph-captured when not
// profiling and not tracing), and copy the per-start cost sums back.
qfs_status run_sweep(qfs_ctx *c, const SweepSpec &sp, std::vector<double> &csum,
                     std::vector<double> &cval) {
  const int ns = (int)sp.slots.size();
  // slot table through a mapped pinned buffer and a copy kernel (see upload_gates)
  if ((size_t)ns > c->h_slots_cap) {
    if (c->h_slots) cudaFreeHost(c->h_slots);
    c->h_slots = nullptr;
    c->h_slots_cap = 0;
    CUDA_TRY(c, cudaHostAlloc((void **)&c->h_slots, (size_t)std::max(ns, 64) * sizeof(Slot), cudaHostAllocMapped));
    c->h_slots_cap = (size_t)std::max(ns, 64);
    c->slots_on_dev = 0;
  }
  // (the previous table's reader, a copy kernel, finished before the previous
  // run_sweep returned: it ends with a stream synchronisation).  Unchanged
  // table (the same active starts and M as the last sweep): nothing to copy —
  // one launch less on the per-sweep host round trip of the short sweeps
  if (ns != c->slots_on_dev || std::memcmp(c->h_slots, sp.slots.data(), ns * sizeof(Slot)) != 0) {
    std::memcpy(c->h_slots, sp.slots.data(), ns * sizeof(Slot));
    c->slots_on_dev = 0;
    Slot *dh = nullptr;
    CUDA_TRY(c, cudaHostGetDevicePointer((void **)&dh, c->h_slots, 0));
    static_assert(sizeof(Slot) == 8, "Slot is copied as double2 halves");
    CUDA_TRY(c, launch_copy_bytes(c->d_slots, dh, ns * sizeof(Slot), c->st));
    c->launches++;
    c->slots_on_dev = ns;
  }
  if (c->d_dbg) {
    std::vector<unsigned long long> init((size_t)4 * c->K);
    for (int i = 0; i < c->K; ++i) { init[4 * i] = ~0ull; init[4 * i + 1] = init[4 * i + 2] = init[4 * i + 3] = 0; }
    CUDA_TRY(c, cudaMemcpy(c->d_dbg, init.data(), init.size() * 8, cudaMemcpyHostToDevice));
  }
  // CUDA graph for the streamed sweep (hundreds of launches); the resident
  // sweep is one launch, where a capture per new (slots, M) shape only costs
  // (C2 cold instantiate 30 -> 8 ms without it)
  ResPlan pl;
  const bool resident = !c->blocks && res_plan(c, sp.M_max, ns, pl);
  const bool use_graph = sp.env_trace == nullptr && !resident && !getenv("QFS_NO_GRAPH");
  if (use_graph) {
    long long key[8] = {ns, sp.M_max, sp.want_val + 2 * sp.want_sig, (long long)(sp.beta * 1e15), sp.S, c->S_cap,
                        c->M_cap, (c->prof ? 2 : 1)};
    if (!c->gexec || std::memcmp(key, c->gkey, sizeof key) != 0) {
      drop_graph(c);
      cudaGraph_t g;
      CUDA_TRY(c, cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
      long long before = c->launches;
      c->capturing = true;
      qfs_status s = issue_sweep(c, sp);
      c->capturing = false;
      cudaError_t e = cudaStreamEndCapture(c->st, &g);
      if (s != QFS_OK) return s;
      if (e != cudaSuccess) return fail(c, QFS_ERR_DEVICE, std::string("graph capture: ") + cudaGetErrorString(e));
      CUDA_TRY(c, cudaGraphInstantiate(&c->gexec, g, 0));
      cudaGraphDestroy(g);
      std::memcpy(c->gkey, key, sizeof key);
      c->glaunches = c->launches - before;
      c->launches = before;
    }
    CUDA_TRY(c, cudaGraphLaunch(c->gexec, c->st));
    c->res_sweeps++;
    c->launches += c->glaunches;
  } else {
    qfs_status s = issue_sweep(c, sp);
    if (s != QFS_OK) return s;
    c->res_sweeps++;
  }
  if (c->copy_defer && c->stg_count > 0) {  // queued sample sets: copy during this sweep's backward
    const qfs_status s = issue_deferred(c);
    if (s != QFS_OK) return s;
  }
  // csum [0, ns) and cval [S_cap, S_cap + ns) in one copy
  const size_t nrb = sp.want_val && c->V > 0 ? (size_t)c->S_cap + ns : (size_t)ns;
  const bool with_check = c->check_pending && !c->check_fetched;  // the gate-check flag rides along
  if (c->prof || c->d_dbg || c->pub_off) {
    // profiling / debug timing read events and buffers right after: a full synchronisation
    CUDA_TRY(c, cudaMemcpyAsync(c->h_csum, c->d_csum, nrb * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    if (with_check) CUDA_TRY(c, cudaMemcpyAsync(c->h_check, c->d_check, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  } else {
    // results published by a kernel into mapped pinned memory; the host spins on the sequence number
    if (!c->h_pubflag) {
      CUDA_TRY(c, cudaHostAlloc((void **)&c->h_pubflag, 64, cudaHostAllocMapped));
      *c->h_pubflag = c->pub_seq;
    }
    double *dh = nullptr;
    unsigned *dchk = nullptr;
    unsigned long long *dflag = nullptr;
    CUDA_TRY(c, cudaHostGetDevicePointer((void **)&dh, c->h_csum, 0));
    CUDA_TRY(c, cudaHostGetDevicePointer((void **)&dchk, c->h_check, 0));
    CUDA_TRY(c, cudaHostGetDevicePointer((void **)&dflag, c->h_pubflag, 0));
    const unsigned long long seq = ++c->pub_seq;
    CUDA_TRY(c, launch_publish(c->d_csum, (int)nrb, with_check ? c->d_check : nullptr, dh, dchk, dflag, seq, c->st));
    c->launches++;
    const qfs_status ws = wait_published(c, seq);
    if (ws != QFS_OK) return ws;
  }
  if (with_check) c->check_fetched = true;
  c->host_read_pending = false;  // the sweep's work, and the gate copy before it, has completed
  csum.assign(c->h_csum, c->h_csum + ns);
  if (sp.want_val && c->V > 0) cval.assign(c->h_cval, c->h_cval + ns);
  else cval.assign(ns, NAN);
  if (c->prof) {
    if (use_graph) prof_collect_graph(c);
    prof_collect(c);
  }
  if (c->d_dbg) {
    std::vector<unsigned long long> h((size_t)4 * c->K);
    CUDA_TRY(c, cudaMemcpy(h.data(), c->d_dbg, h.size() * 8, cudaMemcpyDeviceToHost));
    if (c->dbg_acc.empty()) c->dbg_acc.assign(3, 0.0);
    for (int i = 0; i < c->K; ++i) {
      c->dbg_acc[0] += (double)(h[4 * i + 1] - h[4 * i]);
      c->dbg_acc[1] += (double)(h[4 * i + 2] - h[4 * i + 1]);
      c->dbg_acc[2] += (double)(h[4 * i + 3] - h[4 * i + 2]);
      c->dbg_n++;
    }
  }
  return QFS_OK;
}

// The initial gates are validated on the device (gate_check_kernel: finite,
// unitary to 1e-10, one-qubit slots of the form u (x) I) into a device flag;
// gate_check_result reads it back after the first sweep's synchronisation
// (the caller gets QFS_ERR_NUMERIC instead of results; no host-side O(S K)
// pass on the critical path of every call).
qfs_status gate_check_result(qfs_ctx *c) {
  if (!c->check_pending) return QFS_OK;
  c->check_pending = false;
  if (!c->check_fetched) {
    CUDA_TRY(c, cudaMemcpyAsync(c->h_check, c->d_check, sizeof(unsigned), cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  }
  c->check_fetched = false;
  const unsigned bad = *c->h_check;
  if (bad & 16u) {
    c->have_samples = false;
    return fail(c, QFS_ERR_NUMERIC, "non-finite sample");
  }
  if (bad & 1u) return fail(c, QFS_ERR_NUMERIC, "non-finite initial gate");
  if (bad & 2u) return fail(c, QFS_ERR_NUMERIC, "initial gate not unitary (tol 1e-10)");
  if (bad & 4u) return fail(c, QFS_ERR_NUMERIC, "one-qubit gate slot is not of the form u (x) I (tol 1e-10)");
  if (bad & 8u) return fail(c, QFS_ERR_NUMERIC, "8x8 polar iteration did not converge (singular environment)");
  return QFS_OK;
}

// Device address of a page-locked, mapped host buffer (cudaHostAlloc /
// cudaHostRegister memory, e.g. torch pin_memory(); under unified addressing
// every such buffer is mapped) pinned for this context's device, or nullptr
// (pageable memory, or pinned under another device: staged as before).
const void *pinned_device_ptr(const void *host, int device) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost && a.device == device ? a.devicePointer : nullptr;
}

qfs_status upload_gates(qfs_ctx *c, int s, const double *init) {
  if (!c->h_check) {
    CUDA_TRY(c, cudaHostAlloc((void **)&c->h_check, sizeof(unsigned), cudaHostAllocMapped));
  }
  const size_t gb = (size_t)s * c->gsz * sizeof(double2);
  // a pinned caller buffer is read by the copy kernel in place (no host memcpy
  // into the context's staging buffer; the call is synchronous, so the buffer
  // is not reused before the kernel has read it)
  if (const void *dp = pinned_device_ptr(init, c->device)) {
    c->host_read_pending = true;
    CUDA_TRY(c, launch_copy(c->d_gates, (const double2 *)dp, (long long)s * c->gsz, c->st));
  } else {
  if (gb > c->h_gates_cap) {
    if (c->h_gates) cudaFreeHost(c->h_gates);
    c->h_gates = nullptr;
    c->h_gates_cap = 0;
    CUDA_TRY(c, cudaHostAlloc((void **)&c->h_gates, gb, cudaHostAllocMapped));
    c->h_gates_cap = gb;
  }
  std::memcpy(c->h_gates, init, gb);
  // read by a kernel from the mapped pinned buffer: small uploads never queue
  // on a copy engine behind a caller's large H2D (qfs_set_samples_async)
  double2 *dh = nullptr;
  CUDA_TRY(c, cudaHostGetDevicePointer((void **)&dh, c->h_gates, 0));
  CUDA_TRY(c, launch_copy(c->d_gates, dh, (long long)s * c->gsz, c->st));
  }
  {
    // device-side flag, read back (device -> host, 4 bytes) after the first sweep
    if (!c->d_check) CUDA_TRY(c, cudaMalloc(&c->d_check, sizeof(unsigned)));
    if (c->sample_check_pending)  // the queued sample set's finite check (set_samples_impl, deferred) as bit 4
      CUDA_TRY(c, launch_flag_bit((const unsigned *)c->d_flag, c->d_check, 16u, c->st));
    else
      CUDA_TRY(c, launch_fill_words(c->d_check, 0u, 1, c->st));
    c->sample_check_pending = false;
    if (c->blocks) CUDA_TRY(c, launch_blk_gate_check(c->d_gates, c->d_bg, c->K, c->gsz, s, c->d_check, c->st));
    else CUDA_TRY(c, launch_gate_check(c->d_gates, (long long)s * c->K, c->K, c->d_kinds, c->d_check, c->st));
    c->check_pending = true;
    c->check_fetched = false;
  }
  CUDA_TRY(c, launch_identity_fill(c->d_vprev, (long long)s * c->K, c->st));
  c->launches += 4;  // copy, flag fill, gate check, identity fill
  return QFS_OK;
}

// Emulated ranks (qfs_create_emulated; one start): the start's slots are the
// ranks 0..vr-1, each with its own pool block, states and gate copy.
void push_slots(const qfs_ctx *c, std::vector<Slot> &v, int q, int ml) {
  for (int r = 0; r < c->vr; ++r) v.push_back({q * c->vr + r, ml});
}
const double *replicate_init(const qfs_ctx *c, int s, const double *init, std::vector<double> &buf) {
  if (c->vr == 1) return init;
  const size_t g = (size_t)c->gsz * 2;
  buf.resize((size_t)s * c->vr * g);
  for (int q = 0; q < s; ++q)
    for (int r = 0; r < c->vr; ++r) std::memcpy(buf.data() + ((size_t)q * c->vr + r) * g, init + (size_t)q * g, g * sizeof(double));
  return buf.data();
}
// per-slot cost sums -> per-start: the ranks' training sums add up (each holds
// its own rows); every rank evaluates the full validation set, rank 0's is used
void fold_sums(const qfs_ctx *c, std::vector<double> &csum, std::vector<double> &cval) {
  if (c->vr == 1) return;
  const size_t ns = csum.size() / c->vr;
  for (size_t q = 0; q < ns; ++q) {
    double t = 0.0;
    for (int r = 0; r < c->vr; ++r) t += csum[q * c->vr + r];
    csum[q] = t;
    cval[q] = cval[q * c->vr];
  }
  csum.resize(ns);
  cval.resize(ns);
}

}  // namespace
qfs_status consume_staged(qfs_ctx *c);  // defined with the ABI below
namespace {
qfs_status check_ready(qfs_ctx *c, int s) {
  if (!c) return QFS_ERR_ARG;
  if (c->stg_count > 0) {
    const qfs_status st = consume_staged(c);
    if (st != QFS_OK) return st;
  }
  if (!c->have_samples) return fail(c, QFS_ERR_STATE, "set_samples has not been called");
  if (s < 1) return fail(c, QFS_ERR_ARG, "s must be >= 1");
  if (c->vr > 1 && s != 1) return fail(c, QFS_ERR_ARG, "emulated ranks: one start per call");
  CUDA_TRY(c, cudaSetDevice(c->device));
  return QFS_OK;
}

qfs_status create_common(int n, int k, const int32_t *pairs, int device, qfs_ctx **out) {
  if (!out) return QFS_ERR_ARG;
  *out = nullptr;
  if (n < 2 || n > 26 || k < 1 || !pairs) return QFS_ERR_ARG;
  for (int i = 0; i < k; ++i) {
    int a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a < 0 || b < 0 || a >= n || b >= n || a == b) return QFS_ERR_ARG;
  }
  qfs_ctx *c = new qfs_ctx();
  c->n = n; c->K = k; c->K_alloc = k; c->N = 1LL << n; c->device = device; c->gsz = 16LL * k;
  c->pairs.assign(pairs, pairs + 2 * k);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_pairs, k * sizeof(int2));
  if (e == cudaSuccess) e = cudaMemcpy(c->d_pairs, pairs, k * sizeof(int2), cudaMemcpyHostToDevice);
  c->kinds.assign(k, QFS_GATE_VAR2);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_kinds, k * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(c->d_kinds, 0, k * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&c->d_flag, 4 * sizeof(int));
  c->cur_st = c->st;
  if (const char *fc = getenv("QFS_FWD_CACHE")) c->fwd_cache_mode = atoi(fc);
  if (const char *fp = getenv("QFS_FWD_PAIRS")) c->fwd_pairs = atoi(fp) != 0;
  if (const char *pd = getenv("QFS_PDL")) set_pdl(atoi(pd) != 0);
  if (const char *pa = getenv("QFS_PATH")) c->path = std::max(0, std::min(2, atoi(pa)));
  if (const char *vb = getenv("QFS_VAL_BLOCK")) c->val_block = atoi(vb) != 0;
  if (const char *rc = getenv("QFS_RES_CMAX")) c->res_cmax = std::max(1, std::min(16, atoi(rc)));
  if (const char *rp = getenv("QFS_RES_PER_SM")) c->res_per_sm = atoi(rp) == 2 ? 2 : 1;
  if (const char *rq = getenv("QFS_RES_PAIR")) c->res_pair = std::max(0, std::min(2, atoi(rq)));
  if (const char *uf = getenv("QFS_UNFUSED_POLAR")) c->force_unfused = atoi(uf) != 0;
  if (const char *cd = getenv("QFS_COPY_DEFER")) c->copy_defer = atoi(cd) != 0;
  if (const char *pb = getenv("QFS_PUBLISH")) c->pub_off = atoi(pb) == 0;
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fwd, cudaEventDisableTiming);
  if (const char *bb = getenv("QFS_BWD_BULK")) c->bwd_bulk = atoi(bb) != 0;
  if (const char *bm = getenv("QFS_BULK_MIN_M")) c->bulk_min_m = std::max(1, atoi(bm));
  if (e != cudaSuccess) {
    c->err = std::string("device init: ") + cudaGetErrorString(e);
    *out = c;  // caller can read the error, then destroy
    return QFS_ERR_DEVICE;
  }
  if (getenv("QFS_TAIL_TIMING")) {
    cudaMalloc(&c->d_dbg, (size_t)4 * k * sizeof(unsigned long long));
    cudaMalloc(&c->d_res_dbg, 8 * sizeof(unsigned long long));
    cudaMemset(c->d_res_dbg, 0, 8 * sizeof(unsigned long long));
  }
  *out = c;
  return QFS_OK;
}

}  // namespace

// ======================================================================= ABI ==
extern "C" {

qfs_status qfs_create(int n, int k, const int32_t *pairs, int device, qfs_ctx **out) {
  return create_common(n, k, pairs, device, out);
}

qfs_status qfs_create_blocks(int n, int k, const int32_t *qubits, const int32_t *arity, int device,
                             qfs_ctx **out) {
  if (!out) return QFS_ERR_ARG;
  *out = nullptr;
  if (n < 3 || n > 26 || k < 1 || !qubits || !arity) return QFS_ERR_ARG;
  std::vector<int32_t> pairs(2 * (size_t)k);
  std::vector<BlkGate> bg(k);
  long long off = 0;
  bool any3 = false;
  for (int i = 0; i < k; ++i) {
    const int a = arity[i];
    if (a != 2 && a != 3) return QFS_ERR_ARG;
    for (int j = 0; j < a; ++j) {
      const int q = qubits[3 * i + j];
      if (q < 0 || q >= n) return QFS_ERR_ARG;
      for (int t = 0; t < j; ++t)
        if (qubits[3 * i + t] == q) return QFS_ERR_ARG;
    }
    bg[i].a = a;
    for (int j = 0; j < 3; ++j) bg[i].q[j] = j < a ? qubits[3 * i + j] : 0;
    bg[i].off = (int)off;
    bg[i].kind = QFS_GATE_VAR2;
    off += 1LL << (2 * a);
    any3 = any3 || a == 3;
    pairs[2 * i] = qubits[3 * i];
    pairs[2 * i + 1] = qubits[3 * i + 1];
  }
  qfs_status s = create_common(n, k, pairs.data(), device, out);
  if (s != QFS_OK || !any3) return s;  // all two-qubit: the pair circuit (same packed layout)
  qfs_ctx *c = *out;
  c->blocks = true;
  c->gsz = off;
  c->bgh = bg;
  CUDA_TRY(c, cudaMalloc(&c->d_bg, (size_t)k * sizeof(BlkGate)));
  CUDA_TRY(c, cudaMemcpy(c->d_bg, bg.data(), (size_t)k * sizeof(BlkGate), cudaMemcpyHostToDevice));
  return QFS_OK;
}

qfs_status qfs_create_dist(int n, int k, const int32_t *pairs, int device, void *nccl_comm,
                           int rank, int world, int shard_mode, qfs_ctx **out) {
  if (world < 1 || rank < 0 || rank >= world || (shard_mode != 0 && shard_mode != 1) ||
      (world > 1 && !nccl_comm))
    return QFS_ERR_ARG;
  qfs_status s = create_common(n, k, pairs, device, out);
  if (s != QFS_OK) return s;
  qfs_ctx *c = *out;
  c->comm = (ncclComm_t)nccl_comm;
  c->rank = rank; c->world = world; c->mode = shard_mode;
  if (c->comm) {
    int cr = -1, cn = -1;
    if (ncclCommUserRank(c->comm, &cr) != ncclSuccess || ncclCommCount(c->comm, &cn) != ncclSuccess ||
        cr != rank || cn != world)
      return fail(c, QFS_ERR_ARG, "nccl communicator rank/size mismatch");
  }
  return QFS_OK;
}

qfs_status qfs_create_emulated(int n, int k, const int32_t *pairs, int device, int ranks, qfs_ctx **out) {
  if (ranks < 2 || ranks > 32) return QFS_ERR_ARG;
  qfs_status s = create_common(n, k, pairs, device, out);
  if (s != QFS_OK) return s;
  qfs_ctx *c = *out;
  c->vr = ranks; c->mode = 1; c->world = ranks; c->rank = 0; c->xchg = 1;
  return QFS_OK;
}

qfs_status qfs_set_exchange(qfs_ctx *c, int mode) {
  if (!c) return QFS_ERR_ARG;
  if (mode != 0 && mode != 1) return fail(c, QFS_ERR_ARG, "exchange mode must be 0 (NCCL) or 1 (device)");
  if (c->vr > 1 && mode != 1) return fail(c, QFS_ERR_ARG, "emulated ranks exchange on the device only");
  if (c->blocks) return fail(c, QFS_ERR_ARG, "block circuits run single-GPU");
  if (mode == 1 && c->world > 32) return fail(c, QFS_ERR_ARG, "device exchange: at most 32 ranks");
  if (mode == 1 && c->mode == 1 && c->world > 1 && !c->comm && c->vr == 1)
    return fail(c, QFS_ERR_STATE, "device exchange needs the ranks' NCCL communicator");
  if (mode != c->xchg) {
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    xchg_release(c);
    c->xchg = mode;
    drop_graph(c);
  }
  return QFS_OK;
}

qfs_status qfs_nccl_unique_id(void *id128) {
  if (!id128) return QFS_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return QFS_ERR_DEVICE;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &id, sizeof id);
  return QFS_OK;
}

qfs_status qfs_create_nccl(int n, int k, const int32_t *pairs, int device, const void *id128,
                           int rank, int world, int shard_mode, qfs_ctx **out) {
  if (!id128 || world < 1 || rank < 0 || rank >= world || (shard_mode != 0 && shard_mode != 1))
    return QFS_ERR_ARG;
  qfs_status s = create_common(n, k, pairs, device, out);
  if (s != QFS_OK) return s;
  qfs_ctx *c = *out;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
  if (r != ncclSuccess) return fail(c, QFS_ERR_DEVICE, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  c->comm = comm;
  c->owns_comm = true;
  c->rank = rank; c->world = world; c->mode = shard_mode;
  return QFS_OK;
}

static qfs_status set_samples_impl(qfs_ctx *c, int m_pool, const void *x, const void *y, int v,
                                   const void *xv, const void *yv, cudaMemcpyKind kind,
                                   cudaStream_t ust, bool defer_check = false) {
  if (!c) return QFS_ERR_ARG;
  const bool basis = x == nullptr;  // qfs_set_samples_basis: x_m = e_m (computational basis), not stored
  if (m_pool < 1 || !y || v < 0 || (v > 0 && (!xv || !yv)))
    return fail(c, QFS_ERR_ARG, "bad sample arguments");
  if (basis && (c->mode == 1 || c->vr > 1 || c->blocks))
    return fail(c, QFS_ERR_ARG, "implicit basis inputs: single-rank pair contexts only");
  // emulated ranks (qfs_create_emulated): the caller passes ALL pool rows; rank
  // r keeps rows m = r (mod ranks) as its own [2^n][m_pool / ranks] block
  const int vr = c->vr;
  if (vr > 1 && m_pool % vr) return fail(c, QFS_ERR_CAPACITY, "emulated ranks: m_pool must be divisible by the ranks");
  const long long m_glob = vr > 1 ? m_pool : (long long)m_pool * (c->mode == 1 ? c->world : 1);
  if (m_glob > c->N) return fail(c, QFS_ERR_CAPACITY, "m_pool > 2^n");
  if (vr > 1) m_pool /= vr;  // rows per rank from here on
  if (!offsets_fit(c, std::max((long long)m_pool * vr, (long long)v)))
    return fail(c, QFS_ERR_CAPACITY, "2^n * rows * 16 B >= 4 GiB: beyond the 32-bit offsets of the streamed kernels");
  CUDA_TRY(c, cudaSetDevice(c->device));
  // the cached sweep graph holds the pool pointers: it is rebuilt only when a
  // buffer is reallocated (same shapes: the new contents are used in place).
  // Dropped BEFORE any buffer is freed, so an early return below (non-finite
  // sample, allocation failure) can never leave a graph over freed pools.
  const bool realloc = m_pool != c->m_pool || v != c->V || basis != c->x_basis;
  if (realloc) {
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    drop_graph(c);
  }
  if (m_pool != c->m_pool || basis != c->x_basis || (!basis && !c->d_x)) {
    dfree(c->d_x); dfree(c->d_y);
    if (!basis) CUDA_TRY(c, cudaMalloc(&c->d_x, (size_t)m_pool * vr * c->N * sizeof(double2)));
    CUDA_TRY(c, cudaMalloc(&c->d_y, (size_t)m_pool * vr * c->N * sizeof(double2)));
    c->m_pool = 0;
  }
  c->x_basis = basis;
  if (v != c->V) {
    dfree(c->d_xv); dfree(c->d_yv);
    if (v > 0) {
      CUDA_TRY(c, cudaMalloc(&c->d_xv, (size_t)v * c->N * sizeof(double2)));
      CUDA_TRY(c, cudaMalloc(&c->d_yv, (size_t)v * c->N * sizeof(double2)));
    }
  }
  cudaStream_t st = kind == cudaMemcpyHostToDevice ? c->st : ust;
  const size_t rb = (size_t)c->N * sizeof(double2);
  // stage the row-major pools, then transpose to the sample-minor layout
  if ((size_t)m_pool * rb > c->stage_bytes) {
    dfree(c->d_stage);
    CUDA_TRY(c, cudaMalloc(&c->d_stage, (size_t)m_pool * rb));
    c->stage_bytes = (size_t)m_pool * rb;
  }
  CUDA_TRY(c, launch_fill_words((unsigned *)c->d_flag, 0u, 1, st));  // a kernel, not a copy-engine memset
  // device sources (qfs_set_samples_device, queued async sets) are read in place
  // by kernels: no copy-engine work that could queue behind a concurrent H2D
  const bool dev = kind == cudaMemcpyDeviceToDevice;
  for (int q = basis ? 1 : 0; q < 2; ++q) {
    const double2 *src0 = (const double2 *)(q == 0 ? x : y);
    for (int r = 0; r < vr; ++r) {
      const double2 *src = src0;
      if (vr > 1) {  // rank r's rows r, r + vr, ... gathered into the stage
        CUDA_TRY(c, cudaMemcpy2DAsync(c->d_stage, rb, src0 + (long long)r * c->N, vr * rb, rb, m_pool, kind, st));
        src = c->d_stage;
      } else if (!dev) {
        CUDA_TRY(c, cudaMemcpyAsync(c->d_stage, src, m_pool * rb, kind, st));
        src = c->d_stage;
      }
      CUDA_TRY(c, launch_finite_check((const double *)src, (long long)m_pool * c->N * 2, c->d_flag, st));
      CUDA_TRY(c, launch_transpose(src, (q == 0 ? c->d_x : c->d_y) + (long long)r * m_pool * c->N, m_pool, c->N,
                                   st));
    }
  }
  if (v > 0) {
    if (dev) {
      CUDA_TRY(c, launch_copy(c->d_xv, (const double2 *)xv, (long long)v * c->N, st));
      CUDA_TRY(c, launch_copy(c->d_yv, (const double2 *)yv, (long long)v * c->N, st));
    } else {
      CUDA_TRY(c, cudaMemcpyAsync(c->d_xv, xv, v * rb, kind, st));
      CUDA_TRY(c, cudaMemcpyAsync(c->d_yv, yv, v * rb, kind, st));
    }
    CUDA_TRY(c, launch_finite_check((const double *)c->d_xv, (long long)v * c->N * 2, c->d_flag, st));
    CUDA_TRY(c, launch_finite_check((const double *)c->d_yv, (long long)v * c->N * 2, c->d_flag, st));
  }
  int bad = 0;
  // a queued set consumed by qfs_instantiate (defer_check; single-rank contexts):
  // no host round trip here — the flag travels with the initial-gate check,
  // read back after the first sweep (QFS_ERR_NUMERIC "non-finite sample")
  const bool defer = defer_check && !(c->mode == 1 && c->world > 1 && c->comm);
  if (!defer) {
    CUDA_TRY(c, cudaMemcpyAsync(&bad, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
  }
  c->sample_check_pending = defer;
  c->launches += v > 0 ? 6 : 4;
  c->m_pool = m_pool; c->V = v; c->have_samples = true;
  if (bad) {
    c->have_samples = false;
    return fail(c, QFS_ERR_NUMERIC, "non-finite sample");
  }
  // validation rows over all ranks (sample mode: each rank holds its own
  // validation shard; c_val = (sum over ranks) / V_glob, R11)
  c->V_glob = v;
  if (c->mode == 1 && c->world > 1 && c->comm) {
    // every rank must hold the same number of validation rows (each its own
    // shard): the per-sweep validation all-reduce is then issued by all ranks
    int h[2] = {v, -v};
    CUDA_TRY(c, cudaMemcpyAsync(c->d_flag + 2, h, sizeof h, cudaMemcpyHostToDevice, c->st));
    NCCL_TRY(c, ncclAllReduce(c->d_flag + 2, c->d_flag + 2, 2, ncclInt32, ncclMax, c->comm, c->st));
    CUDA_TRY(c, cudaMemcpyAsync(h, c->d_flag + 2, sizeof h, cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    if (h[0] != -h[1]) {
      c->have_samples = false;
      return fail(c, QFS_ERR_ARG, "sample mode: every rank must pass the same number of validation rows");
    }
    c->V_glob = v * c->world;
  }
  return QFS_OK;
}

// Oldest queued sample set -> the pools (device-to-device through the same
// staging, finite check and transpose as qfs_set_samples), after its H2D copy.
}  // extern "C" (internal helpers below have C++ linkage)
// Enqueue a staged set's H2D copies on the copy stream (after `after`, if given).
qfs_status issue_staged(qfs_ctx *c, qfs_ctx::Staged &g, cudaEvent_t after) {
  if (g.issued) return QFS_OK;
  if (after) CUDA_TRY(c, cudaStreamWaitEvent(c->st_copy, after, 0));
  const size_t bxy = (size_t)g.m_pool * c->N * sizeof(double2), bv = (size_t)g.v * c->N * sizeof(double2);
  CUDA_TRY(c, cudaMemcpyAsync(g.x, g.hx, bxy, cudaMemcpyHostToDevice, c->st_copy));
  CUDA_TRY(c, cudaMemcpyAsync(g.y, g.hy, bxy, cudaMemcpyHostToDevice, c->st_copy));
  if (g.v > 0) {
    CUDA_TRY(c, cudaMemcpyAsync(g.xv, g.hxv, bv, cudaMemcpyHostToDevice, c->st_copy));
    CUDA_TRY(c, cudaMemcpyAsync(g.yv, g.hyv, bv, cudaMemcpyHostToDevice, c->st_copy));
  }
  CUDA_TRY(c, cudaEventRecord(g.ev, c->st_copy));
  g.issued = true;
  return QFS_OK;
}
// After a sweep's graph is enqueued: start the copies of the queued sets not
// yet consumed, behind the sweep's forward phase (QFS_COPY_DEFER).
qfs_status issue_deferred(qfs_ctx *c) {
  for (int q = 0; q < c->stg_count; ++q) {
    qfs_ctx::Staged &g = c->stg[(c->stg_head + q) % 2];
    if (!g.issued) {
      const qfs_status st = issue_staged(c, g, c->ev_fwd);
      if (st != QFS_OK) return st;
    }
  }
  return QFS_OK;
}
qfs_status consume_staged(qfs_ctx *c) {
  qfs_ctx::Staged &g = c->stg[c->stg_head];
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!g.issued) {
    const qfs_status st = issue_staged(c, g, nullptr);  // nothing ran since it was queued
    if (st != QFS_OK) return st;
  }
  CUDA_TRY(c, cudaStreamWaitEvent(c->st, g.ev, 0));
  const qfs_status st =
      set_samples_impl(c, g.m_pool, g.x, g.y, g.v, g.xv, g.yv, cudaMemcpyDeviceToDevice, c->st, true);
  c->stg_head = (c->stg_head + 1) % 2;
  c->stg_count -= 1;
  return st;
}
extern "C" {

qfs_status qfs_set_samples_async(qfs_ctx *c, int m_pool, const double *x, const double *y, int v,
                                 const double *xv, const double *yv) {
  if (!c) return QFS_ERR_ARG;
  if (m_pool < 1 || !x || !y || v < 0 || (v > 0 && (!xv || !yv)))
    return fail(c, QFS_ERR_ARG, "bad sample arguments");
  if ((long long)m_pool * (c->vr > 1 ? 1 : c->mode == 1 ? c->world : 1) > c->N)
    return fail(c, QFS_ERR_CAPACITY, "m_pool > 2^n");
  if (c->stg_count == 2) return fail(c, QFS_ERR_STATE, "two sample sets are already queued");
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (!c->st_copy) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->st_copy, cudaStreamNonBlocking));
  qfs_ctx::Staged &g = c->stg[(c->stg_head + c->stg_count) % 2];
  const size_t bxy = (size_t)m_pool * c->N * sizeof(double2), bv = (size_t)v * c->N * sizeof(double2);
  // both staging slots are sized together: cudaMalloc / cudaFree synchronise,
  // so a first-time allocation of the second slot must not land mid-pipeline
  for (qfs_ctx::Staged &h : c->stg) {
    if (!h.ev) CUDA_TRY(c, cudaEventCreateWithFlags(&h.ev, cudaEventDisableTiming));
    if (bxy > h.cap_xy) {
      if (&h != &g && c->stg_count > 0) continue;  // a queued set still lives there
      dfree(h.x); dfree(h.y);
      CUDA_TRY(c, cudaMalloc(&h.x, bxy));
      CUDA_TRY(c, cudaMalloc(&h.y, bxy));
      h.cap_xy = bxy;
    }
    if (bv > h.cap_v) {
      if (&h != &g && c->stg_count > 0) continue;
      dfree(h.xv); dfree(h.yv);
      CUDA_TRY(c, cudaMalloc(&h.xv, bv));
      CUDA_TRY(c, cudaMalloc(&h.yv, bv));
      h.cap_v = bv;
    }
  }
  g.hx = x; g.hy = y; g.hxv = xv; g.hyv = yv;
  g.m_pool = m_pool;
  g.v = v;
  g.issued = false;
  c->stg_count += 1;
  if (!c->copy_defer) return issue_staged(c, g, nullptr);
  return QFS_OK;
}

qfs_status qfs_set_samples(qfs_ctx *c, int m_pool, const double *x, const double *y, int v,
                           const double *xv, const double *yv) {
  if (c && !x) return fail(c, QFS_ERR_ARG, "bad sample arguments");
  return set_samples_impl(c, m_pool, x, y, v, xv, yv, cudaMemcpyHostToDevice, nullptr);
}

qfs_status qfs_set_samples_basis(qfs_ctx *c, int m_pool, const double *y, int v, const double *xv,
                                 const double *yv) {
  if (!c) return QFS_ERR_ARG;
  if (!y) return fail(c, QFS_ERR_ARG, "bad sample arguments");
  return set_samples_impl(c, m_pool, nullptr, y, v, xv, yv, cudaMemcpyHostToDevice, nullptr);
}

qfs_status qfs_set_samples_device(qfs_ctx *c, int m_pool, const void *dx, const void *dy, int v,
                                  const void *dxv, const void *dyv, void *cuda_stream) {
  if (c && !dx) return fail(c, QFS_ERR_ARG, "bad sample arguments");
  return set_samples_impl(c, m_pool, dx, dy, v, dxv, dyv, cudaMemcpyDeviceToDevice,
                          (cudaStream_t)cuda_stream);
}

qfs_status qfs_trace_sweeps(qfs_ctx *c, int s, const double *init_gates, int m, double beta,
                            int n_sweeps, double *env_trace, double *gate_trace,
                            double *cost_trace, double *sigma_trace) {
  qfs_status st = check_ready(c, s);
  if (st != QFS_OK) return st;
  if (!init_gates || n_sweeps < 0) return fail(c, QFS_ERR_ARG, "bad trace arguments");
  const int wm = c->mode == 1 ? c->world : 1;
  if (m < 1 || m % wm != 0) return fail(c, QFS_ERR_CAPACITY, "M must be >= 1 and divisible by world");
  const int ml = m / wm;
  if (ml > c->m_pool) return fail(c, QFS_ERR_CAPACITY, "M exceeds the pool");
  const int se = s * c->vr;  // slots (emulated ranks: one per rank)
  std::vector<double> rep;
  if ((st = ensure_gates(c, se)) != QFS_OK) return st;
  if ((st = ensure_state(c, se, ml, c->V)) != QFS_OK) return st;
  if ((st = ensure_xchg(c, s)) != QFS_OK) return st;
  if ((st = upload_gates(c, se, replicate_init(c, s, init_gates, rep))) != QFS_OK) return st;
  const size_t tr = (size_t)se * c->gsz;  // gate-major: gate i of start q at s * off_i + q * d_i^2
  if (env_trace && tr > c->env_trace_cap) {
    dfree(c->d_env_trace);
    CUDA_TRY(c, cudaMalloc(&c->d_env_trace, tr * sizeof(double2)));
    c->env_trace_cap = tr;
  }
  SweepSpec sp;
  for (int q = 0; q < s; ++q) push_slots(c, sp.slots, q, ml);
  sp.M_max = ml; sp.want_val = false; sp.beta = beta; sp.S = se; sp.want_sig = sigma_trace != nullptr;
  sp.env_trace = env_trace ? c->d_env_trace : nullptr;
  std::vector<double> csum, cval, hbuf;
  const int vr = c->vr;
  for (int t = 0; t < n_sweeps; ++t) {
    if ((st = run_sweep(c, sp, csum, cval)) != QFS_OK) return st;
    if ((st = gate_check_result(c)) != QFS_OK) return st;
    fold_sums(c, csum, cval);
    if (env_trace) {
      double *dst = env_trace + (size_t)t * s * c->gsz * 2;
      if (vr == 1) {
        CUDA_TRY(c, cudaMemcpy(dst, c->d_env_trace, tr * sizeof(double2), cudaMemcpyDeviceToHost));
      } else {  // [K][s vr][16] -> rank 0's [K][s][16] (pair circuits)
        hbuf.resize(tr * 2);
        CUDA_TRY(c, cudaMemcpy(hbuf.data(), c->d_env_trace, tr * sizeof(double2), cudaMemcpyDeviceToHost));
        for (int i = 0; i < c->K; ++i)
          for (int q = 0; q < s; ++q)
            std::memcpy(dst + ((size_t)i * s + q) * 32, hbuf.data() + ((size_t)i * se + q * vr) * 32, 32 * sizeof(double));
      }
    }
    if (gate_trace)
      for (int q = 0; q < s; ++q)
        CUDA_TRY(c, cudaMemcpy(gate_trace + ((size_t)t * s + q) * c->gsz * 2, c->d_gates + (size_t)q * vr * c->gsz,
                               (size_t)c->gsz * sizeof(double2), cudaMemcpyDeviceToHost));
    if (cost_trace)
      for (int q = 0; q < s; ++q) cost_trace[(size_t)t * s + q] = csum[q] / m;
    if (sigma_trace) {
      std::vector<double> sg((size_t)se * c->K);
      CUDA_TRY(c, cudaMemcpy(sg.data(), c->d_sig, sg.size() * sizeof(double), cudaMemcpyDeviceToHost));
      for (int i = 0; i < c->K; ++i)
        for (int q = 0; q < s; ++q) sigma_trace[((size_t)t * c->K + i) * s + q] = sg[(size_t)q * vr * c->K + i];
    }
  }
  return gate_check_result(c);  // n_sweeps == 0: still report invalid gates
}

qfs_status qfs_bench_sweeps(qfs_ctx *c, int s, const double *init_gates, int m, int n_sweeps,
                            double *sec) {
  qfs_status st = check_ready(c, s);
  if (st != QFS_OK) return st;
  const int wm = c->mode == 1 ? c->world : 1;
  if (!init_gates || n_sweeps < 1 || m < 1 || m % wm || m / wm > c->m_pool)
    return fail(c, QFS_ERR_ARG, "bad bench arguments");
  const int ml = m / wm;
  const int se = s * c->vr;
  std::vector<double> rep;
  if ((st = ensure_gates(c, se)) != QFS_OK) return st;
  if ((st = ensure_state(c, se, ml, c->V)) != QFS_OK) return st;
  if ((st = ensure_xchg(c, s)) != QFS_OK) return st;
  if ((st = upload_gates(c, se, replicate_init(c, s, init_gates, rep))) != QFS_OK) return st;
  SweepSpec sp;
  for (int q = 0; q < s; ++q) push_slots(c, sp.slots, q, ml);
  sp.M_max = ml; sp.S = se;
  std::vector<double> csum, cval;
  cudaEvent_t e0, e1;
  CUDA_TRY(c, cudaEventCreate(&e0));
  CUDA_TRY(c, cudaEventCreate(&e1));
  CUDA_TRY(c, cudaEventRecord(e0, c->st));
  for (int t = 0; t < n_sweeps; ++t) {
    if ((st = run_sweep(c, sp, csum, cval)) != QFS_OK) return st;
    if ((st = gate_check_result(c)) != QFS_OK) return st;
  }
  CUDA_TRY(c, cudaEventRecord(e1, c->st));
  CUDA_TRY(c, cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (sec) *sec = ms * 1e-3;
  return gate_check_result(c);
}

// Controller (readings R7-R14, R16).
qfs_status qfs_instantiate(qfs_ctx *c, int s, const double *init_gates, const qfs_params *p,
                           double *out_gates, qfs_result *out, int *winner) {
  qfs_status st = check_ready(c, s);
  if (st != QFS_OK) return st;
  if (!init_gates || !p || !out_gates || !out) return fail(c, QFS_ERR_ARG, "null argument");
  const int wm = c->mode == 1 ? c->world : 1;
  const long long Nfull = c->N;
  const int pool_g = c->m_pool * wm;  // global pool rows
  if (p->m_init < 1 || p->m_init > pool_g) return fail(c, QFS_ERR_CAPACITY, "m_init > m_pool");
  if (p->m_init % wm) return fail(c, QFS_ERR_CAPACITY, "m_init not divisible by world");
  if (p->max_iter < 1) return fail(c, QFS_ERR_ARG, "max_iter < 1");
  const int se = s * c->vr;  // slots (emulated ranks: one per rank)
  std::vector<double> rep;
  if ((st = ensure_gates(c, se)) != QFS_OK) return st;
  if ((st = ensure_xchg(c, s)) != QFS_OK) return st;
  if ((st = upload_gates(c, se, replicate_init(c, s, init_gates, rep))) != QFS_OK) return st;
  struct S_ {
    int M, it, total, fails, restarts, term, conv_sweep;
    bool has_prev, active;
    double c_prev, c_train, c_val;
  };
  std::vector<S_> A(s);
  for (auto &a : A) {
    a.M = p->m_init; a.it = a.total = a.fails = a.restarts = 0; a.term = -1; a.conv_sweep = -1;
    a.has_prev = false; a.active = true; a.c_prev = 0; a.c_train = NAN; a.c_val = NAN;
  }
  const double otr = p->overtrain_ratio;
  const bool multi_rank = c->world > 1 && c->comm && c->mode == 0;
  std::vector<double> csum, cval;
  for (int t = 1;; ++t) {
    SweepSpec sp;
    sp.S = se; sp.beta = p->beta;
    std::vector<int> act;  // active starts, in slot order
    for (int q = 0; q < s; ++q)
      if (A[q].active) {
        push_slots(c, sp.slots, q, A[q].M / wm);
        act.push_back(q);
        sp.M_max = std::max(sp.M_max, A[q].M / wm);
      }
    sp.want_val = c->V > 0;
    bool any_conv = false, any_active = false;
    if (!sp.slots.empty()) {
      if ((st = ensure_state(c, se, sp.M_max, c->V)) != QFS_OK) return st;
      if ((st = run_sweep(c, sp, csum, cval)) != QFS_OK) return st;
      if ((st = gate_check_result(c)) != QFS_OK) return st;
      fold_sums(c, csum, cval);
      for (size_t j = 0; j < act.size(); ++j) {
        S_ &a = A[act[j]];
        a.c_train = csum[j] / a.M;
        a.c_val = c->V_glob > 0 ? cval[j] / c->V_glob : NAN;
        a.it += 1; a.total += 1;                                               // step 1
        const double cc = a.c_train;
        const bool gen_check = c->V_glob > 0 && std::isfinite(otr) && a.M < Nfull;  // step 2
        bool conv = false;                                                     // step 3
        if (cc <= p->dist_tol) {
          if (!gen_check) conv = true;
          else if (cc < 1e-14) conv = a.c_val <= (1.0 + otr) * p->dist_tol;
          else conv = a.c_val / cc - 1.0 <= otr;
        }
        if (conv) { a.term = QFS_CONVERGED; a.active = false; a.conv_sweep = t; any_conv = true; continue; }
        if (gen_check && a.it >= p->min_iter && a.c_val / cc - 1.0 > otr) {    // step 4
          if (2LL * a.M > pool_g && a.M < Nfull) { a.term = QFS_POOL_EXHAUSTED; a.active = false; continue; }
          a.M = (int)std::min<long long>(2LL * a.M, Nfull);
          a.it = 0; a.fails = 0; a.has_prev = false; a.restarts += 1;
        } else if (p->plateau_window > 0) {                                    // step 5
          if (a.has_prev)
            a.fails = (std::fabs(a.c_prev) - std::fabs(cc) > p->diff_tol_r * std::fabs(cc)) ? 0 : a.fails + 1;
          a.c_prev = cc; a.has_prev = true;
          if (a.it >= p->min_iter && a.fails >= p->plateau_window) { a.term = QFS_PLATEAU; a.active = false; continue; }
        }
        if (a.total >= p->max_iter) { a.term = QFS_MAX_ITER; a.active = false; }  // step 6
      }
    }
    for (auto &a : A) any_active |= a.active;
    if (multi_rank) {  // "any converged" / "any active" across ranks
      int h[2] = {any_conv ? 1 : 0, any_active ? 1 : 0};
      CUDA_TRY(c, cudaMemcpyAsync(c->d_flag, h, sizeof h, cudaMemcpyHostToDevice, c->st));
      NCCL_TRY(c, ncclAllReduce(c->d_flag, c->d_flag, 2, ncclInt32, ncclMax, c->comm, c->st));
      CUDA_TRY(c, cudaMemcpyAsync(h, c->d_flag, sizeof h, cudaMemcpyDeviceToHost, c->st));
      CUDA_TRY(c, cudaStreamSynchronize(c->st));
      any_conv = h[0] != 0;
      any_active = h[1] != 0;
    }
    if (any_conv && p->stop_on_first) {
      for (auto &a : A)
        if (a.active) { a.active = false; a.term = QFS_STOPPED; }
      break;
    }
    if (!any_active) break;
  }
  int win = -1, best = 1 << 30;
  for (int q = 0; q < s; ++q)
    if (A[q].term == QFS_CONVERGED && A[q].conv_sweep < best) { best = A[q].conv_sweep; win = q; }
  if (win < 0) {
    double bc = INFINITY;
    for (int q = 0; q < s; ++q)
      if (A[q].c_train < bc) { bc = A[q].c_train; win = q; }
    if (win < 0) win = 0;
  }
  if (c->vr == 1 && pinned_device_ptr(out_gates, c->device)) {  // pinned caller buffer: one DMA straight into it
    CUDA_TRY(c, cudaMemcpyAsync(out_gates, c->d_gates, (size_t)s * c->gsz * sizeof(double2), cudaMemcpyDeviceToHost,
                                c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
  } else {
    if ((size_t)se * c->gsz * sizeof(double2) > c->h_gates_cap) {  // (only the pinned-input path ran so far)
      if (c->h_gates) cudaFreeHost(c->h_gates);
      c->h_gates = nullptr;
      c->h_gates_cap = 0;
      CUDA_TRY(c, cudaHostAlloc((void **)&c->h_gates, (size_t)se * c->gsz * sizeof(double2), cudaHostAllocMapped));
      c->h_gates_cap = (size_t)se * c->gsz * sizeof(double2);
    }
    CUDA_TRY(c, cudaMemcpyAsync(c->h_gates, c->d_gates, (size_t)se * c->gsz * sizeof(double2),
                                cudaMemcpyDeviceToHost, c->st));
    CUDA_TRY(c, cudaStreamSynchronize(c->st));
    for (int q = 0; q < s; ++q)  // (emulated ranks: rank 0's copy; all ranks hold identical bits)
      std::memcpy(out_gates + (size_t)q * c->gsz * 2, c->h_gates + (size_t)q * c->vr * c->gsz,
                  (size_t)c->gsz * sizeof(double2));
  }
  for (int q = 0; q < s; ++q) {
    out[q].c_train = A[q].c_train; out[q].c_val = A[q].c_val; out[q].sweeps = A[q].total;
    out[q].restarts = A[q].restarts; out[q].final_m = A[q].M; out[q].term = (qfs_term)A[q].term;
  }
  if (winner) *winner = win;
  return QFS_OK;
}

qfs_status qfs_op_apply(qfs_ctx *c, int p0, int p1, const double *g, int dagger, int m,
                        double *psi) {
  if (!c || !g || !psi || m < 1 || p0 < 0 || p1 < 0 || p0 >= c->n || p1 >= c->n || p0 == p1)
    return fail(c, QFS_ERR_ARG, "bad apply arguments");
  CUDA_TRY(c, cudaSetDevice(c->device));
  ApplyParams a{};
  a.n = c->n; a.p0 = p0; a.p1 = p1; a.m = m;
  for (int r = 0; r < 4; ++r)
    for (int q = 0; q < 4; ++q) {
      const double *e = dagger ? g + 2 * (4 * q + r) : g + 2 * (4 * r + q);
      a.g[4 * r + q] = make_double2(e[0], dagger ? -e[1] : e[1]);
    }
  double2 *d = nullptr;
  const size_t bytes = (size_t)m * c->N * sizeof(double2);
  CUDA_TRY(c, cudaMalloc(&d, bytes));
  a.psi = d;
  cudaError_t e = cudaMemcpy(d, psi, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    c->cur_st = c->st;
    LaunchScope ls(c, K_OP, 2.0 * bytes, 32.0 * m * c->N);
    e = launch_apply(a, c->st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e == cudaSuccess) e = cudaMemcpy(psi, d, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(c, QFS_ERR_DEVICE, cudaGetErrorString(e));
  return QFS_OK;
}

qfs_status qfs_op_environment(qfs_ctx *c, int p0, int p1, int m, const double *phi,
                              const double *chi, double *env) {
  if (!c || !phi || !chi || !env || m < 1 || p0 < 0 || p1 < 0 || p0 >= c->n || p1 >= c->n || p0 == p1)
    return fail(c, QFS_ERR_ARG, "bad environment arguments");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t bytes = (size_t)m * c->N * sizeof(double2);
  double2 *dphi = nullptr, *dchi = nullptr;
  double *dpart = nullptr, *dred = nullptr;
  unsigned *dcnt = nullptr;
  Slot *dsl = nullptr;
  BwdParams b{};
  b.n = c->n; b.K = 1;
  b.nb = blocks_per_start((c->N >> 2) * ((m + 31) / 32) * 32, 1, 2);
  cudaError_t e = cudaMalloc(&dphi, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&dchi, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&dpart, (size_t)b.nb * 32 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dred, 32 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&dcnt, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMalloc(&dsl, sizeof(Slot));
  Slot sl{0, m};
  // the backward kernel reads sample-minor views: transpose [m][2^n] -> [2^n][m]
  double2 *dtmp = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&dtmp, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(dtmp, phi, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_transpose(dtmp, dphi, m, c->N, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e == cudaSuccess) e = cudaMemcpy(dtmp, chi, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_transpose(dtmp, dchi, m, c->N, c->st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (dtmp) cudaFree(dtmp);
  if (e == cudaSuccess) e = cudaMemset(dcnt, 0, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemcpy(dsl, &sl, sizeof sl, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    b.slots = dsl; b.g.chi_src = View{dchi, 0, m, 1}; b.g.chi_dst = ViewW{nullptr, 0, 0, 0};
    b.g.phi = View{dphi, 0, m, 1};
    int lo = std::min(p0, p1), hi = std::max(p0, p1);
    b.g.nu = 2; b.g.tp0 = 0; b.g.tp1 = 1; b.g.upd = 0;
    b.g.ins[0] = lo; b.g.ins[1] = hi;
    for (int v = 0; v < 16; ++v)
      b.g.off[v] = v < 4 ? (((long long)(v & 1) << p0) | ((long long)((v >> 1) & 1) << p1)) : 0;
    b.partials = dpart; b.counters = dcnt; b.e_red = dred; b.fuse_polar = 0; b.g.env_gate = 0;
    b.g.upd_gate = -1; b.S = 1;
    c->cur_st = c->st;
    LaunchScope ls(c, K_OP, 2.0 * bytes, 32.0 * m * c->N);
    e = launch_bwd(b, 1, c->st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e == cudaSuccess) e = cudaMemcpy(env, dred, 32 * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(dphi); cudaFree(dchi); cudaFree(dpart); cudaFree(dred); cudaFree(dcnt); cudaFree(dsl);
  if (e != cudaSuccess) return fail(c, QFS_ERR_DEVICE, cudaGetErrorString(e));
  return QFS_OK;
}

qfs_status qfs_op_polar(qfs_ctx *c, int count, const double *env, const double *g_old,
                        double beta, double *g_new, double *sigma_sum) {
  if (!c || count < 1 || !env || !g_old || !g_new || !sigma_sum)
    return fail(c, QFS_ERR_ARG, "bad polar arguments");
  CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t mb = (size_t)count * 16 * sizeof(double2);
  double2 *de = nullptr, *dg = nullptr, *dn = nullptr;
  double *ds = nullptr;
  cudaError_t e = cudaMalloc(&de, mb);
  if (e == cudaSuccess) e = cudaMalloc(&dg, mb);
  if (e == cudaSuccess) e = cudaMalloc(&dn, mb);
  if (e == cudaSuccess) e = cudaMalloc(&ds, count * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(de, env, mb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dg, g_old, mb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    c->cur_st = c->st;
    LaunchScope ls(c, K_OP, 3.0 * mb, 0);
    e = launch_polar_batch(de, dg, beta, dn, ds, count, c->st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
  if (e == cudaSuccess) e = cudaMemcpy(g_new, dn, mb, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(sigma_sum, ds, count * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(de); cudaFree(dg); cudaFree(dn); cudaFree(ds);
  if (e != cudaSuccess) return fail(c, QFS_ERR_DEVICE, cudaGetErrorString(e));
  return QFS_OK;
}

qfs_status qfs_profile_enable(qfs_ctx *c, int on) {
  if (!c) return QFS_ERR_ARG;
  prof_collect(c);
  c->prof = on != 0;
  if (on) {
    for (int q = 0; q < K_NCLASS; ++q) { c->p_ms[q] = c->p_bytes[q] = c->p_flops[q] = 0; c->p_cnt[q] = 0; }
  }
  return QFS_OK;
}

qfs_status qfs_profile_read(qfs_ctx *c, int cap, const char **names, long long *launches,
                            double *ms, double *bytes, double *flops, int *count) {
  if (!c) return QFS_ERR_ARG;
  prof_collect(c);
  for (int q = 0; q < K_NCLASS && q < cap; ++q) {
    if (names) names[q] = kClassName[q];
    if (launches) launches[q] = c->p_cnt[q];
    if (ms) ms[q] = c->p_ms[q];
    if (bytes) bytes[q] = c->p_bytes[q];
    if (flops) flops[q] = c->p_flops[q];
  }
  if (count) *count = K_NCLASS;
  return QFS_OK;
}

long long qfs_launch_count(const qfs_ctx *c) { return c ? c->launches : 0; }

qfs_status qfs_set_gate_kinds(qfs_ctx *c, const int32_t *kinds) {
  if (!c) return QFS_ERR_ARG;
  std::vector<int32_t> k(c->K, QFS_GATE_VAR2);
  if (kinds)
    for (int i = 0; i < c->K; ++i) {
      if (kinds[i] < QFS_GATE_VAR2 || kinds[i] > QFS_GATE_VAR1)
        return fail(c, QFS_ERR_ARG, "gate kind must be 0 (two-qubit variable), 1 (fixed) or 2 (one-qubit variable)");
      if (c->blocks && kinds[i] == QFS_GATE_VAR1 && c->bgh[i].a != 2)
        return fail(c, QFS_ERR_ARG, "one-qubit variable slots must be two-qubit blocks");
      k[i] = kinds[i];
    }
  if (c->blocks) {
    for (int i = 0; i < c->K; ++i) c->bgh[i].kind = k[i];
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemcpy(c->d_bg, c->bgh.data(), (size_t)c->K * sizeof(BlkGate), cudaMemcpyHostToDevice));
    drop_graph(c);
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy(c->d_kinds, k.data(), k.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  c->kinds.swap(k);
  return QFS_OK;
}

qfs_status qfs_set_structure(qfs_ctx *c, int k, const int32_t *pairs) {
  if (!c) return QFS_ERR_ARG;
  if (c->blocks) return fail(c, QFS_ERR_ARG, "qfs_set_structure: not available for block circuits");
  if (k < 1 || !pairs) return fail(c, QFS_ERR_ARG, "bad structure");
  for (int i = 0; i < k; ++i) {
    const int a = pairs[2 * i], b = pairs[2 * i + 1];
    if (a < 0 || b < 0 || a >= c->n || b >= c->n || a == b) return fail(c, QFS_ERR_ARG, "bad qubit pair");
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaStreamSynchronize(c->st));  // no launch of the old structure is in flight
  if (k > c->K_alloc) {
    // structure-dependent buffers are re-planned by the next call (gates, B cache, sigma)
    dfree(c->d_pairs);
    dfree(c->d_kinds);
    CUDA_TRY(c, cudaMalloc(&c->d_pairs, (size_t)k * sizeof(int2)));
    CUDA_TRY(c, cudaMalloc(&c->d_kinds, (size_t)k * sizeof(int)));
    if (c->d_dbg) {
      dfree(c->d_dbg);
      CUDA_TRY(c, cudaMalloc(&c->d_dbg, (size_t)4 * k * sizeof(unsigned long long)));
    }
    c->K_alloc = k;  // gates / B cache / sigma: ensure_gates / ensure_state compare K with K_g / K_s
  }
  CUDA_TRY(c, cudaMemcpy(c->d_pairs, pairs, (size_t)k * sizeof(int2), cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemset(c->d_kinds, 0, (size_t)k * sizeof(int)));
  c->K = k;
  c->gsz = 16LL * k;
  c->pairs.assign(pairs, pairs + 2 * k);
  c->kinds.assign(k, QFS_GATE_VAR2);
  drop_graph(c);
  return QFS_OK;
}

qfs_status qfs_set_path(qfs_ctx *c, int path) {
  if (!c) return QFS_ERR_ARG;
  if (path < 0 || path > 2) return fail(c, QFS_ERR_ARG, "path must be 0 (auto), 1 (streamed) or 2 (resident)");
  if (path != c->path) {
    c->path = path;
    drop_graph(c);
  }
  return QFS_OK;
}
void *qfs_stream(const qfs_ctx *c) { return c ? (void *)c->st : nullptr; }
const char *qfs_last_error(const qfs_ctx *c) { return c ? c->err.c_str() : "null context"; }

void qfs_destroy(qfs_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  if (c->d_dbg && c->dbg_n)
    fprintf(stderr, "[qfs tail timing] per gate launch (avg over %lld): first-CTA-start -> last-CTA-elected %.2f us, "
            "partial reduce %.2f us, polar %.2f us\n", c->dbg_n, c->dbg_acc[0] / c->dbg_n / 1e3,
            c->dbg_acc[1] / c->dbg_n / 1e3, c->dbg_acc[2] / c->dbg_n / 1e3);
  dfree(c->d_dbg);
  if (c->d_res_dbg && c->res_sweeps) {
    unsigned long long h[8];
    cudaMemcpy(h, c->d_res_dbg, sizeof h, cudaMemcpyDeviceToHost);
    const char *nm[8] = {"load", "forward", "env", "reduce", "polar", "uncompute-wait", "chi", "validation"};
    fprintf(stderr, "[qfs resident timing] cluster 0 rank 0, us per launch summed over its slots (%lld launches; K=%d):", c->res_sweeps, c->K);
    for (int q = 0; q < 8; ++q) fprintf(stderr, " %s %.2f", nm[q], h[q] / 1e3 / c->res_sweeps);
    fprintf(stderr, "\n");
  }
  dfree(c->d_res_dbg);
  prof_collect(c);
  drop_graph(c);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  dfree(c->d_pairs); dfree(c->d_kinds); dfree(c->d_bg); dfree(c->d_bpart); dfree(c->d_flag); dfree(c->d_x); dfree(c->d_y); dfree(c->d_xv); dfree(c->d_yv);
  dfree(c->d_gates); dfree(c->d_chi); dfree(c->d_chi2); dfree(c->d_B); dfree(c->d_vb0); dfree(c->d_vb1);
  dfree(c->d_partials); dfree(c->d_ered); dfree(c->d_sig); dfree(c->d_csum); dfree(c->d_rowout);
  c->d_cval = nullptr; dfree(c->d_counters); dfree(c->d_slots); dfree(c->d_env_trace);
  dfree(c->d_stage); dfree(c->d_vprev);
  if (c->h_check) cudaFreeHost(c->h_check);
  if (c->h_pubflag) cudaFreeHost(c->h_pubflag);
  dfree(c->d_check);
  if (c->h_gates) cudaFreeHost(c->h_gates);
  if (c->h_slots) cudaFreeHost(c->h_slots);
  if (c->st_copy) {
    cudaStreamSynchronize(c->st_copy);
    cudaStreamDestroy(c->st_copy);
  }
  for (auto &g : c->stg) {
    dfree(g.x); dfree(g.y); dfree(g.xv); dfree(g.yv);
    if (g.ev) cudaEventDestroy(g.ev);
  }
  if (c->ev_fwd) cudaEventDestroy(c->ev_fwd);
  dfree(c->d_counters1); dfree(c->d_gpart);
  xchg_release(c);
  if (c->h_csum) cudaFreeHost(c->h_csum);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->owns_comm && c->comm) ncclCommDestroy(c->comm);
  delete c;
}

}  // extern "C"
