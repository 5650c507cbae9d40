// qfs_internal.h — launch-parameter structs shared by the runtime
// (qfs_runtime.cu) and the kernels (qfs_kernels.cu).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qfs {

// One active multistart in a lockstep launch: start index and its current
// number of (local) training rows.
struct Slot {
  int s;
  int m;
};

// Strided view of a state array: element (start s, amplitude a, sample m) is
//   base[s * ss + a * sa + m * sm]          (double2 = one complex128)
// Work buffers (chi, B cache) are sample-minor: sa = M_cap, sm = 1, so the
// 32 lanes of a warp (consecutive m) touch one contiguous 512-byte run for any
// gate qubit pair.  The transposed pools use ss = 0, sa = m_pool, sm = 1;
// row-major arrays (validation, unit ops) use sa = 1, sm = 2^n.
struct View {
  const double2 *base;
  long long ss, sa, sm;
  int ident;  // 1: the implicit computational basis (qfs_set_samples_basis): element (a, m) = [a == m]; base unused
};
struct ViewW {
  double2 *base;
  long long ss, sa, sm;
};

// Layout-permuted, sample-blocked state arrays ("perm mode"):
// a start's block holds M_cap / sb sample blocks of [2^n rows][sb samples]
// (elements per block: blk = 2^n sb); in the layout L_i of gate i the
// physical row of natural amplitude a is pi_i(a), with the union bits of
// gates i and i+1 at rows' lowest bits, so the 2^nu rows of one environment
// group are ONE contiguous run of 2^nu * sb * 16 bytes (a single bulk copy).
// A group index G (the source layout's other bits, ascending) and local index
// v map to the destination row  sum_j bit_j(G) << dpos[j]  |  dv[v].
constexpr int kMaxQubits = 26;
struct Scatter {
  int dv[16];
  unsigned char dpos[kMaxQubits];
};

// Per-gate description of the fused backward step for gate i:
//   chi <- G_{i+1}^dag chi (if upd) and E_i += phi_i (x) conj(chi)
// over the 2^nu-amplitude groups spanned by the union of both gates' bits.
struct GateDesc {
  int nu, tp0, tp1, upd;      // union bits; local positions of gate i's pair; update?
  int upd_gate, env_gate;     // i+1 (or -1), i
  int pre;                    // 1: phi does not depend on the previous launch (PDL prefetch)
  uint32_t ins[4];            // union bit positions, ascending (for zero insertion)
  long long off[16];          // amplitude offset of local index v (local bit t <-> loc[t])
  View chi_src;
  ViewW chi_dst;              // base == nullptr: do not write chi back
  View phi;
  // perm mode (bwdt_kernel only): chi_src / phi in permuted blocked layout L_i
  // (one copy per stage) unless *_nat (a natural pool: one copy per row);
  // chi_dst permuted blocked in L_{i-1} through xs
  int perm, chi_nat, phi_nat, sb, n_oth;
  long long blk;
  Scatter xs;
};

struct BwdParams {
  int n, nb, K, S;            // qubits, CTAs per start, gates, total starts (trace layout)
  const Slot *slots;
  GateDesc g;                 // this launch's gate
  const double2 *gates;       // [S][K][16]
  double2 *gates_w;           // same array (written by the polar step)
  const int *kinds;           // [K] gate kinds (0 two-qubit variable, 1 fixed, 2 one-qubit), or nullptr
  double2 *vprev;             // [S][K][16] right singular vectors (warm start) or nullptr
  double *partials;           // [S_act][nb][32]
  unsigned *counters;         // [S_act]
  unsigned *counters1;        // [S_act][40] first-level group tickets (two-level reduction), or nullptr
  double *gpartials;          // [S_act][40][32] group sums
  double *e_red;              // [S_act][32]: reduced E (sample mode: before all-reduce)
  int fuse_polar;             // 1: the last CTA of each start runs the polar update
  int nt;                     // threads per CTA of bwd_kernel (bwd_threads; 0 = default)
  int bulk;                   // 1: bwdt_kernel (bulk copies + mbarrier ring), 0: bwd_kernel (LDGSTS)
  // Device-initiated exchange of the partial environments across the xg ranks
  // of sample mode, done by the last CTA of each start
  // before its polar update: store E into every rank's mailbox as
  // self-validating (32-bit half, epoch) words, wait until all ranks' words of
  // this epoch have landed, sum the xg partials in rank order.
  int xg;                              // > 1: exchange on; ranks
  int xrank;                           // this context's rank; -1: emulated ranks (rank = slot start index)
  int xS;                              // starts per mailbox
  unsigned long long *const *xmbox;    // [xg] rank q's mailbox [2 parity][xg src][xS][64 words]
  unsigned long long *xepoch;          // this context's epoch counters [xS] (emulated: [xg][xS])
  double beta;
  double *sig;                // [S][K] sum sigma, or nullptr
  double2 *env_trace;         // [K][S][16] for this sweep, or nullptr
  unsigned long long *dbg;    // diagnostics: [K][4] globaltimer stamps, or nullptr
};

// Polar update of E (already reduced / all-reduced) for each active start.
struct PolarParams {
  int K, gate, S, n_slots;
  const Slot *slots;
  const int *kinds;           // [K] or nullptr
  const double *e_red;        // [S_act][32]
  double2 *gates;             // [S][K][16]
  double2 *vprev;             // [S][K][16] or nullptr
  double beta;
  double *sig;                // [S][K] or nullptr
  double2 *env_trace;         // [K][S][16] or nullptr
};

// Sweep-end cost: chi' = G_0^dag chi ; sum_m ||chi'_m - x_m||^2 (direct form)
struct FinalParams {
  int n, nb, K;
  const Slot *slots;
  View chi, x;
  int p0, p1;
  int sb;                     // > 0: chi is sample-blocked (natural rows): (m / sb) blk + a sb + m % sb
  long long blk;
  const double2 *gates;       // gate 0 of start s: gates + s*K*16
  double *partials;           // [S_act][nb]
  unsigned *counters;         // [S_act]
  double *out_sum;            // [S_act] raw sum (host divides by M)
};

// Per-gate forward: dst = G_k src for every (quadruple, sample) of every slot.
struct FwdGateParams {
  int n, nb, k, K, rows_fixed; // rows_fixed > 0: that many rows per start (validation)
  int cache_mode;              // bit 0: stores L2::evict_last, bit 1: loads L2::evict_first
  const Slot *slots;
  int p0, p1;
  const double2 *gates;
  View src;
  ViewW dst;
};

// Two consecutive forward gates per pass (fwd2_kernel): B_{k+1}, B_{k+2}.
struct Fwd2Params {
  int n, nb, k, K;
  int nu, tp0, tp1;           // union bits; local positions of gate k+1's pair
  const Slot *slots;
  const double2 *gates;
  uint32_t ins[4];            // union bit positions, ascending
  long long off[16];          // amplitude offset of local index v
  View src;                   // B_k (sample-minor, sm == 1)
  ViewW dst1, dst2;           // B_{k+1}, B_{k+2}
};

// Two-gate forward in perm mode (fwdp_kernel): reads B_k (permuted blocked
// layout L_k; k = 0: the natural x pool through ins / off), writes B_{k+1}
// in L_{k+1} and B_{k+2} in L_{k+2} (dst2.base == nullptr: gate k only).
struct FwdpParams {
  int n, nb, k, K, nu, tp0, tp1, sb, src_nat, n_oth;
  long long blk;
  const Slot *slots;
  const double2 *gates;
  uint32_t ins[4];            // natural source: union bit positions, ascending
  long long off[16];          // natural source: amplitude offset of local v
  int tau[16];                // permuted source: row of local v within the group
  View src;
  ViewW dst1, dst2;           // per-start strides only (ss); rows addressed through the scatters
  Scatter s1, s2;
};

// Whole-row validation forward in shared memory (n <= 13): one CTA per
// (start, validation row); all K gates, then sum ||row - yv_row||^2.
struct ValRowParams {
  int n, K, rows;
  const Slot *slots;
  const int2 *pairs;          // [K]
  const double2 *gates;       // [S][K][16]
  const double2 *xv, *yv;     // row-major [rows][2^n]
  double *row_out;            // [S_act][rows]
};

// Row distance sums (streamed validation end): out[j*rows + r] = ||a - b||^2
struct DistParams {
  int n, rows;
  const Slot *slots;
  View a, b;
  double *row_out;
};

// Cluster-resident sweep (qfs_resident.cu): one cluster of C CTAs per start,
// states of the CTA's sample slice in shared memory, whole sweep + costs.
struct ResParams {
  int n, K, S, C, ld;         // qubits, gates, total starts (trace layout), cluster size, rows per CTA
  int n_slots;
  const Slot *slots;
  const int2 *pairs;          // [K]
  const int *kinds;           // [K] gate kinds, or nullptr
  double2 *gates;             // [S][K][16]: old gates in, new gates out
  const double2 *x, *y;       // pools, sample-minor [2^n][m_pool]
  long long m_pool;
  const double2 *xv, *yv;     // validation rows, row-major [V][2^n]
  int V, want_val;
  double beta;
  double *csum, *cval;        // [n_slots] raw sums ||chi - x||^2, ||C xv - yv||^2
  double *sig;                // [S][K] sum sigma, or nullptr
  double2 *env_trace;         // [K][S][16], or nullptr
  unsigned long long *dbg;    // diagnostics (QFS_TAIL_TIMING): [8] summed globaltimer phases, or nullptr
};

// kernel-level unit ops
struct ApplyParams {
  int n, p0, p1, m;
  double2 g[16];              // already adjointed if requested
  double2 *psi;
};

// ---- launchers (qfs_kernels.cu); all return cudaGetLastError() ----
cudaError_t launch_bwd(const BwdParams &p, int n_slots, cudaStream_t st);
int fwd2_min_blocks();             // CTAs per SM the two-gate forward kernel is compiled for
cudaError_t launch_polar(const PolarParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_final(const FinalParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_fwd_gate(const FwdGateParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_fwd2(const Fwd2Params &p, int n_slots, cudaStream_t st);
cudaError_t launch_fwdp(const FwdpParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_val_row(const ValRowParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_dist(const DistParams &p, int n_slots, cudaStream_t st);
cudaError_t launch_row_reduce(const double *row_in, int rows, double *out, int n_slots,
                              cudaStream_t st);
cudaError_t launch_apply(const ApplyParams &p, cudaStream_t st);
cudaError_t launch_polar_batch(const double2 *env, const double2 *g_old, double beta,
                               double2 *g_new, double *sig, int count, cudaStream_t st);
cudaError_t launch_transpose(const double2 *src, double2 *dst, int rows, long long cols,
                             cudaStream_t st);
cudaError_t launch_finite_check(const double *p, long long n, int *flag, cudaStream_t st);
cudaError_t launch_identity_fill(double2 *v, long long count16, cudaStream_t st);
cudaError_t launch_copy(double2 *dst, const double2 *src, long long count, cudaStream_t st);  // device copy by a kernel
cudaError_t launch_copy_bytes(void *dst, const void *src, size_t bytes, cudaStream_t st);  // 4-byte granular
cudaError_t launch_fill_words(unsigned *dst, unsigned value, long long count, cudaStream_t st);
cudaError_t launch_flag_bit(const unsigned *src, unsigned *dst, unsigned bit, cudaStream_t st);
// hdst / hcheck / hflag: device pointers of mapped pinned host memory
cudaError_t launch_publish(const double *src, int count, const unsigned *check, double *hdst, unsigned *hcheck,
                           unsigned long long *hflag, unsigned long long seq, cudaStream_t st);
cudaError_t launch_gate_check(const double2 *g, long long count, int K, const int *kinds, unsigned *flag,
                              cudaStream_t st);  // initial-gate validation bits into *flag
void set_pdl(bool on);     // launch with programmatic dependent launch (default on)
bool pdl_enabled();
int val_row_max_n();
size_t res_smem_bytes(int n, int K, int ld);  // dynamic shared memory of the resident kernel
size_t res_smem_limit(int minb);  // per-CTA limit when minb CTAs share an SM
int resident_max_clusters(int C, size_t smem); // co-resident clusters of C CTAs (0: cannot launch)
cudaError_t launch_resident(const ResParams &p, int clusters, cudaStream_t st);
// two starts per cluster, one start's polar overlapped with the other's passes
size_t res2_smem_bytes(int n, int K, int ld);
int resident2_max_clusters(int C, size_t smem);
cudaError_t launch_resident_pair(const ResParams &p, int clusters, cudaStream_t st);  // clusters: of start PAIRS
size_t val_blk_smem(int n, int K, int ld);     // shared memory of the block validation kernel
cudaError_t launch_val_block(const ValRowParams &p, int n_slots, cudaStream_t st);
size_t val_cl_smem(int n, int K, int t);      // cluster validation, 2^t CTAs per row
cudaError_t launch_val_cluster(const ValRowParams &p, int n_slots, cudaStream_t st);        // largest n the shared-memory validation forward supports
int bwd_threads(int n_slots);  // threads per CTA of the LDGSTS backward launch
int blocks_per_sm(int nt);  // resident CTAs per SM of the backward kernel at nt threads
size_t bt_smem_bytes(int nu);     // dynamic shared memory of the bulk-copy backward kernel
int bwdt_units_per_cta_min();     // fewest stages a bulk-copy backward CTA is given


// ---------------------------------------------------- multi-qubit blocks --
// qfs_create_blocks circuits (qfs_blocks.cu).  Gate k:
// arity a (2 or 3) on qubits q[0..a-1] (local l = sum_j b(q_j) 2^j), its d x d
// matrix packed at complex offset off of the start's gate block (gsz entries).
struct BlkGate {
  int a, q[3], off, kind;
};
#ifndef QFS_BLK_CTAS_PER_SM
#define QFS_BLK_CTAS_PER_SM 4
#endif
constexpr int kBlkMaxCtas = 148 * QFS_BLK_CTAS_PER_SM;  // CTAs per start of any block launch
struct BlkApplyParams {
  int n, k, dagger, rows_fixed;  // rows_fixed > 0: that many rows per start (validation)
  const Slot *slots;
  const BlkGate *bg;
  const double2 *gates;
  long long gsz;
  View src;
  ViewW dst;
};
struct BlkEnvParams {
  int n, i, K, S;
  const Slot *slots;
  const BlkGate *bg;
  double2 *gates;               // read (old gate) and written (update)
  long long gsz;
  View phi, chi;
  double *partials;             // [S_act][nb][2 d^2]
  unsigned *counters;           // [S_act]
  double beta;
  double *sig;                  // [S][K] or nullptr
  double2 *env_trace;           // gate-major [S * gsz] for this sweep, or nullptr
  unsigned *err;                // bit 8: the 8x8 polar iteration did not converge
};
struct BlkDistParams {
  int n, rows_fixed;
  const Slot *slots;
  View a, b;
  double *partials;             // [S_act][nb]
  unsigned *counters;           // [S_act]
  double *out;                  // [S_act]
};
int blk_ctas(long long items, int n_slots);
cudaError_t launch_blk_apply(const BlkApplyParams &p, int arity, int nb, int n_slots, cudaStream_t st);
cudaError_t launch_blk_env(const BlkEnvParams &p, int arity, int nb, int n_slots, cudaStream_t st);
cudaError_t launch_blk_dist(const BlkDistParams &p, int nb, int n_slots, cudaStream_t st);
cudaError_t launch_blk_gate_check(const double2 *g, const BlkGate *bg, int K, long long gsz, int s, unsigned *flag,
                                  cudaStream_t st);

}  // namespace qfs
