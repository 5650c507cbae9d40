// qfs_kernels.cu — sm_100a kernels of the QFactor-Sample sweep (arXiv 2405.12866).
//
// Hot path of one sweep (§3):
//   fwd_gate_kernel : B_{k+1} = G_k B_k, the B tensors
//   bwd_kernel      : chi <- G_{i+1}^dag chi fused with the environment
//                     E_i = sum phi (x) conj(chi) (Fig. env_calc);
//                     its last CTA per start reduces the CTA partials in order
//                     and runs the half-warp Jacobi polar update u = Y X^dag
//                     (eq:opt_u)
//   final_kernel    : chi <- G_0^dag chi, c_train = (1/M) sum ||chi - x||^2
//   val_row_kernel  : validation cost with the post-sweep gates
// All arithmetic is FP64 (complex128).  Every reduction runs in a fixed order
// (per-thread -> warp shuffle -> CTA -> CTA partials summed in index order by
// the last CTA), so results are deterministic for a given launch shape.
//
// State arrays are sample-minor ([start][amplitude][sample], View in
// qfs_internal.h): a warp's lanes take consecutive samples of the same
// amplitude, so each of a thread's 2^nu amplitude loads is one fully coalesced
// 512-byte warp access whatever qubits the gate acts on.
//
// No code here is shared with the CPU oracle.
#include <cuda_runtime.h>
#include <algorithm>
#include <stdint.h>

#include "qfs_device.cuh"
#include "qfs_internal.h"

namespace qfs {

namespace {

#ifndef QFS_BWD_THREADS
#define QFS_BWD_THREADS 256
#endif
#ifndef QFS_BWD_STAGES
#define QFS_BWD_STAGES 4
#endif
#ifndef QFS_BWD_MINB
#define QFS_BWD_MINB 1
#endif
#ifndef QFS_BWD_HALF_SLOTS
#define QFS_BWD_HALF_SLOTS 2  // starts per launch from which the backward runs 128-thread CTAs, 2 per SM
#endif
#ifndef QFS_BWD_HALF_MINB
#define QFS_BWD_HALF_MINB 2   // resident 128-thread backward CTAs per SM
#endif
#ifndef QFS_WIDE_RED
#define QFS_WIDE_RED 1  // backward, many CTAs per start: one-ticket reduction by all warps of the last CTA
#endif
#ifndef QFS_BWD_BYTEOFF
#define QFS_BWD_BYTEOFF 1  // backward: 32-bit byte offsets from per-start bases for LDGSTS / STG addresses
#endif
#ifndef QFS_BWD_HINT
#define QFS_BWD_HINT 0  // backward L2 hints: 1 phi loads evict_first, 2 chi stores evict_last (A/B)
#endif
#ifndef QFS_BWD_EDRING
#define QFS_BWD_EDRING 1  // backward: chi store offsets carried from issue to use in registers
#endif
#ifndef QFS_FWD2_MINB
#define QFS_FWD2_MINB 2    // two-gate forward: resident CTAs per SM (128 threads each, QFS_FWD2_THREADS)
#endif
#ifndef QFS_FWD2_PF
#define QFS_FWD2_PF 1      // two-gate forward: prefetch the next item's amplitudes into registers
#endif
#ifndef QFS_FWD2_GSMEM
#define QFS_FWD2_GSMEM QFS_FWD2_PF  // re-read gate entries from shared memory (frees 128 registers)
#endif
#ifndef QFS_FWD2_HINT
#define QFS_FWD2_HINT 1    // L2 hints: 1 B_{k+1} stores evict_first, 2 B_{k+2} evict_last, 4 B_k loads evict_first
#endif
constexpr int BWD_THREADS = QFS_BWD_THREADS;
constexpr int BWD_STAGES = QFS_BWD_STAGES;  // LDGSTS pipeline depth of the backward kernel
constexpr int FWD_THREADS = 256;
#ifndef QFS_FWD2_THREADS
#define QFS_FWD2_THREADS 128  // C4 forward 22.1 -> 21.1 ms / 20 steps vs 256 x 1 (finer tail)
#endif
constexpr int FWD2_THREADS = QFS_FWD2_THREADS;  // two-gate forward CTA size
constexpr int FWD_STAGES = 4;   // LDGSTS pipeline depth of the forward kernel
constexpr int VAL_THREADS = 512;
constexpr int RED_THREADS = 256;
constexpr int RED_GS = 16;    // CTAs per first-level group of the backward reduction
constexpr int RED_GMAX = 40;  // >= ceil(max CTAs per start (148 * 4) / RED_GS)


// Polar step of one start by one warp (lanes 16-31 mirror lanes 0-15):
// the kind-aware update of gate_update (E' = (1 - beta) E + beta G_old^dag for
// variable gates); writes G_i, V_i, sum sigma, E trace.
__device__ void polar_write(const double *e32, double2 *gout, double2 *vslot, double beta, int kind,
                            double *sig_out, double2 *env_out, double2 *scratch) {
  const int lane = threadIdx.x & 31, l = lane & 15;
  const double2 e = make_double2(e32[2 * l], e32[2 * l + 1]);
  if (env_out && lane < 16) env_out[l] = e;
  double2 g, v;
  double ss;
  const bool vnew = gate_update(kind, e, gout, beta, vslot, g, v, ss, scratch + 2 * (lane & 16), sig_out != nullptr);
  __syncwarp();
  if (lane < 16 && kind != 1) {
    gout[l] = g;
    if (vslot && vnew) vslot[l] = v;
  }
  if (lane == 0 && sig_out) *sig_out = ss;
}

// Last-CTA election for the per-start reduction of CTA partials, by warp 0
// only (the warp that wrote this CTA's partial): release fence, ticket, and an
// acquire fence in the last CTA.  The other warps never fence or wait.
#ifndef QFS_ELECT_ACQREL
#define QFS_ELECT_ACQREL 1  // ticket as one acq_rel atomic (after a warp barrier) instead of fence + atomic + fence
#endif
__device__ bool warp0_elect_last(unsigned *counter, unsigned nb) {
#if QFS_ELECT_ACQREL
  // the warp's partial stores are ordered before lane 0's release by the warp
  // barrier (release is cumulative); the last CTA's acquire orders the reads of
  // every CTA's partial after it, for all lanes through the second warp barrier
  __syncwarp();
  unsigned last = 0;
  if ((threadIdx.x & 31) == 0) {
    unsigned t;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter) : "memory");
    last = (t == nb - 1) ? 1u : 0u;
    if (last) *counter = 0u;
  }
  last = __shfl_sync(FULL, last, 0);
  __syncwarp();
  return last != 0;
#else
  __threadfence();
  unsigned last = 0;
  if ((threadIdx.x & 31) == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    last = (t == nb - 1) ? 1u : 0u;
    if (last) *counter = 0u;
  }
  last = __shfl_sync(FULL, last, 0);
  if (last) __threadfence();
  return last != 0;
#endif
}

// P-index (0..3) of local amplitude index v for the pair at local bits (TP0, TP1)
template <int TP0, int TP1>
__device__ __forceinline__ int pidx(int v) {
  return ((v >> TP0) & 1) | (((v >> TP1) & 1) << 1);
}

// local index of member l of quadruple q for the pair at local bits (TP0, TP1)
// (the other local bits, ascending, take the bits of q)
template <int NU, int TP0, int TP1>
__host__ __device__ constexpr int pv_idx(int q, int l) {
  int v = ((l & 1) << TP0) | (((l >> 1) & 1) << TP1);
  int bit = 0;
  for (int t = 0; t < NU; ++t) {
    if (t == TP0 || t == TP1) continue;
    v |= ((q >> bit) & 1) << t;
    ++bit;
  }
  return v;
}

template <int NT>
struct BwdShared {
  double2 sQ[16];                          // G_{i+1}^dag
  double2 red[NT / 32][4][16];            // per-warp (per lane-group) E partials
  double sum32[32];
  double2 scratch[64];                     // polar scratch: 32 per half warp
};

// ---------------------------------------------------------------- backward --
// One CTA's share of gate i of the right-to-left sweep (Fig. env_calc
// P:172) for start slot j; ends with warp 0 holding the CTA partial of E_i in
// P.partials (other warps return from here).  Work unit = (group of 2^NU
// amplitudes spanned by both gates' qubits, block of LPT consecutive samples);
// T = 2^(NU-2) threads share a group, thread t owning the Q-quadruple whose
// local bits >= 2 equal t (local bits 0,1 are the Q pair = gate i+1).  Per item:
//   if UPD: chi <- G_{i+1}^dag chi on the own Q-quadruple, written back;
//   NU == 4: the four threads transpose through shared memory so that thread t
//     holds P-quadruple t (members in xor order a = t ^ x), phi is loaded in
//     that order, and all 16 entries of E are accumulated per thread;
//   NU < 4: all-gather of chi by shuffles, accumulators keyed at compile time
//     by (la & PLO, lb & PLO, x) with the target entry fixed by the key and t.
// chi/phi of the next items are staged into shared memory by LDGSTS,
// BWD_STAGES-1 items ahead.  Reductions run in a fixed order (lanes, lane
// groups, warps), so the partial is deterministic for a given launch shape.
template <int NT, int NU, int TP0, int TP1, bool UPD, bool IDENT>
__device__ bool bwd_gate_partial(const BwdParams &P, const GateDesc &G, int jslot, int s,
                                 unsigned Ms, BwdShared<NT> &sh, double2 *stage_buf) {
  constexpr int T = 1 << (NU - 2);
  constexpr int LPT = 32 / T;
  constexpr int NWARP = NT / 32;
  constexpr int PLO = ((TP0 < 2) ? (1 << TP0) : 0) | ((TP1 < 2) ? (1 << TP1) : 0);
  constexpr int NPT_T = (((1 << NU) - 1) & ~((1 << TP0) | (1 << TP1))) >> 2;
  constexpr bool XPOSE = (NU == 4);
  constexpr int AZ = XPOSE ? 1 : T;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane / LPT, ml = lane % LPT;
  const unsigned nmb = (Ms + LPT - 1) / LPT;
  const unsigned units = (1u << (P.n - NU)) * nmb;
  const unsigned chunk = (units + P.nb - 1) / P.nb;
  const unsigned beg = blockIdx.x * chunk;
  const unsigned end = min(units, beg + chunk);
  const FastDiv fdu(nmb);
#if QFS_BWD_HINT & 1
  const uint64_t pol_phi = policy_evict_first();
#endif
#if QFS_BWD_HINT & 2
  const uint64_t pol_chi = policy_evict_last();
#endif

  double2 acc[4][4][AZ];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int x = 0; x < AZ; ++x) acc[p][q][x] = make_double2(0.0, 0.0);

  // element offsets inside one start's block (sample-minor views: sm == 1)
  const double2 *csrc = G.chi_src.base + (long long)s * G.chi_src.ss;
  double2 *cdst = G.chi_dst.base ? G.chi_dst.base + (long long)s * G.chi_dst.ss : nullptr;
  const double2 *fsrc = G.phi.base + (long long)s * G.phi.ss;
  const unsigned csa = (unsigned)G.chi_src.sa, dsa = (unsigned)G.chi_dst.sa, fsa = (unsigned)G.phi.sa;
#if QFS_BWD_BYTEOFF
  const char *cbase = (const char *)csrc, *fbase = (const char *)fsrc;
  char *dbase = (char *)cdst;
#endif
  unsigned offc[4], offd[4], offf[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const unsigned o = (unsigned)G.off[4 * t + l];
    offc[l] = o * csa;
    offd[l] = o * dsa;
    offf[l] = (unsigned)G.off[XPOSE ? (t + 4 * (t ^ l)) : (4 * t + l)] * fsa;
  }
  uint32_t ins[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) ins[q] = G.ins[q];

  const unsigned ustart = beg + warp;
  const int iters = ustart < end ? (int)((end - ustart + NWARP - 1) / NWARP) : 0;
  unsigned lg = 0, lm = 0;  // group base amplitude and sample of the last located item (implicit basis phi)
  auto locate = [&](int k, unsigned &ec, unsigned &ed, unsigned &ef) -> bool {
    const unsigned u = ustart + (unsigned)k * NWARP;
    if (k >= iters) return false;
    unsigned g = fdu.div(u);
    const unsigned m = (u - g * nmb) * LPT + ml;
    if (IDENT) lm = m;
#pragma unroll
    for (int q = 0; q < NU; ++q) g = insert_zero32(g, ins[q]);
    if (IDENT) lg = g;
    ec = g * csa + m;
    ed = g * dsa + m;
    ef = g * fsa + m;
    // every member offset stays inside one start's [2^n][sa] block (32-bit guard, runtime offsets_fit)
    QFS_DASSERT(m >= Ms || ((unsigned long long)(g | (unsigned)G.off[(1 << NU) - 1]) << 0) < (1ull << P.n));
    QFS_DASSERT(m >= Ms || G.phi.ident || (unsigned long long)(g + (unsigned)G.off[(1 << NU) - 1]) * fsa + m < ((unsigned long long)fsa << P.n));
    return m < Ms;
  };
  // chi destination offset of the items in flight (EDRING: computed once, at
  // issue, and rotated through registers; ~0xffffffff marks an invalid item)
#if QFS_BWD_EDRING
  unsigned edr[BWD_STAGES];
#pragma unroll
  for (int q = 0; q < BWD_STAGES; ++q) edr[q] = 0xffffffffu;
#endif
  auto issue_part = [&](int k, bool chi, bool phi) {
    unsigned ec = 0, ed = 0, ef = 0;
    const bool ok = locate(k, ec, ed, ef);
#if QFS_BWD_EDRING
    if (chi) edr[BWD_STAGES - 1] = ok ? ed : 0xffffffffu;
#endif
    double2 *st = stage_buf + (k % BWD_STAGES) * 8 * NT + threadIdx.x;
#if QFS_BWD_BYTEOFF
    // 32-bit byte offsets from the start's base (one start's block < 4 GB):
    // one add per address instead of 64-bit element arithmetic per address
    if (!ok) ec = ef = 0u;  // in bounds; nothing is read (src-size 0)
    if (chi) {
      const unsigned eb = ec << 4;
#pragma unroll
      for (int l = 0; l < 4; ++l) cp_async16(st + l * NT, cbase + (eb + (offc[l] << 4)), ok);
    }
    if (IDENT && phi) {  // implicit basis x_m = e_m (gate 0 of a QF sweep): synthesised, not loaded
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const unsigned a = lg + (unsigned)G.off[XPOSE ? (t + 4 * (t ^ l)) : (4 * t + l)];
        st[(4 + l) * NT] = make_double2(ok && a == lm ? 1.0 : 0.0, 0.0);
      }
    } else if (phi) {
      const unsigned eb = ef << 4;
#pragma unroll
#if QFS_BWD_HINT & 1  // phi = B_i is read once: L2 evict_first
      for (int l = 0; l < 4; ++l)
        cp_async16_hint(st + (4 + l) * NT, fbase + (eb + (offf[l] << 4)), ok, pol_phi);
#else
      for (int l = 0; l < 4; ++l) cp_async16(st + (4 + l) * NT, fbase + (eb + (offf[l] << 4)), ok);
#endif
    }
#else
    if (chi) {
#pragma unroll
      for (int l = 0; l < 4; ++l) cp_async16(st + l * NT, csrc + (ok ? ec + offc[l] : 0u), ok);
    }
    if (phi) {
#pragma unroll
      for (int l = 0; l < 4; ++l) cp_async16(st + (4 + l) * NT, fsrc + (ok ? ef + offf[l] : 0u), ok);
    }
#endif
  };
  auto issue = [&](int k) {
    issue_part(k, true, true);
    cp_async_commit();
  };
  // Prologue.  phi (B_i, written by the forward pass or the x pool) does not
  // depend on the previous backward launch, so with G.pre its first stages are
  // fetched before pdl_wait(), overlapping the previous launch's polar tail.
  // chi and G_{i+1} are written by the previous launch: read after the wait.
  if (G.pre) {
#pragma unroll
    for (int k = 0; k < BWD_STAGES - 1; ++k) issue_part(k, false, true);
    cp_async_commit();
  }
  // dependence on the previous gate: kernel boundary (PDL)
  pdl_wait();
  if (UPD && threadIdx.x < 16) {
    const int a = threadIdx.x >> 2, b = threadIdx.x & 3;
    const double2 g = __ldcg(P.gates + ((long long)s * P.K + G.upd_gate) * 16 + 4 * b + a);
    sh.sQ[threadIdx.x] = cconj(g);  // (G^dag)[a][b]
  }
  if (P.dbg && threadIdx.x == 0) atomicMin(P.dbg + 4 * G.env_gate, gtimer());
#pragma unroll
  for (int k = 0; k < BWD_STAGES - 1; ++k) {
    issue_part(k, true, !G.pre);
    cp_async_commit();
#if QFS_BWD_EDRING
#pragma unroll
    for (int q = 0; q < BWD_STAGES - 1; ++q) edr[q] = edr[q + 1];
#endif
  }
  __syncthreads();
  // G_{i+1}^dag in registers for the whole loop (214 registers, no spill); read
  // from shared memory per item it cost 16 LDS per item (C4 bwd -2.4 % with it here)
#ifndef QFS_BWD_GREG
#define QFS_BWD_GREG 1  // 1: G_{i+1}^dag in registers for the loop; 0: broadcast shared-memory loads per use
#endif
#if QFS_BWD_GREG
  double2 sqr[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) sqr[e] = sh.sQ[e];
#define QFS_SQ(e) sqr[e]
#else
#define QFS_SQ(e) lds_v2(&sh.sQ[e])
#endif

  for (int k = 0; k < iters; ++k) {
    issue(k + BWD_STAGES - 1);
    cp_async_wait<BWD_STAGES - 1>();
#if QFS_BWD_EDRING
    // after the prologue's shifts edr[q] holds item k + q
    const unsigned ed = edr[0];
    const bool valid = ed != 0xffffffffu;
#pragma unroll
    for (int q = 0; q < BWD_STAGES - 1; ++q) edr[q] = edr[q + 1];
#else
    unsigned ec = 0, ed = 0, ef = 0;
    const bool valid = locate(k, ec, ed, ef);
#endif
    double2 *st = stage_buf + (k % BWD_STAGES) * 8 * NT + threadIdx.x;
    double2 c[4], f[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) c[l] = st[l * NT];
#pragma unroll
    for (int l = 0; l < 4; ++l) f[l] = st[(4 + l) * NT];
#ifdef QFS_DIAG_NOCOMPUTE  // diagnostic build: memory traffic only (results invalid)
    if (UPD && cdst && valid) {
      double2 *dp = cdst + ed;
#pragma unroll
      for (int l = 0; l < 4; ++l) dp[offd[l]] = c[l];
    }
    acc[0][0][0].x += c[0].x + f[0].x + c[1].x + f[1].x + c[2].x + f[2].x + c[3].x + f[3].x;
    if (false)
#endif
    if (UPD) {
      double2 o[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o[a], QFS_SQ(4 * a + b), c[b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) c[a] = o[a];
      if (cdst && valid) {
#if QFS_BWD_BYTEOFF
        const unsigned eb = ed << 4;
#pragma unroll
#if QFS_BWD_HINT & 2  // chi is re-read by the next launch: L2 evict_last
        for (int l = 0; l < 4; ++l) st_hint((double2 *)(dbase + (eb + (offd[l] << 4))), c[l], pol_chi);
#else
        for (int l = 0; l < 4; ++l) *(double2 *)(dbase + (eb + (offd[l] << 4))) = c[l];
#endif
#else
        double2 *dp = cdst + ed;
#pragma unroll
        for (int l = 0; l < 4; ++l) dp[offd[l]] = c[l];
#endif
      }
    }
#ifdef QFS_DIAG_NOCOMPUTE
    if (false)
#endif
    if (XPOSE) {
      // transpose through this stage's (already consumed) chi slots
      __syncwarp();
#pragma unroll
      for (int l = 0; l < 4; ++l) st[l * NT] = c[l];
      __syncwarp();
      double2 r[4];
      const int lane_base = threadIdx.x - lane;
#pragma unroll
      for (int x = 0; x < 4; ++x)
        r[x] = stage_buf[(k % BWD_STAGES) * 8 * NT + t * NT + lane_base + (lane ^ (x * LPT))];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          double2 &e = acc[x][y][0];
          e.x = fma(f[x].x, r[y].x, e.x);
          e.x = fma(f[x].y, r[y].y, e.x);
          e.y = fma(f[x].y, r[y].x, e.y);
          e.y = fma(-f[x].x, r[y].y, e.y);
        }
    } else {
#pragma unroll
      for (int x = 0; x < T; ++x) {
        if ((x & NPT_T) != 0) continue;  // partner differs in a non-P bit: no shared P-quadruple
        double2 cx[4];
#pragma unroll
        for (int l = 0; l < 4; ++l) cx[l] = x == 0 ? c[l] : shfl_xor_c(c[l], x * LPT);
#pragma unroll
        for (int la = 0; la < 4; ++la)
#pragma unroll
          for (int lb = 0; lb < 4; ++lb) {
            if (((la ^ lb) & ~PLO & 3) != 0) continue;
            double2 &e = acc[la & PLO][lb & PLO][x < AZ ? x : 0];
            // f[la] * conj(cx[lb])
            e.x = fma(f[la].x, cx[lb].x, e.x);
            e.x = fma(f[la].y, cx[lb].y, e.x);
            e.y = fma(f[la].y, cx[lb].x, e.y);
            e.y = fma(-f[la].x, cx[lb].y, e.y);
          }
      }
    }
  }
  cp_async_wait<0>();
  pdl_trigger();  // all of this CTA's reads of chi/phi are done

  // CTA reduction: over the sample lanes of each lane-group, then lane groups
  // and warps in a fixed order
#pragma unroll
  for (int pa = 0; pa < 4; ++pa)
#pragma unroll
    for (int pb = 0; pb < 4; ++pb)
#pragma unroll
      for (int x = 0; x < AZ; ++x) {
        if (!XPOSE && ((pa & ~PLO) || (pb & ~PLO) || (x & NPT_T))) continue;
        double2 v = acc[pa][pb][x];
#pragma unroll
        for (int o = LPT / 2; o >= 1; o >>= 1) {
          v.x += __shfl_xor_sync(FULL, v.x, o);
          v.y += __shfl_xor_sync(FULL, v.y, o);
        }
        if (ml == 0) {
          int a, b;
          if (XPOSE) {  // acc[x][y]: members t^x, t^y of P-quadruple t
            a = pidx<TP0, TP1>(4 * (t ^ pa));
            b = pidx<TP0, TP1>(4 * (t ^ pb));
          } else {
            a = pidx<TP0, TP1>(pa | (t << 2));
            b = pidx<TP0, TP1>(pb | ((t ^ x) << 2));
          }
          sh.red[warp][XPOSE ? t : 0][4 * a + b] = v;
        }
      }
  __syncthreads();
  if (threadIdx.x >= 32) return false;  // warp 0 finishes the CTA's work
  {
    const int e = threadIdx.x >> 1, im = threadIdx.x & 1;
    double v = 0.0;
#pragma unroll
    for (int wq = 0; wq < NWARP; ++wq)
#pragma unroll
      for (int tq = 0; tq < (XPOSE ? T : 1); ++tq) v += im ? sh.red[wq][tq][e].y : sh.red[wq][tq][e].x;
    P.partials[((long long)jslot * P.nb + blockIdx.x) * 32 + threadIdx.x] = v;
  }
  return true;
}

// Warp 0 of the finishing CTA holds the reduced E (lane = re/im of entry lane/2):
// store it and (fuse_polar) run the gate update (kind: loaded before the
// election so its global load is off the critical path).
// Device-initiated all-reduce of the 4x4 environment over the ranks of sample
// mode (NEXT-2; E is a sum over samples, so the ranks' partials add
// up to the full E).  Warp 0 of the last CTA of start s, lane = real / imag
// part of entry lane / 2.  Each rank writes its partial into parity slot
// (epoch & 1) of EVERY rank's mailbox (peer stores over NVLink; emulated
// ranks: local memory) as two 8-byte words per value, each word = one 32-bit
// half of the double | the 32-bit epoch (the LL protocol: an aligned 8-byte
// store is single-copy atomic, so a word carrying this epoch is complete and
// no memory fence sits on the path — measured: system-scope fences cost ~11 us
// per gate here).  Every rank then polls its own mailbox until all words of
// this epoch have landed and sums the partials in rank order: identical bits
// on all ranks, identical polar updates.  Two parity slots suffice: a rank
// writes epoch t+2 only after it has read every rank's epoch t+1 words, which
// each rank writes only after finishing its epoch t reads.
__device__ double xchg_env(const BwdParams &P, int s, double e) {
  const int lane = threadIdx.x & 31;
  const int r = P.xrank >= 0 ? P.xrank : s;   // emulated: the slot's start index is its rank
  const int sx = P.xrank >= 0 ? s : 0;
  unsigned long long *ep = P.xepoch + (P.xrank >= 0 ? sx : (long long)r * P.xS + sx);
  unsigned long long epn = 0;
  if (lane == 0) {
    epn = *ep + 1;
    *ep = epn;
  }
  epn = __shfl_sync(FULL, epn, 0);
  const unsigned long long tag = (epn & 0xffffffffull) << 32;
  const long long par = (long long)(epn & 1ull);
#ifdef QFS_XCHG_FORCE_SYS  // measurement build: system scope for emulated ranks too
  const bool local = false;
#else
  const bool local = P.xrank < 0;  // real ranks: peer memory over NVLink, system scope
#endif
  const unsigned long long bits = (unsigned long long)__double_as_longlong(e);
  const unsigned long long w0 = (bits & 0xffffffffull) | tag, w1 = (bits >> 32) | tag;
  for (int q = 0; q < P.xg; ++q) {
    unsigned long long *dst = P.xmbox[q] + ((par * P.xg + r) * P.xS + sx) * 64 + 2 * lane;
    if (local) st_ll_gpu(dst, w0, w1);
    else st_ll_sys(dst, w0, w1);
  }
  double t = 0.0;
  for (int q = 0; q < P.xg; ++q) {  // rank order: identical sums everywhere
    const unsigned long long *src = P.xmbox[r] + ((par * P.xg + q) * P.xS + sx) * 64 + 2 * lane;
    unsigned long long a, b;
    for (;;) {
      if (local) ld_ll_gpu(src, a, b);
      else ld_ll_sys(src, a, b);
      if ((a & 0xffffffff00000000ull) == tag && (b & 0xffffffff00000000ull) == tag) break;
      __nanosleep(8);
    }
    t += __longlong_as_double((long long)((a & 0xffffffffull) | (b << 32)));
  }
  return t;
}

template <class SH>  // shared-memory struct with sum32[32] and scratch[64]
__device__ void bwd_finish_e(const BwdParams &P, const GateDesc &G, int jslot, int s, SH &sh, double e, int kind) {
  if (P.xg > 1) e = xchg_env(P, s, e);
  sh.sum32[threadIdx.x] = e;
  if (!P.fuse_polar) P.e_red[(long long)jslot * 32 + threadIdx.x] = e;
  __syncwarp();
  if (P.dbg && threadIdx.x == 0) atomicMax(P.dbg + 4 * G.env_gate + 2, gtimer());
  if (!P.fuse_polar) return;
  const long long gi = (long long)s * P.K + G.env_gate;
  polar_write(sh.sum32, P.gates_w + gi * 16, P.vprev ? P.vprev + gi * 16 : nullptr, P.beta,
              kind, P.sig ? P.sig + gi : nullptr,
              P.env_trace ? P.env_trace + ((long long)G.env_gate * P.S + s) * 16 : nullptr, sh.scratch);
  if (P.dbg && threadIdx.x == 0) atomicMax(P.dbg + 4 * G.env_gate + 3, gtimer());
}

// Warp 0 of the last CTA of a start: sum the CTA partials in CTA order, and
// (fuse_polar) run the polar update of gate i.
template <int NT>
__device__ void bwd_finish(const BwdParams &P, const GateDesc &G, int jslot, int s, BwdShared<NT> &sh, int kind) {
  if (P.dbg && threadIdx.x == 0) atomicMax(P.dbg + 4 * G.env_gate + 1, gtimer());
  const double *pp = P.partials + (long long)jslot * P.nb * 32 + threadIdx.x;
  double e = 0.0;
  // 48 loads in flight per lane, adds in CTA order: one L2 round trip per 48
  // CTAs (at C5, S = 1, nb = 148: 4 round trips instead of 10 with 16)
  constexpr int FLIGHT = 48;
  for (int b0 = 0; b0 < P.nb; b0 += FLIGHT) {
    double xb[FLIGHT];
#pragma unroll
    for (int q = 0; q < FLIGHT; ++q) xb[q] = b0 + q < P.nb ? __ldcg(pp + (long long)(b0 + q) * 32) : 0.0;
#pragma unroll
    for (int q = 0; q < FLIGHT; ++q)
      if (b0 + q < P.nb) e += xb[q];
  }
  bwd_finish_e(P, G, jslot, s, sh, e, kind);
}


// One launch per gate (used in sample-sharded mode and by the unit op).
// WIDE (many CTAs per start, e.g. S = 1): the last CTA to finish sums all CTA
// partials with all of its warps — warp w sums CTAs [w per, (w+1) per) in CTA
// order (one L2 round trip for up to 8 x 24 CTAs), then warp 0 sums the warp
// sums in warp order: deterministic, one ticket on the critical path (C5:
// 2.7 -> 0.95 us per gate).  A separate instantiation, so the few-CTA path
// compiles exactly as before.
template <int NU, int TP0, int TP1, bool UPD, bool WIDE, bool IDENT = false, int NT = BWD_THREADS>
__global__ void __launch_bounds__(NT, NT == BWD_THREADS ? QFS_BWD_MINB : QFS_BWD_HALF_MINB) bwd_kernel(const BwdParams P) {
  __shared__ BwdShared<NT> sh;
  // [BWD_STAGES][8][NT]; 128-byte alignment measured to matter: with
  // static shared memory of 16 * odd bytes in front of it the kernel ran 12 % slower
  extern __shared__ __align__(128) double2 stage_buf[];
  const int jslot = blockIdx.y;
  const Slot sl = P.slots[jslot];
  if constexpr (WIDE) {
    constexpr int NWARP = NT / 32, FL = 24;
    __shared__ unsigned last_cta;
    const bool w0 = bwd_gate_partial<NT, NU, TP0, TP1, UPD, IDENT>(P, P.g, jslot, sl.s, (unsigned)sl.m, sh, stage_buf);
    if (w0) {
      const bool last = warp0_elect_last(&P.counters[jslot], (unsigned)P.nb);
      if (threadIdx.x == 0) last_cta = last ? 1u : 0u;
    }
    __syncthreads();
    if (!last_cta) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (P.dbg && threadIdx.x == 0) atomicMax(P.dbg + 4 * P.g.env_gate + 1, gtimer());
    const int per = (P.nb + NWARP - 1) / NWARP, c0 = warp * per, c1 = min(P.nb, c0 + per);
    const double *pp = P.partials + (long long)jslot * P.nb * 32 + lane;
    double e = 0.0;
    for (int b0 = c0; b0 < c1; b0 += FL) {
      double xb[FL];
#pragma unroll
      for (int q = 0; q < FL; ++q) xb[q] = b0 + q < c1 ? __ldcg(pp + (long long)(b0 + q) * 32) : 0.0;
#pragma unroll
      for (int q = 0; q < FL; ++q)
        if (b0 + q < c1) e += xb[q];
    }
    double *ws = reinterpret_cast<double *>(sh.red);  // free again: warp 0 has read its CTA partial
    ws[warp * 32 + lane] = e;
    __syncthreads();
    if (warp != 0) return;
    const int kind = P.kinds ? __ldg(P.kinds + P.g.env_gate) : 0;
    e = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) e += ws[w * 32 + lane];
    bwd_finish_e(P, P.g, jslot, sl.s, sh, e, kind);
    return;
  }
  if (!bwd_gate_partial<NT, NU, TP0, TP1, UPD, IDENT>(P, P.g, jslot, sl.s, (unsigned)sl.m, sh, stage_buf))
    return;
  const int kind = P.kinds ? __ldg(P.kinds + P.g.env_gate) : 0;
  const int ng = (P.nb + RED_GS - 1) / RED_GS;
  if (ng <= 1 || !P.counters1) {
    if (!warp0_elect_last(&P.counters[jslot], (unsigned)P.nb)) return;
    bwd_finish(P, P.g, jslot, sl.s, sh, kind);
    return;
  }
  // two-level ordered reduction of the CTA partials (many CTAs per start, e.g.
  // S = 1): the last CTA of each group of RED_GS CTAs sums its group in CTA
  // order, the last group to finish sums the group sums in group order — two
  // L2 round trips on the critical path instead of nb / 48
  const int lane = threadIdx.x;
  const int g = blockIdx.x / RED_GS, g0 = g * RED_GS, gsz = min(RED_GS, P.nb - g0);
  if (!warp0_elect_last(&P.counters1[jslot * RED_GMAX + g], (unsigned)gsz)) return;
  if (P.dbg && lane == 0) atomicMax(P.dbg + 4 * P.g.env_gate + 1, gtimer());
  const double *pp = P.partials + ((long long)jslot * P.nb + g0) * 32 + lane;
  double xb[RED_GS];
#pragma unroll
  for (int q = 0; q < RED_GS; ++q) xb[q] = q < gsz ? __ldcg(pp + (long long)q * 32) : 0.0;
  double e = 0.0;
#pragma unroll
  for (int q = 0; q < RED_GS; ++q)
    if (q < gsz) e += xb[q];
  P.gpartials[((long long)jslot * RED_GMAX + g) * 32 + lane] = e;
  if (!warp0_elect_last(&P.counters[jslot], (unsigned)ng)) return;
  const double *gp = P.gpartials + (long long)jslot * RED_GMAX * 32 + lane;
  double yb[RED_GMAX];
#pragma unroll
  for (int q = 0; q < RED_GMAX; ++q) yb[q] = q < ng ? __ldcg(gp + (long long)q * 32) : 0.0;
  e = 0.0;
#pragma unroll
  for (int q = 0; q < RED_GMAX; ++q)
    if (q < ng) e += yb[q];
  bwd_finish_e(P, P.g, jslot, sl.s, sh, e, kind);
}


// ------------------------------------------------- backward, bulk-copy path --
// bwdt_kernel: the same fused step as bwd_kernel (chi <- G_{i+1}^dag chi, E_i,
// last-CTA ordered reduction + polar update of gate i; P:112, P:121-125,
// P:172, eq:opt_u P:59-62), with the tiles moved by the copy engine (B200:
// cp.async.bulk -> SASS UBLKCP, mbarrier -> SYNCS) instead of per-thread LDGSTS.
//
// Layouts (perm mode, qfs_internal.h): B_i and the incoming chi are stored in
// gate i's permuted sample-blocked layout L_i, whose lowest row bits are the
// 2^NU-row union of gates i and i+1 — so a work unit ("stage": one amplitude
// group x one block of sb <= 32 samples) is ONE contiguous 2^NU * sb * 16-byte
// run per array (8 KB at NU = 4, sb = 32): one bulk copy for chi and one for
// phi, where the natural sample-minor layout needed 2^NU row copies of 512 B
// (measured: 512-byte bulk copies are bound by the copy engine's issue rate,
// 3x slower than LDGSTS).  The natural pools (x as phi at i = 0, y as chi at
// i >= K-2) still come row by row.  The updated chi is stored by the
// consumers, one coalesced 32-sample row per STG, straight into the NEXT
// gate's layout L_{i-1} (rows: the Scatter of G and v), so the next launch's
// tiles are contiguous too.
//
// One producer warp fills a ring of BT_STAGES stages (full / empty mbarrier
// pair per stage); consumer warp w owns the stages w, w + BT_CW, ...; lane =
// one sample, all 2^NU amplitudes of it in registers: the chi update and all
// 16 entries of E are lane-local (no transposes, no shuffles; 16 independent
// accumulators).  phi does not depend on the previous launch: with G.pre the
// producer issues the first stages' phi before griddepcontrol.wait (PDL), and
// prefetches phi BT_PF stages ahead into L2 (cp.async.bulk.prefetch.L2).
#ifndef QFS_BT_WARPS
#define QFS_BT_WARPS 6   // + 1 producer = 224 threads: up to 255 registers (8 consumers cap at 168 and spill)
#endif
#ifndef QFS_BT_STAGES
#define QFS_BT_STAGES 12
#endif
#ifndef QFS_BT_PF
#define QFS_BT_PF 4       // phi prefetched into L2 this many stages ahead (0: off)
#endif
#ifndef QFS_BT_HINT
#define QFS_BT_HINT 1     // bit 0: phi (B_i, read once) copies L2::evict_first
#endif
constexpr int BT_CW = QFS_BT_WARPS;           // consumer warps
constexpr int BT_STAGES = QFS_BT_STAGES;
constexpr int BT_THREADS = (BT_CW + 1) * 32;  // + one producer warp
constexpr int BT_SROW = 32;                   // largest sample block (one sample per lane)
// Consumer warp w owns the ring slots w, w + BT_CW, ...: a slot's full barrier
// is then waited on by ONE warp in consecutive rounds, so its phase parity is
// never ambiguous (a warp waiting on a slot two phases ahead of the barrier
// would pass at once — mbarrier parity waits only distinguish adjacent phases).
static_assert(BT_STAGES % BT_CW == 0, "each consumer warp must own whole ring slots");

#ifndef QFS_BT_EARLY
// 1: consumers copy a whole stage (chi and phi) into registers and release the
// slot BEFORE computing (deeper copy pipeline; G^dag from shared memory):
// measured C4 21.1 -> 22.7 us (255 registers, spills), C5 16.5 -> 14.2 us — off
#define QFS_BT_EARLY 0
#endif
struct BtShared {
  uint64_t full[BT_STAGES], empty[BT_STAGES];
  double2 sQ[BT_CW][16];  // QFS_BT_EARLY: G_{i+1}^dag, one copy per consumer warp
  double2 red[BT_CW][16];
  double wsum[(BT_CW + 1) * 32];  // WIDE reduction: per-warp sums of CTA partials
  double sum32[32];
  double2 scratch[64];
  unsigned last_cta;
};

}  // namespace
size_t bt_smem_bytes(int nu) { return (size_t)BT_STAGES * 2 * (1 << nu) * BT_SROW * sizeof(double2); }
namespace {

// destination row of group G, local v (perm-mode scatter)
__device__ __forceinline__ unsigned scatter_base(const Scatter &X, unsigned G, int n_oth) {
  unsigned p = 0;
  for (int j = 0; j < n_oth; ++j) p |= ((G >> j) & 1u) << X.dpos[j];
  return p;
}

template <int NU, int TP0, int TP1, bool UPD, bool WIDE>
__global__ void __launch_bounds__(BT_THREADS, 1) bwdt_kernel(const BwdParams P) {
  constexpr int NV = 1 << NU;
  constexpr int NQ = NV / 4;
  __shared__ BtShared sh;
  extern __shared__ __align__(128) double2 ring[];
  const GateDesc &G = P.g;
  const int jslot = blockIdx.y;
  const Slot sl = P.slots[jslot];
  const int s = sl.s;
  const unsigned Ms = (unsigned)sl.m;
  const int sb = G.sb;                     // sample block (16 or 32)
  const int STAGE = 2 * NV * sb;           // double2 per stage: [chi | phi][v][sb]
  const unsigned nmb = (Ms + sb - 1) / sb;
  const unsigned units = (1u << (P.n - NU)) * nmb;
  const unsigned chunk = (units + P.nb - 1) / P.nb;
  const unsigned beg = min(units, blockIdx.x * chunk), end = min(units, beg + chunk);
  const int nitems = (int)(end - beg);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const FastDiv fdu(nmb);
  // group index G (other bits, ascending) and sample block b of item k
  auto item = [&](int k, unsigned &Gi, unsigned &b) {
    const unsigned u = beg + (unsigned)k;
    Gi = fdu.div(u);
    b = u - Gi * nmb;
  };
  if (threadIdx.x == 0) {
    for (int q = 0; q < BT_STAGES; ++q) {
      mbar_init(&sh.full[q], 1);
      mbar_init(&sh.empty[q], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == BT_CW) {
    // ------------------------------------------------------------ producer
    const double2 *csrc = G.chi_src.base + (long long)s * G.chi_src.ss;
    const double2 *fsrc = G.phi.base + (long long)s * G.phi.ss;
#if QFS_BT_HINT & 1
    const uint64_t pol_f = policy_evict_first();
#endif
    uint32_t ins[NU];
#pragma unroll
    for (int q = 0; q < NU; ++q) ins[q] = G.ins[q];
    const int v = lane & (NV - 1);
    const long long offv = G.off[v];
    // lane l < NV: natural chi row l, NV <= l < 2 NV: natural phi row l - NV;
    // lane 0 / 1: the single permuted chi / phi run
    auto issue = [&](int k, bool chi, bool phi) {
      unsigned Gi, b;
      item(k, Gi, b);
      const unsigned cnt = min((unsigned)sb, Ms - b * sb);
      double2 *stg = ring + (k % BT_STAGES) * STAGE;
      uint64_t *bar = &sh.full[k % BT_STAGES];
      unsigned g = Gi;
#pragma unroll
      for (int q = 0; q < NU; ++q) g = insert_zero32(g, ins[q]);
      if (chi) {
        if (G.chi_nat) {
          if (lane < NV)
            bulk_g2s(stg + v * sb, csrc + ((long long)g + offv) * G.chi_src.sa + b * sb, cnt * 16u, bar);
        } else if (lane == 0) {
          bulk_g2s(stg, csrc + (long long)b * G.blk + ((long long)Gi << NU) * sb, NV * sb * 16u, bar);
        }
      }
      if (phi) {
        double2 *dst = stg + NV * sb;
        if (G.phi_nat) {
          if (lane >= NV && lane < 2 * NV)
            bulk_g2s(dst + v * sb, fsrc + ((long long)g + offv) * G.phi.sa + b * sb, cnt * 16u, bar);
        } else if (lane == 1) {
          const double2 *src = fsrc + (long long)b * G.blk + ((long long)Gi << NU) * sb;
#if QFS_BT_HINT & 1
          bulk_g2s_hint(dst, src, NV * sb * 16u, bar, pol_f);
#else
          bulk_g2s(dst, src, NV * sb * 16u, bar);
#endif
        }
      }
    };
    auto arm = [&](int k) {  // expect the stage's bytes (chi and phi)
      if (lane == 0) {
        unsigned Gi, b;
        item(k, Gi, b);
        const unsigned cnt = min((unsigned)sb, Ms - b * sb);
        const unsigned bytes = ((G.chi_nat ? cnt : (unsigned)sb) + (G.phi_nat ? cnt : (unsigned)sb)) * NV * 16u;
        mbar_arrive_tx(&sh.full[k % BT_STAGES], bytes);
      }
      __syncwarp();
    };
    auto prefetch = [&](int k) {
#if QFS_BT_PF
      if (k < nitems && lane == 0 && !G.phi_nat) {
        unsigned Gi, b;
        item(k, Gi, b);
        bulk_prefetch_l2(fsrc + (long long)b * G.blk + ((long long)Gi << NU) * sb, NV * sb * 16u);
      }
#endif
    };
    const int npre = min(nitems, BT_STAGES);
    if (G.pre) {  // phi of the first stages before the dependence on the previous launch
      for (int k = 0; k < npre; ++k) {
        arm(k);
        issue(k, false, true);
      }
      for (int k = npre; k < npre + QFS_BT_PF; ++k) prefetch(k);
    }
    pdl_wait();
    for (int k = 0; k < npre; ++k) {
      if (!G.pre) arm(k);
      issue(k, true, !G.pre);
    }
    if (!G.pre)
      for (int k = npre; k < npre + QFS_BT_PF; ++k) prefetch(k);
    for (int k = npre; k < nitems; ++k) {
      prefetch(k + QFS_BT_PF);
      mbar_wait(&sh.empty[k % BT_STAGES], ((k / BT_STAGES) - 1) & 1);
      arm(k);
      issue(k, true, true);
    }
  } else {
    // ------------------------------------------------------------ consumers
    pdl_wait();  // G_{i+1} was written by the previous launch's polar update
#if QFS_BT_EARLY
    // G_{i+1}^dag in this warp's shared-memory copy (registers go to the stage copy)
    if (UPD && lane < 16) {
      const int a = lane >> 2, b = lane & 3;  // (G^dag)[a][b] = conj(G[b][a])
      sh.sQ[warp][lane] = cconj(__ldcg(P.gates + ((long long)s * P.K + G.upd_gate) * 16 + 4 * b + a));
    }
    __syncwarp();
#define QFS_BTQ(e) lds_v2(&sh.sQ[warp][e])
#else
    double2 Q[16];
    if (UPD) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)  // (G^dag)[a][b] = conj(G[b][a])
          Q[4 * a + b] = cconj(__ldcg(P.gates + ((long long)s * P.K + G.upd_gate) * 16 + 4 * b + a));
    }
#define QFS_BTQ(e) Q[e]
#endif
    double2 *cdst = G.chi_dst.base ? G.chi_dst.base + (long long)s * G.chi_dst.ss : nullptr;
    double2 acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = make_double2(0.0, 0.0);
    for (int k = warp; k < nitems; k += BT_CW) {
      unsigned Gi, b;
      item(k, Gi, b);
      const bool valid = lane < sb && b * sb + lane < Ms;
      mbar_wait(&sh.full[k % BT_STAGES], (k / BT_STAGES) & 1);
      const double2 *sc = ring + (k % BT_STAGES) * STAGE + lane;
      double2 c[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) c[v] = valid ? sc[v * sb] : make_double2(0.0, 0.0);
#if QFS_BT_EARLY
      double2 fr[NV];  // phi too, then the slot goes back to the producer before any arithmetic
#pragma unroll
      for (int v = 0; v < NV; ++v) fr[v] = valid ? sc[(NV + v) * sb] : make_double2(0.0, 0.0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[k % BT_STAGES]);
#endif
      if (UPD) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          double2 o[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            o[a] = make_double2(0.0, 0.0);
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) cfma(o[a], QFS_BTQ(4 * a + bb), c[4 * q + bb]);
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) c[4 * q + a] = o[a];
        }
        if (cdst && valid) {  // into the next gate's layout L_{i-1}
          const unsigned pg = scatter_base(G.xs, Gi, G.n_oth);
          double2 *dp = cdst + (long long)b * G.blk + lane;
#pragma unroll
          for (int v = 0; v < NV; ++v) dp[(long long)(pg | (unsigned)G.xs.dv[v]) * sb] = c[v];
        }
      }
      // E[l_in][l_out] += phi[v(p, l_in)] conj(chi'[v(p, l_out)]) over the P-quadruples p
#pragma unroll
      for (int p = 0; p < NQ; ++p) {
        double2 f[4];
#pragma unroll
        for (int l = 0; l < 4; ++l)
#if QFS_BT_EARLY
          f[l] = fr[pv_idx<NU, TP0, TP1>(p, l)];
#else
          f[l] = valid ? sc[(NV + pv_idx<NU, TP0, TP1>(p, l)) * sb] : make_double2(0.0, 0.0);
#endif
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int bb = 0; bb < 4; ++bb) {
            const double2 cb = c[pv_idx<NU, TP0, TP1>(p, bb)];
            double2 &e = acc[4 * a + bb];
            e.x = fma(f[a].x, cb.x, e.x);
            e.x = fma(f[a].y, cb.y, e.x);
            e.y = fma(f[a].y, cb.x, e.y);
            e.y = fma(-f[a].x, cb.y, e.y);
          }
      }
#if !QFS_BT_EARLY
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[k % BT_STAGES]);
#endif
    }
#undef QFS_BTQ
    // warp sum over the samples (fixed butterfly order)
#pragma unroll
    for (int e = 0; e < 16; ++e) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        acc[e].x += __shfl_xor_sync(FULL, acc[e].x, o);
        acc[e].y += __shfl_xor_sync(FULL, acc[e].y, o);
      }
    }
    if (lane < 16) {
      double2 w = acc[0];
#pragma unroll
      for (int e = 1; e < 16; ++e)
        if (lane == e) w = acc[e];
      sh.red[warp][lane] = w;
    }
  }
  pdl_trigger();
  __syncthreads();
  // CTA partial: consumer warps in order (warp 0, lane = re / im of entry lane / 2)
  if (warp == 0) {
    const int e = lane >> 1, im = lane & 1;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < BT_CW; ++w) v += im ? sh.red[w][e].y : sh.red[w][e].x;
    P.partials[((long long)jslot * P.nb + blockIdx.x) * 32 + lane] = v;
  }
  const int kind = P.kinds ? __ldg(P.kinds + G.env_gate) : 0;
  if constexpr (WIDE) {
    constexpr int NW = BT_CW + 1, FL = 24;
    if (warp == 0) {
      const bool last = warp0_elect_last(&P.counters[jslot], (unsigned)P.nb);
      if (lane == 0) sh.last_cta = last ? 1u : 0u;
    }
    __syncthreads();
    if (!sh.last_cta) return;
    const int per = (P.nb + NW - 1) / NW, c0 = warp * per, c1 = min(P.nb, c0 + per);
    const double *pp = P.partials + (long long)jslot * P.nb * 32 + lane;
    double e = 0.0;
    for (int b0 = c0; b0 < c1; b0 += FL) {
      double xb[FL];
#pragma unroll
      for (int q = 0; q < FL; ++q) xb[q] = b0 + q < c1 ? __ldcg(pp + (long long)(b0 + q) * 32) : 0.0;
#pragma unroll
      for (int q = 0; q < FL; ++q)
        if (b0 + q < c1) e += xb[q];
    }
    double *ws = sh.wsum;
    ws[warp * 32 + lane] = e;
    __syncthreads();
    if (warp != 0) return;
    e = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) e += ws[w * 32 + lane];
    bwd_finish_e(P, G, jslot, s, sh, e, kind);
  } else {
    if (warp != 0) return;
    if (!warp0_elect_last(&P.counters[jslot], (unsigned)P.nb)) return;
    const double *pp = P.partials + (long long)jslot * P.nb * 32 + lane;
    double e = 0.0;
    constexpr int FLIGHT = 16;
    for (int b0 = 0; b0 < P.nb; b0 += FLIGHT) {
      double xb[FLIGHT];
#pragma unroll
      for (int q = 0; q < FLIGHT; ++q) xb[q] = b0 + q < P.nb ? __ldcg(pp + (long long)(b0 + q) * 32) : 0.0;
#pragma unroll
      for (int q = 0; q < FLIGHT; ++q)
        if (b0 + q < P.nb) e += xb[q];
    }
    bwd_finish_e(P, G, jslot, s, sh, e, kind);
  }
}

// polar step alone (sample-sharded mode, after the NCCL all-reduce of E): one warp per start
__global__ void polar_kernel(const PolarParams P) {
  __shared__ double e32[4][32];
  __shared__ double2 scratch[4][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + w;
  pdl_wait();
  if (j >= P.n_slots) return;
  const Slot sl = P.slots[j];
  e32[w][lane] = P.e_red[(long long)j * 32 + lane];
  __syncwarp();
  const long long gi = (long long)sl.s * P.K + P.gate;
  polar_write(e32[w], P.gates + gi * 16, P.vprev ? P.vprev + gi * 16 : nullptr, P.beta,
              P.kinds ? P.kinds[P.gate] : 0, P.sig ? P.sig + gi : nullptr,
              P.env_trace ? P.env_trace + ((long long)P.gate * P.S + sl.s) * 16 : nullptr, scratch[w]);
}

// --------------------------------------------------------------- final cost --
__global__ void __launch_bounds__(RED_THREADS, 4) final_kernel(const FinalParams P) {
  __shared__ double2 sQ[16];
  __shared__ double red[RED_THREADS / 32];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned Ms = (unsigned)sl.m;
  const unsigned items = Ms << (P.n - 2);
  const unsigned chunk = (items + P.nb - 1) / P.nb;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fdm(Ms);
  pdl_wait();
  if (threadIdx.x < 16) {
    const int a = threadIdx.x >> 2, b = threadIdx.x & 3;
    sQ[threadIdx.x] = cconj(P.gates[(long long)s * P.K * 16 + 4 * b + a]);
  }
  __syncthreads();
  const int lo = min(P.p0, P.p1), hi = max(P.p0, P.p1);
  const unsigned o[4] = {0u, 1u << P.p0, 1u << P.p1, (1u << P.p0) | (1u << P.p1)};
  const double2 *cb = P.chi.base + (long long)s * P.chi.ss;
  const double2 *xb = P.x.base + (long long)s * P.x.ss;
  double acc = 0.0;
  for (unsigned w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const unsigned q = fdm.div(w);
    const unsigned m = w - q * Ms;
    const unsigned base = insert_zero32(insert_zero32(q, lo), hi);
    const double2 *xp = P.x.ident ? nullptr : xb + (long long)base * P.x.sa + (long long)m * P.x.sm;
    double2 v[4], xv[4];
    if (P.sb > 0) {  // perm mode: chi sample-blocked, natural rows (layout L_{-1})
      const double2 *cp = cb + (long long)(m / P.sb) * P.blk + (long long)base * P.sb + m % P.sb;
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] = cp[(long long)o[l] * P.sb];
    } else {
      const double2 *cp = cb + (long long)base * P.chi.sa + (long long)m * P.chi.sm;
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] = cp[(long long)o[l] * P.chi.sa];
    }
#pragma unroll
    for (int l = 0; l < 4; ++l)
      xv[l] = P.x.ident ? make_double2(base + o[l] == m ? 1.0 : 0.0, 0.0) : __ldcs(xp + (long long)o[l] * P.x.sa);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 r = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(r, sQ[4 * a + b], v[b]);
      const double dr = r.x - xv[a].x, di = r.y - xv[a].y;
      acc = fma(dr, dr, acc);
      acc = fma(di, di, acc);
    }
  }
  pdl_trigger();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(FULL, acc, q);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    P.partials[(long long)j * P.nb + blockIdx.x] = t;
  }
  if (!warp0_elect_last(&P.counters[j], (unsigned)P.nb)) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < P.nb; ++b) t += __ldcg(P.partials + (long long)j * P.nb + b);
    P.out_sum[j] = t;
  }
}


// ------------------------------------------------------ forward (per gate) --
// B_{k+1} = G_k B_k for every (quadruple, sample) of every active start.
__global__ void __launch_bounds__(FWD_THREADS, 3) fwd_gate_kernel(const FwdGateParams P) {
  __shared__ double2 sG[16];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned Ms = (unsigned)(P.rows_fixed > 0 ? P.rows_fixed : sl.m);
  const unsigned items = Ms << (P.n - 2);
  const unsigned chunk = (items + P.nb - 1) / P.nb;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fdm(Ms);
  pdl_wait();
  if (threadIdx.x < 16) sG[threadIdx.x] = P.gates[((long long)s * P.K + P.k) * 16 + threadIdx.x];
  __syncthreads();
  const int lo = min(P.p0, P.p1), hi = max(P.p0, P.p1);
  const long long so1 = (1LL << P.p0) * P.src.sa, so2 = (1LL << P.p1) * P.src.sa;
  const long long do1 = (1LL << P.p0) * P.dst.sa, do2 = (1LL << P.p1) * P.dst.sa;
  const long long soff[4] = {0, so1, so2, so1 + so2}, doff[4] = {0, do1, do2, do1 + do2};
  const double2 *src = P.src.base + (long long)s * P.src.ss;
  double2 *dst = P.dst.base + (long long)s * P.dst.ss;
  // LDGSTS pipeline (FWD_STAGES-1 items ahead per thread, own slots only)
  extern __shared__ __align__(128) double2 fstage[];  // [FWD_STAGES][4][FWD_THREADS]
  const unsigned stride = blockDim.x;
  const int iters = beg + threadIdx.x < end ? (int)((end - beg - threadIdx.x + stride - 1) / stride) : 0;
  auto locate = [&](int k, unsigned &base, unsigned &m) -> bool {
    const unsigned w = beg + threadIdx.x + (unsigned)k * stride;
    if (k >= iters) return false;
    const unsigned q = fdm.div(w);
    m = w - q * Ms;
    base = insert_zero32(insert_zero32(q, lo), hi);
    return true;
  };
  const uint64_t pol_ld = policy_evict_first(), pol_st = policy_evict_last();
  const int cm = P.cache_mode;
  auto issue = [&](int k) {
    unsigned base = 0, m = 0;
    const bool ok = locate(k, base, m);
    double2 *stp = fstage + (k % FWD_STAGES) * 4 * FWD_THREADS + threadIdx.x;
    const double2 *sp = src + (long long)base * P.src.sa + (long long)m * P.src.sm;
    if (P.src.ident) {  // implicit basis x_m = e_m
      const unsigned ob[4] = {0u, 1u << P.p0, 1u << P.p1, (1u << P.p0) | (1u << P.p1)};
#pragma unroll
      for (int l = 0; l < 4; ++l) stp[l * FWD_THREADS] = make_double2(ok && base + ob[l] == m ? 1.0 : 0.0, 0.0);
    } else if (cm & 2) {
#pragma unroll
      for (int l = 0; l < 4; ++l) cp_async16_hint(stp + l * FWD_THREADS, ok ? sp + soff[l] : src, ok, pol_ld);
    } else {
#pragma unroll
      for (int l = 0; l < 4; ++l) cp_async16(stp + l * FWD_THREADS, ok ? sp + soff[l] : src, ok);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int k = 0; k < FWD_STAGES - 1; ++k) issue(k);
  for (int k = 0; k < iters; ++k) {
    issue(k + FWD_STAGES - 1);
    cp_async_wait<FWD_STAGES - 1>();
    unsigned base = 0, m = 0;
    locate(k, base, m);
    const double2 *stp = fstage + (k % FWD_STAGES) * 4 * FWD_THREADS + threadIdx.x;
    double2 v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = stp[l * FWD_THREADS];
    double2 *dp = dst + (long long)base * P.dst.sa + (long long)m * P.dst.sm;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 r = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(r, sG[4 * a + b], v[b]);
      if (cm & 1) st_hint(dp + doff[a], r, pol_st);
      else dp[doff[a]] = r;
    }
  }
  cp_async_wait<0>();
  pdl_trigger();
}

// ---------------------------------------------- forward, two gates per pass --
// B_{k+1} = G_k B_k and B_{k+2} = G_{k+1} B_{k+1} in one pass: one thread per
// (2^NU-amplitude group spanned by both pairs, sample), sample fastest (coalesced
// warp accesses for any pair).  Local bits 0,1 = gate k's pair; gate k+1's pair
// sits at local (TP0, TP1).  Per amplitude: 16 B read, 32 B written, instead of
// 32 B read and 32 B written by two single-gate passes.
// Gate entry from shared memory.  With QFS_FWD2_MINB > 1 the load is volatile
// so it is re-issued per use (a broadcast LDS) instead of hoisted: hoisting
// both gates costs 128 registers and pins the kernel at one CTA per SM.
__device__ __forceinline__ double2 gval(const double2 *p) {
#if QFS_FWD2_MINB > 1 || QFS_FWD2_GSMEM
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
#else
  return *p;
#endif
}

template <int NU, int TP0, int TP1, bool IDENT = false>
__global__ void __launch_bounds__(FWD2_THREADS, QFS_FWD2_MINB) fwd2_kernel(const Fwd2Params P) {
  constexpr int NV = 1 << NU;
  constexpr int NQ = NV / 4;
  __shared__ double2 sG[2][16];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned Ms = (unsigned)sl.m;
  const unsigned items = Ms << (P.n - NU);
  const unsigned chunk = (items + P.nb - 1) / P.nb;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fdm(Ms);
  pdl_wait();
  if (threadIdx.x < 32) {
    const int q = threadIdx.x >> 4, e = threadIdx.x & 15;
    sG[q][e] = P.gates[((long long)s * P.K + P.k + q) * 16 + e];
  }
  __syncthreads();
  const double2 *src = P.src.base + (long long)s * P.src.ss;
  double2 *d1 = P.dst1.base + (long long)s * P.dst1.ss;
  double2 *d2 = P.dst2.base + (long long)s * P.dst2.ss;
  const unsigned ssa = (unsigned)P.src.sa, dsa = (unsigned)P.dst1.sa;
  uint32_t ins[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) ins[q] = P.ins[q];
  auto locate = [&](unsigned w) {  // (first amplitude, sample) of item w
    unsigned g = fdm.div(w);
    const unsigned m = w - g * Ms;
#pragma unroll
    for (int q = 0; q < NU; ++q) g = insert_zero32(g, ins[q]);
    QFS_DASSERT(P.src.ident || (unsigned long long)(g + (unsigned)P.off[(1 << NU) - 1]) * ssa + m < ((unsigned long long)ssa << P.n));
    return make_uint2(g, m);
  };
#if QFS_FWD2_HINT
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
#endif
  auto load = [&](unsigned w, double2 *v) {
    const uint2 gm = locate(w);
    if (IDENT) {  // implicit basis x_m = e_m (the first pass of a QF sweep)
#pragma unroll
      for (int u = 0; u < NV; ++u) v[u] = make_double2(gm.x + (unsigned)P.off[u] == gm.y ? 1.0 : 0.0, 0.0);
      return;
    }
    const double2 *sp = src + (gm.x * ssa + gm.y);
#pragma unroll
    for (int u = 0; u < NV; ++u) {
#if QFS_FWD2_HINT & 4
      v[u] = ld_hint(sp + (unsigned)P.off[u] * ssa, pol_first);
#else
      v[u] = sp[(unsigned)P.off[u] * ssa];
#endif
    }
  };
  auto store = [&](double2 *p, const double2 *v, int which) {
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      double2 *q = p + (unsigned)P.off[u] * dsa;
#if QFS_FWD2_HINT & 3
      if ((QFS_FWD2_HINT & 1) && which == 1) st_hint(q, v[u], pol_first);
      else if ((QFS_FWD2_HINT & 2) && which == 2) st_hint(q, v[u], pol_last);
      else *q = v[u];
#else
      *q = v[u];
#endif
    }
  };
  double2 v[NV];
#if QFS_FWD2_PF
  double2 vn[NV];
  if (beg + threadIdx.x < end) load(beg + threadIdx.x, vn);
#endif
  for (unsigned w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const uint2 gm = locate(w);  // recomputed (cheap) instead of carried in registers
    const unsigned o = gm.x * dsa + gm.y;
#if QFS_FWD2_PF
#pragma unroll
    for (int u = 0; u < NV; ++u) v[u] = vn[u];
    if (w + blockDim.x < end) load(w + blockDim.x, vn);  // next item's loads in flight during this one
#else
    load(w, v);
#endif
    // gate k on local bits (0,1)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double2 o4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o4[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o4[a], gval(&sG[0][4 * a + b]), v[4 * q + b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) v[4 * q + a] = o4[a];
    }
    store(d1 + o, v, 1);
    // gate k+1 on local bits (TP0, TP1)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double2 o4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o4[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o4[a], gval(&sG[1][4 * a + b]), v[pv_idx<NU, TP0, TP1>(q, b)]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) v[pv_idx<NU, TP0, TP1>(q, a)] = o4[a];
    }
    store(d2 + o, v, 2);
  }
  pdl_trigger();
}

// ------------------------------------------- forward, perm-mode layouts --
// fwdp_kernel: fwd2_kernel's two gates per pass (B_{k+1} = G_k B_k, B_{k+2} =
// G_{k+1} B_{k+1}) on the layout-permuted sample-blocked arrays of
// perm mode (qfs_internal.h): the source group's 2^NU rows are contiguous in
// B_k's layout L_k (row G 2^NU + tau[v]; at k = 0 the natural x pool through
// ins / off), and each destination row is scattered into the layout of the
// gate that will read it (B_{k+1} in L_{k+1}, B_{k+2} in L_{k+2}) — the layout
// the backward kernel's single contiguous bulk copies need.  The scatter of
// the group index G is a byte-wise table lookup in shared memory (3 x 256
// entries per destination, built before the PDL wait).  dst2.base == nullptr:
// gate k only (the odd tail of the forward pass).
template <int NU, int TP0, int TP1>
__global__ void __launch_bounds__(FWD_THREADS, 1) fwdp_kernel(const FwdpParams P) {
  constexpr int NV = 1 << NU;
  constexpr int NQ = NV / 4;
  __shared__ double2 sG[2][16];
  __shared__ unsigned tab[2][3][256];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned Ms = (unsigned)sl.m;
  const unsigned items = Ms << (P.n - NU);
  const unsigned chunk = (items + P.nb - 1) / P.nb;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fdm(Ms);
  const bool two = P.dst2.base != nullptr;
  for (int e = threadIdx.x; e < 2 * 3 * 256; e += blockDim.x) {  // scatter tables (launch constants)
    const int d = e / 768, byte = (e >> 8) % 3, val = e & 255;
    const Scatter &X = d ? P.s2 : P.s1;
    unsigned p = 0;
    for (int bit = 0; bit < 8; ++bit) {
      const int jj = byte * 8 + bit;
      if (jj < P.n_oth && ((val >> bit) & 1)) p |= 1u << X.dpos[jj];
    }
    tab[d][byte][val] = p;
  }
  pdl_wait();
  if (threadIdx.x < 32) {
    const int q = threadIdx.x >> 4, e = threadIdx.x & 15;
    sG[q][e] = P.gates[((long long)s * P.K + P.k + q) * 16 + e];
  }
  __syncthreads();
  const double2 *src = P.src.base + (long long)s * P.src.ss;
  double2 *d1 = P.dst1.base + (long long)s * P.dst1.ss;
  double2 *d2 = two ? P.dst2.base + (long long)s * P.dst2.ss : nullptr;
  const int sb = P.sb, lsb = sb == 32 ? 5 : 4;
  const long long blk = P.blk;
  uint32_t ins[NU];
#pragma unroll
  for (int q = 0; q < NU; ++q) ins[q] = P.ins[q];
#if QFS_FWD2_HINT
  const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
#endif
  auto load = [&](unsigned w, double2 *v) {
    const unsigned G = fdm.div(w), m = w - G * Ms;
    if (P.src_nat) {
      unsigned g = G;
#pragma unroll
      for (int q = 0; q < NU; ++q) g = insert_zero32(g, ins[q]);
      const double2 *sp = src + (long long)g * P.src.sa + m;
#pragma unroll
      for (int u = 0; u < NV; ++u) v[u] = sp[P.off[u] * P.src.sa];
    } else {
      const double2 *sp = src + (long long)(m >> lsb) * blk + ((long long)G << NU) * sb + (m & (sb - 1));
#pragma unroll
      for (int u = 0; u < NV; ++u) v[u] = sp[P.tau[u] * sb];
    }
  };
  auto store = [&](double2 *base, const Scatter &X, const unsigned (&tb)[3][256], unsigned G, unsigned m,
                   const double2 *v, int which) {
    const unsigned pg = tb[0][G & 255u] | tb[1][(G >> 8) & 255u] | tb[2][G >> 16];
    double2 *bp = base + (long long)(m >> lsb) * blk + (m & (sb - 1));
#pragma unroll
    for (int u = 0; u < NV; ++u) {
      double2 *q = bp + (long long)(pg | (unsigned)X.dv[u]) * sb;
#if QFS_FWD2_HINT & 3
      if ((QFS_FWD2_HINT & 1) && which == 1) st_hint(q, v[u], pol_first);
      else if ((QFS_FWD2_HINT & 2) && which == 2) st_hint(q, v[u], pol_last);
      else *q = v[u];
#else
      *q = v[u];
#endif
    }
  };
  double2 v[NV], vn[NV];
  if (beg + threadIdx.x < end) load(beg + threadIdx.x, vn);
  for (unsigned w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const unsigned G = fdm.div(w), m = w - G * Ms;
#pragma unroll
    for (int u = 0; u < NV; ++u) v[u] = vn[u];
    if (w + blockDim.x < end) load(w + blockDim.x, vn);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {  // gate k on local bits (0, 1)
      double2 o4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o4[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o4[a], gval(&sG[0][4 * a + b]), v[4 * q + b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) v[4 * q + a] = o4[a];
    }
    store(d1, P.s1, tab[0], G, m, v, 1);
    if (!two) continue;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {  // gate k+1 on local bits (TP0, TP1)
      double2 o4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o4[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o4[a], gval(&sG[1][4 * a + b]), v[pv_idx<NU, TP0, TP1>(q, b)]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) v[pv_idx<NU, TP0, TP1>(q, a)] = o4[a];
    }
    store(d2, P.s2, tab[1], G, m, v, 2);
  }
  pdl_trigger();
}

// --------------------------------------------------- validation (row in SMEM) --
// One CTA per (start, validation row): the whole 2^n row lives in shared
// memory, the K gates are applied in order (gate k+1 staged while gate k runs),
// then the row's squared distance to yv.
__global__ void __launch_bounds__(VAL_THREADS) val_row_kernel(const ValRowParams P) {
  extern __shared__ __align__(128) double2 row[];
  __shared__ double2 sG[2][16];
  __shared__ double red[VAL_THREADS / 32];
  const int j = blockIdx.y;
  const int s = P.slots[j].s;
  const int m = blockIdx.x;
  const long long N = 1LL << P.n;
  const double2 *src = P.xv + (long long)m * N;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) row[i] = __ldg(src + i);
  pdl_wait();  // the gates are the ones the backward pass just wrote
  const double2 *gs = P.gates + (long long)s * P.K * 16;
  if (threadIdx.x < 16) sG[0][threadIdx.x] = gs[threadIdx.x];
  __syncthreads();
  for (int k = 0; k < P.K; ++k) {
    const int2 pr = __ldg(P.pairs + k);
    const double2 *G = sG[k & 1];
    double2 nxt;
    const bool stage = threadIdx.x < 16 && k + 1 < P.K;
    if (stage) nxt = gs[(long long)(k + 1) * 16 + threadIdx.x];
    const int lo = min(pr.x, pr.y), hi = max(pr.x, pr.y);
    const long long o1 = 1LL << pr.x, o2 = 1LL << pr.y;
    for (long long r = threadIdx.x; r < (N >> 2); r += blockDim.x) {
      const long long base = insert_zero(insert_zero(r, lo), hi);
      const long long off[4] = {base, base | o1, base | o2, base | o1 | o2};
      double2 v[4], o[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) v[l] = row[off[l]];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o[a], G[4 * a + b], v[b]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) row[off[a]] = o[a];
    }
    if (stage) sG[(k + 1) & 1][threadIdx.x] = nxt;
    __syncthreads();
  }
  const double2 *ref = P.yv + (long long)m * N;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) {
    const double2 a = row[i], b = __ldg(ref + i);
    const double dr = a.x - b.x, di = a.y - b.y;
    acc = fma(dr, dr, acc);
    acc = fma(di, di, acc);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(FULL, acc, q);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    P.row_out[(long long)j * P.rows + m] = t;
  }
}

// per-row squared distance (streamed validation end)
__global__ void __launch_bounds__(RED_THREADS) dist_kernel(const DistParams P) {
  __shared__ double red[RED_THREADS / 32];
  const int j = blockIdx.y, m = blockIdx.x;
  pdl_wait();
  const Slot sl = P.slots[j];
  const long long N = 1LL << P.n;
  const double2 *a = P.a.base + (long long)sl.s * P.a.ss + (long long)m * P.a.sm;
  const double2 *b = P.b.base + (long long)sl.s * P.b.ss + (long long)m * P.b.sm;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) {
    const double2 u = a[i * P.a.sa], v = b[i * P.b.sa];
    const double dr = u.x - v.x, di = u.y - v.y;
    acc = fma(dr, dr, acc);
    acc = fma(di, di, acc);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 16; q >= 1; q >>= 1) acc += __shfl_xor_sync(FULL, acc, q);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    P.row_out[(long long)j * P.rows + m] = t;
  }
}

// out[j] = sum_r row_in[j*rows + r], in row order
__global__ void row_reduce_kernel(const double *row_in, int rows, double *out, int n_slots) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (j >= n_slots) return;
  double t = 0.0;
  for (int r = 0; r < rows; ++r) t += row_in[(long long)j * rows + r];
  out[j] = t;
}

// [rows][cols] -> [cols][rows] (pools to the sample-minor layout), 32x32 tiles
__global__ void transpose_kernel(const double2 *src, double2 *dst, int rows, long long cols) {
  __shared__ double2 tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int r = r0 + dy;
    const long long c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = src[(long long)r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long c = c0 + dy;
    const int r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][dy];
  }
}

__global__ void copy_kernel(double2 *dst, const double2 *src, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void copy_words_kernel(unsigned *dst, const unsigned *src, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// End of a sweep: the per-start cost sums (and, once per call, the gate-check
// flag) written straight into mapped pinned host memory, then the sweep's
// sequence number — the host spins on it (run_sweep) instead of a
// device-to-host copy plus a stream synchronisation (C2: ~10 us less per
// controller step).  One CTA; every value store is ordered before the flag by
// the system-scope fence of its own thread and the CTA barrier.
__global__ void publish_kernel(const double *src, int count, const unsigned *check, double *hdst,
                               unsigned *hcheck, unsigned long long *hflag, unsigned long long seq) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) hdst[i] = src[i];
  if (check && threadIdx.x == 0) *hcheck = *check;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) st_release_sys(hflag, seq);
}

// *dst = (*src != 0) ? bit : 0 (one thread): a deferred check's flag moved
// into the word read back after the first sweep
__global__ void flag_bit_kernel(const unsigned *src, unsigned *dst, unsigned bit) { *dst = *src ? bit : 0u; }

__global__ void fill_words_kernel(unsigned *dst, unsigned value, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = value;
}

// Initial-gate validation on the device (one thread per gate): bit 0 a
// non-finite entry, bit 1 ||G^dag G - I||_max > 1e-10, bit 2 a one-qubit slot
// (kind 2) not of the form u (x) I (tol 1e-10).  OR-ed into *flag.
__global__ void gate_check_kernel(const double2 *g, long long count, int K, const int *kinds, unsigned *flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    double2 G[16];
    unsigned bad = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      G[e] = g[i * 16 + e];
      if (!isfinite(G[e].x) || !isfinite(G[e].y)) bad |= 1u;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {  // conj(G[r][a]) G[r][b]
          re += G[4 * r + a].x * G[4 * r + b].x + G[4 * r + a].y * G[4 * r + b].y;
          im += G[4 * r + a].x * G[4 * r + b].y - G[4 * r + a].y * G[4 * r + b].x;
        }
        if (fabs(re - (a == b ? 1.0 : 0.0)) > 1e-10 || fabs(im) > 1e-10) bad |= 2u;
      }
    if (kinds && kinds[i % K] == 2) {
#pragma unroll
      for (int lo = 0; lo < 4; ++lo)
#pragma unroll
        for (int li = 0; li < 4; ++li) {
          const double2 e = G[4 * lo + li];
          if ((lo >> 1) != (li >> 1)) {
            if (fabs(e.x) > 1e-10 || fabs(e.y) > 1e-10) bad |= 4u;
          } else {
            const double2 f = G[4 * (lo ^ 2) + (li ^ 2)];
            if (fabs(e.x - f.x) > 1e-10 || fabs(e.y - f.y) > 1e-10) bad |= 4u;
          }
        }
    }
    if (bad) atomicOr(flag, bad);
  }
}

__global__ void identity_fill_kernel(double2 *v, long long count16) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count16 * 16;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = make_double2((i % 16) % 5 == 0 ? 1.0 : 0.0, 0.0);
}

// non-finite detection over a sample array (ERR_NUMERIC check on the device)
__global__ void finite_check_kernel(const double *p, long long n, int *flag) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(p[i]);
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---------------------------------------------------------------- unit ops --
__global__ void apply_kernel(const ApplyParams P) {
  const long long N = 1LL << P.n;
  const long long items = (long long)P.m << (P.n - 2);
  const int lo = min(P.p0, P.p1), hi = max(P.p0, P.p1);
  const long long o1 = 1LL << P.p0, o2 = 1LL << P.p1;
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < items;
       w += (long long)gridDim.x * blockDim.x) {
    const long long m = w >> (P.n - 2);
    const long long r = w & ((1LL << (P.n - 2)) - 1);
    const long long base = m * N + insert_zero(insert_zero(r, lo), hi);
    const long long off[4] = {base, base | o1, base | o2, base | o1 | o2};
    double2 v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = P.psi[off[l]];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(o, P.g[4 * a + b], v[b]);
      P.psi[off[a]] = o;
    }
  }
}

// two matrices per warp (one per 16-lane half), cold start (V_0 = I)
__global__ void polar_batch_kernel(const double2 *env, const double2 *g_old, double beta,
                                   double2 *g_new, double *sig, int count) {
  __shared__ double2 scratch[4][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, l = lane & 15;
  const int i = (blockIdx.x * 4 + w) * 2 + (lane >> 4);
  const bool valid = i < count;
  const int ii = valid ? i : count - 1;  // keep the whole warp converged
  double2 e = env[(long long)ii * 16 + l];
  if (beta != 0.0) {
    const double2 go = g_old[(long long)ii * 16 + 4 * (l & 3) + (l >> 2)];
    e = make_double2((1.0 - beta) * e.x + beta * go.x, (1.0 - beta) * e.y - beta * go.y);
  }
  double2 g, v;
  double ss;
  hw_polar(e, nullptr, g, v, ss, scratch[w] + 2 * (lane & 16));
  if (valid) {
    g_new[(long long)i * 16 + l] = g;
    if (l == 0) sig[i] = ss;
  }
}

}  // namespace

// ================================================================ launchers ==
namespace {
bool g_pdl = true;
// Launch kernel k<<<grid, block, smem, st>>>(p), with the programmatic
// stream serialization attribute when PDL is on (the kernel may begin while
// the previous one on the stream drains; see pdl_wait / pdl_trigger).
template <class Prm>
cudaError_t launch_ex(void (*k)(Prm), dim3 grid, dim3 block, size_t smem, cudaStream_t st, const Prm &p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, p);
}
}  // namespace
void set_pdl(bool on) { g_pdl = on; }
bool pdl_enabled() { return g_pdl; }
int val_row_max_n() { return 13; }
// LDGSTS backward shape: 128 threads x 2 CTAs per SM when the launch carries
// at least QFS_BWD_HALF_SLOTS starts (C4, 16 starts: bwd 16.0 -> 15.5 us; the
// finer CTAs overlap one another's reduction tail), else 256 x 1 (C5, one
// start: twice the CTA partials on the per-gate critical path, 11.4 -> 13.5 us)
int bwd_threads(int n_slots) { return n_slots >= QFS_BWD_HALF_SLOTS ? 128 : BWD_THREADS; }
int blocks_per_sm(int nt) { return nt == BWD_THREADS ? QFS_BWD_MINB : QFS_BWD_HALF_MINB; }

cudaError_t launch_bwdt(const BwdParams &p, int n_slots, cudaStream_t st) {
  dim3 grid(p.nb, n_slots), block(BT_THREADS);
  const GateDesc &g = p.g;
  const int smem = (int)bt_smem_bytes(g.nu);
#ifndef QFS_BT_WIDE
#define QFS_BT_WIDE 1
#endif
  const bool wide = QFS_BT_WIDE && p.nb > RED_GS;
#define QFS_BT1(NU, A, B, U, W)                                                                  \
  do {                                                                                           \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      cudaFuncSetAttribute(bwdt_kernel<NU, A, B, U, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)bt_smem_bytes(4));                                               \
      attr = true;                                                                               \
    }                                                                                            \
    launch_ex(bwdt_kernel<NU, A, B, U, W>, grid, block, smem, st, p);                            \
  } while (0)
#define QFS_BT(NU, A, B, U)              \
  do {                                   \
    if (wide) QFS_BT1(NU, A, B, U, true); \
    else QFS_BT1(NU, A, B, U, false);    \
  } while (0)
  if (!g.upd) {
    QFS_BT(2, 0, 1, false);
  } else if (g.nu == 2) {
    if (g.tp0 == 0) QFS_BT(2, 0, 1, true);
    else QFS_BT(2, 1, 0, true);
  } else if (g.nu == 3) {
    if (g.tp0 == 0 && g.tp1 == 2) QFS_BT(3, 0, 2, true);
    else if (g.tp0 == 2 && g.tp1 == 0) QFS_BT(3, 2, 0, true);
    else if (g.tp0 == 1 && g.tp1 == 2) QFS_BT(3, 1, 2, true);
    else QFS_BT(3, 2, 1, true);
  } else {
    if (g.tp0 == 2) QFS_BT(4, 2, 3, true);
    else QFS_BT(4, 3, 2, true);
  }
#undef QFS_BT
#undef QFS_BT1
  return cudaGetLastError();
}

int bwdt_units_per_cta_min() { return 4; }

cudaError_t launch_bwd(const BwdParams &p, int n_slots, cudaStream_t st) {
  if (p.bulk) return launch_bwdt(p, n_slots, st);
  const GateDesc &g = p.g;
  // two-CTA-per-SM shape (128 threads; runtime bwd_threads)
  const bool half = p.nt == 128 && BWD_THREADS != 128;
  const int nt = half ? 128 : BWD_THREADS;
  dim3 grid(p.nb, n_slots), block(nt);
  const int smem = BWD_STAGES * 8 * nt * (int)sizeof(double2);
  const bool wide = QFS_WIDE_RED && p.counters1 && (p.nb + RED_GS - 1) / RED_GS > 1;
#define QFS_BWD1N(NU, A, B, U, W, NT)                                                          \
  do {                                                                                         \
    static bool attr = false;                                                                  \
    if (!attr) {                                                                               \
      cudaFuncSetAttribute(bwd_kernel<NU, A, B, U, W, false, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      attr = true;                                                                             \
    }                                                                                          \
    launch_ex(bwd_kernel<NU, A, B, U, W, false, NT>, grid, block, smem, st, p);                \
  } while (0)
#define QFS_BWD1(NU, A, B, U, W)                    \
  do {                                              \
    if (half) QFS_BWD1N(NU, A, B, U, W, 128);       \
    else QFS_BWD1N(NU, A, B, U, W, BWD_THREADS);    \
  } while (0)
#define QFS_BWD1IN(NU, A, B, U, W, NT)                                                         \
  do {                                                                                         \
    static bool attr = false;                                                                  \
    if (!attr) {                                                                               \
      cudaFuncSetAttribute(bwd_kernel<NU, A, B, U, W, true, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      attr = true;                                                                             \
    }                                                                                          \
    launch_ex(bwd_kernel<NU, A, B, U, W, true, NT>, grid, block, smem, st, p);                 \
  } while (0)
#define QFS_BWD1I(NU, A, B, U, W)                   \
  do {                                              \
    if (half) QFS_BWD1IN(NU, A, B, U, W, 128);      \
    else QFS_BWD1IN(NU, A, B, U, W, BWD_THREADS);   \
  } while (0)
  // IDENT: phi is the implicit basis (gate 0 of a QFactor sweep, qfs_set_samples_basis) —
  // its own instantiation so the common kernels keep their register budget
#define QFS_BWD(NU, A, B, U)                                  \
  do {                                                        \
    if (g.phi.ident) {                                        \
      if (wide) QFS_BWD1I(NU, A, B, U, true);                 \
      else QFS_BWD1I(NU, A, B, U, false);                     \
    } else if (wide) QFS_BWD1(NU, A, B, U, true);             \
    else QFS_BWD1(NU, A, B, U, false);                        \
  } while (0)
  if (!g.upd) {
    QFS_BWD(2, 0, 1, false);
  } else if (g.nu == 2) {
    if (g.tp0 == 0) QFS_BWD(2, 0, 1, true);
    else QFS_BWD(2, 1, 0, true);
  } else if (g.nu == 3) {
    if (g.tp0 == 0 && g.tp1 == 2) QFS_BWD(3, 0, 2, true);
    else if (g.tp0 == 2 && g.tp1 == 0) QFS_BWD(3, 2, 0, true);
    else if (g.tp0 == 1 && g.tp1 == 2) QFS_BWD(3, 1, 2, true);
    else QFS_BWD(3, 2, 1, true);
  } else {
    if (g.tp0 == 2) QFS_BWD(4, 2, 3, true);
    else QFS_BWD(4, 3, 2, true);
  }
#undef QFS_BWD
#undef QFS_BWD1
#undef QFS_BWD1N
#undef QFS_BWD1I
#undef QFS_BWD1IN
  return cudaGetLastError();
}

int fwd2_min_blocks() { return QFS_FWD2_MINB; }

cudaError_t launch_polar(const PolarParams &p, int n_slots, cudaStream_t st) {
  launch_ex(polar_kernel, dim3((n_slots + 3) / 4), dim3(128), 0, st, p);
  return cudaGetLastError();
}

cudaError_t launch_final(const FinalParams &p, int n_slots, cudaStream_t st) {
  launch_ex(final_kernel, dim3(p.nb, n_slots), dim3(RED_THREADS), 0, st, p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_gate(const FwdGateParams &p, int n_slots, cudaStream_t st) {
  const int smem = FWD_STAGES * 4 * FWD_THREADS * (int)sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fwd_gate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  launch_ex(fwd_gate_kernel, dim3(p.nb, n_slots), dim3(FWD_THREADS), smem, st, p);
  return cudaGetLastError();
}

cudaError_t launch_fwd2(const Fwd2Params &p, int n_slots, cudaStream_t st) {
  dim3 grid(p.nb, n_slots), block(FWD2_THREADS);
#define QFS_FWD2(NU, A, B)                                                \
  do {                                                                    \
    if (p.src.ident) launch_ex(fwd2_kernel<NU, A, B, true>, grid, block, 0, st, p); \
    else launch_ex(fwd2_kernel<NU, A, B, false>, grid, block, 0, st, p);  \
  } while (0)
  if (p.nu == 2) {
    if (p.tp0 == 0) QFS_FWD2(2, 0, 1);
    else QFS_FWD2(2, 1, 0);
  } else if (p.nu == 3) {
    if (p.tp0 == 0 && p.tp1 == 2) QFS_FWD2(3, 0, 2);
    else if (p.tp0 == 2 && p.tp1 == 0) QFS_FWD2(3, 2, 0);
    else if (p.tp0 == 1 && p.tp1 == 2) QFS_FWD2(3, 1, 2);
    else QFS_FWD2(3, 2, 1);
  } else {
    if (p.tp0 == 2) QFS_FWD2(4, 2, 3);
    else QFS_FWD2(4, 3, 2);
  }
#undef QFS_FWD2
  return cudaGetLastError();
}

cudaError_t launch_fwdp(const FwdpParams &p, int n_slots, cudaStream_t st) {
  dim3 grid(p.nb, n_slots), block(FWD_THREADS);
#define QFS_FWDP(NU, A, B) launch_ex(fwdp_kernel<NU, A, B>, grid, block, 0, st, p)
  if (p.nu == 2) {
    if (p.tp0 == 0) QFS_FWDP(2, 0, 1);
    else QFS_FWDP(2, 1, 0);
  } else if (p.nu == 3) {
    if (p.tp0 == 0 && p.tp1 == 2) QFS_FWDP(3, 0, 2);
    else if (p.tp0 == 2 && p.tp1 == 0) QFS_FWDP(3, 2, 0);
    else if (p.tp0 == 1 && p.tp1 == 2) QFS_FWDP(3, 1, 2);
    else QFS_FWDP(3, 2, 1);
  } else {
    if (p.tp0 == 2) QFS_FWDP(4, 2, 3);
    else QFS_FWDP(4, 3, 2);
  }
#undef QFS_FWDP
  return cudaGetLastError();
}

cudaError_t launch_val_row(const ValRowParams &p, int n_slots, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(val_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double2) << 13));
    attr_set = true;
  }
  launch_ex(val_row_kernel, dim3(p.rows, n_slots), dim3(VAL_THREADS), sizeof(double2) << p.n, st, p);
  return cudaGetLastError();
}

cudaError_t launch_dist(const DistParams &p, int n_slots, cudaStream_t st) {
  launch_ex(dist_kernel, dim3(p.rows, n_slots), dim3(RED_THREADS), 0, st, p);
  return cudaGetLastError();
}

cudaError_t launch_row_reduce(const double *row_in, int rows, double *out, int n_slots,
                              cudaStream_t st) {
  row_reduce_kernel<<<(n_slots + 127) / 128, 128, 0, st>>>(row_in, rows, out, n_slots);
  return cudaGetLastError();
}

cudaError_t launch_apply(const ApplyParams &p, cudaStream_t st) {
  long long items = (long long)p.m << (p.n - 2);
  long long blocks = (items + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  apply_kernel<<<(unsigned)blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_polar_batch(const double2 *env, const double2 *g_old, double beta,
                               double2 *g_new, double *sig, int count, cudaStream_t st) {
  polar_batch_kernel<<<(count + 7) / 8, 128, 0, st>>>(env, g_old, beta, g_new, sig, count);
  return cudaGetLastError();
}

cudaError_t launch_transpose(const double2 *src, double2 *dst, int rows, long long cols,
                             cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (rows + 31) / 32), block(32, 8);
  transpose_kernel<<<grid, block, 0, st>>>(src, dst, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_finite_check(const double *p, long long n, int *flag, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  finite_check_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_copy(double2 *dst, const double2 *src, long long count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  long long blocks = (count + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  copy_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, src, count);
  return cudaGetLastError();
}

cudaError_t launch_copy_bytes(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  const long long words = (long long)(bytes / 4);
  if (words <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((words + 255) / 256, 148 * 8);
  copy_words_kernel<<<(unsigned)blocks, 256, 0, st>>>((unsigned *)dst, (const unsigned *)src, words);
  return cudaGetLastError();
}

cudaError_t launch_publish(const double *src, int count, const unsigned *check, double *hdst, unsigned *hcheck,
                           unsigned long long *hflag, unsigned long long seq, cudaStream_t st) {
  publish_kernel<<<1, 256, 0, st>>>(src, count, check, hdst, hcheck, hflag, seq);
  return cudaGetLastError();
}

cudaError_t launch_flag_bit(const unsigned *src, unsigned *dst, unsigned bit, cudaStream_t st) {
  flag_bit_kernel<<<1, 1, 0, st>>>(src, dst, bit);
  return cudaGetLastError();
}

cudaError_t launch_fill_words(unsigned *dst, unsigned value, long long count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((count + 255) / 256, 148 * 8);
  fill_words_kernel<<<(unsigned)blocks, 256, 0, st>>>(dst, value, count);
  return cudaGetLastError();
}

cudaError_t launch_gate_check(const double2 *g, long long count, int K, const int *kinds, unsigned *flag,
                              cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((count + 127) / 128, 148 * 4);
  gate_check_kernel<<<(unsigned)blocks, 128, 0, st>>>(g, count, K, kinds, flag);
  return cudaGetLastError();
}

cudaError_t launch_identity_fill(double2 *v, long long count16, cudaStream_t st) {
  if (count16 <= 0) return cudaSuccess;
  long long blocks = (count16 * 16 + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  identity_fill_kernel<<<(unsigned)blocks, 256, 0, st>>>(v, count16);
  return cudaGetLastError();
}

}  // namespace qfs
