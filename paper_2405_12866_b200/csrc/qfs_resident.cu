// qfs_resident.cu — cluster-resident QFactor-Sample sweep for sm_100a.
//
// One thread-block cluster of C CTAs owns one multistart at a time and runs
// its whole sweep (SURVEY.md §8 rows
// a2-a7) out of shared memory: the forward and backward states of the CTA's
// slice of the training samples never leave the SM.  This is the "uncompute"
// variant of the B cache: instead of storing B_1..B_{K-1}
// (P:165's time-memory trade-off) the forward pass keeps only
// phi = B_{K-1} = G_{K-2}...G_0 x, and the backward pass recovers
// B_i = G_i^dag B_{i+1} with the gate's old value (gates are unitary).
//
// Per gate i = K-1 .. 0 (right to left):
//   1. all warps:  E_i partial = sum phi (x) conj(chi) over the CTA's samples
//                  (P:121-125), warp butterfly + warps in order
//   2. warp 0:     cluster barrier, sums the C CTA partials in rank order over
//                  DSMEM (identical bits in every CTA), polar update
//                  G_i <- Y X^dag (eq:opt_u) into the CTA's gate table;
//      warps 1-7:  meanwhile phi <- G_{i-1}^dag phi (uncompute B_{i-1})
//   3. all warps:  chi <- G_i^dag chi (the new value), fused at i = 0 with
//                  c_train = sum ||chi - x||^2 (direct form)
// then the validation rows run forward through the new gates.
// Every reduction has a fixed order, so the result is deterministic for a
// given cluster size.  No code here is shared with the CPU oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "qfs_device.cuh"
#include "qfs_internal.h"

namespace qfs {
namespace {

#ifndef QFS_RES_THREADS
#define QFS_RES_THREADS 256
#endif
constexpr int RES_THREADS = QFS_RES_THREADS;
#ifndef QFS_RES_ENV_UNROLL
#define QFS_RES_ENV_UNROLL 2  // res_env items per unrolled iteration (loads of the next item above the FMAs)
#endif
constexpr int RES_ENV_UNROLL = QFS_RES_ENV_UNROLL;
#ifndef QFS_RES_PUSH
#define QFS_RES_PUSH 1  // resident: CTA partials pushed over DSMEM before the cluster barrier
#endif
#ifndef QFS_RES_FUSE
// resident: chi update of gate i fused with the environment of gate i-1 (one
// pass and one barrier less per gate) — measured slower (C3 442.8 -> 450.9 us
// per sweep, C5c 1452 -> 1501 us: 255 registers and spills), so off
#define QFS_RES_FUSE 0
#endif
#ifndef QFS_RES_PAIRS
#define QFS_RES_PAIRS 1  // resident forward / validation: two gates per shared-memory pass
#endif
#ifndef QFS_RES_SPARE_SMSP
#define QFS_RES_SPARE_SMSP 1  // resident: the uncompute beside the polar leaves warp 0's scheduler alone
#endif
#ifndef QFS_RES_MBAR
// resident: the per-gate cluster exchange of E partials as st.async stores that
// complete on the receiving CTA's mbarrier (only warp 0 waits), instead of a
// cluster-wide barrier.arrive / wait of all threads
#define QFS_RES_MBAR 1
#endif
#ifndef QFS_RES_ALIGN
#define QFS_RES_ALIGN 128  // dynamic shared-memory alignment of the resident / validation kernels
#endif
constexpr int RES_WARPS = RES_THREADS / 32;
constexpr size_t RES_SMEM_MAX = 232448;  // 227 KB opt-in dynamic shared memory per CTA
constexpr size_t RES_SMEM_MAX2 = 113 * 1024;  // two CTAs per SM (228 KB per SM, 1 KB reserved per CTA)

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_size() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cl_count() {
  unsigned r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// split cluster barrier: arrive (release this thread's prior shared-memory
// writes to the cluster) ... wait (acquire the other CTAs' writes)
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }
// load a double from the same shared-memory offset in CTA `rank` of the cluster
// (volatile without a memory clobber: kept after the cluster barrier's wait,
// which clobbers memory, but independent loads can be in flight together)
__device__ __forceinline__ void st_remote_d(double *p, unsigned rank, double v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
// 8-byte store into CTA `rank`'s shared memory at the same offset, completing
// `bytes` on that CTA's mbarrier (same offset) when it has landed
__device__ __forceinline__ void st_async_remote_d(double *p, uint64_t *bar, unsigned rank, double v) {
  unsigned ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}

__device__ __forceinline__ double ld_remote(const double *p, unsigned rank) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
  return v;
}

// psi <- G psi (dag: G^dag psi) on the qubit pair pq for the rows jj < cnt of
// a [2^n][ld] shared-memory state block (sample-minor: quadruple members of
// consecutive items are consecutive samples).  Threads t0, t0 + nt, ...
__device__ void res_apply(double2 *psi, const double2 *G, int2 pq, bool dag, int cnt, const FastDiv &fd,
                          unsigned ld, int n, int t0, int nt) {
  if (cnt <= 0) return;
  double2 g[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) g[e] = dag ? cconj(G[4 * (e & 3) + (e >> 2)]) : G[e];  // (G^dag)[a][b] = conj(G[b][a])
  const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
  const unsigned o1 = (1u << pq.x) * ld, o2 = (1u << pq.y) * ld;
  const unsigned items = (1u << (n - 2)) * (unsigned)cnt;
  for (unsigned q = (unsigned)t0; q < items; q += (unsigned)nt) {
    const unsigned r = fd.div(q);
    const unsigned b = insert_zero32(insert_zero32(r, lo), hi) * ld + (q - r * (unsigned)cnt);
    double2 v[4] = {psi[b], psi[b + o1], psi[b + o2], psi[b + o1 + o2]};
    double2 o[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      o[a] = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < 4; ++k) cfma(o[a], g[4 * a + k], v[k]);
    }
    psi[b] = o[0];
    psi[b + o1] = o[1];
    psi[b + o2] = o[2];
    psi[b + o1 + o2] = o[3];
  }
}


// Two consecutive gates in one pass over a [2^n][ld] shared-memory block: each
// item holds the 2^NU amplitudes spanned by both pairs in registers (gate k on
// local bits (0, 1), gate k+1 on (TP0, TP1)), so the state is read and written
// once per two gates with one barrier instead of two.  Gate entries are
// re-read from shared memory per use.
template <int NU, int TP0, int TP1>
__device__ __forceinline__ constexpr int pair_idx(int q, int l) {
  int v = ((l & 1) << TP0) | (((l >> 1) & 1) << TP1);
  int bit = 0;
  for (int t = 0; t < NU; ++t) {
    if (t == TP0 || t == TP1) continue;
    v |= ((q >> bit) & 1) << t;
    ++bit;
  }
  return v;
}
__device__ __forceinline__ double2 lds_c2(const double2 *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
#ifndef QFS_PAIR_GREG
#define QFS_PAIR_GREG 3  // gate entries of the two-gate pass: 3 read once per item for all its quadruples (default), 0 re-read per use, 1 G1 in registers, 2 both (1, 2 spill)
#endif
template <int NU, int TP0, int TP1>
__device__ void res_apply_pair_t(double2 *psi, const double2 *G1, const double2 *G2, const int (&loc)[4],
                                 const int (&srt)[4], int cnt, const FastDiv &fd, unsigned ld, int n, int t0, int nt) {
  constexpr int NV = 1 << NU, NQ = NV / 4;
  double2 g1r[QFS_PAIR_GREG >= 1 ? 16 : 1], g2r[QFS_PAIR_GREG >= 2 ? 16 : 1];
  if constexpr (QFS_PAIR_GREG >= 1) {
#pragma unroll
    for (int e = 0; e < 16; ++e) g1r[e] = G1[e];
  }
  if constexpr (QFS_PAIR_GREG >= 2) {
#pragma unroll
    for (int e = 0; e < 16; ++e) g2r[e] = G2[e];
  }
  auto ge1 = [&](int e) { if constexpr (QFS_PAIR_GREG >= 1) return g1r[e]; else return lds_c2(G1 + e); };
  auto ge2 = [&](int e) { if constexpr (QFS_PAIR_GREG >= 2) return g2r[e]; else return lds_c2(G2 + e); };
  unsigned ob[NU];  // shared-memory offset of local bit t
#pragma unroll
  for (int t = 0; t < NU; ++t) ob[t] = (1u << loc[t]) * ld;
  auto offs = [&](int u) {  // u is a compile-time constant after unrolling
    unsigned o = 0;
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((u >> t) & 1) o += ob[t];
    return o;
  };
  const unsigned items = (1u << (n - NU)) * (unsigned)cnt;
  for (unsigned q = (unsigned)t0; q < items; q += (unsigned)nt) {
    const unsigned r = fd.div(q);
    unsigned g = r;
#pragma unroll
    for (int t = 0; t < NU; ++t) g = insert_zero32(g, srt[t]);
    const unsigned b = g * ld + (q - r * (unsigned)cnt);
    double2 v[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) v[u] = psi[b + offs(u)];
    if constexpr (QFS_PAIR_GREG == 3) {
      // each gate entry read once per item and applied to all NQ quadruples
      // (same summation order per output as below: bit-identical)
      double2 o[NQ][4];
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int a = 0; a < 4; ++a) o[qq][a] = make_double2(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 g = lds_c2(G1 + 4 * a + c);
#pragma unroll
          for (int qq = 0; qq < NQ; ++qq) cfma(o[qq][a], g, v[4 * qq + c]);
        }
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int a = 0; a < 4; ++a) v[4 * qq + a] = o[qq][a];
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int a = 0; a < 4; ++a) o[qq][a] = make_double2(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 g = lds_c2(G2 + 4 * a + c);
#pragma unroll
          for (int qq = 0; qq < NQ; ++qq) cfma(o[qq][a], g, v[pair_idx<NU, TP0, TP1>(qq, c)]);
        }
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
        for (int a = 0; a < 4; ++a) v[pair_idx<NU, TP0, TP1>(qq, a)] = o[qq][a];
    } else {
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        double2 o[4];
  #pragma unroll
        for (int a = 0; a < 4; ++a) {
          o[a] = make_double2(0.0, 0.0);
  #pragma unroll
          for (int c = 0; c < 4; ++c) cfma(o[a], ge1(4 * a + c), v[4 * qq + c]);
        }
  #pragma unroll
        for (int a = 0; a < 4; ++a) v[4 * qq + a] = o[a];
      }
  #pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        double2 o[4];
  #pragma unroll
        for (int a = 0; a < 4; ++a) {
          o[a] = make_double2(0.0, 0.0);
  #pragma unroll
          for (int c = 0; c < 4; ++c) cfma(o[a], ge2(4 * a + c), v[pair_idx<NU, TP0, TP1>(qq, c)]);
        }
  #pragma unroll
        for (int a = 0; a < 4; ++a) v[pair_idx<NU, TP0, TP1>(qq, a)] = o[a];
      }
  }
#pragma unroll
    for (int u = 0; u < NV; ++u) psi[b + offs(u)] = v[u];
  }
}
__device__ void res_apply_pair(double2 *psi, const double2 *G1, int2 p1, const double2 *G2, int2 p2, int cnt,
                               const FastDiv &fd, unsigned ld, int n, int t0, int nt) {
  // union of the pairs in local order (gate k's pair first, then gate k+1's new
  // qubits ascending) and gate k+1's local positions; fixed-index code only
  const bool x_new = p2.x != p1.x && p2.x != p1.y, y_new = p2.y != p1.x && p2.y != p1.y;
  int l2 = 0, l3 = 0, nu = 2;
  if (x_new && y_new) { l2 = min(p2.x, p2.y); l3 = max(p2.x, p2.y); nu = 4; }
  else if (x_new) { l2 = p2.x; nu = 3; }
  else if (y_new) { l2 = p2.y; nu = 3; }
  auto pos = [&](int q) { return q == p1.x ? 0 : q == p1.y ? 1 : q == l2 ? 2 : 3; };
  const int tp0 = pos(p2.x), tp1 = pos(p2.y);
  const int loc[4] = {p1.x, p1.y, l2, l3};
  int a0 = p1.x, a1 = p1.y, a2 = nu > 2 ? l2 : 31, a3 = nu > 3 ? l3 : 31;  // ascending union bits
  auto cs = [](int &u, int &v) { if (v < u) { const int t = u; u = v; v = t; } };
  cs(a0, a1); cs(a2, a3); cs(a0, a2); cs(a1, a3); cs(a1, a2);
  const int srt[4] = {a0, a1, a2, a3};
  if (nu == 2) {
    if (tp0 == 0) res_apply_pair_t<2, 0, 1>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
    else res_apply_pair_t<2, 1, 0>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
  } else if (nu == 3) {
    if (tp0 == 0 && tp1 == 2) res_apply_pair_t<3, 0, 2>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
    else if (tp0 == 2 && tp1 == 0) res_apply_pair_t<3, 2, 0>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
    else if (tp0 == 1 && tp1 == 2) res_apply_pair_t<3, 1, 2>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
    else res_apply_pair_t<3, 2, 1>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
  } else {
    if (tp0 == 2) res_apply_pair_t<4, 2, 3>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
    else res_apply_pair_t<4, 3, 2>(psi, G1, G2, loc, srt, cnt, fd, ld, n, t0, nt);
  }
}

// Warp butterfly reduce-scatter of 32 per-lane values: lane L ends with the
// sum over the warp of value L (fixed order; 31 shuffles per lane).
__device__ __forceinline__ double warp_reduce_scatter32(double (&acc)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = up ? acc[i] : acc[i + h];
      const double keep = up ? acc[i + h] : acc[i];
      acc[i] = keep + __shfl_xor_sync(FULL, send, h);
    }
  }
  return acc[0];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// E[l_in][l_out] += sum phi[idx(l_in)] conj(chi[idx(l_out)]) over this CTA's
// items; every warp writes its reduced 32 doubles (re/im of the 16
// entries, row-major) to red[warp][.]
__device__ void res_env(const double2 *phi, const double2 *chi, int2 pq, int cnt, const FastDiv &fd,
                        unsigned ld, int n, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) acc[e] = 0.0;
  if (cnt > 0) {
    const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
    const unsigned o1 = (1u << pq.x) * ld, o2 = (1u << pq.y) * ld;
    const unsigned items = (1u << (n - 2)) * (unsigned)cnt;
#pragma unroll RES_ENV_UNROLL
    for (unsigned q = threadIdx.x; q < items; q += RES_THREADS) {
      const unsigned r = fd.div(q);
      const unsigned b = insert_zero32(insert_zero32(r, lo), hi) * ld + (q - r * (unsigned)cnt);
      const double2 f[4] = {phi[b], phi[b + o1], phi[b + o2], phi[b + o1 + o2]};
      const double2 c[4] = {chi[b], chi[b + o1], chi[b + o2], chi[b + o1 + o2]};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // f[a] * conj(c[k])
          double &re = acc[2 * (4 * a + k)], &im = acc[2 * (4 * a + k) + 1];
          re = fma(f[a].x, c[k].x, re);
          re = fma(f[a].y, c[k].y, re);
          im = fma(f[a].y, c[k].x, im);
          im = fma(-f[a].x, c[k].y, im);
        }
    }
  }
  red[warp * 32 + lane] = warp_reduce_scatter32(acc, lane);
}

// Fused backward pass of the resident sweep (QFS_RES_FUSE): chi <- G_i^dag chi
// (gate i on local bits 0, 1) and, from the same registers, the environment of
// gate i-1 (its pair at local (TP0, TP1); phi = B_{i-1} already
// uncomputed) — one shared-memory pass and one barrier instead of two.  Every
// warp writes its reduced 32 doubles (re/im of E_{i-1}'s 16 entries) to
// red[warp][.] like res_env.
template <int NU, int TP0, int TP1>
__device__ void res_chi_env_t(double2 *chi, const double2 *phi, const double2 *G, const int (&loc)[4],
                              const int (&srt)[4], int cnt, const FastDiv &fd, unsigned ld, int n, double *red) {
  constexpr int NV = 1 << NU, NQ = NV / 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) acc[e] = 0.0;
  unsigned ob[NU];
#pragma unroll
  for (int t = 0; t < NU; ++t) ob[t] = (1u << loc[t]) * ld;
  auto offs = [&](int u) {
    unsigned o = 0;
#pragma unroll
    for (int t = 0; t < NU; ++t)
      if ((u >> t) & 1) o += ob[t];
    return o;
  };
  const unsigned items = cnt > 0 ? (1u << (n - NU)) * (unsigned)cnt : 0u;
  for (unsigned q = threadIdx.x; q < items; q += RES_THREADS) {
    const unsigned r = fd.div(q);
    unsigned g = r;
#pragma unroll
    for (int t = 0; t < NU; ++t) g = insert_zero32(g, srt[t]);
    const unsigned b = g * ld + (q - r * (unsigned)cnt);
    double2 v[NV];
#pragma unroll
    for (int u = 0; u < NV; ++u) v[u] = chi[b + offs(u)];
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {  // chi' = G^dag chi, (G^dag)[a][c] = conj(G[c][a])
      double2 o[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        o[a] = make_double2(0.0, 0.0);
#pragma unroll
        for (int c = 0; c < 4; ++c) cfma(o[a], cconj(lds_c2(G + 4 * c + a)), v[4 * qq + c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) v[4 * qq + a] = o[a];
    }
#pragma unroll
    for (int u = 0; u < NV; ++u) chi[b + offs(u)] = v[u];
#pragma unroll
    for (int p = 0; p < NQ; ++p) {  // E[a][k] += phi[a] conj(chi'[k]) on gate i-1's quadruples
      double2 f[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) f[l] = phi[b + offs(pair_idx<NU, TP0, TP1>(p, l))];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 ck = v[pair_idx<NU, TP0, TP1>(p, k)];
          double &re = acc[2 * (4 * a + k)], &im = acc[2 * (4 * a + k) + 1];
          re = fma(f[a].x, ck.x, re);
          re = fma(f[a].y, ck.y, re);
          im = fma(f[a].y, ck.x, im);
          im = fma(-f[a].x, ck.y, im);
        }
    }
  }
  red[warp * 32 + lane] = warp_reduce_scatter32(acc, lane);
}
// dispatch on the union of gate i's pair p1 and gate i-1's pair p2 (the local
// order and template keys of res_apply_pair)
__device__ void res_chi_env(double2 *chi, const double2 *phi, const double2 *G, int2 p1, int2 p2, int cnt,
                            const FastDiv &fd, unsigned ld, int n, double *red) {
  const bool x_new = p2.x != p1.x && p2.x != p1.y, y_new = p2.y != p1.x && p2.y != p1.y;
  int l2 = 0, l3 = 0, nu = 2;
  if (x_new && y_new) { l2 = min(p2.x, p2.y); l3 = max(p2.x, p2.y); nu = 4; }
  else if (x_new) { l2 = p2.x; nu = 3; }
  else if (y_new) { l2 = p2.y; nu = 3; }
  auto pos = [&](int q) { return q == p1.x ? 0 : q == p1.y ? 1 : q == l2 ? 2 : 3; };
  const int tp0 = pos(p2.x), tp1 = pos(p2.y);
  const int loc[4] = {p1.x, p1.y, l2, l3};
  int a0 = p1.x, a1 = p1.y, a2 = nu > 2 ? l2 : 31, a3 = nu > 3 ? l3 : 31;
  auto cs = [](int &u, int &v) { if (v < u) { const int t = u; u = v; v = t; } };
  cs(a0, a1); cs(a2, a3); cs(a0, a2); cs(a1, a3); cs(a1, a2);
  const int srt[4] = {a0, a1, a2, a3};
  if (nu == 2) {
    if (tp0 == 0) res_chi_env_t<2, 0, 1>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
    else res_chi_env_t<2, 1, 0>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
  } else if (nu == 3) {
    if (tp0 == 0 && tp1 == 2) res_chi_env_t<3, 0, 2>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
    else if (tp0 == 2 && tp1 == 0) res_chi_env_t<3, 2, 0>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
    else if (tp0 == 1 && tp1 == 2) res_chi_env_t<3, 1, 2>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
    else res_chi_env_t<3, 2, 1>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
  } else {
    if (tp0 == 2) res_chi_env_t<4, 2, 3>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
    else res_chi_env_t<4, 3, 2>(chi, phi, G, loc, srt, cnt, fd, ld, n, red);
  }
}

struct ResSmem {
  double2 *G;     // [K][16] gate table of the current start (old -> new in place)
  double *red;    // [RES_WARPS][32]
  double *buf;    // [2][32] CTA partial of E (read by the cluster over DSMEM)
  double *cbuf;   // [2] CTA partial costs (train, validation)
  double2 *scr;   // [64] polar scratch (32 per half warp)
  int2 *pr;       // [K] qubit pairs
  int *kinds;     // [K] gate kinds
  double2 *phi;   // [2^n][ld]
  double2 *chi;   // [2^n][ld]
  uint64_t *mbar; // [2] per gate parity (QFS_RES_MBAR)
};

// (offsets from the __shared__ base, no integer casts: the compiler keeps the
// shared state space and emits LDS/STS with 32-bit addresses, not generic
// LD/ST with 64-bit ones)
__device__ __forceinline__ ResSmem res_carve(unsigned char *base, int K, int n, int ld) {
  ResSmem m;
  size_t off = 0;
  m.G = (double2 *)base;
  off += (size_t)K * 16 * sizeof(double2);
  m.red = (double *)(base + off);
  off += RES_WARPS * 32 * sizeof(double);
  m.buf = (double *)(base + off);
  off += (QFS_RES_PUSH ? 2 * 16 * 32 : 64) * sizeof(double);
  m.cbuf = (double *)(base + off);
  off += 2 * sizeof(double);
  m.scr = (double2 *)(base + off);
  off += 64 * sizeof(double2);
  m.pr = (int2 *)(base + off);
  off += (size_t)K * sizeof(int2);
  m.kinds = (int *)(base + off);
  off += (size_t)K * sizeof(int);
  off = (off + 7) & ~(size_t)7;
  m.mbar = (uint64_t *)(base + off);
  off += 2 * sizeof(uint64_t);
  off = (off + 15) & ~(size_t)15;
  m.phi = (double2 *)(base + off);
  m.chi = m.phi + ((size_t)ld << n);
  return m;
}

// MINB = resident CTAs per SM the kernel is compiled for (2: <= 128 registers,
// <= 113 KB shared memory each, so one CTA's polar tail overlaps another
// start's contraction on the same SM).
template <int MINB>
__global__ void __launch_bounds__(RES_THREADS, MINB) res_sweep_kernel(const ResParams P) {
  extern __shared__ __align__(QFS_RES_ALIGN) unsigned char smem_raw[];
  const int K = P.K, n = P.n;
  const unsigned N = 1u << n, ld = (unsigned)P.ld;
  const ResSmem sm = res_carve(smem_raw, K, n, P.ld);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cl_rank(), C = cl_size();

  if (QFS_RES_MBAR && tid == 0) {
    mbar_init(sm.mbar, 1);
    mbar_init(sm.mbar + 1, 1);
    mbar_fence_init();
  }
  pdl_wait();
  for (int k = tid; k < K; k += RES_THREADS) {
    sm.pr[k] = P.pairs[k];
    sm.kinds[k] = P.kinds ? P.kinds[k] : 0;
  }
  if (QFS_RES_MBAR) {  // every CTA's mbarriers initialised before any CTA pushes to them
    cl_arrive();
    cl_wait();
  }
  unsigned mph = 0;  // warp 0: phase parity of mbar[g] in bit g
  // diagnostics: phase times of cluster 0, rank 0 (thread 0), summed over gates
  const bool dbg = P.dbg && cl_id() == 0 && rank == 0 && tid == 0;
  unsigned long long t_prev = 0, ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  auto stamp = [&](int k) {
    if (dbg) {
      const unsigned long long t = gtimer();
      if (k >= 0) ph[k] += t - t_prev;
      t_prev = t;
    }
  };
  stamp(-1);  // start of the launch

  for (int j = (int)cl_id(); j < P.n_slots; j += (int)cl_count()) {
    const Slot sl = P.slots[j];
    const int s = sl.s, M = sl.m;
    const int ms = (M + (int)C - 1) / (int)C;
    const int m0 = (int)rank * ms;
    const int cnt = max(0, min(ms, M - m0));
    const FastDiv fd((unsigned)max(cnt, 1));  // item -> (quadruple, row) of this CTA's rows
    double2 *gglob = P.gates + (long long)s * K * 16;
    for (int q = tid; q < K * 16; q += RES_THREADS) sm.G[q] = gglob[q];
    for (unsigned q = tid; q < N * (unsigned)cnt; q += RES_THREADS) {
      const unsigned a = q / (unsigned)cnt, jj = q - a * (unsigned)cnt;
      const long long gi = (long long)a * P.m_pool + m0 + jj;
      sm.phi[a * ld + jj] = __ldg(P.x + gi);
      sm.chi[a * ld + jj] = __ldg(P.y + gi);
    }
    __syncthreads();
    stamp(0);  // [0] load
    // forward with the previous sweep's gates: phi = B_{K-1} = G_{K-2} ... G_0 x
    if constexpr (QFS_RES_PAIRS && MINB == 1) {  // (the 128-register variant would spill)
      int k = 0;
      for (; k + 2 < K; k += 2) {  // gates k, k+1 (the last gate, K-1, is not applied)
        res_apply_pair(sm.phi, sm.G + 16 * k, sm.pr[k], sm.G + 16 * (k + 1), sm.pr[k + 1], cnt, fd, ld, n, tid,
                       RES_THREADS);
        __syncthreads();
      }
      if (k + 1 < K) {
        res_apply(sm.phi, sm.G + 16 * k, sm.pr[k], false, cnt, fd, ld, n, tid, RES_THREADS);
        __syncthreads();
      }
    } else {
      for (int k = 0; k + 1 < K; ++k) {
        res_apply(sm.phi, sm.G + 16 * k, sm.pr[k], false, cnt, fd, ld, n, tid, RES_THREADS);
        __syncthreads();
      }
    }
    stamp(1);  // [1] forward
    double train = 0.0;
    constexpr bool FUSE = QFS_RES_FUSE && MINB == 1;  // (the 128-register variant would spill)
    if (FUSE) res_env(sm.phi, sm.chi, sm.pr[K - 1], cnt, fd, ld, n, sm.red);  // E_{K-1}; the rest fused below
    for (int i = K - 1; i >= 0; --i) {
      const int par = i & 1;
      if (!FUSE) res_env(sm.phi, sm.chi, sm.pr[i], cnt, fd, ld, n, sm.red);
      __syncthreads();
      stamp(2);  // [2] environment pass
#if QFS_RES_MBAR
      if (warp == 0) {
        // push this CTA's partial into slot [rank] of every cluster CTA's
        // buffer; the stores complete C*256 bytes on each receiver's mbar[par]
        double e = 0.0;
#pragma unroll
        for (int w = 0; w < RES_WARPS; ++w) e += sm.red[w * 32 + lane];
        if (lane == 0) mbar_arrive_tx(sm.mbar + par, C * 32 * (unsigned)sizeof(double));
        __syncwarp();
        for (unsigned c = 0; c < C; ++c) st_async_remote_d(sm.buf + par * 512 + rank * 32 + lane, sm.mbar + par, c, e);
        mbar_wait(sm.mbar + par, (mph >> par) & 1u);
        mph ^= 1u << par;
        e = 0.0;
        for (unsigned c = 0; c < C; ++c) e += sm.buf[par * 512 + c * 32 + lane];  // rank order
#elif QFS_RES_PUSH
      // push this CTA's partial into slot [rank] of every cluster CTA's buffer
      // (remote stores overlap the barrier); after it, all partials are local
      if (warp == 0) {
        double e = 0.0;
#pragma unroll
        for (int w = 0; w < RES_WARPS; ++w) e += sm.red[w * 32 + lane];
        for (unsigned c = 0; c < C; ++c) st_remote_d(sm.buf + par * 512 + rank * 32 + lane, c, e);
      }
      cl_arrive();
      if (warp == 0) {
        cl_wait();
        double e = 0.0;
        for (unsigned c = 0; c < C; ++c) e += sm.buf[par * 512 + c * 32 + lane];  // rank order
#else
      if (warp == 0) {
        double e = 0.0;
#pragma unroll
        for (int w = 0; w < RES_WARPS; ++w) e += sm.red[w * 32 + lane];
        sm.buf[par * 32 + lane] = e;
      }
      cl_arrive();
      if (warp == 0) {
        cl_wait();
        double rv[16];  // all remote loads in flight first, then summed in rank order
#pragma unroll
        for (unsigned c = 0; c < 16; ++c) rv[c] = c < C ? ld_remote(sm.buf + par * 32 + lane, c) : 0.0;
        double e = 0.0;
#pragma unroll
        for (unsigned c = 0; c < 16; ++c)
          if (c < C) e += rv[c];
#endif
        stamp(3);  // [3] CTA + cluster reduction
        const int l = lane & 15;
        double2 ev = make_double2(__shfl_sync(FULL, e, 2 * l), __shfl_sync(FULL, e, 2 * l + 1));
        double2 *gi = sm.G + 16 * i;
        if (P.env_trace && rank == 0 && lane < 16) P.env_trace[((long long)i * P.S + s) * 16 + l] = ev;
        const int kind = sm.kinds[i];
        double2 g, v;
        double ss;
        gate_update(kind, ev, gi, P.beta, nullptr, g, v, ss,
                    sm.scr + 2 * (lane & 16), P.sig != nullptr);
        __syncwarp();
        if (lane < 16 && kind != 1) gi[l] = g;
        if (rank == 0) {
          if (lane < 16 && kind != 1) gglob[16 * i + l] = g;
          if (lane == 0 && P.sig) P.sig[(long long)s * K + i] = ss;
        }
        stamp(4);  // [4] polar
      } else {
        // uncompute B_{i-1} = G_{i-1}^dag B_i with the old G_{i-1}, overlapping the polar
#if QFS_RES_SPARE_SMSP
        // not warp 4: it shares warp 0's scheduler (warp w -> SMSP w % 4), whose
        // polar is a latency-bound chain the uncompute's DFMA would slow down
        if (i > 0 && warp != 4) {
          const int t = tid - 32 - (warp > 4 ? 32 : 0);
          res_apply(sm.phi, sm.G + 16 * (i - 1), sm.pr[i - 1], true, cnt, fd, ld, n, t, RES_THREADS - 64);
        }
#else
        if (i > 0) res_apply(sm.phi, sm.G + 16 * (i - 1), sm.pr[i - 1], true, cnt, fd, ld, n, tid - 32, RES_THREADS - 32);
#endif
#if !QFS_RES_MBAR
        cl_wait();
#endif
      }
      __syncthreads();
      stamp(5);  // [5] wait for the uncompute warps
      if (i > 0) {
        if constexpr (FUSE)  // chi <- G_i^dag chi fused with the environment of gate i-1 (phi = B_{i-1} now)
          res_chi_env(sm.chi, sm.phi, sm.G + 16 * i, sm.pr[i], sm.pr[i - 1], cnt, fd, ld, n, sm.red);
        else
          res_apply(sm.chi, sm.G + 16 * i, sm.pr[i], true, cnt, fd, ld, n, tid, RES_THREADS);
      } else if (cnt > 0) {
        // chi' = G_0^dag chi and c_train = sum ||chi' - x||^2
        const double2 *G = sm.G;
        double2 g[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) g[e] = cconj(G[4 * (e & 3) + (e >> 2)]);
        const int2 pq = sm.pr[0];
        const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
        const unsigned o[4] = {0u, (1u << pq.x), (1u << pq.y), (1u << pq.x) | (1u << pq.y)};
        const unsigned items = (N >> 2) * (unsigned)cnt;
        for (unsigned q = tid; q < items; q += RES_THREADS) {
          const unsigned r = fd.div(q), jj = q - r * (unsigned)cnt;
          const unsigned base = insert_zero32(insert_zero32(r, lo), hi);
          double2 v[4];
#pragma unroll
          for (int l = 0; l < 4; ++l) v[l] = sm.chi[(base | o[l]) * ld + jj];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            double2 rr = make_double2(0.0, 0.0);
#pragma unroll
            for (int k = 0; k < 4; ++k) cfma(rr, g[4 * a + k], v[k]);
            const double2 xv = __ldg(P.x + (long long)(base | o[a]) * P.m_pool + m0 + jj);
            const double dr = rr.x - xv.x, di = rr.y - xv.y;
            train = fma(dr, dr, train);
            train = fma(di, di, train);
          }
        }
      }
      __syncthreads();
      stamp(6);  // [6] chi update
    }
    // validation cost with the post-sweep gates: this CTA's rows
    // v = rank, rank + C, ..., in batches of ld rows through the phi buffer
    double val = 0.0;
    if (P.want_val && P.V > 0) {
      const int rows = (P.V - (int)rank + (int)C - 1) / (int)C;
      for (int b0 = 0; b0 < rows; b0 += (int)ld) {
        const int nb = min((int)ld, rows - b0);
        for (unsigned q = tid; q < N * (unsigned)nb; q += RES_THREADS) {
          const unsigned jj = q / N, a = q - jj * N;
          const long long row = (long long)rank + (long long)C * (b0 + jj);
          sm.phi[a * ld + jj] = __ldg(P.xv + row * N + a);
        }
        __syncthreads();
        const FastDiv fdv((unsigned)nb);
        if constexpr (QFS_RES_PAIRS && MINB == 1) {
          int k = 0;
          for (; k + 1 < K; k += 2) {
            res_apply_pair(sm.phi, sm.G + 16 * k, sm.pr[k], sm.G + 16 * (k + 1), sm.pr[k + 1], nb, fdv, ld, n,
                           tid, RES_THREADS);
            __syncthreads();
          }
          if (k < K) {
            res_apply(sm.phi, sm.G + 16 * k, sm.pr[k], false, nb, fdv, ld, n, tid, RES_THREADS);
            __syncthreads();
          }
        } else {
          for (int k = 0; k < K; ++k) {
            res_apply(sm.phi, sm.G + 16 * k, sm.pr[k], false, nb, fdv, ld, n, tid, RES_THREADS);
            __syncthreads();
          }
        }
        for (unsigned q = tid; q < N * (unsigned)nb; q += RES_THREADS) {
          const unsigned jj = q / N, a = q - jj * N;
          const long long row = (long long)rank + (long long)C * (b0 + jj);
          const double2 u = sm.phi[a * ld + jj], w = __ldg(P.yv + row * N + a);
          const double dr = u.x - w.x, di = u.y - w.y;
          val = fma(dr, dr, val);
          val = fma(di, di, val);
        }
        __syncthreads();
      }
    }
    stamp(7);  // [7] validation
    // costs: threads -> warps (in order) -> CTA -> cluster ranks (in order)
    train = warp_sum(train);
    val = warp_sum(val);
    if (lane == 0) {
      sm.red[warp] = train;
      sm.red[RES_WARPS + warp] = val;
    }
    __syncthreads();
    if (tid == 0) {
      double t = 0.0, v = 0.0;
      for (int w = 0; w < RES_WARPS; ++w) {
        t += sm.red[w];
        v += sm.red[RES_WARPS + w];
      }
      sm.cbuf[0] = t;
      sm.cbuf[1] = v;
    }
    cl_arrive();
    cl_wait();
    if (rank == 0 && tid == 0) {
      double t = 0.0, v = 0.0;
      for (unsigned c = 0; c < C; ++c) {
        t += ld_remote(sm.cbuf, c);
        v += ld_remote(sm.cbuf + 1, c);
      }
      P.csum[j] = t;
      if (P.want_val && P.V > 0) P.cval[j] = v;
    }
    // the next start rewrites the gate table and (later) cbuf: every CTA waits
    // until rank 0 has read the remote costs
    cl_arrive();
    cl_wait();
  }
  if (dbg)  // once per launch: the sums over this cluster's slots
    for (int q = 0; q < 8; ++q) atomicAdd(P.dbg + q, ph[q]);
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// Two starts per cluster, staggered (the default resident kernel when a
// cluster can hold two starts' states; QFS_RES_PAIR).  The per-gate chain of
// one start — E_i partials -> cluster sum -> polar -> chi <- G_i^dag chi ->
// E_{i-1} partials — is serial (the gates are updated one after the
// other, each from the environment of the already-updated ones to its left of
// chi), and its polar / cluster-sum part leaves the FP64 pipe idle.  Here each
// CTA holds its slice of TWO starts A and B and overlaps one start's polar
// with the other start's FP64 passes:
//   warp 0 (PW_A): sums A's CTA partials, pushes them to every CTA of the
//                  cluster (st.async over DSMEM completing on an mbarrier),
//                  waits for the C partials, sums them in rank order, polar
//                  update of A's gate;
//   warp 4 (PW_B): the same for B (warps 0 and 4 share SMSP 0, so the FP64
//                  passes keep two warps on each of the other three);
//   warps 1-3, 5-7 (CW): every FP64 pass of both starts, in the order
//     ... chi_A(i), E_A(i-1) | chi_B(i), E_B(i-1) | phi_A, phi_B <- G(i-2)^dag .. | wait G_A(i-1) ...
//   so B's passes run while A's polar does, and the other way round.
// Named barriers order the roles: ENV_X (CW arrive, PW_X sync: partials of
// E_i written), GATE_X (PW_X arrive, CW sync: new G_i in the gate table), CW
// (the six pass warps among themselves).  Forward, validation and the costs
// run on all eight warps before / after the backward loop, per start.  Every
// reduction keeps a fixed order (warps in order, then cluster ranks in order),
// so results are deterministic for a given cluster size.
constexpr int PW_A = 0, PW_B = 4;
constexpr int CW_THREADS = RES_THREADS - 64;
constexpr int CW_WARPS = CW_THREADS / 32;
enum { NB_CW = 1, NB_ENV_A = 2, NB_ENV_B = 3, NB_GATE_A = 4, NB_GATE_B = 5 };
__device__ __forceinline__ void nb_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}
// E partial over the items t0, t0 + nt, ... (res_env with a thread subset);
// the warp writes its 32 reduced doubles to red_row[lane]
__device__ void res_env_sub(const double2 *phi, const double2 *chi, int2 pq, int cnt, const FastDiv &fd, unsigned ld,
                            int n, int t0, int nt, double *red_row) {
  const int lane = threadIdx.x & 31;
  double acc[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) acc[e] = 0.0;
  if (cnt > 0) {
    const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
    const unsigned o1 = (1u << pq.x) * ld, o2 = (1u << pq.y) * ld;
    const unsigned items = (1u << (n - 2)) * (unsigned)cnt;
#pragma unroll RES_ENV_UNROLL
    for (unsigned q = (unsigned)t0; q < items; q += (unsigned)nt) {
      const unsigned r = fd.div(q);
      const unsigned b = insert_zero32(insert_zero32(r, lo), hi) * ld + (q - r * (unsigned)cnt);
      const double2 f[4] = {phi[b], phi[b + o1], phi[b + o2], phi[b + o1 + o2]};
      const double2 c[4] = {chi[b], chi[b + o1], chi[b + o2], chi[b + o1 + o2]};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // f[a] * conj(c[k])
          double &re = acc[2 * (4 * a + k)], &im = acc[2 * (4 * a + k) + 1];
          re = fma(f[a].x, c[k].x, re);
          re = fma(f[a].y, c[k].y, re);
          im = fma(f[a].y, c[k].x, im);
          im = fma(-f[a].x, c[k].y, im);
        }
    }
  }
  red_row[lane] = warp_reduce_scatter32(acc, lane);
}

// chi' = G_0^dag chi and this thread's share of c_train = sum ||chi' - x||^2
// over the items t0, t0 + nt, ...
__device__ double res_chi0_cost(const double2 *chi, const double2 *G, int2 pq, int cnt, const FastDiv &fd, unsigned ld,
                                int n, const double2 *x, long long m_pool, int m0, int t0, int nt) {
  double train = 0.0;
  if (cnt <= 0) return train;
  double2 g[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) g[e] = cconj(G[4 * (e & 3) + (e >> 2)]);
  const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
  const unsigned o[4] = {0u, (1u << pq.x), (1u << pq.y), (1u << pq.x) | (1u << pq.y)};
  const unsigned items = (1u << (n - 2)) * (unsigned)cnt;
  for (unsigned q = (unsigned)t0; q < items; q += (unsigned)nt) {
    const unsigned r = fd.div(q), jj = q - r * (unsigned)cnt;
    const unsigned base = insert_zero32(insert_zero32(r, lo), hi);
    double2 v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = chi[(base | o[l]) * ld + jj];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 rr = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < 4; ++k) cfma(rr, g[4 * a + k], v[k]);
      const double2 xv = __ldg(x + (long long)(base | o[a]) * m_pool + m0 + jj);
      const double dr = rr.x - xv.x, di = rr.y - xv.y;
      train = fma(dr, dr, train);
      train = fma(di, di, train);
    }
  }
  return train;
}

struct Res2Start {  // one start's view inside the CTA
  double2 *G, *phi, *chi, *scr;
  double *red, *buf;  // [CW_WARPS][32] pass partials; [2][16][32] cluster partials (by rank)
  uint64_t *mbar;     // [2] (gate parity)
  double2 *gglob;
  int j, s, M, cnt, m0;
};

size_t res2_fixed_bytes(int K) {
  size_t b = 2 * (size_t)K * 16 * sizeof(double2)            // gate tables
             + 2 * (CW_WARPS * 32 + 2 * 16 * 32) * sizeof(double)  // red, buf
             + 40 * sizeof(double)                           // cost reduction
             + 4 * sizeof(uint64_t)                          // mbarriers
             + 2 * 64 * sizeof(double2)                      // polar scratch
             + (size_t)K * (sizeof(int2) + sizeof(int));
  return (b + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(RES_THREADS, 1) res_pair_kernel(const ResParams P) {
  extern __shared__ __align__(QFS_RES_ALIGN) unsigned char smem_raw[];
  const int K = P.K, n = P.n;
  const unsigned N = 1u << n, ld = (unsigned)P.ld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned rank = cl_rank(), C = cl_size();
  // carve (offsets from the __shared__ base: LDS/STS addressing)
  size_t off = 0;
  double2 *Gt[2];
  Gt[0] = (double2 *)(smem_raw + off); off += (size_t)K * 16 * sizeof(double2);
  Gt[1] = (double2 *)(smem_raw + off); off += (size_t)K * 16 * sizeof(double2);
  double *redt[2], *buft[2];
  redt[0] = (double *)(smem_raw + off); off += CW_WARPS * 32 * sizeof(double);
  redt[1] = (double *)(smem_raw + off); off += CW_WARPS * 32 * sizeof(double);
  buft[0] = (double *)(smem_raw + off); off += 2 * 16 * 32 * sizeof(double);
  buft[1] = (double *)(smem_raw + off); off += 2 * 16 * 32 * sizeof(double);
  double *cred = (double *)(smem_raw + off); off += 40 * sizeof(double);
  uint64_t *mbar = (uint64_t *)(smem_raw + off); off += 4 * sizeof(uint64_t);
  double2 *scrt[2];
  scrt[0] = (double2 *)(smem_raw + off); off += 64 * sizeof(double2);
  scrt[1] = (double2 *)(smem_raw + off); off += 64 * sizeof(double2);
  int2 *pr = (int2 *)(smem_raw + off); off += (size_t)K * sizeof(int2);
  int *kinds = (int *)(smem_raw + off); off += (size_t)K * sizeof(int);
  off = (off + 15) & ~(size_t)15;
  double2 *st0 = (double2 *)(smem_raw + off);
  const size_t SZ = (size_t)ld << n;  // one [2^n][ld] state block

  if (tid == 0) {
    for (int q = 0; q < 4; ++q) mbar_init(mbar + q, 1);
    mbar_fence_init();
  }
  pdl_wait();
  for (int k = tid; k < K; k += RES_THREADS) {
    pr[k] = P.pairs[k];
    kinds[k] = P.kinds ? P.kinds[k] : 0;
  }
  cl_arrive();  // the mbarriers are initialised before any CTA of the cluster pushes to them
  cl_wait();
  unsigned mph = 0;  // PW: parity bits of the two mbarriers of its start (bit g: gate parity g)

  const int n_pairs = (P.n_slots + 1) / 2;
  for (int pj = (int)cl_id(); pj < n_pairs; pj += (int)cl_count()) {
    Res2Start S[2];
    const bool hasB = 2 * pj + 1 < P.n_slots;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      Res2Start &t = S[x];
      t.j = 2 * pj + x;
      const bool present = x == 0 || hasB;
      const Slot sl = present ? P.slots[t.j] : Slot{};
      t.s = present ? sl.s : 0;
      t.M = present ? sl.m : 0;
      t.m0 = (int)rank * (int)ld;
      t.cnt = max(0, min((int)ld, t.M - t.m0));
      t.G = Gt[x]; t.red = redt[x]; t.buf = buft[x]; t.scr = scrt[x]; t.mbar = mbar + 2 * x;
      t.phi = st0 + (2 * x) * SZ;
      t.chi = st0 + (2 * x + 1) * SZ;
      t.gglob = P.gates + (long long)t.s * K * 16;
    }
    const FastDiv fdA((unsigned)max(S[0].cnt, 1)), fdB((unsigned)max(S[1].cnt, 1));
#pragma unroll
    for (int x = 0; x < 2; ++x) {  // (unrolled: S[] stays in registers)
      if (x == 1 && !hasB) continue;
      for (int q = tid; q < K * 16; q += RES_THREADS) S[x].G[q] = S[x].gglob[q];
      for (unsigned q = tid; q < N * (unsigned)S[x].cnt; q += RES_THREADS) {
        const unsigned a = q / (unsigned)S[x].cnt, jj = q - a * (unsigned)S[x].cnt;
        const long long gi = (long long)a * P.m_pool + S[x].m0 + jj;
        S[x].phi[a * ld + jj] = __ldg(P.x + gi);
        S[x].chi[a * ld + jj] = __ldg(P.y + gi);
      }
    }
    __syncthreads();
    // forward with the previous sweep's gates, both starts: phi = B_{K-1}
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      if (x == 1 && !hasB) continue;
      const FastDiv &fd = x ? fdB : fdA;
      int k = 0;
      for (; k + 2 < K; k += 2) {
        res_apply_pair(S[x].phi, S[x].G + 16 * k, pr[k], S[x].G + 16 * (k + 1), pr[k + 1], S[x].cnt, fd, ld, n, tid,
                       RES_THREADS);
        __syncthreads();
      }
      if (k + 1 < K) {
        res_apply(S[x].phi, S[x].G + 16 * k, pr[k], false, S[x].cnt, fd, ld, n, tid, RES_THREADS);
        __syncthreads();
      }
    }
    // ---- backward, right to left, roles as above ----
    double train[2] = {0.0, 0.0};
    if (warp == PW_A || warp == PW_B) {
      auto pw_run = [&](Res2Start &t, const int ENV, const int GATE) {
        for (int i = K - 1; i >= 0; --i) {
          const int par = i & 1;
          nb_sync(ENV, CW_THREADS + 32);  // the pass warps' partials of E_i are in t.red
          double e = 0.0;
#pragma unroll
          for (int w = 0; w < CW_WARPS; ++w) e += t.red[w * 32 + lane];
          if (lane == 0) mbar_arrive_tx(t.mbar + par, C * 32 * (unsigned)sizeof(double));
          __syncwarp();
          for (unsigned c = 0; c < C; ++c) st_async_remote_d(t.buf + par * 512 + rank * 32 + lane, t.mbar + par, c, e);
          mbar_wait(t.mbar + par, (mph >> par) & 1u);
          mph ^= 1u << par;
          e = 0.0;
          for (unsigned c = 0; c < C; ++c) e += t.buf[par * 512 + c * 32 + lane];  // rank order
          const int l = lane & 15;
          double2 ev = make_double2(__shfl_sync(FULL, e, 2 * l), __shfl_sync(FULL, e, 2 * l + 1));
          double2 *gi = t.G + 16 * i;
          if (P.env_trace && rank == 0 && lane < 16) P.env_trace[((long long)i * P.S + t.s) * 16 + l] = ev;
          const int kind = kinds[i];
          double2 g, v;
          double ss;
          gate_update(kind, ev, gi, P.beta, nullptr, g, v, ss, t.scr + 2 * (lane & 16), P.sig != nullptr);
          __syncwarp();
          if (lane < 16 && kind != 1) gi[l] = g;
          if (rank == 0) {
            if (lane < 16 && kind != 1) t.gglob[16 * i + l] = g;
            if (lane == 0 && P.sig) P.sig[(long long)t.s * K + i] = ss;
          }
          nb_arrive(GATE, CW_THREADS + 32);  // new G_i in the gate table
        }
      };
      if (warp == PW_A) pw_run(S[0], NB_ENV_A, NB_GATE_A);
      else if (hasB) pw_run(S[1], NB_ENV_B, NB_GATE_B);
    } else {
      const int ct = tid - 32 - (warp > PW_B ? 32 : 0);  // 0 .. CW_THREADS-1
      const int cw = ct >> 5;
      auto env = [&](int x, int i) {
        res_env_sub(S[x].phi, S[x].chi, pr[i], S[x].cnt, x ? fdB : fdA, ld, n, ct, CW_THREADS, S[x].red + cw * 32);
        nb_arrive(x ? NB_ENV_B : NB_ENV_A, CW_THREADS + 32);
      };
      env(0, K - 1);
      if (hasB) env(1, K - 1);
      for (int i = K - 1; i >= 0; --i) {
        nb_sync(NB_CW, CW_THREADS);  // E_i passes of both starts done reading phi / chi
        if (i > 0) {  // uncompute B_{i-1} = G_{i-1}^dag B_i with the old G_{i-1}
          res_apply(S[0].phi, S[0].G + 16 * (i - 1), pr[i - 1], true, S[0].cnt, fdA, ld, n, ct, CW_THREADS);
          if (hasB) res_apply(S[1].phi, S[1].G + 16 * (i - 1), pr[i - 1], true, S[1].cnt, fdB, ld, n, ct, CW_THREADS);
        }
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (x == 1 && !hasB) continue;
          nb_sync(x ? NB_GATE_B : NB_GATE_A, CW_THREADS + 32);  // new G_i of start x
          if (i > 0)
            res_apply(S[x].chi, S[x].G + 16 * i, pr[i], true, S[x].cnt, x ? fdB : fdA, ld, n, ct, CW_THREADS);
          else
            train[x] = res_chi0_cost(S[x].chi, S[x].G, pr[0], S[x].cnt, x ? fdB : fdA, ld, n, P.x, P.m_pool,
                                     S[x].m0, ct, CW_THREADS);
          nb_sync(NB_CW, CW_THREADS);  // chi_x(i) and phi_x(i-1) complete
          if (i > 0) env(x, i - 1);
        }
      }
    }
    __syncthreads();
    // validation cost with the post-sweep gates, per start:
    // this CTA's rows v = rank, rank + C, ... in batches of ld rows (phi buffer)
    double val[2] = {0.0, 0.0};
    if (P.want_val && P.V > 0) {
      const int rows = (P.V - (int)rank + (int)C - 1) / (int)C;
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (x == 1 && !hasB) continue;
        for (int b0 = 0; b0 < rows; b0 += (int)ld) {
          const int nb = min((int)ld, rows - b0);
          for (unsigned q = tid; q < N * (unsigned)nb; q += RES_THREADS) {
            const unsigned jj = q / N, a = q - jj * N;
            const long long row = (long long)rank + (long long)C * (b0 + jj);
            S[x].phi[a * ld + jj] = __ldg(P.xv + row * N + a);
          }
          __syncthreads();
          const FastDiv fdv((unsigned)nb);
          int k = 0;
          for (; k + 1 < K; k += 2) {
            res_apply_pair(S[x].phi, S[x].G + 16 * k, pr[k], S[x].G + 16 * (k + 1), pr[k + 1], nb, fdv, ld, n, tid,
                           RES_THREADS);
            __syncthreads();
          }
          if (k < K) {
            res_apply(S[x].phi, S[x].G + 16 * k, pr[k], false, nb, fdv, ld, n, tid, RES_THREADS);
            __syncthreads();
          }
          for (unsigned q = tid; q < N * (unsigned)nb; q += RES_THREADS) {
            const unsigned jj = q / N, a = q - jj * N;
            const long long row = (long long)rank + (long long)C * (b0 + jj);
            const double2 u = S[x].phi[a * ld + jj], w = __ldg(P.yv + row * N + a);
            const double dr = u.x - w.x, di = u.y - w.y;
            val[x] = fma(dr, dr, val[x]);
            val[x] = fma(di, di, val[x]);
          }
          __syncthreads();
        }
      }
    }
    // costs: threads -> warps (in order) -> CTA -> cluster ranks (in order)
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const double t = warp_sum(train[x]), v = warp_sum(val[x]);
      if (lane == 0) {
        cred[(2 * x) * RES_WARPS + warp] = t;
        cred[(2 * x + 1) * RES_WARPS + warp] = v;
      }
    }
    __syncthreads();
    if (tid < 4) {  // cost (tid & 1: validation) of start tid >> 1
      double a = 0.0;
      for (int w = 0; w < RES_WARPS; ++w) a += cred[tid * RES_WARPS + w];
      cred[32 + tid] = a;
    }
    cl_arrive();
    cl_wait();
    if (rank == 0 && tid < (hasB ? 4 : 2)) {
      const int j = 2 * pj + (tid >> 1);
      double a = 0.0;
      for (unsigned c = 0; c < C; ++c) a += ld_remote(cred + 32 + tid, c);
      if ((tid & 1) == 0) P.csum[j] = a;
      else if (P.want_val && P.V > 0) P.cval[j] = a;
    }
    // the next pair rewrites the gate tables and cred: every CTA waits until
    // rank 0 has read the remote costs
    cl_arrive();
    cl_wait();
  }
  pdl_trigger();
}

// Validation cost of the streamed path: one CTA per (start,
// block of ld validation rows); the rows sit in shared memory as a [2^n][ld]
// block (same layout and gate routine as the resident sweep), all K
// post-sweep gates are applied in order, then each row's ||C xv - yv||^2 goes
// to row_out[j][row] (summed over rows in row order by row_reduce_kernel).
// MINB = 2: two CTAs per SM (<= 128 registers, one gate per pass); MINB = 1
// (when the rows' shared memory admits one CTA per SM anyway, e.g. C4's
// ld = 2): two gates per shared-memory pass, half the passes and barriers.
template <int MINB>
__global__ void __launch_bounds__(RES_THREADS, MINB) val_blk_kernel(const ValRowParams P, int ld) {
  extern __shared__ __align__(QFS_RES_ALIGN) unsigned char smem_raw[];
  __shared__ double red[RES_WARPS];
  const int K = P.K, n = P.n;
  const unsigned N = 1u << n;
  double2 *G = (double2 *)smem_raw;
  int2 *pr = (int2 *)(G + K * 16);
  double2 *st = (double2 *)(smem_raw + (((size_t)K * (16 * sizeof(double2) + sizeof(int2)) + 15) & ~(size_t)15));
  const int j = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * ld, nb = min(ld, P.rows - r0);
  for (unsigned q = tid; q < N * (unsigned)nb; q += RES_THREADS) {
    const unsigned jj = q / N, a = q - jj * N;
    st[a * ld + jj] = __ldg(P.xv + (long long)(r0 + jj) * N + a);
  }
  for (int k = tid; k < K; k += RES_THREADS) pr[k] = P.pairs[k];
  pdl_wait();  // the gates are the ones the backward pass just wrote
  const int s = P.slots[j].s;
  for (int q = tid; q < K * 16; q += RES_THREADS) G[q] = P.gates[(long long)s * K * 16 + q];
  __syncthreads();
  const FastDiv fdv((unsigned)nb);
  int k0 = 0;
  if constexpr (MINB == 1) {
    for (; k0 + 1 < K; k0 += 2) {
      res_apply_pair(st, G + 16 * k0, pr[k0], G + 16 * (k0 + 1), pr[k0 + 1], nb, fdv, (unsigned)ld, n, tid,
                     RES_THREADS);
      __syncthreads();
    }
  }
  for (int k = k0; k < K; ++k) {
    res_apply(st, G + 16 * k, pr[k], false, nb, fdv, (unsigned)ld, n, tid, RES_THREADS);
    __syncthreads();
  }
  for (int jj = 0; jj < nb; ++jj) {
    double acc = 0.0;
    const double2 *yr = P.yv + (long long)(r0 + jj) * N;
    for (unsigned a = tid; a < N; a += RES_THREADS) {
      const double2 u = st[a * ld + jj], w = __ldg(yr + a);
      const double dr = u.x - w.x, di = u.y - w.y;
      acc = fma(dr, dr, acc);
      acc = fma(di, di, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < RES_WARPS; ++w) t += red[w];
      P.row_out[(long long)j * P.rows + r0 + jj] = t;
    }
    __syncthreads();
  }
}

// st.shared::cluster of a complex value into CTA `rank` at the same offset
__device__ __forceinline__ void st_remote_c(double2 *p, unsigned rank, double2 v) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 ld_remote_c(const double2 *p, unsigned rank) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(ra) : "memory");
  return v;
}
__device__ __forceinline__ void cl_sync() {
  cl_arrive();
  cl_wait();
}

// Validation for rows too large for one CTA (n = 14: 256 KB): a cluster of C =
// 2^t CTAs (t <= 2 unless shared memory needs 3) holds one row, CTA c the amplitudes whose top t qubits read c.  A
// gate off the top qubits is applied by each CTA to its slice (the block
// routine with n-t local qubits); a gate touching a top qubit is applied to
// quadruples split evenly between the CTAs, members read / written locally or
// over DSMEM, between cluster barriers.  Then each row's ||C xv - yv||^2
// (slices summed in rank order) goes to row_out[j][row].
__global__ void __launch_bounds__(RES_THREADS, 1) val_cl_kernel(const ValRowParams P, int t) {
  extern __shared__ __align__(QFS_RES_ALIGN) unsigned char smem_raw[];
  __shared__ double red[RES_WARPS];
  __shared__ double half_sum_v;
  const int K = P.K, n = P.n;
  const unsigned C = 1u << t, NH = 1u << (n - t), top = (unsigned)(n - t);
  double2 *G = (double2 *)smem_raw;
  int2 *pr = (int2 *)(G + K * 16);
  double2 *st = (double2 *)(smem_raw + (((size_t)K * (16 * sizeof(double2) + sizeof(int2)) + 15) & ~(size_t)15));
  const unsigned rank = cl_rank();
  const int row = blockIdx.x >> t, j = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double2 *xr = P.xv + ((long long)row << n) + (long long)rank * NH;
  for (unsigned a = tid; a < NH; a += RES_THREADS) st[a] = __ldg(xr + a);
  for (int k = tid; k < K; k += RES_THREADS) pr[k] = P.pairs[k];
  pdl_wait();  // the gates are the ones the backward pass just wrote
  const int s = P.slots[j].s;
  for (int q = tid; q < K * 16; q += RES_THREADS) G[q] = P.gates[(long long)s * K * 16 + q];
  __syncthreads();
  const FastDiv one(1u);
  for (int k = 0; k < K; ++k) {
    const int2 pq = pr[k];
    if ((unsigned)max(pq.x, pq.y) < top) {
      res_apply(st, G + 16 * k, pq, false, 1, one, 1u, n - t, tid, RES_THREADS);
      __syncthreads();
      continue;
    }
    cl_sync();  // the partner's half is complete
    const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
    const double2 *g = G + 16 * k;
    const unsigned nq = NH >> 2;  // quadruples per CTA (N/4 = C NH/4 in total)
    for (unsigned q = tid; q < nq; q += RES_THREADS) {
      const unsigned r = rank * nq + q;
      const unsigned base = insert_zero32(insert_zero32(r, lo), hi);
      unsigned own[4], loc[4];
      double2 v[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const unsigned a = base | ((unsigned)(l & 1) << pq.x) | ((unsigned)(l >> 1) << pq.y);
        own[l] = a >> top;
        loc[l] = a & (NH - 1);
        v[l] = own[l] == rank ? st[loc[l]] : ld_remote_c(st + loc[l], own[l]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < 4; ++b) cfma(o, g[4 * a + b], v[b]);
        if (own[a] == rank) st[loc[a]] = o;
        else st_remote_c(st + loc[a], own[a], o);
      }
    }
    cl_sync();  // both halves updated before anyone reads them
  }
  double acc = 0.0;
  const double2 *yr = P.yv + ((long long)row << n) + (long long)rank * NH;
  for (unsigned a = tid; a < NH; a += RES_THREADS) {
    const double2 u = st[a], w = __ldg(yr + a);
    const double dr = u.x - w.x, di = u.y - w.y;
    acc = fma(dr, dr, acc);
    acc = fma(di, di, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < RES_WARPS; ++w) t += red[w];
    half_sum_v = t;
  }
  cl_sync();
  if (rank == 0 && tid == 0) {
    double t_sum = 0.0;
    for (unsigned c = 0; c < C; ++c) t_sum += ld_remote(&half_sum_v, c);
    P.row_out[(long long)j * P.rows + row] = t_sum;
  }
  cl_sync();  // rank 1 stays resident until rank 0 has read its sum
}

}  // namespace

size_t val_cl_smem(int n, int K, int t) {
  return (((size_t)K * 16 * sizeof(double2) + (size_t)K * sizeof(int2) + 15) & ~(size_t)15) +
         ((size_t)1 << (n - t)) * sizeof(double2);
}

cudaError_t launch_val_cluster(const ValRowParams &p, int n_slots, cudaStream_t st) {
  constexpr size_t lim = RES_SMEM_MAX - 256;
  // cluster of 2^t CTAs per row: the smallest that fits, widened (up to 8)
  // while the rows of all starts still fit on the 148 SMs
  // measured at n = 14 (C5, S = 1 / 2 / 4): 4-CTA clusters beat 8-CTA ones
  // (fewer gates on distributed qubits) even with half the SMs idle
  int t = 1;
  while (t < 3 && val_cl_smem(p.n, p.K, t) > lim) ++t;
  while (t < 2 && (long long)p.rows * n_slots * (2 << t) <= 148) ++t;
  if (const char *e = getenv("QFS_VAL_CL_T")) {  // diagnostic override (A/B of the cluster width)
    const int tt = atoi(e);
    if (tt >= 1 && tt <= 3 && val_cl_smem(p.n, p.K, tt) <= lim) t = tt;
  }
  const size_t smem = val_cl_smem(p.n, p.K, t);
  if (smem > lim) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(val_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.rows << t, n_slots);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 1u << t;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, val_cl_kernel, p, t);
}

size_t val_blk_smem(int n, int K, int ld) {
  return (((size_t)K * 16 * sizeof(double2) + (size_t)K * sizeof(int2) + 15) & ~(size_t)15) +
         ((size_t)ld << n) * sizeof(double2);
}

cudaError_t launch_val_block(const ValRowParams &p, int n_slots, cudaStream_t st) {
  // rows per CTA: the most that fit in shared memory, reduced while the grid
  // has fewer CTAs than half the SMs
  constexpr size_t lim = RES_SMEM_MAX - 256;  // the kernel's static reduction array sits beside it
  int ld = 1;
  while (ld < p.rows && val_blk_smem(p.n, p.K, ld + 1) <= lim) ++ld;
  // (fewer, fuller CTAs down to half the SMs: C4, 16 x 16 rows, ld = 2 beats 1 by 3 %)
  while (ld > 1 && (long long)((p.rows + ld - 1) / ld) * n_slots < 74) --ld;
  if (const char *e = getenv("QFS_VAL_BLK_LD")) {  // diagnostic override (A/B)
    const int l = atoi(e);
    if (l >= 1 && l <= p.rows && val_blk_smem(p.n, p.K, l) <= lim) ld = l;
  }
  const size_t smem = val_blk_smem(p.n, p.K, ld);
  if (smem > lim) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(val_blk_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    cudaFuncSetAttribute(val_blk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lim);
    attr = true;
  }
#ifndef QFS_VAL_PAIRS
#define QFS_VAL_PAIRS 1
#endif
  // one CTA per SM either way (shared memory over half the SM's): the pair variant
  const bool one = QFS_VAL_PAIRS && smem + 1024 > RES_SMEM_MAX2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.rows + ld - 1) / ld, n_slots);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return one ? cudaLaunchKernelEx(&cfg, val_blk_kernel<1>, p, ld) : cudaLaunchKernelEx(&cfg, val_blk_kernel<2>, p, ld);
}

size_t res_smem_bytes(int n, int K, int ld) {
  size_t b = (size_t)K * 16 * sizeof(double2) + (RES_WARPS * 32 + (QFS_RES_PUSH ? 2 * 16 * 32 : 64) + 2) * sizeof(double) +
             64 * sizeof(double2) + (size_t)K * (sizeof(int2) + sizeof(int));
  b = (b + 15) & ~(size_t)15;
  b += 2 * ((size_t)ld << n) * sizeof(double2) + 32;  // (+ mbarriers and their alignment)
  return b;
}
int resident_max_clusters_query(int C, size_t smem);
size_t res_smem_limit(int minb) { return minb >= 2 ? RES_SMEM_MAX2 : RES_SMEM_MAX; }

namespace {
template <int MINB>
void res_set_attrs() {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(res_sweep_kernel<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)res_smem_limit(MINB));
    cudaFuncSetAttribute(res_sweep_kernel<MINB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
}
}  // namespace

int resident_max_clusters(int C, size_t smem) {
  // cudaOccupancyMaxActiveClusters is slow (it is queried at every graph
  // capture, and captures follow every change of the active-start set): cache
  // per (cluster size, shared memory)
  // per (cluster size, shared memory); contexts may be driven from several host threads
  static std::map<std::pair<int, size_t>, int> cache;
  static std::mutex mu;
  const auto key = std::make_pair(C, smem);
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int r = resident_max_clusters_query(C, smem);
  cache[key] = r;
  return r;
}

int resident_max_clusters_query(int C, size_t smem) {
  const int minb = smem <= RES_SMEM_MAX2 ? 2 : 1;
  if (minb == 2) res_set_attrs<2>();
  else res_set_attrs<1>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 148);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  int num = 0;
  const cudaError_t e = minb == 2 ? cudaOccupancyMaxActiveClusters(&num, res_sweep_kernel<2>, &cfg)
                                  : cudaOccupancyMaxActiveClusters(&num, res_sweep_kernel<1>, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return num;
}

size_t res2_smem_bytes(int n, int K, int ld) { return res2_fixed_bytes(K) + 4 * ((size_t)ld << n) * sizeof(double2); }

int resident2_max_clusters(int C, size_t smem) {
  static std::map<std::pair<int, size_t>, int> cache;
  static std::mutex mu;
  const auto key = std::make_pair(C, smem);
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(res_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RES_SMEM_MAX);
    cudaFuncSetAttribute(res_pair_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 148);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  int num = 0;
  if (cudaOccupancyMaxActiveClusters(&num, res_pair_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    num = 0;
  }
  cache[key] = num;
  return num;
}

cudaError_t launch_resident_pair(const ResParams &p, int clusters, cudaStream_t st) {
  const size_t smem = res2_smem_bytes(p.n, p.K, p.ld);
  resident2_max_clusters(p.C, smem);  // sets the function attributes
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.C * clusters);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = p.C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, res_pair_kernel, p);
}

cudaError_t launch_resident(const ResParams &p, int clusters, cudaStream_t st) {
  const size_t smem = res_smem_bytes(p.n, p.K, p.ld);
  resident_max_clusters(p.C, smem);  // sets the function attributes
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.C * clusters);
  cfg.blockDim = dim3(RES_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = p.C;
  a[0].val.clusterDim.y = 1;
  a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return smem <= RES_SMEM_MAX2 ? cudaLaunchKernelEx(&cfg, res_sweep_kernel<2>, p)
                               : cudaLaunchKernelEx(&cfg, res_sweep_kernel<1>, p);
}

}  // namespace qfs
