// qfs_kernels.cu — sm_100a kernels of the QFactor-Sample sweep (arXiv 2405.12866).
//
// Hot path of one sweep (§3):
//   fwd_row_kernel / fwd_gate_kernel : B_{k+1} = G_k B_k (the B tensors)
//   bwd_kernel                       : chi <- G_{i+1}^dag chi fused with the
//                                      environment E_i = sum phi (x) conj(chi)
//                                      and, in its last CTA per start, the one-warp
//                                      Jacobi polar update u = Y X^dag (eq:opt_u P:59-62)
//   final_kernel                     : chi <- G_0^dag chi, c_train = (1/M) sum ||chi - x||^2
//   fwd_row_kernel (mode 1)          : validation cost
// All arithmetic is FP64 (complex128).  Every reduction runs in a fixed order
// (per-thread -> warp shuffle -> CTA -> CTA partials summed in index order by
// the last CTA), so results are deterministic for a given launch shape.
//
// No code here is shared with the CPU oracle (oracle/qfso.cpp).
#include <cuda_runtime.h>
#include <stdint.h>

#include "qfs_internal.h"

namespace qfs {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int BWD_THREADS = 256;
constexpr int FWD_THREADS = 512;
constexpr int RED_THREADS = 256;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc += a * b
__device__ __forceinline__ void cfma(double2 &acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__device__ __forceinline__ long long insert_zero(long long v, int pos) {
  long long low = v & ((1LL << pos) - 1);
  return ((v >> pos) << (pos + 1)) | low;
}

// ------------------------------------------------------------ warp polar --
// One-warp one-sided (Hestenes) Jacobi SVD of the 4x4 complex A (shared
// memory, overwritten), followed by G = V X^dag (eq:opt_u: E = X D Y^dag,
// u = Y X^dag with Y = V).  Rounds rotate two disjoint column pairs at once
// ((0,1)(2,3) / (0,2)(1,3) / (0,3)(1,2)); 8 lanes hold one matrix row of the
// pair each (A and V rows); the 2x2 rotation follows the classical formulas
//   zeta = (beta - alpha) / (2|gamma|), t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)),
//   c = 1/sqrt(1 + t^2), s = c t,  [a_j a_k] <- [a_j a_k] [[c, s e^{i phi}], [-s e^{-i phi}, c]]
// with gamma = a_j^dag a_k = |gamma| e^{i phi}.  Converged when no pair has
// |gamma| > 1e-15 ||a_j|| ||a_k||.  Columns with sigma <= 1e-14 sigma_max are
// null; X is completed there by Gram-Schmidt on e_0..e_3 (R5).
__device__ void warp_polar(double2 *sA, double2 *sV, double2 *sX, double2 *sG, double *sig_sum,
                           int lane) {
  if (lane < 16) sV[lane] = make_double2((lane % 5 == 0) ? 1.0 : 0.0, 0.0);
  __syncwarp();
  const int p = (lane >> 2) & 1, r = lane & 3;
  const bool act = lane < 8;
  for (int sweep = 0; sweep < 24; ++sweep) {
    bool any = false;
#pragma unroll 1
    for (int rho = 0; rho < 3; ++rho) {
      int j, k;
      if (rho == 0) { j = 2 * p; k = 2 * p + 1; }
      else if (rho == 1) { j = p; k = p + 2; }
      else { j = p; k = 3 - p; }
      double2 aj = sA[4 * r + j], ak = sA[4 * r + k];
      double2 vj = sV[4 * r + j], vk = sV[4 * r + k];
      double al = aj.x * aj.x + aj.y * aj.y;
      double be = ak.x * ak.x + ak.y * ak.y;
      double gr = aj.x * ak.x + aj.y * ak.y;
      double gi = aj.x * ak.y - aj.y * ak.x;
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        al += __shfl_xor_sync(FULL, al, o);
        be += __shfl_xor_sync(FULL, be, o);
        gr += __shfl_xor_sync(FULL, gr, o);
        gi += __shfl_xor_sync(FULL, gi, o);
      }
      const double ag = sqrt(gr * gr + gi * gi);
      const bool rot = act && ag > 0.0 && ag > 1e-15 * sqrt(al) * sqrt(be);
      __syncwarp();
      if (rot) {
        const double rag = 1.0 / ag;
        const double zeta = (be - al) * 0.5 * rag;
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        const double pr = gr * rag, pi = gi * rag;
        // conj(ph) * a_k and ph * a_j
        double2 ca = make_double2(pr * ak.x + pi * ak.y, pr * ak.y - pi * ak.x);
        double2 pa = make_double2(pr * aj.x - pi * aj.y, pr * aj.y + pi * aj.x);
        sA[4 * r + j] = make_double2(c * aj.x - s * ca.x, c * aj.y - s * ca.y);
        sA[4 * r + k] = make_double2(s * pa.x + c * ak.x, s * pa.y + c * ak.y);
        double2 cv = make_double2(pr * vk.x + pi * vk.y, pr * vk.y - pi * vk.x);
        double2 pv = make_double2(pr * vj.x - pi * vj.y, pr * vj.y + pi * vj.x);
        sV[4 * r + j] = make_double2(c * vj.x - s * cv.x, c * vj.y - s * cv.y);
        sV[4 * r + k] = make_double2(s * pv.x + c * vk.x, s * pv.y + c * vk.y);
      }
      any |= (__any_sync(FULL, rot) != 0);
      __syncwarp();
    }
    if (!any) break;
  }
  // singular values = column norms
  double nn = 0.0;
  if (lane < 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 a = sA[4 * q + lane];
      nn += a.x * a.x + a.y * a.y;
    }
  }
  const double sig = sqrt(nn);
  double sg[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) sg[q] = __shfl_sync(FULL, sig, q);
  const double smax = fmax(fmax(sg[0], sg[1]), fmax(sg[2], sg[3]));
  bool nul[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) nul[q] = !(sg[q] > 1e-14 * smax) || smax == 0.0;
  if (lane < 16) {
    const int jj = lane & 3;
    double2 a = sA[lane];
    sX[lane] = nul[jj] ? make_double2(0.0, 0.0) : make_double2(a.x / sg[jj], a.y / sg[jj]);
  }
  __syncwarp();
  if (lane == 0 && (nul[0] || nul[1] || nul[2] || nul[3])) {
    for (int j = 0; j < 4; ++j) {
      if (!nul[j]) continue;
      for (int e = 0; e < 4; ++e) {
        double2 v[4];
        for (int q = 0; q < 4; ++q) v[q] = make_double2(q == e ? 1.0 : 0.0, 0.0);
        for (int pass = 0; pass < 2; ++pass)
          for (int q = 0; q < 4; ++q) {
            if (q == j || (nul[q] && q > j)) continue;
            double2 d = make_double2(0.0, 0.0);
            for (int rr = 0; rr < 4; ++rr) cfma(d, cconj(sX[4 * rr + q]), v[rr]);
            for (int rr = 0; rr < 4; ++rr) {
              double2 t = cmul(d, sX[4 * rr + q]);
              v[rr].x -= t.x;
              v[rr].y -= t.y;
            }
          }
        double nv = 0.0;
        for (int rr = 0; rr < 4; ++rr) nv += v[rr].x * v[rr].x + v[rr].y * v[rr].y;
        nv = sqrt(nv);
        if (nv > 0.5) {
          for (int rr = 0; rr < 4; ++rr) sX[4 * rr + j] = make_double2(v[rr].x / nv, v[rr].y / nv);
          break;
        }
      }
    }
  }
  __syncwarp();
  if (lane < 16) {
    const int a = lane >> 2, b = lane & 3;
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) cfma(acc, sV[4 * a + q], cconj(sX[4 * b + q]));
    sG[lane] = acc;
  }
  if (lane == 0) *sig_sum = sg[0] + sg[1] + sg[2] + sg[3];
  __syncwarp();
}

// E' = (1 - beta) E + beta G_old^dag into sA, then polar; result written to
// gate slot gout (global) and the optional monitors.
__device__ void polar_from_reduced(const double *e32 /*smem or global, 32 doubles*/,
                                   double2 *gout, double beta, double *sig_out,
                                   double2 *env_out, double2 *sA, double2 *sV, double2 *sX,
                                   double2 *sG, double *sSig, int lane) {
  if (lane < 16) {
    double2 e = make_double2(e32[2 * lane], e32[2 * lane + 1]);
    if (env_out) env_out[lane] = e;
    if (beta != 0.0) {
      const int a = lane >> 2, b = lane & 3;
      double2 go = gout[4 * b + a];  // (G^dag)[a][b] = conj(G[b][a])
      e = make_double2((1.0 - beta) * e.x + beta * go.x, (1.0 - beta) * e.y - beta * go.y);
    }
    sA[lane] = e;
  }
  __syncwarp();
  warp_polar(sA, sV, sX, sG, sSig, lane);
  if (lane < 16) gout[lane] = sG[lane];
  if (lane == 0 && sig_out) *sig_out = *sSig;
}

// Sum NV per-thread values over the CTA: warp shuffles, then warps in order.
// Result in out[0..NV) (shared), valid after the trailing __syncthreads.
template <int NV>
__device__ void block_sum(double (&acc)[NV], double *red /*[nwarps][NV]*/, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if (lane == 0) red[warp * NV + q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NV; q += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += red[w * NV + q];
    out[q] = v;
  }
  __syncthreads();
}

// Last-CTA election for the per-start reduction of CTA partials.
__device__ bool elect_last(unsigned *counter, unsigned nb) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(counter, 1u);
    last = (t == nb - 1);
    if (last) *counter = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// local index v of member l of the P-quadruple w (compile-time)
template <int NU, int TP0, int TP1>
__device__ constexpr int pv(int w, int l) {
  int v = ((l & 1) << TP0) | (((l >> 1) & 1) << TP1);
  int bit = 0;
  for (int t = 0; t < NU; ++t) {
    if (t == TP0 || t == TP1) continue;
    v |= ((w >> bit) & 1) << t;
    ++bit;
  }
  return v;
}

// ---------------------------------------------------------------- backward --
// Gate i of the right-to-left sweep (Fig. env_calc):
//   if UPD: chi <- G_{i+1}^dag chi on the Q pair (local bits 0,1)
//   E_i[a][b] += phi[idx_P(a)] conj(chi[idx_P(b)]) on the P pair (local TP0,TP1)
// Each thread owns whole 2^NU-amplitude groups, so the chi update is in place
// and race-free.  CTA partials -> last CTA per start reduces in CTA order and
// (fuse_polar) runs the one-warp polar update of gate i.
template <int NU, int TP0, int TP1, bool UPD>
__global__ void __launch_bounds__(BWD_THREADS) bwd_kernel(const BwdParams P) {
  constexpr int NV = 1 << NU;
  constexpr int NQ = NV / 4;
  __shared__ double2 sQ[16];
  __shared__ double red[(BWD_THREADS / 32) * 32];
  __shared__ double sum32[32];
  __shared__ double2 sA[16], sV[16], sX[16], sG[16];
  __shared__ double sSig;

  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const int lgG = P.n - NU;
  const long long N = 1LL << P.n;
  const long long items = (long long)sl.m << lgG;
  const long long chunk = (items + P.nb - 1) / P.nb;
  const long long beg = (long long)blockIdx.x * chunk;
  const long long end = min(items, beg + chunk);

  if (UPD && threadIdx.x < 16) {
    const int a = threadIdx.x >> 2, b = threadIdx.x & 3;
    const double2 g = P.gates[((long long)s * P.K + P.upd_gate) * 16 + 4 * b + a];
    sQ[threadIdx.x] = cconj(g);  // (G^dag)[a][b]
  }
  __syncthreads();

  double acc[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) acc[q] = 0.0;

  const double2 *csrc = P.chi_src.base + (long long)s * P.chi_src.stride_s * N;
  double2 *cdst = P.chi_dst.base ? P.chi_dst.base + (long long)s * P.chi_dst.stride_s * N : nullptr;
  const double2 *fsrc = P.phi.base + (long long)s * P.phi.stride_s * N;

  for (long long w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const long long m = w >> lgG;
    long long g = w & ((1LL << lgG) - 1);
#pragma unroll
    for (int t = 0; t < NU; ++t) g = insert_zero(g, P.ins[t]);
    const long long rowoff = m * N + g;
    double2 c[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) c[v] = csrc[rowoff + P.off[v]];
    if (UPD) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double2 o[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          o[a] = make_double2(0.0, 0.0);
#pragma unroll
          for (int b = 0; b < 4; ++b) cfma(o[a], sQ[4 * a + b], c[4 * q + b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) c[4 * q + a] = o[a];
      }
      if (cdst) {
#pragma unroll
        for (int v = 0; v < NV; ++v) cdst[rowoff + P.off[v]] = c[v];
      }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double2 f[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) f[l] = fsrc[rowoff + P.off[pv<NU, TP0, TP1>(q, l)]];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double2 cb = c[pv<NU, TP0, TP1>(q, b)];
          // f[a] * conj(cb)
          acc[8 * a + 2 * b] = fma(f[a].x, cb.x, acc[8 * a + 2 * b]);
          acc[8 * a + 2 * b] = fma(f[a].y, cb.y, acc[8 * a + 2 * b]);
          acc[8 * a + 2 * b + 1] = fma(f[a].y, cb.x, acc[8 * a + 2 * b + 1]);
          acc[8 * a + 2 * b + 1] = fma(-f[a].x, cb.y, acc[8 * a + 2 * b + 1]);
        }
    }
  }

  block_sum<32>(acc, red, sum32);
  if (threadIdx.x < 32)
    P.partials[((long long)j * P.nb + blockIdx.x) * 32 + threadIdx.x] = sum32[threadIdx.x];
  if (!elect_last(&P.counters[j], (unsigned)P.nb)) return;
  if (threadIdx.x < 32) {
    double e = 0.0;
    const double *pp = P.partials + (long long)j * P.nb * 32 + threadIdx.x;
    for (int b = 0; b < P.nb; ++b) e += __ldcg(pp + (long long)b * 32);
    sum32[threadIdx.x] = e;
    if (!P.fuse_polar) P.e_red[(long long)j * 32 + threadIdx.x] = e;
  }
  __syncthreads();
  if (!P.fuse_polar || threadIdx.x >= 32) return;
  double2 *gout = P.gates_w + ((long long)s * P.K + P.env_gate) * 16;
  polar_from_reduced(sum32, gout, P.beta, P.sig ? P.sig + (long long)s * P.K + P.env_gate : nullptr,
                     P.env_trace ? P.env_trace + ((long long)P.env_gate * P.S + s) * 16 : nullptr,
                     sA, sV, sX, sG, &sSig, threadIdx.x);
}

// polar step alone (sample-sharded mode, after the NCCL all-reduce of E)
__global__ void polar_kernel(const PolarParams P) {
  __shared__ double2 sA[4][16], sV[4][16], sX[4][16], sG[4][16];
  __shared__ double sSig[4];
  __shared__ double e32[4][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + w;
  if (j >= P.n_slots) return;
  const Slot sl = P.slots[j];
  e32[w][lane] = P.e_red[(long long)j * 32 + lane];
  __syncwarp();
  double2 *gout = P.gates + ((long long)sl.s * P.K + P.gate) * 16;
  polar_from_reduced(e32[w], gout, P.beta, P.sig ? P.sig + (long long)sl.s * P.K + P.gate : nullptr,
                     P.env_trace ? P.env_trace + ((long long)P.gate * P.S + sl.s) * 16 : nullptr,
                     sA[w], sV[w], sX[w], sG[w], &sSig[w], lane);
}

// --------------------------------------------------------------- final cost --
__global__ void __launch_bounds__(RED_THREADS) final_kernel(const FinalParams P) {
  __shared__ double2 sQ[16];
  __shared__ double red[RED_THREADS / 32];
  __shared__ double tot;
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const long long N = 1LL << P.n;
  const long long items = (long long)sl.m << (P.n - 2);
  const long long chunk = (items + P.nb - 1) / P.nb;
  const long long beg = (long long)blockIdx.x * chunk, end = min(items, beg + chunk);
  if (threadIdx.x < 16) {
    const int a = threadIdx.x >> 2, b = threadIdx.x & 3;
    sQ[threadIdx.x] = cconj(P.gates[(long long)s * P.K * 16 + 4 * b + a]);
  }
  __syncthreads();
  const int lo = min(P.p0, P.p1), hi = max(P.p0, P.p1);
  const long long o1 = 1LL << P.p0, o2 = 1LL << P.p1;
  const double2 *c = P.chi.base + (long long)s * P.chi.stride_s * N;
  const double2 *x = P.x.base + (long long)s * P.x.stride_s * N;
  double acc = 0.0;
  for (long long w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const long long m = w >> (P.n - 2);
    const long long r = w & ((1LL << (P.n - 2)) - 1);
    const long long base = m * N + insert_zero(insert_zero(r, lo), hi);
    const long long off[4] = {0, o1, o2, o1 | o2};
    double2 v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = __ldcg(c + base + off[l]);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(o, sQ[4 * a + b], v[b]);
      const double2 xv = __ldcs(x + base + off[a]);
      const double dr = o.x - xv.x, di = o.y - xv.y;
      acc = fma(dr, dr, acc);
      acc = fma(di, di, acc);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    P.partials[(long long)j * P.nb + blockIdx.x] = t;
  }
  if (!elect_last(&P.counters[j], (unsigned)P.nb)) return;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < P.nb; ++b) t += __ldcg(P.partials + (long long)j * P.nb + b);
    P.out_sum[j] = t;
  }
}

// -------------------------------------------------------- forward (rows) ----
// One CTA per (start, row): the whole 2^n row lives in shared memory; the K
// (or K-1) gates are applied in order, gate k+1 is staged while gate k runs.
__global__ void __launch_bounds__(FWD_THREADS) fwd_row_kernel(const FwdRowParams P) {
  extern __shared__ double2 row[];
  __shared__ double2 sG[2][16];
  __shared__ double red[FWD_THREADS / 32];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const int nrows = P.mode == 0 ? sl.m : P.rows;
  const int m = blockIdx.x;
  if (m >= nrows) return;
  const long long N = 1LL << P.n;
  const int ngates = P.mode == 0 ? P.K - 1 : P.K;
  const double2 *src = P.src.base + ((long long)s * P.src.stride_s + m) * N;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) row[i] = __ldcs(src + i);
  const double2 *gs = P.gates + (long long)s * P.K * 16;
  if (threadIdx.x < 16 && ngates > 0) sG[0][threadIdx.x] = gs[threadIdx.x];
  __syncthreads();
  for (int k = 0; k < ngates; ++k) {
    const int2 pr = __ldg(P.pairs + k);
    const double2 *G = sG[k & 1];
    double2 nxt;
    const bool stage = threadIdx.x < 16 && k + 1 < ngates;
    if (stage) nxt = gs[(long long)(k + 1) * 16 + threadIdx.x];
    const int lo = min(pr.x, pr.y), hi = max(pr.x, pr.y);
    const long long o1 = 1LL << pr.x, o2 = 1LL << pr.y;
    double2 *dst = P.mode == 0 ? P.B + (long long)k * P.b_gate_stride +
                                     ((long long)s * P.b_stride_s + m) * N
                               : nullptr;
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
      if (dst) {
#pragma unroll
        for (int a = 0; a < 4; ++a) dst[off[a]] = o[a];
      }
    }
    if (stage) sG[(k + 1) & 1][threadIdx.x] = nxt;
    __syncthreads();
  }
  if (P.mode == 1) {
    const double2 *ref = P.ref.base + ((long long)s * P.ref.stride_s + m) * N;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < N; i += blockDim.x) {
      const double2 a = row[i], b = __ldcs(ref + i);
      const double dr = a.x - b.x, di = a.y - b.y;
      acc = fma(dr, dr, acc);
      acc = fma(di, di, acc);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
      P.row_out[(long long)j * P.rows + m] = t;
    }
  }
}

// ------------------------------------------------------ forward (per gate) --
__global__ void __launch_bounds__(RED_THREADS) fwd_gate_kernel(const FwdGateParams P) {
  __shared__ double2 sG[16];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const int rows = P.rows_fixed > 0 ? P.rows_fixed : sl.m;
  const long long N = 1LL << P.n;
  const long long items = (long long)rows << (P.n - 2);
  const long long chunk = (items + P.nb - 1) / P.nb;
  const long long beg = (long long)blockIdx.x * chunk, end = min(items, beg + chunk);
  if (threadIdx.x < 16) sG[threadIdx.x] = P.gates[((long long)s * P.K + P.k) * 16 + threadIdx.x];
  __syncthreads();
  const int lo = min(P.p0, P.p1), hi = max(P.p0, P.p1);
  const long long o1 = 1LL << P.p0, o2 = 1LL << P.p1;
  const double2 *src = P.src.base + (long long)s * P.src.stride_s * N;
  double2 *dst = P.dst.base + (long long)s * P.dst.stride_s * N;
  for (long long w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const long long m = w >> (P.n - 2);
    const long long r = w & ((1LL << (P.n - 2)) - 1);
    const long long base = m * N + insert_zero(insert_zero(r, lo), hi);
    const long long off[4] = {base, base | o1, base | o2, base | o1 | o2};
    double2 v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = src[off[l]];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < 4; ++b) cfma(o, sG[4 * a + b], v[b]);
      dst[off[a]] = o;
    }
  }
}

// per-row squared distance (streamed validation end)
__global__ void __launch_bounds__(RED_THREADS) dist_kernel(const DistParams P) {
  __shared__ double red[RED_THREADS / 32];
  const int j = blockIdx.y, m = blockIdx.x;
  const Slot sl = P.slots[j];
  const long long N = 1LL << P.n;
  const double2 *a = P.a.base + ((long long)sl.s * P.a.stride_s + m) * N;
  const double2 *b = P.b.base + ((long long)sl.s * P.b.stride_s + m) * N;
  double acc = 0.0;
  for (long long i = threadIdx.x; i < N; i += blockDim.x) {
    const double2 u = a[i], v = b[i];
    const double dr = u.x - v.x, di = u.y - v.y;
    acc = fma(dr, dr, acc);
    acc = fma(di, di, acc);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
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
  if (j >= n_slots) return;
  double t = 0.0;
  for (int r = 0; r < rows; ++r) t += row_in[(long long)j * rows + r];
  out[j] = t;
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

__global__ void polar_batch_kernel(const double2 *env, const double2 *g_old, double beta,
                                   double2 *g_new, double *sig, int count) {
  __shared__ double2 sA[4][16], sV[4][16], sX[4][16], sG[4][16];
  __shared__ double sSig[4];
  __shared__ double e32[4][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + w;
  if (i >= count) return;
  const double *ep = reinterpret_cast<const double *>(env + (long long)i * 16);
  e32[w][lane] = ep[lane];
  if (lane < 16) g_new[(long long)i * 16 + lane] = g_old[(long long)i * 16 + lane];
  __syncwarp();
  polar_from_reduced(e32[w], g_new + (long long)i * 16, beta, sig + i, nullptr, sA[w], sV[w],
                     sX[w], sG[w], &sSig[w], lane);
}

}  // namespace

// ================================================================ launchers ==
int bwd_threads() { return BWD_THREADS; }
int fwd_row_max_n() { return 13; }

cudaError_t launch_bwd(const BwdParams &p, int n_slots, int tp0, int tp1, bool upd,
                       cudaStream_t st) {
  dim3 grid(p.nb, n_slots), block(BWD_THREADS);
#define QFS_BWD(NU, A, B, U) bwd_kernel<NU, A, B, U><<<grid, block, 0, st>>>(p)
  if (!upd) {
    QFS_BWD(2, 0, 1, false);
  } else if (p.nu == 2) {
    if (tp0 == 0) QFS_BWD(2, 0, 1, true);
    else QFS_BWD(2, 1, 0, true);
  } else if (p.nu == 3) {
    if (tp0 == 0 && tp1 == 2) QFS_BWD(3, 0, 2, true);
    else if (tp0 == 2 && tp1 == 0) QFS_BWD(3, 2, 0, true);
    else if (tp0 == 1 && tp1 == 2) QFS_BWD(3, 1, 2, true);
    else QFS_BWD(3, 2, 1, true);
  } else {
    if (tp0 == 2) QFS_BWD(4, 2, 3, true);
    else QFS_BWD(4, 3, 2, true);
  }
#undef QFS_BWD
  return cudaGetLastError();
}

cudaError_t launch_polar(const PolarParams &p, int n_slots, cudaStream_t st) {
  polar_kernel<<<(n_slots + 3) / 4, 128, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_final(const FinalParams &p, int n_slots, cudaStream_t st) {
  final_kernel<<<dim3(p.nb, n_slots), RED_THREADS, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_row(const FwdRowParams &p, int n_slots, int max_rows, cudaStream_t st) {
  const size_t smem = sizeof(double2) << p.n;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(fwd_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         sizeof(double2) << 13);
    attr_set = true;
  }
  fwd_row_kernel<<<dim3(max_rows, n_slots), FWD_THREADS, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fwd_gate(const FwdGateParams &p, int n_slots, cudaStream_t st) {
  fwd_gate_kernel<<<dim3(p.nb, n_slots), RED_THREADS, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dist(const DistParams &p, int n_slots, cudaStream_t st) {
  dist_kernel<<<dim3(p.rows, n_slots), RED_THREADS, 0, st>>>(p);
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
  polar_batch_kernel<<<(count + 3) / 4, 128, 0, st>>>(env, g_old, beta, g_new, sig, count);
  return cudaGetLastError();
}

}  // namespace qfs
