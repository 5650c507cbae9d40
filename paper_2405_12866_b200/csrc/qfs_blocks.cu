// qfs_blocks.cu — sm_100a kernels for circuits of multi-qubit blocks
// (qfs_create_blocks; "possibly
// multi-qubit" unitary gates, updated without parameterisation).
//
// A block of arity A in {2, 3} acts on qubits q_0..q_{A-1} (as given; local
// index l = sum_j b(q_j) 2^j) with a d x d matrix, d = 2^A.  The sweep is the
// streamed algorithm of qfs_kernels.cu in its
// plain form — one launch per step, no fusion:
//   forward   B_{k+1} = G_k B_k                         (blk_apply_kernel)
//   backward  chi <- G_{i+1}^dag chi                    (blk_apply_kernel, dagger)
//             E_i = sum phi (x) conj(chi), ordered reduction, last CTA runs the
//             gate update (d = 4: the half-warp polar of qfs_device.cuh;
//             d = 8: warp Newton-Schulz polar below)   (blk_env_kernel)
//   cost      sum ||a - b||^2, ordered reduction         (blk_dist_kernel)
// States use the Views of qfs_internal.h (sample-minor work buffers).  No
// code here is shared with the CPU oracle.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "qfs_device.cuh"
#include "qfs_internal.h"

namespace qfs {
namespace {

// per-start ticket with acquire-release semantics at GPU scope (the last-CTA
// election without separate fences, as warp0_elect_last in qfs_kernels.cu)
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned *counter) {
  unsigned t;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(counter) : "memory");
  return t;
}

constexpr int BLK_THREADS = 128;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// first amplitude of block-group r: zeros inserted at the sorted qubit positions
template <int A>
__device__ __forceinline__ unsigned blk_base(unsigned r, const int (&srt)[3]) {
#pragma unroll
  for (int j = 0; j < A; ++j) r = insert_zero32(r, srt[j]);
  return r;
}

struct BlkLocal {
  int q[3], srt[3];
  unsigned off[8];  // amplitude offset of local index l (sum_j b_j 2^{q_j})
};
template <int A>
__device__ __forceinline__ BlkLocal blk_local(const BlkGate &g) {
  BlkLocal b;
#pragma unroll
  for (int j = 0; j < 3; ++j) b.q[j] = b.srt[j] = g.q[j];
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int j = i + 1; j < A; ++j)
      if (b.srt[j] < b.srt[i]) { int t = b.srt[i]; b.srt[i] = b.srt[j]; b.srt[j] = t; }
#pragma unroll
  for (int l = 0; l < (1 << A); ++l) {
    unsigned o = 0;
#pragma unroll
    for (int j = 0; j < A; ++j) o |= (unsigned)((l >> j) & 1) << b.q[j];
    b.off[l] = o;
  }
  return b;
}

// shared-memory load the compiler may not hoist out of the item loop (a
// hoisted 8x8 gate would take 256 registers)
__device__ __forceinline__ double2 lds_c(const double2 *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// --------------------------------------------------------------- apply --
// dst = G_k src (dagger: G_k^dag) for every (group, row) of every slot.
template <int A>
__global__ void __launch_bounds__(BLK_THREADS) blk_apply_kernel(const BlkApplyParams P) {
  constexpr int D = 1 << A;
  __shared__ double2 sG[D * D];
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned rows = P.rows_fixed > 0 ? (unsigned)P.rows_fixed : (unsigned)sl.m;
  const BlkGate bg = P.bg[P.k];
  const double2 *gk = P.gates + (long long)s * P.gsz + bg.off;
  for (int e = threadIdx.x; e < D * D; e += blockDim.x) {
    const int a = e / D, b = e % D;
    sG[e] = P.dagger ? cconj(gk[D * b + a]) : gk[e];  // (G^dag)[a][b] = conj(G[b][a])
  }
  __syncthreads();
  const BlkLocal L = blk_local<A>(bg);
  const unsigned items = (1u << (P.n - A)) * rows;
  const unsigned chunk = (items + gridDim.x - 1) / gridDim.x;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fd(rows);
  const double2 *src = P.src.base + (long long)s * P.src.ss;
  double2 *dst = P.dst.base + (long long)s * P.dst.ss;
  auto load = [&](unsigned w, double2 (&v)[D]) {
    const unsigned r = fd.div(w), m = w - r * rows;  // row fastest: coalesced sample-minor access
    const unsigned base = blk_base<A>(r, L.srt);
#pragma unroll
    for (int l = 0; l < D; ++l) v[l] = src[(long long)(base | L.off[l]) * P.src.sa + (long long)m * P.src.sm];
  };
  double2 vn[D];  // next item's amplitudes, loaded while this one computes
  if (beg + threadIdx.x < end) load(beg + threadIdx.x, vn);
  for (unsigned w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const unsigned r = fd.div(w), m = w - r * rows;
    const unsigned base = blk_base<A>(r, L.srt);
    double2 v[D];
#pragma unroll
    for (int l = 0; l < D; ++l) v[l] = vn[l];
    if (w + blockDim.x < end) load(w + blockDim.x, vn);
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double2 o = make_double2(0.0, 0.0);
#pragma unroll
      for (int b = 0; b < D; ++b) cfma(o, lds_c(&sG[D * a + b]), v[b]);
      dst[(long long)(base | L.off[a]) * P.dst.sa + (long long)m * P.dst.sm] = o;
    }
  }
}

// ------------------------------------------------------------ 8x8 polar --
// Unitary polar factor W of the 8x8 complex E' on one warp (lane holds
// entries lane and lane + 32, row-major), Newton-Schulz X <- X (3I - X^dag X)/2
// from X_0 = E' sqrt(2.9 / ||E'^dag E'||_F): every singular value of X_0 is
// then below sqrt(2.9) < sqrt(3), where the iteration converges (to W for a
// nonsingular E').  Stops when ||X^dag X - I||_F <= 1e-14; returns false if it
// does not within 60 iterations (singular or very ill-conditioned E').  G = W^dag = Y X^dag (eq:opt_u,
// P:59-62, with E' = X D Y^dag), sum sigma = Re Tr(W^dag E').
__device__ __noinline__ bool polar8(const double2 (&e)[2], double2 (&g)[2], double &ss, double2 *sm /*[2][64]*/) {
  const int lane = threadIdx.x & 31;
  double2 *sX = sm, *sT = sm + 64;
  auto xhx = [&](const double2 (&X)[2], double2 (&Y)[2]) {  // Y = X^dag X, X left in sX
    __syncwarp();
    sX[lane] = X[0];
    sX[lane + 32] = X[1];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (lane >> 3) + 4 * h, c = lane & 7;
      double2 y = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) cfma(y, cconj(sX[8 * q + r]), sX[8 * q + c]);
      Y[h] = y;
    }
  };
  double2 x[2] = {e[0], e[1]}, y[2];
  xhx(x, y);
  const double fy = sqrt(warp_sum_d(y[0].x * y[0].x + y[0].y * y[0].y + y[1].x * y[1].x + y[1].y * y[1].y));
  if (!(fy > 0.0)) return false;
  const double sc = sqrt(2.9 / fy);
  x[0].x *= sc; x[0].y *= sc; x[1].x *= sc; x[1].y *= sc;
  bool ok = false;
  for (int it = 0; it < 60; ++it) {
    xhx(x, y);
    double err = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (lane >> 3) + 4 * h, c = lane & 7;
      const double dr = y[h].x - (r == c ? 1.0 : 0.0);
      err += dr * dr + y[h].y * y[h].y;
    }
    err = warp_sum_d(err);
    if (err <= 1e-28) { ok = true; break; }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (lane >> 3) + 4 * h, c = lane & 7;
      sT[lane + 32 * h] = make_double2(0.5 * ((r == c ? 3.0 : 0.0) - y[h].x), -0.5 * y[h].y);
    }
    __syncwarp();
    double2 z[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = (lane >> 3) + 4 * h, c = lane & 7;
      z[h] = make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < 8; ++q) cfma(z[h], sX[8 * r + q], sT[8 * q + c]);
    }
    x[0] = z[0];
    x[1] = z[1];
  }
  // G[r][c] = conj(W[c][r]);  sum sigma = Re sum conj(W) o E'
  __syncwarp();
  sX[lane] = x[0];
  sX[lane + 32] = x[1];
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = (lane >> 3) + 4 * h, c = lane & 7;
    g[h] = cconj(sX[8 * c + r]);
  }
  ss = warp_sum_d(x[0].x * e[0].x + x[0].y * e[0].y + x[1].x * e[1].x + x[1].y * e[1].y);
  return ok;
}


// Fallback for environments Newton-Schulz cannot handle (singular or very
// ill-conditioned E'): one-sided Jacobi on a warp, the 8-column analogue of
// hw_polar (qfs_device.cuh).  Lane l holds rows l>>3 and (l>>3)+4 of column
// c = l & 7 of A = E' V and of V (V_0 = I); round x = 1..7 rotates the
// disjoint column pairs (c, c ^ x) (the 28 pairs of a sweep), until no pair has
// |gamma| > 1e-12 ||a_j|| ||a_k||; sigma_j = ||a_j||, X_j = a_j / sigma_j, null
// columns (sigma_j <= 1e-14 sigma_max) completed by Gram-Schmidt on e_0..e_7
// (as the oracle), G = V X^dag (eq:opt_u), sum sigma.
__device__ __noinline__ void polar8_jacobi(const double2 (&e)[2], double2 (&g)[2], double &ss, double2 *sm) {
  const int lane = threadIdx.x & 31, c = lane & 7, r0 = lane >> 3;
  double mx = fmax(fmax(fabs(e[0].x), fabs(e[0].y)), fmax(fabs(e[1].x), fabs(e[1].y)));
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  const int ex = mx > 0.0 ? ilogb(mx) : 0;
  double2 a[2], v[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    a[h] = make_double2(scalbn(e[h].x, -ex), scalbn(e[h].y, -ex));
    v[h] = make_double2(r0 + 4 * h == c ? 1.0 : 0.0, 0.0);
  }
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool big = false;
#pragma unroll 1
    for (int x = 1; x < 8; ++x) {
      const bool lo = c < (c ^ x);
      double2 aj[2], ak[2], vj[2], vk[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 ap = shfl_xor_c(a[h], x), vp = shfl_xor_c(v[h], x);
        aj[h] = lo ? a[h] : ap; ak[h] = lo ? ap : a[h];
        vj[h] = lo ? v[h] : vp; vk[h] = lo ? vp : v[h];
      }
      double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        al += aj[h].x * aj[h].x + aj[h].y * aj[h].y;
        be += ak[h].x * ak[h].x + ak[h].y * ak[h].y;
        gr += aj[h].x * ak[h].x + aj[h].y * ak[h].y;
        gi += aj[h].x * ak[h].y - aj[h].y * ak[h].x;
      }
#pragma unroll
      for (int o = 8; o <= 16; o <<= 1) {
        al += __shfl_xor_sync(FULL, al, o);
        be += __shfl_xor_sync(FULL, be, o);
        gr += __shfl_xor_sync(FULL, gr, o);
        gi += __shfl_xor_sync(FULL, gi, o);
      }
      const double ag2 = gr * gr + gi * gi, ab = al * be;
      big = big || ag2 > 1e-24 * ab;
      if (ag2 > 0.0 && ag2 > 1e-30 * ab) {  // rotation of hw_polar (rsqrt form)
        const double D = be - al, q4 = 4.0 * ag2, w = fma(D, D, q4), R = w * rsqrt(w);
        const double den = fabs(D) + R, rr = rsqrt(fma(den, den, q4)), cc = den * rr;
        const double f2 = (D >= 0.0 ? 2.0 : -2.0) * rr, spr = f2 * gr, spi = f2 * gi;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (lo) {
            a[h] = make_double2(cc * aj[h].x - (spr * ak[h].x + spi * ak[h].y), cc * aj[h].y - (spr * ak[h].y - spi * ak[h].x));
            v[h] = make_double2(cc * vj[h].x - (spr * vk[h].x + spi * vk[h].y), cc * vj[h].y - (spr * vk[h].y - spi * vk[h].x));
          } else {
            a[h] = make_double2((spr * aj[h].x - spi * aj[h].y) + cc * ak[h].x, (spr * aj[h].y + spi * aj[h].x) + cc * ak[h].y);
            v[h] = make_double2((spr * vj[h].x - spi * vj[h].y) + cc * vk[h].x, (spr * vj[h].y + spi * vj[h].x) + cc * vk[h].y);
          }
        }
      }
    }
    if (!__any_sync(FULL, big)) break;
  }
  double nn = a[0].x * a[0].x + a[0].y * a[0].y + a[1].x * a[1].x + a[1].y * a[1].y;
  nn += __shfl_xor_sync(FULL, nn, 8);
  nn += __shfl_xor_sync(FULL, nn, 16);
  const double sig = sqrt(nn);
  double smax = sig;
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) smax = fmax(smax, __shfl_xor_sync(FULL, smax, o));
  const bool nul = !(sig > 1e-14 * smax) || smax == 0.0;
  double2 *sX = sm, *sV = sm + 64;
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int idx = 8 * (r0 + 4 * h) + c;
    sX[idx] = nul ? make_double2(0.0, 0.0) : make_double2(a[h].x / sig, a[h].y / sig);
    sV[idx] = v[h];
  }
  __syncwarp();
  const unsigned nm = __ballot_sync(FULL, nul && r0 == 0) & 0xffu;  // bit c: column c null
  if (nm && lane == 0) {
    for (int jj = 0; jj < 8; ++jj) {
      if (!((nm >> jj) & 1)) continue;
      for (int e0 = 0; e0 < 8; ++e0) {
        double2 u[8];
        for (int q = 0; q < 8; ++q) u[q] = make_double2(q == e0 ? 1.0 : 0.0, 0.0);
        for (int pass = 0; pass < 2; ++pass)
          for (int q = 0; q < 8; ++q) {
            if (q == jj || (((nm >> q) & 1) && q > jj)) continue;
            double2 d = make_double2(0.0, 0.0);
            for (int rr = 0; rr < 8; ++rr) cfma(d, cconj(sX[8 * rr + q]), u[rr]);
            for (int rr = 0; rr < 8; ++rr) {
              const double2 t = cmul(d, sX[8 * rr + q]);
              u[rr].x -= t.x;
              u[rr].y -= t.y;
            }
          }
        double nv = 0.0;
        for (int rr = 0; rr < 8; ++rr) nv += u[rr].x * u[rr].x + u[rr].y * u[rr].y;
        nv = sqrt(nv);
        if (nv > 0.5) {
          for (int rr = 0; rr < 8; ++rr) sX[8 * rr + jj] = make_double2(u[rr].x / nv, u[rr].y / nv);
          break;
        }
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // G[r][c] = sum_q V[r][q] conj(X[c][q])
    const int r = r0 + 4 * h;
    double2 t = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) cfma(t, sV[8 * r + q], cconj(sX[8 * c + q]));
    g[h] = t;
  }
  double sg = r0 == 0 ? sig : 0.0;  // one lane per column
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) sg += __shfl_xor_sync(FULL, sg, o);
  ss = scalbn(sg, ex);
}

// ---------------------------------------------------------- environment --
// E_i[l_in][l_out] = sum_m sum_r phi_m[idx_r(l_in)] conj(chi_m[idx_r(l_out)])
// (R4): per-thread accumulators, warp butterflies, warps in order,
// CTA partials summed in CTA order by the last CTA (ticket), which then runs
// the gate update of gate i and writes G_i, sum sigma and the environment trace.
template <int A>
__global__ void __launch_bounds__(BLK_THREADS) blk_env_kernel(const BlkEnvParams P) {
  constexpr int D = 1 << A, DD = D * D, NW = BLK_THREADS / 32;
  __shared__ double2 red[NW][DD];
  __shared__ double2 sE[DD];
  __shared__ double2 scratch[128];
  __shared__ unsigned last_cta;
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned rows = (unsigned)sl.m;
  const BlkGate bg = P.bg[P.i];
  const BlkLocal L = blk_local<A>(bg);
  // PARTS lanes share an item, each owning XR rows of E (64 complex
  // accumulators would take 256 registers for d = 8)
#ifndef QFS_BLK_ENV_PARTS
#define QFS_BLK_ENV_PARTS 4
#endif
#ifndef QFS_BLK_ENV_PF
#define QFS_BLK_ENV_PF 1  // items loaded ahead of the one accumulating
#endif
  constexpr int PARTS = A == 3 ? QFS_BLK_ENV_PARTS : 1, XR = D / PARTS;
  const int part = threadIdx.x % PARTS;
  double2 acc[XR * D];
#pragma unroll
  for (int e = 0; e < XR * D; ++e) acc[e] = make_double2(0.0, 0.0);
  const unsigned items = (1u << (P.n - A)) * rows;
  const unsigned chunk = (items + gridDim.x - 1) / gridDim.x;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fd(rows);
  const double2 *ph = P.phi.base + (long long)s * P.phi.ss;
  const double2 *ch = P.chi.base + (long long)s * P.chi.ss;
  auto load = [&](unsigned w, double2 (&f)[XR], double2 (&c)[D]) {
    const unsigned r = fd.div(w), m = w - r * rows;
    const unsigned base = blk_base<A>(r, L.srt);
#pragma unroll
    for (int x = 0; x < XR; ++x)
      f[x] = ph[(long long)(base | L.off[part * XR + x]) * P.phi.sa + (long long)m * P.phi.sm];
#pragma unroll
    for (int l = 0; l < D; ++l) c[l] = ch[(long long)(base | L.off[l]) * P.chi.sa + (long long)m * P.chi.sm];
  };
  const unsigned step = blockDim.x / PARTS;
  double2 fn[XR], cn[D];  // next item's amplitudes, loaded while this one accumulates
  if (beg + threadIdx.x / PARTS < end) load(beg + threadIdx.x / PARTS, fn, cn);
#if QFS_BLK_ENV_PF == 2
  double2 fn2[XR], cn2[D];  // the item after it
  if (beg + threadIdx.x / PARTS + step < end) load(beg + threadIdx.x / PARTS + step, fn2, cn2);
#endif
  for (unsigned w = beg + threadIdx.x / PARTS; w < end; w += step) {
    double2 f[XR], c[D];
#pragma unroll
    for (int x = 0; x < XR; ++x) f[x] = fn[x];
#pragma unroll
    for (int l = 0; l < D; ++l) c[l] = cn[l];
#if QFS_BLK_ENV_PF == 2
#pragma unroll
    for (int x = 0; x < XR; ++x) fn[x] = fn2[x];
#pragma unroll
    for (int l = 0; l < D; ++l) cn[l] = cn2[l];
    if (w + 2 * step < end) load(w + 2 * step, fn2, cn2);
#else
    if (w + step < end) load(w + step, fn, cn);
#endif
#pragma unroll
    for (int x = 0; x < XR; ++x)
#pragma unroll
      for (int y = 0; y < D; ++y) {
        double2 &e = acc[D * x + y];  // f[x] conj(c[y]), row part * XR + x of E
        e.x = fma(f[x].x, c[y].x, e.x);
        e.x = fma(f[x].y, c[y].y, e.x);
        e.y = fma(f[x].y, c[y].x, e.y);
        e.y = fma(-f[x].x, c[y].y, e.y);
      }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < XR * D; ++e) {  // sum over the lanes of this part (xor offsets keep lane % PARTS)
    double re = acc[e].x, im = acc[e].y;
#pragma unroll
    for (int o = 16; o >= PARTS; o >>= 1) {
      re += __shfl_xor_sync(FULL, re, o);
      im += __shfl_xor_sync(FULL, im, o);
    }
    if (lane < PARTS) red[warp][part * XR * D + e] = make_double2(re, im);
  }
  __syncthreads();
  double2 *cta_part = reinterpret_cast<double2 *>(P.partials) + ((long long)j * gridDim.x + blockIdx.x) * DD;
  for (int e = threadIdx.x; e < DD; e += blockDim.x) {
    double2 t = make_double2(0.0, 0.0);
#pragma unroll
    for (int w = 0; w < NW; ++w) { t.x += red[w][e].x; t.y += red[w][e].y; }
    cta_part[e] = t;
  }
  // the CTA barrier orders every thread's partial store before thread 0's
  // release (cumulative); the last CTA's acquire orders the partial loads of
  // all its threads through the next barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atom_add_acq_rel(P.counters + j);
    last_cta = t == gridDim.x - 1 ? 1u : 0u;
    if (last_cta) P.counters[j] = 0u;
  }
  __syncthreads();
  if (!last_cta) return;
  const double2 *pp = reinterpret_cast<const double2 *>(P.partials) + (long long)j * gridDim.x * DD;
  for (int e = threadIdx.x; e < DD; e += blockDim.x) {
    double2 t = make_double2(0.0, 0.0);
    for (unsigned b = 0; b < gridDim.x; ++b) {
      const double2 v = __ldcg(pp + (long long)b * DD + e);
      t.x += v.x;
      t.y += v.y;
    }
    sE[e] = t;
  }
  __syncthreads();
  if (warp != 0) return;
  const long long gi = (long long)s * P.gsz + bg.off;
  double2 *gw = P.gates + gi;
  if (P.env_trace)  // gate-major trace: gate i of start s at S * off_i + s * d^2
    for (int e = lane; e < DD; e += 32) P.env_trace[(long long)P.S * bg.off + (long long)s * DD + e] = sE[e];
  double ss = 0.0;
  if constexpr (D == 4) {
    const int l = lane & 15;
    double2 g, v;
    gate_update(bg.kind, sE[l], gw, P.beta, nullptr, g, v, ss, scratch + 2 * (lane & 16), P.sig != nullptr);
    __syncwarp();
    if (lane < 16 && bg.kind != 1) gw[l] = g;
  } else {
    if (bg.kind == 1) {  // fixed: sum sigma slot = Re Tr(E G)
      double t = 0.0;
      for (int e = lane; e < DD; e += 32) {
        const int a = e / D, b = e % D;
        const double2 gg = gw[D * b + a];
        t += sE[e].x * gg.x - sE[e].y * gg.y;
      }
      ss = warp_sum_d(t);
    } else {
      double2 e2[2], g2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h, a = e / D, b = e % D;
        e2[h] = sE[e];
        if (P.beta != 0.0) {  // E' = (1 - beta) E + beta G_old^dag
          const double2 go = gw[D * b + a];
          e2[h] = make_double2((1.0 - P.beta) * e2[h].x + P.beta * go.x, (1.0 - P.beta) * e2[h].y - P.beta * go.y);
        }
      }
      if (!polar8(e2, g2, ss, scratch)) polar8_jacobi(e2, g2, ss, scratch);
      __syncwarp();
      // row-major G: lane holds entries lane (row lane>>3) and lane + 32 (row 4 + lane>>3)
      gw[lane] = g2[0];
      gw[lane + 32] = g2[1];
    }
  }
  if (lane == 0 && P.sig) P.sig[(long long)s * P.K + P.i] = ss;
}

// ---------------------------------------------------------------- cost --
// out[j] = sum over rows and amplitudes of ||a - b||^2 (P:116-120 direct form;
// P:184 validation), ordered: lanes, warps, CTAs.
__global__ void __launch_bounds__(BLK_THREADS) blk_dist_kernel(const BlkDistParams P) {
  constexpr int NW = BLK_THREADS / 32;
  __shared__ double red[NW];
  __shared__ unsigned last_cta;
  const int j = blockIdx.y;
  const Slot sl = P.slots[j];
  const int s = sl.s;
  const unsigned rows = P.rows_fixed > 0 ? (unsigned)P.rows_fixed : (unsigned)sl.m;
  const unsigned items = (1u << P.n) * rows;
  const unsigned chunk = (items + gridDim.x - 1) / gridDim.x;
  const unsigned beg = blockIdx.x * chunk, end = min(items, beg + chunk);
  const FastDiv fd(rows);
  const double2 *a = P.a.base + (long long)s * P.a.ss, *b = P.b.base + (long long)s * P.b.ss;
  double acc = 0.0;
  for (unsigned w = beg + threadIdx.x; w < end; w += blockDim.x) {
    const unsigned amp = fd.div(w), m = w - amp * rows;
    const double2 u = a[(long long)amp * P.a.sa + (long long)m * P.a.sm];
    const double2 v = b[(long long)amp * P.b.sa + (long long)m * P.b.sm];
    const double dr = u.x - v.x, di = u.y - v.y;
    acc = fma(dr, dr, acc);
    acc = fma(di, di, acc);
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w];
    P.partials[(long long)j * gridDim.x + blockIdx.x] = t;
    const unsigned tk = atom_add_acq_rel(P.counters + j);
    last_cta = tk == gridDim.x - 1 ? 1u : 0u;
    if (last_cta) {
      P.counters[j] = 0u;
      double tot = 0.0;
      for (unsigned c = 0; c < gridDim.x; ++c) tot += __ldcg(P.partials + (long long)j * gridDim.x + c);
      P.out[j] = tot;
    }
  }
}

// ---------------------------------------------------------- gate check --
// finite (bit 1) and unitary to 1e-10 (bit 2) for every block of every start
__global__ void blk_gate_check_kernel(const double2 *g, const BlkGate *bg, int K, long long gsz, int s,
                                      unsigned *flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)s * K;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(t % K);
    const long long st = t / K;
    const int D = 1 << bg[k].a;
    const double2 *G = g + st * gsz + bg[k].off;
    unsigned bad = 0;
    for (int e = 0; e < D * D; ++e)
      if (!isfinite(G[e].x) || !isfinite(G[e].y)) bad |= 1u;
    for (int a = 0; a < D && !bad; ++a)
      for (int b = 0; b < D; ++b) {
        double re = 0.0, im = 0.0;
        for (int r = 0; r < D; ++r) {  // conj(G[r][a]) G[r][b]
          re += G[D * r + a].x * G[D * r + b].x + G[D * r + a].y * G[D * r + b].y;
          im += G[D * r + a].x * G[D * r + b].y - G[D * r + a].y * G[D * r + b].x;
        }
        if (fabs(re - (a == b ? 1.0 : 0.0)) > 1e-10 || fabs(im) > 1e-10) bad |= 2u;
      }
    if (bad) atomicOr(flag, bad);
  }
}

int blk_grid(long long items, int n_slots) {
  long long nb = std::max(1, kBlkMaxCtas / std::max(1, n_slots));
  nb = std::min(nb, (items + BLK_THREADS - 1) / BLK_THREADS);
  return (int)std::max(1LL, std::min<long long>(nb, kBlkMaxCtas));
}

}  // namespace

int blk_ctas(long long items, int n_slots) { return blk_grid(items, n_slots); }

cudaError_t launch_blk_apply(const BlkApplyParams &p, int arity, int nb, int n_slots, cudaStream_t st) {
  dim3 grid(nb, n_slots);
  if (arity == 3) blk_apply_kernel<3><<<grid, BLK_THREADS, 0, st>>>(p);
  else blk_apply_kernel<2><<<grid, BLK_THREADS, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_blk_env(const BlkEnvParams &p, int arity, int nb, int n_slots, cudaStream_t st) {
  dim3 grid(nb, n_slots);
  if (arity == 3) blk_env_kernel<3><<<grid, BLK_THREADS, 0, st>>>(p);
  else blk_env_kernel<2><<<grid, BLK_THREADS, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_blk_dist(const BlkDistParams &p, int nb, int n_slots, cudaStream_t st) {
  blk_dist_kernel<<<dim3(nb, n_slots), BLK_THREADS, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_blk_gate_check(const double2 *g, const BlkGate *bg, int K, long long gsz, int s, unsigned *flag,
                                  cudaStream_t st) {
  const long long cnt = (long long)s * K;
  if (cnt <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>((cnt + 127) / 128, 148 * 4);
  blk_gate_check_kernel<<<(unsigned)blocks, 128, 0, st>>>(g, bg, K, gsz, s, flag);
  return cudaGetLastError();
}

}  // namespace qfs
