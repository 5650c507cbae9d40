// qfs_device.cuh — device helpers shared by the sm_100a kernels of libqfs
// (qfs_kernels.cu: streamed sweep; qfs_resident.cu: cluster-resident sweep):
// complex FP64 arithmetic, bit insertion, PTX wrappers (LDGSTS, PDL, L2
// hints), and the half-warp polar update of a 4x4 complex environment
// (eq:opt_u).  Internal (anonymous namespace); not part of the ABI.
// No code here is shared with the CPU oracle.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace qfs {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// Debug build (build.py --debug: -DQFS_DEBUG, libqfs_debug.so): device-side
// bounds checks of the streamed kernels' 32-bit offsets (compute-sanitizer is
// closed on this pool).  A failed check traps the kernel (the launch reports
// cudaErrorAssert / a device fault) instead of touching memory out of range.
#ifdef QFS_DEBUG
#define QFS_DASSERT(cond)                                                       \
  do {                                                                          \
    if (!(cond)) {                                                              \
      printf("QFS_DASSERT failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);   \
      __trap();                                                                 \
    }                                                                           \
  } while (0)
#else
#define QFS_DASSERT(cond) \
  do {                    \
  } while (0)
#endif
constexpr int JACOBI_MAX_SWEEPS = 20;

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
__device__ __forceinline__ unsigned insert_zero32(unsigned v, int pos) {
  return ((v >> pos) << (pos + 1)) | (v & ((1u << pos) - 1u));
}

// Division by an invariant d (1 <= d < 2^31) for numerators < 2^31:
// q = (umulhi(n, mul) + n) >> l with l = ceil(log2 d), mul = 2^32 (2^l - d) / d + 1.
struct FastDiv {
  unsigned d, mul;
  int l;
  __device__ explicit FastDiv(unsigned dd) : d(dd) {
    l = 0;
    while ((1u << l) < d) ++l;
    mul = (unsigned)((((unsigned long long)1 << 32) * ((1ull << l) - d)) / d + 1);
  }
  __device__ __forceinline__ unsigned div(unsigned n) const { return (__umulhi(n, mul) + n) >> l; }
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// LDGSTS: 16-byte global -> shared copy without a register round trip
// (zero-filled when !valid); .cg = cached in L2 only.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
// L2 eviction-priority policies (createpolicy) and hinted LDGSTS / stores
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_hint(void *smem, const void *gmem, bool valid, uint64_t pol) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(sa), "l"(gmem), "r"(sz),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_hint(double2 *p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ double2 ld_hint(const double2 *p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol)
               : "memory");
  return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ---- bulk async copies (cp.async.bulk, the TMA engine's non-tensor mode) and
// mbarriers (sm_90+; SASS UBLKCP / SYNCS).  A bulk copy moves one contiguous
// run of bytes (16-byte aligned, multiple of 16) from global to shared memory
// and signals the transaction count of an mbarrier when the bytes have landed.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// make the initialised barriers visible to the async proxy (the copy engine)
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// one arrival + bytes the current phase must still receive
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// wait until the phase with the given parity has completed (try_wait: hardware sleep, not a poll)
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "QFS_MBW%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra QFS_MBW%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on bar (the CTA's own shared memory)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, unsigned bytes, uint64_t *bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// bring a contiguous run into L2 ahead of its bulk copy (no shared memory used)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---- system-scope flags for the device-initiated exchange (peer memory over
// NVLink, or local memory for emulated ranks)
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// 16-byte stores / loads of two self-validating 8-byte words (LL protocol:
// each aligned 8-byte word is single-copy atomic, so a word whose flag half
// carries the current epoch is complete — no fences on the exchange path)
__device__ __forceinline__ void st_ll_sys(unsigned long long *p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_ll_sys(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_ll_gpu(unsigned long long *p, unsigned long long a, unsigned long long b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_ll_gpu(const unsigned long long *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// acquire-release fences (lighter than the sequentially consistent
// __threadfence / __threadfence_system = fence.sc)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ double ld_relaxed_sys(const double *p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-stream-serialization attribute may start while the previous
// kernel on the stream drains; everything before pdl_wait() must not depend on
// that kernel's results.  pdl_trigger() lets the next kernel start launching.
// Both are no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// shared-memory load that is re-issued per use (not hoisted into registers)
__device__ __forceinline__ double2 lds_v2(const double2 *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

__device__ __forceinline__ double2 shfl_c(double2 v, int src) {
  return make_double2(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}
__device__ __forceinline__ double2 shfl_xor_c(double2 v, int m) {
  return make_double2(__shfl_xor_sync(FULL, v.x, m), __shfl_xor_sync(FULL, v.y, m));
}

// ------------------------------------------------------------ polar update --
// Half-warp one-sided (Hestenes) Jacobi SVD and polar factor of a 4x4 complex
// matrix; lane l = 4r + j of each 16-lane half holds A[r][j] and V[r][j] in
// registers (both halves of a warp may work on different matrices).
//
//   A_0 = E' V_0 (V_0 = warm-start right singular vectors, any unitary),
//   rounds rotate the disjoint column pairs (j, j ^ x), x = 1, 2, 3:
//     gamma = a_j^dag a_k = |gamma| e^{i phi},  zeta = (||a_k||^2 - ||a_j||^2) / (2|gamma|),
//     t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)),  c = 1/sqrt(1 + t^2),  s = c t,
//     [a_j a_k] <- [a_j a_k] [[c, s e^{i phi}], [-s e^{-i phi}, c]]   (same on V)
//   rotating every pair with |gamma| > 1e-15 ||a_j|| ||a_k||, and stopping after
//   the first sweep in which no pair had |gamma| > 1e-12 ||a_j|| ||a_k|| (the
//   rotations of that sweep are applied; convergence is quadratic, so the
//   residual is far below 1e-12, and no sweep is spent only to verify it, nor
//   chasing rounding noise near 1e-15); then sigma_j = ||a_j||,
//   X_j = a_j / sigma_j (null columns, sigma_j <= 1e-14 sigma_max, completed by
//   Gram-Schmidt on e_0..e_3; R5) and G = V X^dag (eq:opt_u:
//   E = X D Y^dag, u = Y X^dag with Y = V).  Square roots and divisions are
//   rsqrt-based (MUFU.RSQ64H + Newton) to keep the serial chain short.
// On the Jacobi path E' is scaled by an exact power of two first (the polar factor is scale-free).
// scratch: 32 double2 of shared memory per half warp (Newton-Schulz operands;
// the first 16 also serve the null-column completion).
//
// Fast path first (polar_ns): when E' is far enough from singular, its
// unitary polar factor W = X Y^dag is reached by Newton-Schulz iterations
// instead (same result up to rounding; G = W^dag = Y X^dag).
__device__ __forceinline__ double half_sum(double v) {
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Newton-Schulz polar iteration on a half-warp (lane l = 4r + c holds X[r][c]):
//   X_0 = E' / s, s = ||E'||_F / 2 (RMS singular value),
//   X_{k+1} = X_k (3I - X_k^dag X_k) / 2   ->  W, the unitary polar factor of E'.
// Per singular value u = sigma^2 of X_k, f = u - 1 maps to f' = u(3-u)^2/4 - 1
// = -f^2 (3 - f) / 4, |f'| <= f^2 (3 + |f|) / 4 <= f^2 for 0 < u < 2, so
// e_k = ||X_k^dag X_k - I||_F follows e_{k+1} <= e_k^2 (3 + e_k) / 4: the
// iteration count (k <= 10) is the smallest that takes this bound from e_0 to
// <= 1e-16 (unitary to rounding).  Returns false (nothing written) when e_0 > 0.9647 for either
// half of the warp: the Jacobi path below handles that (ill-conditioned or
// singular E').  The decision and the count are warp-uniform.
// The 4x4 products exchange operands through shared memory (scr: 32 double2
// of this half warp: X at [0, 16), T at [16, 32)): one store and eight
// broadcast-friendly loads per product instead of eight 128-bit shuffles.
__device__ bool polar_ns(double2 e, int hb, int r, int c, double2 &g_out, double &ss_out, double2 *scr,
                         bool need_ss = true) {
  const int l = 4 * r + c;
  double2 *sx = scr, *sT = scr + 16;
  auto xhx = [&](double2 X) {  // (X^dag X)[r][c] = sum_q conj(X[q][r]) X[q][c]; leaves X in sx
    __syncwarp();
    sx[l] = X;
    __syncwarp();
    double2 y = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) cfma(y, cconj(sx[4 * q + r]), sx[4 * q + c]);
    return y;
  };
  // E^dag E on the unscaled E' while the Frobenius norm is reduced (the two
  // overlap): X_0 = rs E', Y_0 = rs^2 E'^dag E', rs = 2 / ||E'||_F
  const double2 yp = xhx(e);
  const double fro2 = half_sum(e.x * e.x + e.y * e.y);
  if (!__all_sync(FULL, fro2 > 0.0)) return false;
  const double rs = 2.0 * rsqrt(fro2), rs2 = rs * rs;
  double2 y = make_double2(yp.x * rs2, yp.y * rs2);
  // iteration 0's product X_0 (3I - Y_0)/2 = rs E' (3I - Y_0)/2 does not depend
  // on e_0 (k >= 1 always): issued before e_0's reduction so the shuffles overlap it
  sT[l] = make_double2(0.5 * ((r == c ? 3.0 : 0.0) - y.x), -0.5 * y.y);
  __syncwarp();
  double2 z0 = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < 4; ++q) cfma(z0, sx[4 * r + q], sT[4 * q + c]);
  z0 = make_double2(z0.x * rs, z0.y * rs);
  double2 x;
  const double dre = y.x - (r == c ? 1.0 : 0.0);
  const double e02 = half_sum(dre * dre + y.y * y.y);  // e_0^2
  // iterations needed: smallest k with g_k <= 1e-16, g_0 = e_0, g_{j+1} =
  // g_j^2 (3 + g_j) / 4 — the exact per-value map is f' = -f^2 (3 - f) / 4, so
  // |f'| <= f^2 (3 + |f|) / 4 and e' <= e^2 (3 + e) / 4 (the plain e' <= e^2
  // bound costs ~0.3 iterations more on average at C3 / C4); thresholds on
  // e_0^2, computed offline by bisection and rounded down
  constexpr double th2[10] = {1.33333e-16, 1.53954e-08, 0.000164733, 0.0164122, 0.151213, 0.425849, 0.682251,
                              0.843214, 0.926897, 0.9305720409296991};
  int k = 11;
#pragma unroll
  for (int q = 9; q >= 0; --q)
    if (e02 <= th2[q]) k = q + 1;
  k = max(k, __shfl_xor_sync(FULL, k, 16));
  if (!__all_sync(FULL, k <= 10)) return false;
  x = z0;
  for (int it = 1; it < k; ++it) {
    y = xhx(x);
    const double2 t = make_double2(0.5 * ((r == c ? 3.0 : 0.0) - y.x), -0.5 * y.y);  // (3I - Y)/2
    sT[l] = t;
    __syncwarp();
    double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) cfma(z, sx[4 * r + q], sT[4 * q + c]);
    x = z;
  }
  // G = W^dag: G[r][c] = conj(W[c][r]);  sum sigma = Re Tr(W^dag E') = Re sum conj(W) o E'
  g_out = cconj(shfl_c(x, hb | (4 * c + r)));
  ss_out = need_ss ? half_sum(x.x * e.x + x.y * e.y) : 0.0;  // (skipped when nobody reads it)
  return true;
}

// v0p: warm start V_0 (row-major, this half's matrix) or nullptr for I; read
// only on the Jacobi path, so the Newton-Schulz path has no global load on the
// critical chain.  Returns true when v_out holds new right singular vectors
// (Jacobi ran), false when V was not touched (Newton-Schulz).
__device__ bool hw_polar(double2 e, const double2 *v0p, double2 &g_out, double2 &v_out, double &sig_sum,
                         double2 *scratch, bool need_ss = true) {
  const int lane = threadIdx.x & 31;
  const int hb = lane & 16;         // half-warp base lane
  const int l = lane & 15;
  const int r = l >> 2, j = l & 3;
#ifdef QFS_DIAG_POLAR
  const long long t_ns = clock64();
#endif
  {
    // Newton-Schulz on E' as is: it is scale-free (X_0 = E'/(||E'||_F/2)) and
    // |E'| <= M 2^n cannot overflow the squares.  (The exact power-of-two
    // prescale used to run first for both paths: ilogb / scalbn on the serial
    // chain cost C4 1.4 %, C5 3 %, C3 3 %, C2 5 %; now only the Jacobi path pays.)
    double ss_ns;
    if (polar_ns(e, hb, r, j, g_out, ss_ns, scratch, need_ss)) {
      sig_sum = ss_ns;
#ifdef QFS_DIAG_POLAR
      sig_sum = 100.0 * 1e7 + (double)(clock64() - t_ns);
#endif
      return false;  // the warm start of the Jacobi path is left as it was
    }
  }
  // Jacobi path: exact power-of-two scaling of E'
  double mx = fmax(fabs(e.x), fabs(e.y));
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  const int ex = mx > 0.0 ? ilogb(mx) : 0;
  e.x = scalbn(e.x, -ex);
  e.y = scalbn(e.y, -ex);
  const double2 v0 = v0p ? v0p[l] : make_double2((l % 5 == 0) ? 1.0 : 0.0, 0.0);
  // A_0 = E' V_0
  double2 a = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < 4; ++q) cfma(a, shfl_c(e, hb | (4 * r + q)), shfl_c(v0, hb | (4 * q + j)));
  double2 v = v0;
#ifdef QFS_DIAG_POLAR
  const long long t_start = clock64();
  int n_sweeps = 0;
#endif
  for (int sweep = 0; sweep < JACOBI_MAX_SWEEPS; ++sweep) {
    bool big = false;  // some pair had |gamma|^2 > 1e-24 ||a_j||^2 ||a_k||^2 this sweep
#ifdef QFS_DIAG_POLAR
    ++n_sweeps;
#endif
#pragma unroll
    for (int x = 1; x <= 3; ++x) {
      const double2 ap = shfl_xor_c(a, x);
      const double2 vp = shfl_xor_c(v, x);
      const bool lo = (j & (x == 1 ? 1 : 2)) == 0;
      const double2 aj = lo ? a : ap, ak = lo ? ap : a;
      const double2 vj = lo ? v : vp, vk = lo ? vp : v;
      double al = aj.x * aj.x + aj.y * aj.y;
      double be = ak.x * ak.x + ak.y * ak.y;
      double gr = aj.x * ak.x + aj.y * ak.y;
      double gi = aj.x * ak.y - aj.y * ak.x;
#pragma unroll
      for (int o = 4; o <= 8; o <<= 1) {
        al += __shfl_xor_sync(FULL, al, o);
        be += __shfl_xor_sync(FULL, be, o);
        gr += __shfl_xor_sync(FULL, gr, o);
        gi += __shfl_xor_sync(FULL, gi, o);
      }
      const double ag2 = gr * gr + gi * gi;
      const double ab = al * be;
      big = big || ag2 > 1e-24 * ab;
      if (ag2 > 0.0 && ag2 > 1e-30 * ab) {
        // The same rotation as t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)), c = 1/sqrt(1 + t^2),
        // zeta = D/(2|gamma|), D = beta - alpha, rewritten with two rsqrt and no division:
        //   R = sqrt(D^2 + 4|gamma|^2), den = |D| + R, r = 1/sqrt(den^2 + 4|gamma|^2),
        //   c = den r, s e^{i phi} = 2 sgn(D) r gamma.
        const double D = be - al;
        const double q4 = 4.0 * ag2;
        const double w = fma(D, D, q4);
        const double R = w * rsqrt(w);
        const double den = fabs(D) + R;
        const double r = rsqrt(fma(den, den, q4));
        const double c = den * r;
        const double f2 = (D >= 0.0 ? 2.0 : -2.0) * r;
        const double spr = f2 * gr, spi = f2 * gi;  // s e^{i phi}
        if (lo) {  // a_j' = c a_j - conj(s e^{i phi}) a_k
          a = make_double2(c * aj.x - (spr * ak.x + spi * ak.y), c * aj.y - (spr * ak.y - spi * ak.x));
          v = make_double2(c * vj.x - (spr * vk.x + spi * vk.y), c * vj.y - (spr * vk.y - spi * vk.x));
        } else {   // a_k' = s e^{i phi} a_j + c a_k
          a = make_double2((spr * aj.x - spi * aj.y) + c * ak.x, (spr * aj.y + spi * aj.x) + c * ak.y);
          v = make_double2((spr * vj.x - spi * vj.y) + c * vk.x, (spr * vj.y + spi * vj.x) + c * vk.y);
        }
      }
    }
    if (!__any_sync(FULL, big)) break;
  }
  // sigma_j = ||a_j|| (reduce over rows), sigma_max over columns
  double nn = a.x * a.x + a.y * a.y;
  nn += __shfl_xor_sync(FULL, nn, 4);
  nn += __shfl_xor_sync(FULL, nn, 8);
  const double rs = nn > 0.0 ? rsqrt(nn) : 0.0;
  const double sig = nn * rs;
  double smax = sig;
  smax = fmax(smax, __shfl_xor_sync(FULL, smax, 1));
  smax = fmax(smax, __shfl_xor_sync(FULL, smax, 2));
  const bool nul = !(sig > 1e-14 * smax) || smax == 0.0;
  double2 xx = nul ? make_double2(0.0, 0.0) : make_double2(a.x * rs, a.y * rs);
  if (__any_sync(FULL, nul)) {  // rare: complete the null columns of X
    scratch[l] = xx;
    __syncwarp();
    const unsigned nm = __ballot_sync(FULL, nul && r == 0);  // bit (hb + j): column j null
    const unsigned cols = (nm >> hb) & 0xFu;
    if (l == 0 && cols) {
      for (int jj = 0; jj < 4; ++jj) {
        if (!((cols >> jj) & 1)) continue;
        for (int e0 = 0; e0 < 4; ++e0) {
          double2 u[4];
          for (int q = 0; q < 4; ++q) u[q] = make_double2(q == e0 ? 1.0 : 0.0, 0.0);
          for (int pass = 0; pass < 2; ++pass)
            for (int q = 0; q < 4; ++q) {
              if (q == jj || (((cols >> q) & 1) && q > jj)) continue;
              double2 d = make_double2(0.0, 0.0);
              for (int rr = 0; rr < 4; ++rr) cfma(d, cconj(scratch[4 * rr + q]), u[rr]);
              for (int rr = 0; rr < 4; ++rr) {
                const double2 tq = cmul(d, scratch[4 * rr + q]);
                u[rr].x -= tq.x;
                u[rr].y -= tq.y;
              }
            }
          double nv = 0.0;
          for (int rr = 0; rr < 4; ++rr) nv += u[rr].x * u[rr].x + u[rr].y * u[rr].y;
          nv = sqrt(nv);
          if (nv > 0.5) {
            for (int rr = 0; rr < 4; ++rr) scratch[4 * rr + jj] = make_double2(u[rr].x / nv, u[rr].y / nv);
            break;
          }
        }
      }
    }
    __syncwarp();
    xx = scratch[l];
    __syncwarp();
  }
  // G[r][j] = sum_q V[r][q] conj(X[j][q])
  double2 g = make_double2(0.0, 0.0);
#pragma unroll
  for (int q = 0; q < 4; ++q) cfma(g, shfl_c(v, hb | (4 * r + q)), cconj(shfl_c(xx, hb | (4 * j + q))));
  double ss = sig;                       // each column's lanes hold sigma_j
  ss += __shfl_xor_sync(FULL, ss, 1);
  ss += __shfl_xor_sync(FULL, ss, 2);
  g_out = g;
  v_out = v;
  sig_sum = scalbn(ss, ex);
#ifdef QFS_DIAG_POLAR  // diagnostic build: report sweeps * 1e7 + cycles instead of sum sigma
  sig_sum = (double)n_sweeps * 1e7 + (double)(clock64() - t_start);
#endif
  return true;
}

// Gate update by kind (readings R24-R25; the oracle's gate_update):
//   kind 0: two-qubit variable block, G = polar update of E' (hw_polar);
//   kind 1: fixed gate: G unchanged, ss = Re Tr(E G);
//   kind 2: one-qubit variable gate u on the pair's first qubit, stored as
//           u (x) I: E1[a][b] = E[a][b] + E[a+2][b+2] (partial trace over the
//           p1 bit), the polar update of E1 (x) I is exactly u_new (x) I (its
//           two diagonal copies are averaged so the zeros stay exact), ss = sum
//           of the singular values of E1.
// Half warp, lane l = 4r + c holds e = E[r][c] (before the beta term); gold is
// the old gate (row-major, read-only); both halves may hold different matrices
// but the kind must be warp-uniform.
__device__ bool gate_update(int kind, double2 e, const double2 *gold, double beta, const double2 *v0p, double2 &g,
                            double2 &v, double &ss, double2 *scratch, bool need_ss = true) {
  const int lane = threadIdx.x & 31, hb = lane & 16, l = lane & 15, r = l >> 2, c = l & 3;
  if (kind == 1) {
    g = gold[l];
    const double2 gt = gold[4 * c + r];  // G[c][r]
    ss = need_ss ? half_sum(e.x * gt.x - e.y * gt.y) : 0.0;
    return false;
  }
  const bool blk = (r >> 1) == (c >> 1);
  if (kind == 2) {
    const double2 ea = shfl_c(e, hb | (4 * (r & 1) + (c & 1)));
    const double2 eb = shfl_c(e, hb | (4 * ((r & 1) + 2) + (c & 1) + 2));
    e = blk ? make_double2(ea.x + eb.x, ea.y + eb.y) : make_double2(0.0, 0.0);
    if (beta != 0.0 && blk) {  // (1 - beta) E1 + beta u_old^dag, u_old^dag[a][b] = conj(u_old[b][a])
      const double2 go = gold[4 * (c & 1) + (r & 1)];
      e = make_double2((1.0 - beta) * e.x + beta * go.x, (1.0 - beta) * e.y - beta * go.y);
    }
  } else if (beta != 0.0) {  // E' = (1 - beta) E + beta G_old^dag
    const double2 go = gold[4 * c + r];  // (G^dag)[r][c] = conj(G[c][r])
    e = make_double2((1.0 - beta) * e.x + beta * go.x, (1.0 - beta) * e.y - beta * go.y);
  }
  const bool vnew = hw_polar(e, v0p, g, v, ss, scratch, need_ss);
  if (kind == 2) {
    const double2 ga = shfl_c(g, hb | (4 * (r & 1) + (c & 1)));
    const double2 gb = shfl_c(g, hb | (4 * ((r & 1) + 2) + (c & 1) + 2));
    g = blk ? make_double2(0.5 * (ga.x + gb.x), 0.5 * (ga.y + gb.y)) : make_double2(0.0, 0.0);
    ss *= 0.5;
  }
  return vnew;
}

}  // namespace
}  // namespace qfs
