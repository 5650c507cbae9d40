// Cycle counts of the resident kernel's shared-memory passes in isolation
// (one 256-thread CTA per SM, the C3 / C5c per-CTA shapes), to separate the
// FP64 / shared-memory work of a pass from its fixed costs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_12866_b200/csrc \
//        -I include -I <nccl>/include tools/res_pass_bench.cu -o /tmp/res_pass_bench && /tmp/res_pass_bench
// Passes (cycles per pass, thread 0 of each CTA, averaged over CTAs):
//   0 env (res_env: item loop + warp reduce-scatter), 1 env loop with a plain
//   per-thread sum instead of the reduce-scatter, 2 reduce-scatter alone,
//   3 gate application (res_apply, G^dag), 4 two-gate pass (res_apply_pair),
//   5 __syncthreads alone.  Ideal FP64 time of a pass = items x 64 DFMA / (64 per clock).
#include "qfs_resident.cu"

namespace qfs {
bool pdl_enabled() { return false; }  // (defined in qfs_runtime.cu; unused here)
}

#include <cstdio>
#include <vector>

namespace qfs {
namespace {
__global__ void __launch_bounds__(RES_THREADS, 1)
    pass_bench(int n, int cnt, int ld, int which, int reps, unsigned long long *out, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  double2 *phi = (double2 *)sm;
  double2 *chi = phi + (2 * ((size_t)ld << n) * 16 <= 200 * 1024 ? ((size_t)ld << n) : 0);  // (large shapes: one buffer)
  double2 *G = phi + (chi == phi ? 1 : 2) * ((size_t)ld << n);
  double *red = (double *)(G + 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (unsigned q = tid; q < ((unsigned)ld << n); q += RES_THREADS) {
    phi[q] = make_double2(1e-3 * (q % 97), -1e-3 * (q % 89));
    chi[q] = make_double2(1e-3 * (q % 83), 1e-3 * (q % 79));
  }
  if (tid < 32) {  // two copies of (H (x) H) / 2: unitary, entries +-1/2
    const int e = tid & 15, r = e >> 2, c = e & 3;
    G[tid] = make_double2((__popc(r & c) & 1) ? -0.5 : 0.5, 0.0);
  }
  __syncthreads();
  const FastDiv fd((unsigned)cnt);
  const int2 prs[6] = {{0, 1}, {2, 3}, {4, 5}, {1, 2}, {3, 4}, {n - 2, n - 1}};
  double keep = 0.0;
  const unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const int2 pq = prs[r % 6], pq2 = prs[(r + 1) % 6];
    if (which == 0) {
      res_env(phi, chi, pq, cnt, fd, ld, n, red);
    } else if (which == 1) {
      double acc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) acc[e] = 0.0;
      const int lo = min(pq.x, pq.y), hi = max(pq.x, pq.y);
      const unsigned o1 = (1u << pq.x) * ld, o2 = (1u << pq.y) * ld;
      const unsigned items = (1u << (n - 2)) * (unsigned)cnt;
#pragma unroll RES_ENV_UNROLL
      for (unsigned q = tid; q < items; q += RES_THREADS) {
        const unsigned rr = fd.div(q);
        const unsigned b = insert_zero32(insert_zero32(rr, lo), hi) * ld + (q - rr * (unsigned)cnt);
        const double2 f[4] = {phi[b], phi[b + o1], phi[b + o2], phi[b + o1 + o2]};
        const double2 c[4] = {chi[b], chi[b + o1], chi[b + o2], chi[b + o1 + o2]};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            double &re = acc[2 * (4 * a + k)], &im = acc[2 * (4 * a + k) + 1];
            re = fma(f[a].x, c[k].x, re);
            re = fma(f[a].y, c[k].y, re);
            im = fma(f[a].y, c[k].x, im);
            im = fma(-f[a].x, c[k].y, im);
          }
      }
      double s = 0.0;
#pragma unroll
      for (int e = 0; e < 32; ++e) s += acc[e];
      red[warp * 32 + lane] = s;
    } else if (which == 2) {
      double acc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) acc[e] = phi[(e * 37 + tid + r) & 1023].x;
      red[warp * 32 + lane] = warp_reduce_scatter32(acc, lane);
    } else if (which == 3) {
      res_apply(phi, G, pq, true, cnt, fd, ld, n, tid, RES_THREADS);
    } else if (which == 4) {
      res_apply_pair(phi, G, pq, G + 16, pq2, cnt, fd, ld, n, tid, RES_THREADS);
    }
    __syncthreads();
  }
  const unsigned long long t1 = clock64();
  keep += red[lane] + phi[tid].x;
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / (unsigned long long)reps;
  sink[blockIdx.x * RES_THREADS + tid] = keep;
}
}  // namespace
}  // namespace qfs

int main() {
  using namespace qfs;
  const int shapes[4][2] = {{9, 8}, {10, 4}, {9, 4}, {12, 2}};  // (n, rows per CTA): C3, C5c, C3 at C = 4, C4 validation
  const char *nm[6] = {"env", "env-loop-only", "reduce-scatter", "apply", "apply-pair", "syncthreads"};
  unsigned long long *d_out;
  double *d_sink;
  cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
  cudaMalloc(&d_sink, 148 * RES_THREADS * sizeof(double));
  cudaFuncSetAttribute(pass_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (auto &sh : shapes) {
    const int n = sh[0], cnt = sh[1], ld = cnt;
    const bool one = ((size_t)ld << n) * 2 * 16 > 200 * 1024;  // C4 validation shape: one state buffer (env rows skipped)
    const size_t smem = (one ? 1 : 2) * ((size_t)ld << n) * 16 + 32 * 16 + RES_THREADS * 8;
    const double items = (double)(1 << (n - 2)) * cnt;
    printf("n=%d rows=%d: %.0f items per pass, %.1f per thread; ideal FP64 %.0f cycles (64 DFMA/item)\n", n, cnt, items,
           items / RES_THREADS, items * 64 / 64.0);
    for (int w = 0; w < 6; ++w) {
      if (one && w < 3) continue;
      pass_bench<<<148, RES_THREADS, smem>>>(n, cnt, ld, w == 5 ? 99 : w, 600, d_out, d_sink);
      if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
        return 1;
      }
      std::vector<unsigned long long> h(148);
      cudaMemcpy(h.data(), d_out, 148 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double s = 0;
      for (auto v : h) s += (double)v;
      printf("  %-15s %7.0f cycles per pass (%.2f us at 1.965 GHz)\n", nm[w], s / 148, s / 148 / 1965.0);
    }
  }
  return 0;
}
