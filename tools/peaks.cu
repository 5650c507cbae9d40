// Microbenchmarks for the roofline denominators MEASURED_PEAKS.json lacks:
//   - FP64 DFMA peak (8 independent FMA chains per thread, all SMs)
//   - L2-resident read+write bandwidth (working set well inside the 126 MB L2)
//   - HBM read+write bandwidth (working set >> L2), same access kernel
//   - back-to-back launch latency of an empty kernel (stream and CUDA graph)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 123.456) out[0] = s;
}

// read a, write b (same as a copy): 32 B per element pair (double2 in, double2 out)
__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) { double2 v = a[i]; v.x += 1.0; b[i] = v; }
}
// read-modify-write in place (like the chi update): 32 B per element
__global__ void rmw_kernel(double2 *__restrict__ a, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) { double2 v = a[i]; v.x += 1.0; a[i] = v; }
}
// read only: 16 B per element
__global__ void read_kernel(const double2 *__restrict__ a, size_t n, double *out) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  double s = 0;
  for (; i < n; i += st) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 123.456) out[0] = s;
}
__global__ void empty_kernel() {}
// write only: 16 B per element
__global__ void write_kernel(double2 *__restrict__ a, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) a[i] = make_double2((double)i, 1.0);
}
// `passes` read-modify-write passes over an L2-resident buffer inside one launch
__global__ void rmw_loop_kernel(double2 *__restrict__ a, size_t n, int passes) {
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (int p = 0; p < passes; ++p)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += st) {
      double2 v = a[i]; v.x += 1.0; a[i] = v;
    }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  int clk = 0; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d",
         p.name, p.multiProcessorCount, l2, p.sharedMemPerBlockOptin, clk);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  double *dout; CK(cudaMalloc(&dout, 8));
  // FP64
  {
    int blocks = p.multiProcessorCount * 4, threads = 512, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(dout, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0)); dfma_kernel<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
    }
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf(", \"fp64_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  }
  // bandwidths
  auto bw = [&](size_t bytes_per_array, const char *tag) {
    size_t n = bytes_per_array / 16;
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16)); CK(cudaMemset(b, 0, n * 16));
    int blocks = p.multiProcessorCount * 8, threads = 256;
    float best_c = 1e30f, best_r = 1e30f, best_rd = 1e30f;
    for (int r = 0; r < 8; ++r) {
      CK(cudaEventRecord(e0)); copy_kernel<<<blocks, threads>>>(a, b, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (r) best_c = std::min(best_c, ms);
      CK(cudaEventRecord(e0)); rmw_kernel<<<blocks, threads>>>(a, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); if (r) best_r = std::min(best_r, ms);
      CK(cudaEventRecord(e0)); read_kernel<<<blocks, threads>>>(a, n, dout);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); if (r) best_rd = std::min(best_rd, ms);
    }
    printf(", \"%s_copy_gbs\": %.1f, \"%s_rmw_gbs\": %.1f, \"%s_read_gbs\": %.1f", tag,
           32.0 * n / (best_c * 1e-3) / 1e9, tag, 32.0 * n / (best_r * 1e-3) / 1e9, tag,
           16.0 * n / (best_rd * 1e-3) / 1e9);
    CK(cudaFree(a)); CK(cudaFree(b));
  };
  // L2: 20 passes of read+write over 16 / 32 / 64 MiB inside one launch
  for (size_t mib : {16, 32, 64}) {
    size_t n = (mib << 20) / 16;
    double2 *a; CK(cudaMalloc(&a, n * 16)); CK(cudaMemset(a, 0, n * 16));
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      CK(cudaEventRecord(e0)); rmw_loop_kernel<<<p.multiProcessorCount * 8, 256>>>(a, n, 20);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (r) best = std::min(best, ms);
    }
    printf(", \"l2loop_%zuMiB_rmw_gbs\": %.1f", mib, 20 * 32.0 * n / (best * 1e-3) / 1e9);
    CK(cudaFree(a));
  }
  {  // HBM write-only
    size_t n = (4ull << 30) / 16;
    double2 *a; CK(cudaMalloc(&a, n * 16));
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      CK(cudaEventRecord(e0)); write_kernel<<<p.multiProcessorCount * 8, 256>>>(a, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (r) best = std::min(best, ms);
    }
    printf(", \"hbm_4GiB_write_gbs\": %.1f", 16.0 * n / (best * 1e-3) / 1e9);
    CK(cudaFree(a));
  }
  bw(16ull << 20, "l2_16MiB");
  bw(32ull << 20, "l2_32MiB");
  bw(4ull << 30, "hbm_4GiB");
  // launch latency
  {
    cudaStream_t s; CK(cudaStreamCreate(&s));
    const int L = 2000;
    for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32, 0, s>>>();
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < L; ++i) empty_kernel<<<148, 128, 0, s>>>();
    CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf(", \"launch_stream_us\": %.3f", ms * 1e3 / L);
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < L; ++i) empty_kernel<<<148, 128, 0, s>>>();
    CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(e0, s)); CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf(", \"launch_graph_us\": %.3f", ms * 1e3 / L);
  }
  printf("}\n");
  return 0;
}
