#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
template <int CH>
__global__ void thr(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[CH][2];
  for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) dmma(c[k][0], c[k][1], a, b, c[k][0], c[k][1]);
  double s = 0;
  for (int k = 0; k < CH; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_thr(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8];
  for (int k = 0; k < 8; ++k) c[k] = k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = fma(a, b, c[k]);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *o; cudaMalloc(&o, 148 * 32 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    thr<4><<<148, 32 * warps>>>(o, 10); cudaEventRecord(e0);
    thr<4><<<148, 32 * warps>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * warps * iters * 4 * 512;  // 8x8x4 FMA = 256 FMA = 512 flop per mma per warp
    printf("DMMA warps/SM %2d chains 4: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  thr<1><<<148, 32>>>(o, 10); cudaEventRecord(e0);
  thr<1><<<148, 32>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DMMA dependent-chain latency: %.1f ns per mma (%.1f cycles at 1.965 GHz)\n", ms * 1e6 / iters, ms * 1e6 / iters * 1.965);
  for (int warps : {8, 16, 32}) {
    dfma_thr<<<148, 32 * warps>>>(o, 10); cudaEventRecord(e0);
    dfma_thr<<<148, 32 * warps>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 148.0 * warps * 32 * iters * 8 * 2;
    printf("DFMA warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
