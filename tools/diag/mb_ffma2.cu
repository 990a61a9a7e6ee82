// FFMA2 vs FFMA throughput, alone and with ALU-pipe work (B200):
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o variants/mb tools/diag/mb_ffma2.cu && gpurun -- ./variants/mb
#include <cstdio>
#include <cuda_runtime.h>
// issue-rate microbenchmarks: FFMA vs FFMA2, alone and mixed with ALU-pipe work
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float a, float b, unsigned m) {
  float2 v[8];
  unsigned u[8];
  for (int i = 0; i < 8; ++i) { v[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f - i); u[i] = threadIdx.x + i; }
  float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0 || MODE == 2) { v[i].x = fmaf(v[i].x, a, b); v[i].y = fmaf(v[i].y, a, b); }
        if (MODE == 1 || MODE == 3) v[i] = __ffma2_rn(v[i], A, B);
        if (MODE == 2 || MODE == 3) { u[i] = (u[i] & m) ^ (u[i] >> 3); u[i] = (u[i] | m) ^ (u[i] << 5);}  // 2+2 ALU ops? 
      }
    }
  }
  float s = 0; unsigned t = 0;
  for (int i = 0; i < 8; ++i) { s += v[i].x + v[i].y; t ^= u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + __uint_as_float(t);
}
template <int MODE>
void run(const char* name, float* d, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 4;
  k<MODE><<<blocks, 256>>>(d, 10, 1.0001f, 0.5f, 0x55555555u);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(d, iters, 1.0001f, 0.5f, 0x55555555u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = (double)blocks * 256 * iters * 4 * 8 * 2;
  printf("%s: %.3f ms, %.2f T lane-FMA/s (%.1f lane-FMA/clk/SM at 1.965GHz)\n", name, ms, fma / ms / 1e9, fma / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 4 * 256 * 4);
  int iters = 20000;
  run<0>("FFMA only ", d, iters);
  run<1>("FFMA2 only", d, iters);
  run<2>("FFMA + ALU ", d, iters);
  run<3>("FFMA2 + ALU", d, iters);
  return 0;
}
