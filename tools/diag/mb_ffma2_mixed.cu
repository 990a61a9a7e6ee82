// Cycles per instruction group (FFMA2 / FFMA / LOP3 mixes), CUDA events at 1.965 GHz:
// FFMA2 2.03, FFMA+FFMA 2.05, LOP3 2.01, FFMA2+LOP3 2.35, FFMA+FFMA+LOP3 3.21, FFMA2+2 LOP3 4.19
// -> a packed op holds the FMA pipe two cycles but ONE issue slot; ALU ops are half rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o variants/mb2 tools/diag/mb_ffma2_mixed.cu
#include <cstdio>
#include <cuda_runtime.h>
// cycles per group for: MODE 0: FFMA2 + LOP3 ; 1: FFMA+FFMA+LOP3 ; 2: FFMA2 only ; 3: LOP3 only ; 4: FFMA2 + 2 LOP3; 5: FFMA only(2)
// 6: FFMA2 + MUFU(1/8) ...
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters, float a, float b, unsigned m, long long* cyc) {
  float2 v[8];
  unsigned u[8], w[8];
  for (int i = 0; i < 8; ++i) { v[i] = make_float2(threadIdx.x * 1e-3f + i, threadIdx.x * 2e-3f - i); u[i] = threadIdx.x + i; w[i] = threadIdx.x * 3 + i; }
  float2 A = make_float2(a, a), B = make_float2(b, b);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0 || MODE == 2 || MODE == 4) v[i] = __ffma2_rn(v[i], A, B);
        if (MODE == 1 || MODE == 5) { v[i].x = fmaf(v[i].x, a, b); v[i].y = fmaf(v[i].y, a, b); }
        if (MODE == 0 || MODE == 1 || MODE == 3 || MODE == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(m), "r"(it));
        if (MODE == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(w[i]) : "r"(m), "r"(it));
      }
    }
  }
  long long t1 = clock64();
  float s = 0; unsigned t = 0;
  for (int i = 0; i < 8; ++i) { s += v[i].x + v[i].y; t ^= u[i] ^ w[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + __uint_as_float(t);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE>
void run(const char* name, float* d, long long* dc, int iters) {
  int blocks = 148 * 4;   // 8 warps per SMSP
  k<MODE><<<blocks, 256>>>(d, 10, 1.0001f, 0.5f, 0x55555555u, dc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(d, iters, 1.0001f, 0.5f, 0x55555555u, dc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("%s: %.3f cycles per group per SMSP (events, 1.965 GHz), clock64 %.3f\n", name, ms * 1e-3 * 1.965e9 / (8.0 * iters * 32), (double)c / (8.0 * iters * 32));
}
int main() {
  float* d; cudaMalloc(&d, 148 * 4 * 256 * 4);
  long long* dc; cudaMalloc(&dc, 8);
  int iters = 50000;
  run<2>("FFMA2            ", d, dc, iters);
  run<5>("FFMA+FFMA        ", d, dc, iters);
  run<3>("LOP3             ", d, dc, iters);
  run<0>("FFMA2+LOP3       ", d, dc, iters);
  run<1>("FFMA+FFMA+LOP3   ", d, dc, iters);
  run<4>("FFMA2+LOP3+LOP3  ", d, dc, iters);
  return 0;
}
