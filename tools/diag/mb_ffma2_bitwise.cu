// __ffma2_rn / __fmul2_rn / __fadd2_rn against the scalar _rn operations on 8.4e6 random
// pairs (any bit pattern, denormals, values near 1): 0 mismatches on the B200.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --extended-lambda -o variants/eq tools/diag/mb_ffma2_bitwise.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
__global__ void k(const float* a, const float* b, const float* c, int n, unsigned long long* bad, float* ex) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  float2 A = make_float2(a[2*i], a[2*i+1]), B = make_float2(b[2*i], b[2*i+1]), C = make_float2(c[2*i], c[2*i+1]);
  float2 f = __ffma2_rn(A, B, C), m = __fmul2_rn(A, B), s = __fadd2_rn(A, C);
  float f0 = __fmaf_rn(A.x, B.x, C.x), f1 = __fmaf_rn(A.y, B.y, C.y);
  float m0 = __fmul_rn(A.x, B.x), m1 = __fmul_rn(A.y, B.y);
  float s0 = __fadd_rn(A.x, C.x), s1 = __fadd_rn(A.y, C.y);
  auto ne = [](float u, float v) { return __float_as_uint(u) != __float_as_uint(v) && !(u != u && v != v); };
  if (ne(f.x, f0) || ne(f.y, f1)) { if (atomicAdd(&bad[0], 1ULL) == 0) { ex[0]=A.x; ex[1]=B.x; ex[2]=C.x; ex[3]=f.x; ex[4]=f0; ex[5]=A.y; ex[6]=B.y; ex[7]=C.y; ex[8]=f.y; ex[9]=f1; } }
  if (ne(m.x, m0) || ne(m.y, m1)) atomicAdd(&bad[1], 1ULL);
  if (ne(s.x, s0) || ne(s.y, s1)) atomicAdd(&bad[2], 1ULL);
}
int main() {
  int n = 1 << 24;
  float *h = (float*)malloc(3 * n * 4);
  srand(1);
  for (int i = 0; i < 3 * n; ++i) {
    unsigned r = ((unsigned)rand() << 16) ^ (unsigned)rand();
    int mode = i % 4;
    float v;
    if (mode == 0) { memcpy(&v, &r, 4); }                    // any bit pattern
    else if (mode == 1) v = (float)((double)r / 4294967296.0 * 2 - 1);
    else if (mode == 2) v = (float)((double)r / 4294967296.0) * 1e-20f * ((r & 1) ? 1e-19f : 1.0f);  // tiny/denormal
    else v = 1.0f + (float)(r & 0xff) * 1.1920929e-7f;
    h[i] = v;
  }
  float *d; cudaMalloc(&d, 3 * n * 4); cudaMemcpy(d, h, 3 * n * 4, cudaMemcpyHostToDevice);
  unsigned long long* bad; cudaMalloc(&bad, 24); cudaMemset(bad, 0, 24);
  float* ex; cudaMalloc(&ex, 40);
  k<<<(n / 2 + 255) / 256, 256>>>(d, d + n, d + 2 * n, n, bad, ex);
  unsigned long long hb[3]; cudaMemcpy(hb, bad, 24, cudaMemcpyDeviceToHost);
  float he[10]; cudaMemcpy(he, ex, 40, cudaMemcpyDeviceToHost);
  printf("mismatches fma %llu mul %llu add %llu of %d pairs\n", hb[0], hb[1], hb[2], n / 2);
  if (hb[0]) printf("example: %a*%a+%a = %a (x2) vs %a ; %a*%a+%a = %a vs %a\n", he[0], he[1], he[2], he[3], he[4], he[5], he[6], he[7], he[8], he[9]);
  return 0;
}
