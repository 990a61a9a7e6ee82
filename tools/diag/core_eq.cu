// roll2_core<1, float> against roll2_core<1, float2> on 2.1e6 random pairs of annulus points:
// bit-identical (0 mismatches) once no add takes a bare product (see walk_f32_dev.cuh).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a --extended-lambda -std=c++17 \
//     -I paper_2409_03686_b200/csrc -I include -fmad=true -prec-sqrt=false -prec-div=false \
//     -DEM_TANG_K=4 -DEM_ROLL2_ONE=1 -DEM_ROLL2_DYN=0 -o variants/core_eq tools/diag/core_eq.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "walk_f32_dev.cuh"
using namespace em;
using namespace em::f32;
__global__ void k(const F32Params P, const float* xs, const unsigned* ws, int n, unsigned long long* bad, float* ex) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  float ax = xs[4*i], ay = xs[4*i+1], bx = xs[4*i+2], by = xs[4*i+3];
  unsigned wa = ws[2*i], wb = ws[2*i+1];
  float s2a, s2b, na0, na1, nb0, nb1;
  roll2_core<1, float, unsigned>(P, ax, ay, wa, P.one_bits, s2a, na0, na1);
  roll2_core<1, float, unsigned>(P, bx, by, wb, P.one_bits, s2b, nb0, nb1);
  float2 s2, n0, n1;
  roll2_core<1, float2, uint2>(P, make_float2(ax, bx), make_float2(ay, by), make_uint2(wa, wb), P.one_bits, s2, n0, n1);
  auto ne = [](float u, float v) { return __float_as_uint(u) != __float_as_uint(v) && !(u != u && v != v); };
  if (ne(s2.x, s2a) || ne(s2.y, s2b) || ne(n0.x, na0) || ne(n0.y, nb0) || ne(n1.x, na1) || ne(n1.y, nb1)) {
    if (atomicAdd(bad, 1ULL) == 0) { ex[0]=ax; ex[1]=ay; ex[2]=na0; ex[3]=na1; ex[4]=n0.x; ex[5]=n1.x; ex[6]=bx; ex[7]=by; ex[8]=nb0; ex[9]=nb1; ex[10]=n0.y; ex[11]=n1.y; }
  }
}
int main() {
  F32Params P{};
  // an annulus R = 1, rho = 0.3, A = diag(1.3, 0.8)
  double a0 = 1.3, a1 = 0.8, R = 1.0, rho = 0.3, eps = 1e-5;
  P.Ad[0] = a0; P.Ad[1] = a1; P.Kd[0] = a0*a0; P.Kd[1] = a1*a1; P.ia[0] = 1/a0; P.ia[1] = 1/a1;
  P.oR = R; P.oR2 = R*R; P.hr[0] = rho; P.hr2[0] = rho*rho; P.m2 = a1*a1;
  P.keep = 1 - 4e-6; P.shrink_abs = 1.2e-7;
  double lim = (R - rho) / (2 * a0), rb = std::min(R * a1 / (a0*a0), lim);
  P.rho_h = lim * (1 - 1e-6); P.rho_h2 = P.rho_h * P.rho_h; P.rho_b = rb * (1 - 1e-6); P.rho_b2 = P.rho_b * P.rho_b;
  P.mid2 = 0.65 * 0.65; P.one_bits = 0x3f800000u;
  int n = 1 << 22;
  float* hx = (float*)malloc(2 * n * 4); unsigned* hw = (unsigned*)malloc(n * 4);
  srand(7);
  for (int i = 0; i < n; ++i) {
    double r = rho + (R - rho) * (i % 3 == 0 ? pow(rand() / (double)RAND_MAX, 4.0) : (i % 3 == 1 ? 1 - pow(rand() / (double)RAND_MAX, 4.0) : rand() / (double)RAND_MAX));
    double t = 6.283185307 * rand() / (double)RAND_MAX;
    hx[2*i] = r * cos(t); hx[2*i+1] = r * sin(t);
    hw[i] = ((unsigned)rand() << 16) ^ (unsigned)rand();
  }
  float* dx; unsigned* dw; cudaMalloc(&dx, 2*n*4); cudaMalloc(&dw, n*4);
  cudaMemcpy(dx, hx, 2*n*4, cudaMemcpyHostToDevice); cudaMemcpy(dw, hw, n*4, cudaMemcpyHostToDevice);
  unsigned long long* bad; cudaMalloc(&bad, 8); cudaMemset(bad, 0, 8);
  float* ex; cudaMalloc(&ex, 48);
  k<<<(n/2 + 255)/256, 256>>>(P, dx, dw, n, bad, ex);
  unsigned long long hb; cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
  float he[12]; cudaMemcpy(he, ex, 48, cudaMemcpyDeviceToHost);
  printf("%s mismatching pairs %llu of %d\n", cudaGetErrorString(cudaGetLastError()), hb, n/2);
  if (hb) printf("a: (%a,%a) -> scalar (%a,%a) packed (%a,%a)\nb: (%a,%a) -> scalar (%a,%a) packed (%a,%a)\n", he[0],he[1],he[2],he[3],he[4],he[5],he[6],he[7],he[8],he[9],he[10],he[11]);
  return 0;
}
