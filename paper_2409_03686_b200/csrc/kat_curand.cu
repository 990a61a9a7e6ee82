// kat_curand.cu -- known-answer cross-check of the production RNG against the
// CUDA toolkit's own Philox4x32-10 (curand_Philox4x32_10 from
// curand_philox4x32_x.h, called, not copied).  Test hook only: the walk
// kernels use em::philox4x32_10 (em_rng.cuh), and tests assert both agree.
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>
#include <stdint.h>

namespace em {

__global__ void curand_philox_kernel(const unsigned* in, unsigned* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned* c = in + 6 * i;
  uint4 r = curand_Philox4x32_10(make_uint4(c[0], c[1], c[2], c[3]), make_uint2(c[4], c[5]));
  out[4 * i] = r.x;
  out[4 * i + 1] = r.y;
  out[4 * i + 2] = r.z;
  out[4 * i + 3] = r.w;
}

}  // namespace em

extern "C" int em_curand_philox4x32_blocks(const uint32_t* in6, uint32_t* out4, int n,
                                           int device) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  unsigned *din = nullptr, *dout = nullptr;
  int rc = 0;
  if (cudaMalloc(&din, (size_t)n * 24) != cudaSuccess || cudaMalloc(&dout, (size_t)n * 16) != cudaSuccess)
    rc = -2;
  if (!rc && cudaMemcpy(din, in6, (size_t)n * 24, cudaMemcpyHostToDevice) != cudaSuccess) rc = -2;
  if (!rc) {
    em::curand_philox_kernel<<<(n + 127) / 128, 128>>>(din, dout, n);
    if (cudaGetLastError() != cudaSuccess) rc = -2;
  }
  if (!rc && cudaMemcpy(out4, dout, (size_t)n * 16, cudaMemcpyDeviceToHost) != cudaSuccess) rc = -2;
  cudaFree(din);
  cudaFree(dout);
  cudaSetDevice(prev);
  return rc;
}
