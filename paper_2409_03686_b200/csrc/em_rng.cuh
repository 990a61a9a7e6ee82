// em_rng.cuh -- counter-based RNG for the exit-measure kernels.
//
// philox4x64_10: the reference's stream (S/_kernel.pyx:21-54, S/rng.py:19-62;
//   S/ = /root/reference/pkg/src/exitmeasure/), used by the bit-exact FP64
//   mirror.  mulhi is __umul64hi, the low word a plain 64-bit product.
// philox4x32_10: Salmon et al. (SC'11) Philox4x32 with 10 rounds -- the same
//   function as the CUDA toolkit's curand_Philox4x32_10 (checked against it by
//   a known-answer kernel in tests), used by the production FP32 kernel.  The
//   round keys depend only on the seed, so they are warp-uniform and live in
//   uniform registers.
#pragma once
#include <stdint.h>

namespace em {

struct u64x4 {
  unsigned long long w0, w1, w2, w3;
};

__device__ __forceinline__ u64x4 philox4x64_10(unsigned long long k0, unsigned long long k1,
                                               unsigned long long c0, unsigned long long c1,
                                               unsigned long long c2, unsigned long long c3) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    unsigned long long hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    unsigned long long hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += W0;
    k1 += W1;
  }
  return {c0, c1, c2, c3};
}

// Round keys of Philox4x32-10 for a fixed seed (warp-uniform).
struct PhiloxKey32 {
  unsigned k0[10], k1[10];
};

__host__ __device__ inline PhiloxKey32 philox32_schedule(unsigned key0, unsigned key1) {
  PhiloxKey32 s;
  for (int r = 0; r < 10; ++r) {
    s.k0[r] = key0 + (unsigned)r * 0x9E3779B9u;
    s.k1[r] = key1 + (unsigned)r * 0xBB67AE85u;
  }
  return s;
}

// One 32x32 -> 64 multiply (IMAD.WIDE.U32) yields both halves of a round's
// product; the round keys come from K (kernel params: constant-bank operands
// of the LOP3s), so a block costs 20 IMAD.WIDE + 20 LOP3.
__device__ __forceinline__ uint4 philox4x32_10(const PhiloxKey32& K, unsigned c0, unsigned c1,
                                               unsigned c2, unsigned c3) {
  const unsigned M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)M0 * c0;
    const unsigned long long p1 = (unsigned long long)M1 * c2;
    const unsigned hi0 = (unsigned)(p0 >> 32), lo0 = (unsigned)p0;
    const unsigned hi1 = (unsigned)(p1 >> 32), lo1 = (unsigned)p1;
    c0 = hi1 ^ c1 ^ K.k0[r];
    c1 = lo1;
    c2 = hi0 ^ c3 ^ K.k1[r];
    c3 = lo0;
  }
  return make_uint4(c0, c1, c2, c3);
}

// [0,1) with 23 random bits, built on the FMA/ALU pipes (no I2F): the word's
// top 23 bits become the mantissa of a float in [1,2).
__device__ __forceinline__ float u01_23(unsigned w) {
  return __uint_as_float(0x3f800000u | (w >> 9)) - 1.0f;
}

// (-1,1) symmetric, 23 bits, never exactly +-1: -1 + (2m + 1)/2^23 for the
// word's top 23 bits m; every step below is exact in FP32.
__device__ __forceinline__ float sym11_23(unsigned w) {
  float f = __uint_as_float(0x3f800000u | (w >> 9));  // 1 + m/2^23
  return fmaf(2.0f, f, -3.0f) + 1.1920928955078125e-07f;  // + 2^-23
}

}  // namespace em
