// detmath.cuh -- deterministic log / exp / pow for the synthetic graph
// generator.
//
// CUDA's pow() and glibc's pow() may differ in the last ulp, and the
// generator truncates pow() results to integer ranks, so a host restatement
// built on glibc could not reproduce the device graph edge for edge.  These
// versions use only IEEE-exact operations (+, -, *, /, floor, bit
// manipulation) in a fixed order -- compiled with -fmad=false on the device
// and without FMA contraction on the host they round identically, so the
// CPU oracle (oracle/legend_oracle.c: lo_det_pow) regenerates any edge of a
// benchmark graph bit for bit.  Accuracy: ~1e-15 relative over the ranges
// used (x in [1, 2^40], |y| <= 64).
#pragma once

#include <cstdint>
#include <cstring>

namespace lgd {

__host__ __device__ __forceinline__ uint64_t det_bits(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
#endif
}
__host__ __device__ __forceinline__ double det_from_bits(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double x;
  std::memcpy(&x, &b, 8);
  return x;
#endif
}

// natural log of a positive normal double: x = m 2^e, m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(s), s = (m - 1) / (m + 1), |s| <= 0.1716, odd series to s^25
__host__ __device__ inline double det_log(double x) {
  const uint64_t b = det_bits(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = det_from_bits((b & 0xfffffffffffffull) | (1023ull << 52));
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    e += 1;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double q = 0x1.47ae147ae147bp-4;  // 2/25
  q = q * s2 + 0x1.642c8590b2164p-4;  // 2/23
  q = q * s2 + 0x1.8618618618618p-4;  // 2/21
  q = q * s2 + 0x1.af286bca1af28p-4;  // 2/19
  q = q * s2 + 0x1.e1e1e1e1e1e1ep-4;  // 2/17
  q = q * s2 + 0x1.1111111111111p-3;  // 2/15
  q = q * s2 + 0x1.3b13b13b13b14p-3;  // 2/13
  q = q * s2 + 0x1.745d1745d1746p-3;  // 2/11
  q = q * s2 + 0x1.c71c71c71c71cp-3;  // 2/9
  q = q * s2 + 0x1.2492492492492p-2;  // 2/7
  q = q * s2 + 0x1.999999999999ap-2;  // 2/5
  q = q * s2 + 0x1.5555555555555p-1;  // 2/3
  const double r = s * 2.0 + s * (s2 * q);
  const double de = (double)e;
  return de * 0x1.62e42fee00000p-1 + (r + de * 0x1.a39ef35793c76p-33);
}

// e^y for |y| < 700: y = k ln2 + r, |r| <= ln2 / 2, Taylor to r^17, times 2^k
__host__ __device__ inline double det_exp(double y) {
  const double k = floor(y * 0x1.71547652b82fep+0 + 0.5);
  const double r = (y - k * 0x1.62e42fee00000p-1) - k * 0x1.a39ef35793c76p-33;
  double p = 0x1.952c77030ad4ap-49;  // 1/17!
  p = p * r + 0x1.ae7f3e733b81fp-45;  // 1/16!
  p = p * r + 0x1.ae7f3e733b81fp-41;  // 1/15!
  p = p * r + 0x1.93974a8c07c9dp-37;  // 1/14!
  p = p * r + 0x1.6124613a86d09p-33;  // 1/13!
  p = p * r + 0x1.1eed8eff8d898p-29;  // 1/12!
  p = p * r + 0x1.ae64567f544e4p-26;  // 1/11!
  p = p * r + 0x1.27e4fb7789f5cp-22;  // 1/10!
  p = p * r + 0x1.71de3a556c734p-19;  // 1/9!
  p = p * r + 0x1.a01a01a01a01ap-16;  // 1/8!
  p = p * r + 0x1.a01a01a01a01ap-13;  // 1/7!
  p = p * r + 0x1.6c16c16c16c17p-10;  // 1/6!
  p = p * r + 0x1.1111111111111p-7;   // 1/5!
  p = p * r + 0x1.5555555555555p-5;   // 1/4!
  p = p * r + 0x1.5555555555555p-3;   // 1/3!
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  const int ki = (int)k;
  return p * det_from_bits((uint64_t)(ki + 1023) << 52);
}

// x^y for x >= 1 (the generator's inverse-CDF arguments)
__host__ __device__ inline double det_pow(double x, double y) { return det_exp(y * det_log(x)); }

}  // namespace lgd
