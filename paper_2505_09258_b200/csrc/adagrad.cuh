// adagrad.cuh -- the reference's FP64 Adagrad element update (train.cpp:342-354)
//
//   a = double(S) + g * g;   S' = float(a);
//   theta' = float(double(theta) - lr * g / (sqrt(a) + eps))
//
// bit-identical, with a fast path.  The exact form needs IEEE double sqrt and
// division (~50 instructions per element with CUDA's inline sequences and
// their slow-path branches).  The fast path computes q = lr g / (sqrt(a) +
// eps) to ~2^-50 relative from FP64 MUFU seeds and two Newton steps each,
// then t = theta - q.  float(t_exact) is known when t minus and plus the error
// bound round to the same float; otherwise (and for non-normal operands) the
// caller redoes the element with the exact form.  Both forms take the products, sums and
// conversions in the reference's order, so the result is the reference's to
// the bit either way.
#pragma once

#include <cstdint>

namespace lgd {

// FP64 MUFU seeds (~2^-22 relative): no f32 <-> f64 conversions, which share
// the MIO path with shared-memory traffic
__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// The exact reference update (CUDA's correctly rounded sqrt and division).
__device__ __forceinline__ void adagrad_exact(double g, float& th, float& st, double lr,
                                              double eps) {
  const double a2 = (double)st + g * g;
  st = (float)a2;
  th = (float)((double)th - lr * g / (sqrt(a2) + eps));
}

// Fast path: returns false when the element must be redone exactly (th and st
// are left untouched then).
__device__ __forceinline__ bool adagrad_try_fast(double g, float& th, float& st, double lr,
                                                 double eps) {
  const double a2 = (double)st + g * g;
  const float af = (float)a2;
  const double num = lr * g;
  const double t0 = (double)th;
  // (g = 0 needs no special case: with S > 0, q = 0 and the bound certifies
  // t0; with S = 0 the seed is inf, t is NaN and the exact form runs.  The
  // branch it used to take cost K4 4.5%.)
  // sqrt(a2): s = a2 * rsqrt(a2) from a ~2^-20 seed, two Newton (Heron)
  // steps: the error squares each time, so only the roundings of the last
  // steps remain (< 2^-50 relative)
  const double y = rsqrt_approx(a2);
  const double h = 0.5 * y;
  const double s = a2 * y;
  const double s1 = __fma_rn(h, __fma_rn(-s, s, a2), s);
  const double s2 = __fma_rn(h, __fma_rn(-s1, s1, a2), s1);
  const double den = s2 + eps;
  // 1 / den: ~2^-20 seed, two Newton steps (< 2^-50 relative)
  const double r = rcp_approx(den);
  const double r1 = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
  const double r2 = __fma_rn(r1, __fma_rn(-den, r1, 1.0), r1);
  const double q = num * r2;
  const double t = t0 - q;
  // |t_ref - t| <= B = 2^-46 |q| + 2^-51 |t| (the Newton results are within a
  // few roundings, ~2^-50 |q|, of the exact quotient; t and t_ref each carry
  // one more rounding of 2^-53 |t|).  Rounding to float is monotonic, so when
  // t - B and t + B round to the same float, so does t_ref.  NaN from
  // non-normal operands (the MUFU seeds flush denormals) fails the compare.
  const double bound = __fma_rn(0x1p-46, fabs(q), 0x1p-51 * fabs(t));
  const float lo = (float)(t - bound), hi = (float)(t + bound);
  const bool ok = lo == hi;
  if (ok) {
    st = af;
    th = hi;
  }
  return ok;
}

// One Newton step per seed (~2^-39 relative for q from ~2^-20 seeds): four
// fewer DFMA per element; the certificate widens to B = 2^-36 |q| + 2^-51 |t|,
// so ~5 elements in 10^4 fall back to the exact form.  The K4 default (K4
// +1.5%); profiles/micro/adagrad_probe.cu mode 1 checks it against the exact
// form: 0 mismatches in 4.3e9 random operand triples (fast path 99.953%).
__device__ __forceinline__ bool adagrad_try_fast1(double g, float& th, float& st, double lr,
                                                  double eps) {
  const double a2 = (double)st + g * g;
  const float af = (float)a2;
  const double num = lr * g;
  const double t0 = (double)th;
  const double y = rsqrt_approx(a2);
  const double s = a2 * y;
  const double s1 = __fma_rn(0.5 * y, __fma_rn(-s, s, a2), s);
  const double den = s1 + eps;
  const double r = rcp_approx(den);
  const double r1 = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
  const double q = num * r1;
  const double t = t0 - q;
  const double bound = __fma_rn(0x1p-36, fabs(q), 0x1p-51 * fabs(t));
  const float lo = (float)(t - bound), hi = (float)(t + bound);
  const bool ok = lo == hi;
  if (ok) {
    st = af;
    th = hi;
  }
  return ok;
}

}  // namespace lgd
