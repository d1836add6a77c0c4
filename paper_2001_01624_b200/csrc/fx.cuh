// Exact 128-bit fixed-point accumulation (two 64-bit integer atomics with a carry per
// term; one rounding to fp64 at the end): sums that do not depend on the order in which
// the atomics land.  Used by the Galerkin assemblies (coarse.cu, cpr.cu).
#pragma once

namespace msb {

// v 2^F as a 128-bit two's-complement integer (lo, hi), truncated toward zero
__device__ __forceinline__ void fx_of(double v, int F, unsigned long long& lo, unsigned long long& hi) {
  const bool neg = v < 0.0;
  const double t = ldexp(fabs(v), F);  // < 2^92, exact power-of-two scaling
  hi = (unsigned long long)floor(ldexp(t, -64));
  lo = (unsigned long long)(t - ldexp((double)hi, 64));
  if (neg) {  // two's complement of (hi, lo)
    lo = ~lo + 1ull;
    hi = ~hi + (lo == 0ull ? 1ull : 0ull);
  }
}

__device__ __forceinline__ void fx_add_raw(unsigned long long* e, unsigned long long lo,
                                           unsigned long long hi) {
  const unsigned long long old = atomicAdd(e, lo);
  atomicAdd(e + 1, hi + (old + lo < old ? 1ull : 0ull));
}

__device__ __forceinline__ void fx_add(unsigned long long* e, double v, int F) {
  unsigned long long lo, hi;
  fx_of(v, F, lo, hi);
  fx_add_raw(e, lo, hi);
}

// Unsigned 128-bit fixed point (lo, hi) of t = v 2^F for v >= 0 (fx_add's conversion).
__device__ __forceinline__ void fx_split(double v, int F, unsigned long long& lo,
                                         unsigned long long& hi) {
  const double t = ldexp(v, F);
  hi = (unsigned long long)floor(ldexp(t, -64));
  lo = (unsigned long long)(t - ldexp((double)hi, 64));
}

__device__ __forceinline__ void add128(unsigned long long& lo, unsigned long long& hi,
                                       unsigned long long ylo, unsigned long long yhi) {
  const unsigned long long s = lo + ylo;
  hi += yhi + (s < lo ? 1ull : 0ull);
  lo = s;
}

__device__ __forceinline__ double fx_value(unsigned long long lo, unsigned long long hi, int F) {
  return ldexp(ldexp((double)(long long)hi, 64) + (double)lo, -F);
}

}  // namespace msb
