// log1p(x) reproducing the host C library bit-for-bit.
//
// numpy's Gaussian tail branch computes npy_log1p(-u) with the platform libm
// (glibc on this image), and its result flows straight into the returned
// sample.  CUDA's log1p may differ in the last ulp, so the sketch evaluates
// the classic fdlibm argument-reduction + Remez polynomial algorithm (the
// published algorithm glibc's dbl-64 log1p implements) with explicit
// round-to-nearest operations, fusing exactly the multiply-adds that glibc's
// x86-64 FMA variant (the ifunc chosen on every FMA-capable host) fuses.  tests/
// test_sketch_host.py compiles this header for the host and checks it
// against libm's log1p on millions of inputs.
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define FPI_HD __host__ __device__ __forceinline__
#else
#define FPI_HD inline
#endif

namespace fpi {

#if defined(__CUDA_ARCH__)
FPI_HD double rn_add(double a, double b) { return __dadd_rn(a, b); }
FPI_HD double rn_sub(double a, double b) { return __dsub_rn(a, b); }
FPI_HD double rn_mul(double a, double b) { return __dmul_rn(a, b); }
FPI_HD double rn_div(double a, double b) { return __ddiv_rn(a, b); }
FPI_HD double rn_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
FPI_HD int32_t hi_word(double x) { return (int32_t)__double2hiint(x); }
FPI_HD double with_hi_word(double x, int32_t hi) { return __hiloint2double(hi, __double2loint(x)); }
#else
FPI_HD double rn_add(double a, double b) { volatile double r = a + b; return r; }
FPI_HD double rn_sub(double a, double b) { volatile double r = a - b; return r; }
FPI_HD double rn_mul(double a, double b) { volatile double r = a * b; return r; }
FPI_HD double rn_div(double a, double b) { volatile double r = a / b; return r; }
FPI_HD double rn_fma(double a, double b, double c) { volatile double r = __builtin_fma(a, b, c); return r; }
FPI_HD int32_t hi_word(double x) { uint64_t b; memcpy(&b, &x, 8); return (int32_t)(b >> 32); }
FPI_HD double with_hi_word(double x, int32_t hi) {
  uint64_t b;
  memcpy(&b, &x, 8);
  b = ((uint64_t)(uint32_t)hi << 32) | (b & 0xffffffffull);
  double r;
  memcpy(&r, &b, 8);
  return r;
}
#endif

// Valid for the sampler's arguments x = -u, u in [0, 1) (so x in (-1, 0]);
// the general special cases (x <= -1, inf, nan) are kept for completeness.
FPI_HD double log1p_ieee(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double hfsq, f = 0.0, c = 0.0, s, z, R, u;
  int32_t k, hx, hu = 0, ax;

  hx = hi_word(x);
  ax = hx & 0x7fffffff;
  k = 1;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) {  // x <= -1.0
      if (x == -1.0) return -two54 / 0.0;
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {  // |x| < 2**-29
      if (rn_add(two54, x) > 0.0 && ax < 0x3c900000) return x;
      return rn_fma(-rn_mul(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    if (hx < 0x43400000) {
      u = rn_add(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? rn_sub(1.0, rn_sub(u, x)) : rn_sub(x, rn_sub(u, 1.0));
      c = rn_div(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = rn_sub(u, 1.0);
  }
  hfsq = rn_mul(rn_mul(0.5, f), f);
  const double dk = (double)k;
  if (hu == 0) {  // |f| < 2**-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = rn_fma(dk, ln2_lo, c);
      return rn_fma(dk, ln2_hi, c);
    }
    R = rn_mul(rn_fma(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return rn_sub(f, R);
    return rn_fma(dk, ln2_hi, -rn_sub(rn_sub(R, rn_fma(dk, ln2_lo, c)), f));
  }
  s = rn_div(f, rn_add(2.0, f));
  z = rn_mul(s, s);
  // glibc's dbl-64 evaluation order of the Remez polynomial (pairwise, for ILP):
  // R = z*Lp1 + z^2*(Lp2 + z*Lp3) + z^4*(Lp4 + z*Lp5) + z^6*(Lp6 + z*Lp7)
  {
    const double R2 = rn_fma(z, Lp3, Lp2), R3 = rn_fma(z, Lp5, Lp4), R4 = rn_fma(z, Lp7, Lp6);
    const double z2 = rn_mul(z, z), z4 = rn_mul(z2, z2), z6 = rn_mul(z2, z4);
    R = rn_fma(z, Lp1, rn_mul(z2, R2));
    R = rn_fma(z4, R3, R);
    R = rn_fma(z6, R4, R);
  }
  const double sR = rn_mul(s, rn_add(R, hfsq));
  if (k == 0) return rn_sub(f, rn_sub(hfsq, sR));
  return rn_fma(dk, ln2_hi, -rn_sub(rn_sub(hfsq, rn_add(rn_fma(dk, ln2_lo, c), sR)), f));
}

}  // namespace fpi
