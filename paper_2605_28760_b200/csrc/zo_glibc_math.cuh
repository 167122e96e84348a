// glibc-equivalent log1p for the ziggurat tail (device + host).
//
// numpy's random_standard_normal tail branch calls npy_log1p -> glibc log1p
// (numerics.py:161-168 -> numpy distributions.c).  glibc 2.39 on x86-64 CPUs
// with FMA dispatches to the fdlibm-lineage s_log1p.c compiled with -mfma, and
// GCC contracts specific a*b+c forms into FMAs.  Device libm log1p (and a
// correctly rounded log1p) differ from it on ~4% of tail inputs, so the tail
// value would not be bit-exact.  This restatement spells out every FMA the
// glibc build uses (established by disassembly + 3e8-input comparison against
// the container's libm: 0 mismatches).
//
// The algorithm, its Lp1..Lp7 / ln2_hi / ln2_lo constants and its variable names
// follow fdlibm's s_log1p.c as carried by glibc (sysdeps/ieee754/dbl-64/s_log1p.c),
// which bears this notice:
//
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this
//   software is freely granted, provided that this notice
//   is preserved.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define ZO_HD __host__ __device__ __forceinline__
#else
#define ZO_HD static inline
#endif

namespace zo {

ZO_HD int32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  uint64_t u;
  __builtin_memcpy(&u, &x, 8);
  return (int32_t)(u >> 32);
#endif
}
ZO_HD double with_hi_word(double x, uint32_t h) {
#ifdef __CUDA_ARCH__
  return __hiloint2double((int)h, __double2loint(x));
#else
  uint64_t u;
  __builtin_memcpy(&u, &x, 8);
  u = (u & 0xffffffffULL) | ((uint64_t)h << 32);
  __builtin_memcpy(&x, &u, 8);
  return x;
#endif
}
ZO_HD double fma_rn(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}
// Explicit round-to-nearest mul/add/sub/div so nvcc never contracts them.
ZO_HD double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
ZO_HD double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
ZO_HD double sub_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
ZO_HD double div_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}

// log1p(x) as computed by the container's glibc on an FMA-capable x86-64 host.
ZO_HD double glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
               Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
               Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double hfsq, f = 0.0, c = 0.0, s, z, R, u, dk;
  int32_t k, hx, hu = 0, ax;
  hx = hi_word(x);
  ax = hx & 0x7fffffff;
  k = 1;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) {
      if (x == -1.0) return -__builtin_huge_val();
      return __builtin_nan("");
    }
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return fma_rn(-mul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return add_rn(x, x);
  if (k != 0) {
    if (hx < 0x43400000) {
      u = add_rn(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? sub_rn(1.0, sub_rn(u, x)) : sub_rn(x, sub_rn(u, 1.0));
      c = div_rn(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, (uint32_t)hu | 0x3ff00000u);
    } else {
      k += 1;
      u = with_hi_word(u, (uint32_t)hu | 0x3fe00000u);
      hu = (0x00100000 - hu) >> 2;
    }
    f = sub_rn(u, 1.0);
  }
  dk = (double)k;
  hfsq = mul_rn(mul_rn(0.5, f), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma_rn(dk, ln2_lo, c);
      return fma_rn(dk, ln2_hi, c);
    }
    R = mul_rn(hfsq, fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return sub_rn(f, R);
    return fma_rn(dk, ln2_hi, -sub_rn(sub_rn(R, fma_rn(dk, ln2_lo, c)), f));
  }
  s = div_rn(f, add_rn(2.0, f));
  z = mul_rn(s, s);
  {
    double R2 = fma_rn(z, Lp3, Lp2), R3 = fma_rn(z, Lp5, Lp4), R4 = fma_rn(z, Lp7, Lp6);
    double z2 = mul_rn(z, z), z4 = mul_rn(z2, z2), z6 = mul_rn(z4, z2);
    R = fma_rn(z6, R4, fma_rn(z4, R3, fma_rn(z, Lp1, mul_rn(z2, R2))));
  }
  double q = mul_rn(s, add_rn(hfsq, R));
  if (k == 0) return sub_rn(f, sub_rn(hfsq, q));
  return fma_rn(dk, ln2_hi, -sub_rn(sub_rn(hfsq, add_rn(q, fma_rn(dk, ln2_lo, c))), f));
}

}  // namespace zo
