// fs_glibm.h -- glibc 2.39's exp / log / log1p / pow as x86-64 runs them,
// restated so device code reproduces the host libm bit for bit.
//
// numpy's random module calls the C library for these four functions
// (numpy/random/src/distributions/distributions.c: random_standard_gamma,
// random_beta, the ziggurat exponential/normal tails and wedges,
// random_lognormal), and its result feeds accept/reject tests whose outcome
// decides how many Philox words a variate consumes. CUDA's libm differs from
// glibc by up to 2 ulp, so the device uses these instead.
//
// glibc selects an implementation per CPU with an ifunc: on any x86-64 with
// FMA and AVX2 (the build container and the GPU boxes) it runs the variants
// compiled with -mfma -mavx2 (`__exp_fma`, `__log_fma`, `__pow_fma`,
// `__log1p_fma`). Those are the sources in sysdeps/ieee754/dbl-64 (e_exp.c,
// e_log.c, e_pow.c: the table-driven algorithms; s_log1p.c: fdlibm) with GCC's
// floating-point contraction applied. Every fma below is one that GCC formed
// in those binaries (read from their disassembly); every other multiply and add
// is rounded separately. Tables and coefficients come from the installed libm
// (scripts/gen_glibm.py -> fs_glibm_tables.h).
//
// The header compiles as CUDA device code (nvcc) and as host C/C++ (the CPU
// test tests/glibm/ checks it against the system libm on ~10^8 arguments).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define FS_GLM_FN __device__ __forceinline__
#define FS_GLM_TABLE static __device__ const
#else
#include <math.h>
#include <string.h>
#define FS_GLM_FN static inline
#define FS_GLM_TABLE static const
#endif

#include "fs_glibm_tables.h"

// ---- IEEE helpers: every operation rounds once (no contraction on either side) ----
FS_GLM_FN double glm_asf(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
FS_GLM_FN uint64_t glm_asu(double x) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return u;
#endif
}
#ifdef __CUDA_ARCH__
#define GLM_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GLM_MUL(a, b) __dmul_rn((a), (b))
#define GLM_ADD(a, b) __dadd_rn((a), (b))
#define GLM_SUB(a, b) __dsub_rn((a), (b))
#else
#define GLM_FMA(a, b, c) fma((a), (b), (c))
#define GLM_MUL(a, b) ((a) * (b))
#define GLM_ADD(a, b) ((a) + (b))
#define GLM_SUB(a, b) ((a) - (b))
#endif
FS_GLM_FN double glm_t(const uint64_t* t, int i) { return glm_asf(t[i]); }

#define GLM_INF glm_asf(0x7ff0000000000000ull)
#define GLM_P1009 glm_asf(0x7f00000000000000ull)   // 0x1p1009
#define GLM_PM1022 glm_asf(0x0010000000000000ull)  // 0x1p-1022
#define GLM_P52 4503599627370496.0                 // 0x1p52

FS_GLM_FN double glm_invalid(double x) {
  const double d = GLM_SUB(x, x);
  return d / d;
}

// ---------------------------------------------------------------------------
// exp (e_exp.c; __exp_fma)
// ---------------------------------------------------------------------------
// specialcase(): 2^k outside the normal range (|x| in [512, 1024), or a
// subnormal result)
FS_GLM_FN double glm_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = glm_asf(sbits);
    return GLM_MUL(GLM_FMA(scale, tmp, scale), GLM_P1009);
  }
  sbits += 1022ull << 52;
  const double scale = glm_asf(sbits);
  const double st = GLM_MUL(tmp, scale);
  double y = GLM_ADD(scale, st);
  if (y < 1.0) {
    const double hi = GLM_ADD(y, 1.0);
    const double lo = GLM_ADD(GLM_SUB(scale, y), st);
    const double l2 = GLM_ADD(GLM_ADD(GLM_SUB(1.0, hi), y), lo);
    y = GLM_SUB(GLM_ADD(l2, hi), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return GLM_MUL(y, GLM_PM1022);
}

FS_GLM_FN double glm_exp(double x) {
  const uint64_t ix = glm_asu(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return GLM_ADD(x, 1.0);  // |x| < 2^-54
    if (abstop > 0x408) {                                        // |x| >= 1024, inf, nan
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ff) return GLM_ADD(x, 1.0);
      return (ix >> 63) ? 0.0 : GLM_INF;
    }
    abstop = 0;  // 512 <= |x| < 1024: scale may leave the normal range
  }
  const double invln2n = glm_t(fs_glm_exp_hdr, 0), shift = glm_t(fs_glm_exp_hdr, 1);
  const double kd0 = GLM_FMA(x, invln2n, shift);
  const uint64_t ki = glm_asu(kd0);
  const double kd = GLM_SUB(kd0, shift);
  double r = GLM_FMA(kd, glm_t(fs_glm_exp_hdr, 2), x);
  r = GLM_FMA(kd, glm_t(fs_glm_exp_hdr, 3), r);
  const int idx = 2 * (int)(ki & 127);
  const uint64_t top = ki << 45;
  const double tail = glm_t(fs_glm_exp_tab, idx);
  const uint64_t sbits = fs_glm_exp_tab[idx + 1] + top;
  const double r2 = GLM_MUL(r, r);
  const double a = GLM_ADD(r, tail);
  const double p23 = GLM_FMA(r, glm_t(fs_glm_exp_hdr, 5), glm_t(fs_glm_exp_hdr, 4));
  const double p45 = GLM_FMA(r, glm_t(fs_glm_exp_hdr, 7), glm_t(fs_glm_exp_hdr, 6));
  const double b = GLM_FMA(p23, r2, a);
  const double r4 = GLM_MUL(r2, r2);
  const double tmp = GLM_FMA(r4, p45, b);
  if (abstop == 0) return glm_exp_special(tmp, sbits, ki);
  const double scale = glm_asf(sbits);
  return GLM_FMA(scale, tmp, scale);
}

// ---------------------------------------------------------------------------
// log (e_log.c; __log_fma)
// ---------------------------------------------------------------------------
FS_GLM_FN double glm_log(double x) {
  uint64_t ix = glm_asu(x);
  // LO = asuint64(1 - 0x1p-4), HI = asuint64(1 + 0x1.09p-4): close to 1
  if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const uint64_t* B = fs_glm_log_hdr + 7;
    const double r = GLM_SUB(x, 1.0);
    const double b12 = GLM_FMA(r, glm_t(B, 2), glm_t(B, 1));
    const double b45 = GLM_FMA(r, glm_t(B, 5), glm_t(B, 4));
    const double b78 = GLM_FMA(r, glm_t(B, 8), glm_t(B, 7));
    const double r2 = GLM_MUL(r, r);
    const double q1 = GLM_FMA(r2, glm_t(B, 3), b12);
    const double q2 = GLM_FMA(r2, glm_t(B, 6), b45);
    const double r3 = GLM_MUL(r, r2);
    double q3 = GLM_FMA(r2, glm_t(B, 9), b78);
    q3 = GLM_FMA(r3, glm_t(B, 10), q3);
    double q = GLM_FMA(q3, r3, q2);
    q = GLM_FMA(q, r3, q1);
    const double w = GLM_FMA(r, 134217728.0, r);  // r + r * 0x1p27
    const double rhi = GLM_FMA(-134217728.0, r, w);
    const double rhi2 = GLM_MUL(rhi, rhi);
    const double rlo = GLM_SUB(r, rhi);
    const double b0 = glm_t(B, 0);
    const double hi = GLM_FMA(rhi2, b0, r);
    const double lo0 = GLM_FMA(rhi2, b0, GLM_SUB(r, hi));
    const double lo = GLM_FMA(GLM_MUL(b0, rlo), GLM_ADD(r, rhi), lo0);
    const double y = GLM_FMA(q, r3, lo);
    return GLM_ADD(hi, y);
  }
  const uint32_t top = (uint32_t)(ix >> 48);
  if (top - 0x0010u > 0x7fdfu) {  // x < 0x1p-1022, negative, inf or nan
    if (ix * 2 == 0) return -GLM_INF;
    if (ix == 0x7ff0000000000000ull) return x;
    if ((top & 0x8000) || (top & 0x7ff0) == 0x7ff0) return glm_invalid(x);
    ix = glm_asu(GLM_MUL(x, GLM_P52)) - (52ull << 52);  // subnormal: normalise
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = glm_t(fs_glm_log_tab, 2 * i), logc = glm_t(fs_glm_log_tab, 2 * i + 1);
  const double z = glm_asf(iz);
  const double kd = (double)k;
  const uint64_t* A = fs_glm_log_hdr + 2;
  const double w = GLM_FMA(kd, glm_t(fs_glm_log_hdr, 0), logc);
  const double r = GLM_FMA(z, invc, -1.0);
  const double a12 = GLM_FMA(r, glm_t(A, 2), glm_t(A, 1));
  const double hi = GLM_ADD(r, w);
  const double r2 = GLM_MUL(r, r);
  double lo = GLM_ADD(GLM_SUB(w, hi), r);
  lo = GLM_FMA(kd, glm_t(fs_glm_log_hdr, 1), lo);
  const double rr2 = GLM_MUL(r, r2);
  const double a34 = GLM_FMA(r, glm_t(A, 4), glm_t(A, 3));
  const double l2 = GLM_FMA(r2, glm_t(A, 0), lo);
  const double p = GLM_FMA(a34, r2, a12);
  const double y = GLM_FMA(rr2, p, l2);
  return GLM_ADD(y, hi);
}

// ---------------------------------------------------------------------------
// pow (e_pow.c; __pow_fma)
// ---------------------------------------------------------------------------
// log(x) as hi + *tail with ~2^-68 relative error (log_inline)
FS_GLM_FN double glm_pow_log(uint64_t ix, double* tail) {
  const uint64_t tmp = ix - 0x3fe6955500000000ull;
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double z = glm_asf(iz);
  const double kd = (double)k;
  const uint64_t* T = fs_glm_pow_tab + 4 * i;  // invc, pad, logc, logctail
  const uint64_t* A = fs_glm_pow_hdr + 2;
  const double t1 = GLM_FMA(kd, glm_t(fs_glm_pow_hdr, 0), glm_t(T, 2));
  const double lo1 = GLM_FMA(kd, glm_t(fs_glm_pow_hdr, 1), glm_t(T, 3));
  const double r = GLM_FMA(z, glm_t(T, 0), -1.0);
  const double ar = GLM_MUL(r, glm_t(A, 0));
  const double a12 = GLM_FMA(r, glm_t(A, 2), glm_t(A, 1));
  const double a34 = GLM_FMA(r, glm_t(A, 4), glm_t(A, 3));
  const double t2 = GLM_ADD(r, t1);
  const double lo2 = GLM_ADD(GLM_SUB(t1, t2), r);
  const double ar2 = GLM_MUL(r, ar);
  const double ar3 = GLM_MUL(r, ar2);
  const double lo3 = GLM_FMA(ar, r, -ar2);
  const double hi = GLM_ADD(t2, ar2);
  const double a56 = GLM_FMA(r, glm_t(A, 6), glm_t(A, 5));
  const double lo4 = GLM_ADD(GLM_SUB(t2, hi), ar2);
  const double q = GLM_FMA(a56, ar2, a34);
  const double p = GLM_FMA(ar2, q, a12);
  double lo = GLM_ADD(GLM_ADD(GLM_ADD(lo1, lo2), lo3), lo4);
  lo = GLM_FMA(ar3, p, lo);
  const double y = GLM_ADD(hi, lo);
  *tail = GLM_ADD(GLM_SUB(hi, y), lo);
  return y;
}

FS_GLM_FN double glm_pow_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = glm_asf(sbits);
    return GLM_MUL(GLM_FMA(scale, tmp, scale), GLM_P1009);
  }
  sbits += 1022ull << 52;
  const double scale = glm_asf(sbits);
  const double st = GLM_MUL(tmp, scale);
  double y = GLM_ADD(scale, st);
  if (fabs(y) < 1.0) {
    const double one = y < 0.0 ? -1.0 : 1.0;
    const double lo = GLM_ADD(GLM_SUB(scale, y), st);
    const double hi = GLM_ADD(y, one);
    const double l2 = GLM_ADD(GLM_ADD(GLM_SUB(one, hi), y), lo);
    y = GLM_SUB(GLM_ADD(l2, hi), one);
    if (y == 0.0) y = glm_asf(sbits & 0x8000000000000000ull);
  }
  return GLM_MUL(y, GLM_PM1022);
}

FS_GLM_FN double glm_pow_exp(double x, double xtail, uint64_t sign_bias) {
  uint32_t abstop = (uint32_t)(glm_asu(x) >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) {
      const double one = GLM_ADD(x, 1.0);
      return sign_bias ? -one : one;
    }
    if (abstop > 0x408) {
      const double m = sign_bias ? -1.0 : 1.0;
      return (glm_asu(x) >> 63) ? m * 0.0 : m * GLM_INF;
    }
    abstop = 0;
  }
  const double invln2n = glm_t(fs_glm_exp_hdr, 0), shift = glm_t(fs_glm_exp_hdr, 1);
  const double kd0 = GLM_FMA(x, invln2n, shift);
  const uint64_t ki = glm_asu(kd0);
  const double kd = GLM_SUB(kd0, shift);
  double r = GLM_FMA(kd, glm_t(fs_glm_exp_hdr, 2), x);
  r = GLM_FMA(kd, glm_t(fs_glm_exp_hdr, 3), r);
  r = GLM_ADD(xtail, r);
  const int idx = 2 * (int)(ki & 127);
  const uint64_t top = (ki + sign_bias) << 45;
  const double tail = glm_t(fs_glm_exp_tab, idx);
  const uint64_t sbits = fs_glm_exp_tab[idx + 1] + top;
  const double r2 = GLM_MUL(r, r);
  const double a = GLM_ADD(r, tail);
  const double p23 = GLM_FMA(r, glm_t(fs_glm_exp_hdr, 5), glm_t(fs_glm_exp_hdr, 4));
  const double p45 = GLM_FMA(r, glm_t(fs_glm_exp_hdr, 7), glm_t(fs_glm_exp_hdr, 6));
  const double b = GLM_FMA(p23, r2, a);
  const double r4 = GLM_MUL(r2, r2);
  const double tmp = GLM_FMA(r4, p45, b);
  if (abstop == 0) return glm_pow_special(tmp, sbits, ki);
  const double scale = glm_asf(sbits);
  return GLM_FMA(scale, tmp, scale);
}

// 0: not an integer, 1: odd integer, 2: even integer
FS_GLM_FN int glm_checkint(uint64_t iy) {
  const int e = (int)(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ull << (0x3ff + 52 - e))) return 1;
  return 2;
}
FS_GLM_FN int glm_zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1; }
FS_GLM_FN int glm_issignaling(uint64_t ix) {
  return 2 * (ix ^ 0x0008000000000000ull) > 2 * 0x7ff8000000000000ull;
}

FS_GLM_FN double glm_pow(double x, double y) {
  uint64_t sign_bias = 0;
  uint64_t ix = glm_asu(x);
  const uint64_t iy = glm_asu(y);
  uint32_t topx = (uint32_t)(ix >> 52);
  const uint32_t topy = (uint32_t)(iy >> 52);
  if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ff) - 0x3beu >= 0x43eu - 0x3beu) {
    if (glm_zeroinfnan(iy)) {
      if (2 * iy == 0) return glm_issignaling(ix) ? GLM_ADD(x, y) : 1.0;
      if (ix == 0x3ff0000000000000ull) return glm_issignaling(iy) ? GLM_ADD(x, y) : 1.0;
      if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull)
        return GLM_ADD(x, y);
      if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
      if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
      return GLM_MUL(y, y);
    }
    if (glm_zeroinfnan(ix)) {
      double x2 = GLM_MUL(x, x);
      int neg = 0;
      if ((ix >> 63) && glm_checkint(iy) == 1) {
        x2 = -x2;
        neg = 1;
      }
      if (2 * ix == 0 && (iy >> 63)) return neg ? -GLM_INF : GLM_INF;  // divide by zero
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    // x and y are non-zero finite
    if (ix >> 63) {
      const int yint = glm_checkint(iy);
      if (yint == 0) return glm_invalid(x);
      if (yint == 1) sign_bias = 0x800ull << 7;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ff;
    }
    if ((topy & 0x7ff) - 0x3beu >= 0x43eu - 0x3beu) {
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if ((topy & 0x7ff) < 0x3be) return ix > 0x3ff0000000000000ull ? GLM_ADD(y, 1.0)
                                                                    : GLM_SUB(1.0, y);
      return (ix > 0x3ff0000000000000ull) == (topy < 0x800) ? GLM_INF : 0.0;
    }
    if (topx == 0) {  // subnormal x: normalise
      ix = glm_asu(GLM_MUL(x, GLM_P52)) & 0x7fffffffffffffffull;
      ix -= 52ull << 52;
    }
  }
  double lo;
  const double hi = glm_pow_log(ix, &lo);
  const double ehi = GLM_MUL(y, hi);
  const double elo = GLM_FMA(y, lo, GLM_FMA(hi, y, -ehi));
  return glm_pow_exp(ehi, elo, sign_bias);
}

// ---------------------------------------------------------------------------
// log1p (s_log1p.c, fdlibm; __log1p_fma)
// ---------------------------------------------------------------------------
FS_GLM_FN double glm_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000
  const double ln2_lo = 1.90821492927058770002e-10;  // 0x3dea39ef35793c76
  const double Lp1 = glm_asf(0x3fe5555555555593ull), Lp2 = glm_asf(0x3fd999999997fa04ull),
               Lp3 = glm_asf(0x3fd2492494229359ull), Lp4 = glm_asf(0x3fcc71c51d8e78afull),
               Lp5 = glm_asf(0x3fc7466496cb03deull), Lp6 = glm_asf(0x3fc39a09d078c69full),
               Lp7 = glm_asf(0x3fc2f112df3e5244ull);
  const int32_t hx = (int32_t)(glm_asu(x) >> 32);
  const int32_t ax = hx & 0x7fffffff;
  int k;
  double f, c = 0.0;
  int32_t hu;
  if (hx < 0x3fda827a) {  // x < 0.41422
    if (ax >= 0x3ff00000) {  // x <= -1.0
      if (x == -1.0) return -GLM_INF;
      return glm_invalid(x);
    }
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      return GLM_FMA(-GLM_MUL(x, x), 0.5, x);  // x - x*x*0.5
    }
    if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {  // -0.2929 < x < 0.41422: k = 0
      f = x;
      const double hfsq = GLM_MUL(GLM_MUL(x, 0.5), x);
      const double s = x / GLM_ADD(x, 2.0);
      const double z = GLM_MUL(s, s);
      const double R2 = GLM_FMA(z, Lp3, Lp2), R3 = GLM_FMA(z, Lp5, Lp4), R4 = GLM_FMA(z, Lp7, Lp6);
      const double z2 = GLM_MUL(z, z), z4 = GLM_MUL(z2, z2), z6 = GLM_MUL(z2, z4);
      double R = GLM_FMA(z, Lp1, GLM_MUL(z2, R2));
      R = GLM_FMA(z4, R3, R);
      R = GLM_FMA(z6, R4, R);
      const double sr = GLM_MUL(GLM_ADD(R, hfsq), s);
      return GLM_SUB(f, GLM_SUB(hfsq, sr));
    }
    k = 1;  // -1 < x <= -0.2929
  } else if (hx > 0x7fefffff) {
    return GLM_ADD(x, x);  // inf or nan
  }
  // k != 0
  double u;
  if (hx <= 0x433fffff) {
    u = GLM_ADD(x, 1.0);
    hu = (int32_t)(glm_asu(u) >> 32);
    k = (hu >> 20) - 1023;
    c = k > 0 ? GLM_SUB(1.0, GLM_SUB(u, x)) : GLM_SUB(x, GLM_SUB(u, 1.0));
    c = c / u;
  } else {
    u = x;
    hu = hx;
    k = (hu >> 20) - 1023;
    c = 0.0;
  }
  hu &= 0x000fffff;
  const uint64_t ulo = glm_asu(u) & 0xffffffffull;
  if (hu < 0x6a09e) {
    u = glm_asf(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | ulo);
  } else {
    k += 1;
    u = glm_asf(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | ulo);
    hu = (0x00100000 - hu) >> 2;
  }
  f = GLM_SUB(u, 1.0);
  const double hfsq = GLM_MUL(GLM_MUL(f, 0.5), f);
  const double kd = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return GLM_FMA(kd, ln2_hi, GLM_FMA(kd, ln2_lo, c));
    }
    const double R = GLM_MUL(GLM_FMA(-f, glm_asf(0x3fe5555555555555ull), 1.0), hfsq);
    if (k == 0) return GLM_SUB(f, R);
    const double t = GLM_SUB(GLM_SUB(R, GLM_FMA(kd, ln2_lo, c)), f);
    return GLM_FMA(kd, ln2_hi, -t);
  }
  const double s = f / GLM_ADD(f, 2.0);
  const double z = GLM_MUL(s, s);
  const double R2 = GLM_FMA(z, Lp3, Lp2), R3 = GLM_FMA(z, Lp5, Lp4), R4 = GLM_FMA(z, Lp7, Lp6);
  const double z2 = GLM_MUL(z, z), z4 = GLM_MUL(z2, z2), z6 = GLM_MUL(z2, z4);
  double R = GLM_FMA(z, Lp1, GLM_MUL(z2, R2));
  R = GLM_FMA(z4, R3, R);
  R = GLM_FMA(z6, R4, R);
  const double sr = GLM_MUL(GLM_ADD(R, hfsq), s);
  if (k == 0) return GLM_SUB(f, GLM_SUB(hfsq, sr));
  const double t = GLM_SUB(GLM_SUB(hfsq, GLM_ADD(GLM_FMA(kd, ln2_lo, c), sr)), f);
  return GLM_FMA(kd, ln2_hi, -t);
}
