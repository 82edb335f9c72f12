/* CPU check of csrc/fs_glibm.h against the system libm (test infrastructure).
 * Usage: glibm_check N SEED  -> prints one JSON line of mismatch counts.
 * Arguments: random bit patterns over the whole double range, plus the ranges
 * numpy's distributions feed these functions (uniform (0,1) doubles, gamma and
 * beta exponents 1/alpha, ziggurat tails, lognormal exponents). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "../../paper_2508_03148_b200/csrc/fs_glibm.h"

static uint64_t s0, s1;
static uint64_t next(void) {  /* xorshift128+ */
  uint64_t a = s0, b = s1;
  s0 = b; a ^= a << 23; s1 = a ^ b ^ (a >> 17) ^ (b >> 26);
  return s1 + b;
}
static double unif(void) { return (double)(next() >> 11) * 0x1p-53; }
static double anybits(void) { return glm_asf(next()); }
static int same(double a, double b) {
  uint64_t x = glm_asu(a), y = glm_asu(b);
  if (isnan(a) && isnan(b)) return 1;
  return x == y;
}
static void report(const char* f, double a, double b, double got, double want, long* bad) {
  if (*bad < 5)
    fprintf(stderr, "%s(%a, %a): got %a want %a\n", f, a, b, got, want);
  (*bad)++;
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  s0 = argc > 2 ? strtoull(argv[2], 0, 10) * 0x9E3779B97F4A7C15ull + 1 : 1;
  s1 = 0x0123456789abcdefull ^ s0;
  long bad_exp = 0, bad_log = 0, bad_pow = 0, bad_log1p = 0;
  volatile double sink = 0;
  for (long i = 0; i < n; i++) {
    double x, y, g, w;
    /* exp: any bits; |x| < 800; -0.5 z^2 style arguments (negative, moderate) */
    x = (i % 3 == 0) ? anybits() : (i % 3 == 1) ? (unif() - 0.5) * 1600.0 : -unif() * 40.0;
    g = glm_exp(x); w = exp(x);
    if (!same(g, w)) report("exp", x, 0, g, w, &bad_exp);
    /* log: any bits; (0,1) uniforms; near 1; large */
    x = (i % 4 == 0) ? anybits() : (i % 4 == 1) ? unif() : (i % 4 == 2) ? 1.0 + (unif() - 0.5) * 0.25
                                                         : unif() * 1e6;
    g = glm_log(x); w = log(x);
    if (!same(g, w)) report("log", x, 0, g, w, &bad_log);
    /* log1p: -U for U in [0,1); any bits; small */
    x = (i % 3 == 0) ? -unif() : (i % 3 == 1) ? anybits() : (unif() - 0.5) * 1e-3;
    g = glm_log1p(x); w = log1p(x);
    if (!same(g, w)) report("log1p", x, 0, g, w, &bad_log1p);
    /* pow: U^(1/alpha) (gamma/beta), (1 - a + a Y)^(1/a), any bits */
    switch (i % 4) {
      case 0: x = unif(); y = 1.0 / (0.01 + unif()); break;
      case 1: x = 0.5 + unif() * 4.0; y = 1.0 / (0.01 + unif()); break;
      case 2: x = anybits(); y = anybits(); break;
      default: x = unif() * 8.0; y = (unif() - 0.5) * 200.0; break;
    }
    g = glm_pow(x, y); w = pow(x, y);
    if (!same(g, w)) report("pow", x, y, g, w, &bad_pow);
    sink += g;
  }
  /* special values */
  const double sp[] = {0.0, -0.0, 1.0, -1.0, INFINITY, -INFINITY, NAN, 0x1p-1074, 0x1p-1022,
                       0x1.fffffffffffffp1023, 2.0, 0.5, 3.0, -3.0, 1e-300, 709.78, -745.2, 1024.0,
                       -1024.0, 0x1p-60, -0x1p-60, 0x1p63, -0x1p63};
  const int ns = sizeof(sp) / sizeof(sp[0]);
  for (int a = 0; a < ns; a++) {
    if (!same(glm_exp(sp[a]), exp(sp[a]))) report("exp", sp[a], 0, glm_exp(sp[a]), exp(sp[a]), &bad_exp);
    if (!same(glm_log(sp[a]), log(sp[a]))) report("log", sp[a], 0, glm_log(sp[a]), log(sp[a]), &bad_log);
    if (!same(glm_log1p(sp[a]), log1p(sp[a])))
      report("log1p", sp[a], 0, glm_log1p(sp[a]), log1p(sp[a]), &bad_log1p);
    for (int b = 0; b < ns; b++)
      if (!same(glm_pow(sp[a], sp[b]), pow(sp[a], sp[b])))
        report("pow", sp[a], sp[b], glm_pow(sp[a], sp[b]), pow(sp[a], sp[b]), &bad_pow);
  }
  printf("{\"n\": %ld, \"exp\": %ld, \"log\": %ld, \"log1p\": %ld, \"pow\": %ld}\n", n, bad_exp,
         bad_log, bad_log1p, bad_pow);
  return (bad_exp || bad_log || bad_log1p || bad_pow) ? 1 : 0;
}
