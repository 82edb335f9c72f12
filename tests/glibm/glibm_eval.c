/* csrc/fs_glibm.h compiled for the host, as a shared library for
 * tests/test_boundaries.py (test infrastructure): fn 1 exp, 2 log, 3 log1p,
 * 4 pow(x[i], y[i]) -- the codes of fs_eval / oracle fso_libm. */
#include <stdint.h>
#include "../../paper_2508_03148_b200/csrc/fs_glibm.h"

void glm_eval(int fn, const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    switch (fn) {
      case 1: out[i] = glm_exp(x[i]); break;
      case 2: out[i] = glm_log(x[i]); break;
      case 3: out[i] = glm_log1p(x[i]); break;
      default: out[i] = glm_pow(x[i], y[i]); break;
    }
  }
}
