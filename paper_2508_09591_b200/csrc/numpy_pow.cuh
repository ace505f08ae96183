// smooth_max with numpy's rounding.  Placeholder: correctly rounded pow.
#pragma once
#include "ddmath.cuh"

namespace hm {

HM_HD double np_pow(double x, double y) { return pow_cr(x, y); }

HM_HD double smooth_max_vec_np(const double* z, int n, double gamma, double gamma_inv,
                               double* scratch) {
  double m = z[0];
  for (int i = 1; i < n; ++i) m = z[i] > m ? z[i] : m;
  if (!(m > 0.0)) return 0.0;
  if (isinf(gamma)) return m * 1.0;
  for (int i = 0; i < n; ++i) scratch[i] = np_pow(z[i] / m, gamma);
  double total = pairwise_sum(scratch, n);
  return m * np_pow(total, gamma_inv);
}

}  // namespace hm
