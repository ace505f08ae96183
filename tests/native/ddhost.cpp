// Host build of the product's double-double math (csrc/ddmath.cuh) so the CPU
// test suite can check correct rounding without a GPU.  Test-only.
#include "../../paper_2508_09591_b200/csrc/ddmath.cuh"
#include "../../paper_2508_09591_b200/csrc/numpy_pow.cuh"
extern "C" double hm_host_pow_cr(double x, double y) { return hm::pow_cr(x, y); }
extern "C" double hm_host_smooth_max(const double* z, int n, double gamma) {
  double scratch[256];
  return hm::smooth_max_vec(z, n, gamma, 1.0 / gamma, scratch);
}
extern "C" double hm_host_pairwise(const double* a, int n) { return hm::pairwise_sum(a, n); }
// smooth max over `rows` contiguous vectors of length n (int64 counts)
extern "C" void hm_host_smooth_max_rows(const int64_t* z, long rows, int n, double gamma,
                                        double* out) {
  double buf[256], scratch[256];
  double ginv = 1.0 / gamma;
  for (long r = 0; r < rows; ++r) {
    for (int i = 0; i < n; ++i) buf[i] = (double)z[r * n + i];
    out[r] = hm::smooth_max_vec_np(buf, n, gamma, ginv, scratch);
  }
}
extern "C" void hm_host_np_pow(const double* x, const double* y, double* out, long n) {
  for (long i = 0; i < n; ++i) out[i] = hm::np_pow(x[i], y[i]);
}
