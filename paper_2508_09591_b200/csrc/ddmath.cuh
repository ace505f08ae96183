// Double-double arithmetic for the swap-cost kernel's smooth maximum.
//
// The reference evaluates smooth_max with numpy (swap.py:51-57):
//   m * power(sum(power(z/m, gamma)), 1/gamma)
// and the swap decision is the first-occurrence argmin of those doubles
// (swap.py:240).  To reproduce numpy's rounding the GPU needs (a) the same
// summation order (numpy's pairwise add.reduce, see pairwise_sum below) and
// (b) a pow that returns the correctly rounded double.  pow_cr() evaluates
// exp(y*log(x)) in double-double (~2^-100 relative) and rounds once, so it is
// correctly rounded except when the exact value lies within ~2^-100 of a
// rounding midpoint.
//
// Everything here is __host__ __device__ and must be compiled WITHOUT
// floating-point contraction (nvcc -fmad=false, g++ -ffp-contract=off): the
// error-free transforms rely on every + and * being individually rounded.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define HM_HD __host__ __device__ __forceinline__
#else
#define HM_HD inline
#endif

namespace hm {
namespace dd {

struct ddv {
  double hi, lo;
};

HM_HD ddv two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}

HM_HD ddv quick_two_sum(double a, double b) {
  double s = a + b;
  double e = b - (s - a);
  return {s, e};
}

HM_HD ddv two_prod(double a, double b) {
  double p = a * b;
  double e = fma(a, b, -p);
  return {p, e};
}

HM_HD ddv add(ddv a, ddv b) {
  ddv s = two_sum(a.hi, b.hi);
  ddv t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}

HM_HD ddv add_d(ddv a, double b) {
  ddv s = two_sum(a.hi, b);
  s.lo += a.lo;
  return quick_two_sum(s.hi, s.lo);
}

HM_HD ddv mul(ddv a, ddv b) {
  ddv p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}

HM_HD ddv mul_d(ddv a, double b) {
  ddv p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}

// exp of a double-double: argument reduction by ln2 and 2^-10, degree-9
// Taylor polynomial for expm1, ten squarings, scale by 2^m.
HM_HD ddv exp(ddv a) {
  const ddv kLn2 = {6.9314718055994529e-01, 2.3190468138462996e-17};
  if (a.hi > 709.782712893384) return {INFINITY, 0.0};
  if (a.hi < -745.2) return {0.0, 0.0};
  if (a.hi == 0.0 && a.lo == 0.0) return {1.0, 0.0};
  double m = floor(a.hi / kLn2.hi + 0.5);
  ddv r = add(a, mul_d({-kLn2.hi, -kLn2.lo}, m));
  const double kScale = 1.0 / 1024.0;  // exact power of two
  r.hi *= kScale;
  r.lo *= kScale;
  // inverse factorials 1/n!, n = 2..10, as double-double (exact to 2^-106)
  const ddv kInvFact[9] = {
      {0.5, 0.0},
      {0.16666666666666666, 9.25185853854297e-18},
      {0.041666666666666664, 2.3129646346357427e-18},
      {0.008333333333333333, 1.1564823173178714e-19},
      {0.001388888888888889, -5.300543954373577e-20},
      {0.0001984126984126984, 1.7209558293420705e-22},
      {2.48015873015873e-05, 2.1511947866775882e-23},
      {2.7557319223985893e-06, -1.858393274046472e-22},
      {2.755731922398589e-07, 2.3767714622250297e-23}};
  // Horner: p = r*(1 + r*(1/2! + r*(1/3! + ... + r/10!)))
  ddv s = kInvFact[8];
  for (int n = 7; n >= 0; --n) s = add(mul(s, r), kInvFact[n]);
  s = add_d(mul(s, r), 1.0);
  ddv p = mul(s, r);  // expm1(r)
  for (int i = 0; i < 10; ++i) {
    // expm1(2x) = 2 expm1(x) + expm1(x)^2
    ddv p2 = mul(p, p);
    p = add({2.0 * p.hi, 2.0 * p.lo}, p2);
  }
  ddv e = add_d(p, 1.0);
  int mi = (int)m;
  return {ldexp(e.hi, mi), ldexp(e.lo, mi)};
}

// natural log of a positive finite double, as double-double: x = m 2^e with
// m in [0.5, 1); one Newton step y1 = y0 + m*exp(-y0) - 1 from the libm
// estimate y0 = log(m), plus e*ln2 in double-double (no overflow for
// subnormal x).
HM_HD ddv log(double x) {
  if (x == 1.0) return {0.0, 0.0};
  const ddv kLn2 = {6.9314718055994529e-01, 2.3190468138462996e-17};
  int e;
  double m = frexp(x, &e);
  double y0 = ::log(m);
  ddv ym = {y0, 0.0};
  if (m != 0.5) {
    ddv t = mul_d(exp(ddv{-y0, 0.0}), m);
    t = add_d(t, -1.0);
    ym = add_d(t, y0);
  } else {
    ym = {-kLn2.hi, -kLn2.lo};
  }
  ddv el = two_prod((double)e, kLn2.hi);
  el.lo += (double)e * kLn2.lo;
  el = quick_two_sum(el.hi, el.lo);
  return add(el, ym);
}

}  // namespace dd

// Correctly rounded (to ~2^-100) x^y for the smooth-max domain: x >= 0,
// y > 0 finite.  Special values follow C99 pow.
HM_HD double pow_cr(double x, double y) {
  if (x == 1.0 || y == 0.0) return 1.0;
  if (x == 0.0) return y > 0.0 ? 0.0 : INFINITY;
  if (isinf(y)) return x < 1.0 ? (y > 0.0 ? 0.0 : INFINITY) : (y > 0.0 ? INFINITY : 0.0);
  if (y == 1.0) return x;
  dd::ddv l = dd::log(x);
  // y * l exactly enough: y is a double, l a double-double
  dd::ddv yl = dd::mul_d(l, y);
  dd::ddv r = dd::exp(yl);
  return r.hi + r.lo;
}

// numpy's add.reduce over a contiguous run of n doubles (pairwise summation,
// numpy/_core/src/umath/loops_utils.h.src pairwise_sum): n < 8 sequential
// from 0.0, 8 <= n <= 128 eight interleaved accumulators folded
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the remainder sequentially,
// n > 128 halving at a multiple of 8 (one level: n <= 256 supported, no
// recursion so the device stack size stays static).
HM_HD double pairwise_block(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res += a[i];
  return res;
}

HM_HD double pairwise_sum(const double* a, int n) {
  if (n <= 128) return pairwise_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_block(a, n2) + pairwise_block(a + n2, n - n2);
}

// smooth_max of one count vector (swap.py:51-57).  `gamma_inv` must be the
// double 1.0/gamma exactly as Python computes it.  gamma == inf gives the
// exact maximum.  `scratch` holds n doubles.
HM_HD double smooth_max_vec(const double* z, int n, double gamma, double gamma_inv,
                            double* scratch) {
  double m = z[0];
  for (int i = 1; i < n; ++i) m = z[i] > m ? z[i] : m;
  if (!(m > 0.0)) return 0.0;
  if (isinf(gamma)) return m * 1.0;
  for (int i = 0; i < n; ++i) scratch[i] = pow_cr(z[i] / m, gamma);
  double total = pairwise_sum(scratch, n);
  return m * pow_cr(total, gamma_inv);
}

}  // namespace hm
