// Probe of the vrcp14pd rounding used by numpy's SVML pow (__svml_pow8_ha):
// rr = vrndscalepd(vrcp14pd(m), 1/32) for the vgetmantpd mantissa m in
// [0.5, 1).  Prints whether rcp14 depends only on the top b mantissa bits and
// the exact m thresholds where rr steps down by 1/32; those thresholds are the
// HM_NP_RCP_THRESH table in paper_2508_09591_b200/csrc/numpy_pow.cuh.
// Build/run on an AVX-512 host:  gcc -O1 -mavx512f svml_pow_probe.c -lm && ./a.out
#include <immintrin.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <math.h>
static double rr_of(double m) {
  __m512d v = _mm512_set1_pd(m);
  __m512d r = _mm512_rcp14_pd(v);
  __m512d s = _mm512_roundscale_pd(r, 0x58);
  double out[8]; _mm512_storeu_pd(out, s); return out[0];
}
static double rcp14(double m) {
  double out[8]; _mm512_storeu_pd(out, _mm512_rcp14_pd(_mm512_set1_pd(m))); return out[0];
}
static uint64_t bits(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
static double from(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
int main() {
  // does rcp14 depend only on the top b mantissa bits?
  for (int b = 10; b <= 24; b += 2) {
    int same = 1;
    for (uint64_t i = 0; i < 200000; i++) {
      uint64_t u = bits(0.75) + i * 7919ull * 1000003ull % (bits(1.5) - bits(0.75));
      uint64_t mask = ~((1ull << (52 - b)) - 1);
      if (rcp14(from(u)) != rcp14(from(u & mask))) { same = 0; break; }
    }
    printf("top %d bits determine rcp14: %d\n", b, same);
  }
  // thresholds of rndscale(rcp14(m), 1/32): m where rr changes, scanning m in [0.75, 1.5)
  double prev = rr_of(0.5);
  uint64_t lo = bits(0.5), hi = bits(1.0);
  // coarse scan at 2^-20 steps then refine by binary search
  uint64_t step = 1ull << 28;
  for (uint64_t u = lo + step; u < hi; u += step) {
    double cur = rr_of(from(u));
    if (cur != prev) {
      uint64_t a = u - step, c = u;  // rr(a) == prev, rr(c) == cur
      while (c - a > 1) { uint64_t mid = a + (c - a) / 2; if (rr_of(from(mid)) == prev) a = mid; else c = mid; }
      printf("T %.17g %a %.17g->%.17g\n", from(c), from(c), prev, cur);
      prev = cur;
    }
  }
  return 0;
}
