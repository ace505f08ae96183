// numpy's float64 power, restated for the GPU (and host), bit for bit.
//
// numpy 2.3 on an AVX512_SKX host evaluates np.power(float64, float64) with
// Intel SVML's __svml_pow8_ha (numpy/_core/src/umath/svml, BSD-3-Clause),
// which is NOT correctly rounded (~5% of results differ by 1 ulp from the
// correctly rounded value).  The reference's swap decision is the argmin of
// smooth-max costs computed with that pow (swap.py:51-57, 240), so the
// decision on near-ties depends on SVML's exact rounding.  This header
// restates the __svml_pow8_ha main path operation by operation (one lane):
// log2(x) via getmant/getexp, a 32-entry table indexed by the 5-bit rounded
// vrcp14pd reciprocal and a degree-8 polynomial with a double-double
// correction; y*log2(x) with round-toward-zero products; 2^t via a shifter
// (round-down add), a 16-entry 2^(j/16) table and a degree-6 polynomial.
// vrcp14pd depends only on the top 16 mantissa bits; its rounding to 1/32 is
// reproduced by the measured threshold table kRcpThresh (probed on the
// instruction, tests/native/svml_pow_probe.c).  Special operands (x <= 0 or
// non-finite, y non-finite, |y*log2 x| > 1021.5) take SVML's scalar rare path;
// here they follow C99 pow with a correctly rounded result.
// (vgetmantpd imm 0xa normalises to [1/2, 1).)
//
// The constants below are numpy's table __svml_dpow_ha_data_internal_avx512
// (extracted by tests/native/extract_svml_pow.py from the installed numpy).
// Compile without contraction (nvcc -fmad=false / g++ -ffp-contract=off).
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>
#if !defined(__CUDA_ARCH__)
#include <fenv.h>
#endif

#include "ddmath.cuh"

namespace hm {
namespace npsvml {

#define HM_NP_kLogHiA \
  0x0000000000000000ull, 0xbfa6bad3758e0000ull, 0xbfb663f6fac90000ull, 0xbfc08c588cda8000ull, \
  0xbfc5c01a39fc0000ull, 0xbfcacf5e2db50000ull, 0xbfcfbc16b9028000ull, 0xbfd24407ab0e0000ull, \
  0xbfd49a784bcd0000ull, 0xbfd6e221cd9d0000ull, 0xbfd91bba891f0000ull, 0xbfdb47ebf7388000ull, \
  0xbfdd6753e0330000ull, 0xbfdf7a8568cb0000ull, 0xbfe0c10500d64000ull, 0xbfe1bf311e95e000ull,
#define HM_NP_kLogHiB \
  0x3fda8ff971810000ull, 0x3fd8a8980abfc000ull, 0x3fd6cb0f6865c000ull, 0x3fd4f6fbb2cec000ull, \
  0x3fd32bfee3710000ull, 0x3fd169c053640000ull, 0x3fcf5fd8a9060000ull, 0x3fcbfc67a8000000ull, \
  0x3fc8a8980abf8000ull, 0x3fc563dc29ff8000ull, 0x3fc22dadc2ab0000ull, 0x3fbe0b1ae8f30000ull, \
  0x3fb7d60496d00000ull, 0x3fb1bb32a6000000ull, 0x3fa77394c9da0000ull, 0x3f9743ee86200000ull,
#define HM_NP_kLogLoA \
  0x0000000000000000ull, 0xbd5fb0e626c0de13ull, 0xbd33167ccc538261ull, 0x3d2871a7610e40bdull, \
  0x3d54bc302ffa76fbull, 0x3d436c101ee13440ull, 0x3d47f5dc57266758ull, 0xbd3ce60916e52e91ull, \
  0xbd5b8afe492bf6ffull, 0xbd49bcaf1aa4168aull, 0xbd5708b4b2b5056cull, 0xbd250520a377c7ecull, \
  0x3d55f101c141e670ull, 0xbd3b3b3864c60011ull, 0x3d45669df6a2b592ull, 0x3d5fe43895d8ac46ull,
#define HM_NP_kLogLoB \
  0x3d44bc302ffa76fbull, 0xbd266cccab240e90ull, 0x3d41d406db502403ull, 0x3d3661e393a16b95ull, \
  0xbd51979a5db68722ull, 0xbd4d4f1b95e0ff45ull, 0x3d5f1a4847f7b278ull, 0xbd3667f21fa8423full, \
  0x3d5e9933354dbf17ull, 0x3d56590643906f2aull, 0x3d5a4b69691d7994ull, 0xbd054cda62d3926eull, \
  0xbd512ce6312ebb82ull, 0x3d552743318a8a57ull, 0xbd54e55443478fe0ull, 0xbd495539356f93dcull,
#define HM_NP_kExpHi \
  0x3ff0000000000000ull, 0x3ff0b5586cf9890full, 0x3ff172b83c7d517bull, 0x3ff2387a6e756238ull, \
  0x3ff306fe0a31b715ull, 0x3ff3dea64c123422ull, 0x3ff4bfdad5362a27ull, 0x3ff5ab07dd485429ull, \
  0x3ff6a09e667f3bcdull, 0x3ff7a11473eb0187ull, 0x3ff8ace5422aa0dbull, 0x3ff9c49182a3f090ull, \
  0x3ffae89f995ad3adull, 0x3ffc199bdd85529cull, 0x3ffd5818dcfba487ull, 0x3ffea4afa2a490daull,
#define HM_NP_kExpLo \
  0x0000000000000000ull, 0x3c979aa65d837b6dull, 0xbc801b15eaa59348ull, 0x3c968efde3a8a894ull, \
  0x3c834d754db0abb6ull, 0x3c859f48a72a4c6dull, 0x3c7690cebb7aafb0ull, 0x3c9063e1e21c5409ull, \
  0xbc93b3efbf5e2228ull, 0xbc7b32dcb94da51dull, 0x3c8db72fc1f0eab4ull, 0x3c71affc2b91ce27ull, \
  0x3c8c1a7792cb3387ull, 0x3c736eae30af0cb3ull, 0x3c74a385a63d07a7ull, 0xbc8ff7128fd391f0ull,

constexpr uint64_t kC0 = 0x40071547652b82feull;
constexpr uint64_t kP400 = 0xc0627a394386376full;
constexpr uint64_t kP440 = 0x4054873cf87141d1ull;
constexpr uint64_t kP480 = 0xc04715473528efc1ull;
constexpr uint64_t kP4c0 = 0x403a617607e55815ull;
constexpr uint64_t kP500 = 0xc02ec709dc3b71a1ull;
constexpr uint64_t kP540 = 0x4022776c50effbdeull;
constexpr uint64_t kP580 = 0xc0171547652b82fcull;
constexpr uint64_t kP5c0 = 0x400ec709dc3a03fdull;
constexpr uint64_t kP600 = 0xbc8778d9c7190437ull;
constexpr uint64_t kP640 = 0x3c8777df70b75d10ull;
constexpr uint64_t kShifter = 0x42f8000000003ff0ull;
constexpr uint64_t kMaskR = 0xbfffffffffffffffull;
constexpr uint64_t kQ700 = 0x3f24a1d7f58c2d59ull;
constexpr uint64_t kQ740 = 0x3f55d7472783d279ull;
constexpr uint64_t kQ780 = 0x3f83b2ad1b14ebaaull;
constexpr uint64_t kQ7c0 = 0x3fac6b08d4ad8eb9ull;
constexpr uint64_t kQ800 = 0x3fcebfbdff84554dull;
constexpr uint64_t kQ840 = 0x3fe62e42fefa398bull;
constexpr uint64_t kRange = 0x408fec0000000000ull;

#if defined(__CUDACC__)
__constant__ uint64_t kLogHiA_d[16] = {HM_NP_kLogHiA};
__constant__ uint64_t kLogHiB_d[16] = {HM_NP_kLogHiB};
__constant__ uint64_t kLogLoA_d[16] = {HM_NP_kLogLoA};
__constant__ uint64_t kLogLoB_d[16] = {HM_NP_kLogLoB};
__constant__ uint64_t kExpHi_d[16] = {HM_NP_kExpHi};
__constant__ uint64_t kExpLo_d[16] = {HM_NP_kExpLo};
#endif
static const uint64_t kLogHiA_h[16] = {HM_NP_kLogHiA};
static const uint64_t kLogHiB_h[16] = {HM_NP_kLogHiB};
static const uint64_t kLogLoA_h[16] = {HM_NP_kLogLoA};
static const uint64_t kLogLoB_h[16] = {HM_NP_kLogLoB};
static const uint64_t kExpHi_h[16] = {HM_NP_kExpHi};
static const uint64_t kExpLo_h[16] = {HM_NP_kExpLo};

#if defined(__CUDA_ARCH__)
#define HM_NP_TAB(name, i) name##_d[i]
#else
#define HM_NP_TAB(name, i) name##_h[i]
#endif

// m thresholds where round(vrcp14(m) * 32) / 32 steps down by 1/32, m in [0.75, 1.5)
// m thresholds where round(vrcp14(m) * 32) / 32 steps down by 1/32, m in [0.5, 1)
#define HM_NP_RCP_THRESH \
  0.5039520263671875, 0.51201629638671875, 0.5203399658203125, 0.5289306640625, \
  0.53781890869140625, 0.54698944091796875, 0.5565338134765625, 0.56638336181640625, \
  0.5765838623046875, 0.58715057373046875, 0.59814453125, 0.6095123291015625, \
  0.62137603759765625, 0.6336517333984375, 0.6464691162109375, 0.6598052978515625, \
  0.67369842529296875, 0.68816375732421875, 0.70330047607421875, 0.71909332275390625, \
  0.73563385009765625, 0.7529449462890625, 0.77109527587890625, 0.7901153564453125, \
  0.81014251708984375, 0.83116912841796875, 0.85334014892578125, 0.876708984375, \
  0.90142822265625, 0.9275360107421875, 0.95523834228515625, 0.98464202880859375

HM_HD double as_d(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
HM_HD uint64_t as_u(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

// explicit-rounding primitives ({rn,rz,rd}-sae in the SVML code)
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double mul_rz(double a, double b) { return __dmul_rz(a, b); }
__device__ __forceinline__ double fma_rz(double a, double b, double c) { return __fma_rz(a, b, c); }
__device__ __forceinline__ double add_rz(double a, double b) { return __dadd_rz(a, b); }
__device__ __forceinline__ double add_rd(double a, double b) { return __dadd_rd(a, b); }
__device__ __forceinline__ double sub_rz(double a, double b) { return __dsub_rz(a, b); }
#else
inline double fma_rn(double a, double b, double c) { return fma(a, b, c); }
inline double with_mode(int mode, double (*f)(double, double, double), double a, double b, double c) {
  int old = fegetround();
  fesetround(mode);
  volatile double va = a, vb = b, vc = c;
  volatile double r = f(va, vb, vc);
  fesetround(old);
  return r;
}
inline double op_mul(double a, double b, double) { return a * b; }
inline double op_add(double a, double b, double) { return a + b; }
inline double op_fma(double a, double b, double c) { return fma(a, b, c); }
inline double op_sub(double a, double b, double) { return a - b; }
inline double mul_rz(double a, double b) { return with_mode(FE_TOWARDZERO, op_mul, a, b, 0.0); }
inline double fma_rz(double a, double b, double c) { return with_mode(FE_TOWARDZERO, op_fma, a, b, c); }
inline double add_rz(double a, double b) { return with_mode(FE_TOWARDZERO, op_add, a, b, 0.0); }
inline double add_rd(double a, double b) { return with_mode(FE_DOWNWARD, op_add, a, b, 0.0); }
inline double sub_rz(double a, double b) { return with_mode(FE_TOWARDZERO, op_sub, a, b, 0.0); }
#endif

// one lane of __svml_pow8_ha; returns false when SVML would take its rare path
HM_HD bool pow_main(double x, double y, double* out) {
  // special-lane masks: vfpclasspd x 0xdf, y 0x99
  if (!(x > 0.0) || isinf(x) || isnan(x) || isinf(y) || isnan(y)) return false;
  // vgetmantpd imm 0xa: mantissa in [0.5, 1); vgetexppd: floor(log2 x)
  int e;
  double m = frexp(x, &e);           // x = m * 2^e, m in [0.5, 1)
  double ex = (double)(e - 1);
  // vrcp14pd + vrndscalepd(1/32) -> rr in [1, 2]: measured threshold table
  const double th[32] = {HM_NP_RCP_THRESH};
  int k = 0;
  for (int i = 0; i < 32; ++i) k += m >= th[i];
  double rr = 2.0 - 0.03125 * k;
  uint64_t ib = as_u(rr) >> 47;
  int j = (int)(ib & 15u);
  bool hi_tab = (ib >> 4) & 1u;
  double l_hi = as_d(hi_tab ? HM_NP_TAB(kLogHiB, j) : HM_NP_TAB(kLogHiA, j));
  double l_lo = as_d(hi_tab ? HM_NP_TAB(kLogLoB, j) : HM_NP_TAB(kLogLoA, j));
  if (rr < 1.5) ex = ex + 1.0;
  double R = fma_rn(m * 0.5, rr, -0.5);
  double R2 = R * R;
  double p9 = fma_rn(as_d(kP400), R, as_d(kP440));
  double p2 = fma_rn(as_d(kP480), R, as_d(kP4c0));
  double p7 = fma_rn(as_d(kP500), R, as_d(kP540));
  double p3 = fma_rn(as_d(kP580), R, as_d(kP5c0));
  double p15 = fma_rn(as_d(kP600), R, as_d(kP640));
  p9 = fma_rn(R2, p9, p2);
  double R4 = R2 * R2;
  p7 = fma_rn(R2, p7, p3);
  p9 = fma_rn(R4, p9, p7);
  p9 = fma_rn(R2, p9, p15);
  double P = fma_rn(R, p9, l_lo);
  double H0 = l_hi + ex;
  const double c0 = as_d(kC0);
  double S = fma_rn(c0, R, H0);
  double d6 = S - H0;
  double z4 = fma_rn(-R, d6, S);
  double z14 = fma_rn(R, c0, -d6);
  double z5 = S - z4;
  z14 = fma_rn(-z14, R, z14);
  double z12 = fma_rn(d6, R, -z5);
  double z7 = z14 - z12;
  double z8 = P + z7;
  double lh = z4 + z8;                 // log2(x), high part
  double th_ = mul_rz(lh, y);
  double z9 = lh - z4;
  double tl = fma_rz(y, lh, -th_);
  double ll = z8 - z9;                 // log2(x), low part
  tl = fma_rz(y, ll, tl);
  double t = add_rz(th_, tl);          // y * log2(x)
  double tz = t - th_;
  double sh = add_rd(t, as_d(kShifter));
  // vreducepd imm 0x41: t - floor(16 t)/16, final subtraction truncated (probed)
  double red = sub_rz(t, floor(t * 16.0) * 0.0625);
  double z6 = tl - tz;
  double r = red + z6;
  r = as_d(as_u(r) & kMaskR);
  if (!(fabs(t) <= as_d(kRange))) return false;
  uint64_t sb = as_u(sh);
  int j2 = (int)(sb & 15u);
  double e_hi = as_d(HM_NP_TAB(kExpHi, j2));
  double e_lo = as_d(HM_NP_TAB(kExpLo, j2));
  double r2 = r * r;
  double q1 = fma_rn(as_d(kQ700), r, as_d(kQ740));
  double q11 = fma_rn(as_d(kQ780), r, as_d(kQ7c0));
  double q15 = fma_rn(as_d(kQ800), r, as_d(kQ840));
  q1 = fma_rn(r2, q1, q11);
  q1 = fma_rn(r2, q1, q15);
  q1 = fma_rn(r, q1, e_lo);
  q1 = fma_rn(e_hi, q1, e_hi);
  double scale = as_d((sb << 48) & 0x7ff0000000000000ull);
  *out = q1 * scale;
  return true;
}

}  // namespace npsvml

// np.power(x, y) for float64 as numpy computes it (AVX512_SKX host).
HM_HD double np_pow(double x, double y) {
  double r;
  if (npsvml::pow_main(x, y, &r)) return r;
  return pow_cr(x, y);
}

// smooth_max of one vector with numpy's rounding (swap.py:51-57).
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
