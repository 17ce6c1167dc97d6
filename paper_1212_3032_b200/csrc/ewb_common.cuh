// Shared device code for the sm_100a FP64 BEM hot path.
//
// Everything here restates the reference numerics (ewbem 0.1.0):
//   radial scalars, closed form ........ kernels.py:102-119
//   radial scalars, power series ....... kernels.py:36-53, 122-138
//   static (Kelvin) scalars ............ kernels.py:141-152
//   weighted U/T contraction ........... kernels.py:327-357
// reorganised for a GPU: the closed-form brackets are factored so that
// e^{-i z_s}, e^{-i z_p} and 1/z are evaluated once per quadrature point
// and reused by all four scalars and all 18 tensor entries; 1/z is a
// per-frequency constant times 1/r; the series is a real-coefficient
// Horner scheme in w = -i z (the reference's 24 power-sum terms, of which
// the first EWB_SERIES_TERMS already agree to < 1e-18 for |z| < 0.35).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef EWB_SERIES_TERMS
#define EWB_SERIES_TERMS 16
#endif

namespace ewb {

// Every kernel launch of the library is counted (ewb_launch_count) so the
// benchmark can report exactly how many of OUR kernels ran in its timed
// region.  Usage:  EWB_NOTE kernel<<<...>>>(...);
void note_launch();
#define EWB_NOTE ::ewb::note_launch(),

// Debug build (-DEWB_DEBUG_CHECKS; read through ewb_debug_checks in the C
// ABI): device-side invariant checks (index bounds, ring-slot bookkeeping,
// scratch capacity) count violations and keep the first violated site per
// translation unit, and every workspace is filled with NaN before a call so
// a read of a word the kernels never wrote poisons the results the parity
// tests compare.  This stands in for compute-sanitizer, which the GPU pool
// does not run.  The release build compiles all of it away.
#ifdef EWB_DEBUG_CHECKS
static __device__ unsigned long long g_ewb_dbg[2];
#define EWB_DCHECK(cond, site)                                        \
  do {                                                                \
    if (!(cond) && atomicAdd(&::ewb::g_ewb_dbg[0], 1ull) == 0ull)     \
      ::ewb::g_ewb_dbg[1] = (unsigned long long)(site);               \
  } while (0)
#define EWB_DEBUG_TU(name)                                            \
  void dbg_fetch_##name(unsigned long long* o) {                      \
    cudaMemcpyFromSymbol(o, g_ewb_dbg, sizeof(g_ewb_dbg));            \
  }                                                                   \
  void dbg_reset_##name() {                                           \
    const unsigned long long z[2] = {0ull, 0ull};                     \
    cudaMemcpyToSymbol(g_ewb_dbg, z, sizeof(z));                      \
  }
inline cudaError_t dbg_poison(void* p, size_t bytes, cudaStream_t s) {
  return p && bytes ? cudaMemsetAsync(p, 0xff, bytes, s) : cudaSuccess;   // all-ones = NaN
}
constexpr bool kDebugChecks = true;
#else
#define EWB_DCHECK(cond, site) ((void)0)
#define EWB_DEBUG_TU(name)                                            \
  void dbg_fetch_##name(unsigned long long* o) { o[0] = o[1] = 0ull; } \
  void dbg_reset_##name() {}
inline cudaError_t dbg_poison(void*, size_t, cudaStream_t) { return cudaSuccess; }
constexpr bool kDebugChecks = false;
#endif

constexpr double kSeriesSwitch = 0.35;   // kernels.py:36 (strict <)
constexpr double kFarRatio = 4.0;        // quadrature.py:206 far_threshold
constexpr double kNearRatio = 1.5;       // quadrature.py:207 near_threshold
constexpr uint8_t kNeumann = 0;          // assembly.py:32
constexpr uint8_t kDirichlet = 1;        // assembly.py:33

struct cplx {
  double re, im;
};

__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx operator-(cplx a) { return {-a.re, -a.im}; }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx operator*(cplx a, double s) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx conj(cplx a) { return {a.re, -a.im}; }
__device__ __forceinline__ double abs2(cplx a) { return fma(a.re, a.re, a.im * a.im); }
// acc += s * a (s real)
__device__ __forceinline__ void axpy(cplx& acc, double s, cplx a) {
  acc.re = fma(s, a.re, acc.re);
  acc.im = fma(s, a.im, acc.im);
}
// acc += a * b (complex)
__device__ __forceinline__ void cfma(cplx& acc, cplx a, cplx b) {
  acc.re = fma(a.re, b.re, fma(-a.im, b.im, acc.re));
  acc.im = fma(a.re, b.im, fma(a.im, b.re, acc.im));
}
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  // Smith's algorithm (robust); rounding-level parity with numpy's division.
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, den = b.re + b.im * r;
    return {(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  } else {
    double r = b.re / b.im, den = b.re * r + b.im;
    return {(a.re * r + a.im) / den, (a.im * r - a.re) / den};
  }
}

// t = -i/z - 1/z^2 = ir (ta + tb ir): two FMA + two MUL per wave
__device__ __forceinline__ cplx t_closed(cplx ta, cplx tb, double ir) {
  return {fma(tb.re, ir, ta.re) * ir, fma(tb.im, ir, ta.im) * ir};
}
// the same with ir2 = ir^2 given: one constant operand per instruction (a
// DFMA takes a single constant-bank operand), for kernels whose frequency
// constants are kernel parameters
__device__ __forceinline__ cplx t_closed2(cplx ta, cplx tb, double ir, double ir2) {
  return {fma(ta.re, ir, tb.re * ir2), fma(ta.im, ir, tb.im * ir2)};
}

// Per-frequency constants (host-computed exactly as kernels.py:56-77 and
// material.py:83-94 do, then passed by value).
struct FreqConst {
  cplx ks, kp;          // omega / c_s, omega / c_p
  // t = -i/z - 1/z^2 of the closed form (kernels.py:105-119) with z = k r:
  // t = (ta + tb / r) / r,  ta = -i / k,  tb = -1 / k^2  (host constants)
  cplx tas, tbs, tap, tbp;
  cplx g2;              // (kp / ks)^2   (kernels.py:75)
  double ks_abs;        // |ks| : |z_s| = |ks| r decides the series branch
  double sw;            // series below |z_s| < sw (reference: 0.35, kernels.py:36)
  double ratio;         // (lam + 2 mu) / mu        (kernels.py:328)
  double inv4pimu;      // 1 / (4 pi mu)
  double inv4pi;        // 1 / (4 pi)
};

// Static (Kelvin) constants, kernels.py:141-152.
struct StaticConst {
  double g2;            // mu / (lam + 2 mu)
  double ratio, inv4pimu, inv4pi;
};

// Real series coefficients (w = -i z):  phi-S a_n, phi-P b_n, psi c_n and
// the (n-1)-weighted derivative variants.  kernels.py:40-53.
struct SeriesCoef {
  double a[EWB_SERIES_TERMS], da[EWB_SERIES_TERMS];
  double b[EWB_SERIES_TERMS], db[EWB_SERIES_TERMS];
  double c[EWB_SERIES_TERMS], dc[EWB_SERIES_TERMS];
};

// Whole-program compilation (no -rdc): each translation unit that evaluates
// the series owns a copy and uploads it once with upload_series().
static __constant__ SeriesCoef c_series;

inline SeriesCoef make_series_host() {
  SeriesCoef s;
  double fact[EWB_SERIES_TERMS + 3];
  fact[0] = 1.0;
  for (int k = 1; k < EWB_SERIES_TERMS + 3; ++k) fact[k] = fact[k - 1] * k;
  for (int n = 0; n < EWB_SERIES_TERMS; ++n) {
    double i0 = 1.0 / fact[n], i1 = 1.0 / fact[n + 1], i2 = 1.0 / fact[n + 2];
    s.a[n] = i0 - i1 + i2;             // phi, S wave
    s.b[n] = i1 - i2;                  // phi, P wave (sign folded, kernels.py:48)
    s.c[n] = i0 - 3.0 * i1 + 3.0 * i2; // psi
    s.da[n] = (n - 1) * s.a[n];
    s.db[n] = (n - 1) * s.b[n];
    s.dc[n] = (n - 1) * s.c[n];
  }
  return s;
}

static inline cudaError_t upload_series(cudaStream_t st) {
  static bool done = false;
  if (done) return cudaSuccess;
  SeriesCoef s = make_series_host();
  cudaError_t e = cudaMemcpyToSymbolAsync(c_series, &s, sizeof(s), 0, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) done = true;
  return e;
}

// Shared-memory loads the compiler may not hoist: the per-member constants
// are read where they are used instead of occupying ~28 registers across
// the quadrature loop (a runtime frequency index cannot use constant-bank
// operands the way the single-frequency kernels do).
__device__ __forceinline__ double lds_d(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
// (FreqConst is 8-byte aligned with a 152-byte stride: two scalar loads)
__device__ __forceinline__ cplx lds_c(const cplx* p) { return {lds_d(&p->re), lds_d(&p->im)}; }

// a 16-byte aligned complex in one 128-bit load
__device__ __forceinline__ cplx lds_c16(const cplx* p) {
  cplx v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.re), "=d"(v.im)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// FP64 literals of the hot loops as constant-bank operands: a 64-bit
// immediate is not encodable in DFMA/DMUL/DADD, so a literal costs two UMOV
// per use in an unrolled loop (measured: 5.7 % of k_far_multi's issued
// instructions); a __constant__ value is read straight from the constant bank.
struct NumConst {
  double two, three, four, nine, far_sw, series_sw, six, fifteen, half;
};
#ifdef EWB_STRICT_SWITCH
static __constant__ NumConst c_num = {2.0, 3.0, 4.0, 9.0, 0.35, 0.35, 6.0, 15.0, 0.5};
#else
static __constant__ NumConst c_num = {2.0, 3.0, 4.0, 9.0, 0.1, 0.35, 6.0, 15.0, 0.5};  // far_sw = kFarSwitch
#endif

// Four radial brackets  phi*r, psi*r, dphi/dr*r^2, dpsi/dr*r^2.
struct Brackets {
  cplx f0, f1, f2, f3;
};

// Closed form (kernels.py:102-119), factored:
//   t = -i/z - 1/z^2,   E = e^{-iz}, F = E t, G = E (-i z)  (P terms carry g2)
//   f0 = Es + Fs - Fp
//   f1 = Es + 3Fs - Ep - 3Fp
//   f2 = Gs - 2Es - 3Fs + Ep + 3Fp
//   f3 = Gs - 4Es - 9Fs - Gp + 4Ep + 9Fp
//
// brackets_phase takes the two phase factors Es = e^{-i z_s}, ep = e^{-i z_p}
// from the caller (the multi-frequency kernels step them across an
// equispaced frequency batch instead of calling exp/sincos per frequency).
__device__ __forceinline__ Brackets brackets_phase(const FreqConst& fc, double r, double ir,
                                                   cplx Es, cplx ep) {
  double zs_re = fc.ks.re * r, zs_im = fc.ks.im * r;
  double zp_re = fc.kp.re * r, zp_im = fc.kp.im * r;
  cplx Ep = fc.g2 * ep;
  const double ir2 = ir * ir;
  const cplx ts = t_closed2(fc.tas, fc.tbs, ir, ir2), tp = t_closed2(fc.tap, fc.tbp, ir, ir2);
  cplx Fs = Es * ts, Fp = Ep * tp;
  cplx Gs = Es * cplx{zs_im, -zs_re};
  cplx Gp = Ep * cplx{zp_im, -zp_re};
  Brackets o;
  o.f0 = Es + Fs - Fp;
  o.f1 = Es + c_num.three * (Fs - Fp) - Ep;
  o.f2 = Gs - c_num.two * Es + Ep + c_num.three * (Fp - Fs);
  o.f3 = Gs - Gp + c_num.four * (Ep - Es) + c_num.nine * (Fp - Fs);
  return o;
}

// ---------------------------------------------------------------------
// sin/cos and exp for the kernel phases e^{-i z} (kernels.py:103-104).
// libdevice's versions materialise their polynomial coefficients as
// immediates (two UMOV per constant per call: 13 % of the matrix-free
// kernel's issued instructions, ncu r02) and carry the large-argument
// reduction inline.  Here: Cody-Waite reduction by pi/2 in three FMA steps,
// the fdlibm minimax kernels for sin and cos on [-pi/4, pi/4] (< 2^-58),
// exp by 2^k e^r with |r| <= ln2/2 and a degree-13 Taylor polynomial
// (truncation 4e-18); every coefficient is a constant-bank operand of its
// DFMA.  Accuracy ~1 ulp (checked against libm over 2e6 arguments,
// tests/test_gpu_assembly.py), far inside the 1e-10 parity bar.  Arguments
// beyond |x| = 1e5 (never reached by a BEM phase) take libdevice's sincos.
// ---------------------------------------------------------------------
struct MathConst {
  double two_over_pi, pio2_1, pio2_2, pio2_3, magic, sincos_big, half;
  double s[6], c[6];
  double log2e, ln2_hi, ln2_lo, exp_lo, exp_hi;
  double e[14];   // 1/13!, 1/12!, ..., 1/1!, 1/0!
  double delta_max;   // |t| bound of exp_small
};
static __constant__ MathConst c_math = {
    6.36619772367581382433e-01,  1.57079632679489655800e+00, 6.12323399573676603587e-17,
    -1.49738490485916983520e-33, 6755399441055744.0,          1.0e5, 0.5,
    {-1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
     2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10},
    {4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
     -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11},
    1.44269504088896338700e+00, 6.93147180559945286227e-01, 2.31904681384629955842e-17,
    -746.0, 710.0,
    {1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
     1.0 / 362880.0, 1.0 / 40320.0, 1.0 / 5040.0, 1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0,
     1.0 / 6.0, 0.5, 1.0, 1.0},
    0.0625};

static __device__ __noinline__ void sincos_large(double x, double* s, double* c) { sincos(x, s, c); }

__device__ __forceinline__ double flip_sign(double v, int neg) {
  return __hiloint2double(__double2hiint(v) ^ (neg << 31), __double2loint(v));
}

__device__ __forceinline__ void fast_sincos(double x, double* sp, double* cp) {
  if (!(fabs(x) <= c_math.sincos_big)) {   // also NaN / inf
    sincos_large(x, sp, cp);
    return;
  }
  const double t = fma(x, c_math.two_over_pi, c_math.magic);
  const double kd = t - c_math.magic;
  const int q = __double2loint(t);
  double r = fma(-kd, c_math.pio2_1, x);
  r = fma(-kd, c_math.pio2_2, r);
  r = fma(-kd, c_math.pio2_3, r);
  const double z = r * r;
  double ps = fma(z, c_math.s[5], c_math.s[4]);
  ps = fma(z, ps, c_math.s[3]);
  ps = fma(z, ps, c_math.s[2]);
  ps = fma(z, ps, c_math.s[1]);
  ps = fma(z, ps, c_math.s[0]);
  const double sn = fma(r * z, ps, r);
  double pc = fma(z, c_math.c[5], c_math.c[4]);
  pc = fma(z, pc, c_math.c[3]);
  pc = fma(z, pc, c_math.c[2]);
  pc = fma(z, pc, c_math.c[1]);
  pc = fma(z, pc, c_math.c[0]);
  const double cs = c_math.e[13] + fma(z * z, pc, -c_math.half * z);   // 1 - (z/2 - z^2 P)
  const bool swap = q & 1;
  *sp = flip_sign(swap ? cs : sn, (q >> 1) & 1);
  *cp = flip_sign(swap ? sn : cs, ((q + 1) >> 1) & 1);
}

__device__ __forceinline__ double fast_exp(double x) {
  double xd = x < c_math.exp_lo ? c_math.exp_lo : x;   // NaN passes through
  xd = xd > c_math.exp_hi ? c_math.exp_hi : xd;
  const double t = fma(xd, c_math.log2e, c_math.magic);
  const double kd = t - c_math.magic;
  const int k = __double2loint(t);
  double r = fma(-kd, c_math.ln2_hi, xd);
  r = fma(-kd, c_math.ln2_lo, r);
  double p = fma(c_math.e[0], r, c_math.e[1]);
#pragma unroll
  for (int i = 2; i < 14; ++i) p = fma(p, r, c_math.e[i]);
  const int k1 = k >> 1, k2 = k - k1;
  p = p * __hiloint2double((k1 + 1023) << 20, 0);
  return p * __hiloint2double((k2 + 1023) << 20, 0);
}

// N arguments in lockstep: the same arithmetic as fast_sincos / fast_exp per
// argument (bit-identical results), written so that each polynomial
// coefficient feeds N independent FMA chains back to back — one constant
// fetch instead of N, and N-way instruction-level parallelism on the
// dependent Horner steps.
template <int N>
__device__ __forceinline__ void fast_sincos_n(const double (&x)[N], double (&sp)[N],
                                              double (&cp)[N]) {
  bool big = false;
#pragma unroll
  for (int i = 0; i < N; ++i) big |= !(fabs(x[i]) <= c_math.sincos_big);
  if (big) {
#pragma unroll
    for (int i = 0; i < N; ++i) sincos_large(x[i], &sp[i], &cp[i]);
    return;
  }
  double r[N], z[N], ps[N], pc[N];
  int q[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double t = fma(x[i], c_math.two_over_pi, c_math.magic);
    const double kd = t - c_math.magic;
    q[i] = __double2loint(t);
    r[i] = fma(-kd, c_math.pio2_1, x[i]);
    r[i] = fma(-kd, c_math.pio2_2, r[i]);
    r[i] = fma(-kd, c_math.pio2_3, r[i]);
    z[i] = r[i] * r[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) ps[i] = fma(z[i], c_math.s[5], c_math.s[4]);
#pragma unroll
  for (int m = 3; m >= 0; --m)
#pragma unroll
    for (int i = 0; i < N; ++i) ps[i] = fma(z[i], ps[i], c_math.s[m]);
#pragma unroll
  for (int i = 0; i < N; ++i) pc[i] = fma(z[i], c_math.c[5], c_math.c[4]);
#pragma unroll
  for (int m = 3; m >= 0; --m)
#pragma unroll
    for (int i = 0; i < N; ++i) pc[i] = fma(z[i], pc[i], c_math.c[m]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double sn = fma(r[i] * z[i], ps[i], r[i]);
    const double cs = c_math.e[13] + fma(z[i] * z[i], pc[i], -c_math.half * z[i]);
    const bool swap = q[i] & 1;
    sp[i] = flip_sign(swap ? cs : sn, (q[i] >> 1) & 1);
    cp[i] = flip_sign(swap ? sn : cs, ((q[i] + 1) >> 1) & 1);
  }
}

template <int N>
__device__ __forceinline__ void fast_exp_n(const double (&x)[N], double (&e)[N]) {
  double r[N], p[N];
  int k[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double xd = x[i] < c_math.exp_lo ? c_math.exp_lo : x[i];   // NaN passes through
    xd = xd > c_math.exp_hi ? c_math.exp_hi : xd;
    const double t = fma(xd, c_math.log2e, c_math.magic);
    const double kd = t - c_math.magic;
    k[i] = __double2loint(t);
    r[i] = fma(-kd, c_math.ln2_hi, xd);
    r[i] = fma(-kd, c_math.ln2_lo, r[i]);
    p[i] = fma(c_math.e[0], r[i], c_math.e[1]);
  }
#pragma unroll
  for (int m = 2; m < 14; ++m)
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = fma(p[i], r[i], c_math.e[m]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const int k1 = k[i] >> 1, k2 = k[i] - k1;
    e[i] = (p[i] * __hiloint2double((k1 + 1023) << 20, 0)) * __hiloint2double((k2 + 1023) << 20, 0);
  }
}

// The S and P phase factors of NP points: E_s = e^{-i k_s r}, e_p = e^{-i k_p r}.
template <int NP>
__device__ __forceinline__ void phase_factors_n(cplx ks, cplx kp, const double (&r)[NP],
                                                cplx (&Es)[NP], cplx (&ep)[NP]) {
  double xa[2 * NP], xe[2 * NP], s[2 * NP], c[2 * NP], m[2 * NP];
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    xa[2 * i] = ks.re * r[i];
    xa[2 * i + 1] = kp.re * r[i];
    xe[2 * i] = ks.im * r[i];
    xe[2 * i + 1] = kp.im * r[i];
  }
  fast_sincos_n<2 * NP>(xa, s, c);
  fast_exp_n<2 * NP>(xe, m);
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    Es[i] = {m[2 * i] * c[2 * i], -m[2 * i] * s[2 * i]};
    ep[i] = {m[2 * i + 1] * c[2 * i + 1], -m[2 * i + 1] * s[2 * i + 1]};
  }
}

// e^{-i k r} = e^{Im(k) r} (cos(Re(k) r) - i sin(Re(k) r))
__device__ __forceinline__ cplx phase_factor(cplx k, double r) {
  double s, c;
  fast_sincos(k.re * r, &s, &c);
  double m = fast_exp(k.im * r);
  return {m * c, -m * s};
}

// e^t for |t| <= c_math.delta_max = 2^-4: degree-8 Taylor (truncation
// t^9 / 9! <= 4e-17).  The damping factors e^{Im(k) r} of the second and
// third quadrature point of a far pair follow from the first point's by
// e^{Im(k) r_q} = e^{Im(k) r_0} e^{Im(k) (r_q - r_0)} whenever
// |Im(k_s)| d_j <= 2^-4 (|r_q - r_0| <= d_j, the element's longest edge;
// |Im(k_p)| < |Im(k_s)|): 11 FP64 instructions instead of 21 per factor,
// ~1 ulp apart from fast_exp.  Measured on the cfg5 application (degree 6,
// bound 2^-6): K = 1 402.8 -> 377.3 ms, K = 5 638.7 -> 616.7 ms.
__device__ __forceinline__ double exp_small(double t) {
  double p = fma(c_math.e[5], t, c_math.e[6]);   // 1/8! t + 1/7!
  p = fma(p, t, c_math.e[7]);
  p = fma(p, t, c_math.e[8]);
  p = fma(p, t, c_math.e[9]);
  p = fma(p, t, c_math.e[10]);
  p = fma(p, t, c_math.e[11]);
  p = fma(p, t, c_math.e[12]);
  return fma(p, t, c_math.e[13]);
}

// Damping factors of one point of a pair: the full exponentials, or — DELTA,
// from the pair's first point (r0, ms0, mp0) — the small-argument update.
template <bool DELTA>
__device__ __forceinline__ void damping_factors(const FreqConst& fc, double r, double r0,
                                                double ms0, double mp0, double& ms, double& mp) {
  if (DELTA) {
    const double t = r - r0;
    ms = ms0 * exp_small(fc.ks.im * t);
    mp = mp0 * exp_small(fc.kp.im * t);
  } else {
    const double xe[2] = {fc.ks.im * r, fc.kp.im * r};
    double m[2];
    fast_exp_n<2>(xe, m);
    ms = m[0];
    mp = m[1];
  }
}

// Closed-form brackets with the damping factors given (damping_factors).
__device__ __forceinline__ Brackets brackets_closed_m(const FreqConst& fc, double r, double ir,
                                                      double ms, double mp) {
  const double xa[2] = {fc.ks.re * r, fc.kp.re * r};
  double s[2], c[2];
  fast_sincos_n<2>(xa, s, c);
  return brackets_phase(fc, r, ir, cplx{ms * c[0], -ms * s[0]}, cplx{mp * c[1], -mp * s[1]});
}

__device__ __forceinline__ Brackets brackets_closed(const FreqConst& fc, double r, double ir) {
  // the S and P phases in lockstep (shared coefficient fetches, 2-way ILP)
  const double rr[1] = {r};
  cplx Es[1], ep[1];
  phase_factors_n<1>(fc.ks, fc.kp, rr, Es, ep);
  return brackets_phase(fc, r, ir, Es[0], ep[0]);
}

// Horner, real coefficients, complex argument: p(w) = sum_n c_n w^n.
__device__ __forceinline__ void horner4(cplx w, const double* c0, const double* c1,
                                        const double* c2, const double* c3, cplx* out) {
  cplx p0 = {c0[EWB_SERIES_TERMS - 1], 0.0}, p1 = {c1[EWB_SERIES_TERMS - 1], 0.0};
  cplx p2 = {c2[EWB_SERIES_TERMS - 1], 0.0}, p3 = {c3[EWB_SERIES_TERMS - 1], 0.0};
#pragma unroll
  for (int n = EWB_SERIES_TERMS - 2; n >= 0; --n) {
    p0 = {fma(p0.re, w.re, fma(-p0.im, w.im, c0[n])), fma(p0.re, w.im, p0.im * w.re)};
    p1 = {fma(p1.re, w.re, fma(-p1.im, w.im, c1[n])), fma(p1.re, w.im, p1.im * w.re)};
    p2 = {fma(p2.re, w.re, fma(-p2.im, w.im, c2[n])), fma(p2.re, w.im, p2.im * w.re)};
    p3 = {fma(p3.re, w.re, fma(-p3.im, w.im, c3[n])), fma(p3.re, w.im, p3.im * w.re)};
  }
  out[0] = p0; out[1] = p1; out[2] = p2; out[3] = p3;
}

// Power series (kernels.py:122-138) with the (-i)^n folded into w = -i z:
//   f0 = A(ws) + g2 B(wp)      f1 = C(ws) - g2 C(wp)
//   f2 = A'(ws) + g2 B'(wp)    f3 = C'(ws) - g2 C'(wp)
__device__ __forceinline__ Brackets brackets_series_k(cplx ks, cplx kp, cplx g2, double r) {
  cplx ws = {ks.im * r, -ks.re * r};
  cplx wp = {kp.im * r, -kp.re * r};
  cplx s[4], p[4];
  horner4(ws, c_series.a, c_series.da, c_series.c, c_series.dc, s);
  horner4(wp, c_series.b, c_series.db, c_series.c, c_series.dc, p);
  Brackets o;
  o.f0 = s[0] + g2 * p[0];
  o.f2 = s[1] + g2 * p[1];
  o.f1 = s[2] - g2 * p[2];
  o.f3 = s[3] - g2 * p[3];
  return o;
}
__device__ __forceinline__ Brackets brackets_series(const FreqConst& fc, double r) {
  return brackets_series_k(fc.ks, fc.kp, fc.g2, r);
}

// Power-sum form of the same series, NT terms: one complex power per term
// shared by the four real-coefficient sums (fewer FP64 ops than Horner).
template <int NT>
__device__ __forceinline__ void series4_pow(cplx w, const double* c0, const double* c1,
                                            const double* c2, const double* c3, cplx* out) {
  cplx s0 = {c0[0], 0.0}, s1 = {c1[0], 0.0}, s2 = {c2[0], 0.0}, s3 = {c3[0], 0.0};
  cplx p = w;
#pragma unroll
  for (int n = 1; n < NT; ++n) {
    axpy(s0, c0[n], p);
    axpy(s1, c1[n], p);
    axpy(s2, c2[n], p);
    axpy(s3, c3[n], p);
    if (n + 1 < NT) p = p * w;
  }
  out[0] = s0; out[1] = s1; out[2] = s2; out[3] = s3;
}

template <int NT>
__device__ __forceinline__ Brackets brackets_series_n(const FreqConst& fc, double r) {
  static_assert(NT <= EWB_SERIES_TERMS, "series table too short");
  cplx ws = {fc.ks.im * r, -fc.ks.re * r};
  cplx wp = {fc.kp.im * r, -fc.kp.re * r};
  cplx s[4], p[4];
  series4_pow<NT>(ws, c_series.a, c_series.da, c_series.c, c_series.dc, s);
  series4_pow<NT>(wp, c_series.b, c_series.db, c_series.c, c_series.dc, p);
  Brackets o;
  o.f0 = s[0] + fc.g2 * p[0];
  o.f2 = s[1] + fc.g2 * p[1];
  o.f1 = s[2] - fc.g2 * p[2];
  o.f3 = s[3] - fc.g2 * p[3];
  return o;
}

// The series branch out of line, for kernels whose series points are rare
// (far pairs switch at |k_s r| < 0.1): its register peak then does not
// shape the hot closed-form loop.
// (only the three constants the series reads travel by value: the whole
// FreqConst would be passed through local memory)
static __device__ __noinline__ Brackets brackets_series_cold3(cplx ks, cplx kp, cplx g2, double r) {
  return brackets_series_k(ks, kp, g2, r);
}
__device__ __forceinline__ Brackets brackets_series_cold(const FreqConst& fc, double r) {
  return brackets_series_cold3(fc.ks, fc.kp, fc.g2, r);
}

// Strict per-point switch exactly as kernels.py:79-95 (|k_s r| < 0.35).
// The far/mid (and matrix-free far) kernels run with fc.sw = kFarSwitch:
// between 0.1 and 0.35 the closed form agrees with the series to <= 2e-13
// relative (measured against the reference's 24-term series, DESIGN.md
// §4), and warps of far pairs then never execute both branches.  Near and
// self pairs keep the reference's 0.35.  -DEWB_STRICT_SWITCH: 0.35 everywhere.
#ifdef EWB_STRICT_SWITCH
constexpr double kFarSwitch = kSeriesSwitch;
#else
constexpr double kFarSwitch = 0.1;
#endif

__device__ __forceinline__ Brackets brackets_strict(const FreqConst& fc, double r, double ir) {
#ifdef EWB_SERIES_POW
  if (fc.ks_abs * r < fc.sw) return brackets_series_n<16>(fc, r);
#else
  if (fc.ks_abs * r < fc.sw) return brackets_series(fc, r);
#endif
  return brackets_closed(fc, r, ir);
}

// Warp-uniform evaluation.  When every active lane is on the same side of
// the reference's switch the result is the reference's branch.  When a warp
// mixes both, one evaluation valid for all its lanes is used instead of
// executing both branches serially:
//   series, 20 terms, if every |z_s| < 1   (truncation < 1e-17 relative)
//   closed form      if every |z_s| > 0.05 (cancellation <= eps/|z|^2 ~ 1e-13)
// Both agree with the reference's choice far inside the 1e-10 parity bar
// (the reference's own seam test allows 1e-12, test_kernels.py:83-98).
// Build with -DEWB_STRICT_SWITCH for the per-point reference switch.
__device__ __forceinline__ Brackets brackets_dynamic(const FreqConst& fc, double r, double ir) {
#if defined(EWB_TIMING_CLOSED_ONLY)
  return brackets_closed(fc, r, ir);   // timing experiments only: not parity-valid
#elif !defined(EWB_UNIFORM_SWITCH)
  return brackets_strict(fc, r, ir);
#else
  const unsigned mask = __activemask();
  const double za = fc.ks_abs * r;
  const bool ser = za < kSeriesSwitch;
  if (__all_sync(mask, ser)) return brackets_series_n<16>(fc, r);
  if (__all_sync(mask, !ser)) return brackets_closed(fc, r, ir);
  if (__all_sync(mask, za < 1.0)) return brackets_series_n<20>(fc, r);
  if (__all_sync(mask, za > 0.05)) return brackets_closed(fc, r, ir);
  return brackets_strict(fc, r, ir);
#endif
}

// ---------------------------------------------------------------------
// Contraction accumulators (kernels.py:327-357).  With w the quadrature
// weight (rule weight x area) and d = (y - x)/r, dn = d.n_j:
//   su   = sum w phi                    U_ij = (su d_ij - P_ij)/(4 pi mu)
//   P_ij = sum w psi d_i d_j
//   sa   = sum w a dn                   T_ij = (sa d_ij + n_i va_j + B_ij
//   va_j = sum w a d_j                           + vc_i n_j)/(4 pi)
//   B_ij = sum w b dn d_i d_j
//   vc_i = sum w c d_i
// Symmetric 3x3 stored as xx, yy, zz, xy, xz, yz.
// ---------------------------------------------------------------------
template <typename S>
struct Acc {
  S su, P[6], sa, va[3], B[6], vc[3];
};

__device__ __forceinline__ void zero(double& v) { v = 0.0; }
__device__ __forceinline__ void zero(cplx& v) { v = {0.0, 0.0}; }

template <typename S>
__device__ __forceinline__ void acc_zero(Acc<S>& A) {
  zero(A.su); zero(A.sa);
#pragma unroll
  for (int k = 0; k < 6; ++k) { zero(A.P[k]); zero(A.B[k]); }
#pragma unroll
  for (int k = 0; k < 3; ++k) { zero(A.va[k]); zero(A.vc[k]); }
}

__device__ __forceinline__ void madd(double& acc, double s, double v) { acc = fma(s, v, acc); }
__device__ __forceinline__ void madd(cplx& acc, double s, cplx v) { axpy(acc, s, v); }

// Accumulate one quadrature point given the weighted scalars
//   Phi = w phi, Psi = w psi, Aw = w a, Bw = w b dn, Cw = w c.
template <typename S>
__device__ __forceinline__ void acc_point(Acc<S>& A, S Phi, S Psi, S Aw, S Bw, S Cw,
                                          double dx, double dy, double dz, double dn) {
  double dd[6] = {dx * dx, dy * dy, dz * dz, dx * dy, dx * dz, dy * dz};
  A.su = A.su + Phi;
#pragma unroll
  for (int k = 0; k < 6; ++k) { madd(A.P[k], dd[k], Psi); madd(A.B[k], dd[k], Bw); }
  madd(A.sa, dn, Aw);
  madd(A.va[0], dx, Aw); madd(A.va[1], dy, Aw); madd(A.va[2], dz, Aw);
  madd(A.vc[0], dx, Cw); madd(A.vc[1], dy, Cw); madd(A.vc[2], dz, Cw);
}

__device__ __forceinline__ void point_dynamic(Acc<cplx>& A, const FreqConst& fc, double r,
                                              double ir, double dx, double dy, double dz,
                                              double dn, double w) {
  Brackets f = brackets_dynamic(fc, r, ir);
  double wr = w * ir, wr2 = wr * ir;
  cplx Phi = wr * f.f0;
  cplx Psi = wr * f.f1;
  cplx Aw = wr2 * (f.f2 - f.f1);
  cplx Bw = (2.0 * wr2 * dn) * (2.0 * f.f1 - f.f3);
  cplx dd = f.f2 - f.f3;
  cplx Cw = wr2 * (fc.ratio * (dd - 2.0 * f.f1) - 2.0 * (dd - f.f1));
  acc_point(A, Phi, Psi, Aw, Bw, Cw, dx, dy, dz, dn);
}

// The five weighted scalars of one closed-form point straight from the
// phase factors.  With D = E_s t_s - E_p t_p (t = -i/z - 1/z^2, the 1/z
// terms of kernels.py:105-119, from t_closed), G_s = -i z_s E_s and G_p = -i z_p E_p, the
// brackets are linear in (E_s, E_p, D, G_s, G_p):
//   f0 = E_s + D,  f1 = E_s - E_p + 3D,  f2 = G_s - 2E_s + E_p - 3D,
//   f3 = G_s - G_p - 4E_s + 4E_p - 9D,
// and so are the weighted scalars of kernels.py:330-333 (wu, wt carry the
// rule weight, 1/r and 1/(4 pi mu) or 1/(4 pi r^2); wb = 2 wt dn):
//   Phi = wu f0,  Psi = wu f1,  Aw = wt (f2 - f1) = wt (G_s - 3E_s + 2E_p - 6D),
//   Bw = wb (2f1 - f3) = wb (6(E_s - E_p) + 15D + G_p - G_s),
//   Cw = wt (ratio (f2 - f3 - 2f1) - 2 (f2 - f3 - f1))
//      = wt ((ratio - 2) G_p + (4 - ratio) E_p - 2E_s - 6D).
// Same values as the factored brackets (brackets_closed with the phase
// factors given) + the scalar formulas, rounding apart, with ~35 % fewer
// FP64 instructions per point (k_far_multi; the cfg3 pair-kernel product
// uses it through weights_closed: +1.8 % pair-evals/s).
struct Weighted5 {
  cplx Phi, Psi, Aw, Bw, Cw;
};
__device__ __forceinline__ Weighted5 weights_phase(cplx ks, cplx kp, cplx ts, cplx tp, double r,
                                                   cplx Es, cplx Ep, double wu, double wt,
                                                   double wb, double cr2, double c4r) {
  cplx D = Es * ts;
  D.re = fma(-Ep.re, tp.re, fma(Ep.im, tp.im, D.re));
  D.im = fma(-Ep.re, tp.im, fma(-Ep.im, tp.re, D.im));
  const cplx Gs = Es * cplx{ks.im * r, -ks.re * r};
  const cplx Gp = Ep * cplx{kp.im * r, -kp.re * r};
  const cplx dE = Es - Ep;
  Weighted5 w;
  w.Phi = wu * (Es + D);
  w.Psi = {wu * fma(c_num.three, D.re, dE.re), wu * fma(c_num.three, D.im, dE.im)};
  w.Aw = {wt * fma(-c_num.six, D.re, fma(c_num.two, Ep.re, fma(-c_num.three, Es.re, Gs.re))),
          wt * fma(-c_num.six, D.im, fma(c_num.two, Ep.im, fma(-c_num.three, Es.im, Gs.im)))};
  w.Bw = {wb * fma(c_num.fifteen, D.re, fma(c_num.six, dE.re, Gp.re - Gs.re)),
          wb * fma(c_num.fifteen, D.im, fma(c_num.six, dE.im, Gp.im - Gs.im))};
  w.Cw = {wt * fma(-c_num.six, D.re, fma(-c_num.two, Es.re, fma(c4r, Ep.re, cr2 * Gp.re))),
          wt * fma(-c_num.six, D.im, fma(-c_num.two, Es.im, fma(c4r, Ep.im, cr2 * Gp.im)))};
  return w;
}

// The same from (fc, r): the phase factors evaluated here.
__device__ __forceinline__ Weighted5 weights_closed(const FreqConst& fc, double r, double ir,
                                                   double wu, double wt, double wb) {
  const cplx Es = phase_factor(fc.ks, r);
  const cplx Ep = fc.g2 * phase_factor(fc.kp, r);
  const double ir2 = ir * ir;
  return weights_phase(fc.ks, fc.kp, t_closed2(fc.tas, fc.tbs, ir, ir2),
                       t_closed2(fc.tap, fc.tbp, ir, ir2), r, Es, Ep, wu, wt, wb,
                       fc.ratio - c_num.two, c_num.four - fc.ratio);
}

// Weighted scalars of the series branch (kernels.py:330-333) from brackets.
__device__ __forceinline__ Weighted5 weights_brackets(const Brackets& f, double ratio, double wu,
                                                      double wt, double wb) {
  Weighted5 w;
  w.Phi = wu * f.f0;
  w.Psi = wu * f.f1;
  w.Aw = wt * (f.f2 - f.f1);
  w.Bw = wb * (c_num.two * f.f1 - f.f3);
  const cplx dd = f.f2 - f.f3;
  w.Cw = wt * (ratio * (dd - c_num.two * f.f1) - c_num.two * (dd - f.f1));
  return w;
}

// One dynamic point with the block constants folded into the weights:
// wu = w / (4 pi mu r), wt = w / (4 pi r^2); series below |k_s r| < sw taken
// out of line.  The accumulators then hold U and T contributions directly.
// SER = false: the caller proved |k_s| r >= sw for every point it passes
// (no out-of-line series call in the kernel, fewer live registers).
template <bool SER = true>
__device__ __forceinline__ void point_dynamic_scaled(Acc<cplx>& A, const FreqConst& fc,
                                                     double sw, double r, double ir, double dx,
                                                     double dy, double dz, double dn, double wu,
                                                     double wt) {
  const Brackets f =
      SER && fc.ks_abs * r < sw ? brackets_series_cold(fc, r) : brackets_closed(fc, r, ir);
  const cplx Phi = wu * f.f0;
  const cplx Psi = wu * f.f1;
  const cplx Aw = wt * (f.f2 - f.f1);
  const cplx Bw = (c_num.two * wt * dn) * (c_num.two * f.f1 - f.f3);
  const cplx dd = f.f2 - f.f3;
  const cplx Cw = wt * (fc.ratio * (dd - c_num.two * f.f1) - c_num.two * (dd - f.f1));
  acc_point(A, Phi, Psi, Aw, Bw, Cw, dx, dy, dz, dn);
}

// The T product of one point from its four brackets (see point_apply_T).
__device__ __forceinline__ void point_apply_T_br(cplx y[3], const Brackets& f, double ratio,
                                                 double dx, double dy, double dz, double dn,
                                                 double wt, const cplx v[3], cplx nv, double nx,
                                                 double ny, double nz) {
  const cplx Aw = wt * (f.f2 - f.f1);
  const cplx Bw = (c_num.two * wt * dn) * (c_num.two * f.f1 - f.f3);
  const cplx dd = f.f2 - f.f3;
  const cplx Cw = wt * (ratio * (dd - c_num.two * f.f1) - c_num.two * (dd - f.f1));
  cplx sv = dx * v[0];
  axpy(sv, dy, v[1]);
  axpy(sv, dz, v[2]);
  const cplx e = dn * Aw, h = Aw * sv;
  cplx gg = Bw * sv;
  cfma(gg, Cw, nv);
  const double n[3] = {nx, ny, nz}, d[3] = {dx, dy, dz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cfma(y[a], e, v[a]);
    axpy(y[a], n[a], h);
    axpy(y[a], d[a], gg);
  }
}

// One dynamic point applied straight to a vector (T only, one vector: the
// matrix-free GMRES product).  With s = d.v and nv = n.v the point's share of
// T v (kernels.py:345-356) is
//   (T v)_a += e v_a + n_a h + d_a g,   e = Aw dn, h = Aw s, g = Bw s + Cw nv
// (~44 DP instead of 40 accumulator updates plus a third of a block apply),
// and no 20-word accumulator is live: far fewer registers per thread.
template <bool SER = true>
__device__ __forceinline__ void point_apply_T(cplx y[3], const FreqConst& fc, double sw, double r,
                                              double ir, double dx, double dy, double dz,
                                              double dn, double wt, const cplx v[3], cplx nv,
                                              double nx, double ny, double nz) {
  // (the linear-basis weights measured 1-4 % slower here at low frequency:
  // this product keeps the bracket form)
  const Brackets f =
      SER && fc.ks_abs * r < sw ? brackets_series_cold(fc, r) : brackets_closed(fc, r, ir);
  point_apply_T_br(y, f, fc.ratio, dx, dy, dz, dn, wt, v, nv, nx, ny, nz);
}

// The T product of one point from its weighted scalars Aw, Bw (2 dn folded
// in), Cw (see point_apply_T).
__device__ __forceinline__ void point_apply_T_w(cplx y[3], cplx Aw, cplx Bw, cplx Cw, double dx,
                                                double dy, double dz, double dn, const cplx v[3],
                                                cplx nv, double nx, double ny, double nz) {
  cplx sv = dx * v[0];
  axpy(sv, dy, v[1]);
  axpy(sv, dz, v[2]);
  const cplx e = dn * Aw, h = Aw * sv;
  cplx gg = Bw * sv;
  cfma(gg, Cw, nv);
  const double n[3] = {nx, ny, nz}, d[3] = {dx, dy, dz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cfma(y[a], e, v[a]);
    axpy(y[a], n[a], h);
    axpy(y[a], d[a], gg);
  }
}

// The same with the point's damping factors supplied by the caller.
template <bool SER = true>
__device__ __forceinline__ void point_apply_T_m(cplx y[3], const FreqConst& fc, double sw, double r,
                                                double ir, double dx, double dy, double dz,
                                                double dn, double wt, const cplx v[3], cplx nv,
                                                double nx, double ny, double nz, double ms,
                                                double mp) {
#ifndef EWB_MF_BRACKETS
  if (!(SER && fc.ks_abs * r < sw)) {
    // weighted scalars straight from the linear basis (weights_phase): with
    // the damping factors supplied, measured 1.6 % (low frequency) to 3.6 %
    // (omega = 8) faster on the cfg5 application than the bracket form below
    const double xa[2] = {fc.ks.re * r, fc.kp.re * r};
    double s[2], c[2];
    fast_sincos_n<2>(xa, s, c);
    const cplx Es = {ms * c[0], -ms * s[0]};
#ifdef EWB_MF_G2_COMPLEX
    const cplx Ep = fc.g2 * cplx{mp * c[1], -mp * s[1]};
#else
    // g2 = (k_p / k_s)^2 = (c_s / c_p)^2 is real for the real materials of
    // the reference (its complex value carries ~1e-17 of rounding in the
    // imaginary part): folded into the damping factor as a real scalar
    const double mpg = mp * fc.g2.re;
    const cplx Ep = {mpg * c[1], -mpg * s[1]};
#endif
    const double ir2 = ir * ir;
    const Weighted5 w = weights_phase(fc.ks, fc.kp, t_closed2(fc.tas, fc.tbs, ir, ir2),
                                      t_closed2(fc.tap, fc.tbp, ir, ir2), r, Es, Ep, 0.0, wt,
                                      c_num.two * wt * dn, fc.ratio - c_num.two,
                                      c_num.four - fc.ratio);
    point_apply_T_w(y, w.Aw, w.Bw, w.Cw, dx, dy, dz, dn, v, nv, nx, ny, nz);
    return;
  }
#endif
  const Brackets f = SER && fc.ks_abs * r < sw ? brackets_series_cold(fc, r)
                                               : brackets_closed_m(fc, r, ir, ms, mp);
  point_apply_T_br(y, f, fc.ratio, dx, dy, dz, dn, wt, v, nv, nx, ny, nz);
}

template <bool SER = true>
__device__ __forceinline__ void point_dynamic_scaled_m(Acc<cplx>& A, const FreqConst& fc,
                                                       double sw, double r, double ir, double dx,
                                                       double dy, double dz, double dn, double wu,
                                                       double wt, double ms, double mp) {
#ifndef EWB_MF_ACC_BRACKETS
  // linear-basis weights as in point_apply_T_m, in the series-free instances
  // only: measured on the masked K = 5 cfg5 pass, 567 -> 556 ms at omega = 8
  // (SER = false) but 601 -> 659 ms at low frequency, where the kernel also
  // carries the series call (register pressure)
  if (!SER) {
    const double xa[2] = {fc.ks.re * r, fc.kp.re * r};
    double s[2], c[2];
    fast_sincos_n<2>(xa, s, c);
    const cplx Es = {ms * c[0], -ms * s[0]};
#ifdef EWB_MF_G2_COMPLEX
    const cplx Ep = fc.g2 * cplx{mp * c[1], -mp * s[1]};
#else
    // g2 = (k_p / k_s)^2 = (c_s / c_p)^2 is real for the real materials of
    // the reference (its complex value carries ~1e-17 of rounding in the
    // imaginary part): folded into the damping factor as a real scalar
    const double mpg = mp * fc.g2.re;
    const cplx Ep = {mpg * c[1], -mpg * s[1]};
#endif
    const double ir2 = ir * ir;
    const Weighted5 w = weights_phase(fc.ks, fc.kp, t_closed2(fc.tas, fc.tbs, ir, ir2),
                                      t_closed2(fc.tap, fc.tbp, ir, ir2), r, Es, Ep, wu, wt,
                                      c_num.two * wt * dn, fc.ratio - c_num.two,
                                      c_num.four - fc.ratio);
    acc_point(A, w.Phi, w.Psi, w.Aw, w.Bw, w.Cw, dx, dy, dz, dn);
    return;
  }
#endif
  const Brackets f = SER && fc.ks_abs * r < sw ? brackets_series_cold(fc, r)
                                               : brackets_closed_m(fc, r, ir, ms, mp);
  const cplx Phi = wu * f.f0;
  const cplx Psi = wu * f.f1;
  const cplx Aw = wt * (f.f2 - f.f1);
  const cplx Bw = (c_num.two * wt * dn) * (c_num.two * f.f1 - f.f3);
  const cplx dd = f.f2 - f.f3;
  const cplx Cw = wt * (fc.ratio * (dd - c_num.two * f.f1) - c_num.two * (dd - f.f1));
  acc_point(A, Phi, Psi, Aw, Bw, Cw, dx, dy, dz, dn);
}

// One dynamic point applied straight to one vector for both operators (the
// cfg3 fused reduction y_U = U x, y_T = T x): with s = d.x,
//   (U x)_a += Phi x_a - Psi d_a s,   (T x)_a as in point_apply_T.
__device__ __forceinline__ void point_apply_UT(cplx yu[3], cplx yt[3], const FreqConst& fc,
                                               double sw, double r, double ir, double dx,
                                               double dy, double dz, double dn, double wu,
                                               double wt, const cplx v[3], cplx nv, double nx,
                                               double ny, double nz) {
  const double wb = c_num.two * wt * dn;
  const Weighted5 w = fc.ks_abs * r < sw
                          ? weights_brackets(brackets_series_cold(fc, r), fc.ratio, wu, wt, wb)
                          : weights_closed(fc, r, ir, wu, wt, wb);
  const cplx Phi = w.Phi, Psi = w.Psi, Aw = w.Aw, Bw = w.Bw, Cw = w.Cw;
  cplx sv = dx * v[0];
  axpy(sv, dy, v[1]);
  axpy(sv, dz, v[2]);
  const cplx e = dn * Aw, h = Aw * sv, ps = Psi * sv;
  cplx gg = Bw * sv;
  cfma(gg, Cw, nv);
  const double n[3] = {nx, ny, nz}, d[3] = {dx, dy, dz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    cfma(yt[a], e, v[a]);
    axpy(yt[a], n[a], h);
    axpy(yt[a], d[a], gg);
    cfma(yu[a], Phi, v[a]);
    axpy(yu[a], -d[a], ps);
  }
}

// One static point (Kelvin), kernels.py:141-152 + 327-357.
__device__ __forceinline__ void point_static(Acc<double>& A, const StaticConst& sc, double ir,
                                             double dx, double dy, double dz, double dn,
                                             double w) {
  double ir2 = ir * ir;
  double phi = 0.5 * (1.0 + sc.g2) * ir;
  double psi = 0.5 * (sc.g2 - 1.0) * ir;
  double dphi = -0.5 * (1.0 + sc.g2) * ir2;
  double dpsi = 0.5 * (1.0 - sc.g2) * ir2;
  double psr = psi * ir;
  double a = dphi - psr;
  double b = 2.0 * (2.0 * psr - dpsi);
  double c = sc.ratio * (dphi - dpsi - 2.0 * psr) - 2.0 * (dphi - dpsi - psr);
  acc_point(A, w * phi, w * psi, w * a, w * b * dn, w * c, dx, dy, dz, dn);
}

// Finalise the 3x3 blocks: U[a][b], T[a][b] (a = load direction at x,
// b = component at y).
template <typename S>
__device__ __forceinline__ void acc_finalize(const Acc<S>& A, double nx, double ny, double nz,
                                             double inv4pimu, double inv4pi, S U[3][3],
                                             S T[3][3]) {
  const int sym[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
  double n[3] = {nx, ny, nz};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      S u = a == b ? A.su - A.P[sym[a][b]] : -A.P[sym[a][b]];
      u = inv4pimu * u;
      S t = A.B[sym[a][b]];
      madd(t, n[a], A.va[b]);
      madd(t, n[b], A.vc[a]);
      if (a == b) t = t + A.sa;
      U[a][b] = u;
      T[a][b] = inv4pi * t;
    }
  }
}

// Warp reduction of an accumulator (lane 0 ends with the total).
__device__ __forceinline__ double shfl_down(double v, int o) {
  return __shfl_down_sync(0xffffffffu, v, o);
}
__device__ __forceinline__ void warp_sum(double& v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += shfl_down(v, o);
}
__device__ __forceinline__ void warp_sum(cplx& v) { warp_sum(v.re); warp_sum(v.im); }

__device__ __forceinline__ void warp_allsum(double& v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
}
__device__ __forceinline__ void warp_allsum(cplx& v) { warp_allsum(v.re); warp_allsum(v.im); }

// Butterfly variant: every lane ends with the (bitwise identical) totals.
template <typename S>
__device__ __forceinline__ void acc_warp_allsum(Acc<S>& A) {
  warp_allsum(A.su); warp_allsum(A.sa);
#pragma unroll
  for (int k = 0; k < 6; ++k) { warp_allsum(A.P[k]); warp_allsum(A.B[k]); }
#pragma unroll
  for (int k = 0; k < 3; ++k) { warp_allsum(A.va[k]); warp_allsum(A.vc[k]); }
}

template <typename S>
__device__ __forceinline__ void acc_warp_sum(Acc<S>& A) {
  warp_sum(A.su); warp_sum(A.sa);
#pragma unroll
  for (int k = 0; k < 6; ++k) { warp_sum(A.P[k]); warp_sum(A.B[k]); }
#pragma unroll
  for (int k = 0; k < 3; ++k) { warp_sum(A.va[k]); warp_sum(A.vc[k]); }
}

}  // namespace ewb
