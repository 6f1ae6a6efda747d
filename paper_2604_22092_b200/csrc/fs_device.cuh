// fs_device.cuh — device math shared by every kernel: the counter-based
// uniform sources, the piecewise erfcx, the holding-time hazards and the
// shedding profiles.  Everything that feeds a parity-checked value is
// written with explicit IEEE rounding (the library is built -fmad=false as
// well), so the bits match the reference's numpy float64 / float32
// arithmetic step by step.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "../../include/flashspread.h"

namespace fs {

// ---------------------------------------------------------------------------
// splitmix64-style mixer — /root/reference/pkg/src/spreadsim/rng.py:31-67
// ---------------------------------------------------------------------------
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;        // rng.py:31
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;        // rng.py:32
constexpr uint64_t kStepMult = 0xA24BAED4963EE407ull;    // rng.py:33
constexpr uint64_t kStreamMult = 0x9FB21C651E98DF25ull;  // rng.py:34
constexpr double kInv2p53 = 1.1102230246251565e-16;      // 2**-53, rng.py:36

__host__ __device__ __forceinline__ uint64_t avalanche(uint64_t x) {  // rng.py:48-51
  x = (x ^ (x >> 30)) * kMix1;
  x = (x ^ (x >> 27)) * kMix2;
  return x ^ (x >> 31);
}
// per-(seed, step) key, hoisted out of the per-node work (rng.py:56)
__host__ __device__ __forceinline__ uint64_t splitmix_step_key(uint64_t seed, uint64_t step) {
  return avalanche(seed ^ (step * kStepMult));
}
// uniform in [0,1) with 53 random bits (rng.py:57, 66-67)
__device__ __forceinline__ double splitmix_uniform(uint64_t step_key, uint64_t stream) {
  uint64_t b = avalanche(step_key ^ (stream * kStreamMult));
  return (double)(b >> 11) * kInv2p53;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  key = (seed lo, seed hi),
// counter = (stream lo, stream hi, step lo, step hi); the uniform takes the
// top 53 bits of (x1 << 32 | x0).  north_star extension: no reference.
// ---------------------------------------------------------------------------
struct Philox4 { uint32_t x0, x1, x2, x3; };

__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
}

__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c.x0, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c.x2, hi1, lo1);
    c = Philox4{hi1 ^ c.x1 ^ k0, lo1, hi0 ^ c.x3 ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// not inlined: the step kernels carry it for the rng="philox" option only, and
// its 10 rounds' state would otherwise weigh on their register allocation
static __device__ __noinline__ double philox_uniform(uint64_t seed, uint64_t step, uint64_t stream) {
  Philox4 c{(uint32_t)stream, (uint32_t)(stream >> 32), (uint32_t)step, (uint32_t)(step >> 32)};
  Philox4 o = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint64_t b = ((uint64_t)o.x1 << 32) | (uint64_t)o.x0;
  return (double)(b >> 11) * kInv2p53;
}

// ---------------------------------------------------------------------------
// erfcx — the reference's piecewise form, hazards.py:84-105:
//   identity exp(z^2) erfc(z) on [0, 3.5], 4-term asymptotic series above,
//   reflection 2 exp(z^2) - erfcx(-z) below 0.
// ---------------------------------------------------------------------------
constexpr double kBranchZ = 3.5;                       // hazards.py:35
constexpr double kSqrtPi = 1.7724538509055159;         // math.sqrt(math.pi)
constexpr double kSqrt2OverPi = 0.7978845608028654;    // math.sqrt(2/pi)
constexpr double kSqrt2 = 1.4142135623730951;          // math.sqrt(2.0)

__device__ __forceinline__ double erfcx_positive(double z) {
  if (z <= kBranchZ) return __dmul_rn(exp(__dmul_rn(z, z)), erfc(z));
  double inv2 = __ddiv_rn(1.0, __dmul_rn(z, z));
  double poly = __dadd_rn(0.75, __dmul_rn(inv2, -1.875));
  poly = __dadd_rn(-0.5, __dmul_rn(inv2, poly));
  poly = __dadd_rn(1.0, __dmul_rn(inv2, poly));
  return __ddiv_rn(poly, __dmul_rn(z, kSqrtPi));
}

__device__ __forceinline__ double erfcx_piecewise(double z) {
  if (z < 0.0) return __dsub_rn(__dmul_rn(2.0, exp(__dmul_rn(z, z))), erfcx_positive(-z));
  return erfcx_positive(z);
}

// log-normal hazard in f64, hazards.py:122-132 (h(0) = 0, inf denominator -> 0)
__device__ __forceinline__ double hazard_lognormal_f64(double tau, double mu, double sigma) {
  if (!(tau > 0.0)) return 0.0;
  double z = __ddiv_rn(__dsub_rn(log(tau), mu), __dmul_rn(sigma, kSqrt2));
  double denom = __dmul_rn(__dmul_rn(tau, sigma), erfcx_piecewise(z));
  if (isinf(denom)) return 0.0;
  return __ddiv_rn(kSqrt2OverPi, denom);
}

// Weibull(k, lambda) hazard: (k/lambda) (tau/lambda)^(k-1).  north_star
// extension; oracle/spreadsim_port.py uses the same
// operation order.
__device__ __forceinline__ double hazard_weibull_f64(double tau, double k, double lam) {
  if (!(tau > 0.0)) return (k == 1.0) ? __ddiv_rn(1.0, lam) : 0.0;
  double x = __ddiv_rn(tau, lam);
  return __dmul_rn(__ddiv_rn(k, lam), pow(x, __dsub_rn(k, 1.0)));
}

// Erlang(k, r) hazard: r (r tau)^(k-1)/(k-1)! / sum_{n<k} (r tau)^n / n!,
// evaluated with the running term t_n = t_{n-1} * x / n.
__device__ __forceinline__ double hazard_erlang_f64(double tau, int k, double r) {
  if (!(tau > 0.0)) return (k == 1) ? r : 0.0;
  double x = __dmul_rn(r, tau);
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < k; ++n) {
    term = __ddiv_rn(__dmul_rn(term, x), (double)n);
    sum = __dadd_rn(sum, term);
  }
  return __ddiv_rn(__dmul_rn(r, term), sum);
}

// ---- fp32 variants (FS_HAZ_F32): same piecewise formulas in float; the
// z<0 reflection is rewritten exp(-z^2)/... to stay finite in fp32.
__device__ __forceinline__ float erfcx_positive_f32(float z) {
  if (z <= 3.5f) return expf(z * z) * erfcf(z);
  float inv2 = 1.0f / (z * z);
  return (1.0f + inv2 * (-0.5f + inv2 * (0.75f + inv2 * (-1.875f)))) / (z * 1.7724538509f);
}
__device__ __forceinline__ float hazard_lognormal_f32(float tau, float mu, float sigma) {
  if (!(tau > 0.0f)) return 0.0f;
  float z = (logf(tau) - mu) / (sigma * 1.4142135624f);
  float ex;
  if (z < 0.0f) {
    // erfcx(z) = 2 e^{z^2} - erfcx(-z); h = c / (tau sigma erfcx(z)).  For
    // z << 0 the first term dominates: use h = c e^{-z^2} / (tau sigma (2 - e^{-z^2} erfcx(-z)))
    float emz2 = expf(-z * z);
    float d = tau * sigma * (2.0f - emz2 * erfcx_positive_f32(-z));
    return 0.7978845608f * emz2 / d;
  }
  ex = erfcx_positive_f32(z);
  return 0.7978845608f / (tau * sigma * ex);
}
__device__ __forceinline__ float hazard_weibull_f32(float tau, float k, float lam) {
  if (!(tau > 0.0f)) return (k == 1.0f) ? 1.0f / lam : 0.0f;
  return (k / lam) * powf(tau / lam, k - 1.0f);
}
__device__ __forceinline__ float hazard_erlang_f32(float tau, int k, float r) {
  if (!(tau > 0.0f)) return (k == 1) ? r : 0.0f;
  float x = r * tau, term = 1.0f, sum = 1.0f;
  for (int n = 1; n < k; ++n) { term = term * x / (float)n; sum += term; }
  return r * term / sum;
}

// the hazards other than the f64 log-normal, out of line: a call per drain
// where they are used, and no register pressure where they are not
static __device__ __noinline__ float nodal_rate_other(int kind, double p0, double p1, float age, int prec) {
  switch (kind) {
    case FS_HZ_LOGNORMAL: return hazard_lognormal_f32(age, (float)p0, (float)p1);
    case FS_HZ_WEIBULL:
      return prec == FS_HAZ_F64 ? __double2float_rn(hazard_weibull_f64((double)age, p0, p1))
                                : hazard_weibull_f32(age, (float)p0, (float)p1);
    case FS_HZ_ERLANG:
      return prec == FS_HAZ_F64 ? __double2float_rn(hazard_erlang_f64((double)age, (int)p0, p1))
                                : hazard_erlang_f32(age, (int)p0, (float)p1);
    default: return 0.0f;
  }
}

// rate of a nodal compartment at age `age` (f32 storage value), cast to the
// f32 rate buffer exactly as renewal.py:474-480 (f64 math, f32 store)
__device__ __forceinline__ float nodal_rate(int kind, double p0, double p1, float age, int prec) {
  if (kind == FS_HZ_EXPONENTIAL) return __double2float_rn(p0);
  if (kind == FS_HZ_LOGNORMAL && prec == FS_HAZ_F64) return __double2float_rn(hazard_lognormal_f64((double)age, p0, p1));
  return nodal_rate_other(kind, p0, p1, age, prec);
}

// shedding profile s(tau), hazards.py:196-218 (f64)
__device__ __forceinline__ double shedding_f64(int kind, double mu, double sigma, double peak, double tau) {
  if (kind == FS_SHED_CONSTANT) return 1.0;
  if (kind == FS_SHED_LN_HAZARD) return hazard_lognormal_f64(tau, mu, sigma);
  // density_peak: lognormal_pdf(tau) / lognormal_pdf(mode), hazards.py:149-158
  if (!(tau > 0.0)) return __ddiv_rn(0.0, peak);
  double zs = __ddiv_rn(__dsub_rn(log(tau), mu), sigma);
  double num = exp(__dmul_rn(__dmul_rn(-0.5, zs), zs));
  double den = __dmul_rn(__dmul_rn(tau, sigma), 2.5066282746310002);  // math.sqrt(2*pi)
  return __ddiv_rn(__ddiv_rn(num, den), peak);
}

// Bernoulli decision u < q with q = -expm1(-rate*tau) in f64
// (renewal.py:533-535).  The bracket t - t^2/2 <= q <= t settles almost
// every draw without the expm1; the bracket is widened by 1e-12 relative,
// far beyond the few-ulp disagreement of two libm expm1s.
__device__ __forceinline__ bool bernoulli_fire(double u, float rate, double tau) {
  double x = __dmul_rn(-(double)rate, tau);  // -(rates.astype(f64)) * tau
  double t = -x;
  if (u >= __dmul_rn(t, 1.000000000001)) return false;
  double lo = __dmul_rn(__dsub_rn(t, __dmul_rn(__dmul_rn(0.5, t), t)), 0.999999999999);
  if (u < lo) return true;
  return u < -expm1(x);
}

// ---------------------------------------------------------------------------
// storage-type helpers (promote on load, cast on store; renewal.py:358-367)
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

}  // namespace fs
