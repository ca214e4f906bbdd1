// ssqa_device.cuh -- device-side building blocks shared by every sweep kernel.
//
// Counter RNG (rng.hpp:10-67), the exact FP64 update of update_spins
// (annealer.cpp:258-300) and the integer field/energy algebra that replaces
// the reference's double field tiles (annealer.cpp:91-256).
#pragma once

#include <cstdint>

namespace ssqa_dev {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr uint32_t kStreamSpinInit = 1;    // rng.hpp:21
constexpr uint32_t kStreamSweepNoise = 2;  // rng.hpp:22

// splitmix64 finalizer, rng.hpp:10-15.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// CounterRng key, rng.hpp:33-34.
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint32_t stream) {
  return mix64(mix64(seed) ^ (0x100000000ull + stream));
}

// spin_counter, rng.hpp:65-67.
__host__ __device__ __forceinline__ uint64_t spin_counter(uint64_t cycle, uint32_t k,
                                                          uint32_t i) {
  return (cycle << 32) | (uint64_t(k) << 20) | uint64_t(i);
}

// Top five bits of mix64(x0): x ^ (x >> 31) leaves bits 63..59 of x
// unchanged, so only the high word of the second product is needed.
__device__ __forceinline__ uint32_t mix64_top5(uint64_t x0) {
  uint64_t x = x0 + kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
  // high 32 bits of the low 64-bit product x * C2
  const uint32_t c2lo = 0x133111ebu, c2hi = 0x94d049bbu;
  uint32_t top = __umulhi(lo, c2lo) + lo * c2hi + hi * c2lo;
  return top >> 27;
}

// mix64_top5 for an argument that already includes mix64's "+= golden".
__device__ __forceinline__ uint32_t mix64_top5_pre(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
  const uint32_t c2lo = 0x133111ebu, c2hi = 0x94d049bbu;
  return (__umulhi(lo, c2lo) + lo * c2hi + hi * c2lo) >> 27;
}

// High 32 bits of the final splitmix product for an argument that already
// includes mix64's "+= golden" (the top five bits decide the noise level;
// comparing the whole word against t << 27 avoids the shift).
__device__ __forceinline__ uint32_t mix64_top32_pre(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
  const uint32_t c2lo = 0x133111ebu, c2hi = 0x94d049bbu;
  return __umulhi(lo, c2lo) + lo * c2hi + hi * c2lo;
}

// Noise level of update_spins (annealer.cpp:277-278):
//   u = (raw >> 11) * 2^-53;  u < 7/16 -> 0,  u < 23/32 -> -1,  else +1.
// Both thresholds are exact multiples of 2^-5, so the comparison reduces to
// the top five bits t of raw: t < 14 -> 0, t < 23 -> -1, else +1.
// Returns 0, 1, 2 for the noise values 0.0, -1.0, +1.0.
__device__ __forceinline__ int noise_index(uint32_t top5) {
  return top5 < 14u ? 0 : (top5 < 23u ? 1 : 2);
}

// Everything update_spins needs besides the per-spin data; doubles are the
// reference's own values, products formed exactly as the reference forms
// them (n_rnd * {0,-1,+1}, jperp * {+1,-1}).
struct UpdateConsts {
  double noise[3];   // n_rnd * 0.0, n_rnd * -1.0, n_rnd * 1.0
  double jp_pos;     // jperp * 1.0
  double jp_neg;     // jperp * -1.0
  double i0;
  double hi_clamp;   // i0 - alpha
  double lo_clamp;   // -i0
};

__device__ __forceinline__ UpdateConsts make_consts(double n_rnd, double jperp, double i0,
                                                    double alpha) {
  UpdateConsts c;
  c.noise[0] = __dmul_rn(n_rnd, 0.0);
  c.noise[1] = __dmul_rn(n_rnd, -1.0);
  c.noise[2] = __dmul_rn(n_rnd, 1.0);
  c.jp_pos = __dmul_rn(jperp, 1.0);
  c.jp_neg = __dmul_rn(jperp, -1.0);
  c.i0 = i0;
  c.hi_clamp = __dsub_rn(i0, alpha);
  c.lo_clamp = -i0;
  return c;
}

// One (i, k) update, annealer.cpp:269-295, in the reference's operation
// order with round-to-nearest adds and no contraction.
//   field   : h_i + sum_j J_ij sigma_jk (exact double)
//   nidx    : noise_index(top5 of raw(spin_counter(cycle, k, i)))
//   up, dn  : delayed neighbour spins sigma_{k+1}, sigma_{k-1} (+-1)
// Returns the clamped accumulator; the new spin is (acc >= 0.0 ? +1 : -1).
__device__ __forceinline__ double update_one(const UpdateConsts& c, double field, int nidx,
                                             int up, int dn, bool bidirectional,
                                             double acc) {
  double input = field;
  const double nz = nidx == 0 ? c.noise[0] : (nidx == 1 ? c.noise[1] : c.noise[2]);
  input = __dadd_rn(input, nz);
  input = __dadd_rn(input, up > 0 ? c.jp_pos : c.jp_neg);
  if (bidirectional) input = __dadd_rn(input, dn > 0 ? c.jp_pos : c.jp_neg);
  const double s = __dadd_rn(acc, input);
  return (s >= c.i0) ? c.hi_clamp : ((s < c.lo_clamp) ? c.lo_clamp : s);
}

// update_one with the noise level chosen straight from the top five RNG
// bits (branch-free selects): t5 < 14 -> noise[0], t5 < 23 -> noise[1],
// else noise[2].
__device__ __forceinline__ double update_fast(const UpdateConsts& c, double field,
                                              uint32_t t5, int up, int dn, bool bidirectional,
                                              double acc) {
  const bool rest = t5 < 14u, neg = t5 < 23u;
  double nz = neg ? c.noise[1] : c.noise[2];
  nz = rest ? c.noise[0] : nz;
  double input = __dadd_rn(field, nz);
  input = __dadd_rn(input, up > 0 ? c.jp_pos : c.jp_neg);
  if (bidirectional) input = __dadd_rn(input, dn > 0 ? c.jp_pos : c.jp_neg);
  const double s = __dadd_rn(acc, input);
  const double lo = (s < c.lo_clamp) ? c.lo_clamp : s;
  return (s >= c.i0) ? c.hi_clamp : lo;
}

// Exact v * 2^-p for int32 v without the XU-pipe I2F.F64: the bit pattern
// hi:(v ^ 2^31) with hi = exponent of 2^(52-p) encodes (2^52 + v + 2^31) *
// 2^-p exactly; subtracting (2^52 + 2^31) * 2^-p (exact, same binade) leaves
// v * 2^-p.  magic_hi = 0x43300000 - (p << 20), magic = (2^52 + 2^31) * 2^-p.
struct I2D {
  uint32_t magic_hi;
  double magic;
};

__host__ __device__ inline I2D make_i2d(int p) {
  I2D c;
  c.magic_hi = 0x43300000u - (uint32_t(p) << 20);
  double m = 4503601774854144.0;  // 2^52 + 2^31
  for (int k = 0; k < p; ++k) m *= 0.5;
  c.magic = m;
  return c;
}

__device__ __forceinline__ double scaled_i32(int v, const I2D& c) {
  const double d = __hiloint2double(int(c.magic_hi), int(uint32_t(v) ^ 0x80000000u));
  return __dsub_rn(d, c.magic);
}

// Fast-path constants (valid when every parameter is finite and
// n_rnd * 2^p is an integer NR): the noise joins the integer field
// (field + n_rnd*nz == (S + H' + nz*NR) * 2^-p exactly), the coupling term
// jperp * (+-1) is jperp with its sign bit flipped, and signs of finite,
// never -0.0 accumulators come from the high word.
struct FastConsts {
  int nr;              // n_rnd * 2^p
  uint32_t jp_hi, jp_lo;  // bits of jperp * 1.0
  double i0, hi_clamp, lo_clamp;
};

template <bool BIDIR>
__device__ __forceinline__ double update_fast2(const FastConsts& c, const I2D& i2d, int s_h1,
                                               uint32_t top, int up, int dn, double acc) {
  const int nzi = top < 0x70000000u ? 0 : (top < 0xB8000000u ? -c.nr : c.nr);
  double input = scaled_i32(s_h1 + nzi, i2d);
  input = __dadd_rn(input, __hiloint2double(int(c.jp_hi ^ (uint32_t(up) & 0x80000000u)),
                                            int(c.jp_lo)));
  if (BIDIR)
    input = __dadd_rn(input, __hiloint2double(int(c.jp_hi ^ (uint32_t(dn) & 0x80000000u)),
                                              int(c.jp_lo)));
  const double s = __dadd_rn(acc, input);
  const double lo = (s < c.lo_clamp) ? c.lo_clamp : s;
  return (s >= c.i0) ? c.hi_clamp : lo;
}

// Exact double of an integer field scaled by 2^-p (|v| < 2^53).
__device__ __forceinline__ double scaled(long long v, double scale) {
  return __dmul_rn(double(v), scale);
}

}  // namespace ssqa_dev
