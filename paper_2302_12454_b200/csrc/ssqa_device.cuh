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

// ---- Issue-lean noise draw for the fused epilogue --------------------------
// The epilogue is bound by instruction issue and by the ALU pipe (LOP3 /
// SHF / ISETP / SEL), while the FMA pipe (IMAD) sits mostly idle.  This
// restatement of raw(spin_counter(cycle, k, i)) >> 59 (rng.hpp:10-15, 36-38)
// moves the 64-bit shifts onto the FMA pipe as multiplies by powers of two
// held in registers (mul.hi by 2^s == >> (32 - s), mul.lo by 2^s == << s),
// forms the counter sum with one wide multiply-add, and keeps three-input
// XORs on the ALU.  `base` = key + spin_counter(cycle, k, 0) * golden +
// golden (mix64's first add), so x0 = base + i * golden.
//   p4 = 4, p32 = 32: opaque to ptxas (kept in registers) so it cannot turn
//   the multiplies back into shifts.
// Returns the top five bits of the draw.
#ifndef SSQA_RNG_FMA
#define SSQA_RNG_FMA 1  // 1: shifts as IMAD.HI / IMAD.SHL (FMA pipe); 0: funnel shifts (ALU)
#endif
__device__ __forceinline__ uint32_t noise_top5(uint64_t base, uint32_t i, uint32_t p4,
                                               uint32_t p32) {
  uint32_t lo, hi;
  // x0 = base + i * golden (mod 2^64)
  asm("{\n\t.reg .u64 w;\n\t"
      "mad.wide.u32 w, %2, 0x7f4a7c15, %3;\n\t"
      "mov.b64 {%0, %1}, w;\n\t"
      "mad.lo.u32 %1, %2, 0x9e3779b9, %1;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(i), "l"(base));
  uint32_t l1, h1;
#if SSQA_RNG_FMA
  // x ^= x >> 30
  l1 = lo ^ __umulhi(lo, p4) ^ (hi * p4);
  h1 = hi ^ __umulhi(hi, p4);
#else
  l1 = lo ^ __funnelshift_r(lo, hi, 30);
  h1 = hi ^ (hi >> 30);
#endif
  // x *= 0xbf58476d1ce4e5b9
  uint32_t l2, h2;
  asm("{\n\t.reg .u64 w;\n\t"
      "mul.wide.u32 w, %2, 0x1ce4e5b9;\n\t"
      "mov.b64 {%0, %1}, w;\n\t"
      "mad.lo.u32 %1, %2, 0xbf58476d, %1;\n\t"
      "mad.lo.u32 %1, %3, 0x1ce4e5b9, %1;\n\t}"
      : "=r"(l2), "=r"(h2)
      : "r"(l1), "r"(h1));
  uint32_t l3, h3;
#if SSQA_RNG_FMA
  // x ^= x >> 27
  l3 = l2 ^ __umulhi(l2, p32) ^ (h2 * p32);
  h3 = h2 ^ __umulhi(h2, p32);
#else
  l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  h3 = h2 ^ (h2 >> 27);
#endif
  // high word of x * 0x94d049bb133111eb; its top five bits are the draw's
  // (the final x ^= x >> 31 leaves bits 63..59 unchanged)
  const uint32_t top = __umulhi(l3, 0x133111ebu) + l3 * 0x94d049bbu + h3 * 0x133111ebu;
  return __umulhi(top, p32);  // top >> 27
}

// noise_top5 for the issue-lean epilogue: the counter sum with the row's
// i * golden pinned in registers (add / add-with-carry), the low-word shifts
// as funnel shifts (ALU) and the high-word shifts as high products by 2^2 /
// 2^5 (FMA pipe), the last product as one multiply-high-add.
__device__ __forceinline__ uint32_t noise_top5_v4(uint64_t base, uint32_t iG_lo, uint32_t iG_hi,
                                                  uint32_t p4, uint32_t p32) {
  uint32_t lo, hi;
  asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;"
      : "=r"(lo), "=r"(hi)
      : "r"(uint32_t(base)), "r"(uint32_t(base >> 32)), "r"(iG_lo), "r"(iG_hi));
  const uint32_t l1 = lo ^ __funnelshift_r(lo, hi, 30);
  const uint32_t h1 = hi ^ __umulhi(hi, p4);
  uint32_t l2, h2;
  asm("{\n\t.reg .u64 w;\n\t"
      "mul.wide.u32 w, %2, 0x1ce4e5b9;\n\t"
      "mov.b64 {%0, %1}, w;\n\t"
      "mad.lo.u32 %1, %2, 0xbf58476d, %1;\n\t"
      "mad.lo.u32 %1, %3, 0x1ce4e5b9, %1;\n\t}"
      : "=r"(l2), "=r"(h2)
      : "r"(l1), "r"(h1));
  const uint32_t l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  const uint32_t h3 = h2 ^ __umulhi(h2, p32);
  uint32_t top;
  asm("mad.hi.u32 %0, %1, 0x133111eb, %2;"
      : "=r"(top)
      : "r"(l3), "r"(l3 * 0x94d049bbu + h3 * 0x133111ebu));
  return top >> 27;
}

// Noise level of update_spins (annealer.cpp:277-278) scaled to the integer
// field: nz_lut[t5] = 0 (t5 < 14), -NR (t5 < 23), +NR, NR = n_rnd * 2^p,
// |NR| <= 127 -- one conflict-free shared byte load instead of two compares
// and two selects (32 bytes span 8 banks; lanes of one word broadcast).
__device__ __forceinline__ void fill_noise_lut(int8_t* lut, int nr, int t) {
  if (t < 32) lut[t] = int8_t(t < 14 ? 0 : (t < 23 ? -nr : nr));
}
__device__ __forceinline__ int noise_lut(const int8_t* lut, uint32_t t5) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(uint32_t(__cvta_generic_to_shared(lut)) + t5));
  return v;
}

// update_fast2 with the noise already in the integer field and the bias of
// the magic-number conversion folded into it: xb = (S + H' + nz NR) ^ 2^31
// (i.e. + 2^31 mod 2^32, added once per row on the host side of the loop).
template <bool BIDIR>
__device__ __forceinline__ double update_fast3(const FastConsts& c, const I2D& i2d, uint32_t xb,
                                               int up, int dn, double acc) {
  double input = __dsub_rn(__hiloint2double(int(i2d.magic_hi), int(xb)), i2d.magic);
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
