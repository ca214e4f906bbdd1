// quantize.cpp -- host quantizer: IsingModel doubles -> int8 J', int32 H'.
//
// Replaces DenseProblem's 1-byte coupling codes (annealer.cpp:32-89) with
// an exact integer image: J' = J * 2^p, H' = h * 2^p for the smallest
// p >= 0 that makes every coupling and bias an integer.  Because sigma is
// +-1, the reference's double field h_i + sum_j J_ij sigma_j is then exactly
// (H'_i + S_i) * 2^-p with the integer contraction S = J' sigma, and the
// replica energy -1/2 sum_i sigma_i (F_i + h_i) + offset is exactly
// -1/2 * (sum_i sigma_i (S_i + 2 H'_i)) * 2^-p + offset (annealer.cpp:246-256)
// -- the only rounding left is the final "+ offset", which the device
// performs with the same operands.  Models with no such p (non-dyadic
// couplings) or |J'| > 127 are rejected: the engine has no CPU fallback.
#include <cmath>
#include <cstdlib>
#include <string>

#include "engine.h"

namespace ssqa_engine {

namespace {

// Smallest p in [0, 62] with v * 2^p integral, or -1.
int dyadic_exponent(double v) {
  if (!std::isfinite(v)) return -1;
  if (v == 0.0) return 0;
  for (int p = 0; p <= 62; ++p) {
    double x = std::ldexp(v, p);
    if (x == std::floor(x)) return p;
  }
  return -1;
}

}  // namespace

int quantize(int n, const double* h, const double* J, double offset, Quantized* q,
             std::string* why) {
  int p = 0;
  for (int i = 0; i < n; ++i) {
    int e = dyadic_exponent(h[i]);
    if (e < 0) {
      *why = "bias " + std::to_string(i) + " is not a dyadic rational";
      return SSQA_EUNSUP;
    }
    if (e > p) p = e;
  }
  for (size_t v = 0; v < size_t(n) * n; ++v) {
    int e = dyadic_exponent(J[v]);
    if (e < 0) {
      *why = "coupling " + std::to_string(v / n) + "," + std::to_string(v % n) +
             " is not a dyadic rational";
      return SSQA_EUNSUP;
    }
    if (e > p) p = e;
  }
  q->n = n;
  q->npad = (n + 127) / 128 * 128;
  q->p = p;
  q->offset = offset;
  q->scale = std::ldexp(1.0, -p);
  q->J.assign(size_t(q->npad) * q->npad, 0);
  q->H.assign(size_t(q->npad), 0);
  q->max_abs_j = 0;
  q->max_abs_h = 0;
  // Row i of J' holds the coefficients the reference multiplies into field
  // i: jpad[j*stride + i] = coupling_row(j)[i] (annealer.cpp:52-55, 107).
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j) {
      double x = std::ldexp(J[size_t(j) * n + i], p);
      if (std::fabs(x) > 127.0) {
        *why = "coupling magnitude exceeds int8 at scale 2^" + std::to_string(p);
        return SSQA_EUNSUP;
      }
      int v = int(x);
      q->J[size_t(i) * q->npad + j] = int8_t(v);
      if (std::abs(v) > q->max_abs_j) q->max_abs_j = std::abs(v);
    }
  }
  // FP4 (e2m1) image: representable integers 0, 1, 2, 3, 4, 6 (+ sign).
  {
    auto code = [](int v) -> int {
      const int a = v < 0 ? -v : v;
      int c;
      switch (a) {
        case 0: c = 0; break;
        case 1: c = 2; break;
        case 2: c = 4; break;
        case 3: c = 5; break;
        case 4: c = 6; break;
        case 6: c = 7; break;
        default: return -1;
      }
      return c | (v < 0 ? 8 : 0);
    };
    q->fp4_ok = true;
    q->J4.assign(size_t(q->npad) * (q->npad / 2), 0);
    for (int i = 0; i < q->npad && q->fp4_ok; ++i) {
      for (int j = 0; j < q->npad; ++j) {
        const int c = code(q->J[size_t(i) * q->npad + j]);
        if (c < 0) {
          q->fp4_ok = false;
          break;
        }
        q->J4[size_t(i) * (q->npad / 2) + j / 2] |= uint8_t(c << (4 * (j & 1)));
      }
    }
    if (!q->fp4_ok) q->J4.clear();
  }
  // |H'| < 2^29 keeps S + 2H' inside int32 for every n < 2^20.
  for (int i = 0; i < n; ++i) {
    double x = std::ldexp(h[i], p);
    if (std::fabs(x) >= double(1 << 29)) {
      *why = "bias magnitude exceeds the int32 field range at scale 2^" + std::to_string(p);
      return SSQA_EUNSUP;
    }
    int v = int(x);
    q->H[i] = v;
    if (std::abs(v) > q->max_abs_h) q->max_abs_h = std::abs(v);
  }
  return SSQA_OK;
}

}  // namespace ssqa_engine
