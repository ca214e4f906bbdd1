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
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstring>
#include <cmath>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"

namespace ssqa_engine {

namespace {

// Smallest p in [0, 62] with v * 2^p integral, or -1.  Read off the IEEE
// bits: v = F * 2^(E - 1075) with F the significand (implicit 1 for normal
// numbers), so the lowest set bit of v has weight 2^(E - 1075 + ctz(F)).
int dyadic_exponent(double v) {
  uint64_t b;
  std::memcpy(&b, &v, sizeof b);
  const int E = int((b >> 52) & 0x7ff);
  if (E == 0x7ff) return -1;  // inf / nan
  uint64_t F = b & ((1ull << 52) - 1);
  if (E == 0 && F == 0) return 0;  // +-0
  if (E != 0) F |= 1ull << 52;
  const int low = (E == 0 ? 1 : E) - 1075 + __builtin_ctzll(F);
  const int p = low >= 0 ? 0 : -low;
  return p <= 62 ? p : -1;
}

// f(lo, hi) over [0, n) on all hardware threads (n up to 2^20 rows).
template <class F>
void parallel_for(int n, F&& f) {
  const int nt = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), n / 32 + 1));
  if (nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int lo = int(int64_t(n) * t / nt), hi = int(int64_t(n) * (t + 1) / nt);
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

void atomic_max(std::atomic<int>& a, int v) {
  int cur = a.load();
  while (v > cur && !a.compare_exchange_weak(cur, v)) {
  }
}
void atomic_min(std::atomic<long long>& a, long long v) {
  long long cur = a.load();
  while (v < cur && !a.compare_exchange_weak(cur, v)) {
  }
}

}  // namespace

bool build_fp4x2(const Quantized& q, std::vector<uint8_t>* out) {
  out->assign(size_t(q.npad) * q.npad, 0);
  std::atomic<bool> ok{true};
  parallel_for(q.npad, [&](int lo, int hi) {
    for (int i = lo; i < hi; ++i) {
      const int8_t* row = &q.J[size_t(i) * q.npad];
      uint8_t* o = out->data() + size_t(i) * q.npad;
      for (int j = 0; j < q.npad; ++j) {
        const int v = row[j];
        const int m = v < 0 ? -v : v;
        if (m > 12 || kFp4x2A[m] < 0) {
          ok = false;
          return;
        }
        const uint32_t s = v < 0 ? 8u : 0u;
        const size_t a = fp4x2_byte_a(j);
        const int sh = fp4x2_shift(j);
        if (kFp4x2A[m]) o[a] |= uint8_t((uint32_t(kFp4x2A[m]) | s) << sh);
        if (kFp4x2B[m]) o[a + 64] |= uint8_t((uint32_t(kFp4x2B[m]) | s) << sh);
      }
    }
  });
  return ok.load();
}

int dyadic_exponent_of(double v) { return dyadic_exponent(v); }

int quantize(int n, const double* h, const double* J, double offset, Quantized* q,
             std::string* why, int p_min) {
  // scale exponent: the largest dyadic exponent of any bias or coupling
  // (at least p_min, so several instances can share one scale)
  int p = std::max(0, p_min);
  for (int i = 0; i < n; ++i) {
    int e = dyadic_exponent(h[i]);
    if (e < 0) {
      *why = "bias " + std::to_string(i) + " is not a dyadic rational";
      return SSQA_EUNSUP;
    }
    if (e > p) p = e;
  }
  {
    std::atomic<int> pmax{p};
    std::atomic<long long> bad{LLONG_MAX};  // first non-dyadic coupling (row-major index)
    parallel_for(n, [&](int lo, int hi) {
      int pl = 0;
      for (int r = lo; r < hi; ++r) {
        const double* row = J + size_t(r) * n;
        for (int c = 0; c < n; ++c) {
          const int e = dyadic_exponent(row[c]);
          if (e < 0) {
            atomic_min(bad, (long long)r * n + c);
            break;
          }
          if (e > pl) pl = e;
        }
      }
      atomic_max(pmax, pl);
    });
    if (bad.load() != LLONG_MAX) {
      const long long v = bad.load();
      *why = "coupling " + std::to_string(v / n) + "," + std::to_string(v % n) +
             " is not a dyadic rational";
      return SSQA_EUNSUP;
    }
    p = pmax.load();
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
  // i: jpad[j*stride + i] = coupling_row(j)[i] (annealer.cpp:52-55, 107) --
  // a transpose of the (row-major) model matrix, done in 64x64 blocks.
  {
    constexpr int kB = 64;
    const int nb = (n + kB - 1) / kB;
    const double up = std::ldexp(1.0, p);
    std::atomic<int> maxj{0};
    std::atomic<bool> overflow{false};
    parallel_for(nb, [&](int lo, int hi) {
      int ml = 0;
      for (int bi = lo; bi < hi; ++bi) {
        const int i0 = bi * kB, i1 = std::min(n, i0 + kB);
        for (int j0 = 0; j0 < n; j0 += kB) {
          const int j1 = std::min(n, j0 + kB);
          for (int j = j0; j < j1; ++j) {
            const double* src = J + size_t(j) * n;
            for (int i = i0; i < i1; ++i) {
              const double x = src[i] * up;  // exact: a power-of-two scale of a dyadic value
              if (std::fabs(x) > 127.0) {
                overflow = true;
                return;
              }
              const int v = int(x);
              q->J[size_t(i) * q->npad + j] = int8_t(v);
              ml = std::max(ml, std::abs(v));
            }
          }
        }
      }
      atomic_max(maxj, ml);
    });
    if (overflow.load()) {
      *why = "coupling magnitude exceeds int8 at scale 2^" + std::to_string(p);
      return SSQA_EUNSUP;
    }
    q->max_abs_j = maxj.load();
  }
  // FP4 (e2m1) image: representable integers 0, 1, 2, 3, 4, 6 (+ sign).
  {
    static const int kCode[9] = {0, 2, 4, 5, 6, -1, 7, -1, -1};  // |v| -> e2m1 magnitude code
    q->fp4_ok = q->max_abs_j <= 6 && q->max_abs_j != 5;
    if (q->fp4_ok) {
      q->J4.assign(size_t(q->npad) * (q->npad / 2), 0);
      std::atomic<bool> ok{true};
      parallel_for(q->npad, [&](int lo, int hi) {
        for (int i = lo; i < hi; ++i) {
          const int8_t* row = &q->J[size_t(i) * q->npad];
          uint8_t* out = &q->J4[size_t(i) * (q->npad / 2)];
          for (int j = 0; j < q->npad; ++j) {
            const int v = row[j];
            const int c = kCode[v < 0 ? -v : v];
            if (c < 0) {
              ok = false;
              return;
            }
            out[j / 2] |= uint8_t((c | (v < 0 ? 8 : 0)) << (4 * (j & 1)));
          }
        }
      });
      q->fp4_ok = ok.load();
    }
    if (!q->fp4_ok) q->J4.clear();
  }
  // FP4 pair image when the single one does not exist: J' = A1 + A2.
  q->fp4x2_ok = false;
  if (!q->fp4_ok && fp4x2_splittable(q->max_abs_j)) {
    q->fp4x2_ok = build_fp4x2(*q, &q->J4);
    if (!q->fp4x2_ok) q->J4.clear();
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
