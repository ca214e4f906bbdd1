// host/instances.cpp -- C entry points of include/ssqa_host.h.
#include <algorithm>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>
#include <stdexcept>
#include <string>

#include "ssqa/gi.hpp"
#include "ssqa/model.hpp"
#include "ssqa/rng.hpp"
#include "ssqa_host.h"

namespace {

thread_local std::string g_host_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_host_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_host_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_host_err = e.what();
    return 3;
  }
}

constexpr uint32_t kStreamDenseCoupling = 8;
constexpr uint32_t kStreamDenseBias = 9;

// Run f(lo, hi) over [0, n) on all hardware threads.
template <class F>
void parallel_rows(int n, F&& f) {
  const int nt = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), n / 64 + 1));
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int lo = int(int64_t(n) * t / nt), hi = int(int64_t(n) * (t + 1) / nt);
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

const char* ssqa_host_last_error(void) { return g_host_err.c_str(); }

int ssqa_gi_ising(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                  double c2, double* h, double* J, double* offset) {
  return guard([&] {
    ssqa::gi_ising_arrays(ssqa::generate_gi(n_nodes, edge_prob, seed, permute != 0, c1, c2), h, J,
                          offset);
  });
}

int ssqa_gi_compact(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                    double c2, uint8_t* adj, double* h, double* offset) {
  return guard([&] {
    ssqa::gi_compact(ssqa::generate_gi(n_nodes, edge_prob, seed, permute != 0, c1, c2), adj, h,
                     offset);
  });
}

int ssqa_dense_ising(int n, int kind, uint64_t seed, double* h, double* J, double* offset) {
  return guard([&] {
    if (n < 1) throw std::invalid_argument("n must be >= 1");
    if (kind != 0 && kind != 1) throw std::invalid_argument("kind must be 0 or 1");
    const ssqa::CounterRng cj(seed, kStreamDenseCoupling), ch(seed, kStreamDenseBias);
    // Coupling (i, j), i < j, is drawn at counter i*n + j; every row is
    // filled independently (the mirror entries recompute their draw), so the
    // matrix is written sequentially by all threads.
    auto draw = [&](int a, int b) {  // a < b
      const uint64_t c = uint64_t(a) * uint64_t(n) + uint64_t(b);
      return kind == 0 ? double(int(cj.below(c, 16)) - 8) : ((cj.raw(c) >> 63) ? 1.0 : -1.0);
    };
    parallel_rows(n, [&](int lo, int hi) {
      for (int i = lo; i < hi; ++i) {
        double* row = J + size_t(i) * n;
        h[i] = kind == 0 ? double(int(ch.below(uint64_t(i), 16)) - 8) : 0.0;
        for (int j = 0; j < i; ++j) row[j] = draw(j, i);
        row[i] = 0.0;
        for (int j = i + 1; j < n; ++j) row[j] = draw(i, j);
      }
    });
    *offset = 0.0;
  });
}

int ssqa_ising_energy(int n, const double* h, const double* J, double offset,
                      const int8_t* spins, double* out) {
  return guard([&] {
    ssqa::IsingModel m(n, offset);
    for (int i = 0; i < n; ++i) {
      m.set_bias(i, h[i]);
      for (int j = i + 1; j < n; ++j) m.set_coupling(i, j, J[size_t(i) * n + j]);
    }
    *out = ssqa::ising_energy(m, ssqa::SpinVector(spins, spins + n));
  });
}

}  // extern "C"
