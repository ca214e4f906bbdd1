// host/inputs.cpp -- the engine's input side: IsingModel, the minimal
// QuboModel the reference API hands around, and the GI instance builder.
//
// Only what the annealing path consumes lives here (SURVEY.md section 8.1
// rows a12 and f2): model/graph text I/O, mapping decode/verify and the
// other toolkit utilities of proj/src/{model,gi}.cpp are out of scope.
//
// The GI builder does not materialise the O(n^4) penalty QUBO the way the
// reference's build_gi_qubo (gi.cpp:146-184) does.  Every off-diagonal
// entry of that QUBO receives exactly one contribution, so it is a closed
// form of the two adjacency matrices (the Kronecker structure of the GI
// penalty):
//   a = (u, i), b = (v, j), spin index (u-1) n + (i-1), u = graph-2 vertex,
//   i = graph-1 role:
//     Q_aa = -2 c1
//     Q_ab =  2 c1            u == v xor i == j      (one-hot rows / columns)
//     Q_ab =  c2              u != v, i != j, A1(i,j) != A2(u,v)
//     Q_ab =  0               otherwise
// and the Ising map x = (s+1)/2 (model.cpp:139-161) then gives
//   J_ab = -Q_ab / 4 (only where Q_ab != 0, so untouched entries stay +0.0),
//   h_a  = c1 - sum_{b != a, ascending, Q_ab != 0} Q_ab / 4,
//   offset = 2 c1 n + sum_a ( -c1 + sum_{b > a, ascending, Q_ab != 0} Q_ab / 4 ),
// accumulated in exactly that order, so the doubles equal the reference's
// bit for bit for any c1, c2 (tests/golden/gi_instances.npz pins it).
// Graph draws follow generate_gi (gi.cpp:102-144): edge (u, v), u < v, is
// present iff uniform01(u (n+1) + v) < p under key (seed, kStreamGiEdges);
// the relabelling is a Fisher-Yates pass u = n .. 2 with w = 1 + below(u, u)
// under (seed, kStreamGiPerm).
#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>

#include "ssqa/gi.hpp"
#include "ssqa/model.hpp"
#include "ssqa/rng.hpp"
#include "ssqa_host.h"

namespace ssqa {

namespace {

[[noreturn]] void bad_index(const char* what, int i, int n) {
  throw std::out_of_range(std::string(what) + " index " + std::to_string(i) +
                          " not in [0, " + std::to_string(n) + ")");
}

inline void need_index(int i, int n, const char* what) {
  if (unsigned(i) >= unsigned(n)) bad_index(what, i, n);
}

inline void need_node(int u, int n) {
  if (u < 1 || u > n)
    throw std::invalid_argument("graph node " + std::to_string(u) + " not in [1, " +
                                std::to_string(n) + "]");
}

// Symmetric 0/1 adjacency of a 1-based graph, stored 0-based.
std::vector<uint8_t> adjacency(const Graph& g) {
  const int n = g.n_nodes;
  std::vector<uint8_t> a(size_t(n) * n, 0);
  for (const auto& e : g.edges) {
    a[size_t(e.first - 1) * n + (e.second - 1)] = 1;
    a[size_t(e.second - 1) * n + (e.first - 1)] = 1;
  }
  return a;
}

void check_penalties(double c1, double c2) {
  if (!(c1 > 0.0) || !(c2 > 0.0)) throw std::invalid_argument("GI penalties c1, c2 must be > 0");
}

}  // namespace

// ------------------------------------------------------------------ spins
SpinVector bits_to_spins(const BitVector& x) {
  SpinVector s(x.size());
  std::transform(x.begin(), x.end(), s.begin(), [](uint8_t b) -> int8_t {
    if (b > 1) throw std::invalid_argument("bit vector holds a value other than 0/1");
    return b ? 1 : -1;
  });
  return s;
}

BitVector spins_to_bits(const SpinVector& s) {
  BitVector x(s.size());
  std::transform(s.begin(), s.end(), x.begin(), [](int8_t v) -> uint8_t {
    if (v != 1 && v != -1) throw std::invalid_argument("spin vector holds a value other than +-1");
    return v > 0;
  });
  return x;
}

// ------------------------------------------------------------- QuboModel
QuboModel::QuboModel(int n, double constant) : n_(n), constant_(constant) {
  if (n < 1) throw std::invalid_argument("QuboModel: n must be >= 1");
  q_.assign(size_t(n) * size_t(n), 0.0);
}

size_t QuboModel::index(int i, int j) const {
  need_index(i, n_, "variable");
  need_index(j, n_, "variable");
  return i <= j ? size_t(i) * n_ + j : size_t(j) * n_ + i;
}

double QuboModel::coeff(int i, int j) const { return q_[index(i, j)]; }
void QuboModel::set_coeff(int i, int j, double value) { q_[index(i, j)] = value; }
void QuboModel::add_coeff(int i, int j, double value) { q_[index(i, j)] += value; }

double qubo_energy(const QuboModel& q, const BitVector& x) {
  if (x.size() != size_t(q.n())) throw std::invalid_argument("bit vector length != model size");
  double e = q.constant();
  for (int i = 0; i < q.n(); ++i) {
    if (x[i] > 1) throw std::invalid_argument("bit vector holds a value other than 0/1");
    if (!x[i]) continue;
    e += q.coeff(i, i);
    for (int j = i + 1; j < q.n(); ++j)
      if (x[j]) e += q.coeff(i, j);
  }
  return e;
}

// ------------------------------------------------------------ IsingModel
IsingModel::IsingModel(int n, double offset) : n_(n), offset_(offset) {
  if (n < 1) throw std::invalid_argument("IsingModel: n must be >= 1");
  h_.assign(size_t(n), 0.0);
  j_.assign(size_t(n) * size_t(n), 0.0);
}

double IsingModel::bias(int i) const {
  need_index(i, n_, "spin");
  return h_[size_t(i)];
}

void IsingModel::set_bias(int i, double value) {
  need_index(i, n_, "spin");
  h_[size_t(i)] = value;
}

double IsingModel::coupling(int i, int j) const {
  need_index(i, n_, "spin");
  need_index(j, n_, "spin");
  return j_[size_t(i) * n_ + j];
}

void IsingModel::set_coupling(int i, int j, double value) {
  need_index(i, n_, "spin");
  need_index(j, n_, "spin");
  if (i == j) throw std::invalid_argument("IsingModel: no self-coupling (i == j)");
  j_[size_t(i) * n_ + j] = value;
  j_[size_t(j) * n_ + i] = value;
}

// H(s) = offset - sum_i h_i s_i - sum_{i<j} J_ij s_i s_j in row order.
double ising_energy(const IsingModel& m, const SpinVector& s) {
  const int n = m.n();
  if (s.size() != size_t(n)) throw std::invalid_argument("spin vector length != model size");
  double e = m.offset();
  for (int i = 0; i < n; ++i) {
    if (s[i] != 1 && s[i] != -1)
      throw std::invalid_argument("spin vector holds a value other than +-1");
    e -= m.bias(i) * s[i];
    const double* row = m.coupling_row(i);
    for (int j = i + 1; j < n; ++j) e -= row[j] * s[i] * s[j];
  }
  return e;
}

double ising_flip_delta(const IsingModel& m, const SpinVector& s, int i) {
  if (s.size() != size_t(m.n())) throw std::invalid_argument("spin vector length != model size");
  need_index(i, m.n(), "spin");
  double f = m.bias(i);
  const double* row = m.coupling_row(i);
  for (int j = 0; j < m.n(); ++j) f += row[j] * s[j];
  return 2.0 * s[i] * f;
}

// x = (s + 1) / 2: h_a = -Q_aa/2 - sum_{b != a} Q_ab/4 (ascending b), J_ab =
// -Q_ab/4, offset = C + sum_a (Q_aa/2 + sum_{b > a} Q_ab/4); zero entries
// are skipped so they leave no -0.0 behind.
IsingModel qubo_to_ising(const QuboModel& q) {
  const int n = q.n();
  IsingModel m(n);
  double off = q.constant();
  for (int a = 0; a < n; ++a) {
    const double qd = q.coeff(a, a);
    double h = -0.5 * qd;
    off += 0.5 * qd;
    for (int b = 0; b < n; ++b) {
      if (b == a) continue;
      const double v = q.coeff(a, b);
      if (v == 0.0) continue;
      h -= 0.25 * v;
      if (b > a) {
        m.set_coupling(a, b, -0.25 * v);
        off += 0.25 * v;
      }
    }
    m.set_bias(a, h);
  }
  m.set_offset(off);
  return m;
}

// ------------------------------------------------------------------ graphs
bool Graph::has_edge(int u, int v) const {
  const std::pair<int, int> e(std::min(u, v), std::max(u, v));
  return std::binary_search(edges.begin(), edges.end(), e);
}

void Graph::add_edge(int u, int v) {
  need_node(u, n_nodes);
  need_node(v, n_nodes);
  if (u == v) throw std::invalid_argument("graph edge is a self-loop");
  edges.emplace_back(std::min(u, v), std::max(u, v));
}

void Graph::normalize() {
  for (const auto& e : edges) {
    need_node(e.first, n_nodes);
    need_node(e.second, n_nodes);
    if (e.first >= e.second) throw std::invalid_argument("graph edge not stored as u < v");
  }
  std::sort(edges.begin(), edges.end());
  if (std::adjacent_find(edges.begin(), edges.end()) != edges.end())
    throw std::invalid_argument("graph holds a duplicate edge");
}

GiInstance generate_gi(int n_nodes, double edge_prob, uint64_t seed, bool permute, double c1,
                       double c2) {
  if (n_nodes < 1) throw std::invalid_argument("generate_gi: n_nodes must be >= 1");
  if (!(edge_prob >= 0.0 && edge_prob <= 1.0))
    throw std::invalid_argument("generate_gi: edge_prob must lie in [0, 1]");
  check_penalties(c1, c2);
  const int n = n_nodes;
  GiInstance g;
  g.c1 = c1;
  g.c2 = c2;
  g.graph1.n_nodes = g.graph2.n_nodes = n;
  const CounterRng edges(seed, kStreamGiEdges);
  for (int u = 1; u < n; ++u)  // counters ascend, so the list comes out sorted
    for (int v = u + 1; v <= n; ++v)
      if (edges.uniform01(uint64_t(u) * uint64_t(n + 1) + uint64_t(v)) < edge_prob)
        g.graph1.edges.emplace_back(u, v);
  // lab[u] = graph-2 name of graph-1 vertex u
  std::vector<int> lab(size_t(n) + 1);
  std::iota(lab.begin(), lab.end(), 0);
  if (permute) {
    const CounterRng perm(seed, kStreamGiPerm);
    for (int u = n; u >= 2; --u) std::swap(lab[u], lab[1 + int(perm.below(uint64_t(u), uint64_t(u)))]);
  }
  for (const auto& e : g.graph1.edges)
    g.graph2.edges.emplace_back(std::min(lab[e.first], lab[e.second]),
                                std::max(lab[e.first], lab[e.second]));
  std::sort(g.graph2.edges.begin(), g.graph2.edges.end());
  std::vector<int> truth(static_cast<size_t>(n));
  for (int u = 1; u <= n; ++u) truth[size_t(lab[u] - 1)] = u;
  g.truth_perm = std::move(truth);
  return g;
}

namespace {

// Q_ab of the GI penalty in closed form (see the header comment); a, b are
// 0-based spin indices (u-1) n + (i-1).
struct GiPenalty {
  int n;
  double c1, c2;
  const uint8_t* A1;  // graph-1 adjacency (roles)
  const uint8_t* A2;  // graph-2 adjacency (vertices)
  double operator()(int a, int b) const {
    if (a == b) return -2.0 * c1;
    const int u = a / n, i = a % n, v = b / n, j = b % n;
    if ((u == v) != (i == j)) return 2.0 * c1;
    // here u != v and i != j (a != b)
    return A1[size_t(i) * n + j] != A2[size_t(u) * n + v] ? c2 : 0.0;
  }
};

}  // namespace

QuboModel build_gi_qubo(const GiInstance& inst) {
  const int n = inst.graph1.n_nodes;
  if (n != inst.graph2.n_nodes) throw std::invalid_argument("GI graphs differ in node count");
  check_penalties(inst.c1, inst.c2);
  const std::vector<uint8_t> a1 = adjacency(inst.graph1), a2 = adjacency(inst.graph2);
  const GiPenalty Q{n, inst.c1, inst.c2, a1.data(), a2.data()};
  const int N = n * n;
  QuboModel q(N, 2.0 * inst.c1 * n);
  for (int a = 0; a < N; ++a)
    for (int b = a; b < N; ++b) {
      const double v = Q(a, b);
      if (v != 0.0) q.set_coeff(a, b, v);
    }
  return q;
}

// The Ising model of the GI penalty straight from the adjacency matrices
// (no N x N QUBO): same values and accumulation order as
// qubo_to_ising(build_gi_qubo(inst)).  h, J (N x N, mirrored), offset.
void gi_ising_arrays(const GiInstance& inst, double* h, double* J, double* offset) {
  const int n = inst.graph1.n_nodes;
  if (n != inst.graph2.n_nodes) throw std::invalid_argument("GI graphs differ in node count");
  check_penalties(inst.c1, inst.c2);
  const std::vector<uint8_t> a1 = adjacency(inst.graph1), a2 = adjacency(inst.graph2);
  const GiPenalty Q{n, inst.c1, inst.c2, a1.data(), a2.data()};
  const int N = n * n;
  std::fill(J, J + size_t(N) * N, 0.0);
  double off = 2.0 * inst.c1 * n;
  for (int a = 0; a < N; ++a) {
    const double qd = Q(a, a);
    double ha = -0.5 * qd;
    off += 0.5 * qd;
    double* row = J + size_t(a) * N;
    for (int b = 0; b < N; ++b) {
      if (b == a) continue;
      const double v = Q(a, b);
      if (v == 0.0) continue;
      ha -= 0.25 * v;
      row[b] = -0.25 * v;
      if (b > a) off += 0.25 * v;
    }
    h[a] = ha;
  }
  *offset = off;
}

// The pair of generate_gi as two 0/1 adjacency matrices (0-based, n x n,
// graph 1 then graph 2) and the Ising biases / offset of its penalty in
// closed form: with deg1 / deg2 the vertex degrees and m = |E1| = |E2|,
//   h_(u,i) = c1 - c1 (n-1) - c2/4 [deg2(u)(n-1-deg1(i)) + (n-1-deg2(u)) deg1(i)]
//   offset  = 2 c1 n - c1 n^2 + c1 n^2 (n-1) / 2 + c2/4 M,
//   M = m (n(n-1) - 2m) + (n(n-1)/2 - m) 2m   (edge-mismatch pairs a < b).
// Exact (hence equal to the reference's accumulation) whenever c1 and c2 are
// dyadic, the only case the engine accepts; the device generator
// (ssqa_problem_create_gi) builds J' from the same adjacency matrices.
void gi_compact(const GiInstance& inst, uint8_t* adj, double* h, double* offset) {
  const int n = inst.graph1.n_nodes;
  const std::vector<uint8_t> a1 = adjacency(inst.graph1), a2 = adjacency(inst.graph2);
  std::copy(a1.begin(), a1.end(), adj);
  std::copy(a2.begin(), a2.end(), adj + size_t(n) * n);
  std::vector<int> d1(size_t(n), 0), d2(size_t(n), 0);
  for (int x = 0; x < n; ++x)
    for (int y = 0; y < n; ++y) {
      d1[size_t(x)] += a1[size_t(x) * n + y];
      d2[size_t(x)] += a2[size_t(x) * n + y];
    }
  const double c1 = inst.c1, c2 = inst.c2;
  for (int u = 0; u < n; ++u)
    for (int i = 0; i < n; ++i) {
      const long mis = long(d2[size_t(u)]) * (n - 1 - d1[size_t(i)]) +
                       long(n - 1 - d2[size_t(u)]) * d1[size_t(i)];
      h[size_t(u) * n + i] = c1 - c1 * double(n - 1) - 0.25 * c2 * double(mis);
    }
  const double m = double(inst.graph1.edges.size());
  const double nn1 = double(n) * double(n - 1);
  const double M = m * (nn1 - 2.0 * m) + (nn1 / 2.0 - m) * 2.0 * m;
  *offset = 2.0 * c1 * n - c1 * double(n) * n + c1 * double(n) * n * (n - 1) / 2.0 + 0.25 * c2 * M;
}

}  // namespace ssqa
