// host/annealer.cpp -- the reference annealer API (ssqa/annealer.hpp) on top
// of the C ABI (include/ssqa_cuda.h).  The facade owns no numerics: it
// converts types, forwards to the device engine and turns error codes back
// into the reference's exceptions (annealer.cpp:25-30, 365-373).
#include "ssqa/annealer.hpp"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <memory>
#include <stdexcept>
#include <string>

#include "ssqa_cuda.h"
#include "engine.h"

namespace ssqa {

namespace {

ssqa_params_c to_c(const SsqaParams& p) {
  ssqa_params_c c{};
  c.r = p.r;
  c.jperp_min = p.jperp_min;
  c.jperp_max = p.jperp_max;
  c.beta = p.beta;
  c.tau = p.tau;
  c.delay = p.delay;
  c.i0 = p.i0;
  c.n_rnd = p.n_rnd;
  c.alpha = p.alpha;
  c.sc = p.sc;
  c.bidirectional = p.bidirectional ? 1 : 0;
  return c;
}

ssqa_ssa_params_c to_c(const SsaParams& p) {
  ssqa_ssa_params_c c{};
  c.i0_min = p.i0_min;
  c.i0_max = p.i0_max;
  c.beta = p.beta;
  c.tau = p.tau;
  c.n_rnd = p.n_rnd;
  c.alpha = p.alpha;
  c.sc = p.sc;
  return c;
}

void check(int rc) {
  if (rc == SSQA_OK) return;
  const std::string msg = ssqa_last_error();
  if (rc == SSQA_EINVAL || rc == SSQA_EUNSUP) throw std::invalid_argument(msg);
  if (rc == SSQA_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

struct ProblemHandle {
  ssqa_problem p = nullptr;
  ~ProblemHandle() { ssqa_problem_destroy(p); }
};
struct BatchHandle {
  ssqa_batch b = nullptr;
  ~BatchHandle() { ssqa_batch_destroy(b); }
};

void upload(const IsingModel& m, int device, ProblemHandle& h) {
  check(ssqa_problem_create(m.n(), m.biases().data(), m.coupling_data(), m.offset(), device,
                            &h.p));
}

// One problem holding every model (one per trial): ssqa_problem_create_many.
void upload_many(const std::vector<IsingModel>& ms, int device, ProblemHandle& h) {
  if (ms.empty()) throw std::invalid_argument("no models");
  const int n = ms.front().n();
  std::vector<double> hs, js, offs;
  hs.reserve(ms.size() * size_t(n));
  js.reserve(ms.size() * size_t(n) * n);
  for (const IsingModel& m : ms) {
    if (m.n() != n) throw std::invalid_argument("instances must have the same size");
    hs.insert(hs.end(), m.biases().begin(), m.biases().end());
    js.insert(js.end(), m.coupling_data(), m.coupling_data() + size_t(n) * n);
    offs.push_back(m.offset());
  }
  check(ssqa_problem_create_many(int(ms.size()), n, hs.data(), js.data(), offs.data(), device,
                                 &h.p));
}

// A one-trial batch carrying an explicit lattice (per-step API).
void load(BatchHandle& bh, ProblemHandle& ph, const ReplicaLattice& lat, SsqaParams p,
          uint64_t seed) {
  if (p.sc < 1) p.sc = 1;  // the per-step API never reads sc
  ssqa_params_c c = to_c(p);
  check(ssqa_batch_create(ph.p, &c, 1, 0, SSQA_ENGINE_AUTO, &bh.b));
  check(ssqa_batch_set_seeds(bh.b, &seed));
  std::vector<double> hist;
  for (const auto& h : lat.history) hist.insert(hist.end(), h.begin(), h.end());
  std::vector<double> acc = lat.is_acc;
  if (acc.empty()) acc.assign(lat.sigma.size(), 0.0);
  if (hist.empty())
    for (int s = 0; s <= p.delay; ++s) hist.insert(hist.end(), lat.sigma.begin(), lat.sigma.end());
  check(ssqa_batch_write_lattice(bh.b, 0, lat.sigma.data(), acc.data(), hist.data(), lat.cycle));
}

}  // namespace

void SsqaParams::validate(int n) const {
  ssqa_params_c c = to_c(*this);
  check(ssqa_params_validate(&c, n));
}

double jperp_schedule(long cycle, const SsqaParams& p) {
  ssqa_params_c c = to_c(p);
  double v = 0.0;
  check(ssqa_jperp_schedule(cycle, &c, &v));
  return v;
}

const std::vector<double>& ReplicaLattice::delayed_sigma() const {
  return history[size_t(cycle % (delay + 1))];
}

ReplicaLattice init_lattice(int n, int replicas, int delay, uint64_t seed) {
  // The device init kernel needs a problem handle; an all-zero n-spin problem
  // made on the device does (no host model, no upload).
  if (n < 1) throw std::invalid_argument("init_lattice needs n >= 1");
  ProblemHandle ph;
  check(ssqa_problem_create_zero(n, 0, &ph.p));
  SsqaParams p;
  p.r = replicas;
  p.delay = delay;
  p.sc = 1;
  ssqa_params_c c = to_c(p);
  BatchHandle bh;
  check(ssqa_batch_create(ph.p, &c, 1, 0, SSQA_ENGINE_AUTO, &bh.b));
  check(ssqa_batch_set_seeds(bh.b, &seed));
  check(ssqa_batch_init(bh.b));
  ReplicaLattice lat;
  lat.n = n;
  lat.replicas = replicas;
  lat.delay = delay;
  const size_t nr = size_t(n) * replicas;
  lat.sigma.resize(nr);
  lat.is_acc.resize(nr);
  std::vector<double> hist((size_t(delay) + 1) * nr);
  check(ssqa_batch_read_lattice(bh.b, 0, lat.sigma.data(), lat.is_acc.data(), hist.data(),
                                &lat.cycle));
  for (int s = 0; s <= delay; ++s)
    lat.history.emplace_back(hist.begin() + s * nr, hist.begin() + (s + 1) * nr);
  return lat;
}

void ssqa_sweep(ReplicaLattice& lat, const IsingModel& m, double jperp, const SsqaParams& p,
                uint64_t seed, long cycle) {
  if (lat.n != m.n() || lat.replicas != p.r)
    throw std::invalid_argument("lattice dimensions do not match model/params");
  if (cycle != lat.cycle) throw std::invalid_argument("sweep cycle does not match lattice history");
  ProblemHandle ph;
  upload(m, 0, ph);
  BatchHandle bh;
  load(bh, ph, lat, p, seed);
  check(ssqa_batch_sweep_with(bh.b, jperp, p.i0));
  const size_t nr = lat.sigma.size();
  std::vector<double> hist((size_t(lat.delay) + 1) * nr);
  lat.is_acc.resize(nr);
  check(ssqa_batch_read_lattice(bh.b, 0, lat.sigma.data(), lat.is_acc.data(), hist.data(),
                                &lat.cycle));
  lat.history.assign(size_t(lat.delay) + 1, {});
  for (int s = 0; s <= lat.delay; ++s)
    lat.history[size_t(s)].assign(hist.begin() + s * nr, hist.begin() + (s + 1) * nr);
}

std::vector<double> replica_energies(const ReplicaLattice& lat, const IsingModel& m) {
  if (lat.n != m.n()) throw std::invalid_argument("lattice does not match model");
  ProblemHandle ph;
  upload(m, 0, ph);
  SsqaParams p;
  p.r = lat.replicas;
  p.delay = 0;
  ReplicaLattice flat = lat;
  flat.delay = 0;
  flat.history.clear();
  flat.cycle = 0;
  BatchHandle bh;
  load(bh, ph, flat, p, 0);
  std::vector<double> e(size_t(lat.replicas));
  check(ssqa_batch_energies(bh.b, e.data()));
  return e;
}

namespace {

// Batch outputs -> AnnealResult (trace rows carry `r` energies per cycle and
// the jperp the reference records with them, annealer.cpp:343).
template <class JperpAt>
std::vector<AnnealResult> to_results(int T, int n, int r, long sc,
                                     const std::vector<ssqa_result_c>& res,
                                     const std::vector<int8_t>& best,
                                     const std::vector<double>& trace, bool record_trace,
                                     JperpAt jperp_at) {
  std::vector<AnnealResult> out(static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) {
    AnnealResult& a = out[size_t(t)];
    a.best_energy = res[size_t(t)].best_energy;
    a.best_replica = res[size_t(t)].best_replica;
    a.reached_target = res[size_t(t)].reached_target != 0;
    a.first_hit_cycle = res[size_t(t)].first_hit_cycle;
    a.cycles_used = res[size_t(t)].cycles_used;
    a.wall_seconds = res[size_t(t)].wall_seconds;
    a.best_state.assign(best.begin() + size_t(t) * n, best.begin() + size_t(t + 1) * n);
    if (record_trace) {
      const double* tr = trace.data() + size_t(t) * (sc + 1) * r;
      for (long cyc = 0; cyc <= a.cycles_used; ++cyc) {
        const double jp = jperp_at(cyc);
        for (int k = 0; k < r; ++k) a.trace.push_back({cyc, k, tr[size_t(cyc) * r + k], jp});
      }
    }
  }
  return out;
}

}  // namespace

std::vector<AnnealResult> ssqa_run_batch(const IsingModel& m, const SsqaParams& p,
                                         const std::vector<uint64_t>& seeds,
                                         std::optional<double> target_energy,
                                         const RunOptions& opts, const EngineOptions& eng) {
  p.validate(m.n());
  if (seeds.empty()) return {};
  ProblemHandle ph;
  upload(m, eng.device, ph);
  const int T = int(seeds.size());
  ssqa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * m.n());
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1) * p.r);
  check(ssqa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                       target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                       opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                       opts.record_trace ? trace.data() : nullptr));
  return to_results(T, m.n(), p.r, p.sc, res, best, trace, opts.record_trace,
                    [&p](long c) { return jperp_schedule(c, p); });
}

AnnealResult ssqa_run(const IsingModel& m, const SsqaParams& p, uint64_t seed,
                      std::optional<double> target_energy, const RunOptions& opts) {
  return ssqa_run_batch(m, p, {seed}, target_energy, opts).front();
}

// ---- J' row shards over several GPUs, driven from one host thread ----------
// (the Python driver is paper_2302_12454_b200/rowshard.py.)
// NCCL is bound at run time (dlopen of libnccl.so.2): the engine library has
// no link-time dependency on it and single-GPU callers never load it.
namespace {

struct Nccl {
  using Comm = void*;
  int (*CommInitAll)(Comm*, int, const int*) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  static constexpr int kUint8 = 1;  // ncclUint8

  static Nccl& get() {
    static Nccl n = [] {
      Nccl x;
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!h) throw std::runtime_error(std::string("NCCL not found: ") + dlerror());
      auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + name);
        return p;
      };
      x.CommInitAll = reinterpret_cast<decltype(x.CommInitAll)>(sym("ncclCommInitAll"));
      x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
      x.AllGather = reinterpret_cast<decltype(x.AllGather)>(sym("ncclAllGather"));
      x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
      x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
      x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(sym("ncclGetErrorString"));
      return x;
    }();
    return n;
  }
  void ok(int rc) const {
    if (rc != 0) throw std::runtime_error(std::string("NCCL: ") + GetErrorString(rc));
  }
};

void cuda_ok(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace

std::vector<AnnealResult> ssqa_run_row_sharded(const IsingModel& m, const SsqaParams& p,
                                               const std::vector<uint64_t>& seeds,
                                               const std::vector<int>& devices,
                                               std::optional<double> target_energy,
                                               const RunOptions& opts, RowShardExchange exchange) {
  p.validate(m.n());
  if (seeds.empty()) return {};
  if (devices.empty()) throw std::invalid_argument("ssqa_run_row_sharded: no devices");
  const int G = int(devices.size()), T = int(seeds.size());
  struct Shard {
    ProblemHandle ph;
    BatchHandle bh;
    void* buf = nullptr;  // two halves (cycle parity) of G chunks in shard order
    cudaEvent_t packed[2] = {nullptr, nullptr};  // this shard's chunk of that parity is written
    cudaStream_t stream = nullptr;
    int device = 0;
    ~Shard() {
      cudaSetDevice(device);
      for (cudaEvent_t e : packed)
        if (e) cudaEventDestroy(e);
      if (buf) cudaFree(buf);
    }
  };
  std::vector<Shard> sh(static_cast<size_t>(G));
  const ssqa_params_c c = to_c(p);
  size_t nb = 0;
  for (int g = 0; g < G; ++g) {
    Shard& s = sh[size_t(g)];
    s.device = devices[size_t(g)];
    upload(m, s.device, s.ph);
    check(ssqa_batch_create(s.ph.p, &c, T, opts.record_trace ? 1 : 0, SSQA_ENGINE_TCGEN05,
                            &s.bh.b));
    check(ssqa_batch_set_shard(s.bh.b, g, G));
    check(ssqa_batch_set_seeds(s.bh.b, seeds.data()));
    nb = size_t(ssqa_batch_shard_bytes(s.bh.b));
    s.stream = static_cast<cudaStream_t>(ssqa_batch_stream(s.bh.b));
    cuda_ok(cudaSetDevice(s.device));
    cuda_ok(cudaMalloc(&s.buf, 2 * nb * size_t(G)));
    for (cudaEvent_t& e : s.packed) cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // NCCL needs distinct devices; a device listed twice (several shards on one
  // GPU, e.g. to check the sharding on a single-GPU box) takes the copy
  // exchange below, which is also what `exchange` = kPeerCopy asks for
  bool distinct = true;
  for (int g = 0; g < G; ++g)
    for (int h = 0; h < g; ++h) distinct = distinct && devices[size_t(g)] != devices[size_t(h)];
  const bool use_nccl = (G > 1 || ssqa_engine::tune().nccl1 > 0) && distinct &&
                        exchange == RowShardExchange::kNccl;
  std::vector<Nccl::Comm> comms(static_cast<size_t>(G), nullptr);
  const Nccl* nccl = nullptr;
  if (use_nccl) {
    nccl = &Nccl::get();
    nccl->ok(nccl->CommInitAll(comms.data(), G, devices.data()));
  }
  auto destroy_comms = [&] {
    if (nccl)
      for (Nccl::Comm cm : comms)
        if (cm) nccl->CommDestroy(cm);
  };
  try {
    for (Shard& s : sh)
      check(ssqa_batch_shard_begin(s.bh.b, target_energy ? 1 : 0, target_energy.value_or(0.0),
                                   opts.stop_at_target ? 1 : 0));
    for (long cyc = 0; cyc <= p.sc; ++cyc) {
      // Chunks alternate between two halves by cycle parity: a GPU rewrites
      // its chunk of a half two cycles later, after its merge of the cycle
      // in between, which needed every peer's next chunk -- sent only after
      // that peer had merged (and so read or received) this one.
      const int par = int(cyc & 1);
      auto half = [&](Shard& s) { return static_cast<char*>(s.buf) + size_t(par) * nb * size_t(G); };
      // pass: each GPU updates its rows and packs them into its own chunk
      for (int g = 0; g < G; ++g) {
        Shard& s = sh[size_t(g)];
        check(ssqa_batch_shard_pass(s.bh.b, half(s) + size_t(g) * nb));
        if (G > 1 && !use_nccl) {
          cuda_ok(cudaSetDevice(s.device));
          cuda_ok(cudaEventRecord(s.packed[par], s.stream));
        }
      }
      if (use_nccl) {
        // in-place all-gather of the chunks, ordered on each engine stream
        nccl->ok(nccl->GroupStart());
        for (int g = 0; g < G; ++g) {
          Shard& s = sh[size_t(g)];
          nccl->ok(nccl->AllGather(half(s) + size_t(g) * nb, half(s), nb, Nccl::kUint8,
                                   comms[size_t(g)], s.stream));
        }
        nccl->ok(nccl->GroupEnd());
      } else if (G > 1) {
        // copy exchange: every GPU pulls the peers' chunks on its own stream
        // once they are packed (cudaMemcpyPeerAsync over NVLink)
        for (int g = 0; g < G; ++g) {
          Shard& d = sh[size_t(g)];
          cuda_ok(cudaSetDevice(d.device));
          for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            Shard& src = sh[size_t(h)];
            cuda_ok(cudaStreamWaitEvent(d.stream, src.packed[par], 0));
            cuda_ok(cudaMemcpyPeerAsync(half(d) + size_t(h) * nb, d.device,
                                        half(src) + size_t(h) * nb, src.device, nb, d.stream));
          }
        }
      }
      for (Shard& s : sh) check(ssqa_batch_shard_merge(s.bh.b, half(s)));
    }
    for (Shard& s : sh) check(ssqa_batch_shard_end(s.bh.b));
  } catch (...) {
    destroy_comms();
    throw;
  }
  // identical results on every GPU: read shard 0's
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * m.n());
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1) * p.r);
  for (size_t g = 1; g < sh.size(); ++g) check(ssqa_batch_synchronize(sh[g].bh.b));
  check(ssqa_batch_fetch(sh[0].bh.b, res.data(), best.data(),
                         opts.record_trace ? trace.data() : nullptr));
  destroy_comms();
  return to_results(T, m.n(), p.r, p.sc, res, best, trace, opts.record_trace,
                    [&p](long cy) { return jperp_schedule(cy, p); });
}

std::vector<AnnealResult> ssqa_run_instances(const std::vector<IsingModel>& models,
                                             const SsqaParams& p,
                                             const std::vector<uint64_t>& seeds,
                                             std::optional<double> target_energy,
                                             const RunOptions& opts, const EngineOptions& eng) {
  if (models.size() != seeds.size()) throw std::invalid_argument("one model per seed");
  if (seeds.empty()) return {};
  const int n = models.front().n();
  p.validate(n);
  ProblemHandle ph;
  upload_many(models, eng.device, ph);
  const int T = int(seeds.size());
  ssqa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * n);
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1) * p.r);
  check(ssqa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                       target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                       opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                       opts.record_trace ? trace.data() : nullptr));
  return to_results(T, n, p.r, p.sc, res, best, trace, opts.record_trace,
                    [&p](long c) { return jperp_schedule(c, p); });
}

std::vector<AnnealResult> ssqa_run_gi_instances(int n_nodes, double edge_prob, bool permute,
                                                double c1, double c2,
                                                const std::vector<uint64_t>& instance_seeds,
                                                const SsqaParams& p,
                                                const std::vector<uint64_t>& seeds,
                                                std::optional<double> target_energy,
                                                const RunOptions& opts, const EngineOptions& eng) {
  if (instance_seeds.size() != seeds.size()) throw std::invalid_argument("one instance per seed");
  if (seeds.empty()) return {};
  const int n = n_nodes * n_nodes;
  p.validate(n);
  ProblemHandle ph;
  check(ssqa_problem_create_gi(int(seeds.size()), n_nodes, edge_prob, instance_seeds.data(),
                               permute ? 1 : 0, c1, c2, eng.device, &ph.p));
  const int T = int(seeds.size());
  ssqa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * n);
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1) * p.r);
  check(ssqa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                       target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                       opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                       opts.record_trace ? trace.data() : nullptr));
  return to_results(T, n, p.r, p.sc, res, best, trace, opts.record_trace,
                    [&p](long c) { return jperp_schedule(c, p); });
}

std::vector<AnnealResult> ssa_run_gi_instances(int n_nodes, double edge_prob, bool permute,
                                               double c1, double c2,
                                               const std::vector<uint64_t>& instance_seeds,
                                               const SsaParams& p,
                                               const std::vector<uint64_t>& seeds,
                                               std::optional<double> target_energy,
                                               const RunOptions& opts, const EngineOptions& eng) {
  if (instance_seeds.size() != seeds.size()) throw std::invalid_argument("one instance per seed");
  if (seeds.empty()) return {};
  const int n = n_nodes * n_nodes;
  p.validate(n);
  ProblemHandle ph;
  check(ssqa_problem_create_gi(int(seeds.size()), n_nodes, edge_prob, instance_seeds.data(),
                               permute ? 1 : 0, c1, c2, eng.device, &ph.p));
  const int T = int(seeds.size());
  ssqa_ssa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * n);
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1));
  check(ssqa_ssa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                           target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                           opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                           opts.record_trace ? trace.data() : nullptr));
  return to_results(T, n, 1, p.sc, res, best, trace, opts.record_trace,
                    [](long) { return 0.0; });
}

std::vector<double> SsaParams::i0_levels() const {
  ssqa_ssa_params_c c = to_c(*this);
  double buf[65];
  int count = 0;
  check(ssqa_i0_levels(&c, buf, &count));
  return std::vector<double>(buf, buf + count);
}

long SsaParams::cycles_per_iteration() const { return long(i0_levels().size()) * tau; }

void SsaParams::validate(int n) const {
  ssqa_ssa_params_c c = to_c(*this);
  check(ssqa_ssa_params_validate(&c, n));
}

double i0_schedule(long cycle, const SsaParams& p) {
  ssqa_ssa_params_c c = to_c(p);
  double v = 0.0;
  check(ssqa_i0_schedule(cycle, &c, &v));
  return v;
}

std::vector<AnnealResult> ssa_run_batch(const IsingModel& m, const SsaParams& p,
                                        const std::vector<uint64_t>& seeds,
                                        std::optional<double> target_energy,
                                        const RunOptions& opts, const EngineOptions& eng) {
  p.validate(m.n());
  if (seeds.empty()) return {};
  ProblemHandle ph;
  upload(m, eng.device, ph);
  const int T = int(seeds.size());
  ssqa_ssa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * m.n());
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1));
  check(ssqa_ssa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                           target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                           opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                           opts.record_trace ? trace.data() : nullptr));
  return to_results(T, m.n(), 1, p.sc, res, best, trace, opts.record_trace,
                    [](long) { return 0.0; });
}

AnnealResult ssa_run(const IsingModel& m, const SsaParams& p, uint64_t seed,
                     std::optional<double> target_energy, const RunOptions& opts) {
  return ssa_run_batch(m, p, {seed}, target_energy, opts).front();
}

std::vector<AnnealResult> ssa_run_instances(const std::vector<IsingModel>& models,
                                            const SsaParams& p,
                                            const std::vector<uint64_t>& seeds,
                                            std::optional<double> target_energy,
                                            const RunOptions& opts, const EngineOptions& eng) {
  if (models.size() != seeds.size()) throw std::invalid_argument("one model per seed");
  if (seeds.empty()) return {};
  const int n = models.front().n();
  p.validate(n);
  ProblemHandle ph;
  upload_many(models, eng.device, ph);
  const int T = int(seeds.size());
  ssqa_ssa_params_c c = to_c(p);
  std::vector<ssqa_result_c> res(seeds.size());
  std::vector<int8_t> best(size_t(T) * n);
  std::vector<double> trace;
  if (opts.record_trace) trace.resize(size_t(T) * (p.sc + 1));
  check(ssqa_ssa_run_batch(ph.p, &c, seeds.data(), T, target_energy ? 1 : 0,
                           target_energy.value_or(0.0), opts.record_trace ? 1 : 0,
                           opts.stop_at_target ? 1 : 0, eng.engine, res.data(), best.data(),
                           opts.record_trace ? trace.data() : nullptr));
  return to_results(T, n, 1, p.sc, res, best, trace, opts.record_trace,
                    [](long) { return 0.0; });
}

}  // namespace ssqa
