// ref_adapter.cpp -- TEST INFRASTRUCTURE ONLY (see oracle_api.h).
//
// Exposes the unmodified reference library (compiled from
// /root/reference/proj/src with -Dssqa=ssqa_ref) through a plain C ABI so
// the pytest suite and bench.py's reference arm can drive it with ctypes.
// Nothing here re-implements reference logic: every call forwards to the
// reference function named in its comment.
#include <chrono>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ssqa/annealer.hpp"
#include "ssqa/bench.hpp"
#include "ssqa/gi.hpp"
#include "ssqa/model.hpp"
#include "ssqa/rng.hpp"

#include "oracle_api.h"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

ssqa_ref::IsingModel make_model(int n, const double* h, const double* J, double offset) {
  ssqa_ref::IsingModel m(n, offset);
  for (int i = 0; i < n; ++i) {
    m.set_bias(i, h[i]);
    for (int j = i + 1; j < n; ++j) m.set_coupling(i, j, J[size_t(i) * n + j]);
  }
  return m;
}

ssqa_ref::SsqaParams make_params(const orc_ssqa_params* p) {
  ssqa_ref::SsqaParams q;
  q.r = p->r;
  q.jperp_min = p->jperp_min;
  q.jperp_max = p->jperp_max;
  q.beta = p->beta;
  q.tau = p->tau;
  q.delay = p->delay;
  q.i0 = p->i0;
  q.n_rnd = p->n_rnd;
  q.alpha = p->alpha;
  q.sc = p->sc;
  q.bidirectional = p->bidirectional != 0;
  return q;
}

ssqa_ref::SsaParams make_ssa(const orc_ssa_params* p) {
  ssqa_ref::SsaParams q;
  q.i0_min = p->i0_min;
  q.i0_max = p->i0_max;
  q.beta = p->beta;
  q.tau = p->tau;
  q.n_rnd = p->n_rnd;
  q.alpha = p->alpha;
  q.sc = p->sc;
  return q;
}

void load_lattice(ssqa_ref::ReplicaLattice& lat, int n, int r, int d, const double* sigma,
                  const double* acc, const double* hist, long cycle) {
  const size_t nr = size_t(n) * r;
  lat.n = n;
  lat.replicas = r;
  lat.delay = d;
  lat.cycle = cycle;
  lat.sigma.assign(sigma, sigma + nr);
  lat.is_acc.assign(acc, acc + nr);
  lat.history.assign(size_t(d) + 1, {});
  for (int s = 0; s <= d; ++s) lat.history[s].assign(hist + s * nr, hist + (s + 1) * nr);
}

void store_lattice(const ssqa_ref::ReplicaLattice& lat, double* sigma, double* acc,
                   double* hist) {
  const size_t nr = lat.sigma.size();
  std::memcpy(sigma, lat.sigma.data(), nr * sizeof(double));
  std::memcpy(acc, lat.is_acc.data(), nr * sizeof(double));
  for (size_t s = 0; s < lat.history.size(); ++s)
    std::memcpy(hist + s * nr, lat.history[s].data(), nr * sizeof(double));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// rng.hpp:10-15
uint64_t ref_mix64(uint64_t x) { return ssqa_ref::mix64(x); }
// rng.hpp:33-34
uint64_t ref_rng_key(uint64_t seed, uint32_t stream) {
  return ssqa_ref::CounterRng(seed, stream).key();
}
// rng.hpp:36-38
uint64_t ref_rng_raw(uint64_t seed, uint32_t stream, uint64_t counter) {
  return ssqa_ref::CounterRng(seed, stream).raw(counter);
}
// rng.hpp:41-43
double ref_rng_uniform01(uint64_t seed, uint32_t stream, uint64_t counter) {
  return ssqa_ref::CounterRng(seed, stream).uniform01(counter);
}
// rng.hpp:65-67
uint64_t ref_spin_counter(uint64_t cycle, int replica, int spin) {
  return ssqa_ref::spin_counter(cycle, replica, spin);
}

// annealer.cpp:375-380
int ref_jperp_schedule(long cycle, const orc_ssqa_params* p, double* out) {
  return guarded([&] { *out = ssqa_ref::jperp_schedule(cycle, make_params(p)); });
}

// annealer.cpp:432-447
int ref_init_lattice(int n, int r, int d, uint64_t seed, double* sigma, double* acc,
                     double* hist) {
  return guarded([&] {
    ssqa_ref::ReplicaLattice lat = ssqa_ref::init_lattice(n, r, d, seed);
    store_lattice(lat, sigma, acc, hist);
  });
}

// annealer.cpp:449-463
int ref_ssqa_sweep(int n, const double* h, const double* J, double offset, double jperp,
                   const orc_ssqa_params* p, uint64_t seed, long cycle, double* sigma,
                   double* acc, double* hist, long* lat_cycle) {
  return guarded([&] {
    ssqa_ref::IsingModel m = make_model(n, h, J, offset);
    ssqa_ref::SsqaParams q = make_params(p);
    ssqa_ref::ReplicaLattice lat;
    load_lattice(lat, n, q.r, q.delay, sigma, acc, hist, *lat_cycle);
    ssqa_ref::ssqa_sweep(lat, m, jperp, q, seed, cycle);
    store_lattice(lat, sigma, acc, hist);
    *lat_cycle = lat.cycle;
  });
}

// annealer.cpp:465-472
int ref_replica_energies(int n, const double* h, const double* J, double offset, int r,
                         const double* sigma, double* out) {
  return guarded([&] {
    ssqa_ref::IsingModel m = make_model(n, h, J, offset);
    ssqa_ref::ReplicaLattice lat;
    lat.n = n;
    lat.replicas = r;
    lat.sigma.assign(sigma, sigma + size_t(n) * r);
    auto e = ssqa_ref::replica_energies(lat, m);
    std::memcpy(out, e.data(), e.size() * sizeof(double));
  });
}

// annealer.cpp:474-487 (ssqa_run -> run_lattice 313-361)
int ref_ssqa_run(int n, const double* h, const double* J, double offset,
                 const orc_ssqa_params* p, uint64_t seed, int has_target, double target,
                 int record_trace, int stop_at_target, orc_result* out, int8_t* best_state,
                 double* trace_energy) {
  return guarded([&] {
    ssqa_ref::IsingModel m = make_model(n, h, J, offset);
    ssqa_ref::RunOptions opts;
    opts.record_trace = record_trace != 0;
    opts.stop_at_target = stop_at_target != 0;
    std::optional<double> tgt;
    if (has_target) tgt = target;
    ssqa_ref::AnnealResult res = ssqa_ref::ssqa_run(m, make_params(p), seed, tgt, opts);
    out->best_energy = res.best_energy;
    out->best_replica = res.best_replica;
    out->reached_target = res.reached_target;
    out->first_hit_cycle = res.first_hit_cycle;
    out->cycles_used = res.cycles_used;
    out->trace_len = long(res.trace.size());
    out->wall_seconds = res.wall_seconds;
    if (best_state) {
      for (size_t i = 0; i < res.best_state.size(); ++i) best_state[i] = res.best_state[i];
    }
    if (trace_energy) {
      for (size_t i = 0; i < res.trace.size(); ++i) trace_energy[i] = res.trace[i].energy;
    }
  });
}

// annealer.cpp:403-408
int ref_i0_schedule(long cycle, const orc_ssa_params* p, double* out) {
  return guarded([&] { *out = ssqa_ref::i0_schedule(cycle, make_ssa(p)); });
}

// annealer.cpp:489-501 (ssa_run -> run_lattice)
int ref_ssa_run(int n, const double* h, const double* J, double offset, const orc_ssa_params* p,
                uint64_t seed, int has_target, double target, int record_trace,
                int stop_at_target, orc_result* out, int8_t* best_state, double* trace_energy) {
  return guarded([&] {
    ssqa_ref::IsingModel m = make_model(n, h, J, offset);
    ssqa_ref::RunOptions opts;
    opts.record_trace = record_trace != 0;
    opts.stop_at_target = stop_at_target != 0;
    std::optional<double> tgt;
    if (has_target) tgt = target;
    ssqa_ref::AnnealResult res = ssqa_ref::ssa_run(m, make_ssa(p), seed, tgt, opts);
    out->best_energy = res.best_energy;
    out->best_replica = res.best_replica;
    out->reached_target = res.reached_target;
    out->first_hit_cycle = res.first_hit_cycle;
    out->cycles_used = res.cycles_used;
    out->trace_len = long(res.trace.size());
    out->wall_seconds = res.wall_seconds;
    if (best_state)
      for (size_t i = 0; i < res.best_state.size(); ++i) best_state[i] = res.best_state[i];
    if (trace_energy)
      for (size_t i = 0; i < res.trace.size(); ++i) trace_energy[i] = res.trace[i].energy;
  });
}

// ssqa_run (annealer.cpp:474-487) for every seed on `workers` threads over ONE
// shared model (as run_trials shares its problem, bench.cpp:365-407); used by
// bench.py's CPU baseline for the dense configs, whose model is too large
// to rebuild per call.  best_energy[t] receives each trial's best energy.
int ref_ssqa_run_many(int n, const double* h, const double* J, double offset,
                      const orc_ssqa_params* p, const uint64_t* seeds, int trials, int workers,
                      double* best_energy) {
  return guarded([&] {
    const ssqa_ref::IsingModel m = make_model(n, h, J, offset);
    const ssqa_ref::SsqaParams q = make_params(p);
    ssqa_ref::RunOptions opts;
    opts.record_trace = false;
    opts.stop_at_target = false;
    std::vector<std::thread> th;
    std::vector<std::string> errs(size_t(std::max(1, workers)));
    for (int w = 0; w < std::max(1, workers); ++w)
      th.emplace_back([&, w] {
        try {
          for (int t = w; t < trials; t += std::max(1, workers))
            best_energy[t] = ssqa_ref::ssqa_run(m, q, seeds[t], {}, opts).best_energy;
        } catch (const std::exception& e) {
          errs[size_t(w)] = e.what();
        }
      });
    for (auto& x : th) x.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// gi.cpp:102-184 + model.cpp:139-161
int ref_gi_ising(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                 double c2, double* h, double* J, double* offset) {
  return guarded([&] {
    ssqa_ref::GiInstance inst =
        ssqa_ref::generate_gi(n_nodes, edge_prob, seed, permute != 0, c1, c2);
    ssqa_ref::IsingModel m = ssqa_ref::qubo_to_ising(ssqa_ref::build_gi_qubo(inst));
    const int n = m.n();
    for (int i = 0; i < n; ++i) {
      h[i] = m.bias(i);
      std::memcpy(J + size_t(i) * n, m.coupling_row(i), size_t(n) * sizeof(double));
    }
    *offset = m.offset();
  });
}

// bench.cpp:359-432
int ref_run_trials(const orc_ssqa_params* p, int n_nodes, double edge_prob, int permute,
                   double c1, double c2, int fresh_instance, uint64_t gi_seed, int trials,
                   long ec, double p_target, uint64_t base_seed, int workers,
                   orc_trial* outcomes, double* p_s, double* t_mean, double* tts_seconds,
                   int* tts_kind) {
  return guarded([&] {
    ssqa_ref::BenchConfig cfg;
    cfg.engine = ssqa_ref::Engine::kSsqa;
    cfg.ssqa = make_params(p);
    cfg.problem.n_nodes = n_nodes;
    cfg.problem.edge_prob = edge_prob;
    cfg.problem.permute = permute != 0;
    cfg.problem.c1 = c1;
    cfg.problem.c2 = c2;
    cfg.problem.fresh_instance = fresh_instance != 0;
    cfg.problem.gi_seed = gi_seed;
    cfg.trials = trials;
    cfg.ec = ec;
    cfg.p_target = p_target;
    cfg.base_seed = base_seed;
    cfg.workers = workers;
    ssqa_ref::BenchRecord rec = ssqa_ref::run_trials(cfg);
    for (size_t t = 0; t < rec.per_trial.size(); ++t) {
      outcomes[t].seed = rec.per_trial[t].seed;
      outcomes[t].reached_target = rec.per_trial[t].reached_target;
      outcomes[t].first_hit_cycle = rec.per_trial[t].first_hit_cycle;
      outcomes[t].best_energy = rec.per_trial[t].best_energy;
      outcomes[t].wall_seconds = rec.per_trial[t].wall_seconds;
    }
    *p_s = rec.p_s;
    *t_mean = rec.t_mean_s;
    *tts_seconds = rec.tts.seconds;
    *tts_kind = int(rec.tts.kind);
  });
}

// make_manifest("bench", ...) of a run_trials (bench.cpp:519-531) serialised
// to `buf` (manifest replay fixture for the facade's replay_manifest).
long ref_bench_manifest(const orc_ssqa_params* p, int n_nodes, double edge_prob, int permute,
                        double c1, double c2, int fresh_instance, uint64_t gi_seed, int trials,
                        long ec, double p_target, uint64_t base_seed, int workers, char* buf,
                        long cap) {
  long len = -1;
  int rc = guarded([&] {
    ssqa_ref::BenchConfig cfg;
    cfg.engine = ssqa_ref::Engine::kSsqa;
    cfg.ssqa = make_params(p);
    cfg.problem.n_nodes = n_nodes;
    cfg.problem.edge_prob = edge_prob;
    cfg.problem.permute = permute != 0;
    cfg.problem.c1 = c1;
    cfg.problem.c2 = c2;
    cfg.problem.fresh_instance = fresh_instance != 0;
    cfg.problem.gi_seed = gi_seed;
    cfg.trials = trials;
    cfg.ec = ec;
    cfg.p_target = p_target;
    cfg.base_seed = base_seed;
    cfg.workers = workers;
    ssqa_ref::BenchRecord rec = ssqa_ref::run_trials(cfg);
    const std::string js = ssqa_ref::make_manifest("bench", cfg, {}, {rec}, {}).dump(1);
    len = long(js.size());
    if (len + 1 > cap) throw std::runtime_error("buffer too small");
    std::memcpy(buf, js.c_str(), size_t(len) + 1);
  });
  return rc ? -1 : len;
}

}  // extern "C"
