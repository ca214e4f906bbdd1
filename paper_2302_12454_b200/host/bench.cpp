// host/bench.cpp -- run_trials / replica_sweep / run_cases (ssqa/bench.hpp)
// over device batches.  Trial semantics follow proj/src/bench.cpp:359-477:
// seeds base_seed + t, fixed budget (stop_at_target = false, 336), sc = ec/r
// (363), GI target 0 (309-313), fresh per-trial instances seeded by
// CounterRng(base_seed, kStreamTrialInstance).raw(t) (373, 388).
#include "ssqa/bench.hpp"

#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <stdexcept>
#include <exception>
#include <thread>

#include "ssqa/gi.hpp"
#include "ssqa/rng.hpp"

namespace ssqa {

namespace {

std::string fmt(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.6g", v);
  return buf;
}

IsingModel gi_model(const ProblemSpec& p, uint64_t seed) {
  const GiInstance inst = generate_gi(p.n_nodes, p.edge_prob, seed, p.permute, p.c1, p.c2);
  const int n = p.n_nodes * p.n_nodes;
  IsingModel m(n);
  std::vector<double> h(static_cast<size_t>(n)), J(static_cast<size_t>(n) * n);
  double off = 0.0;
  gi_ising_arrays(inst, h.data(), J.data(), &off);
  for (int i = 0; i < n; ++i) {
    m.set_bias(i, h[size_t(i)]);
    for (int j = i + 1; j < n; ++j)
      if (J[size_t(i) * n + j] != 0.0) m.set_coupling(i, j, J[size_t(i) * n + j]);
  }
  m.set_offset(off);
  return m;
}

}  // namespace

std::string engine_name(Engine e) {
  switch (e) {
    case Engine::kSsqa: return "ssqa";
    case Engine::kSsa: return "ssa";
    case Engine::kSa: return "sa";
  }
  throw std::logic_error("bad engine enum");
}

Engine engine_from_name(const std::string& name) {
  if (name == "ssqa") return Engine::kSsqa;
  if (name == "ssa") return Engine::kSsa;
  if (name == "sa") return Engine::kSa;
  throw std::invalid_argument("unknown engine '" + name + "' (ssqa|ssa|sa)");
}

void ProblemSpec::validate() const {
  const bool gi = n_nodes > 0, file = !model_file.empty();
  if (gi == file) throw std::invalid_argument("problem needs exactly one of: GI node count, model file");
  if (gi) {
    if (edge_prob < 0.0 || edge_prob > 1.0) throw std::invalid_argument("edge_prob outside [0, 1]");
    if (c1 <= 0.0 || c2 <= 0.0) throw std::invalid_argument("penalties must be positive");
  }
}

void BenchConfig::validate() const {
  problem.validate();
  if (trials < 1) throw std::invalid_argument("trials must be >= 1");
  if (ec < 1) throw std::invalid_argument("ec must be >= 1");
  if (p_target <= 0.0 || p_target >= 1.0) throw std::invalid_argument("p_target must lie in (0, 1)");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (engine == Engine::kSsqa) {
    if (ssqa.r < 1) throw std::invalid_argument("replica count required (>= 1)");
    if (ec / ssqa.r < 1) throw std::invalid_argument("ec too small for replica count");
  }
}

long compute_ec(int r, long sc) {
  if (r < 1 || sc < 1) throw std::invalid_argument("compute_ec needs r >= 1, sc >= 1");
  return long(r) * sc;
}

double TtsValue::value_or_inf() const {
  if (kind == Kind::kFinite) return seconds;
  if (kind == Kind::kSaturatedZero) return 0.0;
  return std::numeric_limits<double>::infinity();
}

std::string TtsValue::csv_field() const {
  if (kind == Kind::kFinite) return fmt(seconds);
  return kind == Kind::kSaturatedZero ? "0" : "-";
}

// t * ln(1 - p_target) / ln(1 - p_s) (bench.cpp:144-160).
TtsValue compute_tts(double p_s, double t_seconds, double p_target) {
  if (p_target <= 0.0 || p_target >= 1.0) throw std::invalid_argument("p_target must lie in (0, 1)");
  if (p_s < 0.0 || p_s > 1.0) throw std::invalid_argument("p_s outside [0, 1]");
  if (t_seconds <= 0.0) throw std::invalid_argument("t must be > 0");
  TtsValue v;
  if (p_s == 0.0) {
    v.kind = TtsValue::Kind::kUndefined;
  } else if (p_s == 1.0) {
    v.kind = TtsValue::Kind::kSaturatedZero;
  } else {
    v.kind = TtsValue::Kind::kFinite;
    v.seconds = t_seconds * std::log(1.0 - p_target) / std::log(1.0 - p_s);
  }
  return v;
}

BenchRecord run_trials(const BenchConfig& cfg) {
  cfg.validate();
  if (cfg.engine == Engine::kSa)
    throw std::invalid_argument("the B200 engine runs the lattice engines (ssqa, ssa) only");
  const bool ssa = cfg.engine == Engine::kSsa;
  const bool gi = cfg.problem.n_nodes > 0;
  const int r = ssa ? 1 : cfg.ssqa.r;  // bench.cpp:362-363
  const long budget = cfg.ec / r;
  SsqaParams p = cfg.ssqa;
  p.sc = budget;
  SsaParams ps = cfg.ssa;
  ps.sc = budget;
  RunOptions opts;
  opts.stop_at_target = false;
  EngineOptions eng0;
  // run_engine (bench.cpp:332-357) for a set of seeds on one model.
  auto run = [&](const IsingModel& m, const std::vector<uint64_t>& s, double target,
                 const EngineOptions& eng) {
    return ssa ? ssa_run_batch(m, ps, s, target, opts, eng)
               : ssqa_run_batch(m, p, s, target, opts, eng);
  };

  std::vector<uint64_t> seeds(size_t(cfg.trials));
  for (int t = 0; t < cfg.trials; ++t) seeds[size_t(t)] = cfg.base_seed + uint64_t(t);
  if (!gi)
    throw std::invalid_argument(
        "model files are not read by the engine facade: load the model in the caller and "
        "call ssqa_run / the C ABI");
  const int n = cfg.problem.n_nodes * cfg.problem.n_nodes;
  const bool fresh = cfg.problem.fresh_instance;
  const bool device_gi = ssa || (p.r <= 256 && p.delay <= 30);  // tcgen05 shapes
  // Fresh instance per trial (bench.cpp:387-389): seeds CounterRng(base_seed,
  // kStreamTrialInstance).raw(t), every instance built on the device.
  std::vector<uint64_t> inst(size_t(cfg.trials));
  if (fresh) {
    const CounterRng irng(cfg.base_seed, kStreamTrialInstance);
    for (int t = 0; t < cfg.trials; ++t) inst[size_t(t)] = irng.raw(uint64_t(t));
  }
  std::optional<IsingModel> pinned;
  if (!fresh) pinned.emplace(gi_model(cfg.problem, cfg.problem.gi_seed));
  const double target = 0.0;  // GI ground state (bench.cpp:309-313)

  // One block of trials [lo, hi) on one GPU.
  auto block = [&](int lo, int hi, int device) -> std::vector<AnnealResult> {
    EngineOptions eng = eng0;
    eng.device = device;
    const std::vector<uint64_t> s(seeds.begin() + lo, seeds.begin() + hi);
    if (!fresh) return run(*pinned, s, target, eng);
    const std::vector<uint64_t> is(inst.begin() + lo, inst.begin() + hi);
    if (device_gi) {
      const ProblemSpec& ps_ = cfg.problem;
      return ssa ? ssa_run_gi_instances(ps_.n_nodes, ps_.edge_prob, ps_.permute, ps_.c1, ps_.c2,
                                        is, ps, s, target, opts, eng)
                 : ssqa_run_gi_instances(ps_.n_nodes, ps_.edge_prob, ps_.permute, ps_.c1,
                                         ps_.c2, is, p, s, target, opts, eng);
    }
    // shapes only the SIMT engine takes: one device run per instance
    std::vector<AnnealResult> out;
    for (size_t t = 0; t < s.size(); ++t)
      out.push_back(run(gi_model(cfg.problem, is[t]), {s[t]}, target, eng).front());
    return out;
  };

  // GPUs share the battery in contiguous trial blocks, one host thread each
  // (the reference's worker pool over trials, bench.cpp:399-407).
  const std::vector<int> devs = cfg.devices.empty() ? std::vector<int>{cfg.device} : cfg.devices;
  const int G = std::max(1, std::min(int(devs.size()), cfg.trials));
  std::vector<std::vector<AnnealResult>> parts(static_cast<size_t>(G));
  std::vector<std::exception_ptr> errs(static_cast<size_t>(G));
  auto work = [&](int gi_) {
    const int lo = int(int64_t(cfg.trials) * gi_ / G), hi = int(int64_t(cfg.trials) * (gi_ + 1) / G);
    try {
      parts[size_t(gi_)] = block(lo, hi, devs[size_t(gi_)]);
    } catch (...) {
      errs[size_t(gi_)] = std::current_exception();
    }
  };
  if (G == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) th.emplace_back(work, g);
    for (auto& x : th) x.join();
  }
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
  std::vector<AnnealResult> results;
  results.reserve(size_t(cfg.trials));
  for (auto& part : parts)
    for (auto& a : part) results.push_back(std::move(a));
  BenchRecord rec;
  rec.engine = cfg.engine;
  rec.n = n;
  rec.r = r;
  rec.ec = ssa ? cfg.ec : compute_ec(r, budget);  // bench.cpp:414-417
  rec.tau = ssa ? cfg.ssa.tau : cfg.ssqa.tau;
  rec.trials = cfg.trials;
  rec.base_seed = cfg.base_seed;
  int hits = 0;
  double t_sum = 0.0;
  for (int t = 0; t < cfg.trials; ++t) {
    const AnnealResult& a = results[size_t(t)];
    rec.per_trial.push_back(
        {seeds[size_t(t)], a.reached_target, a.first_hit_cycle, a.best_energy, a.wall_seconds});
    hits += a.reached_target ? 1 : 0;
    t_sum += a.wall_seconds;
  }
  rec.p_s = double(hits) / cfg.trials;
  rec.t_mean_s = t_sum / cfg.trials;
  rec.tts = compute_tts(rec.p_s, rec.t_mean_s > 0.0 ? rec.t_mean_s : 1e-12, cfg.p_target);
  return rec;
}

std::vector<BenchRecord> replica_sweep(const BenchConfig& cfg, const std::vector<int>& r_values) {
  if (cfg.engine != Engine::kSsqa)
    throw std::invalid_argument("replica sweep applies to the replica engine only");
  if (r_values.empty()) throw std::invalid_argument("no replica counts given");
  std::vector<BenchRecord> out;
  for (int r : r_values) {
    BenchConfig c = cfg;
    c.ssqa.r = r;
    out.push_back(run_trials(c));
  }
  return out;
}

std::vector<CaseSpec> case_suite() {
  return {{"case1", 10000, 50, 2},
          {"case2", 10000, 100, 1},
          {"case3", 20000, 50, 4},
          {"case4", 20000, 100, 2},
          {"case5", 40000, 100, 4}};
}

std::vector<BenchRecord> run_cases(const BenchConfig& cfg) {
  if (cfg.engine != Engine::kSsqa)
    throw std::invalid_argument("the case suite is defined for the replica engine only");
  std::vector<BenchRecord> out;
  for (const CaseSpec& cs : case_suite()) {
    if (cs.ec / cfg.ssqa.r / (long(cs.tau) * (cfg.ssqa.beta + 1)) != cs.iterations)
      throw std::invalid_argument(
          "case iteration counts need r*(beta+1)*tau to divide ec as tabulated "
          "(r=25, beta=3 reproduces them)");
    BenchConfig c = cfg;
    c.ec = cs.ec;
    c.ssqa.tau = cs.tau;
    BenchRecord rec = run_trials(c);
    rec.label = cs.label;
    out.push_back(std::move(rec));
  }
  return out;
}

namespace {

std::ofstream open_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  if (records.empty()) throw std::invalid_argument("no records to write");
  std::ofstream f(path);
  if (!f) throw std::runtime_error("cannot write " + path);
  return f;
}

}  // namespace

void write_results_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream f = open_csv(records, path);
  f << "engine,n,r,ec,tau,trials,p_s,t_mean_s,tts_s,seed\n";
  for (const auto& r : records)
    f << engine_name(r.engine) << "," << r.n << "," << r.r << "," << r.ec << "," << r.tau << ","
      << r.trials << "," << fmt(r.p_s) << "," << fmt(r.t_mean_s) << "," << r.tts.csv_field()
      << "," << r.base_seed << "\n";
  if (!f) throw std::runtime_error("write failed: " + path);
}

void write_sweep_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream f = open_csv(records, path);
  f << "r,p_s,t_mean_s,tts_s\n";
  for (const auto& r : records)
    f << r.r << "," << fmt(r.p_s) << "," << fmt(r.t_mean_s) << "," << r.tts.csv_field() << "\n";
  if (!f) throw std::runtime_error("write failed: " + path);
}

void write_cases_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream f = open_csv(records, path);
  f << "case,ec,tau,p_s,t_mean_s,tts_s\n";
  for (const auto& r : records)
    f << r.label << "," << r.ec << "," << r.tau << "," << fmt(r.p_s) << "," << fmt(r.t_mean_s)
      << "," << r.tts.csv_field() << "\n";
  if (!f) throw std::runtime_error("write failed: " + path);
}

}  // namespace ssqa
