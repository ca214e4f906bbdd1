// host/manifest.cpp -- JSON forms of the bench records and run manifests
// (bench.hpp: BenchConfig/TtsValue/BenchRecord::to_json/from_json,
// make_manifest, replay_manifest), in the reference's schema
// (bench.cpp:124-300, 519-584) so manifests written by either side replay on
// the other.  Replays re-run on the GPU through run_trials/replica_sweep/
// run_cases and compare the outcomes bitwise.  Built only with nlohmann/json.
#include "ssqa/bench.hpp"

#ifdef SSQA_HAVE_JSON

#include <ctime>
#include <stdexcept>
#include <string>

namespace ssqa {

namespace {

constexpr const char* kManifestVersion = "0.1.0";

// Every expected key present, nothing else (the reference's strictness).
void expect_keys(const nlohmann::json& j, std::initializer_list<const char*> keys,
                 const char* where) {
  if (!j.is_object()) throw std::runtime_error(std::string(where) + ": not an object");
  for (const char* k : keys)
    if (!j.contains(k)) throw std::runtime_error(std::string(where) + ": missing key '" + k + "'");
  for (auto it = j.begin(); it != j.end(); ++it) {
    bool ok = false;
    for (const char* k : keys) ok = ok || it.key() == k;
    if (!ok) throw std::runtime_error(std::string(where) + ": unknown key '" + it.key() + "'");
  }
}

std::string utc_timestamp() {
  const std::time_t now = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&now, &tm);
  char buf[32];
  std::strftime(buf, sizeof(buf), "%Y-%m-%dT%H:%M:%SZ", &tm);
  return buf;
}

}  // namespace

nlohmann::json TtsValue::to_json() const {
  nlohmann::json j;
  j["defined"] = kind != Kind::kUndefined;
  j["saturated"] = kind == Kind::kSaturatedZero;
  j["seconds"] = kind == Kind::kFinite ? nlohmann::json(seconds) : nlohmann::json(nullptr);
  return j;
}

TtsValue TtsValue::from_json(const nlohmann::json& j) {
  expect_keys(j, {"defined", "saturated", "seconds"}, "tts");
  TtsValue v;
  if (!j.at("defined").get<bool>()) {
    v.kind = Kind::kUndefined;
  } else if (j.at("saturated").get<bool>()) {
    v.kind = Kind::kSaturatedZero;
  } else {
    v.kind = Kind::kFinite;
    v.seconds = j.at("seconds").get<double>();
  }
  return v;
}

nlohmann::json BenchConfig::to_json() const {
  nlohmann::json j;
  j["engine"] = engine_name(engine);
  j["ssqa"] = nlohmann::json{{"r", ssqa.r},
                             {"jperp_min", ssqa.jperp_min},
                             {"jperp_max", ssqa.jperp_max},
                             {"beta", ssqa.beta},
                             {"tau", ssqa.tau},
                             {"delay", ssqa.delay},
                             {"i0", ssqa.i0},
                             {"n_rnd", ssqa.n_rnd},
                             {"alpha", ssqa.alpha},
                             {"bidirectional", ssqa.bidirectional}};
  j["ssa"] = nlohmann::json{{"i0_min", ssa.i0_min}, {"i0_max", ssa.i0_max},
                            {"beta", ssa.beta},     {"tau", ssa.tau},
                            {"n_rnd", ssa.n_rnd},   {"alpha", ssa.alpha}};
  j["sa"] = nlohmann::json{{"t_init", sa.t_init}, {"t_final", sa.t_final},
                           {"delta_it", sa.delta_it}};
  nlohmann::json pr;
  pr["n_nodes"] = problem.n_nodes;
  pr["edge_prob"] = problem.edge_prob;
  pr["permute"] = problem.permute;
  pr["c1"] = problem.c1;
  pr["c2"] = problem.c2;
  pr["fresh_instance"] = problem.fresh_instance;
  pr["gi_seed"] = problem.gi_seed;
  pr["model_file"] = problem.model_file;
  pr["target_energy"] =
      problem.target_energy ? nlohmann::json(*problem.target_energy) : nlohmann::json(nullptr);
  j["problem"] = pr;
  j["trials"] = trials;
  j["ec"] = ec;
  j["p_target"] = p_target;
  j["base_seed"] = base_seed;
  j["workers"] = workers;
  return j;
}

BenchConfig BenchConfig::from_json(const nlohmann::json& j) {
  expect_keys(j, {"engine", "ssqa", "ssa", "sa", "problem", "trials", "ec", "p_target",
                  "base_seed", "workers"},
              "config");
  BenchConfig c;
  c.engine = engine_from_name(j.at("engine").get<std::string>());
  const nlohmann::json& q = j.at("ssqa");
  expect_keys(q, {"r", "jperp_min", "jperp_max", "beta", "tau", "delay", "i0", "n_rnd", "alpha",
                  "bidirectional"},
              "config.ssqa");
  q.at("r").get_to(c.ssqa.r);
  q.at("jperp_min").get_to(c.ssqa.jperp_min);
  q.at("jperp_max").get_to(c.ssqa.jperp_max);
  q.at("beta").get_to(c.ssqa.beta);
  q.at("tau").get_to(c.ssqa.tau);
  q.at("delay").get_to(c.ssqa.delay);
  q.at("i0").get_to(c.ssqa.i0);
  q.at("n_rnd").get_to(c.ssqa.n_rnd);
  q.at("alpha").get_to(c.ssqa.alpha);
  q.at("bidirectional").get_to(c.ssqa.bidirectional);
  const nlohmann::json& s = j.at("ssa");
  expect_keys(s, {"i0_min", "i0_max", "beta", "tau", "n_rnd", "alpha"}, "config.ssa");
  s.at("i0_min").get_to(c.ssa.i0_min);
  s.at("i0_max").get_to(c.ssa.i0_max);
  s.at("beta").get_to(c.ssa.beta);
  s.at("tau").get_to(c.ssa.tau);
  s.at("n_rnd").get_to(c.ssa.n_rnd);
  s.at("alpha").get_to(c.ssa.alpha);
  const nlohmann::json& a = j.at("sa");
  expect_keys(a, {"t_init", "t_final", "delta_it"}, "config.sa");
  a.at("t_init").get_to(c.sa.t_init);
  a.at("t_final").get_to(c.sa.t_final);
  a.at("delta_it").get_to(c.sa.delta_it);
  const nlohmann::json& p = j.at("problem");
  expect_keys(p, {"n_nodes", "edge_prob", "permute", "c1", "c2", "fresh_instance", "gi_seed",
                  "model_file", "target_energy"},
              "config.problem");
  p.at("n_nodes").get_to(c.problem.n_nodes);
  p.at("edge_prob").get_to(c.problem.edge_prob);
  p.at("permute").get_to(c.problem.permute);
  p.at("c1").get_to(c.problem.c1);
  p.at("c2").get_to(c.problem.c2);
  p.at("fresh_instance").get_to(c.problem.fresh_instance);
  p.at("gi_seed").get_to(c.problem.gi_seed);
  p.at("model_file").get_to(c.problem.model_file);
  if (!p.at("target_energy").is_null()) c.problem.target_energy = p.at("target_energy").get<double>();
  j.at("trials").get_to(c.trials);
  j.at("ec").get_to(c.ec);
  j.at("p_target").get_to(c.p_target);
  j.at("base_seed").get_to(c.base_seed);
  j.at("workers").get_to(c.workers);
  return c;
}

nlohmann::json BenchRecord::to_json() const {
  nlohmann::json outs = nlohmann::json::array();
  for (const TrialOutcome& t : per_trial)
    outs.push_back(nlohmann::json{{"seed", t.seed},
                                  {"reached_target", t.reached_target},
                                  {"first_hit_cycle", t.first_hit_cycle},
                                  {"best_energy", t.best_energy},
                                  {"wall_seconds", t.wall_seconds}});
  nlohmann::json j;
  j["label"] = label;
  j["engine"] = engine_name(engine);
  j["n"] = n;
  j["r"] = r;
  j["ec"] = ec;
  j["tau"] = tau;
  j["trials"] = trials;
  j["p_s"] = p_s;
  j["t_mean_s"] = t_mean_s;
  j["tts"] = tts.to_json();
  j["seed"] = base_seed;
  j["per_trial"] = outs;
  return j;
}

BenchRecord BenchRecord::from_json(const nlohmann::json& j) {
  expect_keys(j, {"label", "engine", "n", "r", "ec", "tau", "trials", "p_s", "t_mean_s", "tts",
                  "seed", "per_trial"},
              "record");
  BenchRecord rec;
  j.at("label").get_to(rec.label);
  rec.engine = engine_from_name(j.at("engine").get<std::string>());
  j.at("n").get_to(rec.n);
  j.at("r").get_to(rec.r);
  j.at("ec").get_to(rec.ec);
  j.at("tau").get_to(rec.tau);
  j.at("trials").get_to(rec.trials);
  j.at("p_s").get_to(rec.p_s);
  j.at("t_mean_s").get_to(rec.t_mean_s);
  rec.tts = TtsValue::from_json(j.at("tts"));
  j.at("seed").get_to(rec.base_seed);
  for (const nlohmann::json& t : j.at("per_trial")) {
    expect_keys(t, {"seed", "reached_target", "first_hit_cycle", "best_energy", "wall_seconds"},
                "per_trial");
    TrialOutcome o;
    t.at("seed").get_to(o.seed);
    t.at("reached_target").get_to(o.reached_target);
    t.at("first_hit_cycle").get_to(o.first_hit_cycle);
    t.at("best_energy").get_to(o.best_energy);
    t.at("wall_seconds").get_to(o.wall_seconds);
    rec.per_trial.push_back(o);
  }
  return rec;
}

nlohmann::json make_manifest(const std::string& kind, const BenchConfig& cfg,
                             const std::vector<int>& r_values,
                             const std::vector<BenchRecord>& records,
                             const std::vector<std::string>& output_paths) {
  nlohmann::json recs = nlohmann::json::array();
  for (const BenchRecord& r : records) recs.push_back(r.to_json());
  nlohmann::json m;
  m["kind"] = kind;
  m["version"] = kManifestVersion;
  m["created_utc"] = utc_timestamp();
  m["config"] = cfg.to_json();
  m["r_values"] = r_values;
  m["outputs"] = output_paths;
  m["records"] = recs;
  return m;
}

ReplayResult replay_manifest(const nlohmann::json& manifest, std::optional<int> workers_override) {
  expect_keys(manifest, {"kind", "version", "created_utc", "config", "r_values", "outputs",
                         "records"},
              "manifest");
  BenchConfig cfg = BenchConfig::from_json(manifest.at("config"));
  if (workers_override) cfg.workers = *workers_override;
  const std::string kind = manifest.at("kind").get<std::string>();
  ReplayResult out;
  if (kind == "bench") {
    out.records.push_back(run_trials(cfg));
  } else if (kind == "sweep") {
    out.records = replica_sweep(cfg, manifest.at("r_values").get<std::vector<int>>());
  } else if (kind == "cases") {
    out.records = run_cases(cfg);
  } else {
    throw std::runtime_error("unknown manifest kind '" + kind + "'");
  }
  auto differ = [&out](const std::string& why) {
    if (out.match) out.mismatch = why;
    out.match = false;
  };
  const nlohmann::json& want = manifest.at("records");
  if (want.size() != out.records.size()) {
    differ("record count differs");
    return out;
  }
  for (size_t i = 0; i < want.size(); ++i) {
    const BenchRecord a = BenchRecord::from_json(want[i]);
    const BenchRecord& b = out.records[i];
    if (a.per_trial.size() != b.per_trial.size()) {
      differ("trial count differs in record " + std::to_string(i));
      continue;
    }
    for (size_t t = 0; t < a.per_trial.size(); ++t) {
      const TrialOutcome &x = a.per_trial[t], &y = b.per_trial[t];
      if (x.seed != y.seed || x.reached_target != y.reached_target ||
          x.first_hit_cycle != y.first_hit_cycle || x.best_energy != y.best_energy) {
        differ("trial " + std::to_string(t) + " of record " + std::to_string(i) + " differs");
        break;
      }
    }
  }
  return out;
}

}  // namespace ssqa

#endif  // SSQA_HAVE_JSON
