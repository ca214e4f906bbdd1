/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C interface shared by the two CPU checkers under oracle/:
 *   - ref_*  : the unmodified reference C++ sources (/root/reference/proj/src)
 *              compiled into oracle/_ref/libssqa_ref.so through ref_adapter.cpp
 *              (namespace renamed ssqa -> ssqa_ref at compile time);
 *   - orc_*  : ssqa_oracle.c, a scalar C restatement of the same hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load these libraries, and only as checkers or the CPU
 * baseline.  The product (paper_2302_12454_b200) never links them.
 *
 * Layouts follow the reference ReplicaLattice (annealer.hpp:68-81):
 * sigma/acc are [i*r + k] doubles, history is (delay+1) consecutive
 * snapshots of that layout.  J is the dense mirrored n*n double matrix of
 * IsingModel (model.hpp:60-66).
 */
#ifndef SSQA_ORACLE_API_H
#define SSQA_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors ssqa::SsqaParams (annealer.hpp:14-30). */
typedef struct {
  int r;
  double jperp_min;
  double jperp_max;
  int beta;
  int tau;
  int delay;
  double i0;
  double n_rnd;
  double alpha;
  long sc;
  int bidirectional;
} orc_ssqa_params;

/* Mirrors ssqa::SsaParams (annealer.hpp:38-50). */
typedef struct {
  double i0_min;
  double i0_max;
  double beta;
  int tau;
  double n_rnd;
  double alpha;
  long sc;
} orc_ssa_params;

/* Mirrors the scalar fields of ssqa::AnnealResult (annealer.hpp:102-111). */
typedef struct {
  double best_energy;
  int best_replica;
  int reached_target;
  long first_hit_cycle;
  long cycles_used;
  long trace_len;
  double wall_seconds;
} orc_result;

/* Mirrors ssqa::TrialOutcome (bench.hpp:75-81). */
typedef struct {
  uint64_t seed;
  int reached_target;
  long first_hit_cycle;
  double best_energy;
  double wall_seconds;
} orc_trial;

/* Return codes: 0 ok, 1 invalid argument, 2 other error (see *_last_error). */

/* ---- reference adapter (oracle/_ref/libssqa_ref.so) ---- */
const char* ref_last_error(void);
uint64_t ref_mix64(uint64_t x);
uint64_t ref_rng_key(uint64_t seed, uint32_t stream);
uint64_t ref_rng_raw(uint64_t seed, uint32_t stream, uint64_t counter);
double ref_rng_uniform01(uint64_t seed, uint32_t stream, uint64_t counter);
uint64_t ref_spin_counter(uint64_t cycle, int replica, int spin);
int ref_jperp_schedule(long cycle, const orc_ssqa_params* p, double* out);
int ref_init_lattice(int n, int r, int d, uint64_t seed, double* sigma, double* acc,
                     double* hist);
int ref_ssqa_sweep(int n, const double* h, const double* J, double offset, double jperp,
                   const orc_ssqa_params* p, uint64_t seed, long cycle, double* sigma,
                   double* acc, double* hist, long* lat_cycle);
int ref_replica_energies(int n, const double* h, const double* J, double offset, int r,
                         const double* sigma, double* out);
int ref_ssqa_run(int n, const double* h, const double* J, double offset,
                 const orc_ssqa_params* p, uint64_t seed, int has_target, double target,
                 int record_trace, int stop_at_target, orc_result* out, int8_t* best_state,
                 double* trace_energy);
int ref_ssqa_run_many(int n, const double* h, const double* J, double offset,
                      const orc_ssqa_params* p, const uint64_t* seeds, int trials, int workers,
                      double* best_energy);
long ref_bench_manifest(const orc_ssqa_params* p, int n_nodes, double edge_prob, int permute,
                        double c1, double c2, int fresh_instance, uint64_t gi_seed, int trials,
                        long ec, double p_target, uint64_t base_seed, int workers, char* buf,
                        long cap);
int ref_i0_schedule(long cycle, const orc_ssa_params* p, double* out);
int ref_ssa_run(int n, const double* h, const double* J, double offset, const orc_ssa_params* p,
                uint64_t seed, int has_target, double target, int record_trace,
                int stop_at_target, orc_result* out, int8_t* best_state, double* trace_energy);
int ref_gi_ising(int n_nodes, double edge_prob, uint64_t seed, int permute, double c1,
                 double c2, double* h, double* J, double* offset);
int ref_run_trials(const orc_ssqa_params* p, int n_nodes, double edge_prob, int permute,
                   double c1, double c2, int fresh_instance, uint64_t gi_seed, int trials,
                   long ec, double p_target, uint64_t base_seed, int workers,
                   orc_trial* outcomes, double* p_s, double* t_mean, double* tts_seconds,
                   int* tts_kind);

/* ---- C restatement (oracle/_build/libssqa_oracle.so) ---- */
const char* orc_last_error(void);
uint64_t orc_mix64(uint64_t x);
uint64_t orc_rng_key(uint64_t seed, uint32_t stream);
uint64_t orc_rng_raw(uint64_t seed, uint32_t stream, uint64_t counter);
double orc_rng_uniform01(uint64_t seed, uint32_t stream, uint64_t counter);
uint64_t orc_spin_counter(uint64_t cycle, int replica, int spin);
int orc_jperp_schedule(long cycle, const orc_ssqa_params* p, double* out);
int orc_init_lattice(int n, int r, int d, uint64_t seed, double* sigma, double* acc,
                     double* hist);
int orc_ssqa_sweep(int n, const double* h, const double* J, double offset, double jperp,
                   const orc_ssqa_params* p, uint64_t seed, long cycle, double* sigma,
                   double* acc, double* hist, long* lat_cycle);
int orc_replica_energies(int n, const double* h, const double* J, double offset, int r,
                         const double* sigma, double* out);
int orc_ssqa_run(int n, const double* h, const double* J, double offset,
                 const orc_ssqa_params* p, uint64_t seed, int has_target, double target,
                 int record_trace, int stop_at_target, orc_result* out, int8_t* best_state,
                 double* trace_energy);
int orc_i0_schedule(long cycle, const orc_ssa_params* p, double* out);
int orc_ssa_run(int n, const double* h, const double* J, double offset, const orc_ssa_params* p,
                uint64_t seed, int has_target, double target, int record_trace,
                int stop_at_target, orc_result* out, int8_t* best_state, double* trace_energy);

#ifdef __cplusplus
}
#endif

#endif
