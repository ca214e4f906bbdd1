/*
 * ssqa_oracle.c -- TEST INFRASTRUCTURE ONLY: a scalar C restatement of the
 * reference SSQA hot path, used as the parity checker for the CUDA engine.
 * It is never linked into, or called by, the product.
 *
 * Parity is pinned two ways (tests/test_oracle_golden.py):
 *   1. the frozen RNG / schedule / clamp / delay known-answer tests of
 *      proj/tests/test_rng.cpp:40-56,122 and proj/tests/test_annealer.cpp:76-304;
 *   2. bitwise agreement with the reference itself (oracle/_ref, built from
 *      /root/reference by oracle/Makefile) through committed fixtures in
 *      tests/golden/ produced by scripts/make_golden.py.
 *
 * Each function cites the reference file:line it restates.  Arithmetic
 * order follows the production path (not the RefSweeper test helper): the
 * J sum starts at zero, runs over ascending j and the bias is added last
 * (annealer.cpp:91-95, 124-128); energies sum over ascending i
 * (annealer.cpp:246-256).  Compiled with -ffp-contract=off; every product
 * in the sweep is exact (sigma is +-1, noise is 0/+-1), so contraction could
 * not change a bit anyway.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_api.h"

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* rng.hpp:10-15 -- splitmix64 finalizer. */
uint64_t orc_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* rng.hpp:33-34 -- key = mix64(mix64(seed) ^ (2^32 + stream)). */
uint64_t orc_rng_key(uint64_t seed, uint32_t stream) {
  return orc_mix64(orc_mix64(seed) ^ (0x100000000ull + stream));
}

static uint64_t raw_k(uint64_t key, uint64_t counter) {
  return orc_mix64(key + counter * 0x9e3779b97f4a7c15ull); /* rng.hpp:36-38 */
}

uint64_t orc_rng_raw(uint64_t seed, uint32_t stream, uint64_t counter) {
  return raw_k(orc_rng_key(seed, stream), counter);
}

/* rng.hpp:41-43 */
double orc_rng_uniform01(uint64_t seed, uint32_t stream, uint64_t counter) {
  return (double)(orc_rng_raw(seed, stream, counter) >> 11) * 0x1.0p-53;
}

/* rng.hpp:65-67 */
uint64_t orc_spin_counter(uint64_t cycle, int replica, int spin) {
  return (cycle << 32) | ((uint64_t)replica << 20) | (uint64_t)spin;
}

enum { kStreamSpinInit = 1, kStreamSweepNoise = 2 }; /* rng.hpp:20-28 */

/* annealer.cpp:20-30, 365-373 -- SsqaParams::validate. */
static int validate(int n, const orc_ssqa_params* p) {
  if (n < 1 || n >= (1 << 20)) return fail(1, "spin count out of range");
  if (p->sc < 1 || p->sc >= (1L << 31)) return fail(1, "sc out of range");
  if (p->n_rnd < 0.0) return fail(1, "n_rnd must be >= 0");
  if (p->alpha <= 0.0) return fail(1, "alpha must be > 0");
  if (p->r < 1 || p->r >= (1 << 12)) return fail(1, "replica count out of range");
  if (p->jperp_max < p->jperp_min) return fail(1, "jperp_max < jperp_min");
  if (p->beta < 1) return fail(1, "beta must be >= 1");
  if (p->tau < 1) return fail(1, "tau must be >= 1");
  if (p->delay < 0) return fail(1, "delay must be >= 0");
  if (p->i0 <= 0.0) return fail(1, "i0 must be > 0");
  return 0;
}

/* annealer.cpp:375-380 */
static double jperp_at(long cycle, const orc_ssqa_params* p) {
  long c = cycle % ((long)p->tau * (p->beta + 1));
  long step = c / p->tau;
  return p->jperp_min + (double)step * (p->jperp_max - p->jperp_min) / p->beta;
}

int orc_jperp_schedule(long cycle, const orc_ssqa_params* p, double* out) {
  if (cycle < 0) return fail(1, "cycle must be >= 0");
  *out = jperp_at(cycle, p);
  return 0;
}

/* annealer.cpp:432-447 -- sigma = pm1(raw(spin_counter(0,k,i))), acc = 0. */
int orc_init_lattice(int n, int r, int d, uint64_t seed, double* sigma, double* acc,
                     double* hist) {
  const uint64_t key = orc_rng_key(seed, kStreamSpinInit);
  const size_t nr = (size_t)n * r;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < r; ++k)
      sigma[(size_t)i * r + k] = (raw_k(key, orc_spin_counter(0, k, i)) >> 63) ? 1.0 : -1.0;
  for (size_t v = 0; v < nr; ++v) acc[v] = 0.0;
  for (int s = 0; s <= d; ++s) memcpy(hist + s * nr, sigma, nr * sizeof(double));
  return 0;
}

/* annealer.cpp:216-242 with the tile contract of 91-95 / 124-128:
 * fields[i*r+k] = h_i + (0 + sum_{j ascending} J_ij sigma_jk). */
static void compute_fields(int n, int r, const double* h, const double* J,
                           const double* sigma, double* fields) {
  for (int i = 0; i < n; ++i) {
    const double* row = J + (size_t)i * n;
    for (int k = 0; k < r; ++k) {
      double a = 0.0;
      for (int j = 0; j < n; ++j) a += row[j] * sigma[(size_t)j * r + k];
      fields[(size_t)i * r + k] = h[i] + a;
    }
  }
}

/* annealer.cpp:246-256 */
static void energies_from_fields(int n, int r, const double* h, double offset,
                                 const double* sigma, const double* fields, double* e) {
  for (int k = 0; k < r; ++k) e[k] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < r; ++k)
      e[k] += sigma[(size_t)i * r + k] * (fields[(size_t)i * r + k] + h[i]);
  for (int k = 0; k < r; ++k) e[k] = -0.5 * e[k] + offset;
}

/* annealer.cpp:258-300 -- three-level noise, delayed coupling, clamp, sign. */
static void update_spins(int n, int r, int d, double* sigma, double* acc, double* hist,
                         const double* fields, double jperp, double i0, double n_rnd,
                         double alpha, int bidirectional, uint64_t noise_key, long cycle) {
  const size_t nr = (size_t)n * r;
  double* hi = hist + (size_t)(cycle % (d + 1)) * nr;
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < r; ++k) {
      const size_t v = (size_t)i * r + k;
      double input = fields[v];
      double u = (double)(raw_k(noise_key, orc_spin_counter((uint64_t)cycle, k, i)) >> 11) *
                 0x1.0p-53;
      input += n_rnd * (u < 0.4375 ? 0.0 : (u < 0.71875 ? -1.0 : 1.0));
      int kup = (k + 1 == r) ? 0 : k + 1;
      input += jperp * hi[(size_t)i * r + kup];
      if (bidirectional) {
        int kdn = (k == 0) ? r - 1 : k - 1;
        input += jperp * hi[(size_t)i * r + kdn];
      }
      double s = acc[v] + input;
      double clamped = (s >= i0) ? i0 - alpha : ((s < -i0) ? -i0 : s);
      acc[v] = clamped;
      sigma[v] = (clamped >= 0.0) ? 1.0 : -1.0;
    }
  }
  memcpy(hi, sigma, nr * sizeof(double)); /* annealer.cpp:298 */
}

/* annealer.cpp:449-463 */
int orc_ssqa_sweep(int n, const double* h, const double* J, double offset, double jperp,
                   const orc_ssqa_params* p, uint64_t seed, long cycle, double* sigma,
                   double* acc, double* hist, long* lat_cycle) {
  (void)offset;
  if (cycle != *lat_cycle) return fail(1, "sweep cycle does not match lattice history");
  double* fields = malloc(sizeof(double) * (size_t)n * p->r);
  if (!fields) return fail(2, "out of memory");
  compute_fields(n, p->r, h, J, sigma, fields);
  update_spins(n, p->r, p->delay, sigma, acc, hist, fields, jperp, p->i0, p->n_rnd, p->alpha,
               p->bidirectional, orc_rng_key(seed, kStreamSweepNoise), cycle);
  free(fields);
  *lat_cycle = cycle + 1;
  return 0;
}

/* annealer.cpp:465-472 */
int orc_replica_energies(int n, const double* h, const double* J, double offset, int r,
                         const double* sigma, double* out) {
  double* fields = malloc(sizeof(double) * (size_t)n * r);
  if (!fields) return fail(2, "out of memory");
  compute_fields(n, r, h, J, sigma, fields);
  energies_from_fields(n, r, h, offset, sigma, fields, out);
  free(fields);
  return 0;
}

/* annealer.cpp:313-361 -- run_lattice, shared by SSQA and SSA. */
typedef double (*cycle_fn)(long cycle, const void* ctx);

static int run_lattice(int n, const double* h, const double* J, double offset, int r, int d,
                       double n_rnd, double alpha, int bidirectional, long sc, cycle_fn jperp_f,
                       cycle_fn i0_f, const void* ctx, uint64_t seed, int has_target,
                       double target, int record_trace, int stop_at_target, orc_result* out,
                       int8_t* best_state, double* trace_energy) {
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const size_t nr = (size_t)n * r;
  double* sigma = malloc(sizeof(double) * nr);
  double* acc = malloc(sizeof(double) * nr);
  double* hist = malloc(sizeof(double) * nr * (d + 1));
  double* fields = malloc(sizeof(double) * nr);
  double* energy = malloc(sizeof(double) * r);
  if (!sigma || !acc || !hist || !fields || !energy) return fail(2, "out of memory");
  orc_init_lattice(n, r, d, seed, sigma, acc, hist);
  const uint64_t noise_key = orc_rng_key(seed, kStreamSweepNoise);

  out->best_energy = INFINITY;
  out->best_replica = 0;
  out->reached_target = 0;
  out->first_hit_cycle = -1;
  out->trace_len = 0;
  const double kTargetTol = 1e-9; /* annealer.hpp:113 */

  long cycle = 0;
  for (;; ++cycle) {
    const int final_scan = (cycle == sc);
    /* scan_state, annealer.cpp:327-345 */
    compute_fields(n, r, h, J, sigma, fields);
    energies_from_fields(n, r, h, offset, sigma, fields, energy);
    for (int k = 0; k < r; ++k) {
      if (energy[k] < out->best_energy) {
        out->best_energy = energy[k];
        out->best_replica = k;
        if (best_state)
          for (int i = 0; i < n; ++i) best_state[i] = sigma[(size_t)i * r + k] > 0.0 ? 1 : -1;
        if (has_target && !out->reached_target && out->best_energy <= target + kTargetTol) {
          out->reached_target = 1;
          out->first_hit_cycle = cycle;
        }
      }
      if (record_trace) {
        if (trace_energy) trace_energy[out->trace_len] = energy[k];
        out->trace_len++;
      }
    }
    if (final_scan) break;
    if (stop_at_target && out->reached_target) break; /* annealer.cpp:351 */
    update_spins(n, r, d, sigma, acc, hist, fields, jperp_f(cycle, ctx), i0_f(cycle, ctx), n_rnd,
                 alpha, bidirectional, noise_key, cycle);
  }
  out->cycles_used = cycle;
  clock_gettime(CLOCK_MONOTONIC, &t1);
  out->wall_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  free(sigma);
  free(acc);
  free(hist);
  free(fields);
  free(energy);
  return 0;
}

static double ssqa_jperp(long c, const void* ctx) { return jperp_at(c, (const orc_ssqa_params*)ctx); }
static double ssqa_i0(long c, const void* ctx) { (void)c; return ((const orc_ssqa_params*)ctx)->i0; }

/* annealer.cpp:474-487 */
int orc_ssqa_run(int n, const double* h, const double* J, double offset,
                 const orc_ssqa_params* p, uint64_t seed, int has_target, double target,
                 int record_trace, int stop_at_target, orc_result* out, int8_t* best_state,
                 double* trace_energy) {
  int rc = validate(n, p);
  if (rc) return rc;
  return run_lattice(n, h, J, offset, p->r, p->delay, p->n_rnd, p->alpha, p->bidirectional,
                     p->sc, ssqa_jperp, ssqa_i0, p, seed, has_target, target, record_trace,
                     stop_at_target, out, best_state, trace_energy);
}

/* annealer.cpp:382-408 -- SsaParams::validate, i0_levels, i0_schedule. */
static int ssa_levels(const orc_ssa_params* p, double* levels, int* count) {
  int k = 0;
  for (double v = p->i0_min; v <= p->i0_max * (1.0 + 1e-12); v /= p->beta) {
    levels[k++] = v;
    if (k > 64) return fail(1, "i0 schedule has too many levels");
  }
  *count = k;
  return 0;
}

static int ssa_validate(int n, const orc_ssa_params* p) {
  if (n < 1 || n >= (1 << 20)) return fail(1, "spin count out of range");
  if (p->sc < 1 || p->sc >= (1L << 31)) return fail(1, "sc out of range");
  if (p->n_rnd < 0.0) return fail(1, "n_rnd must be >= 0");
  if (p->alpha <= 0.0) return fail(1, "alpha must be > 0");
  if (p->i0_min <= 0.0 || p->i0_min > p->i0_max) return fail(1, "need 0 < i0_min <= i0_max");
  if (p->beta <= 0.0 || p->beta >= 1.0) return fail(1, "beta must be in (0, 1)");
  if (p->tau < 1) return fail(1, "tau must be >= 1");
  return 0;
}

typedef struct {
  double levels[66];
  int count;
  int tau;
} ssa_ctx;

static double ssa_jperp(long c, const void* ctx) { (void)c; (void)ctx; return 0.0; }
static double ssa_i0(long c, const void* ctx) {
  const ssa_ctx* s = (const ssa_ctx*)ctx;
  long cc = c % ((long)s->count * s->tau);
  return s->levels[cc / s->tau];
}

int orc_i0_schedule(long cycle, const orc_ssa_params* p, double* out) {
  if (cycle < 0) return fail(1, "cycle must be >= 0");
  ssa_ctx s;
  int rc = ssa_levels(p, s.levels, &s.count);
  if (rc) return rc;
  s.tau = p->tau;
  *out = ssa_i0(cycle, &s);
  return 0;
}

/* annealer.cpp:489-501 */
int orc_ssa_run(int n, const double* h, const double* J, double offset, const orc_ssa_params* p,
                uint64_t seed, int has_target, double target, int record_trace,
                int stop_at_target, orc_result* out, int8_t* best_state, double* trace_energy) {
  int rc = ssa_validate(n, p);
  if (rc) return rc;
  ssa_ctx s;
  rc = ssa_levels(p, s.levels, &s.count);
  if (rc) return rc;
  s.tau = p->tau;
  return run_lattice(n, h, J, offset, 1, 0, p->n_rnd, p->alpha, 0, p->sc, ssa_jperp, ssa_i0, &s,
                     seed, has_target, target, record_trace, stop_at_target, out, best_state,
                     trace_energy);
}
