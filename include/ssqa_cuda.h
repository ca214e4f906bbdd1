/*
 * ssqa_cuda.h -- C ABI of the B200 SSQA engine (libssqa_b200.so).
 *
 * This is the drop-in boundary for the reference's annealing loop
 * (/root/reference/proj).  The reference has no FFI of its own: its hot
 * path is the C++ call chain ssqa_run -> run_lattice -> compute_fields /
 * energies_from_fields / update_spins (src/annealer.cpp:216-361, 474-487)
 * and its batched caller run_trials (src/bench.cpp:359-432).  Each entry
 * point below names the reference interface it replaces.  The C++ facade in
 * include/ssqa/{rng,model,gi,annealer,bench}.hpp (same names as the reference headers) is built on top
 * of these entry points; INTEGRATION.md shows the binding a maintainer adds.
 *
 * Conventions
 *  - Plain pointers and sizes only; all pointers are HOST pointers unless a
 *    name says otherwise.  No exceptions cross the ABI.
 *  - Every function returns SSQA_OK (0) or an error code; ssqa_last_error()
 *    returns the calling thread's last message.  SSQA_EINVAL corresponds to
 *    the reference's std::invalid_argument (annealer.cpp:25-30, 365-373),
 *    SSQA_ERANGE to std::out_of_range, SSQA_ECUDA/SSQA_EUNSUP to failures the
 *    reference cannot have (device errors; models the int8 engine cannot
 *    represent exactly -- there is no CPU fallback).
 *  - Lattice arrays use the reference ReplicaLattice layout [i*r + k]
 *    (annealer.hpp:68-81); history is (delay+1) consecutive snapshots.
 *  - A problem handle owns one device and one CUDA stream.  Distinct handles
 *    may be used from distinct threads concurrently (the reference's
 *    run_trials calls ssqa_run from W threads, bench.cpp:379-407).
 */
#ifndef SSQA_CUDA_H
#define SSQA_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSQA_OK 0
#define SSQA_EINVAL 1  /* std::invalid_argument in the reference */
#define SSQA_ERANGE 2  /* std::out_of_range in the reference */
#define SSQA_ECUDA 3   /* CUDA runtime / launch failure */
#define SSQA_EUNSUP 4  /* model not exactly representable by the int8 engine */

typedef struct ssqa_problem_s* ssqa_problem;
typedef struct ssqa_batch_s* ssqa_batch;

/* Mirrors ssqa::SsqaParams (annealer.hpp:14-30), field for field. */
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
} ssqa_params_c;

/* Mirrors ssqa::SsaParams (annealer.hpp:38-50), field for field: the
 * single-network engine whose accumulator bound climbs the geometric ladder
 * i0_min, i0_min/beta, ... <= i0_max every tau cycles and wraps. */
typedef struct {
  double i0_min;
  double i0_max;
  double beta;
  int tau;
  double n_rnd;
  double alpha;
  long sc;
} ssqa_ssa_params_c;

/* Scalar fields of ssqa::AnnealResult (annealer.hpp:102-111).  wall_seconds
 * of a batched run is the batch's device time divided by the trial count. */
typedef struct {
  double best_energy;
  int best_replica;
  int reached_target;
  long first_hit_cycle;
  long cycles_used;
  double wall_seconds;
} ssqa_result_c;

/* Engine selection for ssqa_batch_create (SSQA_ENGINE_AUTO picks the
 * tcgen05 kernel whenever the shape allows it). */
#define SSQA_ENGINE_AUTO 0
#define SSQA_ENGINE_SIMT 1    /* CUDA-core int8 field + fused epilogue */
#define SSQA_ENGINE_TCGEN05 2 /* fused tcgen05/TMEM/TMA sweep kernel */

const char* ssqa_last_error(void);
const char* ssqa_version(void);

/* ---- Device memory pool (no reference counterpart: the reference's lattice
 * lives in std::vector, annealer.cpp:432-447) ---------------------------------
 * Problem and batch buffers come from a process-wide caching allocator:
 * destroyed handles return their blocks to it and the next handle of the same
 * shape reuses them, so repeated ssqa_run_batch calls pay no cudaMalloc /
 * cudaFree.  Blocks are released when an allocation would otherwise fail, or
 * here.  ssqa_pool_trim returns the bytes released (device -1: all devices). */
long long ssqa_pool_trim(int device);
int ssqa_pool_stats(int device, long long* cached_bytes, long long* in_use_bytes);

/* ---- Problem: replaces DenseProblem (annealer.cpp:40-89) -------------------
 * h[n], J[n*n] (dense, mirrored, zero diagonal: IsingModel storage,
 * model.hpp:59-66) and offset are quantized once to int8 J' = J*2^p and
 * int32 H' = h*2^p with the smallest p >= 0 that makes both integral, then
 * uploaded to `device`.  |J'| <= 127 gives int8 couplings, up to 32639 int16
 * ones (ssqa_problem_int16); SSQA_EUNSUP beyond that.
 * The device copy is shared by every batch created on the handle. */
int ssqa_problem_create(int n, const double* h, const double* J, double offset, int device,
                        ssqa_problem* out);
int ssqa_problem_destroy(ssqa_problem prob);
/* Fresh instances per trial (run_trials with fresh_instance, bench.cpp:387-389):
 * `count` models of n spins -- h[count*n], J[count*n*n], offsets[count] --
 * quantized at one common scale and stacked on the device.  A batch on such
 * a problem must have trials == count; trial t anneals instance t (tcgen05
 * engine, one trial per column tile).  ssqa_problem_count() is 1 for
 * ssqa_problem_create problems. */
int ssqa_problem_create_many(int count, int n, const double* h, const double* J,
                             const double* offsets, int device, ssqa_problem* out);
int ssqa_problem_count(ssqa_problem prob);
/* Problems built on the device, with no host model (SURVEY.md 8.1 f2 and the
 * BASELINE C4/C5 instances): the same quantized problem as
 *   ssqa_problem_create(ssqa_dense_ising(n, kind, seed))          (dense), and
 *   ssqa_problem_create_many(qubo_to_ising(build_gi_qubo(generate_gi(
 *       n_nodes, edge_prob, seeds[t], permute, c1, c2))) for t < count)   (GI;
 *   count == 1 gives a single-instance problem), gi.cpp:102-184 --
 * the GI graph pairs are drawn on the host, J' is written on the device from
 * their adjacency matrices (the penalty's closed form); dyadic c1, c2 only. */
int ssqa_problem_create_dense(int n, int kind, uint64_t seed, int device, ssqa_problem* out);
int ssqa_problem_create_gi(int count, int n_nodes, double edge_prob, const uint64_t* seeds,
                           int permute, double c1, double c2, int device, ssqa_problem* out);
/* The all-zero n-spin problem (h = 0, J = 0, offset 0), made on the device:
 * what init_lattice / lattice-only batches need without uploading a model. */
int ssqa_problem_create_zero(int n, int device, ssqa_problem* out);
/* Device image of a problem: J' int8 [count*npad][npad], H' int32 [count*npad],
 * offsets [count] (any pointer may be NULL). */
int ssqa_problem_export(ssqa_problem prob, int8_t* J, int32_t* H, double* offsets);
/* Quantizer report: padded size, scale exponent p, max |J'|, max |H'|. */
int ssqa_problem_info(ssqa_problem prob, int* n, int* n_pad, int* shift_p, int* max_abs_j,
                      int* max_abs_h);

/* 1 when the problem also holds an FP4 (e2m1) image of J' (couplings all in
 * {0, +-1, +-2, +-3, +-4, +-6}); the tcgen05 engine then streams 4-bit
 * operands (tcgen05.mma kind::mxf4 with unit block scales). */
int ssqa_problem_fp4(ssqa_problem prob);
/* 1 when the couplings need int16 (127 < max |J'| <= 32639): J' is held as two
 * int8 planes J' = 256 Ahi + Alo and the tcgen05 engine runs one int8 MMA per
 * plane (replicas <= 128; the SIMT engine refuses such problems). */
int ssqa_problem_int16(ssqa_problem prob);

/* Host-only dry run of the quantizer (no device touched): the scale and
 * ranges ssqa_problem_create would use, or SSQA_EUNSUP with the reason. */
int ssqa_quantize_info(int n, const double* h, const double* J, int* n_pad, int* shift_p,
                       int* max_abs_j, int* max_abs_h);

/* Host-only dry run of the column tiling (no device touched): how a batch of
 * `trials` x `replicas` columns over n spins would be laid out on `sms` SMs
 * by the tcgen05 engine with 4- or 8-bit operands -- columns per tile, column
 * tiles, trials per tile and row parts per tile (1: whole tiles; > 1: each
 * tile's rows split over that many CTAs). */
int ssqa_plan_geometry(int n, int replicas, int trials, int sms, int operand_bits,
                       int* tile_cols, int* tiles, int* trials_per_tile, int* row_parts);

/* ---- Validation: SsqaParams::validate (annealer.cpp:365-373) ---------- */
int ssqa_params_validate(const ssqa_params_c* p, int n);
/* jperp_schedule (annealer.cpp:375-380); SSQA_EINVAL for cycle < 0. */
int ssqa_jperp_schedule(long cycle, const ssqa_params_c* p, double* out);

/* ---- SSA: SsaParams::validate / i0_levels (annealer.cpp:382-397) and
 * i0_schedule (annealer.cpp:403-408).  SSQA_EINVAL for a ladder of more than
 * 64 levels, as the reference; also for an empty ladder (NaN bounds), where
 * the reference would divide by zero. */
int ssqa_ssa_params_validate(const ssqa_ssa_params_c* p, int n);
int ssqa_i0_schedule(long cycle, const ssqa_ssa_params_c* p, double* out);
/* SsaParams::i0_levels (annealer.cpp:389-397): writes the ladder to
 * levels[0..*count) (room for 64 doubles). */
int ssqa_i0_levels(const ssqa_ssa_params_c* p, double* levels, int* count);

/* ---- One-shot runs: ssqa_run (annealer.cpp:474-487) over a batch of seeds.
 * Trial t runs ssqa_run(model, p, seeds[t], target, {record_trace,
 * stop_at_target}) exactly; results[t] gets the AnnealResult scalars,
 * best_states[t*n..] (int8 +-1, may be NULL) the best state and
 * trace[t*(sc+1)*r ..] (may be NULL unless record_trace) the TracePoint
 * energies in the reference order (cycle-major, replica-minor; entries past
 * a trial's cycles_used stay untouched). */
int ssqa_run_batch(ssqa_problem prob, const ssqa_params_c* p, const uint64_t* seeds,
                   int trials, int has_target, double target, int record_trace,
                   int stop_at_target, int engine, ssqa_result_c* results,
                   int8_t* best_states, double* trace);

/* ssa_run (annealer.cpp:489-501) over a batch of seeds: the same lattice
 * engine with r = 1, delay = 0, jperp = 0 and the per-cycle bound
 * i0_schedule(cycle, p).  Arguments and outputs as ssqa_run_batch (trace
 * holds sc+1 energies per trial; best_replica is always 0). */
int ssqa_ssa_run_batch(ssqa_problem prob, const ssqa_ssa_params_c* p, const uint64_t* seeds,
                       int trials, int has_target, double target, int record_trace,
                       int stop_at_target, int engine, ssqa_result_c* results,
                       int8_t* best_states, double* trace);

/* ---- Batches: device-resident state for `trials` x p->r replica columns.
 * Replaces the per-trial ReplicaLattice of run_lattice (annealer.cpp:319-321);
 * run_trials' thread pool (bench.cpp:399-407) becomes the batch. */
int ssqa_batch_create(ssqa_problem prob, const ssqa_params_c* p, int trials, int record_trace,
                      int engine, ssqa_batch* out);
/* A batch of ssa_run trials (annealer.cpp:489-501); every batch entry point
 * below applies, with r = 1 and delay = 0.  ssqa_batch_sweep follows the
 * i0 ladder at the lattice cycle. */
int ssqa_batch_create_ssa(ssqa_problem prob, const ssqa_ssa_params_c* p, int trials,
                          int record_trace, int engine, ssqa_batch* out);
int ssqa_batch_destroy(ssqa_batch b);
/* CUDA stream (cudaStream_t) the batch enqueues on; for event timing. */
void* ssqa_batch_stream(ssqa_batch b);
/* Engine the batch resolved to (SSQA_ENGINE_SIMT / SSQA_ENGINE_TCGEN05). */
int ssqa_batch_engine(ssqa_batch b);
/* Bits per coupling/spin operand the contraction streams: 4 (e2m1 FP4,
 * tcgen05 kind::mxf4) or 8 (int8). */
int ssqa_batch_operand_bits(ssqa_batch b);
/* Upload per-trial seeds (host array of `trials`). */
int ssqa_batch_set_seeds(ssqa_batch b, const uint64_t* seeds);
/* Asynchronous full run on the batch stream: init_lattice + run_lattice
 * for every trial (annealer.cpp:313-361).  No host synchronisation. */
int ssqa_batch_launch(ssqa_batch b, int has_target, double target, int stop_at_target);
/* Wait for the batch stream and copy results back (as ssqa_run_batch). */
int ssqa_batch_fetch(ssqa_batch b, ssqa_result_c* results, int8_t* best_states,
                     double* trace);
/* Number of kernel launches the last ssqa_batch_launch enqueued. */
long ssqa_batch_launch_count(ssqa_batch b);
/* Device time of the last ssqa_batch_launch (CUDA events recorded on the
 * batch stream around everything the launch enqueued); waits for it. */
int ssqa_batch_elapsed_ms(ssqa_batch b, double* ms);
/* Block until everything queued on the batch stream has finished. */
int ssqa_batch_synchronize(ssqa_batch b);
/* Measurement hook: time `iters` back-to-back launches of the engine's field
 * contraction on the current state (CUDA events on the batch stream) and
 * return the mean duration of one launch.  State is not modified. */
int ssqa_batch_profile_field(ssqa_batch b, int iters, double* ms_per_launch);

/* ---- GPU row shards (J' row-sharded across GPUs) ------
 * Every GPU g of G holds the same problem and a batch with the same seeds and
 * params; ssqa_batch_set_shard(b, g, G) makes it update only spin rows
 * [g*npad/G, (g+1)*npad/G).  Per cycle c = 0..sc:
 *   ssqa_batch_shard_pass(b, chunk)   contraction of its rows against the full
 *       sigma(c), update of its rows, and packs sigma(c+1) of its rows
 *       (1 bit per spin) plus its per-column int64 energy partials into
 *       `chunk` (device memory, ssqa_batch_shard_bytes(b) bytes);
 *   all-gather of the G chunks (e.g. ncclAllGather, in shard order);
 *   ssqa_batch_shard_merge(b, chunks) unpacks every shard's rows into
 *       sigma(c+1), sums the energy partials and scans cycle c
 *       (best tracking, trace, stop-at-target) exactly as run_lattice.
 * Bracket the cycles with ssqa_batch_shard_begin (reset + init_lattice) and
 * ssqa_batch_shard_end; ssqa_batch_fetch then returns the results (identical
 * on every GPU).  All calls enqueue on ssqa_batch_stream(b); order the
 * collective on that stream.  tcgen05 engine, int8 operands; npad/128 must
 * be divisible by G. */
int ssqa_batch_set_shard(ssqa_batch b, int shard, int nshards);
long ssqa_batch_shard_bytes(ssqa_batch b);
int ssqa_batch_shard_begin(ssqa_batch b, int has_target, double target, int stop_at_target);
int ssqa_batch_shard_pass(ssqa_batch b, void* chunk);
int ssqa_batch_shard_merge(ssqa_batch b, const void* chunks);
int ssqa_batch_shard_end(ssqa_batch b);

/* Peer push instead of a collective library: the pack kernel of
 * ssqa_batch_shard_pass_to stores this shard's chunk straight into dests[d]
 * (this shard's slot in GPU d's exchange region, a peer pointer from
 * ssqa_ipc_open -- NVLink stores) and its last block raises *flags[d] = epoch
 * (system-scope release); ssqa_batch_shard_merge_from waits until its own
 * flags[0..G) all reach epoch (system-scope acquire) and merges `chunks`.
 * Use epoch = cycle + 1 and two exchange regions by epoch parity: a GPU can
 * only write epoch e + 2 after every GPU has merged epoch e.  ndest <= 8. */
int ssqa_batch_shard_pass_to(ssqa_batch b, void* const* dests, unsigned* const* flags, int ndest,
                             unsigned epoch);
int ssqa_batch_shard_merge_from(ssqa_batch b, const void* chunks, const unsigned* flags,
                                int nflags, unsigned epoch);
/* The exchange fused into the shard pass itself (FP4 operands with the table
 * epilogue: ssqa_batch_shard_direct_ok): the tcgen05 epilogue stores every
 * spin word of its rows into its own FP4 slot AND into each peer's
 * (peer_sig4[d] = peer d's ssqa_batch_sig4 pointer, IPC-mapped; same slot
 * ring on every GPU), its last CTA pushes the per-column int64 energy
 * partials to peer_parts[d] (this shard's row of peer d's parts half for the
 * epoch's parity) and raises *flags[d] = epoch.  ssqa_batch_shard_merge_direct
 * waits on its own G flags, sums the G int64 partial rows at `parts`
 * (part_stride bytes apart), refreshes the int8 slot from the FP4 slot and
 * scans.
 * No pack kernel, no staging buffer, no collective call. */
int ssqa_batch_shard_direct_ok(ssqa_batch b);
int ssqa_batch_sig4(ssqa_batch b, void** dev_ptr_out);
int ssqa_batch_shard_pass_direct(ssqa_batch b, void* const* peer_sig4, void* const* peer_parts,
                                 unsigned* const* flags, int npeer, unsigned epoch);
int ssqa_batch_shard_merge_direct(ssqa_batch b, const void* parts, long long part_stride,
                                  const unsigned* flags, int nflags, unsigned epoch);
/* Exchange regions: a zeroed device block of its own (CUDA IPC maps whole
 * allocations), its 64-byte IPC handle, and the peer mapping of a handle
 * from another process of the node. */
int ssqa_exchange_alloc(int device, long long bytes, void** dev_ptr_out);
int ssqa_exchange_free(void* dev_ptr);
int ssqa_ipc_handle(const void* dev_ptr, void* handle_out);
int ssqa_ipc_open(const void* handle, int device, void** dev_ptr_out);
int ssqa_ipc_close(void* dev_ptr);

/* ---- Per-step API: init_lattice / ssqa_sweep / replica_energies
 * (annealer.cpp:432-472), applied to every trial of the batch. ---------- */
/* init_lattice(n, r, delay, seeds[t]) for each trial; lattice cycle = 0. */
int ssqa_batch_init(ssqa_batch b);
/* `count` consecutive ssqa_sweep calls with the batch's own jperp schedule
 * (jperp_schedule(cycle, p), i0 = p->i0), starting at the lattice cycle. */
int ssqa_batch_sweep(ssqa_batch b, long count);
/* One ssqa_sweep with an explicit coupling strength and bound, as the
 * reference per-step API allows (annealer.hpp:89-90, test_annealer.cpp:343-347). */
int ssqa_batch_sweep_with(ssqa_batch b, double jperp, double i0);
/* replica_energies of every trial's current state: out[t*r + k]. */
int ssqa_batch_energies(ssqa_batch b, double* out);
/* Read / write one trial's lattice in the reference layout.  hist holds
 * (delay+1)*n*r doubles; cycle is ReplicaLattice::cycle. */
int ssqa_batch_read_lattice(ssqa_batch b, int trial, double* sigma, double* acc, double* hist,
                            long* cycle);
int ssqa_batch_write_lattice(ssqa_batch b, int trial, const double* sigma, const double* acc,
                             const double* hist, long cycle);

#ifdef __cplusplus
}
#endif

#endif /* SSQA_CUDA_H */
