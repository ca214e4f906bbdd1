// capi.cu -- the C ABI of include/ssqa_cuda.h: problem upload, batches, the
// run loop (run_lattice, annealer.cpp:313-361) and the per-step parity API.
#include "devpool.h"
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.h"
#include "quantize_kernels.cuh"
#include "generate_kernels.cuh"
#include "ssqa/gi.hpp"
#include "ssqa/rng.hpp"
#include "simt_kernels.cuh"
#include "sweep_tc.h"
#include "../../include/ssqa_tune.h"

using namespace ssqa_engine;

namespace ssqa_engine {
TuneOverrides& tune() {
  static TuneOverrides t;
  return t;
}
}  // namespace ssqa_engine

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = code == SSQA_ECUDA ? msg + tc_watchdog_message() : msg;
  return code;
}

#define CU(call)                                                                    \
  do {                                                                              \
    cudaError_t e__ = (call);                                                       \
    if (e__ != cudaSuccess)                                                         \
      return set_err(SSQA_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)

// Batch timing events.  Inside a stream capture (rowshard.capture_run) a plain
// record only orders the capture; the external form makes it a real record
// node, so elapsed-time queries work after every graph replay.
cudaError_t record_event(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, st);
}

#define CHECK_LAUNCH()                                                                 \
  do {                                                                                 \
    cudaError_t e__ = cudaGetLastError();                                              \
    if (e__ != cudaSuccess)                                                            \
      return set_err(SSQA_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e__)); \
  } while (0)

constexpr long kMaxCycles = 1L << 31;  // annealer.cpp:20
constexpr int kMaxReplicas = 1 << 12;  // annealer.cpp:21
constexpr int kMaxSpins = 1 << 20;     // annealer.cpp:22
constexpr double kTargetTol = 1e-9;    // annealer.hpp:113

// annealer.cpp:25-30 + 365-373
int validate(const ssqa_params_c* p, int n) {
  if (!p) return set_err(SSQA_EINVAL, "null params");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  if (p->sc < 1 || p->sc >= kMaxCycles) return set_err(SSQA_EINVAL, "sc out of range");
  if (p->n_rnd < 0.0) return set_err(SSQA_EINVAL, "n_rnd must be >= 0");
  if (p->alpha <= 0.0) return set_err(SSQA_EINVAL, "alpha must be > 0");
  if (p->r < 1 || p->r >= kMaxReplicas)
    return set_err(SSQA_EINVAL, "replica count out of range");
  if (p->jperp_max < p->jperp_min) return set_err(SSQA_EINVAL, "jperp_max < jperp_min");
  if (p->beta < 1) return set_err(SSQA_EINVAL, "beta must be >= 1");
  if (p->tau < 1) return set_err(SSQA_EINVAL, "tau must be >= 1");
  if (p->delay < 0) return set_err(SSQA_EINVAL, "delay must be >= 0");
  if (p->i0 <= 0.0) return set_err(SSQA_EINVAL, "i0 must be > 0");
  return SSQA_OK;
}

// annealer.cpp:375-380, evaluated on the host so the device sees the
// reference's own doubles.
double jperp_at(long cycle, const ssqa_params_c& p) {
  long c = cycle % (long(p.tau) * (p.beta + 1));
  long step = c / p.tau;
  return p.jperp_min + double(step) * (p.jperp_max - p.jperp_min) / p.beta;
}

// annealer.cpp:382-387 (SsaParams::validate) and 389-397 (i0_levels).
int ssa_validate(const ssqa_ssa_params_c* p, int n) {
  if (!p) return set_err(SSQA_EINVAL, "null params");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  if (p->sc < 1 || p->sc >= kMaxCycles) return set_err(SSQA_EINVAL, "sc out of range");
  if (p->n_rnd < 0.0) return set_err(SSQA_EINVAL, "n_rnd must be >= 0");
  if (p->alpha <= 0.0) return set_err(SSQA_EINVAL, "alpha must be > 0");
  if (p->i0_min <= 0.0 || p->i0_min > p->i0_max)
    return set_err(SSQA_EINVAL, "need 0 < i0_min <= i0_max");
  if (p->beta <= 0.0 || p->beta >= 1.0) return set_err(SSQA_EINVAL, "beta must be in (0, 1)");
  if (p->tau < 1) return set_err(SSQA_EINVAL, "tau must be >= 1");
  return SSQA_OK;
}

int ssa_levels(const ssqa_ssa_params_c* p, std::vector<double>* levels) {
  levels->clear();
  for (double v = p->i0_min; v <= p->i0_max * (1.0 + 1e-12); v /= p->beta) {
    levels->push_back(v);
    if (levels->size() > 64) return set_err(SSQA_EINVAL, "i0 schedule has too many levels");
  }
  // The reference would divide by zero here (NaN bounds); refuse instead.
  if (levels->empty()) return set_err(SSQA_EINVAL, "i0 schedule is empty");
  return SSQA_OK;
}

// annealer.cpp:403-408
double i0_level_at(long cycle, const std::vector<double>& levels, int tau) {
  const long c = cycle % (long(levels.size()) * tau);
  return levels[size_t(c / tau)];
}

// The accumulator bound of cycle c: the constant p.i0 of ssqa_run
// (annealer.cpp:485) or the SSA ladder (annealer.cpp:499).
double i0_at(const ssqa_batch_s* b, long cycle) {
  return b->ssa ? i0_level_at(cycle, b->ssa_levels, b->ssa_tau) : b->p.i0;
}

int num_sms(int device) {
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v;
}

// Column tiling: whole trials per tile, as few tiles as the SM count allows.
// tcgen05 engine, large problems: when there are few column tiles and many
// row tiles, widen the tiles (more trials per tile -> each J' row tile is
// streamed by fewer CTAs, larger MMA N) and split each tile's rows over rs
// CTAs (row split, one CTA per SM).  fp4: FP4 operands need tile_cols <= 240.
// CTA pairs pay where the operand feed binds (C4: 64 row tiles, C5: 256);
// at C3's 20 row tiles they cost ~15 % (scripts/geom_sweep.py).
constexpr int kPairMinRowTiles = 64;

Geom make_geom(int n, int npad, int R, int T, int sms, int engine, bool fp4, bool per_trial,
               bool i16 = false) {
  Geom g;
  g.n = n;
  g.npad = npad;
  g.R = R;
  g.T = T;
  // int16 planes: two accumulators per buffer, 4 x tile columns of TMEM
  const int max_cols = i16 ? 128 : 256;
  int tpt = std::max(1, (T + sms - 1) / sms);
  if (R <= max_cols) tpt = std::min(tpt, max_cols / R);
  else tpt = 1;
  tpt = std::max(1, std::min(tpt, T));
  if (per_trial) tpt = 1;  // multi-instance problems: each tile reads its trial's J'
  int rs = 1;
  const int nrt = npad / 128;
  if (engine == SSQA_ENGINE_TCGEN05 && R <= max_cols && !per_trial) {
    // FP4 tiles <= 240 columns (scale-factor TMEM columns); int8 tiles <= 192:
    // smaller operand stages leave room for a deeper TMA pipeline (C4 measured:
    // 0.76 ms/sweep at 192 columns vs 0.84 at 256)
    const int cap = i16 ? 128 : (fp4 ? 240 : 192);
    int wide = std::max(1, std::min(T, cap / R));
    if (tune().wide > 0) wide = std::max(1, std::min(wide, tune().wide));
    const int wtiles = (T + wide - 1) / wide;
    if (nrt >= 16 && nrt < kPairMinRowTiles && tune().wide <= 0) {
      // Mid-size problems (C3's N = 2500 with a short battery, e.g. one GPU's
      // block of a trial-sharded run): epilogue-bound, so pick the (trials per
      // tile, row parts) that minimise the busiest CTA's sweep -- measured on
      // C3 blocks of 128 / 256 / 512 trials (scripts/geom_sweep.py), in units
      // of one epilogue column of one row tile:
      //   whole tiles   nrt * (cols + 40 k) * 1.05            (FP64 epilogue)
      //   row split     ceil(nrt / rs) * (cols + 122 k) + 159 (table epilogue,
      //                 cross-CTA stamps once per pass),  k = npad / 2560
      const double k = double(npad) / 2560.0;
      double best = 1e300;
      int best_tpt = tpt, best_rs = 1;
      for (int w = 1; w <= std::max(1, std::min(T, cap / R)); ++w) {
        const int tiles = (T + w - 1) / w;
        if (tiles > sms) continue;
        const int te = (T + tiles - 1) / tiles;
        const int cols = (te * R + 15) / 16 * 16;
        const double whole = nrt * (cols + 40.0 * k) * 1.05;
        if (whole < best) best = whole, best_tpt = te, best_rs = 1;
        for (int r2 = 2; r2 <= std::min(nrt, sms / tiles); ++r2) {
          const double split = double((nrt + r2 - 1) / r2) * (cols + 122.0 * k) + 159.0;
          if (split < best) best = split, best_tpt = te, best_rs = r2;
        }
      }
      tpt = best_tpt;
      rs = best_rs;
    } else if (nrt >= 16 && wide > tpt && wtiles * 2 <= sms) {
      // worth it when the wide tiling still fills the SMs with >= 2 parts per tile
      tpt = (T + wtiles - 1) / wtiles;  // as even as the tile count allows
      rs = std::min(nrt, sms / wtiles);
      // an even part count lets the parts run as CTA pairs (M = 256 MMAs);
      // worth one idle SM per tile from 5 parts up
      if (rs >= 5 && (rs & 1) && nrt % 2 == 0 && nrt >= kPairMinRowTiles) rs -= 1;
    }
    {
      const int want = tune().rs;  // test / tuning override
      if (want >= 1) {
        const int tiles = (T + tpt - 1) / tpt;
        rs = std::max(1, std::min({want, nrt, std::max(1, sms / tiles)}));
      }
    }
  }
  g.tpt = tpt;
  g.tile_cols = (tpt * R + 15) / 16 * 16;
  g.ntiles = (T + tpt - 1) / tpt;
  g.ccols = g.ntiles * g.tile_cols;
  g.rs = rs;
  return g;
}

template <class T>
int dalloc(T** p, size_t count) {
  CU(pmalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T)));
  return SSQA_OK;
}

void dfree(void* p) {
  if (p) pool_free(p);
}

int8_t* slot_ptr(ssqa_batch_s* b, int s) { return b->d_sig + size_t(s) * b->slot_elems; }

int pick_free(const ssqa_batch_s* b) {
  for (int s = 0; s < b->nslots; ++s) {
    if (s == b->cur) continue;
    if (std::find(b->phys.begin(), b->phys.end(), s) != b->phys.end()) continue;
    return s;
  }
  return -1;  // unreachable: nslots = delay + 3
}

// Give cur and every history snapshot its own slot so one trial's lattice
// can be rewritten without touching the others (ssqa_batch_write_lattice).
int normalize_slots(ssqa_batch_s* b) {
  std::vector<int> roles;
  roles.push_back(b->cur);
  for (int s : b->phys) roles.push_back(s);
  std::vector<int> sorted = roles;
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end()) return SSQA_OK;
  int8_t* fresh = nullptr;
  int rc = dalloc(&fresh, b->slot_elems * b->nslots);
  if (rc) return rc;
  for (size_t r = 0; r < roles.size(); ++r) {
    CU(cudaMemcpyAsync(fresh + r * b->slot_elems, slot_ptr(b, roles[r]), b->slot_elems,
                       cudaMemcpyDeviceToDevice, b->prob->stream));
  }
  CU(cudaStreamSynchronize(b->prob->stream));
  pool_free(b->d_sig);
  b->d_sig = fresh;
  b->cur = 0;
  for (size_t s = 0; s < b->phys.size(); ++s) b->phys[s] = int(s) + 1;
  return SSQA_OK;
}

// One SIMT sweep of the whole batch at b->cycle (update_spins semantics),
// optionally followed by the scan.  do_update = 0 computes energies only.
int simt_sweep(ssqa_batch_s* b, double jperp, double i0, int do_update, const ScanArgs* scan) {
  const Geom& g = b->g;
  cudaStream_t st = b->prob->stream;
  launch_field_simt(g, b->prob->d_J, slot_ptr(b, b->cur), b->d_S, st);
  CHECK_LAUNCH();
  const int src = b->phys[size_t(b->cycle % (b->d + 1))];
  const int dst = do_update ? pick_free(b) : b->cur;
  StepArgs a{b->cycle, jperp, i0, b->p.n_rnd, b->p.alpha, b->p.bidirectional, do_update};
  launch_energy_update_simt(g, b->d_S, b->prob->d_H, b->prob->q.scale, b->d_seeds,
                            slot_ptr(b, b->cur), slot_ptr(b, src), slot_ptr(b, dst), b->d_acc,
                            b->d_E, a, st);
  CHECK_LAUNCH();
  b->launches += 2;
  if (scan) {
    launch_scan(g, b->d_E, *scan, slot_ptr(b, b->cur), b->d_best_e, b->d_best_k, b->d_reached,
                b->d_first_hit, b->d_cycles_used, b->d_active, b->d_best_state, b->d_trace, st);
    CHECK_LAUNCH();
    b->launches += 1;
  }
  if (do_update) {
    b->phys[size_t(b->cycle % (b->d + 1))] = dst;
    b->cur = dst;
    b->cycle += 1;
  }
  return SSQA_OK;
}

int init_state(ssqa_batch_s* b) {
  cudaStream_t st = b->prob->stream;
  b->cur = 0;
  std::fill(b->phys.begin(), b->phys.end(), 0);
  b->cycle = 0;
  b->lattice_stale = false;
  launch_init(b->g, b->d_seeds, slot_ptr(b, 0), b->d_acc, st);
  CHECK_LAUNCH();
  b->launches += 1;
  return SSQA_OK;
}

// FP4 / FP4-pair images of a device-built J' (every instance of the problem),
// with the rules of ssqa_problem_create: the e2m1 image when every coupling
// is representable, otherwise the pair image when every |J'| splits.
cudaError_t build_images(ssqa_problem_s* pr, int* d_stats) {
  Quantized& q = pr->q;
  const size_t np2 = size_t(q.npad) * q.npad, cnt = size_t(pr->count);
  int flag = 0;
  cudaError_t e = cudaSuccess;
  q.fp4_ok = q.max_abs_j <= 6 && q.max_abs_j != 5;
  if (q.fp4_ok) {
    e = cudaMemsetAsync(d_stats, 0, sizeof(int), pr->stream);
    if (e == cudaSuccess) e = pmalloc(&pr->d_J4, cnt * np2 / 2);
    if (e == cudaSuccess) launch_qfp4(pr->d_J, cnt * np2, pr->d_J4, d_stats, pr->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, d_stats, sizeof(int), cudaMemcpyDeviceToHost, pr->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
    if (e == cudaSuccess && flag) {
      q.fp4_ok = false;
      pool_free(pr->d_J4);
      pr->d_J4 = nullptr;
    }
  }
  if (e == cudaSuccess && !q.fp4_ok && fp4x2_splittable(q.max_abs_j)) {
    flag = 0;
    e = cudaMemsetAsync(d_stats, 0, sizeof(int), pr->stream);
    if (e == cudaSuccess) e = pmalloc(&pr->d_J4, cnt * np2);
    for (size_t c = 0; c < cnt && e == cudaSuccess; ++c)
      launch_qfp4x2(pr->d_J + c * np2, q.npad, pr->d_J4 + c * np2, d_stats, pr->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, d_stats, sizeof(int), cudaMemcpyDeviceToHost, pr->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
    q.fp4x2_ok = e == cudaSuccess && !flag;
    if (!q.fp4x2_ok && pr->d_J4) {
      pool_free(pr->d_J4);
      pr->d_J4 = nullptr;
    }
  }
  return e;
}

}  // namespace

extern "C" {

const char* ssqa_last_error(void) { return g_err.c_str(); }

int ssqa_tune_set(const char* key, long value) {
  if (!key) return set_err(SSQA_EINVAL, "ssqa_tune_set: null key");
  TuneOverrides& t = tune();
  const std::string k(key);
  const int v = int(value);
  if (k == "tab") t.tab = v;
  else if (k == "fp4") t.fp4 = v;
  else if (k == "rs") t.rs = v;
  else if (k == "wide") t.wide = v;
  else if (k == "epi") t.epi = v;
  else if (k == "cta2") t.cta2 = v;
  else if (k == "stages") t.stages = v;
  else if (k == "nps") t.nps = v;
  else if (k == "exp") t.exp = v;
  else if (k == "i16") t.i16 = v;
  else if (k == "nccl1") t.nccl1 = v;
  else if (k == "tskip") t.tskip = v;
  else return set_err(SSQA_EINVAL, "ssqa_tune_set: unknown key '" + k + "'");
  return SSQA_OK;
}

int ssqa_tune_trace(const char* path) {
  tune().trace = path ? path : "";
  return SSQA_OK;
}

void ssqa_tune_reset(void) { tune() = TuneOverrides(); }
const char* ssqa_version(void) { return "ssqa-b200 0.1.0"; }

int ssqa_params_validate(const ssqa_params_c* p, int n) { return validate(p, n); }

int ssqa_jperp_schedule(long cycle, const ssqa_params_c* p, double* out) {
  if (cycle < 0) return set_err(SSQA_EINVAL, "cycle must be >= 0");
  *out = jperp_at(cycle, *p);
  return SSQA_OK;
}

int ssqa_problem_create(int n, const double* h, const double* J, double offset, int device,
                        ssqa_problem* out) {
  if (!out || !h || !J) return set_err(SSQA_EINVAL, "null argument");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  // The quantizer of csrc/quantize.cpp, run on the device: the doubles are
  // uploaded once, scanned for the scale, scaled + transposed into J' and
  // packed into the FP4 image there (quantize_kernels.cu); only the n biases
  // and a few scalars go through the host.
  int p = 0;
  for (int i = 0; i < n; ++i) {
    const int e = dyadic_exponent_of(h[i]);
    if (e < 0) return set_err(SSQA_EUNSUP, "bias " + std::to_string(i) + " is not a dyadic rational");
    p = std::max(p, e);
  }
  auto* pr = new ssqa_problem_s();
  Quantized& q = pr->q;
  q.n = n;
  q.npad = (n + 127) / 128 * 128;
  q.offset = offset;
  pr->device = device;
  const size_t nn = size_t(n) * n, np2 = size_t(q.npad) * q.npad;
  double* d_Jd = nullptr;
  int* d_stats = nullptr;  // [0] pmax, [1] maxabs, [2] overflow, [3] not_fp4, [4..5] bad (u64)
  int st[6] = {0, 0, 0, 0, 0, 0};
  std::string fail;
  auto cleanup = [&]() {
    if (d_Jd) pool_free(d_Jd);
    if (d_stats) pool_free(d_stats);
  };
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = pmalloc(&d_Jd, nn * sizeof(double));
  if (e == cudaSuccess) e = pmalloc(&d_stats, sizeof(st));
  if (e == cudaSuccess) e = pmalloc(&pr->d_J, np2);
  if (e == cudaSuccess) {
    const unsigned long long none = ~0ull;
    cudaMemsetAsync(d_stats, 0, sizeof(st), pr->stream);
    cudaMemcpyAsync(d_stats + 4, &none, sizeof(none), cudaMemcpyHostToDevice, pr->stream);
    e = cudaMemcpyAsync(d_Jd, J, nn * sizeof(double), cudaMemcpyHostToDevice, pr->stream);
  }
  if (e == cudaSuccess) {
    launch_qscan(d_Jd, nn, d_stats, reinterpret_cast<unsigned long long*>(d_stats + 4),
                 pr->stream);
    e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
  if (e == cudaSuccess) {
    unsigned long long bad;
    std::memcpy(&bad, st + 4, sizeof bad);
    if (bad != ~0ull) {
      fail = "coupling " + std::to_string(bad / n) + "," + std::to_string(bad % n) +
             " is not a dyadic rational";
    } else {
      p = std::max(p, st[0]);
      launch_qtranspose(d_Jd, n, q.npad, std::ldexp(1.0, p), pr->d_J, d_stats + 1, d_stats + 2,
                        pr->stream);
      e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
      if (e == cudaSuccess && st[2] && tune().i16 != 0) {
        // |J'| > 127: int16 couplings as two int8 planes (engine.h Quantized::i16)
        int16_t* d_J16 = nullptr;
        st[1] = st[2] = 0;
        e = cudaMemcpyAsync(d_stats + 1, st + 1, 2 * sizeof(int), cudaMemcpyHostToDevice, pr->stream);
        if (e == cudaSuccess) e = pmalloc(&d_J16, np2 * sizeof(int16_t));
        if (e == cudaSuccess) {
          launch_qtranspose16(d_Jd, n, q.npad, std::ldexp(1.0, p), d_J16, d_stats + 1,
                              d_stats + 2, pr->stream);
          e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
        if (e == cudaSuccess && !st[2]) {
          pool_free(pr->d_J);
          pr->d_J = nullptr;
          e = pmalloc(&pr->d_J, 2 * np2);
          if (e == cudaSuccess) launch_qplanes16(d_J16, q.npad, reinterpret_cast<uint8_t*>(pr->d_J), pr->stream);
          if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
          q.i16 = true;
        }
        if (d_J16) pool_free(d_J16);
      }
      if (e == cudaSuccess && st[2])
        fail = std::string("coupling magnitude exceeds ") +
               (tune().i16 != 0 ? "int16 (32639)" : "int8") + " at scale 2^" + std::to_string(p);
    }
  }
  if (e == cudaSuccess && fail.empty()) {
    q.p = p;
    q.scale = std::ldexp(1.0, -p);
    q.max_abs_j = st[1];
    // biases: H' = h * 2^p, |H'| < 2^29 keeps S + 2H' inside int32
    std::vector<int32_t> H(size_t(q.npad), 0);
    for (int i = 0; i < n && fail.empty(); ++i) {
      const double x = std::ldexp(h[i], p);
      if (std::fabs(x) >= double(1 << 29))
        fail = "bias magnitude exceeds the int32 field range at scale 2^" + std::to_string(p);
      else
        H[size_t(i)] = int32_t(x);
      q.max_abs_h = std::max(q.max_abs_h, std::abs(H[size_t(i)]));
    }
    if (fail.empty()) {
      e = pmalloc(&pr->d_H, H.size() * sizeof(int32_t));
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(pr->d_H, H.data(), H.size() * sizeof(int32_t),
                            cudaMemcpyHostToDevice, pr->stream);
      // FP4 (e2m1) image when every coupling is 0, +-1, +-2, +-3, +-4 or +-6
      q.fp4_ok = !q.i16 && q.max_abs_j <= 6 && q.max_abs_j != 5;
      if (e == cudaSuccess && q.fp4_ok) {
        e = pmalloc(&pr->d_J4, np2 / 2);
        if (e == cudaSuccess) {
          launch_qfp4(pr->d_J, np2, pr->d_J4, d_stats + 3, pr->stream);
          e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
        if (e == cudaSuccess && st[3]) {
          q.fp4_ok = false;
          pool_free(pr->d_J4);
          pr->d_J4 = nullptr;
        }
      }
      // otherwise the FP4 pair image J' = A1 + A2 (|J'| <= 12, != 11)
      if (e == cudaSuccess && !q.i16 && !q.fp4_ok && fp4x2_splittable(q.max_abs_j)) {
        st[3] = 0;
        e = cudaMemcpyAsync(d_stats + 3, st + 3, sizeof(int), cudaMemcpyHostToDevice, pr->stream);
        if (e == cudaSuccess) e = pmalloc(&pr->d_J4, np2);
        if (e == cudaSuccess) {
          launch_qfp4x2(pr->d_J, q.npad, pr->d_J4, d_stats + 3, pr->stream);
          e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
        q.fp4x2_ok = e == cudaSuccess && !st[3];
        if (!q.fp4x2_ok && pr->d_J4) {
          pool_free(pr->d_J4);
          pr->d_J4 = nullptr;
        }
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
    }
  }
  cleanup();
  if (e != cudaSuccess) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_ECUDA, std::string("problem upload: ") + cudaGetErrorString(e));
  }
  if (!fail.empty()) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_EUNSUP, fail);
  }
  *out = pr;
  return SSQA_OK;
}

int ssqa_problem_fp4(ssqa_problem pr) {
  return !pr ? 0 : pr->q.fp4_ok ? 1 : pr->q.fp4x2_ok ? 2 : 0;
}

int ssqa_problem_int16(ssqa_problem pr) { return pr && pr->q.i16 ? 1 : 0; }

int ssqa_problem_create_many(int count, int n, const double* h, const double* J,
                             const double* offsets, int device, ssqa_problem* out) {
  if (!out || !h || !J || !offsets) return set_err(SSQA_EINVAL, "null argument");
  if (count < 1) return set_err(SSQA_EINVAL, "count must be >= 1");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  const size_t nn = size_t(n) * n;
  // one scale for all instances: the largest exponent any of them needs
  std::vector<ssqa_engine::Quantized> qs(static_cast<size_t>(count));
  std::string why;
  int p = 0;
  for (int c = 0; c < count; ++c) {
    int rc = quantize(n, h + size_t(c) * n, J + size_t(c) * nn, offsets[c], &qs[size_t(c)], &why);
    if (rc) return set_err(rc, "instance " + std::to_string(c) + ": " + why);
    p = std::max(p, qs[size_t(c)].p);
  }
  for (int c = 0; c < count; ++c)
    if (qs[size_t(c)].p != p) {
      int rc = quantize(n, h + size_t(c) * n, J + size_t(c) * nn, offsets[c], &qs[size_t(c)],
                        &why, p);
      if (rc) return set_err(rc, "instance " + std::to_string(c) + ": " + why);
    }
  auto* pr = new ssqa_problem_s();
  pr->q = qs[0];
  pr->count = count;
  bool fp4 = true;
  for (auto& q : qs) {
    pr->q.max_abs_j = std::max(pr->q.max_abs_j, q.max_abs_j);
    pr->q.max_abs_h = std::max(pr->q.max_abs_h, q.max_abs_h);
    fp4 = fp4 && q.fp4_ok;
    pr->offsets.push_back(q.offset);
  }
  pr->q.fp4_ok = fp4;
  // no common single image: the pair image when every instance splits
  bool fp4x2 = !fp4 && fp4x2_splittable(pr->q.max_abs_j);
  pr->q.fp4x2_ok = fp4x2;
  const size_t npad = size_t(pr->q.npad);
  pr->q.J.resize(size_t(count) * npad * npad);
  pr->q.H.resize(size_t(count) * npad);
  if (fp4) pr->q.J4.resize(size_t(count) * npad * (npad / 2));
  else if (fp4x2) pr->q.J4.resize(size_t(count) * npad * npad);
  else pr->q.J4.clear();
  for (int c = 0; c < count; ++c) {
    const Quantized& q = qs[size_t(c)];
    if (c > 0) {
      std::copy(q.J.begin(), q.J.end(), pr->q.J.begin() + size_t(c) * npad * npad);
      std::copy(q.H.begin(), q.H.end(), pr->q.H.begin() + size_t(c) * npad);
      if (fp4) std::copy(q.J4.begin(), q.J4.end(), pr->q.J4.begin() + size_t(c) * npad * (npad / 2));
    }
    if (fp4x2) {
      std::vector<uint8_t> img;
      if (build_fp4x2(q, &img))
        std::copy(img.begin(), img.end(), pr->q.J4.begin() + size_t(c) * npad * npad);
      else
        fp4x2 = false;
    }
  }
  pr->q.fp4x2_ok = fp4x2;
  if (!fp4 && !fp4x2) pr->q.J4.clear();
  qs.clear();
  pr->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = pmalloc(&pr->d_J, pr->q.J.size());
  if (e == cudaSuccess) e = pmalloc(&pr->d_H, pr->q.H.size() * sizeof(int32_t));
  if (e == cudaSuccess) e = pmalloc(&pr->d_offsets, size_t(count) * sizeof(double));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pr->d_J, pr->q.J.data(), pr->q.J.size(), cudaMemcpyHostToDevice, pr->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pr->d_H, pr->q.H.data(), pr->q.H.size() * sizeof(int32_t),
                        cudaMemcpyHostToDevice, pr->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pr->d_offsets, pr->offsets.data(), size_t(count) * sizeof(double),
                        cudaMemcpyHostToDevice, pr->stream);
  if (e == cudaSuccess && (fp4 || fp4x2)) {
    e = pmalloc(&pr->d_J4, pr->q.J4.size());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(pr->d_J4, pr->q.J4.data(), pr->q.J4.size(), cudaMemcpyHostToDevice,
                          pr->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
  if (e != cudaSuccess) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_ECUDA, std::string("problem upload: ") + cudaGetErrorString(e));
  }
  *out = pr;
  return SSQA_OK;
}

// ---- problems built on the device (generate_kernels.cu) -------------------
int ssqa_problem_create_dense(int n, int kind, uint64_t seed, int device, ssqa_problem* out) {
  if (!out) return set_err(SSQA_EINVAL, "null argument");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  if (kind != 0 && kind != 1) return set_err(SSQA_EINVAL, "kind must be 0 or 1");
  auto* pr = new ssqa_problem_s();
  Quantized& q = pr->q;
  q.n = n;
  q.npad = (n + 127) / 128 * 128;
  q.p = 0;  // integer couplings and biases
  q.scale = 1.0;
  q.offset = 0.0;
  pr->device = device;
  int* d_stats = nullptr;
  int st[2] = {0, 0};
  const size_t np2 = size_t(q.npad) * q.npad;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = pmalloc(&d_stats, 4 * sizeof(int));
  if (e == cudaSuccess) e = pmalloc(&pr->d_J, np2);
  if (e == cudaSuccess) e = pmalloc(&pr->d_H, size_t(q.npad) * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_stats, 0, 4 * sizeof(int), pr->stream);
  if (e == cudaSuccess) {
    // CounterRng(seed, 8 / 9).key() (host/instances.cpp: the host builder's streams)
    const uint64_t kj = ssqa::CounterRng(seed, 8).key(), kh = ssqa::CounterRng(seed, 9).key();
    launch_gen_dense(n, q.npad, kind, kj, kh, pr->d_J, pr->d_H, d_stats, d_stats + 1, pr->stream);
    e = cudaMemcpyAsync(st, d_stats, sizeof(st), cudaMemcpyDeviceToHost, pr->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
  if (e == cudaSuccess) {
    q.max_abs_j = st[0];
    q.max_abs_h = st[1];
    e = build_images(pr, d_stats + 2);
  }
  if (d_stats) pool_free(d_stats);
  if (e != cudaSuccess) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_ECUDA, std::string("problem generation: ") + cudaGetErrorString(e));
  }
  *out = pr;
  return SSQA_OK;
}

int ssqa_problem_create_gi(int count, int n_nodes, double edge_prob, const uint64_t* seeds,
                           int permute, double c1, double c2, int device, ssqa_problem* out) {
  if (!out || !seeds) return set_err(SSQA_EINVAL, "null argument");
  if (count < 1) return set_err(SSQA_EINVAL, "count must be >= 1");
  if (n_nodes < 1 || size_t(n_nodes) * n_nodes >= size_t(kMaxSpins))
    return set_err(SSQA_EINVAL, "n_nodes out of range");
  const int nn = n_nodes, N = nn * nn;
  std::vector<uint8_t> adj(size_t(count) * 2 * nn * nn);
  std::vector<double> h(size_t(N));
  std::vector<double> offsets(static_cast<size_t>(count));
  auto* pr = new ssqa_problem_s();
  Quantized& q = pr->q;
  q.n = N;
  q.npad = (N + 127) / 128 * 128;
  pr->count = count;
  pr->device = device;
  std::vector<int32_t> H(size_t(count) * q.npad, 0);
  std::string fail;
  int p = 0, jo = 0, jm = 0;
  try {
    // couplings -2 c1 / 4 (one-hot) and -c2 / 4 (edge mismatch)
    const double jo_d = -0.25 * (2.0 * c1), jm_d = -0.25 * c2;
    const int e1 = dyadic_exponent_of(jo_d), e2 = dyadic_exponent_of(jm_d);
    if (e1 < 0 || e2 < 0) throw std::invalid_argument("GI penalties must be dyadic rationals");
    std::vector<std::vector<double>> hs(static_cast<size_t>(count));
    for (int c = 0; c < count; ++c) {
      hs[size_t(c)].resize(size_t(N));
      ssqa::gi_compact(ssqa::generate_gi(nn, edge_prob, seeds[c], permute != 0, c1, c2),
                       adj.data() + size_t(c) * 2 * nn * nn, hs[size_t(c)].data(),
                       &offsets[size_t(c)]);
    }
    // the scale the quantizer would find: every coupling value present and
    // every bias.  One-hot couplings exist from n = 2; edge-mismatch ones in
    // an instance with 0 < |E| < n(n-1)/2 edges.
    p = nn >= 2 ? e1 : 0;
    for (int c = 0; c < count; ++c) {
      long m2 = 0;  // 2 |E1|
      for (int x = 0; x < nn * nn; ++x) m2 += adj[size_t(c) * 2 * nn * nn + size_t(x)];
      if (m2 > 0 && m2 < long(nn) * (nn - 1)) p = std::max(p, e2);
    }
    for (auto& hv : hs)
      for (double v : hv) {
        const int e = dyadic_exponent_of(v);
        if (e < 0) throw std::invalid_argument("bias is not a dyadic rational");
        p = std::max(p, e);
      }
    jo = int(std::ldexp(jo_d, p));
    jm = int(std::ldexp(jm_d, p));
    if (std::abs(jo) > 127 || std::abs(jm) > 127)
      throw std::invalid_argument("coupling magnitude exceeds int8 at scale 2^" + std::to_string(p));
    for (int c = 0; c < count; ++c)
      for (int i = 0; i < N; ++i) {
        const double x = std::ldexp(hs[size_t(c)][size_t(i)], p);
        if (std::fabs(x) >= double(1 << 29))
          throw std::invalid_argument("bias magnitude exceeds the int32 field range");
        H[size_t(c) * q.npad + size_t(i)] = int32_t(x);
        q.max_abs_h = std::max(q.max_abs_h, std::abs(int32_t(x)));
      }
  } catch (const std::exception& ex) {
    fail = ex.what();
  }
  if (!fail.empty()) {
    delete pr;
    return set_err(SSQA_EUNSUP, fail);
  }
  q.p = p;
  q.scale = std::ldexp(1.0, -p);
  q.offset = offsets[0];
  pr->offsets = offsets;
  const size_t np2 = size_t(q.npad) * q.npad;
  uint8_t* d_adj = nullptr;
  int* d_stats = nullptr;
  int mj = 0;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = pmalloc(&d_stats, 4 * sizeof(int));
  if (e == cudaSuccess) e = pmalloc(&d_adj, adj.size());
  if (e == cudaSuccess) e = pmalloc(&pr->d_J, size_t(count) * np2);
  if (e == cudaSuccess) e = pmalloc(&pr->d_H, H.size() * sizeof(int32_t));
  if (e == cudaSuccess) e = pmalloc(&pr->d_offsets, size_t(count) * sizeof(double));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_stats, 0, 4 * sizeof(int), pr->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_adj, adj.data(), adj.size(), cudaMemcpyHostToDevice, pr->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pr->d_H, H.data(), H.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                        pr->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(pr->d_offsets, offsets.data(), size_t(count) * sizeof(double),
                        cudaMemcpyHostToDevice, pr->stream);
  if (e == cudaSuccess) {
    launch_gen_gi(count, nn, q.npad, jo, jm, d_adj, pr->d_J, d_stats, pr->stream);
    e = cudaMemcpyAsync(&mj, d_stats, sizeof(int), cudaMemcpyDeviceToHost, pr->stream);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
  if (e == cudaSuccess) {
    q.max_abs_j = mj;
    e = build_images(pr, d_stats + 2);
  }
  if (d_adj) pool_free(d_adj);
  if (d_stats) pool_free(d_stats);
  if (e != cudaSuccess) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_ECUDA, std::string("problem generation: ") + cudaGetErrorString(e));
  }
  *out = pr;
  return SSQA_OK;
}

int ssqa_problem_create_zero(int n, int device, ssqa_problem* out) {
  if (!out) return set_err(SSQA_EINVAL, "null argument");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  auto* pr = new ssqa_problem_s();
  Quantized& q = pr->q;
  q.n = n;
  q.npad = (n + 127) / 128 * 128;
  q.fp4_ok = true;  // all-zero couplings are e2m1-exact
  pr->device = device;
  const size_t np2 = size_t(q.npad) * q.npad;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pr->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = pmalloc(&pr->d_J, np2);
  if (e == cudaSuccess) e = pmalloc(&pr->d_J4, np2 / 2);
  if (e == cudaSuccess) e = pmalloc(&pr->d_H, size_t(q.npad) * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(pr->d_J, 0, np2, pr->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(pr->d_J4, 0, np2 / 2, pr->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(pr->d_H, 0, size_t(q.npad) * sizeof(int32_t), pr->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(pr->stream);
  if (e != cudaSuccess) {
    ssqa_problem_destroy(pr);
    return set_err(SSQA_ECUDA, std::string("problem allocation: ") + cudaGetErrorString(e));
  }
  *out = pr;
  return SSQA_OK;
}

int ssqa_problem_export(ssqa_problem pr, int8_t* J, int32_t* H, double* offsets) {
  if (!pr) return set_err(SSQA_EINVAL, "null problem");
  CU(cudaSetDevice(pr->device));
  CU(cudaStreamSynchronize(pr->stream));
  const size_t np = size_t(pr->q.npad), cnt = size_t(pr->count);
  if (J) CU(cudaMemcpy(J, pr->d_J, cnt * np * np * (pr->q.i16 ? 2 : 1), cudaMemcpyDeviceToHost));
  if (H) CU(cudaMemcpy(H, pr->d_H, cnt * np * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (offsets) {
    if (pr->count > 1) std::copy(pr->offsets.begin(), pr->offsets.end(), offsets);
    else offsets[0] = pr->q.offset;
  }
  return SSQA_OK;
}

int ssqa_problem_count(ssqa_problem pr) { return pr ? pr->count : 0; }

int ssqa_quantize_info(int n, const double* h, const double* J, int* n_pad, int* shift_p,
                       int* max_abs_j, int* max_abs_h) {
  if (!h || !J) return set_err(SSQA_EINVAL, "null argument");
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  Quantized q;
  std::string why;
  int rc = quantize(n, h, J, 0.0, &q, &why);
  if (rc) return set_err(rc, why);
  if (n_pad) *n_pad = q.npad;
  if (shift_p) *shift_p = q.p;
  if (max_abs_j) *max_abs_j = q.max_abs_j;
  if (max_abs_h) *max_abs_h = q.max_abs_h;
  return SSQA_OK;
}

int ssqa_plan_geometry(int n, int replicas, int trials, int sms, int operand_bits,
                       int* tile_cols, int* tiles, int* trials_per_tile, int* row_parts) {
  if (n < 1 || n >= kMaxSpins) return set_err(SSQA_EINVAL, "spin count out of range");
  if (replicas < 1 || trials < 1 || sms < 1) return set_err(SSQA_EINVAL, "bad batch shape");
  if (operand_bits != 4 && operand_bits != 8) return set_err(SSQA_EINVAL, "operand bits: 4 or 8");
  const int npad = (n + 127) / 128 * 128;
  const Geom g = make_geom(n, npad, replicas, trials, sms, SSQA_ENGINE_TCGEN05, operand_bits == 4,
                           false);
  if (tile_cols) *tile_cols = g.tile_cols;
  if (tiles) *tiles = g.ntiles;
  if (trials_per_tile) *trials_per_tile = g.tpt;
  if (row_parts) *row_parts = g.rs;
  return SSQA_OK;
}

int ssqa_problem_destroy(ssqa_problem pr) {
  if (!pr) return SSQA_OK;
  cudaSetDevice(pr->device);
  // blocks go back to the pool (devpool.h): nothing may still read them
  if (pr->stream) cudaStreamSynchronize(pr->stream);
  dfree(pr->d_J);
  dfree(pr->d_H);
  dfree(pr->d_J4);
  dfree(pr->d_offsets);
  if (pr->stream) cudaStreamDestroy(pr->stream);
  delete pr;
  return SSQA_OK;
}

int ssqa_problem_info(ssqa_problem pr, int* n, int* n_pad, int* shift_p, int* max_abs_j,
                      int* max_abs_h) {
  if (!pr) return set_err(SSQA_EINVAL, "null problem");
  if (n) *n = pr->q.n;
  if (n_pad) *n_pad = pr->q.npad;
  if (shift_p) *shift_p = pr->q.p;
  if (max_abs_j) *max_abs_j = pr->q.max_abs_j;
  if (max_abs_h) *max_abs_h = pr->q.max_abs_h;
  return SSQA_OK;
}

}  // extern "C"

namespace {

// Shared by ssqa_batch_create and ssqa_batch_create_ssa; `levels`/`tau`
// describe an SSA bound ladder (levels == nullptr for SSQA batches).
int create_batch(ssqa_problem pr, const ssqa_params_c* p, int trials, int record_trace,
                 int engine, const std::vector<double>* levels, int tau, ssqa_batch* out) {
  int rc = SSQA_OK;
  if (trials < 1) return set_err(SSQA_EINVAL, "trials must be >= 1");
  if (pr->count > 1) {
    if (trials != pr->count)
      return set_err(SSQA_EINVAL, "a multi-instance problem needs one trial per instance");
    if (engine == SSQA_ENGINE_SIMT)
      return set_err(SSQA_EUNSUP, "multi-instance problems need the tcgen05 engine");
  }
  CU(cudaSetDevice(pr->device));
  int eng = engine;
  // int16 couplings: tcgen05 only, tiles of <= 128 replica columns
  const bool tc_ok = tc_supported(pr->q.npad, p->r, p->delay) && (!pr->q.i16 || p->r <= 128);
  if (eng == SSQA_ENGINE_AUTO) eng = tc_ok ? SSQA_ENGINE_TCGEN05 : SSQA_ENGINE_SIMT;
  if (eng == SSQA_ENGINE_TCGEN05 && !tc_ok)
    return set_err(SSQA_EUNSUP, "tcgen05 engine does not support this shape");
  if (pr->q.i16 && eng != SSQA_ENGINE_TCGEN05)
    return set_err(SSQA_EUNSUP, "int16 couplings need the tcgen05 engine (replicas <= 128)");
  if (pr->count > 1 && eng != SSQA_ENGINE_TCGEN05)
    return set_err(SSQA_EUNSUP, "multi-instance problems need the tcgen05 engine");
  if (eng != SSQA_ENGINE_SIMT && eng != SSQA_ENGINE_TCGEN05)
    return set_err(SSQA_EINVAL, "unknown engine");

  auto* b = new ssqa_batch_s();
  b->prob = pr;
  b->p = *p;
  if (levels) {
    b->ssa = true;
    b->ssa_levels = *levels;
    b->ssa_tau = tau;
  }
  b->engine = eng;
  b->record_trace = record_trace;
  b->d = p->delay;
  b->nslots = p->delay + 3;
  const bool any_fp4 = pr->q.fp4_ok || pr->q.fp4x2_ok;
  b->g = make_geom(pr->q.n, pr->q.npad, p->r, trials, num_sms(pr->device), eng, any_fp4,
                   pr->count > 1, pr->q.i16);
  b->slot_elems = size_t(b->g.ccols) * b->g.npad;
  b->phys.assign(size_t(b->d) + 1, 0);
  const int T = trials;
  rc = SSQA_OK;
  auto A = [&](auto** ptr, size_t count) {
    if (rc == SSQA_OK) rc = dalloc(ptr, count);
  };
  A(&b->d_sig, b->slot_elems * b->nslots);
  A(&b->d_acc, b->slot_elems);
  A(&b->d_seeds, size_t(T));
  A(&b->d_jperp, size_t(p->sc) + 1);
  A(&b->d_E, size_t(b->g.ccols));
  if (eng == SSQA_ENGINE_SIMT) A(&b->d_S, b->slot_elems);
  if (eng == SSQA_ENGINE_TCGEN05 && any_fp4) A(&b->d_sig4, b->slot_elems * b->nslots / 2);
  A(&b->d_best_e, size_t(T));
  A(&b->d_best_k, size_t(T));
  A(&b->d_reached, size_t(T));
  A(&b->d_first_hit, size_t(T));
  A(&b->d_cycles_used, size_t(T));
  A(&b->d_active, size_t(T));
  A(&b->d_best_state, size_t(T) * pr->q.n);
  if (eng == SSQA_ENGINE_TCGEN05) A(&b->d_best_packed, size_t(T) * pr->q.npad);
  if (record_trace) A(&b->d_trace, size_t(T) * (p->sc + 1) * p->r);
  if (levels) A(&b->d_i0, size_t(p->sc) + 1);
  if (rc) {
    ssqa_batch_destroy(b);
    return rc;
  }
  // any failure from here on releases the batch (and its pool blocks)
  auto init = [&]() -> int {
    std::vector<double> jp(size_t(p->sc) + 1);
    for (long c = 0; c <= p->sc; ++c) jp[size_t(c)] = jperp_at(c, *p);
    CU(cudaMemcpy(b->d_jperp, jp.data(), jp.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (levels) {
      std::vector<double> i0t(size_t(p->sc) + 1);
      for (long c = 0; c <= p->sc; ++c) i0t[size_t(c)] = i0_at(b, c);
      CU(cudaMemcpy(b->d_i0, i0t.data(), i0t.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    CU(cudaMemset(b->d_sig, 0, b->slot_elems * b->nslots));
    if (b->d_sig4) CU(cudaMemset(b->d_sig4, 0, b->slot_elems * b->nslots / 2));
    CU(cudaMemset(b->d_acc, 0, b->slot_elems * sizeof(double)));
    CU(cudaEventCreate(&b->ev0));
    CU(cudaEventCreate(&b->ev1));
    return SSQA_OK;
  };
  rc = init();
  if (rc) {
    const std::string keep = g_err;
    ssqa_batch_destroy(b);
    g_err = keep;
    return rc;
  }
  *out = b;
  return SSQA_OK;
}

}  // namespace

extern "C" {

int ssqa_batch_create(ssqa_problem pr, const ssqa_params_c* p, int trials, int record_trace,
                      int engine, ssqa_batch* out) {
  if (!pr || !out) return set_err(SSQA_EINVAL, "null argument");
  int rc = validate(p, pr->q.n);
  if (rc) return rc;
  return create_batch(pr, p, trials, record_trace, engine, nullptr, 1, out);
}

int ssqa_ssa_params_validate(const ssqa_ssa_params_c* p, int n) {
  int rc = ssa_validate(p, n);
  if (rc) return rc;
  std::vector<double> levels;
  return ssa_levels(p, &levels);
}

int ssqa_i0_schedule(long cycle, const ssqa_ssa_params_c* p, double* out) {
  if (!p || !out) return set_err(SSQA_EINVAL, "null argument");
  if (cycle < 0) return set_err(SSQA_EINVAL, "cycle must be >= 0");
  std::vector<double> levels;
  int rc = ssa_levels(p, &levels);
  if (rc) return rc;
  *out = i0_level_at(cycle, levels, p->tau);
  return SSQA_OK;
}

int ssqa_i0_levels(const ssqa_ssa_params_c* p, double* out, int* count) {
  if (!p || !out || !count) return set_err(SSQA_EINVAL, "null argument");
  std::vector<double> levels;
  int rc = ssa_levels(p, &levels);
  if (rc) return rc;
  std::copy(levels.begin(), levels.end(), out);
  *count = int(levels.size());
  return SSQA_OK;
}

int ssqa_batch_create_ssa(ssqa_problem pr, const ssqa_ssa_params_c* p, int trials,
                          int record_trace, int engine, ssqa_batch* out) {
  if (!pr || !out) return set_err(SSQA_EINVAL, "null argument");
  int rc = ssa_validate(p, pr->q.n);
  if (rc) return rc;
  std::vector<double> levels;
  rc = ssa_levels(p, &levels);
  if (rc) return rc;
  // LatticeRunSpec of ssa_run (annealer.cpp:492-500): one replica, no delay,
  // jperp == 0 (jperp_schedule of this struct is +0.0 at every cycle).
  ssqa_params_c q{};
  q.r = 1;
  q.jperp_min = 0.0;
  q.jperp_max = 0.0;
  q.beta = 1;
  q.tau = 1;
  q.delay = 0;
  q.i0 = levels[0];
  q.n_rnd = p->n_rnd;
  q.alpha = p->alpha;
  q.sc = p->sc;
  q.bidirectional = 0;
  return create_batch(pr, &q, trials, record_trace, engine, &levels, p->tau, out);
}

int ssqa_ssa_run_batch(ssqa_problem prob, const ssqa_ssa_params_c* p, const uint64_t* seeds,
                       int trials, int has_target, double target, int record_trace,
                       int stop_at_target, int engine, ssqa_result_c* results,
                       int8_t* best_states, double* trace) {
  ssqa_batch b = nullptr;
  int rc = ssqa_batch_create_ssa(prob, p, trials, record_trace, engine, &b);
  if (rc) return rc;
  rc = ssqa_batch_set_seeds(b, seeds);
  if (!rc) rc = ssqa_batch_launch(b, has_target, target, stop_at_target);
  if (!rc) rc = ssqa_batch_fetch(b, results, best_states, record_trace ? trace : nullptr);
  std::string keep = g_err;
  ssqa_batch_destroy(b);
  g_err = keep;
  return rc;
}

int ssqa_batch_destroy(ssqa_batch b) {
  if (!b) return SSQA_OK;
  cudaSetDevice(b->prob->device);
  cudaStreamSynchronize(b->prob->stream);
  for (void* ptr : {(void*)b->d_sig, (void*)b->d_sig4, (void*)b->d_acc, (void*)b->d_seeds, (void*)b->d_jperp, (void*)b->d_i0, b->d_split,
                    (void*)b->d_S, (void*)b->d_E, (void*)b->d_best_e, (void*)b->d_best_k,
                    (void*)b->d_reached, (void*)b->d_first_hit, (void*)b->d_cycles_used,
                    (void*)b->d_active, (void*)b->d_best_state, (void*)b->d_best_packed,
                    (void*)b->d_trace, (void*)b->d_push_ctr})
    dfree(ptr);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  delete b;
  return SSQA_OK;
}

void* ssqa_batch_stream(ssqa_batch b) { return b ? (void*)b->prob->stream : nullptr; }
int ssqa_batch_engine(ssqa_batch b) { return b ? b->engine : -1; }
int ssqa_batch_operand_bits(ssqa_batch b) {
  if (!b) return -1;
  return (b->engine == SSQA_ENGINE_TCGEN05 && tc_uses_fp4(b)) ? 4 : 8;
}
long ssqa_batch_launch_count(ssqa_batch b) { return b ? b->launches : -1; }

int ssqa_batch_elapsed_ms(ssqa_batch b, double* ms) {
  if (!b || !ms) return set_err(SSQA_EINVAL, "null argument");
  CU(cudaSetDevice(b->prob->device));
  CU(cudaEventSynchronize(b->ev1));
  float f = 0.f;
  CU(cudaEventElapsedTime(&f, b->ev0, b->ev1));
  *ms = double(f);
  return SSQA_OK;
}

int ssqa_batch_synchronize(ssqa_batch b) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  CU(cudaSetDevice(b->prob->device));
  CU(cudaStreamSynchronize(b->prob->stream));
  return SSQA_OK;
}

int ssqa_batch_profile_field(ssqa_batch b, int iters, double* ms_per_launch) {
  if (!b || !ms_per_launch || iters < 1) return set_err(SSQA_EINVAL, "bad argument");
  if (b->prob->count > 1) return set_err(SSQA_EUNSUP, "field profile of a multi-instance batch");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  int32_t* S = b->d_S;
  bool tmp = false;
  if (!S) {
    int rc = dalloc(&S, b->slot_elems);
    if (rc) return rc;
    tmp = true;
  }
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  CU(cudaEventRecord(e0, st));
  for (int i = 0; i < iters; ++i) launch_field_simt(b->g, b->prob->d_J, slot_ptr(b, b->cur), S, st);
  CHECK_LAUNCH();
  CU(cudaEventRecord(e1, st));
  CU(cudaEventSynchronize(e1));
  float f = 0.f;
  CU(cudaEventElapsedTime(&f, e0, e1));
  *ms_per_launch = double(f) / iters;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (tmp) pool_free(S);
  return SSQA_OK;
}

int ssqa_batch_set_seeds(ssqa_batch b, const uint64_t* seeds) {
  if (!b || !seeds) return set_err(SSQA_EINVAL, "null argument");
  CU(cudaSetDevice(b->prob->device));
  CU(cudaMemcpyAsync(b->d_seeds, seeds, size_t(b->g.T) * sizeof(uint64_t),
                     cudaMemcpyHostToDevice, b->prob->stream));
  CU(cudaStreamSynchronize(b->prob->stream));
  b->seeds_set = true;
  return SSQA_OK;
}

int ssqa_batch_launch(ssqa_batch b, int has_target, double target, int stop_at_target) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  if (!b->seeds_set) return set_err(SSQA_EINVAL, "seeds not set");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  b->launches = 0;
  CU(record_event(b->ev0, st));
  launch_reset_results(b->g.T, b->p.sc, b->d_best_e, b->d_best_k, b->d_reached,
                       b->d_first_hit, b->d_cycles_used, b->d_active, st);
  CHECK_LAUNCH();
  b->launches += 1;
  int rc = init_state(b);
  if (rc) return rc;
  ScanArgs sa{};
  sa.sc = b->p.sc;
  sa.scale = b->prob->q.scale;
  sa.offset = b->prob->q.offset;
  sa.has_target = has_target;
  sa.target_tol = target + kTargetTol;
  sa.stop_at_target = stop_at_target;
  sa.record_trace = b->record_trace;
  if (b->engine == SSQA_ENGINE_TCGEN05) {
    rc = tc_run(b, sa);
    if (rc) return set_err(rc, tc_last_error());
  } else {
    for (long c = 0; c <= b->p.sc; ++c) {
      sa.cycle = c;
      const double jp = jperp_at(c, b->p);
      rc = simt_sweep(b, jp, i0_at(b, c), c < b->p.sc ? 1 : 0, &sa);
      if (rc) return rc;
    }
  }
  CU(record_event(b->ev1, st));
  return SSQA_OK;
}

int ssqa_batch_fetch(ssqa_batch b, ssqa_result_c* results, int8_t* best_states,
                     double* trace) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  CU(cudaStreamSynchronize(st));
  const int T = b->g.T;
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, b->ev0, b->ev1));
  if (results) {
    std::vector<double> be(T);
    std::vector<int> bk(T), re(T);
    std::vector<long> fh(T), cu(T);
    CU(cudaMemcpy(be.data(), b->d_best_e, T * sizeof(double), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(bk.data(), b->d_best_k, T * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(re.data(), b->d_reached, T * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(fh.data(), b->d_first_hit, T * sizeof(long), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(cu.data(), b->d_cycles_used, T * sizeof(long), cudaMemcpyDeviceToHost));
    for (int t = 0; t < T; ++t) {
      results[t].best_energy = be[t];
      results[t].best_replica = bk[t];
      results[t].reached_target = re[t];
      results[t].first_hit_cycle = fh[t];
      results[t].cycles_used = cu[t];
      results[t].wall_seconds = 1e-3 * double(ms) / T;
    }
  }
  if (best_states)
    CU(cudaMemcpy(best_states, b->d_best_state, size_t(T) * b->g.n, cudaMemcpyDeviceToHost));
  if (trace) {
    if (!b->record_trace) return set_err(SSQA_EINVAL, "batch was created without a trace");
    CU(cudaMemcpy(trace, b->d_trace, size_t(T) * (b->p.sc + 1) * b->p.r * sizeof(double),
                  cudaMemcpyDeviceToHost));
  }
  return SSQA_OK;
}

int ssqa_run_batch(ssqa_problem prob, const ssqa_params_c* p, const uint64_t* seeds,
                   int trials, int has_target, double target, int record_trace,
                   int stop_at_target, int engine, ssqa_result_c* results,
                   int8_t* best_states, double* trace) {
  ssqa_batch b = nullptr;
  int rc = ssqa_batch_create(prob, p, trials, record_trace, engine, &b);
  if (rc) return rc;
  rc = ssqa_batch_set_seeds(b, seeds);
  if (!rc) rc = ssqa_batch_launch(b, has_target, target, stop_at_target);
  if (!rc) rc = ssqa_batch_fetch(b, results, best_states, record_trace ? trace : nullptr);
  std::string keep = g_err;
  ssqa_batch_destroy(b);
  g_err = keep;
  return rc;
}

// ---- GPU row shards ------------------------------------
int ssqa_batch_set_shard(ssqa_batch b, int shard, int nshards) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  if (nshards < 1 || shard < 0 || shard >= nshards)
    return set_err(SSQA_EINVAL, "shard index out of range");
  if (b->engine != SSQA_ENGINE_TCGEN05)
    return set_err(SSQA_EUNSUP, "row shards need the tcgen05 engine");
  const int nrt = b->g.npad / 128;
  if (nrt % nshards != 0)
    return set_err(SSQA_EUNSUP, "padded spin count / 128 must divide into the shards");
  if (b->prob->count > 1) return set_err(SSQA_EUNSUP, "row shards of a multi-instance problem");
  if (b->d > 30) return set_err(SSQA_EUNSUP, "tcgen05 engine supports delay <= 30");
  b->shard = shard;
  b->nshards = nshards;
  return SSQA_OK;
}

long ssqa_batch_shard_bytes(ssqa_batch b) {
  if (!b) return -1;
  const long rows = long(b->g.npad) / b->nshards;
  return long(b->g.ccols) * (rows / 32) * 4 + long(b->g.ccols) * 8;
}

int ssqa_batch_shard_begin(ssqa_batch b, int has_target, double target, int stop_at_target) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  if (!b->seeds_set) return set_err(SSQA_EINVAL, "seeds not set");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  b->launches = 0;
  CU(record_event(b->ev0, st));
  launch_reset_results(b->g.T, b->p.sc, b->d_best_e, b->d_best_k, b->d_reached,
                       b->d_first_hit, b->d_cycles_used, b->d_active, st);
  CHECK_LAUNCH();
  b->launches += 1;
  int rc = init_state(b);
  if (rc) return rc;
  // FP4 / FP4-pair operands: the passes read and write the FP4 spin slots
  if (tc_uses_fp4(b)) {
    launch_pack_fp4(b->d_sig, b->d_sig4, size_t(b->nslots) * b->slot_elems / 2, st);
    CHECK_LAUNCH();
    b->launches += 1;
  }
  b->sh_has_target = has_target;
  b->sh_target_tol = target + kTargetTol;
  b->sh_stop = stop_at_target;
  return SSQA_OK;
}

}  // extern "C"

namespace {

int shard_scan_advance(ssqa_batch b, bool upd, int dst);

int shard_pass(ssqa_batch b, const PeerPush& pp) {
  if (b->cycle > b->p.sc) return set_err(SSQA_EINVAL, "run already complete");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  const int nrt = b->g.npad / 128 / b->nshards;
  CU(cudaMemsetAsync(b->d_E, 0, size_t(b->g.ccols) * sizeof(long long), st));
  int rc = tc_shard_pass(b, b->shard * nrt, nrt, reinterpret_cast<unsigned long long*>(b->d_E));
  if (rc) return set_err(rc, tc_last_error());
  // sigma(c+1) rows of this shard sit in the slot the kernel picked (ring rule)
  const int dst = b->cycle < b->p.sc ? pick_free(b) : b->cur;
  if (tc_uses_fp4(b))
    launch_shard_pack_fp4(b->g, b->d_sig4 + size_t(dst) * b->slot_elems / 2, b->shard * nrt * 128,
                          nrt * 128, reinterpret_cast<const unsigned long long*>(b->d_E), pp, st);
  else
    launch_shard_pack(b->g, slot_ptr(b, dst), b->shard * nrt * 128, nrt * 128,
                      reinterpret_cast<const unsigned long long*>(b->d_E), pp, st);
  CHECK_LAUNCH();
  b->launches += 2;
  return SSQA_OK;
}

int shard_merge(ssqa_batch b, const void* chunks, const PeerWait& pw) {
  if (b->cycle > b->p.sc) return set_err(SSQA_EINVAL, "run already complete");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  const bool upd = b->cycle < b->p.sc;
  const int dst = upd ? pick_free(b) : b->cur;
  uint8_t* dst4 = tc_uses_fp4(b) ? b->d_sig4 + size_t(dst) * b->slot_elems / 2 : nullptr;
  launch_shard_unpack(b->g, slot_ptr(b, dst), dst4, chunks, size_t(ssqa_batch_shard_bytes(b)),
                      b->nshards, b->g.npad / b->nshards, upd, b->d_E, pw, st);
  CHECK_LAUNCH();
  return shard_scan_advance(b, upd, dst);
}

// after a merge: scan cycle c on the merged energies, advance the slot ring
int shard_scan_advance(ssqa_batch b, bool upd, int dst) {
  cudaStream_t st = b->prob->stream;
  ScanArgs sa{};
  sa.cycle = b->cycle;
  sa.sc = b->p.sc;
  sa.scale = b->prob->q.scale;
  sa.offset = b->prob->q.offset;
  sa.has_target = b->sh_has_target;
  sa.target_tol = b->sh_target_tol;
  sa.stop_at_target = b->sh_stop;
  sa.record_trace = b->record_trace;
  launch_scan(b->g, b->d_E, sa, slot_ptr(b, b->cur), b->d_best_e, b->d_best_k, b->d_reached,
              b->d_first_hit, b->d_cycles_used, b->d_active, b->d_best_state, b->d_trace, st);
  CHECK_LAUNCH();
  b->launches += 2;
  if (upd) {
    b->phys[size_t(b->cycle % (b->d + 1))] = dst;
    b->cur = dst;
  }
  b->cycle += 1;  // sc + 1 marks the run complete
  return SSQA_OK;
}

}  // namespace

extern "C" {

int ssqa_batch_shard_pass(ssqa_batch b, void* chunk) {
  if (!b || !chunk) return set_err(SSQA_EINVAL, "null argument");
  PeerPush pp{};
  pp.dst[0] = static_cast<uint8_t*>(chunk);
  pp.n = 1;
  return shard_pass(b, pp);
}

int ssqa_batch_shard_merge(ssqa_batch b, const void* chunks) {
  if (!b || !chunks) return set_err(SSQA_EINVAL, "null argument");
  return shard_merge(b, chunks, PeerWait{nullptr, 0u, 0});
}

int ssqa_batch_shard_pass_to(ssqa_batch b, void* const* dests, unsigned* const* flags, int ndest,
                             unsigned epoch) {
  if (!b || !dests || !flags) return set_err(SSQA_EINVAL, "null argument");
  if (ndest < 1 || ndest > kMaxPeers) return set_err(SSQA_EINVAL, "1..8 destinations");
  CU(cudaSetDevice(b->prob->device));
  if (!b->d_push_ctr) {
    int rc = dalloc(&b->d_push_ctr, 1);
    if (rc) return rc;
    CU(cudaMemsetAsync(b->d_push_ctr, 0, sizeof(unsigned), b->prob->stream));
  }
  PeerPush pp{};
  for (int d = 0; d < ndest; ++d) {
    if (!dests[d] || !flags[d]) return set_err(SSQA_EINVAL, "null destination");
    pp.dst[d] = static_cast<uint8_t*>(dests[d]);
    pp.flag[d] = flags[d];
  }
  pp.n = ndest;
  pp.counter = b->d_push_ctr;
  pp.epoch = epoch;
  return shard_pass(b, pp);
}

int ssqa_batch_shard_merge_from(ssqa_batch b, const void* chunks, const unsigned* flags,
                                int nflags, unsigned epoch) {
  if (!b || !chunks || !flags) return set_err(SSQA_EINVAL, "null argument");
  if (nflags != b->nshards) return set_err(SSQA_EINVAL, "one flag per shard");
  return shard_merge(b, chunks, PeerWait{flags, epoch, nflags});
}

int ssqa_batch_shard_direct_ok(ssqa_batch b) {
  return (b && b->engine == SSQA_ENGINE_TCGEN05 && b->prob->count == 1 && tc_shard_direct_ok(b))
             ? 1 : 0;
}

int ssqa_batch_sig4(ssqa_batch b, void** dev_ptr_out) {
  if (!b || !dev_ptr_out) return set_err(SSQA_EINVAL, "null argument");
  if (!b->d_sig4) return set_err(SSQA_EUNSUP, "batch has no FP4 spin slots");
  *dev_ptr_out = b->d_sig4;
  return SSQA_OK;
}

int ssqa_batch_shard_pass_direct(ssqa_batch b, void* const* peer_sig4, void* const* peer_parts,
                                 unsigned* const* flags, int npeer, unsigned epoch) {
  if (!b || !peer_sig4 || !peer_parts || !flags) return set_err(SSQA_EINVAL, "null argument");
  if (npeer < 1 || npeer > kMaxPeers) return set_err(SSQA_EINVAL, "1..8 peers");
  if (b->cycle > b->p.sc) return set_err(SSQA_EINVAL, "run already complete");
  if (!ssqa_batch_shard_direct_ok(b))
    return set_err(SSQA_EUNSUP, "fused shard exchange needs FP4 operands and the table epilogue");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  if (!b->d_push_ctr) {
    int rc = dalloc(&b->d_push_ctr, 1);
    if (rc) return rc;
    CU(cudaMemsetAsync(b->d_push_ctr, 0, sizeof(unsigned), st));
  }
  long long delta[kMaxPeers];
  unsigned long long* parts[kMaxPeers];
  for (int d = 0; d < npeer; ++d) {
    if (!peer_sig4[d] || !peer_parts[d] || !flags[d]) return set_err(SSQA_EINVAL, "null peer");
    delta[d] = reinterpret_cast<const char*>(peer_sig4[d]) - reinterpret_cast<const char*>(b->d_sig4);
    parts[d] = static_cast<unsigned long long*>(peer_parts[d]);
  }
  const int nrt = b->g.npad / 128 / b->nshards;
  CU(cudaMemsetAsync(b->d_E, 0, size_t(b->g.ccols) * sizeof(long long), st));
  int rc = tc_shard_pass_direct(b, b->shard * nrt, nrt, reinterpret_cast<unsigned long long*>(b->d_E),
                                delta, parts, flags, npeer, epoch, b->d_push_ctr);
  if (rc) return set_err(rc, tc_last_error());
  b->launches += 1;
  return SSQA_OK;
}

int ssqa_batch_shard_merge_direct(ssqa_batch b, const void* parts, long long part_stride,
                                  const unsigned* flags, int nflags, unsigned epoch) {
  if (!b || !parts || !flags) return set_err(SSQA_EINVAL, "null argument");
  if (part_stride < (long long)b->g.ccols * 8 || part_stride % 8)
    return set_err(SSQA_EINVAL, "partial rows need ccols * 8 bytes, 8-aligned");
  if (nflags != b->nshards) return set_err(SSQA_EINVAL, "one flag per shard");
  if (b->cycle > b->p.sc) return set_err(SSQA_EINVAL, "run already complete");
  CU(cudaSetDevice(b->prob->device));
  cudaStream_t st = b->prob->stream;
  const bool upd = b->cycle < b->p.sc;
  const int dst = upd ? pick_free(b) : b->cur;
  launch_shard_merge_direct(b->g, slot_ptr(b, dst), b->d_sig4 + size_t(dst) * b->slot_elems / 2,
                            parts, size_t(part_stride), b->nshards, upd, b->d_E,
                            PeerWait{flags, epoch, nflags}, st);
  CHECK_LAUNCH();
  return shard_scan_advance(b, upd, dst);
}

int ssqa_exchange_alloc(int device, long long bytes, void** dev_ptr_out) {
  if (!dev_ptr_out || bytes < 1) return set_err(SSQA_EINVAL, "bad argument");
  CU(cudaSetDevice(device));
  // a pool block is a cudaMalloc allocation of its own: IPC maps it from its base
  CU(pmalloc(dev_ptr_out, size_t(bytes)));
  CU(cudaMemset(*dev_ptr_out, 0, size_t(bytes)));
  return SSQA_OK;
}

int ssqa_exchange_free(void* dev_ptr) {
  if (dev_ptr) {
    CU(cudaDeviceSynchronize());  // no kernel of this process still uses it
    pool_free(dev_ptr);
  }
  return SSQA_OK;
}

int ssqa_ipc_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return set_err(SSQA_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  std::memcpy(handle_out, &h, sizeof(h));
  return SSQA_OK;
}

int ssqa_ipc_open(const void* handle, int device, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return set_err(SSQA_EINVAL, "null argument");
  CU(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  CU(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return SSQA_OK;
}

int ssqa_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return set_err(SSQA_EINVAL, "null argument");
  CU(cudaIpcCloseMemHandle(dev_ptr));
  return SSQA_OK;
}

int ssqa_batch_shard_end(ssqa_batch b) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  CU(cudaSetDevice(b->prob->device));
  CU(record_event(b->ev1, b->prob->stream));
  b->cycle = b->p.sc;
  return SSQA_OK;
}

int ssqa_batch_init(ssqa_batch b) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  if (!b->seeds_set) return set_err(SSQA_EINVAL, "seeds not set");
  CU(cudaSetDevice(b->prob->device));
  int rc = init_state(b);
  if (rc) return rc;
  CU(cudaStreamSynchronize(b->prob->stream));
  return SSQA_OK;
}

int ssqa_batch_sweep_with(ssqa_batch b, double jperp, double i0) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  CU(cudaSetDevice(b->prob->device));
  int rc = b->engine == SSQA_ENGINE_TCGEN05 ? tc_sweep(b, jperp, i0)
                                            : simt_sweep(b, jperp, i0, 1, nullptr);
  if (rc) return rc == SSQA_ECUDA && b->engine == SSQA_ENGINE_TCGEN05
                     ? set_err(rc, tc_last_error()) : rc;
  CU(cudaStreamSynchronize(b->prob->stream));
  return SSQA_OK;
}

int ssqa_batch_sweep(ssqa_batch b, long count) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  for (long s = 0; s < count; ++s) {
    if (b->cycle + 1 >= kMaxCycles) return set_err(SSQA_EINVAL, "cycle out of range");
    int rc = ssqa_batch_sweep_with(b, jperp_at(b->cycle, b->p), i0_at(b, b->cycle));
    if (rc) return rc;
  }
  return SSQA_OK;
}

int ssqa_batch_energies(ssqa_batch b, double* out) {
  if (!b || !out) return set_err(SSQA_EINVAL, "null argument");
  if (b->prob->count > 1) return set_err(SSQA_EUNSUP, "energies of a multi-instance batch");
  CU(cudaSetDevice(b->prob->device));
  const Geom& g = b->g;
  // fields + integer energies of the current state (no update, no scan)
  cudaStream_t st = b->prob->stream;
  int32_t* S = b->d_S;
  bool tmp = false;
  if (!S) {
    int rc = dalloc(&S, b->slot_elems);
    if (rc) return rc;
    tmp = true;
  }
  launch_field_simt(g, b->prob->d_J, slot_ptr(b, b->cur), S, st);
  CHECK_LAUNCH();
  StepArgs a{b->cycle, 0.0, b->p.i0, b->p.n_rnd, b->p.alpha, 0, 0};
  launch_energy_update_simt(g, S, b->prob->d_H, b->prob->q.scale, b->d_seeds,
                            slot_ptr(b, b->cur), slot_ptr(b, b->cur), slot_ptr(b, b->cur),
                            b->d_acc, b->d_E, a, st);
  CHECK_LAUNCH();
  std::vector<long long> E(g.ccols);
  CU(cudaMemcpyAsync(E.data(), b->d_E, E.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                     st));
  CU(cudaStreamSynchronize(st));
  if (tmp) pool_free(S);
  const double scale = b->prob->q.scale, offset = b->prob->q.offset;
  for (int t = 0; t < g.T; ++t)
    for (int k = 0; k < g.R; ++k)
      out[size_t(t) * g.R + k] = -0.5 * (double(E[col_of(g, t, k)]) * scale) + offset;
  return SSQA_OK;
}

int ssqa_batch_read_lattice(ssqa_batch b, int trial, double* sigma, double* acc, double* hist,
                            long* cycle) {
  if (!b) return set_err(SSQA_EINVAL, "null batch");
  if (trial < 0 || trial >= b->g.T) return set_err(SSQA_ERANGE, "trial index out of range");
  if (b->lattice_stale)
    return set_err(SSQA_EINVAL, "lattice state is not kept after a fused run; re-init first");
  CU(cudaSetDevice(b->prob->device));
  CU(cudaStreamSynchronize(b->prob->stream));
  const Geom& g = b->g;
  const int n = g.n, R = g.R;
  std::vector<int8_t> col(n);
  std::vector<double> acol(n);
  auto read_slot = [&](int slot, double* dst) -> int {
    for (int k = 0; k < R; ++k) {
      CU(cudaMemcpy(col.data(), slot_ptr(b, slot) + size_t(col_of(g, trial, k)) * g.npad, n,
                    cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) dst[size_t(i) * R + k] = double(col[i]);
    }
    return SSQA_OK;
  };
  int rc;
  if (sigma && (rc = read_slot(b->cur, sigma))) return rc;
  if (hist)
    for (int s = 0; s <= b->d; ++s)
      if ((rc = read_slot(b->phys[s], hist + size_t(s) * n * R))) return rc;
  if (acc) {
    for (int k = 0; k < R; ++k) {
      CU(cudaMemcpy(acol.data(), b->d_acc + size_t(col_of(g, trial, k)) * g.npad,
                    n * sizeof(double), cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) acc[size_t(i) * R + k] = acol[i];
    }
  }
  if (cycle) *cycle = b->cycle;
  return SSQA_OK;
}

int ssqa_batch_write_lattice(ssqa_batch b, int trial, const double* sigma, const double* acc,
                             const double* hist, long cycle) {
  if (!b || !sigma || !acc || !hist) return set_err(SSQA_EINVAL, "null argument");
  if (trial < 0 || trial >= b->g.T) return set_err(SSQA_ERANGE, "trial index out of range");
  if (cycle < 0 || cycle >= kMaxCycles) return set_err(SSQA_EINVAL, "cycle out of range");
  CU(cudaSetDevice(b->prob->device));
  int rc = normalize_slots(b);
  if (rc) return rc;
  const Geom& g = b->g;
  const int n = g.n, R = g.R;
  std::vector<int8_t> col(g.npad, 0);
  std::vector<double> acol(g.npad, 0.0);
  auto write_slot = [&](int slot, const double* src) -> int {
    for (int k = 0; k < R; ++k) {
      for (int i = 0; i < n; ++i) {
        const double v = src[size_t(i) * R + k];
        if (v != 1.0 && v != -1.0) return set_err(SSQA_EINVAL, "spin entry not -1/+1");
        col[i] = v > 0 ? 1 : -1;
      }
      CU(cudaMemcpy(slot_ptr(b, slot) + size_t(col_of(g, trial, k)) * g.npad, col.data(),
                    g.npad, cudaMemcpyHostToDevice));
    }
    return SSQA_OK;
  };
  if ((rc = write_slot(b->cur, sigma))) return rc;
  for (int s = 0; s <= b->d; ++s)
    if ((rc = write_slot(b->phys[s], hist + size_t(s) * n * R))) return rc;
  for (int k = 0; k < R; ++k) {
    for (int i = 0; i < n; ++i) acol[i] = acc[size_t(i) * R + k];
    CU(cudaMemcpy(b->d_acc + size_t(col_of(g, trial, k)) * g.npad, acol.data(),
                  g.npad * sizeof(double), cudaMemcpyHostToDevice));
  }
  b->cycle = cycle;
  return SSQA_OK;
}

}  // extern "C"
