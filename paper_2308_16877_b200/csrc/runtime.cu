// runtime.cu — host side of the C-ABI (include/hpac_offload.h): validation
// with the reference's error taxonomy, arena accounting, grid resolution,
// kernel dispatch, statistics, host-buffer (end-to-end) entry, metrics.
#include <cuda_runtime.h>

#include <cmath>
#include <limits>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "engine.h"
#include "hpac_offload.h"

#define HPAC_API extern "C" __attribute__((visibility("default")))

namespace hpac {
size_t engine_thread_smem(EngineParams& p);
int engine_thread_max_in(int app);
int engine_thread_max_out(int app);
cudaError_t engine_thread_launch(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st);
bool engine_stream_eligible(const EngineParams& p);
size_t engine_stream_smem(const EngineParams& p);
cudaError_t engine_stream_launch(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st);
bool engine_bs_iact_eligible(const EngineParams& p);
size_t engine_bs_iact_smem(EngineParams& p);
cudaError_t engine_bs_iact_launch(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st);
size_t engine_team_seq_smem(EngineParams& p, int block);
cudaError_t engine_team_seq_launch(const EngineParams& p, int team_end, int block, size_t smem,
                                   cudaStream_t st);
size_t binomial_team_smem(EngineParams& p);
cudaError_t binomial_team_launch(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st);
cudaError_t mape_launch(const double* a, const double* b, int64_t n, double* d_sum,
                        unsigned long long* d_inf, cudaStream_t st);
cudaError_t mcr_launch(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* d_cnt,
                       cudaStream_t st);
}  // namespace hpac

using namespace hpac;

namespace {

int fail(char* err, size_t len, int code, const char* fmt, ...) {
  if (err && len) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, len, fmt, ap);
    va_end(ap);
  }
  return code;
}

int cuda_fail(char* err, size_t len, cudaError_t e, const char* where) {
  return fail(err, len, HPAC_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

// Per-host-thread launch scratch: a ring of slots, each with its own device
// counters, pinned readback and events, so an asynchronous launch's counter
// readback can never be overwritten by (or upload the counters of) the next
// call; launches on different streams use different slots. A slot is reused
// only after its previous readback completed (`done`).
constexpr int kScratchSlots = 8;
struct ScratchSlot {
  unsigned long long* d_cnt = nullptr;
  unsigned long long* h_cnt = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, done = nullptr;
  bool in_flight = false;  // readback enqueued, not yet waited for
};
struct Scratch {
  int device = -1;
  ScratchSlot slot[kScratchSlots];
  int next = 0;
  // the last asynchronous launch (hpac_stats_fetch)
  int pending = -1;
  cudaStream_t pending_stream = nullptr;
  hpac_stats_t pending_base{};
};
thread_local Scratch g_scratch;
// set by the zero-copy host entry around its launch: generic per-thread engine
thread_local bool g_force_thread_engine = false;

// Largest double x with sqrt_rn(x) <= t: sqrt is correctly rounded and
// monotone, so sqrt_rn(ssq) <= t  <=>  ssq <= x (the iACT hit test of
// iact.hpp:60-70 without the square root).
static double sqrt_threshold_square(double t) {
  if (!(t >= 0.0)) return -1.0;
  if (std::isinf(t)) return t;
  double x = t * t;
  if (std::isinf(x)) x = std::numeric_limits<double>::max();
  while (x > 0.0 && std::sqrt(x) > t) x = std::nextafter(x, 0.0);
  for (;;) {
    const double y = std::nextafter(x, std::numeric_limits<double>::infinity());
    if (std::isinf(y) || std::sqrt(y) > t) break;
    x = y;
  }
  return x;
}

void scratch_release() {
  for (ScratchSlot& s : g_scratch.slot) {
    if (s.done) cudaEventSynchronize(s.done);
    if (s.d_cnt) cudaFree(s.d_cnt);
    if (s.h_cnt) cudaFreeHost(s.h_cnt);
    for (cudaEvent_t ev : {s.ev0, s.ev1, s.done})
      if (ev) cudaEventDestroy(ev);
    s = ScratchSlot{};
  }
  g_scratch.pending = -1;
  g_scratch.device = -1;
}

cudaError_t scratch_ready() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_scratch.device == dev && g_scratch.slot[0].d_cnt) return cudaSuccess;
  if (g_scratch.device >= 0) {  // the thread moved to another device
    int cur = dev;
    cudaSetDevice(g_scratch.device);
    scratch_release();
    cudaSetDevice(cur);
  }
  const size_t bytes = sizeof(unsigned long long) * kNumCounters;
  for (ScratchSlot& s : g_scratch.slot) {
    if ((e = cudaMalloc(&s.d_cnt, bytes)) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&s.h_cnt, bytes)) != cudaSuccess) return e;
    if ((e = cudaEventCreate(&s.ev0)) != cudaSuccess) return e;
    if ((e = cudaEventCreate(&s.ev1)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  g_scratch.device = dev;
  return cudaSuccess;
}

// Next free slot: waits for the slot's previous readback if it is still in
// flight (only after kScratchSlots outstanding asynchronous launches).
cudaError_t scratch_acquire(int* idx) {
  const int i = g_scratch.next;
  g_scratch.next = (i + 1) % kScratchSlots;
  ScratchSlot& s = g_scratch.slot[i];
  if (s.in_flight) {
    cudaError_t e = cudaEventSynchronize(s.done);
    if (e != cudaSuccess) return e;
    s.in_flight = false;
  }
  if (g_scratch.pending == i) g_scratch.pending = -1;
  *idx = i;
  return cudaSuccess;
}

bool kind_uses_modulus(int k) {
  return k == HPAC_PERFO_SMALL || k == HPAC_PERFO_LARGE || k == HPAC_PERFO_HERDED_SMALL ||
         k == HPAC_PERFO_HERDED_LARGE;
}

// grid.hpp:27-37
int validate_grid(const hpac_grid_t* g, char* err, size_t el) {
  if (!g) return fail(err, el, HPAC_ERR_CONFIG, "grid is null");
  if (g->num_teams < 1) return fail(err, el, HPAC_ERR_CONFIG, "num_teams must be positive");
  if (g->threads_per_team < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "threads_per_team must be positive");
  if (g->warp_size < 1 || g->warp_size > 64)
    return fail(err, el, HPAC_ERR_CONFIG, "warp_size must be in [1, 64]");
  if (g->threads_per_team % g->warp_size != 0)
    return fail(err, el, HPAC_ERR_CONFIG, "warp_size (%d) must divide threads_per_team (%d)",
                g->warp_size, g->threads_per_team);
  if (g->items_per_thread < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "items_per_thread must be positive");
  return 0;
}

// ApproxSpec::validate + Taf/Iact/PerfoConfig::validate (directive.hpp:72-84,
// taf.hpp:19-23, iact.hpp:24-29, perfo.hpp:27-34)
int validate_spec(const hpac_spec_t* s, char* err, size_t el) {
  switch (s->technique) {
    case HPAC_TECH_TAF:
      if (s->taf_h_size < 1) return fail(err, el, HPAC_ERR_CONFIG, "TAF history size must be >= 1");
      if (s->taf_p_size < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "TAF prediction size must be >= 1");
      if (!(s->taf_threshold >= 0.0))
        return fail(err, el, HPAC_ERR_CONFIG, "TAF threshold must be >= 0");
      break;
    case HPAC_TECH_IACT:
      if (s->iact_table_size < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "iACT table size must be >= 1");
      if (!(s->iact_threshold >= 0.0))
        return fail(err, el, HPAC_ERR_CONFIG, "iACT threshold must be >= 0");
      if (s->iact_tables_per_warp < 0)
        return fail(err, el, HPAC_ERR_CONFIG, "tables_per_warp must be >= 1");
      break;
    case HPAC_TECH_PERFO:
      if (s->perfo_kind < 0 || s->perfo_kind > HPAC_PERFO_RANDOM)
        return fail(err, el, HPAC_ERR_CONFIG, "unknown perforation kind");
      if (kind_uses_modulus(s->perfo_kind)) {
        if (s->perfo_modulus < 2)
          return fail(err, el, HPAC_ERR_CONFIG, "perforation modulus must be >= 2");
      } else if (s->perfo_skip_percent < 1 || s->perfo_skip_percent > 99) {
        return fail(err, el, HPAC_ERR_CONFIG, "perforation skip percent must be in [1, 99]");
      }
      break;
    default:
      return fail(err, el, HPAC_ERR_CONFIG, "ApproxSpec must carry exactly one technique payload");
  }
  if (s->level < HPAC_LEVEL_THREAD || s->level > HPAC_LEVEL_TEAM)
    return fail(err, el, HPAC_ERR_CONFIG, "unknown decision level");
  if (s->technique == HPAC_TECH_IACT && s->n_input_sections < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "iACT requires at least one input section");
  if ((s->technique == HPAC_TECH_IACT || s->technique == HPAC_TECH_TAF) &&
      s->n_output_sections < 1)
    return fail(err, el, HPAC_ERR_CONFIG, "memoization requires at least one output section");
  return 0;
}

// Region dims from the app (engine.hpp:26-33 input_dims/output_dims).
int bind_region(hpac_region_t* r, char* err, size_t el, int64_t n = 1) {
  // buffers are only required for non-empty launches (an empty device
  // array may legitimately be NULL)
  const bool need = n > 0;
  switch (r->app) {
    case HPAC_APP_TABLE:
      if (need && !r->table_out) return fail(err, el, HPAC_ERR_CONFIG, "region has no evaluate function");
      if (need && r->input_dims > 0 && !r->in)
        return fail(err, el, HPAC_ERR_CONFIG, "region declares inputs but has no load_input");
      if (r->output_dims < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "region output_dims must be >= 1");
      if (r->input_dims < 0) return fail(err, el, HPAC_ERR_CONFIG, "region input_dims must be >= 0");
      return 0;
    case HPAC_APP_SYNTHETIC:
      if (r->synthetic_profile < 0 || r->synthetic_profile > 2)
        return fail(err, el, HPAC_ERR_CONFIG, "unknown synthetic profile");
      r->input_dims = 1;
      r->output_dims = 1;
      return 0;
    case HPAC_APP_BLACKSCHOLES:
      r->input_dims = 5;
      r->output_dims = 1;
      if (need && !r->in) return fail(err, el, HPAC_ERR_CONFIG, "region declares inputs but has no load_input");
      return 0;
    case HPAC_APP_BINOMIAL:
      r->input_dims = 5;
      r->output_dims = 1;
      if (need && !r->in) return fail(err, el, HPAC_ERR_CONFIG, "region declares inputs but has no load_input");
      if (r->binomial_steps < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "binomial_price: n_steps must be >= 1");
      return 0;
    case HPAC_APP_KMEANS:
      if (r->kmeans_dims < 1 || r->kmeans_k < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "kmeans dims and k must be >= 1");
      if (need && (!r->in || !r->centroids))
        return fail(err, el, HPAC_ERR_CONFIG, "kmeans region needs points and centroids");
      r->input_dims = r->kmeans_dims;
      r->output_dims = r->kmeans_k;
      return 0;
    case HPAC_APP_LAVAMD:
      if (r->lavamd_boxes1d < 1 || r->lavamd_particles < 1)
        return fail(err, el, HPAC_ERR_CONFIG, "lavamd: boxes1d and particles must be >= 1");
      if (!(r->lavamd_alpha > 0.0)) return fail(err, el, HPAC_ERR_CONFIG, "lavamd: alpha must be > 0");
      if (need && (!r->in || !r->table_out || !r->out))
        return fail(err, el, HPAC_ERR_CONFIG, "lavamd region needs rv (in), qv (table_out) and fv (out)");
      r->input_dims = 0;
      r->output_dims = 4;
      return 0;
  }
  return fail(err, el, HPAC_ERR_UNSUPPORTED, "unsupported application id %d", r->app);
}

uint64_t taf_state_bytes(int h, int dims) { return (uint64_t)dims * (uint64_t)h * 8u + 16u; }
uint64_t table_group_bytes(int tpw, int tsize, int in_dims, int out_dims) {
  return (uint64_t)tpw * (uint64_t)tsize * (uint64_t)(in_dims + out_dims) * 8u +
         (uint64_t)tpw * 2u * 4u;
}

// bind_technique arena charges (engine.hpp:83-116): the per-team bump
// allocator fails at the first allocation that crosses the budget,
// reporting required = used + length (arena.hpp:37-38).
int arena_account(const hpac_grid_t* g, const hpac_region_t* r, const hpac_spec_t* s, int tpw,
                  uint64_t* required, uint64_t* available, char* err, size_t el) {
  const uint64_t cap = g->shared_mem_budget_bytes;
  uint64_t used = 0, per = 0;
  int count = 0;
  *available = cap;
  if (s->technique == HPAC_TECH_TAF) {
    per = taf_state_bytes(s->taf_h_size, r->output_dims);
    count = g->threads_per_team;
  } else if (s->technique == HPAC_TECH_IACT) {
    per = table_group_bytes(tpw, s->iact_table_size, r->input_dims, r->output_dims);
    count = g->threads_per_team / g->warp_size;
  }
  if (count > 0 && per > 0) {
    uint64_t fit = cap / per;  // allocations that fit
    if (fit < (uint64_t)count) {
      *required = (fit + 1) * per;
      return fail(err, el, HPAC_ERR_ARENA_OVERFLOW,
                  "shared arena overflow: required %llu bytes, available %llu bytes",
                  (unsigned long long)*required, (unsigned long long)cap);
    }
    used = per * (uint64_t)count;
  }
  if (s->level == HPAC_LEVEL_TEAM) {
    if (used + 8 > cap) {
      *required = used + 8;
      return fail(err, el, HPAC_ERR_ARENA_OVERFLOW,
                  "shared arena overflow: required %llu bytes, available %llu bytes",
                  (unsigned long long)*required, (unsigned long long)cap);
    }
    used += 8;
  }
  *required = used;
  return 0;
}

struct Prepared {
  EngineParams p{};
  int kind = 0;  // 0 = per-thread engine, 1 = team seq, 2 = binomial team
  int nblocks = 0;
  int block = 0;
  int team_end = 0;
  size_t smem = 0;
  bool empty = false;
};

// Full launch-time validation in the reference's order (engine.hpp:135-186),
// then the B200 engine's own limits (HPAC_ERR_UNSUPPORTED).
int prepare(const hpac_grid_t* g, int64_t n, int32_t mapping, const hpac_region_t* region,
            const hpac_spec_t* spec, const hpac_launch_t* launch, Prepared& pr,
            hpac_stats_t* stats, char* err, size_t el) {
  int rc;
  if ((rc = validate_grid(g, err, el))) return rc;
  if (mapping != HPAC_MAP_PER_THREAD && mapping != HPAC_MAP_PER_TEAM)
    return fail(err, el, HPAC_ERR_CONFIG, "unknown work mapping");
  if (n < 0) return fail(err, el, HPAC_ERR_CONFIG, "problem size must be non-negative");
  const bool per_team = mapping == HPAC_MAP_PER_TEAM;
  const int64_t cap = per_team ? (int64_t)g->num_teams * g->items_per_thread
                               : (int64_t)g->num_teams * g->threads_per_team * g->items_per_thread;
  if (n > cap)
    return fail(err, el, HPAC_ERR_CONFIG,
                "grid capacity %lld cannot cover problem size %lld (increase num_teams, "
                "threads_per_team, or items_per_thread)",
                (long long)cap, (long long)n);
  if (!region) return fail(err, el, HPAC_ERR_CONFIG, "region is null");
  hpac_region_t r = *region;
  if ((rc = bind_region(&r, err, el, n))) return rc;

  EngineParams& p = pr.p;
  std::memset(&p, 0, sizeof p);
  p.region = r;
  p.in_dims = r.input_dims;
  p.out_dims = r.output_dims;
  p.tech = -1;
  p.level = HPAC_LEVEL_THREAD;
  int tpw = 0;
  if (spec) {
    if ((rc = validate_spec(spec, err, el))) return rc;
    p.tech = spec->technique;
    p.level = spec->level;
    if (spec->technique == HPAC_TECH_IACT) {
      if (r.input_dims < 1) return fail(err, el, HPAC_ERR_CONFIG, "iACT requires a region with inputs");
      tpw = spec->iact_tables_per_warp > 0 ? spec->iact_tables_per_warp : g->warp_size;
      if (tpw < 1 || g->warp_size % tpw != 0)
        return fail(err, el, HPAC_ERR_CONFIG, "tables_per_warp (%d) must divide warp_size (%d)",
                    tpw, g->warp_size);
    }
    uint64_t req = 0, avail = 0;
    rc = arena_account(g, &r, spec, tpw, &req, &avail, err, el);
    if (stats) {
      stats->arena_required = req;
      stats->arena_available = avail;
    }
    if (rc) return rc;
    if (spec->technique == HPAC_TECH_PERFO &&
        (spec->perfo_kind == HPAC_PERFO_INI || spec->perfo_kind == HPAC_PERFO_FINI) &&
        ((r.app == HPAC_APP_TABLE && r.encounters) || r.app == HPAC_APP_LAVAMD))
      return fail(err, el, HPAC_ERR_CONFIG,
                  "INI/FINI perforation requires a fixed trip count per thread");
    p.taf_h = spec->taf_h_size;
    p.taf_p = spec->taf_p_size;
    p.taf_thr = spec->taf_threshold;
    p.tsize = spec->iact_table_size;
    p.tpw = tpw;
    p.iact_thr = spec->iact_threshold;
    p.iact_thr2 = sqrt_threshold_square(spec->iact_threshold);
    p.perfo_kind = spec->perfo_kind;
    p.perfo_mod = spec->perfo_modulus;
    p.perfo_pct = spec->perfo_skip_percent;
    p.perfo_seed = spec->perfo_seed;
  }
  p.voting = spec && p.level != HPAC_LEVEL_THREAD;

  // schedule
  p.n = n;
  p.num_teams = g->num_teams;
  p.tpt = g->threads_per_team;
  p.ws = g->warp_size;
  p.wpt = g->threads_per_team / g->warp_size;
  p.stride = per_team ? (int64_t)g->num_teams : (int64_t)g->num_teams * g->threads_per_team;
  p.steps = n <= 0 ? 0 : (n + p.stride - 1) / p.stride;
  p.fast_ws = (p.ws <= 32 && 32 % p.ws == 0) ? 1 : 0;
  p.has_enc = ((r.app == HPAC_APP_TABLE && r.encounters) || r.app == HPAC_APP_LAVAMD) ? 1 : 0;
  p.staged = r.app == HPAC_APP_LAVAMD ? 1 : 0;
  p.barrier_eval = (r.flags & HPAC_REGION_BARRIER_IN_EVALUATE) ? 1 : 0;
  p.accumulate = (r.flags & HPAC_REGION_STORE_ACCUMULATE) ? 1 : 0;
  p.paths = launch ? launch->paths : nullptr;

  int tb = 0, te = g->num_teams;
  if (launch && (launch->team_begin != 0 || launch->team_end != 0)) {
    tb = launch->team_begin;
    te = launch->team_end;
    if (tb < 0 || te > g->num_teams || tb > te)
      return fail(err, el, HPAC_ERR_CONFIG, "team range [%d, %d) outside [0, %d)", tb, te,
                  g->num_teams);
  }
  p.team_begin = tb;
  pr.team_end = te;
  pr.empty = (te == tb) || n == 0;

  // ---- B200 engine limits ------------------------------------------------
  if (r.app == HPAC_APP_LAVAMD) {
    const long long boxes = (long long)r.lavamd_boxes1d * r.lavamd_boxes1d * r.lavamd_boxes1d;
    if (!per_team)
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "LavaMD runs one box per team (per-team mapping)");
    if (r.lavamd_particles != g->threads_per_team)
      return fail(err, el, HPAC_ERR_CONFIG,
                  "lavamd: particles per box (%d) must equal threads_per_team (%d)",
                  r.lavamd_particles, g->threads_per_team);
    if (n > boxes)
      return fail(err, el, HPAC_ERR_CONFIG, "lavamd: %lld items exceed %lld boxes", (long long)n,
                  boxes);
    if ((reinterpret_cast<uintptr_t>(r.in) & 31) != 0)
      return fail(err, el, HPAC_ERR_UNSUPPORTED,
                  "lavamd: rv must be 32-byte aligned (one double4 per particle)");
    if (g->threads_per_team > 1024)
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "threads_per_team > 1024 is not supported");
    p.per_team = 1;
    {
      // tiled box order for L2 reuse of the 27-neighbourhoods (whole grid only;
      // HPAC_LAVA_TILE=0 keeps the natural order)
      const char* lt = getenv("HPAC_LAVA_TILE");
      const int b1 = r.lavamd_boxes1d;
      const bool whole = tb == 0 && te == g->num_teams && (long long)g->num_teams == boxes && n == boxes;
      p.box_tile = (lt && strcmp(lt, "0") == 0) || !whole ? 0 : (b1 % 32 == 0 ? 32 : (b1 % 16 == 0 ? 16 : 0));
    }
    pr.kind = 0;
    pr.block = p.tpt;
    pr.nblocks = te - tb;
    pr.smem = engine_thread_smem(p);
  } else if (!per_team) {
    if (r.app == HPAC_APP_BINOMIAL)
      return fail(err, el, HPAC_ERR_UNSUPPORTED,
                  "binomial region runs under per-team mapping (bench/run.hpp:44)");
    if (g->threads_per_team > 1024)
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "threads_per_team > 1024 is not supported");
    if (r.input_dims > engine_thread_max_in(r.app))
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "region input_dims %d exceeds %d", r.input_dims,
                  engine_thread_max_in(r.app));
    if (r.app != HPAC_APP_KMEANS && r.output_dims > engine_thread_max_out(r.app))
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "region output_dims %d exceeds %d",
                  r.output_dims, engine_thread_max_out(r.app));
    if (r.app == HPAC_APP_KMEANS && spec && spec->technique == HPAC_TECH_TAF)
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "TAF on the K-Means region is not supported");
    if (r.app == HPAC_APP_KMEANS && spec && spec->technique == HPAC_TECH_IACT && r.out)
      return fail(err, el, HPAC_ERR_UNSUPPORTED,
                  "iACT on K-Means keeps labels only; pass out = NULL");
    if (r.app == HPAC_APP_KMEANS) p.out_dims = 1;  // payload = label
    pr.kind = 0;
    pr.block = p.tpt;
    pr.nblocks = te - tb;
    // K-Means filtered argmin on the FP64 tensor op (AppKmeans::warp_eval)
    // for its shape: 32 dims, k % 8 == 0, labels only, whole hardware warps;
    // HPAC_KM_DMMA=0 keeps the per-lane CUDA-core filter (A/B tests)
    if (r.app == HPAC_APP_KMEANS) {
      const char* km = getenv("HPAC_KM_DMMA");
      p.warp_eval = r.kmeans_dims == 32 && r.kmeans_k % 8 == 0 && !r.out &&
                    !(r.flags & HPAC_REGION_KMEANS_FAST_MATH) && p.tpt % 32 == 0 && p.tpt <= 256 &&
                    (reinterpret_cast<uintptr_t>(r.in) & 15) == 0 && !(km && strcmp(km, "0") == 0);
    }
    pr.smem = engine_thread_smem(p);
    // streaming variant (engine_stream.cu: barrier-free lane kernel) where it applies;
    // HPAC_ENGINE=thread forces the generic engine (A/B parity tests)
    const char* force = getenv("HPAC_ENGINE");
    if (engine_stream_eligible(p) && !(force && strcmp(force, "thread") == 0) &&
        !g_force_thread_engine) {
      pr.kind = 3;
      pr.smem = engine_stream_smem(p);
    }
    // iACT on Blackscholes: decide-then-price engine (engine_bs_iact.cu)
    if (engine_bs_iact_eligible(p) && !(force && strcmp(force, "thread") == 0) &&
        !g_force_thread_engine) {
      pr.kind = 4;
      pr.smem = engine_bs_iact_smem(p);
    }
  } else {
    if (r.app == HPAC_APP_KMEANS)
      return fail(err, el, HPAC_ERR_UNSUPPORTED, "K-Means region runs under per-thread mapping");
    if (r.app == HPAC_APP_BINOMIAL) {
      pr.kind = 2;
      pr.block = 64;
      pr.nblocks = te - tb;
      pr.smem = binomial_team_smem(p);
    } else {
      if (r.input_dims > engine_thread_max_in(r.app) ||
          r.output_dims > engine_thread_max_out(r.app))
        return fail(err, el, HPAC_ERR_UNSUPPORTED, "region dims exceed the engine limits");
      pr.kind = 1;
      pr.block = 128;
      pr.nblocks = (te - tb + pr.block - 1) / pr.block;
      pr.smem = engine_team_seq_smem(p, pr.block);
    }
  }
  if (pr.smem > 227 * 1024)
    return fail(err, el, HPAC_ERR_UNSUPPORTED,
                "technique state needs %zu bytes of shared memory per CTA (max 232448)", pr.smem);
  return 0;
}

cudaError_t launch_prepared(const Prepared& pr, cudaStream_t st) {
  if (pr.empty) return cudaSuccess;
  switch (pr.kind) {
    case 0: return engine_thread_launch(pr.p, pr.nblocks, pr.smem, st);
    case 1: return engine_team_seq_launch(pr.p, pr.team_end, pr.block, pr.smem, st);
    case 2: return binomial_team_launch(pr.p, pr.nblocks, pr.smem, st);
    case 3: return engine_stream_launch(pr.p, pr.nblocks, pr.smem, st);
    case 4: return engine_bs_iact_launch(pr.p, pr.nblocks, pr.smem, st);
  }
  return cudaErrorInvalidValue;
}

void counters_to_stats(const unsigned long long* c, hpac_stats_t* st) {
  st->total_invocations = c[kCntTotal];
  st->approx_invocations = c[kCntApprox];
  st->divergent_warp_steps = c[kCntDivergent];
  st->total_warp_steps = c[kCntWarpSteps];
  st->resident_warps = (int32_t)c[kCntResidentWarps];
  st->lattice_fallbacks = c[kCntLatticeFallback];
  st->lattice_nodes = c[kCntLatticeNodes];
}

// Map device-side faults to the reference's exceptions.
int finish_status(const unsigned long long* c, hpac_stats_t* st, int app, char* err, size_t el) {
  if (c[kCntBarrierKey] != ~0ull) {
    st->barrier_divergence_detected = 1;
    st->fail_step = (int64_t)(c[kCntBarrierKey] >> 32);
    st->fail_team = (int32_t)(c[kCntBarrierKey] & 0xffffffffu);
    st->fail_missing = (int32_t)c[kCntBarrierMissing];
    return fail(err, el, HPAC_ERR_BARRIER_DIVERGENCE,
                "barrier divergence in team %d at step %lld: %d thread(s) never arrived",
                st->fail_team, (long long)st->fail_step, st->fail_missing);
  }
  if (c[kCntAppError]) {
    if (app == HPAC_APP_BINOMIAL)
      return fail(err, el, HPAC_ERR_CONFIG,
                  "binomial_price: invalid option parameters or lattice outside the "
                  "risk-neutral range");
    return fail(err, el, HPAC_ERR_CONFIG, "black_scholes_call: invalid option parameters");
  }
  return 0;
}

}  // namespace

// Internal handles for captured loops (the K-Means Lloyd graph, kmeans.cu):
// the region is validated once, then launched from inside a CUDA graph with
// caller-owned counters (accumulating across iterations), a device seed and
// a preallocated DMMA operand block.
namespace hpac {
int region_prepare(const hpac_grid_t* g, int64_t n, int32_t mapping, const hpac_region_t* region,
                   const hpac_spec_t* spec, unsigned long long* d_counters,
                   const unsigned long long* seed_ptr, const double* km_aux, void** handle,
                   char* err, size_t el) {
  Prepared* pr = new Prepared;
  hpac_stats_t st{};
  int rc = prepare(g, n, mapping, region, spec, nullptr, *pr, &st, err, el);
  if (rc) {
    delete pr;
    return rc;
  }
  pr->p.counters = d_counters;
  pr->p.seed_ptr = seed_ptr;
  pr->p.km_aux = km_aux;
  *handle = pr;
  return HPAC_OK;
}
cudaError_t region_launch(const void* handle, cudaStream_t st) {
  return launch_prepared(*static_cast<const Prepared*>(handle), st);
}
void region_free(void* handle) { delete static_cast<Prepared*>(handle); }
}  // namespace hpac

// ===========================================================================
// C-ABI
// ===========================================================================
HPAC_API int hpac_abi_version(void) { return HPAC_ABI_VERSION; }

HPAC_API const char* hpac_status_name(int status) {
  switch (status) {
    case HPAC_OK: return "OK";
    case HPAC_ERR_CONFIG: return "ConfigError";
    case HPAC_ERR_ARENA_OVERFLOW: return "ArenaOverflowError";
    case HPAC_ERR_BARRIER_DIVERGENCE: return "BarrierDivergenceError";
    case HPAC_ERR_CUDA: return "CudaError";
    case HPAC_ERR_DIRECTIVE: return "DirectiveError";
    case HPAC_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "?";
}

// BenchmarkInfo table + resolve_grid, bench/run.hpp:41-97 ("lavamd" is the
// framework's extension, one box of particles per team).
HPAC_API int hpac_resolve_grid(const char* benchmark, int64_t n, const hpac_grid_t* ov,
                               hpac_grid_t* out, int32_t* mapping_out, char* err, size_t el) {
  struct Info {
    const char* id;
    long long default_n;
    int tpt, ws, ipt, mapping;
  };
  static const Info table[] = {
      {"blackscholes", 65536, 64, 32, 16, HPAC_MAP_PER_THREAD},
      {"binomial", 16384, 64, 32, 8, HPAC_MAP_PER_TEAM},
      {"kmeans", 4096, 64, 32, 4, HPAC_MAP_PER_THREAD},
      {"synthetic-constant", 16384, 64, 32, 32, HPAC_MAP_PER_THREAD},
      {"synthetic-slow-drift", 16384, 64, 32, 32, HPAC_MAP_PER_THREAD},
      {"synthetic-noise", 16384, 64, 32, 32, HPAC_MAP_PER_THREAD},
      // extension: one box per team, lane = particle (128 = 4 whole warps;
      // grid.hpp:27-37 needs warp_size | threads_per_team), item = box
      {"lavamd", 512, 128, 32, 1, HPAC_MAP_PER_TEAM},
  };
  if (!benchmark) return fail(err, el, HPAC_ERR_CONFIG, "benchmark is null");
  const Info* info = nullptr;
  for (const Info& i : table)
    if (std::strcmp(i.id, benchmark) == 0) info = &i;
  if (!info) return fail(err, el, HPAC_ERR_CONFIG, "unknown benchmark '%s'", benchmark);
  hpac_grid_t z{};
  if (!ov) ov = &z;
  long long nn = n > 0 ? n : info->default_n;
  hpac_grid_t g;
  g.threads_per_team = ov->threads_per_team > 0 ? ov->threads_per_team : info->tpt;
  g.warp_size = ov->warp_size > 0 ? ov->warp_size : info->ws;
  g.items_per_thread = ov->items_per_thread > 0 ? ov->items_per_thread : info->ipt;
  g.shared_mem_budget_bytes = ov->shared_mem_budget_bytes ? ov->shared_mem_budget_bytes : 48 * 1024;
  if (ov->num_teams > 0) {
    g.num_teams = ov->num_teams;
  } else {
    long long per_team = info->mapping == HPAC_MAP_PER_TEAM
                             ? g.items_per_thread
                             : (long long)g.threads_per_team * g.items_per_thread;
    long long t = (nn + per_team - 1) / per_team;
    g.num_teams = (int)(t < 1 ? 1 : t);
  }
  *out = g;
  if (mapping_out) *mapping_out = info->mapping;
  return HPAC_OK;
}

HPAC_API int hpac_region_bind(hpac_region_t* region, char* err, size_t el) {
  if (!region) return fail(err, el, HPAC_ERR_CONFIG, "region is null");
  return bind_region(region, err, el);
}

HPAC_API int hpac_arena_required(const hpac_grid_t* g, const hpac_region_t* region,
                                 const hpac_spec_t* spec, uint64_t* required,
                                 uint64_t* available, char* err, size_t el) {
  int rc;
  if ((rc = validate_grid(g, err, el))) return rc;
  hpac_region_t r = *region;
  if ((rc = bind_region(&r, err, el))) return rc;
  if ((rc = validate_spec(spec, err, el))) return rc;
  int tpw = spec->iact_tables_per_warp > 0 ? spec->iact_tables_per_warp : g->warp_size;
  return arena_account(g, &r, spec, tpw, required, available, err, el);
}

HPAC_API int hpac_run_region(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                             const hpac_region_t* region, const hpac_spec_t* spec,
                             const hpac_launch_t* launch, hpac_stats_t* stats, char* err,
                             size_t el) {
  hpac_stats_t local{};
  if (!stats) stats = &local;
  std::memset(stats, 0, sizeof *stats);
  if (err && el) err[0] = 0;
  Prepared pr;
  int rc = prepare(grid, n, mapping, region, spec, launch, pr, stats, err, el);
  if (rc) return rc;
  cudaStream_t st = launch ? (cudaStream_t)launch->stream : nullptr;
  bool sync = !launch || launch->synchronous;
  cudaError_t e = scratch_ready();
  if (e != cudaSuccess) return cuda_fail(err, el, e, "scratch");
  int si = 0;
  if ((e = scratch_acquire(&si)) != cudaSuccess) return cuda_fail(err, el, e, "scratch slot");
  ScratchSlot& slot = g_scratch.slot[si];
  // counters: zero, barrier key = ~0
  unsigned long long init[kNumCounters];
  std::memset(init, 0, sizeof init);
  init[kCntBarrierKey] = ~0ull;
  std::memcpy(slot.h_cnt, init, sizeof init);
  if ((e = cudaMemcpyAsync(slot.d_cnt, slot.h_cnt, sizeof init, cudaMemcpyHostToDevice, st)) !=
      cudaSuccess)
    return cuda_fail(err, el, e, "counter init");
  pr.p.counters = slot.d_cnt;
  // events bracket the kernel(s) only: the counter copies stay outside
  if ((e = cudaEventRecord(slot.ev0, st)) != cudaSuccess) return cuda_fail(err, el, e, "event");
  if ((e = launch_prepared(pr, st)) != cudaSuccess) return cuda_fail(err, el, e, "kernel launch");
  if ((e = cudaEventRecord(slot.ev1, st)) != cudaSuccess) return cuda_fail(err, el, e, "event");
  e = cudaMemcpyAsync(slot.h_cnt, slot.d_cnt, sizeof init, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(err, el, e, "counter readback");
  if ((e = cudaEventRecord(slot.done, st)) != cudaSuccess) return cuda_fail(err, el, e, "event");
  slot.in_flight = true;
  if (!sync) {
    // counters stay in this launch's slot; hpac_stats_fetch reads them
    g_scratch.pending = si;
    g_scratch.pending_stream = st;
    g_scratch.pending_base = *stats;
    return HPAC_OK;
  }
  if ((e = cudaEventSynchronize(slot.done)) != cudaSuccess) return cuda_fail(err, el, e, "kernel");
  slot.in_flight = false;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, slot.ev0, slot.ev1);
  counters_to_stats(slot.h_cnt, stats);
  stats->kernel_ms = ms;
  return finish_status(slot.h_cnt, stats, pr.p.region.app, err, el);
}

HPAC_API int hpac_stats_fetch(hpac_stats_t* stats) {
  if (g_scratch.pending < 0) return HPAC_ERR_CONFIG;
  ScratchSlot& slot = g_scratch.slot[g_scratch.pending];
  cudaError_t e = cudaEventSynchronize(slot.done);
  if (e != cudaSuccess) return HPAC_ERR_CUDA;
  slot.in_flight = false;
  *stats = g_scratch.pending_base;
  counters_to_stats(slot.h_cnt, stats);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, slot.ev0, slot.ev1);
  stats->kernel_ms = ms;
  g_scratch.pending = -1;
  char buf[8];
  return finish_status(slot.h_cnt, stats, -1, buf, sizeof buf);
}

// Device-usable address of page-locked (pinned) host memory, else null.
const void* pinned_device_ptr(const void* p) {
  if (!p) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Private stream-ordered pool for the host-buffer entry: memory is kept
// across calls (release threshold = max), so repeated end-to-end calls do
// not re-map device memory every time (the default pool trims at syncs).
cudaMemPool_t host_entry_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[16] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) return pools[dev] = nullptr;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return pools[dev];
}

namespace hpac {
// the binomial pipeline's per-launch workspace comes from the same retained pool
cudaMemPool_t bino_pool() { return ::host_entry_pool(); }
}  // namespace hpac

namespace {
// items [c0, c1) of every row of the [rows x G] matrix of `rec`-double
// records, rows cut at n (the last row may be ragged): one 2-D copy for the
// whole rows of the block, one 1-D copy for the ragged part
cudaError_t copy_column_block(double* dst, const double* src, int64_t n, int64_t G, int64_t c0,
                              int64_t c1, int rec, cudaMemcpyKind kind, cudaStream_t s) {
  if (c1 <= c0 || n <= c0) return cudaSuccess;
  const int64_t full = n >= c1 ? (n - c1) / G + 1 : 0;  // rows whose block is entirely < n
  const size_t pitch = (size_t)G * rec * 8, width = (size_t)(c1 - c0) * rec * 8;
  cudaError_t e = cudaSuccess;
  if (full > 0)
    e = cudaMemcpy2DAsync(dst + (size_t)c0 * rec, pitch, src + (size_t)c0 * rec, pitch, width,
                          (size_t)full, kind, s);
  const int64_t r0 = full * G + c0;  // the block's first item in the next row
  if (e == cudaSuccess && r0 < n) {
    const int64_t cnt = (n - r0) < (c1 - c0) ? (n - r0) : (c1 - c0);
    e = cudaMemcpyAsync(dst + (size_t)r0 * rec, src + (size_t)r0 * rec, (size_t)cnt * rec * 8, kind, s);
  }
  return e;
}
}  // namespace

static int run_region_host_impl(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                                const hpac_region_t* host_region, const hpac_spec_t* spec,
                                int32_t team_begin, int32_t team_end, hpac_stats_t* stats,
                                char* err, size_t el);

// End-to-end entry with host buffers: H2D inputs, run, D2H outputs.
HPAC_API int hpac_run_region_host(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                                  const hpac_region_t* host_region, const hpac_spec_t* spec,
                                  hpac_stats_t* stats, char* err, size_t el) {
  return run_region_host_impl(grid, n, mapping, host_region, spec, 0, 0, stats, err, el);
}

// The same for one team range: only its column block of items moves.
HPAC_API int hpac_run_region_host_teams(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                                        const hpac_region_t* host_region, const hpac_spec_t* spec,
                                        int32_t team_begin, int32_t team_end, hpac_stats_t* stats,
                                        char* err, size_t el) {
  return run_region_host_impl(grid, n, mapping, host_region, spec, team_begin, team_end, stats,
                              err, el);
}

static int run_region_host_impl(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                                const hpac_region_t* host_region, const hpac_spec_t* spec,
                                int32_t team_begin, int32_t team_end, hpac_stats_t* stats,
                                char* err, size_t el) {
  if (!host_region) return fail(err, el, HPAC_ERR_CONFIG, "region is null");
  const bool ranged = team_begin != 0 || team_end != 0;
  int64_t col0 = 0, col1 = 0, colG = 0;  // the range's column block (ranged only)
  if (ranged) {
    int vr = validate_grid(grid, err, el);
    if (vr) return vr;
    if (host_region->app != HPAC_APP_BLACKSCHOLES && host_region->app != HPAC_APP_BINOMIAL)
      return fail(err, el, HPAC_ERR_UNSUPPORTED,
                  "team-range host entry: Blackscholes and Binomial regions only");
    if (team_begin < 0 || team_end > grid->num_teams || team_begin > team_end)
      return fail(err, el, HPAC_ERR_CONFIG, "team range [%d, %d) outside [0, %d)", team_begin,
                  team_end, grid->num_teams);
    const int64_t w = mapping == HPAC_MAP_PER_TEAM ? 1 : grid->threads_per_team;
    col0 = team_begin * w;
    col1 = team_end * w;
    colG = (int64_t)grid->num_teams * w;
  }
  hpac_region_t r = *host_region;
  int rc = bind_region(&r, err, el);
  if (rc) return rc;
  const size_t nn = (size_t)(n > 0 ? n : 0);
  size_t in_bytes = 0, tab_bytes = 0, enc_bytes = 0, out_bytes = 0, cen_bytes = 0, lab_bytes = 0;
  switch (r.app) {
    case HPAC_APP_TABLE:
      in_bytes = r.in ? nn * r.input_dims * 8 : 0;
      tab_bytes = nn * r.output_dims * 8;
      enc_bytes = r.encounters ? nn * 4 : 0;
      out_bytes = r.out ? nn * r.output_dims * 8 : 0;
      break;
    case HPAC_APP_SYNTHETIC: out_bytes = r.out ? nn * 8 : 0; break;
    case HPAC_APP_BLACKSCHOLES:
    case HPAC_APP_BINOMIAL:
      in_bytes = nn * 40;
      out_bytes = r.out ? nn * 8 : 0;
      break;
    case HPAC_APP_LAVAMD: {
      const size_t parts = (size_t)r.lavamd_boxes1d * r.lavamd_boxes1d * r.lavamd_boxes1d *
                           (size_t)r.lavamd_particles;
      in_bytes = parts * 32;   // rv (v, x, y, z) of every box (neighbours)
      tab_bytes = parts * 8;   // qv
      out_bytes = parts * 32;  // fv (accumulated in place)
      break;
    }
    case HPAC_APP_KMEANS:
      in_bytes = nn * r.kmeans_dims * 8;
      cen_bytes = (size_t)r.kmeans_k * r.kmeans_dims * 8;
      out_bytes = r.out ? nn * r.kmeans_k * 8 : 0;
      lab_bytes = r.labels ? nn * 4 : 0;
      break;
  }
  cudaStream_t st = nullptr;
  cudaError_t e;
  std::vector<void*> bufs;
  cudaError_t alloc_e = cudaSuccess;  // first allocation / copy failure
  const char* alloc_what = nullptr;
  auto dalloc = [&](size_t bytes, const void* src, bool copy, const char* what) -> void* {
    if (!bytes || alloc_e != cudaSuccess) return nullptr;
    void* d = nullptr;
    cudaMemPool_t pool = host_entry_pool();
    cudaError_t ae = pool ? cudaMallocFromPoolAsync(&d, bytes, pool, st) : cudaMallocAsync(&d, bytes, st);
    if (ae == cudaSuccess) {
      bufs.push_back(d);
      if (copy && src) ae = cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st);
    }
    if (ae != cudaSuccess) {
      alloc_e = ae;
      alloc_what = what;
      return nullptr;
    }
    return d;
  };
  auto release = [&]() {
    for (void* b : bufs) cudaFreeAsync(b, st);
    cudaStreamSynchronize(st);
  };
  hpac_region_t d = r;
  // Zero-copy for the stream-once regions (Blackscholes; the K-Means labels
  // region): when the caller's buffers are pinned, the kernel reads the
  // inputs and writes the outputs over PCIe in place, so the host->device
  // and device->host transfers overlap each other and the compute instead
  // of running back to back. The generic per-thread engine is used: its
  // independent per-lane loads keep more PCIe reads in flight than one bulk
  // copy per team. HPAC_HOST_COPY=1 keeps the staged path.
  const bool zc_app = r.app == HPAC_APP_BLACKSCHOLES || (r.app == HPAC_APP_KMEANS && !r.out);
  const char* hc = getenv("HPAC_HOST_COPY");
  const bool zero_copy = zc_app && !(hc && strcmp(hc, "1") == 0) && pinned_device_ptr(r.in) &&
                         (!r.out || pinned_device_ptr(r.out)) &&
                         (!r.labels || pinned_device_ptr(r.labels));
  if (zero_copy) {
    d.in = (const double*)pinned_device_ptr(r.in);
    d.out = (double*)pinned_device_ptr(r.out);
    d.labels = (int32_t*)pinned_device_ptr(r.labels);
    d.centroids = (const double*)dalloc(cen_bytes, r.centroids, true, "centroids");  // read per CTA: stage
  } else {
    d.in = (const double*)dalloc(in_bytes, r.in, !ranged, "inputs");
    d.table_out = (const double*)dalloc(tab_bytes, r.table_out, true, "table_out");
    d.encounters = (const int32_t*)dalloc(enc_bytes, r.encounters, true, "encounters");
    // outputs start from the caller's contents where an item can be left
    // untouched (perforation skips, accumulating stores, LavaMD's fv +=);
    // the option regions otherwise write every item, so nothing is copied in
    const bool keeps = (spec && spec->technique == HPAC_TECH_PERFO) ||
                       !(r.app == HPAC_APP_BLACKSCHOLES || r.app == HPAC_APP_BINOMIAL);
    d.out = (double*)dalloc(out_bytes, r.out, keeps && !ranged, "outputs");
    if (ranged && alloc_e == cudaSuccess) {  // the range's column block only
      cudaError_t ce = copy_column_block(const_cast<double*>(d.in), r.in, n, colG, col0, col1, 5,
                                         cudaMemcpyHostToDevice, st);
      if (ce == cudaSuccess && keeps && d.out)
        ce = copy_column_block(d.out, r.out, n, colG, col0, col1, 1, cudaMemcpyHostToDevice, st);
      if (ce != cudaSuccess) {
        alloc_e = ce;
        alloc_what = "the team range's inputs";
      }
    }
    d.centroids = (const double*)dalloc(cen_bytes, r.centroids, true, "centroids");
    d.labels = (int32_t*)dalloc(lab_bytes, r.labels, true, "labels");
  }
  if (alloc_e != cudaSuccess) {
    release();
    cudaGetLastError();
    return fail(err, el, HPAC_ERR_CUDA, "CUDA error staging %s: %s", alloc_what,
                cudaGetErrorString(alloc_e));
  }
  hpac_launch_t L{};
  L.stream = st;
  L.synchronous = 1;
  L.team_begin = team_begin;
  L.team_end = team_end;
  g_force_thread_engine = zero_copy;
  rc = hpac_run_region(grid, n, mapping, &d, spec, &L, stats, err, el);
  g_force_thread_engine = false;
  if (stats) stats->zero_copy = zero_copy ? 1 : 0;
  if (rc == HPAC_OK && !zero_copy) {
    if (out_bytes && ranged &&
        (e = copy_column_block(r.out, d.out, n, colG, col0, col1, 1, cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess)
      rc = cuda_fail(err, el, e, "copying outputs to the host");
    if (out_bytes && !ranged &&
        (e = cudaMemcpyAsync(r.out, d.out, out_bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      rc = cuda_fail(err, el, e, "copying outputs to the host");
    if (rc == HPAC_OK && lab_bytes &&
        (e = cudaMemcpyAsync(r.labels, d.labels, lab_bytes, cudaMemcpyDeviceToHost, st)) !=
            cudaSuccess)
      rc = cuda_fail(err, el, e, "copying labels to the host");
  }
  for (void* b : bufs) cudaFreeAsync(b, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess && rc == HPAC_OK)
    rc = cuda_fail(err, el, e, "host entry");
  return rc;
}

// ---- metrics (metrics.hpp:17-45), device buffers -------------------------
HPAC_API int hpac_mape(const double* a, const double* b, int64_t n, void* stream, double* result) {
  if (n <= 0) {
    *result = 0.0;
    return HPAC_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* d_sum;
  unsigned long long* d_inf;
  if (cudaMallocAsync(&d_sum, 16, st) != cudaSuccess) return HPAC_ERR_CUDA;
  d_inf = reinterpret_cast<unsigned long long*>(d_sum + 1);
  cudaMemsetAsync(d_sum, 0, 16, st);
  if (mape_launch(a, b, n, d_sum, d_inf, st) != cudaSuccess) return HPAC_ERR_CUDA;
  double h[2];
  cudaMemcpyAsync(h, d_sum, 16, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_sum, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return HPAC_ERR_CUDA;
  unsigned long long infc;
  std::memcpy(&infc, &h[1], 8);
  *result = infc ? INFINITY : h[0] / (double)n;
  return HPAC_OK;
}

HPAC_API int hpac_mcr(const int32_t* a, const int32_t* b, int64_t n, void* stream, double* result) {
  if (n <= 0) {
    *result = 0.0;
    return HPAC_OK;
  }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* d;
  if (cudaMallocAsync(&d, 8, st) != cudaSuccess) return HPAC_ERR_CUDA;
  cudaMemsetAsync(d, 0, 8, st);
  if (mcr_launch(a, b, n, d, st) != cudaSuccess) return HPAC_ERR_CUDA;
  unsigned long long h;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return HPAC_ERR_CUDA;
  *result = (double)h / (double)n;
  return HPAC_OK;
}
