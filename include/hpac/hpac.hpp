// hpac/hpac.hpp — C++ host API over the C-ABI (include/hpac_offload.h).
//
// Mirrors the reference's approx-region API so a simtac user switches by
// changing the namespace (paths relative to /root/reference/proj/include/simtac/):
//
//   hpac::GridConfig, WorkMapping         <- grid.hpp:14-54
//   hpac::ApproxSpec, parse_directive     <- directive.hpp:59-84, :522-554
//   hpac::Region (+ app builders)         <- engine.hpp:26-33, bench/*.hpp
//   hpac::run_region -> LaunchResult      <- engine.hpp:132-134, :35-54
//   hpac::kmeans_benchmark                <- bench/kmeans.hpp:62-144
//   exceptions                            <- errors.hpp:12-62, directive.hpp:120
//
// Header-only; link libhpac_b200.so. Buffers are device pointers (the
// caller owns them); run_region_host takes host pointers instead.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>

#include "hpac_offload.h"

namespace hpac {

// ---- errors (errors.hpp:12-62) --------------------------------------------
class SimtError : public std::runtime_error {
 public:
  explicit SimtError(const std::string& w) : std::runtime_error(w) {}
};
class ConfigError : public SimtError {
 public:
  explicit ConfigError(const std::string& w) : SimtError(w) {}
};
class ArenaOverflowError : public SimtError {
 public:
  ArenaOverflowError(const std::string& w, std::size_t req, std::size_t avail)
      : SimtError(w), required_bytes(req), available_bytes(avail) {}
  std::size_t required_bytes, available_bytes;
};
class BarrierDivergenceError : public SimtError {
 public:
  BarrierDivergenceError(const std::string& w, int team, long long step, int missing)
      : SimtError(w), team_id(team), step(step), missing(missing) {}
  int team_id;
  long long step;
  int missing;
};
class DirectiveError : public SimtError {
 public:
  DirectiveError(const std::string& w, int code, long long offset)
      : SimtError(w), code(code), offset(offset) {}
  int code;
  long long offset;
};
class UnsupportedError : public SimtError {
 public:
  explicit UnsupportedError(const std::string& w) : SimtError(w) {}
};
class CudaError : public SimtError {
 public:
  explicit CudaError(const std::string& w) : SimtError(w) {}
};

namespace detail {
inline void check(int rc, const char* err, const hpac_stats_t* st = nullptr) {
  switch (rc) {
    case HPAC_OK: return;
    case HPAC_ERR_CONFIG: throw ConfigError(err);
    case HPAC_ERR_ARENA_OVERFLOW:
      throw ArenaOverflowError(err, st ? st->arena_required : 0, st ? st->arena_available : 0);
    case HPAC_ERR_BARRIER_DIVERGENCE:
      throw BarrierDivergenceError(err, st ? st->fail_team : 0, st ? st->fail_step : 0,
                                   st ? st->fail_missing : 0);
    case HPAC_ERR_UNSUPPORTED: throw UnsupportedError(err);
    case HPAC_ERR_CUDA: throw CudaError(err);
    default: throw SimtError(err);
  }
}
}  // namespace detail

// ---- grid (grid.hpp:14-54) --------------------------------------------------
enum class WorkMapping : int32_t { kPerThread = HPAC_MAP_PER_THREAD, kPerTeam = HPAC_MAP_PER_TEAM };

struct GridConfig {
  int num_teams = 1;
  int threads_per_team = 32;
  int warp_size = 32;
  int items_per_thread = 1;
  std::size_t shared_mem_budget_bytes = 48 * 1024;

  int total_threads() const { return num_teams * threads_per_team; }
  int warps_per_team() const { return threads_per_team / warp_size; }
  hpac_grid_t c() const {
    return {num_teams, threads_per_team, warp_size, items_per_thread, shared_mem_budget_bytes};
  }
};

// bench::resolve_grid (bench/run.hpp:81-97)
inline GridConfig resolve_grid(const std::string& benchmark, long long n, const GridConfig* ov = nullptr,
                               WorkMapping* mapping = nullptr) {
  hpac_grid_t o{}, out{};
  if (ov) o = {ov->num_teams, ov->threads_per_team, ov->warp_size, ov->items_per_thread,
               ov->shared_mem_budget_bytes};
  int32_t m = 0;
  char err[512];
  detail::check(hpac_resolve_grid(benchmark.c_str(), n, &o, &out, &m, err, sizeof err), err);
  if (mapping) *mapping = static_cast<WorkMapping>(m);
  return {out.num_teams, out.threads_per_team, out.warp_size, out.items_per_thread,
          out.shared_mem_budget_bytes};
}

// ---- spec (directive.hpp:59-84) -------------------------------------------
enum class Technique : int32_t { kTaf = HPAC_TECH_TAF, kIact = HPAC_TECH_IACT, kPerfo = HPAC_TECH_PERFO };
enum class Level : int32_t { kThread = HPAC_LEVEL_THREAD, kWarp = HPAC_LEVEL_WARP, kTeam = HPAC_LEVEL_TEAM };
enum class PerfoKind : int32_t {
  kSmall = HPAC_PERFO_SMALL, kLarge = HPAC_PERFO_LARGE, kIni = HPAC_PERFO_INI, kFini = HPAC_PERFO_FINI,
  kHerdedSmall = HPAC_PERFO_HERDED_SMALL, kHerdedLarge = HPAC_PERFO_HERDED_LARGE,
  kRandom = HPAC_PERFO_RANDOM
};

struct ApproxSpec {
  hpac_spec_t s{};
  std::string text;  // canonical directive (unparse)

  Technique technique() const { return static_cast<Technique>(s.technique); }
  Level level() const { return static_cast<Level>(s.level); }

  static ApproxSpec taf(int h, int p, double thr, Level lv = Level::kThread) {
    ApproxSpec a;
    a.s.technique = HPAC_TECH_TAF;
    a.s.level = static_cast<int32_t>(lv);
    a.s.taf_h_size = h;
    a.s.taf_p_size = p;
    a.s.taf_threshold = thr;
    a.s.n_output_sections = 1;
    return a;
  }
  static ApproxSpec iact(int table_size, double thr, int tables_per_warp = 0,
                         Level lv = Level::kThread) {
    ApproxSpec a;
    a.s.technique = HPAC_TECH_IACT;
    a.s.level = static_cast<int32_t>(lv);
    a.s.iact_table_size = table_size;
    a.s.iact_threshold = thr;
    a.s.iact_tables_per_warp = tables_per_warp;
    a.s.n_input_sections = a.s.n_output_sections = 1;
    return a;
  }
  static ApproxSpec perfo(PerfoKind kind, int arg, Level lv = Level::kThread, uint64_t seed = 0) {
    ApproxSpec a;
    a.s.technique = HPAC_TECH_PERFO;
    a.s.level = static_cast<int32_t>(lv);
    a.s.perfo_kind = static_cast<int32_t>(kind);
    if (kind == PerfoKind::kIni || kind == PerfoKind::kFini || kind == PerfoKind::kRandom)
      a.s.perfo_skip_percent = arg;
    else
      a.s.perfo_modulus = arg;
    a.s.perfo_seed = seed;
    return a;
  }
};

// parse_directive (directive.hpp:522)
inline ApproxSpec parse_directive(const std::string& text) {
  ApproxSpec a;
  int32_t code = -1;
  int64_t off = -1;
  char buf[2048];
  int rc = hpac_parse_directive(text.c_str(), &a.s, &code, &off, buf, sizeof buf);
  if (rc == HPAC_ERR_DIRECTIVE) throw DirectiveError(buf, code, off);
  detail::check(rc, buf);
  a.text = buf;
  return a;
}

// unparse (directive.hpp:528-554)
inline std::string unparse(const ApproxSpec& a) {
  if (!a.text.empty()) return a.text;
  char buf[1024];
  detail::check(hpac_unparse(&a.s, buf, sizeof buf), "unparse failed");
  return buf;
}

// ---- regions (engine.hpp:26-33 + bench/*.hpp builders) -----------------------
struct Region {
  hpac_region_t r{};
};

inline Region table_region(int input_dims, int output_dims, const double* in, const double* table_out,
                           double* out, const int32_t* encounters = nullptr, int flags = 0) {
  Region g;
  g.r.app = HPAC_APP_TABLE;
  g.r.input_dims = input_dims;
  g.r.output_dims = output_dims;
  g.r.in = in;
  g.r.table_out = table_out;
  g.r.out = out;
  g.r.encounters = encounters;
  g.r.flags = flags;
  return g;
}
inline Region synthetic_region(int profile, uint64_t seed, double* out) {
  Region g;
  g.r.app = HPAC_APP_SYNTHETIC;
  g.r.synthetic_profile = profile;
  g.r.seed = seed;
  g.r.out = out;
  return g;
}
inline Region blackscholes_region(const double* options, double* prices) {
  Region g;
  g.r.app = HPAC_APP_BLACKSCHOLES;
  g.r.in = options;
  g.r.out = prices;
  return g;
}
inline Region binomial_region(const double* options, int n_steps, double* prices, bool american = true,
                              bool put = true) {
  Region g;
  g.r.app = HPAC_APP_BINOMIAL;
  g.r.in = options;
  g.r.out = prices;
  g.r.binomial_steps = n_steps;
  g.r.binomial_american = american;
  g.r.binomial_put = put;
  return g;
}
inline Region kmeans_region(const double* points, int dims, const double* centroids, int k,
                            int32_t* labels, double* distances = nullptr) {
  Region g;
  g.r.app = HPAC_APP_KMEANS;
  g.r.in = points;
  g.r.kmeans_dims = dims;
  g.r.centroids = centroids;
  g.r.kmeans_k = k;
  g.r.labels = labels;
  g.r.out = distances;
  return g;
}

// LavaMD (extension): one home box per item under
// WorkMapping::kPerTeam with threads_per_team == particles; rv (v,x,y,z) and
// qv per particle (32-byte aligned rv), fv accumulated in place.
inline Region lavamd_region(const double* rv, const double* qv, double* fv, int boxes1d, int particles,
                            double alpha = 0.5) {
  Region g;
  g.r.app = HPAC_APP_LAVAMD;
  g.r.in = rv;
  g.r.table_out = qv;
  g.r.out = fv;
  g.r.lavamd_boxes1d = boxes1d;
  g.r.lavamd_particles = particles;
  g.r.lavamd_alpha = alpha;
  return g;
}

// ---- launch (engine.hpp:35-54, :132-134) --------------------------------------
struct KernelStats {
  uint64_t total_invocations = 0, approx_invocations = 0, divergent_warp_steps = 0,
           total_warp_steps = 0;
};

struct LaunchResult {
  KernelStats stats;
  int resident_warps = 0;
  double kernel_ms = 0.0;  // measured device time (replaces the cost model's device_time)
  double approx_rate() const {
    return stats.total_invocations == 0
               ? 0.0
               : static_cast<double>(stats.approx_invocations) / stats.total_invocations;
  }
  double divergent_fraction() const {
    return stats.total_warp_steps == 0
               ? 0.0
               : static_cast<double>(stats.divergent_warp_steps) / stats.total_warp_steps;
  }
};

namespace detail {
inline LaunchResult to_result(const hpac_stats_t& st) {
  LaunchResult lr;
  lr.stats = {st.total_invocations, st.approx_invocations, st.divergent_warp_steps,
              st.total_warp_steps};
  lr.resident_warps = st.resident_warps;
  lr.kernel_ms = st.kernel_ms;
  return lr;
}
}  // namespace detail

inline LaunchResult run_region(const GridConfig& grid, long long n, WorkMapping mapping,
                               const Region& region, const ApproxSpec* spec, void* stream = nullptr,
                               uint8_t* paths = nullptr) {
  hpac_grid_t g = grid.c();
  hpac_launch_t L{};
  L.stream = stream;
  L.paths = paths;
  L.synchronous = 1;
  hpac_stats_t st{};
  char err[1024];
  int rc = hpac_run_region(&g, n, static_cast<int32_t>(mapping), &region.r, spec ? &spec->s : nullptr,
                           &L, &st, err, sizeof err);
  detail::check(rc, err, &st);
  return detail::to_result(st);
}

inline LaunchResult run_region_host(const GridConfig& grid, long long n, WorkMapping mapping,
                                    const Region& host_region, const ApproxSpec* spec) {
  hpac_grid_t g = grid.c();
  hpac_stats_t st{};
  char err[1024];
  int rc = hpac_run_region_host(&g, n, static_cast<int32_t>(mapping), &host_region.r,
                                spec ? &spec->s : nullptr, &st, err, sizeof err);
  detail::check(rc, err, &st);
  return detail::to_result(st);
}

// One team range [team_begin, team_end) of the grid with host buffers: only
// the range's items move (the per-rank call of a multi-GPU split).
inline LaunchResult run_region_host_teams(const GridConfig& grid, long long n, WorkMapping mapping,
                                          const Region& host_region, const ApproxSpec* spec,
                                          int team_begin, int team_end) {
  hpac_grid_t g = grid.c();
  hpac_stats_t st{};
  char err[1024];
  int rc = hpac_run_region_host_teams(&g, n, static_cast<int32_t>(mapping), &host_region.r,
                                      spec ? &spec->s : nullptr, team_begin, team_end, &st, err,
                                      sizeof err);
  detail::check(rc, err, &st);
  return detail::to_result(st);
}

// ---- K-Means (bench/kmeans.hpp:62-144) --------------------------------------
struct KmeansResult {
  int iterations = 0;
  bool converged = false;
  KernelStats stats;
  double region_ms = 0.0, update_ms = 0.0;
  bool graph = false;  // the iterations ran as one CUDA graph launch
};

inline KmeansResult kmeans_benchmark(const double* points, long long n, int dims, int k,
                                     double* centroids, int32_t* assignments, const GridConfig& grid,
                                     const ApproxSpec* spec, int max_iters = 40, void* stream = nullptr,
                                     hpac_allreduce_fn allreduce = nullptr, void* user = nullptr) {
  hpac_kmeans_problem_t p{};
  p.n_points = n;
  p.dims = dims;
  p.k = k;
  p.points = points;
  p.centroids = centroids;
  p.assignments = assignments;
  p.max_iters = max_iters;
  p.allreduce = allreduce;
  p.allreduce_user = user;
  hpac_grid_t g = grid.c();
  hpac_kmeans_result_t r{};
  char err[1024];
  int rc = hpac_kmeans_run(&g, &p, spec ? &spec->s : nullptr, stream, &r, err, sizeof err);
  detail::check(rc, err, &r.stats);
  KmeansResult out;
  out.iterations = r.iterations;
  out.converged = r.converged;
  out.stats = {r.stats.total_invocations, r.stats.approx_invocations, r.stats.divergent_warp_steps,
               r.stats.total_warp_steps};
  out.region_ms = r.region_ms;
  out.update_ms = r.update_ms;
  out.graph = r.graph != 0;
  return out;
}

}  // namespace hpac
