// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library (simtac,
// header-only C++20), compiled straight from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libsimtac_ref.so. Nothing from the
// reference is copied into this repository; this file only adapts the
// reference's own API (run_region, the bench Regions and generators,
// parse_directive, taf_reference_oracle, kmeans_benchmark, mape/mcr) to the
// flat C structs of include/hpac_offload.h so Python tests and bench.py's
// reference arm can call it.
//
// Used for: pinning oracle/hpac_oracle.c (differential tests), generating
// the golden fixtures under tests/golden/, and timing the reference's CPU
// path (bench.py --impl reference, cpu_baseline).
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "hpac_offload.h"
#include "simtac/bench/binomial.hpp"
#include "simtac/bench/blackscholes.hpp"
#include "simtac/bench/kmeans.hpp"
#include "simtac/bench/run.hpp"
#include "simtac/bench/synthetic.hpp"
#include "simtac/directive.hpp"
#include "simtac/engine.hpp"
#include "simtac/metrics.hpp"
#include "simtac/taf_oracle.hpp"

using namespace simtac;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

void put_err(char* err, size_t len, const std::string& msg) {
  if (!err || !len) return;
  std::strncpy(err, msg.c_str(), len - 1);
  err[len - 1] = 0;
}

// hpac_spec_t -> ApproxSpec (directive.hpp:59-84)
bool to_spec(const hpac_spec_t* s, ApproxSpec& out, std::string& why) {
  out = ApproxSpec{};
  switch (s->technique) {
    case HPAC_TECH_TAF:
      out.technique = Technique::kTaf;
      out.taf = TafConfig{s->taf_h_size, s->taf_p_size, s->taf_threshold};
      break;
    case HPAC_TECH_IACT: {
      out.technique = Technique::kIact;
      IactConfig c;
      c.table_size = s->iact_table_size;
      c.threshold = s->iact_threshold;
      if (s->iact_tables_per_warp != 0) c.tables_per_warp = s->iact_tables_per_warp;
      out.iact = c;
      break;
    }
    case HPAC_TECH_PERFO: {
      out.technique = Technique::kPerfo;
      PerfoConfig c;
      switch (s->perfo_kind) {
        case HPAC_PERFO_SMALL: c.kind = PerfoKind::kSmall; break;
        case HPAC_PERFO_LARGE: c.kind = PerfoKind::kLarge; break;
        case HPAC_PERFO_INI: c.kind = PerfoKind::kIni; break;
        case HPAC_PERFO_FINI: c.kind = PerfoKind::kFini; break;
        case HPAC_PERFO_HERDED_SMALL: c.kind = PerfoKind::kHerdedSmall; break;
        case HPAC_PERFO_HERDED_LARGE: c.kind = PerfoKind::kHerdedLarge; break;
        default: why = "perforation kind not in the reference"; return false;
      }
      c.modulus = s->perfo_modulus;
      c.skip_percent = s->perfo_skip_percent;
      out.perfo = c;
      break;
    }
    default: why = "unknown technique"; return false;
  }
  switch (s->level) {
    case HPAC_LEVEL_THREAD: out.level = Level::kThread; break;
    case HPAC_LEVEL_WARP: out.level = Level::kWarp; break;
    case HPAC_LEVEL_TEAM: out.level = Level::kTeam; break;
    default: why = "unknown level"; return false;
  }
  ArraySection sec{"x", {1, 0}, SectionDim::literal(1), SectionDim::literal(1)};
  for (int i = 0; i < s->n_input_sections; ++i) out.inputs.push_back(sec);
  for (int i = 0; i < s->n_output_sections; ++i) out.outputs.push_back(sec);
  return true;
}

GridConfig to_grid(const hpac_grid_t* g) {
  GridConfig c;
  c.num_teams = g->num_teams;
  c.threads_per_team = g->threads_per_team;
  c.warp_size = g->warp_size;
  c.items_per_thread = g->items_per_thread;
  c.shared_mem_budget_bytes = g->shared_mem_budget_bytes;
  return c;
}

void fill_stats(const LaunchResult& lr, hpac_stats_t* st) {
  st->total_invocations = lr.stats.total_invocations;
  st->approx_invocations = lr.stats.approx_invocations;
  st->divergent_warp_steps = lr.stats.divergent_warp_steps;
  st->total_warp_steps = lr.stats.total_warp_steps;
  st->resident_warps = lr.resident_warps;
  st->barrier_divergence_detected = lr.stats.barrier_divergence_detected;
}

// Run `region` through the reference engine, mapping exceptions to status
// codes (engine.hpp:128-131, errors.hpp).
int run_guarded(const hpac_grid_t* g, int64_t n, int32_t mapping, const Region& region,
                const hpac_spec_t* s, hpac_stats_t* st, char* err, size_t errlen) {
  std::memset(st, 0, sizeof *st);
  ApproxSpec spec;
  if (s) {
    std::string why;
    if (!to_spec(s, spec, why)) {
      put_err(err, errlen, why);
      return HPAC_ERR_UNSUPPORTED;
    }
  }
  try {
    LaunchResult lr = run_region(to_grid(g), n,
                                 mapping == HPAC_MAP_PER_TEAM ? WorkMapping::kPerTeam
                                                              : WorkMapping::kPerThread,
                                 region, s ? &spec : nullptr);
    fill_stats(lr, st);
    return HPAC_OK;
  } catch (const ArenaOverflowError& e) {
    st->arena_required = e.required_bytes;
    st->arena_available = e.available_bytes;
    put_err(err, errlen, e.what());
    return HPAC_ERR_ARENA_OVERFLOW;
  } catch (const BarrierDivergenceError& e) {
    st->barrier_divergence_detected = 1;
    st->fail_team = e.team_id;
    st->fail_step = e.step;
    st->fail_missing = static_cast<int32_t>(e.missing_threads.size());
    put_err(err, errlen, e.what());
    return HPAC_ERR_BARRIER_DIVERGENCE;
  } catch (const ConfigError& e) {
    put_err(err, errlen, e.what());
    return HPAC_ERR_CONFIG;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return HPAC_ERR_CONFIG;
  }
}

// Path logging: an (item, encounter) is approximate unless the reference
// called evaluate for it (lane 0 of the team under per-team mapping).
struct PathLog {
  uint8_t* paths = nullptr;
  bool per_team = false;
  void init(int64_t n, const int32_t* enc) {
    if (!paths) return;
    for (int64_t i = 0; i < n; ++i) {
      int e = enc ? enc[i] : 1;
      uint8_t bits = 0;
      for (int r = 0; r < e && r < 8; ++r) bits |= uint8_t(1u << r);
      paths[i] = bits;
    }
  }
  void evaluated(const LaneCtx& ctx) {
    if (!paths || ctx.encounter >= 8) return;
    if (per_team && ctx.thread_in_team != 0) return;
    paths[ctx.index] &= uint8_t(~(1u << ctx.encounter));
  }
};

}  // namespace

REF_API int ref_abi_version() { return HPAC_ABI_VERSION; }

// Generic TABLE region through the reference engine (any pure region).
REF_API int ref_run_region(const hpac_grid_t* g, int64_t n, int32_t mapping,
                           const hpac_region_t* r, const hpac_spec_t* s, hpac_stats_t* st,
                           uint8_t* paths, char* err, size_t errlen) {
  PathLog log;
  log.paths = paths;
  log.per_team = mapping == HPAC_MAP_PER_TEAM;
  Region region;
  std::vector<double> kdist;
  const int32_t* enc = nullptr;
  switch (r->app) {
    case HPAC_APP_TABLE: {
      int in_dims = r->input_dims, out_dims = r->output_dims;
      region.input_dims = in_dims;
      region.output_dims = out_dims;
      enc = r->encounters;
      if (enc) region.encounters = [enc](const LaneCtx& c) { return int(enc[c.index]); };
      if (in_dims > 0 && r->in)
        region.load_input = [r, in_dims](const LaneCtx& c, std::span<double> in) {
          for (int d = 0; d < in_dims; ++d) in[d] = r->in[c.index * in_dims + d];
        };
      if (r->table_out) {
        bool barrier = (r->flags & HPAC_REGION_BARRIER_IN_EVALUATE) != 0;
        region.evaluate = [r, out_dims, barrier, &log](LaneCtx& c, std::span<const double>,
                                                      std::span<double> o) {
          if (barrier) c.team_barrier();
          for (int d = 0; d < out_dims; ++d) o[d] = r->table_out[c.index * out_dims + d];
          log.evaluated(c);
        };
      }
      bool acc = (r->flags & HPAC_REGION_STORE_ACCUMULATE) != 0;
      region.store = [r, out_dims, acc](const LaneCtx& c, std::span<const double> o) {
        if (!r->out) return;
        for (int d = 0; d < out_dims; ++d) {
          if (acc)
            r->out[c.index * out_dims + d] += o[d];
          else
            r->out[c.index * out_dims + d] = o[d];
        }
      };
      break;
    }
    case HPAC_APP_SYNTHETIC: {
      auto prof = static_cast<bench::SyntheticProfile>(r->synthetic_profile);
      uint64_t seed = r->seed;
      region.input_dims = 1;
      region.output_dims = 1;
      region.load_input = [prof, seed](const LaneCtx& c, std::span<double> in) {
        in[0] = bench::synthetic_value(prof, c.index, seed);
      };
      region.evaluate = [prof, seed, &log](LaneCtx& c, std::span<const double>,
                                           std::span<double> o) {
        o[0] = bench::synthetic_eval(bench::synthetic_value(prof, c.index, seed));
        log.evaluated(c);
      };
      region.store = [r](const LaneCtx& c, std::span<const double> o) {
        if (r->out) r->out[c.index] = o[0];
      };
      break;
    }
    case HPAC_APP_BLACKSCHOLES:
    case HPAC_APP_BINOMIAL: {
      const bench::BsOption* opts = reinterpret_cast<const bench::BsOption*>(r->in);
      region.input_dims = 5;
      region.output_dims = 1;
      region.load_input = [opts](const LaneCtx& c, std::span<double> in) {
        const bench::BsOption& o = opts[c.index];
        in[0] = o.spot;
        in[1] = o.strike;
        in[2] = o.rate;
        in[3] = o.vol;
        in[4] = o.maturity;
      };
      if (r->app == HPAC_APP_BLACKSCHOLES) {
        region.evaluate = [opts, &log](LaneCtx& c, std::span<const double>, std::span<double> o) {
          o[0] = bench::black_scholes_call(opts[c.index]);
          log.evaluated(c);
        };
      } else {
        int steps = r->binomial_steps;
        bool am = r->binomial_american, put = r->binomial_put;
        region.evaluate = [opts, steps, am, put, &log](LaneCtx& c, std::span<const double>,
                                                      std::span<double> o) {
          o[0] = bench::binomial_price(opts[c.index], steps, am, put);
          log.evaluated(c);
        };
      }
      region.store = [r](const LaneCtx& c, std::span<const double> o) {
        if (r->out) r->out[c.index] = o[0];
      };
      break;
    }
    case HPAC_APP_KMEANS: {
      int dims = r->kmeans_dims, k = r->kmeans_k;
      region.input_dims = dims;
      region.output_dims = k;
      region.load_input = [r, dims](const LaneCtx& c, std::span<double> in) {
        for (int d = 0; d < dims; ++d) in[d] = r->in[c.index * dims + d];
      };
      region.evaluate = [r, dims, k, &log](LaneCtx& c, std::span<const double>,
                                           std::span<double> out) {
        const double* pt = r->in + c.index * dims;
        for (int cc = 0; cc < k; ++cc) {
          double ssq = 0.0;
          for (int d = 0; d < dims; ++d) {
            double diff = pt[d] - r->centroids[cc * dims + d];
            ssq += diff * diff;
          }
          out[cc] = std::sqrt(ssq);
        }
        log.evaluated(c);
      };
      region.store = [r, k](const LaneCtx& c, std::span<const double> o) {
        if (r->out)
          for (int cc = 0; cc < k; ++cc) r->out[c.index * k + cc] = o[cc];
        if (r->labels) {
          int best = 0;
          double bd = o[0];
          for (int cc = 1; cc < k; ++cc)
            if (o[cc] < bd) {
              bd = o[cc];
              best = cc;
            }
          r->labels[c.index] = best;
        }
      };
      break;
    }
    default: put_err(err, errlen, "unsupported app"); return HPAC_ERR_UNSUPPORTED;
  }
  log.init(n, enc);
  return run_guarded(g, n, mapping, region, s, st, err, errlen);
}

// ---- application math + generators (bench/*.hpp) ------------------------
REF_API int ref_black_scholes_call(const double* o, double* price) {
  try {
    *price = bench::black_scholes_call({o[0], o[1], o[2], o[3], o[4]});
    return 0;
  } catch (const std::exception&) {
    return HPAC_ERR_CONFIG;
  }
}

REF_API int ref_binomial_price(const double* o, int n_steps, int american, int is_put,
                               double* price) {
  try {
    *price = bench::binomial_price({o[0], o[1], o[2], o[3], o[4]}, n_steps, american, is_put);
    return 0;
  } catch (const std::exception&) {
    return HPAC_ERR_CONFIG;
  }
}

// ---- the reference's stock benchmark regions and plain loops ---------------
// bench.py's reference arm times these: bench::binomial_region /
// bench::blackscholes_region (bench/binomial.hpp:74-94,
// bench/blackscholes.hpp:72-92) through run_region exactly as
// bench::detail::run_benchmark builds them (bench/run.hpp:133-165), and the
// plain per-option loops binomial_reference / blackscholes_reference
// (bench/binomial.hpp:96-102, bench/blackscholes.hpp:94-98).
static std::vector<bench::BsOption> to_options(const double* o, int64_t n) {
  std::vector<bench::BsOption> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i)
    v[i] = bench::BsOption{o[5 * i], o[5 * i + 1], o[5 * i + 2], o[5 * i + 3], o[5 * i + 4]};
  return v;
}

REF_API int ref_bench_binomial_run(const double* opts, int64_t n, int n_steps,
                                   const hpac_grid_t* g, const hpac_spec_t* s, double* prices,
                                   hpac_stats_t* st, char* err, size_t errlen) {
  const std::vector<bench::BsOption> options = to_options(opts, n);
  std::vector<double> out(static_cast<size_t>(n), 0.0);
  Region region = bench::binomial_region(options, n_steps, out);
  int rc = run_guarded(g, n, HPAC_MAP_PER_TEAM, region, s, st, err, errlen);
  if (prices) std::memcpy(prices, out.data(), sizeof(double) * static_cast<size_t>(n));
  return rc;
}

REF_API int ref_bench_blackscholes_run(const double* opts, int64_t n, const hpac_grid_t* g,
                                       const hpac_spec_t* s, double* prices, hpac_stats_t* st,
                                       char* err, size_t errlen) {
  const std::vector<bench::BsOption> options = to_options(opts, n);
  std::vector<double> out(static_cast<size_t>(n), 0.0);
  Region region = bench::blackscholes_region(options, out);
  int rc = run_guarded(g, n, HPAC_MAP_PER_THREAD, region, s, st, err, errlen);
  if (prices) std::memcpy(prices, out.data(), sizeof(double) * static_cast<size_t>(n));
  return rc;
}

REF_API void ref_binomial_reference(const double* opts, int64_t n, int n_steps, double* prices) {
  std::vector<double> out = bench::binomial_reference(to_options(opts, n), n_steps);
  std::memcpy(prices, out.data(), sizeof(double) * static_cast<size_t>(n));
}

REF_API void ref_blackscholes_reference(const double* opts, int64_t n, double* prices) {
  std::vector<double> out = bench::blackscholes_reference(to_options(opts, n));
  std::memcpy(prices, out.data(), sizeof(double) * static_cast<size_t>(n));
}

REF_API double ref_synthetic_value(int profile, int64_t i, uint64_t seed) {
  return bench::synthetic_value(static_cast<bench::SyntheticProfile>(profile), i, seed);
}

REF_API void ref_make_bs_portfolio(int64_t n, uint64_t seed, int base_block, double jitter,
                                   double* out) {
  auto p = bench::make_bs_portfolio(n, seed, base_block, jitter);
  std::memcpy(out, p.data(), sizeof(double) * 5 * static_cast<size_t>(n));
}

REF_API void ref_make_binomial_portfolio(int64_t n, uint64_t seed, double jitter, double* out) {
  auto p = bench::make_binomial_portfolio(n, seed, jitter);
  std::memcpy(out, p.data(), sizeof(double) * 5 * static_cast<size_t>(n));
}

REF_API void ref_make_blobs(int64_t n, int dims, int k, uint64_t seed, double separation,
                            double* out) {
  auto p = bench::make_blobs(n, dims, k, seed, separation);
  std::memcpy(out, p.points.data(), sizeof(double) * static_cast<size_t>(n) * dims);
}

// ---- K-Means Lloyd loop (bench/kmeans.hpp:62-144) -------------------------
REF_API int ref_kmeans_benchmark(const double* points, int64_t n, int dims, int k,
                                 const hpac_grid_t* g, const hpac_spec_t* s, int max_iters,
                                 int32_t* assignments, int32_t* iterations, int32_t* converged,
                                 hpac_stats_t* st, char* err, size_t errlen) {
  std::memset(st, 0, sizeof *st);
  bench::KmeansProblem p;
  p.dims = dims;
  p.k = k;
  p.n_points = n;
  p.points.assign(points, points + static_cast<size_t>(n) * dims);
  ApproxSpec spec;
  if (s) {
    std::string why;
    if (!to_spec(s, spec, why)) {
      put_err(err, errlen, why);
      return HPAC_ERR_UNSUPPORTED;
    }
  }
  try {
    bench::KmeansResult res =
        bench::kmeans_benchmark(p, to_grid(g), s ? &spec : nullptr, CostModel{}, max_iters);
    for (int64_t i = 0; i < n; ++i) assignments[i] = res.assignments[i];
    *iterations = res.iterations;
    *converged = res.converged;
    st->total_invocations = res.stats.total_invocations;
    st->approx_invocations = res.stats.approx_invocations;
    st->divergent_warp_steps = res.stats.divergent_warp_steps;
    st->total_warp_steps = res.stats.total_warp_steps;
    return HPAC_OK;
  } catch (const ArenaOverflowError& e) {
    st->arena_required = e.required_bytes;
    st->arena_available = e.available_bytes;
    put_err(err, errlen, e.what());
    return HPAC_ERR_ARENA_OVERFLOW;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return HPAC_ERR_CONFIG;
  }
}

// ---- TAF primitives (taf.hpp, taf_oracle.hpp) -----------------------------
REF_API double ref_rsd(const double* w, int len) {
  return rsd(std::span<const double>(w, static_cast<size_t>(len)));
}

// taf_step over a stream; same contract as oracle_taf_drive.
REF_API int64_t ref_taf_drive(int h, int p, double thr, const double* stream, int64_t len,
                              int64_t invocations, uint8_t* approx, double* outputs) {
  TafState st(TafConfig{h, p, thr});
  int64_t pos = 0, k = 0;
  for (; k < invocations; ++k) {
    if (!st.predicting() && pos >= len) break;
    TafStepResult r = taf_step(st, [&]() { return stream[pos++]; });
    approx[k] = r.took_approx_path;
    outputs[k] = r.output;
  }
  return k;
}

REF_API int64_t ref_taf_reference_oracle(int h, int p, double thr, const double* stream,
                                         int64_t len, int64_t invocations, uint8_t* approx,
                                         double* outputs) {
  auto tr = taf_reference_oracle(std::span<const double>(stream, static_cast<size_t>(len)),
                                 TafConfig{h, p, thr}, invocations);
  for (size_t i = 0; i < tr.size(); ++i) {
    approx[i] = tr[i].took_approx_path;
    outputs[i] = tr[i].output;
  }
  return static_cast<int64_t>(tr.size());
}

// ---- directive parser (directive.hpp) --------------------------------------
REF_API int ref_parse_directive(const char* text, hpac_spec_t* out, int32_t* code,
                                int64_t* offset, char* err, size_t errlen) {
  std::memset(out, 0, sizeof *out);
  try {
    ApproxSpec s = parse_directive(text);
    out->technique = static_cast<int32_t>(s.technique);
    out->level = static_cast<int32_t>(s.level);
    if (s.taf) {
      out->taf_h_size = s.taf->h_size;
      out->taf_p_size = s.taf->p_size;
      out->taf_threshold = s.taf->threshold;
    }
    if (s.iact) {
      out->iact_table_size = s.iact->table_size;
      out->iact_threshold = s.iact->threshold;
      out->iact_tables_per_warp = s.iact->tables_per_warp.value_or(0);
    }
    if (s.perfo) {
      out->perfo_kind = static_cast<int32_t>(s.perfo->kind);
      out->perfo_modulus = s.perfo->modulus;
      out->perfo_skip_percent = s.perfo->skip_percent;
    }
    out->n_input_sections = static_cast<int32_t>(s.inputs.size());
    out->n_output_sections = static_cast<int32_t>(s.outputs.size());
    put_err(err, errlen, unparse(s));  // canonical form on success
    return HPAC_OK;
  } catch (const DirectiveError& e) {
    *code = static_cast<int32_t>(e.code);
    *offset = static_cast<int64_t>(e.offset);
    put_err(err, errlen, e.what());
    return HPAC_ERR_DIRECTIVE;
  } catch (const std::exception& e) {
    *code = -1;
    *offset = -1;
    put_err(err, errlen, e.what());
    return HPAC_ERR_CONFIG;
  }
}

// ---- grid defaults (bench/run.hpp:41-97) -----------------------------------
REF_API int ref_resolve_grid(const char* benchmark, int64_t n, const hpac_grid_t* ov,
                             hpac_grid_t* out, int32_t* mapping) {
  try {
    const bench::BenchmarkInfo& info = bench::benchmark_info(benchmark);
    bench::TrialSetup s;
    s.items_per_thread = ov->items_per_thread;
    s.num_teams = ov->num_teams;
    s.threads_per_team = ov->threads_per_team;
    s.warp_size = ov->warp_size;
    if (ov->shared_mem_budget_bytes) s.shared_mem_budget_bytes = ov->shared_mem_budget_bytes;
    long long nn = n > 0 ? n : info.default_n;
    GridConfig g = bench::resolve_grid(info, s, nn);
    out->num_teams = g.num_teams;
    out->threads_per_team = g.threads_per_team;
    out->warp_size = g.warp_size;
    out->items_per_thread = g.items_per_thread;
    out->shared_mem_budget_bytes = g.shared_mem_budget_bytes;
    *mapping = info.mapping == WorkMapping::kPerTeam ? HPAC_MAP_PER_TEAM : HPAC_MAP_PER_THREAD;
    return HPAC_OK;
  } catch (const std::exception&) {
    return HPAC_ERR_CONFIG;
  }
}

// ---- metrics (metrics.hpp) --------------------------------------------------
REF_API double ref_mape(const double* a, const double* b, int64_t n) {
  return mape(std::span<const double>(a, static_cast<size_t>(n)),
              std::span<const double>(b, static_cast<size_t>(n)));
}

REF_API double ref_mcr(const int32_t* a, const int32_t* b, int64_t n) {
  std::vector<int> x(a, a + n), y(b, b + n);
  return mcr(x, y);
}
