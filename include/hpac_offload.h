/*
 * hpac_offload.h — C-ABI of the B200-native approximate-region engine.
 *
 * This is the drop-in boundary for the reference's approximate-region hot
 * path. Every entry point cites the reference interface it replaces
 * (paths relative to /root/reference/proj/include/simtac/):
 *
 *   hpac_run_region       <- run_region(grid, n, mapping, region, spec, model)
 *                            engine.hpp:132-134 (returns LaunchResult, engine.hpp:35-54)
 *   hpac_resolve_grid     <- bench::resolve_grid + benchmark_info   bench/run.hpp:41-97
 *   hpac_parse_directive  <- parse_directive                        directive.hpp:522
 *   hpac_unparse          <- unparse                                directive.hpp:528-554
 *   hpac_arena_required   <- bind_technique arena charges           engine.hpp:75-117
 *   hpac_make_*           <- make_bs_portfolio / make_binomial_portfolio / make_blobs
 *                            bench/blackscholes.hpp:42-68, bench/binomial.hpp:54-69,
 *                            bench/kmeans.hpp:25-47
 *   hpac_kmeans_run       <- kmeans_benchmark (Lloyd loop)           bench/kmeans.hpp:62-144
 *   hpac_mape / hpac_mcr  <- mape / mcr                              metrics.hpp:17-45
 *
 * A reference `Region` (engine.hpp:26-33) carries std::function callbacks,
 * which cannot cross to the device; here a region is an application id
 * (hpac_region_t.app) plus caller-owned buffers. HPAC_APP_TABLE is the
 * generic region: load_input reads `in`, evaluate returns `table_out`
 * (precomputed accurate outputs), store writes `out`; it expresses any pure
 * reference Region over a work index.
 *
 * Plain C types only; no torch or CUDA types in signatures (streams are
 * passed as void*, i.e. a cudaStream_t).
 *
 * Status codes map the reference exception taxonomy (errors.hpp:12-62):
 *   ConfigError -> HPAC_ERR_CONFIG, ArenaOverflowError -> HPAC_ERR_ARENA_OVERFLOW,
 *   BarrierDivergenceError -> HPAC_ERR_BARRIER_DIVERGENCE,
 *   DirectiveError -> HPAC_ERR_DIRECTIVE.
 */
#ifndef HPAC_OFFLOAD_H
#define HPAC_OFFLOAD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPAC_ABI_VERSION 4 /* v4: hpac_run_region_host_teams; v3: status-returning all-reduce hooks */

/* ---- status codes ------------------------------------------------------ */
#define HPAC_OK 0
#define HPAC_ERR_CONFIG 1
#define HPAC_ERR_ARENA_OVERFLOW 2
#define HPAC_ERR_BARRIER_DIVERGENCE 3
#define HPAC_ERR_CUDA 4
#define HPAC_ERR_DIRECTIVE 5
#define HPAC_ERR_UNSUPPORTED 6

/* ---- enums (values match the reference enum order) --------------------- */
/* WorkMapping, grid.hpp:14 */
#define HPAC_MAP_PER_THREAD 0
#define HPAC_MAP_PER_TEAM 1
/* Technique, directive.hpp:18; NONE = accurate baseline (null spec) */
#define HPAC_TECH_TAF 0
#define HPAC_TECH_IACT 1
#define HPAC_TECH_PERFO 2
/* Level, hierarchy.hpp:15 */
#define HPAC_LEVEL_THREAD 0
#define HPAC_LEVEL_WARP 1
#define HPAC_LEVEL_TEAM 2
/* PerfoKind, perfo.hpp:11; RANDOM is an extension (unpinned) */
#define HPAC_PERFO_SMALL 0
#define HPAC_PERFO_LARGE 1
#define HPAC_PERFO_INI 2
#define HPAC_PERFO_FINI 3
#define HPAC_PERFO_HERDED_SMALL 4
#define HPAC_PERFO_HERDED_LARGE 5
#define HPAC_PERFO_RANDOM 6
/* Applications (bench/*.hpp); LAVAMD is an extension (unpinned) */
#define HPAC_APP_TABLE 0
#define HPAC_APP_SYNTHETIC 1
#define HPAC_APP_BLACKSCHOLES 2
#define HPAC_APP_BINOMIAL 3
#define HPAC_APP_KMEANS 4
#define HPAC_APP_LAVAMD 5
/* SyntheticProfile, bench/synthetic.hpp:14 */
#define HPAC_SYNTH_CONSTANT 0
#define HPAC_SYNTH_SLOW_DRIFT 1
#define HPAC_SYNTH_NOISE 2
/* hpac_region_t.flags */
#define HPAC_REGION_STORE_ACCUMULATE 1   /* store adds into out (out[i] += o) */
#define HPAC_REGION_BARRIER_IN_EVALUATE 2 /* evaluate calls team_barrier() (machine.hpp:32) */
#define HPAC_REGION_KMEANS_FAST_MATH 4   /* K-Means distances with FMA contraction */

/* GridConfig, grid.hpp:16-54 */
typedef struct hpac_grid {
  int32_t num_teams;
  int32_t threads_per_team;
  int32_t warp_size;
  int32_t items_per_thread;
  uint64_t shared_mem_budget_bytes; /* default 48 KiB (grid.hpp:21) */
} hpac_grid_t;

/* ApproxSpec, directive.hpp:59-84 (one technique payload, flattened). */
typedef struct hpac_spec {
  int32_t technique;
  int32_t level;
  /* TafConfig, taf.hpp:14-25 */
  int32_t taf_h_size;
  int32_t taf_p_size;
  double taf_threshold;
  /* IactConfig, iact.hpp:16-41 */
  int32_t iact_table_size;
  int32_t iact_tables_per_warp; /* 0 = unset (one table per lane) */
  double iact_threshold;
  /* PerfoConfig, perfo.hpp:22-36 */
  int32_t perfo_kind;
  int32_t perfo_modulus;      /* SMALL / LARGE / HERDED_* */
  int32_t perfo_skip_percent; /* INI / FINI / RANDOM */
  int32_t reserved0;
  uint64_t perfo_seed; /* RANDOM only */
  /* in(...) / out(...) section counts; the engine only validates them
     (ApproxSpec::validate, directive.hpp:79-82) */
  int32_t n_input_sections;
  int32_t n_output_sections;
} hpac_spec_t;

/* KernelStats + LaunchResult decision stats (cost.hpp:50-57, engine.hpp:35-54).
   The cost model's estimated_cost/device_time are replaced by measured time. */
typedef struct hpac_stats {
  uint64_t total_invocations;
  uint64_t approx_invocations;
  uint64_t divergent_warp_steps;
  uint64_t total_warp_steps;
  int32_t resident_warps;
  int32_t barrier_divergence_detected;
  /* ArenaOverflowError{required, available} (arena.hpp:37-38) */
  uint64_t arena_required;
  uint64_t arena_available;
  /* BarrierDivergenceError{team, step, missing} (errors.hpp:49-62) */
  int64_t fail_step;
  int32_t fail_team;
  int32_t fail_missing;
  /* measured device time of the region kernel(s), milliseconds */
  double kernel_ms;
  /* binomial American-put lattices recomputed on the full triangle because
     the early-exercise boundary check failed (diagnostic; normally 0) */
  uint64_t lattice_fallbacks;
  /* binomial lattices: node updates actually executed (the full triangle is
     N(N+1)/2 per evaluated option; early-exercise tracking skips nodes whose
     value is the analytic exercise value) */
  uint64_t lattice_nodes;
  /* hpac_run_region_host: 1 = the kernel read/wrote the caller's pinned
     buffers in place (zero-copy), 0 = staged through device buffers */
  int32_t zero_copy;
  int32_t reserved0;
} hpac_stats_t;

/* Region descriptor (replaces engine.hpp:26-33). Pointers are caller-owned;
   device pointers for hpac_run_region, host pointers for hpac_run_region_host. */
typedef struct hpac_region {
  int32_t app;
  int32_t input_dims;  /* TABLE: caller sets; apps: filled from the app */
  int32_t output_dims; /* TABLE: caller sets; apps: filled from the app */
  int32_t flags;
  /* application parameters */
  int32_t synthetic_profile;
  int32_t binomial_steps;    /* lattice steps (bench/run.hpp:33 default 32) */
  int32_t binomial_american; /* binomial_price(american, is_put), binomial.hpp:16 */
  int32_t binomial_put;
  int32_t kmeans_dims;
  int32_t kmeans_k;
  int32_t lavamd_boxes1d; /* LAVAMD: boxes per dimension */
  int32_t lavamd_particles; /* LAVAMD: particles per box */
  uint64_t seed; /* SYNTHETIC noise seed */
  double lavamd_alpha;
  /* buffers */
  const double* in;          /* TABLE: n*input_dims; BS/BINOMIAL: n*5 options (S,K,r,vol,T);
                                KMEANS: n*d points (AoS); LAVAMD: rv n*4 */
  const double* table_out;   /* TABLE: n*output_dims accurate outputs; LAVAMD: qv n */
  const int32_t* encounters; /* TABLE: optional per-item encounter counts (NULL = 1) */
  double* out;               /* n*output_dims outputs; KMEANS: optional n*k distances */
  const double* centroids;   /* KMEANS: k*d */
  int32_t* labels;           /* KMEANS: n labels = argmin of the stored distances */
} hpac_region_t;

/* Launch controls. */
typedef struct hpac_launch {
  void* stream;       /* cudaStream_t (NULL = default stream) */
  int32_t team_begin; /* execute logical teams [team_begin, team_end); 0,0 = all */
  int32_t team_end;
  uint8_t* paths;     /* optional device buffer of n bytes: bit r set iff encounter r
                         of item i took the approximate path (per-team: lane 0) */
  int32_t synchronous; /* 1: wait and fill stats; 0: enqueue only (stats via
                          hpac_stats_fetch after the stream drains) */
  int32_t reserved;
} hpac_launch_t;

int hpac_abi_version(void);
const char* hpac_status_name(int status);

/* Default grid for a reference benchmark id ("blackscholes", "binomial",
   "kmeans", "synthetic-constant", "synthetic-slow-drift", "synthetic-noise",
   "lavamd"); nonzero override fields win (bench/run.hpp:81-97). */
int hpac_resolve_grid(const char* benchmark, int64_t n, const hpac_grid_t* overrides,
                      hpac_grid_t* out, int32_t* mapping_out, char* err, size_t errlen);

/* Directive text <-> spec (directive.hpp:522-554). On HPAC_ERR_DIRECTIVE,
   *err_code / *err_offset carry ParseErrorCode (directive.hpp:86-100) and
   the byte offset. */
int hpac_parse_directive(const char* text, hpac_spec_t* out, int32_t* err_code,
                         int64_t* err_offset, char* err, size_t errlen);
int hpac_unparse(const hpac_spec_t* spec, char* buf, size_t len);

/* Fill region dims from the app (no-op for TABLE). */
int hpac_region_bind(hpac_region_t* region, char* err, size_t errlen);

/* Per-team arena bytes bind_technique would charge; HPAC_ERR_ARENA_OVERFLOW
   with stats-style required/available when over budget. */
int hpac_arena_required(const hpac_grid_t* grid, const hpac_region_t* region,
                        const hpac_spec_t* spec, uint64_t* required, uint64_t* available,
                        char* err, size_t errlen);

/* Run one approximate region over [0, n) on the device. spec == NULL is
   the accurate baseline. */
int hpac_run_region(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                    const hpac_region_t* region, const hpac_spec_t* spec,
                    const hpac_launch_t* launch, hpac_stats_t* stats, char* err,
                    size_t errlen);

/* Same call with HOST buffers: copies inputs host->device, runs, copies
   outputs device->host (the reference-facing end-to-end entry). For the
   stream-once regions (Blackscholes, the K-Means labels region) with
   page-locked caller buffers the kernel reads and writes them in place
   instead (zero-copy over PCIe/C2C, both directions overlapped with the
   compute; stats->zero_copy = 1); HPAC_HOST_COPY=1 forces staging. */
int hpac_run_region_host(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                         const hpac_region_t* host_region, const hpac_spec_t* spec,
                         hpac_stats_t* stats, char* err, size_t errlen);

/* hpac_run_region_host for the logical teams [team_begin, team_end) of the
   grid only (the multi-GPU split of one global grid, machine.hpp:77-84:
   each rank runs a contiguous team range with the global stride). The
   range's items form a column block of the [steps x G] item matrix
   (per-team: columns [team_begin, team_end) of G = num_teams; per-thread:
   columns [team_begin, team_end) x threads_per_team of G = num_teams x
   threads_per_team), so only that block moves each way (2-D copies); items
   outside it are neither read nor written. Blackscholes and Binomial
   regions. team_begin = team_end = 0: the whole grid (= hpac_run_region_host). */
int hpac_run_region_host_teams(const hpac_grid_t* grid, int64_t n, int32_t mapping,
                               const hpac_region_t* host_region, const hpac_spec_t* spec,
                               int32_t team_begin, int32_t team_end, hpac_stats_t* stats,
                               char* err, size_t errlen);

/* Stats of the last asynchronous launch on this thread (after stream sync). */
int hpac_stats_fetch(hpac_stats_t* stats);

/* ---- K-Means Lloyd loop (bench/kmeans.hpp:62-144) ---------------------- */
/* Sum-reduction hook for the per-iteration centroid partials: a packed
   device buffer [k*dims sum changes | k count changes | 1 changed] (doubles;
   the iteration's moves: +x into a point's new cluster, -x out of its old
   one). Multi-GPU callers all-reduce it across ranks (e.g. ncclAllReduce /
   torch all_reduce over NCCL); NULL = single device. The hook returns 0 on
   success; any other value aborts the run with HPAC_ERR_CUDA (a failed
   all-reduce would otherwise leave each rank on its local partials). */
typedef int (*hpac_allreduce_fn)(double* buf, int64_t count, void* user, void* stream);

typedef struct hpac_kmeans_problem {
  int64_t n_points;     /* points in this shard */
  int32_t dims;
  int32_t k;
  const double* points; /* device, n*dims (AoS) */
  double* centroids;    /* device, k*dims; in: initial centroids when
                           HPAC_KMEANS_CENTROIDS_GIVEN, else Forgy init from
                           the first k points (kmeans.hpp:66-71); out: final */
  int32_t* assignments; /* device, n labels (out) */
  int32_t max_iters;
  int32_t flags;        /* HPAC_REGION_KMEANS_FAST_MATH | HPAC_KMEANS_CENTROIDS_GIVEN |
                           HPAC_KMEANS_HOST_LOOP */
  uint64_t perfo_seed_base; /* RANDOM perforation: seed of iteration i = base + i */
  hpac_allreduce_fn allreduce;
  void* allreduce_user;
  double* reduce_buf;   /* optional device buffer of k*dims + k + 1 doubles */
} hpac_kmeans_problem_t;

#define HPAC_KMEANS_CENTROIDS_GIVEN 8
/* Drive the loop from the host, one synchronised iteration at a time. By
   default (no all-reduce hook) the whole loop is ONE CUDA graph launch: a
   conditional WHILE node whose body is one iteration, with convergence
   decided on the device (no host round trip per iteration). */
#define HPAC_KMEANS_HOST_LOOP 16

typedef struct hpac_kmeans_result {
  int32_t iterations;  /* region launches executed */
  int32_t converged;   /* stopped because no label changed */
  hpac_stats_t stats;  /* summed over launches */
  double region_ms;    /* device time in the distance region kernels */
  double update_ms;    /* device time in the centroid update kernels */
  int32_t graph;       /* 1: the iterations ran as one CUDA graph launch */
} hpac_kmeans_result_t;

int hpac_kmeans_run(const hpac_grid_t* grid, const hpac_kmeans_problem_t* problem,
                    const hpac_spec_t* spec, void* stream, hpac_kmeans_result_t* result,
                    char* err, size_t errlen);

/* Native NCCL all-reduce usable as hpac_kmeans_problem_t.allreduce:
   `user` = the caller's ncclComm_t; sums the packed buffer in place on the
   given stream. NCCL is loaded at run time (libnccl.so.2); 0 = unavailable.
   hpac_nccl_allreduce returns HPAC_OK, HPAC_ERR_UNSUPPORTED (no NCCL / no
   communicator) or HPAC_ERR_CUDA (ncclAllReduce failed);
   hpac_nccl_check polls the communicator's asynchronous error state. */
int hpac_nccl_available(void);
int hpac_nccl_allreduce(double* buf, int64_t count, void* user, void* stream);
int hpac_nccl_check(void* comm);
/* Multi-process communicator for the hook (one process per GPU): rank 0
   writes a 128-byte NCCL unique id, the caller broadcasts it, every rank
   joins (ncclGetUniqueId / ncclCommInitRank). */
int hpac_nccl_unique_id(uint8_t* id128);
int hpac_nccl_comm_init_rank(int nranks, const uint8_t* id128, int rank, void** comm);
/* ncclCommInitAll over `ndev` local devices (one process owning them all);
   comms receives ndev ncclComm_t handles. */
int hpac_nccl_comm_init_all(int ndev, const int* devlist, void** comms);
int hpac_nccl_comm_destroy(void* comm);

/* ---- host generators (same libstdc++ distributions as the reference) --- */
int hpac_make_bs_portfolio(int64_t n, uint64_t seed, int32_t base_block, double jitter,
                           double* out /* n*5 */);
int hpac_make_binomial_portfolio(int64_t n, uint64_t seed, double jitter,
                                 double* out /* n*5 */);
int hpac_make_blobs(int64_t n, int32_t dims, int32_t k, uint64_t seed, double separation,
                    double* out /* n*dims */);

/* LavaMD inputs (extension; Rodinia lavaMD init restated): per particle
   rv = (v, x, y, z) and qv, each value (splitmix64(seed ^ (5*i + c)) % 10 + 1) / 10. */
int hpac_make_lavamd(int32_t boxes1d, int32_t particles, uint64_t seed, double* rv /* P*4 */,
                     double* qv /* P */);

/* ---- quality metrics (metrics.hpp:17-45); device buffers --------------- */
int hpac_mape(const double* accurate, const double* approximate, int64_t n, void* stream,
              double* result);
int hpac_mcr(const int32_t* accurate, const int32_t* approximate, int64_t n, void* stream,
             double* result);

/* ---- roofline support ------------------------------------------------- */
/* Measured FP64 (DFMA) throughput of this device in TFLOP/s: MEASURED_PEAKS.json
   carries HBM and bf16 peaks only, and the regions here compute in FP64, so
   the FP64 roofline denominators are measured in-run by these probes. */
int hpac_probe_fp64_peak(double* tflops);
/* FP64 tensor-op (DMMA m8n8k4) peak, TFLOP/s: the K-Means DMMA filter's roofline. */
int hpac_probe_dmma_peak(double* tflops);

/* ---- diagnostics ------------------------------------------------------ */
/* Evaluate one of the accurate-path math functions element-wise on device
   buffers (test support for csrc/fastmath.cuh; no reference counterpart).
   The BS kinds read AoS option records (5 doubles per element; n records)
   and write NaN where black_scholes_call would throw. */
enum {
  HPAC_FM_EXP = 0, HPAC_FM_LOG = 1, HPAC_FM_ERFC = 2, HPAC_FM_BS = 3,
  HPAC_FM_LIBDEVICE_EXP = 4, HPAC_FM_LIBDEVICE_LOG = 5, HPAC_FM_LIBDEVICE_ERFC = 6,
  HPAC_FM_LIBDEVICE_BS = 7
};
int hpac_fm_eval(int32_t kind, const double* x, double* y, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HPAC_OFFLOAD_H */
