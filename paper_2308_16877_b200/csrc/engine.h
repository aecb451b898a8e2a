// engine.h — launch parameters shared by the host runtime and the kernels.
#pragma once

#include <cstdint>

#include "hpac_offload.h"

namespace hpac {

// Device counters (one block of u64 per launch).
enum Counter : int {
  kCntTotal = 0,
  kCntApprox = 1,
  kCntDivergent = 2,
  kCntWarpSteps = 3,
  kCntResidentWarps = 4,
  kCntAppError = 5,       // nonzero: an app evaluate raised ConfigError
  kCntBarrierKey = 6,     // min over (step << 32 | team) of barrier divergence; ~0 = none
  kCntBarrierMissing = 7, // missing-thread count of the team that set the key
  kCntLatticeFallback = 8,  // binomial boundary-tracking fallbacks
  kCntLatticeNodes = 9,     // binomial node updates executed
  kNumCounters = 10,
};

struct EngineParams {
  // schedule (machine.hpp:77-84)
  int64_t n;
  int64_t steps;
  int64_t stride;
  int32_t num_teams;
  int32_t tpt;   // threads per team
  int32_t ws;    // logical warp size
  int32_t wpt;   // logical warps per team
  int32_t team_begin;
  int32_t fast_ws;  // ws divides 32 -> logical warps are lane segments of a HW warp
  // technique
  int32_t tech;  // -1 = accurate
  int32_t level;
  int32_t voting;
  int32_t taf_h, taf_p;
  double taf_thr;
  int32_t tsize, tpw;
  double iact_thr;
  int32_t perfo_kind, perfo_mod, perfo_pct;
  uint64_t perfo_seed;
  // region
  hpac_region_t region;
  int32_t in_dims, out_dims;
  int32_t has_enc, barrier_eval, accumulate;
  int32_t per_team;  // lane-level engine under per-team mapping (all lanes share idx)
  int32_t staged;    // app stages shared data per round (AppLavaMD)
  int32_t warp_eval; // app evaluates a hardware warp's items cooperatively (AppKmeans DMMA)
  const double* km_aux;  // AppKmeans warp_eval: DMMA B fragments [k*32], norms [k], max norm
                         // (preallocated by a captured Lloyd loop; else per launch)
  const unsigned long long* seed_ptr;  // device perforation seed (captured loops); null = perfo_seed
  // shared-memory carve-up (doubles unless noted)
  int32_t smem_taf_off;   // TAF ring (smem variant)
  int32_t smem_last_off;  // TAF last (smem variant)
  int32_t smem_tab_off;   // iACT tables
  int32_t smem_scratch_off;  // app scratch (centroids / payload)
  int32_t smem_ctl_off;   // control words (int, counts)
  int32_t ctl_ints;
  int32_t lat_bmax;       // binomial: register block bound
  // Blackscholes iACT engine (engine_bs_iact.cu): lookups decide a chunk of
  // q_steps steps, then the CTA prices the queued misses densely
  int32_t q_steps;
  int32_t box_tile;       // LavaMD: tiled box order (T, 0 = natural order; full grid only)
  double iact_thr2;       // largest ssq with sqrt_rn(ssq) <= iact_thr (exact test, no sqrt)
  // outputs
  uint8_t* paths;
  unsigned long long* counters;
};

}  // namespace hpac
