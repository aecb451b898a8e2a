// engine_thread.cu — the approximate-region engine for the per-thread work
// mapping (WorkMapping::kPerThread, grid.hpp:14), i.e. run_region
// (engine.hpp:132-402) for regions whose threads own distinct work items.
//
// Mapping onto the hardware: one CTA = one logical team; one CUDA thread =
// one logical thread; a logical warp of `ws` lanes is a lane segment of a
// hardware warp when ws divides 32 (votes = __ballot_sync + __popc on the
// segment, iACT writer = shuffle butterfly), otherwise a shared-memory
// group (generic path). Per-thread technique state lives in registers
// (TAF window as a shift register for h <= 8, perforation counters) and
// per-warp iACT tables live in shared memory. The grid-stride schedule is
// the reference's: item = tid + step * G with G = num_teams * tpt, so each
// thread's decision stream is identical to the reference's.
#include <cuda_runtime.h>

#include <cstdio>

#include "apps.cuh"
#include "engine.h"
#include "hpac_device.cuh"

namespace hpac {

constexpr int kTechNone = 3;

namespace {

// Triple-buffered shared counters: one __syncthreads per use.
struct CtlLayout {
  // ints
  static constexpr int kTeamYes = 0;   // [3]
  static constexpr int kTeamAct = 3;   // [3]
  static constexpr int kBarMax = 6;    // [3] barrier-divergence max arrivals
  static constexpr int kBarMiss = 9;   // [3]
  static constexpr int kGeneric = 16;  // generic-ws per-logical-warp words start here
};

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v, unsigned mask) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

}  // namespace

// TAF window in registers for single-output apps (h <= 8); multi-output
// windows live in a shared ring [dim][slot][thread] so they hold no
// registers across the accurate path (LavaMD's pair loop)
int engine_thread_max_out(int app);
static inline bool taf_window_in_registers(const EngineParams& p) {
  return p.taf_h <= 8 && engine_thread_max_out(p.region.app) == 1;
}

// i-th box of the tiled order: tile columns of T x T boxes (x fastest, then
// y), z-plane by z-plane inside a column; b1 % T == 0
__device__ __forceinline__ int lava_tile_order(int i, int b1, int T) {
  const int col = T * T * b1;
  const int tile = i / col, r = i - tile * col;
  const int z = r / (T * T), rr = r - z * T * T;
  const int nt = b1 / T;
  const int x = (tile % nt) * T + rr % T, y = (tile / nt) * T + rr / T;
  return x + b1 * (y + b1 * z);
}

template <class App, int TECH, int HREG, int MAXT>
__global__ void __launch_bounds__(MAXT, MAXT > 256 ? 1
                                       : (App::min_blocks_256(TECH) > 0 ? App::min_blocks_256(TECH)
                                                                         : App::MIN_BLOCKS_256))
    engine_thread_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int IN_MAX = App::IN_MAX;
  constexpr int OUT_MAX = App::OUT_MAX;

  const int local = threadIdx.x;
  // LavaMD: boxes in T x T x all-z tile columns (z-planes of a tile in
  // order) so a box's 27-neighbourhood is still in L2 from the previous plane;
  // teams are independent, so the processing order changes nothing else
  const int team = p.box_tile > 0 ? lava_tile_order((int)blockIdx.x, p.region.lavamd_boxes1d, p.box_tile)
                                  : p.team_begin + (int)blockIdx.x;
  const int64_t tid = (int64_t)team * p.tpt + local;
  const int64_t owner = p.per_team ? (int64_t)team : tid;  // machine.hpp:77-80
  const int ws = p.ws;
  const int lane = local % ws;   // logical lane
  const int wloc = local / ws;   // logical warp within the team
  const int hw_lane = local & 31;
  const int hw_warp = local >> 5;
  const int hw_count = min(32, p.tpt - hw_warp * 32);
  const unsigned hw_mask = hw_count == 32 ? 0xffffffffu : ((1u << hw_count) - 1u);
  const bool fast = p.fast_ws != 0;
  const int seg_base = hw_lane - lane;  // fast path only
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << seg_base);
  int* ctl = reinterpret_cast<int*>(smem + p.smem_ctl_off);
  int* gw = ctl + CtlLayout::kGeneric;  // generic-ws words: [wpt][4] + tables [T][3]
  for (int i = local; i < p.ctl_ints; i += blockDim.x) ctl[i] = 0;
  App::init(p, smem + p.smem_scratch_off);
  __syncthreads();

  // ---- TAF state (TafState, taf.hpp:59-163) -------------------------------
  int taf_mode = kTafFilling, taf_rem = 0, taf_count = 0, taf_head = 0;
  // TAF window: registers [slot][dim] oldest first for single-output apps
  // (REGWIN), else a shared ring [dim][slot][thread] of compile-time length
  // HREG (HREG > 0) or of runtime length p.taf_h (HREG == 0)
  constexpr bool REGWIN = HREG > 0 && OUT_MAX == 1;
  constexpr int HW = HREG > 0 ? HREG : 1;
  double win[REGWIN ? HW : 1][REGWIN ? OUT_MAX : 1];
  const double taf_t2 = p.taf_thr * p.taf_thr;
  const double taf_t_lo = taf_t2 * (1.0 - 1e-9) - 1e-27, taf_t_hi = taf_t2 * (1.0 + 1e-9) + 1e-27;
  double last[OUT_MAX];
#pragma unroll
  for (int d = 0; d < OUT_MAX; ++d) last[d] = 0.0;
#pragma unroll
  for (int i = 0; i < (REGWIN ? HW : 1); ++i)
#pragma unroll
    for (int d = 0; d < (REGWIN ? OUT_MAX : 1); ++d) win[i][d] = 0.0;
  double* ring = smem + p.smem_taf_off;  // [d][slot][tpt] (smem variant)

  // ---- iACT per-table bookkeeping (MemoTable, iact.hpp:58-145) -----------
  const int tpw = TECH == HPAC_TECH_IACT ? p.tpw : 1;
  const int group = ws / tpw;                       // lanes sharing one table
  const int T = p.wpt * tpw;                        // tables in this team
  const int tab = wloc * tpw + lane / group;        // this lane's table
  const int D = p.in_dims + p.out_dims;
  double* tabs = smem + p.smem_tab_off;             // [(slot*D + c) * T + tab]
  int rr = 0, occ = 0;

  // ---- perforation counters (engine.hpp:70-71) -----------------------------
  int64_t pcount = 0, hcount = 0;
  const uint64_t perfo_seed = p.seed_ptr ? (uint64_t)*p.seed_ptr : p.perfo_seed;
  int64_t trip = 0;
  if (TECH == HPAC_TECH_PERFO &&
      (p.perfo_kind == HPAC_PERFO_INI || p.perfo_kind == HPAC_PERFO_FINI))
    trip = trip_count(owner, p.stride, p.n, p.steps);

  // ---- stats ---------------------------------------------------------------
  unsigned long long s_total = 0, s_approx = 0, s_warp = 0, s_div = 0;
  bool touched = false;
  bool app_error = false;
  int round_ctr = 0;  // global round counter for triple buffers

  for (int64_t step = 0; step < p.steps; ++step) {
    const int64_t idx = owner + step * p.stride;
    const bool active = idx < p.n;
    int enc = 1;
    if (p.has_enc && active) enc = App::encounters(p, idx);
    int rounds = 1;
    if (p.has_enc) {
      // team max of encounters (engine.hpp:194-215); block-uniform
      __shared__ int s_rounds[2];
      if (local == 0) s_rounds[step & 1] = 0;
      __syncthreads();
      if (active) atomicMax(&s_rounds[step & 1], enc);
      __syncthreads();
      rounds = s_rounds[step & 1];
    }
    int arrivals = 0;
    uint8_t pbits = 0;

    for (int round = 0; round < rounds; ++round, ++round_ctr) {
      const int buf = round_ctr % 3;
      const bool in_round = active && round < enc;

      // ---- predicate phase (engine.hpp:221-251) ----------------------------
      double in[IN_MAX];
      bool loaded = false;
      bool pred = false;
      int hit = -1, near = -1;
      double min_d = dinf();
      if (in_round) {
        if (TECH == HPAC_TECH_TAF) {
          pred = taf_mode == kTafPredicting;
        } else if (TECH == HPAC_TECH_IACT) {
          App::load(p, idx, in);
          loaded = true;
          // MemoTable::lookup / min_distance / nearest_slot in one scan
          double hit_d = 0.0, near_d = dinf();
          for (int s = 0; s < occ; ++s) {
            double ssq = 0.0;
#pragma unroll
            for (int c = 0; c < IN_MAX; ++c)
              if (c < p.in_dims) {
                double df = __dsub_rn(tabs[(s * D + c) * T + tab], in[c]);
                ssq = __dadd_rn(ssq, __dmul_rn(df, df));
              }
            double dd = __dsqrt_rn(ssq);
            if (dd <= p.iact_thr && (hit < 0 || dd < hit_d)) {
              hit = s;
              hit_d = dd;
            }
            if (dd < near_d) {
              near_d = dd;
              near = s;
            }
          }
          min_d = near_d;
          pred = hit >= 0;
        } else if (TECH == HPAC_TECH_PERFO) {
          const bool herded = p.perfo_kind == HPAC_PERFO_HERDED_SMALL ||
                              p.perfo_kind == HPAC_PERFO_HERDED_LARGE;
          pred = perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, perfo_seed,
                                   herded ? hcount : pcount, trip, owner);
        }
      }

      // ---- decision hierarchy (hierarchy.hpp:33-70, engine.hpp:257-298) ----
      bool approx = pred;
      bool team_any = true;
      if (TECH != kTechNone && p.voting) {
        if (p.level == HPAC_LEVEL_TEAM) {
          int* yes = ctl + CtlLayout::kTeamYes;
          int* act = ctl + CtlLayout::kTeamAct;
          if (local == 0) {
            yes[(buf + 1) % 3] = 0;
            act[(buf + 1) % 3] = 0;
          }
          unsigned bv = __ballot_sync(hw_mask, in_round && pred);
          unsigned ba = __ballot_sync(hw_mask, in_round);
          if (hw_lane == 0 && ba) {
            atomicAdd(&yes[buf], __popc(bv));
            atomicAdd(&act[buf], __popc(ba));
          }
          __syncthreads();
          int ty = yes[buf], ta = act[buf];
          team_any = ta > 0;
          approx = 2 * ty > ta;  // majority_decision, hierarchy.hpp:33-35
          if (active && team_any) arrivals += 1;  // the vote's framework barrier
        } else if (fast) {
          unsigned bv = __ballot_sync(hw_mask, in_round && pred) & seg_mask;
          unsigned ba = __ballot_sync(hw_mask, in_round) & seg_mask;
          approx = 2 * __popc(bv) > __popc(ba);
        } else {
          int* w = gw + wloc * 4;
          __syncthreads();
          if (lane == 0) {
            w[0] = 0;
            w[1] = 0;
          }
          __syncthreads();
          if (in_round) {
            atomicAdd(&w[1], 1);
            if (pred) atomicAdd(&w[0], 1);
          }
          __syncthreads();
          approx = 2 * w[0] > w[1];
        }
      }

      // ---- team staging outside the region (staged apps: LavaMD). Decisions
      // come first: they never read the staged data (TAF/perforation), and a
      // round in which no lane of the team evaluates stages nothing.
      if (p.staged)
        App::round_begin(p, idx, round, smem + p.smem_scratch_off, active, in_round && !approx);

      // ---- warp-cooperative evaluation (AppKmeans DMMA): the hardware warp
      // evaluates its lanes' items together, converged, before the per-lane
      // bookkeeping below consumes the results
      double wout = 0.0;
      if constexpr (App::WARP_EVAL) {  // launched only with p.warp_eval
        bool want = in_round && !approx;
        // iACT forced approximation with an empty table falls back (below)
        if (TECH == HPAC_TECH_IACT && in_round && approx && hit < 0 && occ <= 0) want = true;
        if (__any_sync(0xffffffffu, want))
          wout = App::warp_eval(p, idx, want, smem + p.smem_scratch_off, hw_lane);
      }

      // ---- lane execution (engine.hpp:303-347) -----------------------------
      double out[OUT_MAX];
#pragma unroll
      for (int d = 0; d < OUT_MAX; ++d) out[d] = 0.0;
      bool cand = false;
      if (in_round) {
        if (approx) {
          if (TECH == HPAC_TECH_TAF) {
            // TafState::emit_approx, taf.hpp:114-117
#pragma unroll
            for (int d = 0; d < OUT_MAX; ++d) out[d] = last[d];
            if (taf_mode == kTafPredicting && --taf_rem == 0) {
              taf_count = 0;
              taf_head = 0;
              taf_mode = kTafFilling;
            }
            App::store(p, idx, out, local);
          } else if (TECH == HPAC_TECH_IACT) {
            int slot = hit >= 0 ? hit : (occ > 0 ? near : -1);
            if (slot >= 0) {
#pragma unroll
              for (int d = 0; d < OUT_MAX; ++d)
                if (d < p.out_dims) out[d] = tabs[(slot * D + p.in_dims + d) * T + tab];
              App::store(p, idx, out, local);
            } else {
              approx = false;  // empty table: accurate fallback (engine.hpp:327-331)
            }
          }
          // perforation: output untouched
        }
        if (!approx) {
          if constexpr (App::WARP_EVAL) {
            out[0] = wout;
          } else {
            if (!loaded) App::load(p, idx, in);
            if (!App::eval(p, idx, in, out, smem + p.smem_scratch_off, local, round)) app_error = true;
          }
          if (p.barrier_eval) arrivals += 1;
          App::store(p, idx, out, local);
          if (TECH == HPAC_TECH_TAF) {
            // TafState::observe_accurate, taf.hpp:94-108
            bool full;
            if constexpr (REGWIN) {
#pragma unroll
              for (int i = 0; i + 1 < HW; ++i) win[i][0] = win[i + 1][0];
              win[HW - 1][0] = out[0];
              if (taf_count < HREG) ++taf_count;
              full = taf_count == HREG;
            } else {
              const int h = HREG > 0 ? HREG : p.taf_h;
              int slot;
              if (taf_count < h) {
                slot = taf_head + taf_count;
                if (slot >= h) slot -= h;
                ++taf_count;
              } else {
                slot = taf_head;
                taf_head = taf_head + 1 == h ? 0 : taf_head + 1;
              }
#pragma unroll
              for (int d = 0; d < OUT_MAX; ++d)
                if (d < p.out_dims) ring[(d * h + slot) * p.tpt + local] = out[d];
              full = taf_count == h;
            }
#pragma unroll
            for (int d = 0; d < OUT_MAX; ++d) last[d] = out[d];
            bool check = (taf_mode == kTafFilling && full) || taf_mode == kTafChecking;
            if (taf_mode == kTafPredicting) {
              if (--taf_rem == 0) {
                taf_count = 0;
                taf_head = 0;
                taf_mode = kTafFilling;
              }
            } else if (check) {
              // every output dimension must pass (taf.hpp:134-140)
              bool pass = true;
              if constexpr (REGWIN) {
                double col[HW];
#pragma unroll
                for (int i = 0; i < HW; ++i) col[i] = win[i][0];
                pass = taf_window_passes<HW>(col, p.taf_thr);
              } else if constexpr (HREG > 0) {
#pragma unroll
                for (int d = 0; d < OUT_MAX; ++d)
                  if (d < p.out_dims && pass)
                    pass = taf_ring_passes_fixed<HW>(ring + d * HW * p.tpt + local, p.tpt, taf_head,
                                                     p.taf_thr, taf_t_lo, taf_t_hi);
              } else {
                for (int d = 0; d < p.out_dims && pass; ++d)
                  pass = taf_ring_passes(ring + d * p.taf_h * p.tpt + local, p.tpt, p.taf_h,
                                         taf_head, taf_count, p.taf_thr);
              }
              if (pass) {
                taf_rem = p.taf_p;
                taf_mode = kTafPredicting;
              } else {
                taf_mode = kTafChecking;
              }
            }
          }
          if (TECH == HPAC_TECH_IACT && hit < 0) cand = true;
        }
        s_total += 1;
        if (approx) {
          s_approx += 1;
          if (round < 8) pbits |= (uint8_t)(1u << round);
        }
      }

      // ---- iACT write phase (engine.hpp:351-366, iact.hpp:166-180) ----------
      if (TECH == HPAC_TECH_IACT) {
        double bd = cand ? min_d : -1.0;
        int bl = lane;
        if (fast) {
          for (int off = group >> 1; off > 0; off >>= 1) {
            double od = __shfl_xor_sync(hw_mask, bd, off);
            int ol = __shfl_xor_sync(hw_mask, bl, off);
            if (writer_better(od, ol, bd, bl)) {
              bd = od;
              bl = ol;
            }
          }
          __syncwarp(hw_mask);
        } else {
          unsigned long long* tk = reinterpret_cast<unsigned long long*>(gw + p.wpt * 4);
          int* tl = gw + p.wpt * 4 + 2 * T;
          __syncthreads();
          if (lane % group == 0) {
            tk[tab] = 0ull;
            tl[tab] = 1 << 30;
          }
          __syncthreads();
          // candidate keys: +1 so that a real distance 0 beats "no candidate"
          unsigned long long key =
              cand ? (unsigned long long)__double_as_longlong(min_d) + 1ull : 0ull;
          if (cand) atomicMax(&tk[tab], key);
          __syncthreads();
          if (cand && key == tk[tab]) atomicMin(&tl[tab], lane);
          __syncthreads();
          bd = tk[tab] ? 0.0 : -1.0;
          bl = tl[tab];
        }
        if (bd >= 0.0) {
          if (lane == bl) {
            // MemoTable::insert at the round-robin cursor, iact.hpp:124-135
#pragma unroll
            for (int c = 0; c < IN_MAX; ++c)
              if (c < p.in_dims) tabs[(rr * D + c) * T + tab] = in[c];
#pragma unroll
            for (int d = 0; d < OUT_MAX; ++d)
              if (d < p.out_dims) tabs[(rr * D + p.in_dims + d) * T + tab] = out[d];
          }
          rr = rr + 1 == p.tsize ? 0 : rr + 1;
          occ = occ + 1 < p.tsize ? occ + 1 : p.tsize;
        }
        if (fast)
          __syncwarp(hw_mask);
        else
          __syncthreads();
      }

      // ---- perforation counters + warp stats (engine.hpp:368-378) -----------
      bool any_lw, mixed;
      if (fast) {
        unsigned ba = __ballot_sync(hw_mask, in_round) & seg_mask;
        unsigned bx = __ballot_sync(hw_mask, in_round && approx) & seg_mask;
        any_lw = ba != 0;
        mixed = bx != 0 && bx != ba;
      } else {
        int* w = gw + wloc * 4;
        __syncthreads();
        if (lane == 0) {
          w[2] = 0;
          w[3] = 0;
        }
        __syncthreads();
        if (in_round) atomicAdd(&w[approx ? 3 : 2], 1);
        __syncthreads();
        any_lw = (w[2] + w[3]) > 0;
        mixed = w[2] > 0 && w[3] > 0;
      }
      if (TECH == HPAC_TECH_PERFO) {
        if (in_round) pcount += 1;
        if (any_lw) hcount += 1;
      }
      if (lane == 0 && any_lw) {
        touched = true;
        s_warp += 1;
        if (mixed) s_div += 1;
      }
      (void)team_any;
    }

    if (p.paths && active && (!p.per_team || local == 0)) p.paths[idx] = pbits;

    // ---- TeamState::end_step barrier check (machine.hpp:53-61) -------------
    if (p.barrier_eval) {
      const int b = step % 3;
      int* bmax = ctl + CtlLayout::kBarMax;
      int* bmiss = ctl + CtlLayout::kBarMiss;
      if (local == 0) {
        bmax[(b + 1) % 3] = 0;
        bmiss[(b + 1) % 3] = 0;
      }
      __syncthreads();
      if (active) atomicMax(&bmax[b], arrivals);
      __syncthreads();
      if (active && arrivals < bmax[b]) atomicAdd(&bmiss[b], 1);
      __syncthreads();
      if (local == 0 && bmiss[b] > 0) {
        unsigned long long key = ((unsigned long long)step << 32) | (unsigned)team;
        unsigned long long prev = atomicMin(&p.counters[kCntBarrierKey], key);
        if (key < prev) atomicExch(&p.counters[kCntBarrierMissing], (unsigned long long)bmiss[b]);
      }
    }
  }

  // ---- reduce stats: one atomic per hardware warp per counter -----------------
  s_total = warp_sum_u64(s_total, hw_mask);
  s_approx = warp_sum_u64(s_approx, hw_mask);
  s_warp = warp_sum_u64(s_warp, hw_mask);
  s_div = warp_sum_u64(s_div, hw_mask);
  unsigned long long s_res = warp_sum_u64((lane == 0 && touched) ? 1ull : 0ull, hw_mask);
  unsigned any_err = __ballot_sync(hw_mask, app_error);
  if (hw_lane == 0) {
    if (s_total) atomicAdd(&p.counters[kCntTotal], s_total);
    if (s_approx) atomicAdd(&p.counters[kCntApprox], s_approx);
    if (s_div) atomicAdd(&p.counters[kCntDivergent], s_div);
    if (s_warp) atomicAdd(&p.counters[kCntWarpSteps], s_warp);
    if (s_res) atomicAdd(&p.counters[kCntResidentWarps], s_res);
    if (any_err) atomicAdd(&p.counters[kCntAppError], 1ull);
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------
template <class App, int TECH>
static cudaError_t launch_tech(const EngineParams& p, int nblocks, size_t smem,
                               cudaStream_t st) {
  // TAF: register shift-register window for single-output regions, h <= 8
  // compile-time window length for h <= 8 (registers for single-output
  // apps, a fixed-length shared ring otherwise); h > 8: runtime-length ring
  int hreg = 0;
  if (TECH == HPAC_TECH_TAF && p.taf_h <= 8) hreg = p.taf_h;
#define HPAC_LAUNCH(H)                                                                  \
  {                                                                                     \
    auto k = p.tpt <= 256 ? engine_thread_kernel<App, TECH, H, 256>                     \
                          : engine_thread_kernel<App, TECH, H, 1024>;                   \
    if (smem > 48 * 1024) {                                                             \
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)smem);                                  \
      if (e != cudaSuccess) return e;                                                   \
    }                                                                                   \
    k<<<nblocks, p.tpt, smem, st>>>(p);                                                 \
    return cudaGetLastError();                                                          \
  }
  if constexpr (TECH == HPAC_TECH_TAF) {
    switch (hreg) {
      case 1: HPAC_LAUNCH(1);
      case 2: HPAC_LAUNCH(2);
      case 3: HPAC_LAUNCH(3);
      case 4: HPAC_LAUNCH(4);
      case 5: HPAC_LAUNCH(5);
      case 6: HPAC_LAUNCH(6);
      case 7: HPAC_LAUNCH(7);
      case 8: HPAC_LAUNCH(8);
      default: HPAC_LAUNCH(0);
    }
  }
  HPAC_LAUNCH(0);
#undef HPAC_LAUNCH
}

template <class App>
static cudaError_t launch_app(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st) {
  // techniques the runtime rejects for an app are not instantiated
  switch (p.tech) {
    case HPAC_TECH_TAF:
      if constexpr (App::HAS_TAF) return launch_tech<App, HPAC_TECH_TAF>(p, nblocks, smem, st);
      return cudaErrorInvalidValue;
    case HPAC_TECH_IACT:
      if constexpr (App::HAS_IACT) return launch_tech<App, HPAC_TECH_IACT>(p, nblocks, smem, st);
      return cudaErrorInvalidValue;
    case HPAC_TECH_PERFO: return launch_tech<App, HPAC_TECH_PERFO>(p, nblocks, smem, st);
    default: return launch_tech<App, kTechNone>(p, nblocks, smem, st);
  }
}

// Dynamic shared memory for the per-thread engine; fills the offsets.
size_t engine_thread_smem(EngineParams& p) {
  size_t off = 0;  // in doubles
  p.smem_taf_off = 0;
  p.smem_last_off = 0;
  if (p.tech == HPAC_TECH_TAF && !taf_window_in_registers(p)) {
    p.smem_taf_off = (int)off;
    off += (size_t)p.out_dims * p.taf_h * p.tpt;
  }
  p.smem_tab_off = (int)off;
  if (p.tech == HPAC_TECH_IACT)
    off += (size_t)p.tsize * (p.in_dims + p.out_dims) * p.wpt * p.tpw;
  off = (off + 1) & ~(size_t)1;  // 16-byte aligned scratch (vector staging)
  p.smem_scratch_off = (int)off;
  if (p.region.app == HPAC_APP_KMEANS && !p.warp_eval)  // centroids + squared norms
    off += (size_t)p.region.kmeans_k * p.region.kmeans_dims + p.region.kmeans_k + 1;
  if (p.region.app == HPAC_APP_LAVAMD) off += (size_t)p.region.lavamd_particles * 5 + 64;  // + exp table
  p.smem_ctl_off = (int)off;
  // control ints: 16 fixed + generic-ws words (4 per logical warp + 3 per table)
  size_t ctl_ints = 16 + 4 * (size_t)p.wpt + 3 * (size_t)p.wpt * (p.tpw > 0 ? p.tpw : 1) + 4;
  p.ctl_ints = (int)ctl_ints;
  off += (ctl_ints + 1) / 2 + 1;
  return off * sizeof(double);
}

int engine_thread_max_in(int app) {
  switch (app) {
    case HPAC_APP_TABLE: return AppTable::IN_MAX;
    case HPAC_APP_SYNTHETIC: return AppSynthetic::IN_MAX;
    case HPAC_APP_BLACKSCHOLES: return AppBlackScholes::IN_MAX;
    case HPAC_APP_KMEANS: return AppKmeans::IN_MAX;
    case HPAC_APP_LAVAMD: return 0;
  }
  return 0;
}
int engine_thread_max_out(int app) {
  switch (app) {
    case HPAC_APP_TABLE: return AppTable::OUT_MAX;
    case HPAC_APP_SYNTHETIC: return AppSynthetic::OUT_MAX;
    case HPAC_APP_BLACKSCHOLES: return AppBlackScholes::OUT_MAX;
    case HPAC_APP_KMEANS: return AppKmeans::OUT_MAX;
    case HPAC_APP_LAVAMD: return AppLavaMD::OUT_MAX;
  }
  return 0;
}

}  // namespace hpac
cudaMemPool_t host_entry_pool();  // runtime.cu: the library's retained pool
namespace hpac {

size_t kmeans_aux_bytes(int k) { return ((size_t)k * 33 + 1) * sizeof(double); }

// Per-launch K-Means DMMA operand block (AppKmeans::warp_eval): B fragments
// [(j*4 + m)*32 + L] (double2) = c[8j + L/4][8m + 2(L%4) .. +1], then the
// squared norms (dimension-order fma, as AppKmeans::init) and their maximum.
__global__ void kmeans_dmma_aux_kernel(const double* __restrict__ cent, int k, double* aux) {
  double2* bf = reinterpret_cast<double2*>(aux);
  for (int e = threadIdx.x; e < k * 16; e += blockDim.x) {
    const int L = e & 31, m = (e >> 5) & 3, j = e >> 7;
    const double* src = cent + (8 * j + (L >> 2)) * 32 + 8 * m + 2 * (L & 3);
    bf[e] = make_double2(src[0], src[1]);
  }
  double* cc = aux + k * 32;
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double s = 0.0;
    for (int d = 0; d < 32; ++d) s = fma(cent[c * 32 + d], cent[c * 32 + d], s);
    cc[c] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // max norm; NaN if any centroid is non-finite (warp_eval then certifies
    // nothing and every point takes the reference path)
    double mx = 0.0;
    bool finite = true;
    for (int c = 0; c < k; ++c) {
      finite = finite && isfinite(cc[c]);
      mx = fmax(mx, cc[c]);
    }
    cc[k] = finite ? mx : __longlong_as_double(0x7ff8000000000000ll);
  }
}

cudaError_t engine_thread_launch(const EngineParams& p, int nblocks, size_t smem,
                                 cudaStream_t st) {
  if (p.region.app == HPAC_APP_KMEANS && p.warp_eval) {
    const int k = p.region.kmeans_k;
    double* aux = const_cast<double*>(p.km_aux);  // preallocated (captured loop)
    cudaError_t e = cudaSuccess;
    // per-launch block from the retained pool (no physical re-mapping inside
    // the timed stream work); a captured loop passes its own
    cudaMemPool_t pool = p.km_aux ? nullptr : host_entry_pool();
    if (!aux && (e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&aux),
                                                    kmeans_aux_bytes(k), pool, st)
                          : cudaMallocAsync(&aux, kmeans_aux_bytes(k), st)) != cudaSuccess)
      return e;
    kmeans_dmma_aux_kernel<<<1, 256, 0, st>>>(p.region.centroids, k, aux);
    EngineParams q = p;
    q.km_aux = aux;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = launch_app<AppKmeansDmma>(q, nblocks, smem, st);
    if (p.km_aux) return e;
    cudaError_t f = cudaFreeAsync(aux, st);
    return e != cudaSuccess ? e : f;
  }
  switch (p.region.app) {
    case HPAC_APP_TABLE: return launch_app<AppTable>(p, nblocks, smem, st);
    case HPAC_APP_SYNTHETIC: return launch_app<AppSynthetic>(p, nblocks, smem, st);
    case HPAC_APP_BLACKSCHOLES: return launch_app<AppBlackScholes>(p, nblocks, smem, st);
    case HPAC_APP_KMEANS: return launch_app<AppKmeans>(p, nblocks, smem, st);
    case HPAC_APP_LAVAMD: return launch_app<AppLavaMD>(p, nblocks, smem, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hpac
