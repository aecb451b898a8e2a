// engine_stream.cu — the streaming variants of the per-thread engine
// (run_region, engine.hpp:132-402, WorkMapping::kPerThread) for
// single-encounter regions whose accurate path is a pure function of one
// AoS input record: Blackscholes (bench/blackscholes.hpp:72-92).
//
// Same decisions, stats and outputs as engine_thread.cu (and therefore the
// reference); two kernels:
//  * bs_lane_kernel (the default): barrier-free — each thread reads its own
//    record with read-only loads only when it evaluates, votes are warp
//    ballots or one __syncthreads_count per step (team level), 64 registers
//    (32 warps/SM). C1 exact 82 us per 4 M options vs 90 us for the tile
//    kernel on the same math (profiles/r04_bs_lane_ab.txt).
//  * bs_stream_kernel (HPAC_STREAM_TMA=1, A/B tests): the team's input tile of
//    step s+1 (tpt consecutive 40 B records, one contiguous span) is fetched
//    by ONE thread with a 1-D bulk TMA copy (cp.async.bulk ...
//    mbarrier::complete_tx) into a double-buffered shared tile while the team
//    computes step s; a tile is not fetched at all when every active thread
//    of the team is known to take the approximate path at s+1 (TAF regime
//    with >= 2 predictions left, or a perforation skip). The team vote is a
//    __syncthreads_count, the warp vote a segment-masked __ballot_sync.
// Per-thread counters are 32-bit and reduced once per thread at the end.
// Eligibility (runtime.cu): per-thread mapping, no encounters, no barrier in
// evaluate, warp_size | 32, threads_per_team a multiple of 32 and <= 256,
// technique none / TAF (h <= 8) / perforation.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "apps.cuh"
#include "engine.h"
#include "hpac_device.cuh"
#include "tma.cuh"

namespace hpac {

namespace {

constexpr int kStreamMaxT = 256;
constexpr int kTechNoneStream = 3;  // accurate baseline (spec == NULL)
constexpr int kRec = 5;  // doubles per option record

__device__ __forceinline__ unsigned long long warp_sum_u32(unsigned v) {
  unsigned long long s = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

}  // namespace

// One CUDA thread runs PAIR logical threads of the team: local and
// local + tpt/PAIR (both in hardware-aligned 32-lane segments, so warp votes
// stay segment ballots per logical set). Two independent options per thread
// double the FP64 instruction-level parallelism of the accurate path (the
// kernel is latency-bound on DFMA chains at one option per thread) and halve
// the per-option share of the step bookkeeping.
template <int TECH, int LEVEL, int HREG, int PAIR>
__global__ void __launch_bounds__(kStreamMaxT / PAIR, (PAIR == 2 ? 4 : 3))
    bs_stream_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  const int tpt = p.tpt;
  const int half = tpt / PAIR;  // physical threads
  double* tile = smem;                                             // [2][tpt*5]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * tpt * kRec);  // [2]

  const int phys = threadIdx.x;
  const int team = p.team_begin + (int)blockIdx.x;
  const int64_t G = p.stride;
  const int ws = p.ws;
  const int hw_lane = phys & 31;
  const int lane = hw_lane % ws;  // logical lane (half is a multiple of 32)
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << (hw_lane - lane));
  const double* __restrict__ in = p.region.in;
  double* __restrict__ out = p.region.out;
  const int64_t team_base = (int64_t)team * tpt;
  // per-team schedule bounds, once: steps [0, full) see a whole tile, step
  // `full` (if < tsteps) a ragged one, steps >= tsteps nothing
  const int64_t rem0 = p.n - team_base;  // items at or after this team's step-0 base
  const int tsteps = rem0 <= 0 ? 0 : (int)(p.steps < (rem0 - 1) / G + 1 ? p.steps : (rem0 - 1) / G + 1);
  const int full = rem0 < tpt ? 0 : (int)(p.steps < (rem0 - tpt) / G + 1 ? p.steps : (rem0 - tpt) / G + 1);
  const int ragged = tsteps > full ? (int)(rem0 - (int64_t)full * G) : 0;  // count at step `full`
  const int nsteps = (int)p.steps;
  // bulk copies need 16-byte aligned source and size: tpt*40 B per tile is a
  // multiple of 16 when tpt is even (always, tpt % 32 == 0); the ragged last
  // tile of the grid and misaligned buffers fall back to per-thread loads.
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  auto tile_count = [&](int s) -> int { return s < full ? tpt : (s == full ? ragged : 0); };
  auto tile_tma = [&](int s) -> bool { return aligned && s < full; };
  const uint32_t tile_bytes = (uint32_t)(tpt * kRec * 8);

  if (phys == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase0 = 0, phase1 = 0;
  bool loaded_cur = nsteps > 0 && tile_tma(0);
  if (phys == 0 && loaded_cur) {
    mbar_expect_tx(&bar[0], tile_bytes);
    tma_load_1d(tile, in + team_base * kRec, tile_bytes, &bar[0]);
  }
  // thread 0's bookkeeping: a load into buffer b that no consumer waited for
  // is still "outstanding"; it must be retired before the buffer is re-armed
  // (an mbarrier must not see a second arrive while its phase is pending)
  bool issued0 = loaded_cur, issued1 = false;

  // per logical thread k: local = phys + k*half, tid = team_base + local
  constexpr int HW = HREG > 0 ? HREG : 1;
  int taf_mode[PAIR], taf_rem[PAIR], taf_count[PAIR];
  double win[PAIR][HW], last[PAIR];
  int trip[PAIR];
#pragma unroll
  for (int k = 0; k < PAIR; ++k) {
    taf_mode[k] = kTafFilling;
    taf_rem[k] = 0;
    taf_count[k] = 0;
    last[k] = 0.0;
#pragma unroll
    for (int i = 0; i < HW; ++i) win[k][i] = 0.0;
    trip[k] = 0;
    if (TECH == HPAC_TECH_PERFO &&
        (p.perfo_kind == HPAC_PERFO_INI || p.perfo_kind == HPAC_PERFO_FINI))
      trip[k] = (int)trip_count(team_base + phys + k * half, G, p.n, p.steps);
  }

  unsigned c_total = 0, c_approx = 0, c_warp = 0, c_div = 0, c_res = 0;
  bool app_error = false;
  const double* src_step = in + (team_base + phys) * kRec;  // logical 0's record at step s
  double* dst_step = out ? out + team_base + phys : nullptr;
  uint8_t* path_step = p.paths ? p.paths + team_base + phys : nullptr;

  for (int step = 0; step < nsteps; ++step) {
    const int cnt = tile_count(step);
    const int buf = step & 1;
    bool active[PAIR], pred[PAIR], approx[PAIR];
    bool need_next = false;
    const int cnt_next = tile_count(step + 1);
#pragma unroll
    for (int k = 0; k < PAIR; ++k) {
      const int local = phys + k * half;
      const int64_t tid = team_base + local;
      active[k] = local < cnt;  // idx = tid + step*G < n
      // ---- predicate (engine.hpp:221-251); for 1-encounter regions the
      // per-thread and herded perforation counters both equal `step`
      pred[k] = false;
      if (active[k]) {
        if (TECH == HPAC_TECH_TAF) pred[k] = taf_mode[k] == kTafPredicting;
        if (TECH == HPAC_TECH_PERFO)
          pred[k] = perfo_should_skip32(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step,
                                        trip[k], tid);
      }
      // known approximate at step+1 (thread level decisions only depend on
      // the thread's own state; any approximate lane needs no input)
      if (step + 1 < nsteps && local < cnt_next) {
        bool nn = true;
        if (TECH == HPAC_TECH_TAF && LEVEL == HPAC_LEVEL_THREAD)
          nn = !(taf_mode[k] == kTafPredicting && taf_rem[k] >= 2);
        if (TECH == HPAC_TECH_PERFO)
          nn = !perfo_should_skip32(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step + 1,
                                    trip[k], tid);
        need_next = need_next || nn;
      }
      approx[k] = pred[k];
    }

    // ---- team barrier: frees tile[buf^1] (consumed at step-1), team vote,
    // and "does anybody need the next tile" in bar.red ops
    if (TECH != kTechNoneStream && LEVEL == HPAC_LEVEL_TEAM) {
      int yes = 0;
#pragma unroll
      for (int k = 0; k < PAIR; ++k) yes += __syncthreads_count(active[k] && pred[k]);
      const bool ta = 2 * yes > cnt;  // majority_decision over the team's active threads
#pragma unroll
      for (int k = 0; k < PAIR; ++k) approx[k] = ta;
    }
    const int any_next = __syncthreads_or(need_next);
    if (LEVEL == HPAC_LEVEL_WARP && TECH != kTechNoneStream) {
#pragma unroll
      for (int k = 0; k < PAIR; ++k) {
        const unsigned bv = __ballot_sync(0xffffffffu, active[k] && pred[k]) & seg_mask;
        const unsigned ba = __ballot_sync(0xffffffffu, active[k]) & seg_mask;
        approx[k] = 2 * __popc(bv) > __popc(ba);
      }
    }
    bool loaded_next = false;
    if (any_next && tile_tma(step + 1)) {
      loaded_next = true;
      if (phys == 0) {
        const int nb = buf ^ 1;
        if (nb ? issued1 : issued0) mbar_wait(&bar[nb], (nb ? phase1 : phase0) ^ 1);
        mbar_expect_tx(&bar[nb], tile_bytes);
        tma_load_1d(tile + nb * tpt * kRec, in + (team_base + (int64_t)(step + 1) * G) * kRec,
                    tile_bytes, &bar[nb]);
        if (nb)
          issued1 = true;
        else
          issued0 = true;
      }
    }

    // ---- lane execution (engine.hpp:303-347): both logical threads' inputs
    // first, then both evaluations in one straight-line block
    bool ev[PAIR];
    bool any_ev = false;
#pragma unroll
    for (int k = 0; k < PAIR; ++k) {
      ev[k] = active[k] && !approx[k];
      any_ev = any_ev || ev[k];
    }
    double v[PAIR];
#pragma unroll
    for (int k = 0; k < PAIR; ++k) v[k] = 0.0;
    if (any_ev) {
      double rec[PAIR][kRec];
      if (loaded_cur) {
        mbar_wait(&bar[buf], buf ? phase1 : phase0);
#pragma unroll
        for (int k = 0; k < PAIR; ++k) {
          const double* t = tile + buf * tpt * kRec + (phys + k * half) * kRec;
#pragma unroll
          for (int c = 0; c < kRec; ++c) rec[k][c] = t[c];
        }
      } else {
#pragma unroll
        for (int k = 0; k < PAIR; ++k) {
          const double* o = src_step + (int64_t)k * half * kRec;
#pragma unroll
          for (int c = 0; c < kRec; ++c) rec[k][c] = ev[k] ? __ldg(o + c) : 1.0;
        }
      }
      // an approximate or inactive logical thread prices a dummy valid
      // option (1,1,0,0,1) alongside; its result is discarded
#pragma unroll
      for (int k = 0; k < PAIR; ++k)
        if (!ev[k]) {
          rec[k][0] = 1.0;
          rec[k][1] = 1.0;
          rec[k][2] = 0.0;
          rec[k][3] = 0.0;
          rec[k][4] = 1.0;
        }
#pragma unroll
      for (int k = 0; k < PAIR; ++k)
        if (!bs_call(rec[k][0], rec[k][1], rec[k][2], rec[k][3], rec[k][4], v[k]) && ev[k])
          app_error = true;
    }

#pragma unroll
    for (int k = 0; k < PAIR; ++k) {
      if (!active[k]) continue;
      double* o = dst_step ? dst_step + (int64_t)k * half : nullptr;
      if (approx[k]) {
        if (TECH == HPAC_TECH_TAF) {
          // TafState::emit_approx, taf.hpp:114-117
          if (o) __stcs(o, last[k]);
          if (taf_mode[k] == kTafPredicting && --taf_rem[k] == 0) {
            taf_count[k] = 0;
            taf_mode[k] = kTafFilling;
          }
        }
        // perforation: output untouched
      } else {
        if (o) __stcs(o, v[k]);
        if (TECH == HPAC_TECH_TAF) {
          // TafState::observe_accurate, taf.hpp:94-108
#pragma unroll
          for (int i = 0; i + 1 < HW; ++i) win[k][i] = win[k][i + 1];
          win[k][HW - 1] = v[k];
          if (taf_count[k] < HREG) ++taf_count[k];
          last[k] = v[k];
          const bool check = (taf_mode[k] == kTafFilling && taf_count[k] == HREG) ||
                             taf_mode[k] == kTafChecking;
          if (taf_mode[k] == kTafPredicting) {
            if (--taf_rem[k] == 0) {
              taf_count[k] = 0;
              taf_mode[k] = kTafFilling;
            }
          } else if (check) {
            if (taf_window_passes<HW>(win[k], p.taf_thr)) {
              taf_rem[k] = p.taf_p;
              taf_mode[k] = kTafPredicting;
            } else {
              taf_mode[k] = kTafChecking;
            }
          }
        }
      }
      c_total += 1;
      if (approx[k]) c_approx += 1;
      if (path_step) path_step[(int64_t)k * half] = approx[k] ? 1 : 0;
    }
    // every thread observes the completion of a loaded tile it did not read,
    // so the buffer's phase stays in step for the whole team
    if (loaded_cur) {
      if (buf)
        phase1 ^= 1;
      else
        phase0 ^= 1;
    }
    loaded_cur = loaded_next;

    // ---- warp stats (cost.hpp:66-86), per logical set
#pragma unroll
    for (int k = 0; k < PAIR; ++k) {
      const unsigned ba = __ballot_sync(0xffffffffu, active[k]) & seg_mask;
      const unsigned bx = __ballot_sync(0xffffffffu, active[k] && approx[k]) & seg_mask;
      if (lane == 0 && ba) {
        c_res |= 1u << k;
        c_warp += 1;
        if (bx != 0 && bx != ba) c_div += 1;
      }
    }
    src_step += G * kRec;
    if (dst_step) dst_step += G;
    if (path_step) path_step += G;
  }
  // a tile may have been fetched speculatively and then not read by anybody
  // (every lane approximated): thread 0 retires the last copy of each
  // buffer so none is in flight when the CTA exits
  if (phys == 0) {
    if (issued0) mbar_wait(&bar[0], phase0 ^ 1);
    if (issued1) mbar_wait(&bar[1], phase1 ^ 1);
  }

  const unsigned long long s_total = warp_sum_u32(c_total);
  const unsigned long long s_approx = warp_sum_u32(c_approx);
  const unsigned long long s_warp = warp_sum_u32(c_warp);
  const unsigned long long s_div = warp_sum_u32(c_div);
  const unsigned long long s_res = warp_sum_u32(__popc(c_res));
  const unsigned any_err = __ballot_sync(0xffffffffu, app_error);
  if (hw_lane == 0) {
    if (s_total) atomicAdd(&p.counters[kCntTotal], s_total);
    if (s_approx) atomicAdd(&p.counters[kCntApprox], s_approx);
    if (s_div) atomicAdd(&p.counters[kCntDivergent], s_div);
    if (s_warp) atomicAdd(&p.counters[kCntWarpSteps], s_warp);
    if (s_res) atomicAdd(&p.counters[kCntResidentWarps], s_res);
    if (any_err) atomicAdd(&p.counters[kCntAppError], 1ull);
  }
}

// Barrier-free variant (the default): every thread loads its own 40 B
// record with read-only 64-bit loads when it evaluates, and nothing else.
// Same schedule, decisions, stats and outputs as bs_stream_kernel. The
// tile staging above wins nothing once the accurate path is the FP64
// fastmath closed form: a warp's five loads cover 1,280 contiguous bytes, the
// other resident warps hide the HBM latency, and dropping the two barriers,
// the mbarrier waits and the double-buffered tile per step frees the
// registers and issue slots they took. Approximate lanes load nothing (TAF
// predictions, perforation skips), like the tile version's skipped fetches.
// Team votes keep one __syncthreads_count per step.
#ifndef HPAC_LANE_MINB
#define HPAC_LANE_MINB 4  // 256-thread blocks per SM: <= 64 registers
#endif
template <int TECH, int LEVEL, int HREG>
__global__ void __launch_bounds__(kStreamMaxT, HPAC_LANE_MINB) bs_lane_kernel(const EngineParams p) {
  const int tpt = p.tpt;
  const int phys = threadIdx.x;
  const int team = p.team_begin + (int)blockIdx.x;
  const int64_t G = p.stride;
  const int ws = p.ws;
  const int hw_lane = phys & 31;
  const int lane = hw_lane % ws;
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << (hw_lane - lane));
  const int64_t team_base = (int64_t)team * tpt;
  const int64_t tid = team_base + phys;
  const int nsteps = (int)p.steps;
  // this thread's items: idx = tid + s*G < n for s < my_steps
  const int64_t rem = p.n - tid;
  const int my_steps = rem <= 0 ? 0 : (int)(p.steps < (rem - 1) / G + 1 ? p.steps : (rem - 1) / G + 1);
  const int64_t team_rem = p.n - team_base;  // active threads of the team at step s: team_rem - s*G

  constexpr int HW = HREG > 0 ? HREG : 1;
  int taf_mode = kTafFilling, taf_rem = 0, taf_count = 0;
  double win[HW], last = 0.0;
#pragma unroll
  for (int i = 0; i < HW; ++i) win[i] = 0.0;
  int trip = 0;
  if (TECH == HPAC_TECH_PERFO && (p.perfo_kind == HPAC_PERFO_INI || p.perfo_kind == HPAC_PERFO_FINI))
    trip = (int)trip_count(tid, G, p.n, p.steps);

  // per-step bookkeeping kept to what the directive needs: the total and
  // warp-step counts follow from my_steps at the end (a segment has an active
  // lane at step s iff s < its lanes' largest my_steps), and only
  // thread-level decisions can split a segment (warp/team votes are uniform)
  unsigned c_approx = 0, c_div = 0;
  bool app_error = false;
  const double* src = p.region.in + tid * kRec;
  double* const out = p.region.out;
  uint8_t* const paths = p.paths;
  int64_t idx = tid;

  for (int step = 0; step < nsteps; ++step) {
    const bool active = step < my_steps;
    // ---- predicate (engine.hpp:221-251); 1-encounter regions: the
    // per-thread and herded perforation counters both equal `step`
    bool pred = false;
    if (active) {
      if (TECH == HPAC_TECH_TAF) pred = taf_mode == kTafPredicting;
      if (TECH == HPAC_TECH_PERFO)
        pred = perfo_should_skip32(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step, trip,
                                   tid);
    }
    bool approx = pred;
    if (TECH != kTechNoneStream && LEVEL == HPAC_LEVEL_TEAM) {
      const int yes = __syncthreads_count(active && pred);
      const int64_t tr = team_rem - (int64_t)step * G;
      const int cnt = tr <= 0 ? 0 : (tr < tpt ? (int)tr : tpt);
      approx = 2 * yes > cnt;  // majority_decision over the team's active threads
    }
    if (TECH != kTechNoneStream && LEVEL == HPAC_LEVEL_WARP) {
      const unsigned bv = __ballot_sync(0xffffffffu, active && pred) & seg_mask;
      const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
      approx = 2 * __popc(bv) > __popc(ba);
    }
    // ---- lane execution (engine.hpp:303-347)
    if (active) {
      if (approx) {
        if (TECH == HPAC_TECH_TAF) {
          // TafState::emit_approx, taf.hpp:114-117
          if (out) __stcs(out + idx, last);
          if (taf_mode == kTafPredicting && --taf_rem == 0) {
            taf_count = 0;
            taf_mode = kTafFilling;
          }
        }
        // perforation: output untouched
      } else {
        double v = 0.0;
        if (!bs_call(__ldg(src), __ldg(src + 1), __ldg(src + 2), __ldg(src + 3), __ldg(src + 4), v))
          app_error = true;
        if (out) __stcs(out + idx, v);
        if (TECH == HPAC_TECH_TAF) {
          // TafState::observe_accurate, taf.hpp:94-108
#pragma unroll
          for (int i = 0; i + 1 < HW; ++i) win[i] = win[i + 1];
          win[HW - 1] = v;
          if (taf_count < HREG) ++taf_count;
          last = v;
          const bool check =
              (taf_mode == kTafFilling && taf_count == HREG) || taf_mode == kTafChecking;
          if (taf_mode == kTafPredicting) {
            if (--taf_rem == 0) {
              taf_count = 0;
              taf_mode = kTafFilling;
            }
          } else if (check) {
            if (taf_window_passes<HW>(win, p.taf_thr)) {
              taf_rem = p.taf_p;
              taf_mode = kTafPredicting;
            } else {
              taf_mode = kTafChecking;
            }
          }
        }
      }
      if (approx) c_approx += 1;
      if (paths) paths[idx] = approx ? 1 : 0;
    }
    // ---- divergent warp steps (cost.hpp:66-86): thread-level decisions only
    if (TECH != kTechNoneStream && LEVEL == HPAC_LEVEL_THREAD) {
      const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
      const unsigned bx = __ballot_sync(0xffffffffu, active && approx) & seg_mask;
      if (lane == 0 && bx != 0 && bx != ba) c_div += 1;
    }
    src += G * kRec;
    idx += G;
  }
  // warp steps and resident warps of the logical warp (segment): the
  // segment's largest my_steps, at its lane 0
  int seg_steps = my_steps;
  for (int o = 1; o < ws && o < 32; o <<= 1)
    seg_steps = max(seg_steps, __shfl_xor_sync(0xffffffffu, seg_steps, o));
  const unsigned c_total = (unsigned)my_steps;
  const unsigned c_warp = lane == 0 ? (unsigned)seg_steps : 0u;
  const bool resident = lane == 0 && seg_steps > 0;

  const unsigned long long s_total = warp_sum_u32(c_total);
  const unsigned long long s_approx = warp_sum_u32(c_approx);
  const unsigned long long s_warp = warp_sum_u32(c_warp);
  const unsigned long long s_div = warp_sum_u32(c_div);
  const unsigned long long s_res = warp_sum_u32(resident ? 1u : 0u);
  const unsigned any_err = __ballot_sync(0xffffffffu, app_error);
  if (hw_lane == 0) {
    if (s_total) atomicAdd(&p.counters[kCntTotal], s_total);
    if (s_approx) atomicAdd(&p.counters[kCntApprox], s_approx);
    if (s_div) atomicAdd(&p.counters[kCntDivergent], s_div);
    if (s_warp) atomicAdd(&p.counters[kCntWarpSteps], s_warp);
    if (s_res) atomicAdd(&p.counters[kCntResidentWarps], s_res);
    if (any_err) atomicAdd(&p.counters[kCntAppError], 1ull);
  }
}

bool engine_stream_eligible(const EngineParams& p) {
  if (p.region.app != HPAC_APP_BLACKSCHOLES) return false;
  if (p.per_team || p.has_enc || p.barrier_eval || p.staged) return false;
  if (p.steps >= 0x7fffffff) return false;  // 32-bit step counters
  if (!p.fast_ws || p.tpt % 32 != 0 || p.tpt > kStreamMaxT) return false;
  if (p.tech == HPAC_TECH_IACT) return false;
  if (p.tech == HPAC_TECH_TAF && p.taf_h > 8) return false;
  return true;
}

size_t engine_stream_smem(const EngineParams& p) {
  return (size_t)2 * p.tpt * kRec * sizeof(double) + 2 * sizeof(uint64_t);
}

template <int TECH, int LEVEL, int H>
static void stream_launch_h(const EngineParams& p, int nblocks, size_t smem, cudaStream_t st) {
  // two logical threads per CUDA thread (tpt % 64 == 0) only on request
  // (HPAC_STREAM_PAIR=1): measured 97.0 us unpaired vs 98.6 us paired on C1
  // exact (profiles/r02g_bs_pair_ab.txt) — the paired kernel needs 100-119
  // registers, so its doubled ILP is paid for with half the resident warps
  const char* pe = getenv("HPAC_STREAM_PAIR");
  const bool pair_on = pe && strcmp(pe, "1") == 0;
  const char* te = getenv("HPAC_STREAM_TMA");
  const bool tma_on = te && strcmp(te, "1") == 0;
  if (p.tpt % 64 == 0 && pair_on)
    bs_stream_kernel<TECH, LEVEL, H, 2><<<nblocks, p.tpt / 2, smem, st>>>(p);
  else if (tma_on)
    bs_stream_kernel<TECH, LEVEL, H, 1><<<nblocks, p.tpt, smem, st>>>(p);
  else
    bs_lane_kernel<TECH, LEVEL, H><<<nblocks, p.tpt, 0, st>>>(p);
}

template <int TECH, int LEVEL>
static cudaError_t stream_launch_level(const EngineParams& p, int nblocks, size_t smem,
                                       cudaStream_t st) {
  if (TECH == HPAC_TECH_TAF) {
    switch (p.taf_h) {
#define HPAC_S(H) \
  case H: stream_launch_h<TECH, LEVEL, H>(p, nblocks, smem, st); break;
      HPAC_S(1) HPAC_S(2) HPAC_S(3) HPAC_S(4) HPAC_S(5) HPAC_S(6) HPAC_S(7) HPAC_S(8)
#undef HPAC_S
      default: return cudaErrorInvalidValue;
    }
  } else {
    stream_launch_h<TECH, LEVEL, 0>(p, nblocks, smem, st);
  }
  return cudaGetLastError();
}

template <int TECH>
static cudaError_t stream_launch_tech(const EngineParams& p, int nblocks, size_t smem,
                                      cudaStream_t st) {
  if (!p.voting) return stream_launch_level<TECH, HPAC_LEVEL_THREAD>(p, nblocks, smem, st);
  if (p.level == HPAC_LEVEL_WARP) return stream_launch_level<TECH, HPAC_LEVEL_WARP>(p, nblocks, smem, st);
  return stream_launch_level<TECH, HPAC_LEVEL_TEAM>(p, nblocks, smem, st);
}

cudaError_t engine_stream_launch(const EngineParams& p, int nblocks, size_t smem,
                                 cudaStream_t st) {
  switch (p.tech) {
    case HPAC_TECH_TAF: return stream_launch_tech<HPAC_TECH_TAF>(p, nblocks, smem, st);
    case HPAC_TECH_PERFO: return stream_launch_tech<HPAC_TECH_PERFO>(p, nblocks, smem, st);
    default:
      return stream_launch_level<kTechNoneStream, HPAC_LEVEL_THREAD>(p, nblocks, smem, st);
  }
}

}  // namespace hpac
