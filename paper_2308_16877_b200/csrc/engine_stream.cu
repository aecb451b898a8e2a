// engine_stream.cu — the streaming variant of the per-thread engine
// (run_region, engine.hpp:132-402, WorkMapping::kPerThread) for
// single-encounter regions whose accurate path is a pure function of one
// AoS input record: Blackscholes (bench/blackscholes.hpp:72-92).
//
// Same decisions, stats and outputs as engine_thread.cu (and therefore the
// reference); what changes is how the HBM side is driven:
//  * the team's input tile of step s+1 (tpt consecutive 40 B records, one
//    contiguous span) is fetched by ONE thread with a 1-D bulk TMA copy
//    (cp.async.bulk ... mbarrier::complete_tx) into a double-buffered shared
//    tile while the team computes step s, so the FP64-bound evaluation never
//    waits on an HBM round trip;
//  * a tile is not fetched at all when every active thread of the team is
//    known to take the approximate path at s+1 (TAF regime with >= 2
//    predictions left, or a perforation skip) — TAF/perforation then save the
//    input bytes as well as the flops;
//  * the team vote is a __syncthreads_count (no shared atomics), the warp
//    vote a segment-masked __ballot_sync; per-thread counters are 32-bit and
//    reduced once per thread at the end.
// Eligibility (runtime.cu): per-thread mapping, no encounters, no barrier in
// evaluate, warp_size | 32, threads_per_team a multiple of 32 and <= 256,
// technique none / TAF (h <= 8) / perforation.
#include <cuda_runtime.h>

#include "apps.cuh"
#include "engine.h"
#include "hpac_device.cuh"

namespace hpac {

namespace {

constexpr int kStreamMaxT = 256;
constexpr int kTechNoneStream = 3;  // accurate baseline (spec == NULL)
constexpr int kRec = 5;  // doubles per option record

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum_u32(unsigned v) {
  unsigned long long s = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

}  // namespace

template <int TECH, int LEVEL, int HREG>
__global__ void __launch_bounds__(kStreamMaxT, (HREG > 5 ? 3 : 4)) bs_stream_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  const int tpt = p.tpt;
  double* tile = smem;                                             // [2][tpt*5]
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * tpt * kRec);  // [2]

  const int local = threadIdx.x;
  const int team = p.team_begin + (int)blockIdx.x;
  const int64_t tid = (int64_t)team * tpt + local;
  const int64_t G = p.stride;
  const int ws = p.ws;
  const int lane = local % ws;
  const int hw_lane = local & 31;
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << (hw_lane - lane));
  const double* __restrict__ in = p.region.in;
  double* __restrict__ out = p.region.out;
  const int64_t team_base = (int64_t)team * tpt;
  // bulk copies need 16-byte aligned source and size: tpt*40 B per tile is a
  // multiple of 16 when tpt is even (always, tpt % 32 == 0); the ragged last
  // tile of the grid and misaligned buffers fall back to per-thread loads.
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0;

  auto tile_count = [&](int64_t s) -> int {
    const int64_t b = team_base + s * G;
    const int64_t c = p.n - b;
    return c <= 0 ? 0 : (c >= tpt ? tpt : (int)c);
  };
  auto tile_tma = [&](int64_t s) -> bool {
    return aligned && s < p.steps && tile_count(s) == tpt;
  };

  if (local == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t phase0 = 0, phase1 = 0;
  if (local == 0 && p.steps > 0 && tile_tma(0)) {
    mbar_expect_tx(&bar[0], (uint32_t)(tpt * kRec * 8));
    tma_load_1d(tile, in + team_base * kRec, (uint32_t)(tpt * kRec * 8), &bar[0]);
  }
  bool loaded_cur = p.steps > 0 && tile_tma(0);
  // thread 0's bookkeeping: a load into buffer b that no consumer waited for
  // is still "outstanding"; it must be retired before the buffer is re-armed
  // (an mbarrier must not see a second arrive while its phase is pending)
  bool issued0 = loaded_cur, issued1 = false;

  // TAF state (TafState, taf.hpp:59-163): register shift register, oldest first
  int taf_mode = kTafFilling, taf_rem = 0, taf_count = 0;
  double win[HREG > 0 ? HREG : 1];
#pragma unroll
  for (int i = 0; i < (HREG > 0 ? HREG : 1); ++i) win[i] = 0.0;
  double last = 0.0;
  int64_t trip = 0;
  if (TECH == HPAC_TECH_PERFO &&
      (p.perfo_kind == HPAC_PERFO_INI || p.perfo_kind == HPAC_PERFO_FINI))
    trip = trip_count(tid, G, p.n, p.steps);

  unsigned c_total = 0, c_approx = 0, c_warp = 0, c_div = 0;
  bool touched = false, app_error = false;

  for (int64_t step = 0; step < p.steps; ++step) {
    const int cnt = tile_count(step);
    const bool active = local < cnt;  // idx = tid + step*G < n
    const int64_t idx = tid + step * G;
    const int buf = (int)(step & 1);

    // ---- predicate (engine.hpp:221-251); for 1-encounter regions the
    // per-thread and herded perforation counters both equal `step`
    bool pred = false;
    if (active) {
      if (TECH == HPAC_TECH_TAF) pred = taf_mode == kTafPredicting;
      if (TECH == HPAC_TECH_PERFO)
        pred = perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step,
                                 trip, tid);
    }
    // known approximate at step+1 (thread level decisions only depend on
    // the thread's own state; any approximate lane needs no input)
    bool need_next = false;
    if (step + 1 < p.steps && local < tile_count(step + 1)) {
      need_next = true;
      if (TECH == HPAC_TECH_TAF && LEVEL == HPAC_LEVEL_THREAD)
        need_next = !(taf_mode == kTafPredicting && taf_rem >= 2);
      if (TECH == HPAC_TECH_PERFO)
        need_next = !perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed,
                                       step + 1, trip, tid);
    }

    // ---- team barrier: frees tile[buf^1] (consumed at step-1), team vote,
    // and "does anybody need the next tile" in one or two bar.red ops
    bool approx = pred;
    if (TECH != kTechNoneStream && LEVEL == HPAC_LEVEL_TEAM) {
      const int yes = __syncthreads_count(active && pred);
      approx = 2 * yes > cnt;  // majority_decision over the team's active threads
    }
    const int any_next = __syncthreads_or(need_next);
    if (LEVEL == HPAC_LEVEL_WARP && TECH != kTechNoneStream) {
      const unsigned bv = __ballot_sync(0xffffffffu, active && pred) & seg_mask;
      const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
      approx = 2 * __popc(bv) > __popc(ba);
    }
    bool loaded_next = false;
    if (any_next && tile_tma(step + 1)) {
      loaded_next = true;
      if (local == 0) {
        const int nb = buf ^ 1;
        if (nb ? issued1 : issued0) mbar_wait(&bar[nb], (nb ? phase1 : phase0) ^ 1);
        mbar_expect_tx(&bar[nb], (uint32_t)(tpt * kRec * 8));
        tma_load_1d(tile + nb * tpt * kRec, in + (team_base + (step + 1) * G) * kRec,
                    (uint32_t)(tpt * kRec * 8), &bar[nb]);
        if (nb)
          issued1 = true;
        else
          issued0 = true;
      }
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
        double rec[kRec];
        if (loaded_cur) {
          mbar_wait(&bar[buf], buf ? phase1 : phase0);
          const double* t = tile + buf * tpt * kRec + local * kRec;
#pragma unroll
          for (int c = 0; c < kRec; ++c) rec[c] = t[c];
        } else {
          const double* o = in + idx * kRec;
#pragma unroll
          for (int c = 0; c < kRec; ++c) rec[c] = __ldg(o + c);
        }
        double v = 0.0;
        if (!bs_call(rec[0], rec[1], rec[2], rec[3], rec[4], v)) app_error = true;
        if (out) __stcs(out + idx, v);
        if (TECH == HPAC_TECH_TAF) {
          // TafState::observe_accurate, taf.hpp:94-108
#pragma unroll
          for (int i = 0; i + 1 < (HREG > 0 ? HREG : 1); ++i) win[i] = win[i + 1];
          win[(HREG > 0 ? HREG : 1) - 1] = v;
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
            if (taf_window_passes<(HREG > 0 ? HREG : 1)>(win, p.taf_thr)) {
              taf_rem = p.taf_p;
              taf_mode = kTafPredicting;
            } else {
              taf_mode = kTafChecking;
            }
          }
        }
      }
      c_total += 1;
      if (approx) c_approx += 1;
      if (p.paths) p.paths[idx] = approx ? 1 : 0;
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

    // ---- warp stats (cost.hpp:66-86)
    const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
    const unsigned bx = __ballot_sync(0xffffffffu, active && approx) & seg_mask;
    if (lane == 0 && ba) {
      touched = true;
      c_warp += 1;
      if (bx != 0 && bx != ba) c_div += 1;
    }
  }
  // a tile may have been fetched speculatively and then not read by anybody
  // (every lane approximated): thread 0 retires the last copy of each
  // buffer so none is in flight when the CTA exits
  if (local == 0) {
    if (issued0) mbar_wait(&bar[0], phase0 ^ 1);
    if (issued1) mbar_wait(&bar[1], phase1 ^ 1);
  }

  const unsigned long long s_total = warp_sum_u32(c_total);
  const unsigned long long s_approx = warp_sum_u32(c_approx);
  const unsigned long long s_warp = warp_sum_u32(c_warp);
  const unsigned long long s_div = warp_sum_u32(c_div);
  const unsigned long long s_res = warp_sum_u32((lane == 0 && touched) ? 1u : 0u);
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
  if (!p.fast_ws || p.tpt % 32 != 0 || p.tpt > kStreamMaxT) return false;
  if (p.tech == HPAC_TECH_IACT) return false;
  if (p.tech == HPAC_TECH_TAF && p.taf_h > 8) return false;
  return true;
}

size_t engine_stream_smem(const EngineParams& p) {
  return (size_t)2 * p.tpt * kRec * sizeof(double) + 2 * sizeof(uint64_t);
}

template <int TECH, int LEVEL>
static cudaError_t stream_launch_level(const EngineParams& p, int nblocks, size_t smem,
                                       cudaStream_t st) {
  if (TECH == HPAC_TECH_TAF) {
    switch (p.taf_h) {
#define HPAC_S(H) \
  case H: bs_stream_kernel<TECH, LEVEL, H><<<nblocks, p.tpt, smem, st>>>(p); break;
      HPAC_S(1) HPAC_S(2) HPAC_S(3) HPAC_S(4) HPAC_S(5) HPAC_S(6) HPAC_S(7) HPAC_S(8)
#undef HPAC_S
      default: return cudaErrorInvalidValue;
    }
  } else {
    bs_stream_kernel<TECH, LEVEL, 0><<<nblocks, p.tpt, smem, st>>>(p);
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
