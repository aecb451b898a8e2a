// engine_bs_iact.cu — iACT (memo(in:...)) on the Blackscholes region under
// the per-thread mapping: run_region (engine.hpp:132-402) with the iACT
// lookup / vote / writer protocol (engine.hpp:238-242, 318-332, 351-366;
// iact.hpp:43-180), restructured for the GPU.
//
// Why a dedicated engine: iACT decisions depend only on the inputs (the
// table holds past misses' inputs; a hit copies a stored output but never
// looks at it), so the accurate evaluations can be taken out of the
// lockstep loop. The lockstep engine (engine_thread.cu) evaluates the miss
// lanes of a warp while the hit lanes idle, with an HBM round trip per step,
// and was slower than not approximating (0.45x at memo(in:2:0.5)).
//
// Here one CTA = one logical team (64..256 threads); per step:
//  * the team's input tile (tpt consecutive 40 B records, one contiguous
//    span) arrives by bulk TMA into a 4-tile ring, three steps ahead;
//  * every lane looks its record up in its table (shared memory, exact
//    no-FMA squared distance; the hit test sqrt_rn(ssq) <= thr is the exact
//    ssq <= thr2 with thr2 found on the host, and square roots are taken
//    only for near-ties, so decisions are bit-identical), votes
//    (segment ballot / __syncthreads_count), and the per-table writer (max
//    min-distance miss lane, ties to the lowest lane; shuffle butterfly over
//    the lanes sharing the table) inserts its INPUT and its ITEM INDEX at the
//    round-robin cursor;
//  * a lane that must evaluate appends its item to the CTA's miss queue; a
//    lane that approximates appends (item, producing item) to the hit queue
//    (items packed step << 8 | thread in 32 bits).
// Every q_steps steps (and after the last) the CTA prices the queued misses
// densely — two options per thread, records re-read through L2, no lane
// idling behind a hit — and then
// copies each hit's output from its producer (an earlier miss of the same
// team; visible after the barrier).
//
// Stats and path bits are the reference's (cost.hpp:66-86): they depend on
// decisions only. Eligibility (runtime.cu): Blackscholes, per-thread mapping,
// iACT, warp_size | 32, threads_per_team a multiple of 32 and <= 256, no
// encounters / barrier flags.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "apps.cuh"
#include "engine.h"
#include "hpac_device.cuh"
#include "tma.cuh"

namespace hpac {

namespace {
constexpr int kIactMaxT = 256;
constexpr int kRecD = 5;          // doubles per option record
constexpr int kRing = 4;          // input tiles in flight (prefetch distance 3)
constexpr int kQueueItems = 512;  // queued items per queue between flushes

struct IactLayout {
  // offsets in doubles from the dynamic smem base
  int tile, tab_in, tab_src, q_miss, q_hit, q_src, ctl, total;
};

// items are packed (step << 8 | local) in 32 bits: the producing item of a
// hit is always in the same team (steps < 2^23, tpt <= 256)
__host__ __device__ inline IactLayout iact_layout(int tpt, int T, int tsize, int q_steps) {
  IactLayout L;
  const int cap = q_steps * tpt;
  L.tile = 0;                                    // [kRing][tpt*5]
  L.tab_in = L.tile + kRing * tpt * kRecD;       // [(slot*5 + c)*T + tab]
  L.tab_src = L.tab_in + tsize * kRecD * T;      // int32 [slot*T + tab]
  L.q_miss = L.tab_src + (tsize * T + 1) / 2;    // int32 [cap]
  L.q_hit = L.q_miss + (cap + 1) / 2;            // int32 [cap]
  L.q_src = L.q_hit + (cap + 1) / 2;             // int32 [cap]
  L.ctl = L.q_src + (cap + 1) / 2;               // kRing mbarriers + 2 counters
  L.total = L.ctl + kRing + 1;
  return L;
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned v) {
  unsigned long long s = v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
}  // namespace

// TS: compile-time table size (1..8; slots in registers of the unrolled
// lookup so the per-slot distance chains run in parallel), 0 = runtime size
template <int LEVEL, int TS>
__global__ void __launch_bounds__(kIactMaxT) bs_iact_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  const int tpt = p.tpt;
  const int local = threadIdx.x;
  const int team = p.team_begin + (int)blockIdx.x;
  const int64_t team_base = (int64_t)team * tpt;
  const int64_t G = p.stride;
  const int ws = p.ws;
  const int lane = local % ws;
  const int wloc = local / ws;
  const int hw_lane = local & 31;
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << (hw_lane - lane));
  const int tpw = p.tpw;
  const int group = ws / tpw;  // lanes sharing one table (a power of two)
  const int T = p.wpt * tpw;
  const int tab = wloc * tpw + lane / group;
  const int tsize = p.tsize;
  const double thr2 = p.iact_thr2;
  const IactLayout L = iact_layout(tpt, T, tsize, p.q_steps);
  double* tile = smem + L.tile;
  double* tab_in = smem + L.tab_in;
  int* tab_src = reinterpret_cast<int*>(smem + L.tab_src);
  int* q_miss = reinterpret_cast<int*>(smem + L.q_miss);
  int* q_hit = reinterpret_cast<int*>(smem + L.q_hit);
  int* q_src = reinterpret_cast<int*>(smem + L.q_src);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.ctl);  // [kRing]
  int* qc = reinterpret_cast<int*>(smem + L.ctl + kRing);     // [0] misses, [1] hits
  const double* __restrict__ in = p.region.in;
  double* __restrict__ out = p.region.out;
  auto item = [&](int packed) -> int64_t {
    return team_base + (packed & 255) + (int64_t)(packed >> 8) * G;
  };

  // per-team schedule bounds (as engine_stream.cu)
  const int64_t rem0 = p.n - team_base;
  const int tsteps = rem0 <= 0 ? 0 : (int)(p.steps < (rem0 - 1) / G + 1 ? p.steps : (rem0 - 1) / G + 1);
  const int full = rem0 < tpt ? 0 : (int)(p.steps < (rem0 - tpt) / G + 1 ? p.steps : (rem0 - tpt) / G + 1);
  const int ragged = tsteps > full ? (int)(rem0 - (int64_t)full * G) : 0;
  const int nsteps = (int)p.steps;
  const bool aligned = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  auto tile_count = [&](int s) -> int { return s < full ? tpt : (s == full ? ragged : 0); };
  auto tile_tma = [&](int s) -> bool { return aligned && s < full; };
  const uint32_t tile_bytes = (uint32_t)(tpt * kRecD * 8);
  auto issue = [&](int s) {
    uint64_t* b = &bar[s % kRing];
    mbar_expect_tx(b, tile_bytes);
    tma_load_1d(tile + (s % kRing) * tpt * kRecD, in + (team_base + (int64_t)s * G) * kRecD,
                tile_bytes, b);
  };

  if (local == 0) {
#pragma unroll
    for (int r = 0; r < kRing; ++r) mbar_init(&bar[r], 1);
    mbar_fence_init();
    qc[0] = 0;
    qc[1] = 0;
    // every tile loaded is consumed by a full team at its step (s < full)
    for (int s = 0; s < kRing - 1; ++s)
      if (tile_tma(s)) issue(s);
  }
  int rr = 0, occ = 0;  // MemoTable cursor / occupancy, identical across the group
  unsigned c_total = 0, c_approx = 0, c_warp = 0, c_div = 0;
  bool touched = false, app_error = false;

  for (int step = 0; step < nsteps; ++step) {
    const int cnt = tile_count(step);
    const bool active = local < cnt;
    const int me = (step << 8) | local;
    // everyone is done with the ring slot of step-1 and the queues are reset
    __syncthreads();
    if (local == 0 && tile_tma(step + kRing - 1)) issue(step + kRing - 1);

    // ---- load_input + MemoTable lookup (iact.hpp:58-110): nearest slot by
    // IEEE distance sqrt(sum of no-FMA squares), lowest slot on ties; the hit
    // test sqrt_rn(ssq) <= thr is ssq <= thr2 exactly, and the square roots
    // are only taken when two candidates' ssq are close enough to round to
    // the same distance
    double x[kRecD];
    int near = -1;
    double near_q = dinf();
    if (active) {
      if (tile_tma(step)) {
        mbar_wait(&bar[step % kRing], (uint32_t)((step / kRing) & 1));
        const double* t = tile + (step % kRing) * tpt * kRecD + local * kRecD;
#pragma unroll
        for (int c = 0; c < kRecD; ++c) x[c] = t[c];
      } else {
        const double* o = in + item(me) * kRecD;
#pragma unroll
        for (int c = 0; c < kRecD; ++c) x[c] = __ldg(o + c);
      }
      if constexpr (TS > 0) {
        // all slots' squared distances first (independent chains), then the
        // in-order selection
        double q[TS];
#pragma unroll
        for (int s = 0; s < TS; ++s) {
          double ssq = 0.0;
#pragma unroll
          for (int c = 0; c < kRecD; ++c) {
            const double df = __dsub_rn(tab_in[(s * kRecD + c) * T + tab], x[c]);
            ssq = __dadd_rn(ssq, __dmul_rn(df, df));
          }
          q[s] = ssq;
        }
#pragma unroll
        for (int s = 0; s < TS; ++s) {
          if (s < occ && q[s] < near_q) {
            bool take = true;
            if (near >= 0 && q[s] >= near_q * (1.0 - 0x1p-48))
              take = __dsqrt_rn(q[s]) < __dsqrt_rn(near_q);
            if (take) {
              near_q = q[s];
              near = s;
            }
          }
        }
      } else {
        for (int s = 0; s < occ; ++s) {
          double ssq = 0.0;
#pragma unroll
          for (int c = 0; c < kRecD; ++c) {
            const double df = __dsub_rn(tab_in[(s * kRecD + c) * T + tab], x[c]);
            ssq = __dadd_rn(ssq, __dmul_rn(df, df));
          }
          if (ssq < near_q) {
            bool take = true;
            if (near >= 0 && ssq >= near_q * (1.0 - 0x1p-48))
              take = __dsqrt_rn(ssq) < __dsqrt_rn(near_q);
            if (take) {
              near_q = ssq;
              near = s;
            }
          }
        }
      }
    }
    const bool pred = active && near >= 0 && near_q <= thr2;

    // ---- decision hierarchy (hierarchy.hpp:33-70)
    bool approx = pred;
    if (LEVEL == HPAC_LEVEL_WARP) {
      const unsigned bv = __ballot_sync(0xffffffffu, pred) & seg_mask;
      const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
      approx = 2 * __popc(bv) > __popc(ba);
    } else if (LEVEL == HPAC_LEVEL_TEAM) {
      approx = 2 * __syncthreads_count(pred) > cnt;
    }

    // ---- lane execution (engine.hpp:318-332): approximate = the slot's
    // output (nearest slot when forced); empty table = accurate fallback
    int kind = 0;  // 1 = price (queue), 2 = copy from the producing item
    int src = 0;
    bool cand = false;
    if (active) {
      if (approx) {
        if (near >= 0) {
          kind = 2;
          src = tab_src[near * T + tab];
        } else {
          approx = false;
        }
      }
      if (!approx) {
        kind = 1;
        cand = !pred;  // a miss that evaluates is a writer candidate
      }
      c_total += 1;
      if (approx) c_approx += 1;
      if (p.paths) p.paths[item(me)] = approx ? 1 : 0;
    }

    // ---- writer (iact.hpp:166-180): max min-distance candidate, lowest
    // lane; with one lane per table the candidate writes itself
    if (group > 1) {
      double bd = cand ? __dsqrt_rn(near_q) : -1.0;
      int bl = lane;
      for (int off = group >> 1; off > 0; off >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, bd, off);
        const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
        if (writer_better(od, ol, bd, bl)) {
          bd = od;
          bl = ol;
        }
      }
      if (bd >= 0.0) {
        if (lane == bl) {
#pragma unroll
          for (int c = 0; c < kRecD; ++c) tab_in[(rr * kRecD + c) * T + tab] = x[c];
          tab_src[rr * T + tab] = me;
        }
        rr = rr + 1 == tsize ? 0 : rr + 1;
        occ = occ + 1 < tsize ? occ + 1 : tsize;
      }
    } else if (cand) {
#pragma unroll
      for (int c = 0; c < kRecD; ++c) tab_in[(rr * kRecD + c) * T + tab] = x[c];
      tab_src[rr * T + tab] = me;
      rr = rr + 1 == tsize ? 0 : rr + 1;
      occ = occ + 1 < tsize ? occ + 1 : tsize;
    }

    // ---- queue pushes (warp-aggregated)
    {
      const unsigned lt = (1u << hw_lane) - 1u;
      const unsigned bm = __ballot_sync(0xffffffffu, kind == 1);
      const unsigned bh = __ballot_sync(0xffffffffu, kind == 2);
      int base_m = 0, base_h = 0;
      if (hw_lane == 0) {
        if (bm) base_m = atomicAdd(&qc[0], __popc(bm));
        if (bh) base_h = atomicAdd(&qc[1], __popc(bh));
      }
      base_m = __shfl_sync(0xffffffffu, base_m, 0);
      base_h = __shfl_sync(0xffffffffu, base_h, 0);
      if (kind == 1) {
        q_miss[base_m + __popc(bm & lt)] = me;
      } else if (kind == 2) {
        const int q = base_h + __popc(bh & lt);
        q_hit[q] = me;
        q_src[q] = src;
      }
    }

    // ---- warp stats (cost.hpp:66-86)
    {
      const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
      const unsigned bx = __ballot_sync(0xffffffffu, active && approx) & seg_mask;
      if (lane == 0 && ba) {
        touched = true;
        c_warp += 1;
        if (bx != 0 && bx != ba) c_div += 1;
      }
    }
    __syncwarp();  // table inserts visible to the group's next lookups

    // ---- flush: dense pricing of the misses (records re-read through L2),
    // then the hits' copies from their producers
    if ((step + 1) % p.q_steps == 0 || step + 1 == nsteps) {
      __syncthreads();
      const int mc = qc[0], hc = qc[1];
      const int nt = blockDim.x;
      for (int i = local; i < mc; i += 2 * nt) {
        const int j = i + nt < mc ? i + nt : i;
        const int64_t e0 = item(q_miss[i]), e1 = item(q_miss[j]);
        const double* r0 = in + e0 * kRecD;
        const double* r1 = in + e1 * kRecD;
        double a[kRecD], b[kRecD];
#pragma unroll
        for (int c = 0; c < kRecD; ++c) {
          a[c] = __ldg(r0 + c);
          b[c] = __ldg(r1 + c);
        }
        double v0, v1;
        const bool ok0 = bs_call(a[0], a[1], a[2], a[3], a[4], v0);
        const bool ok1 = bs_call(b[0], b[1], b[2], b[3], b[4], v1);
        if (!ok0 || !ok1) app_error = true;
        if (out) {
          __stcs(out + e0, v0);
          if (j != i) __stcs(out + e1, v1);
        }
      }
      __syncthreads();
      if (out)
        for (int i = local; i < hc; i += nt) __stcs(out + item(q_hit[i]), __ldcg(out + item(q_src[i])));
      if (local == 0) {
        qc[0] = 0;
        qc[1] = 0;
      }
      // the next step's leading barrier orders the reset before new pushes
    }
  }

  const unsigned long long s_total = warp_sum(c_total);
  const unsigned long long s_approx = warp_sum(c_approx);
  const unsigned long long s_warp = warp_sum(c_warp);
  const unsigned long long s_div = warp_sum(c_div);
  const unsigned long long s_res = warp_sum((lane == 0 && touched) ? 1u : 0u);
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

// ---------------------------------------------------------------------------
// Per-lane tables (tables_per_warp == warp_size, the default), thread or warp
// level: no lane ever reads another lane's table, so the table lives in the
// lane's registers and the whole decision stream of a chunk of 32 steps runs
// without shared memory or barriers (warp votes are one ballot per step). The
// warp then prices its chunk's misses densely (two per thread) into a shared
// 32 x 32 output tile, resolves the hits (a producer earlier in the chunk
// from the tile, an older one from the slot's remembered price), and stores
// the tile coalesced. Warps are independent: one CTA = one team.
// ---------------------------------------------------------------------------
constexpr int kLaneChunk = 32;

#ifndef HPAC_IACT_LANE_MINB
#define HPAC_IACT_LANE_MINB 1  // min 256-thread-equivalent blocks (register cap)
#endif
#ifndef HPAC_IACT_LANE_PAIR
#define HPAC_IACT_LANE_PAIR 0  // 1: price two misses per iteration (117 vs 131 us at 0)
#endif
template <int LEVEL, int TS>
__global__ void __launch_bounds__(kIactMaxT, HPAC_IACT_LANE_MINB) bs_iact_lane_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  const int local = threadIdx.x;
  const int warp = local >> 5, lane = local & 31;
  const int team = p.team_begin + (int)blockIdx.x;
  const int64_t tid = (int64_t)team * p.tpt + local;
  const int64_t G = p.stride;
  const int ws = p.ws;
  const int sl = lane % ws;  // logical lane
  const unsigned seg_mask = ws >= 32 ? 0xffffffffu : (((1u << ws) - 1u) << (lane - sl));
  const double thr2 = p.iact_thr2;
  const double* __restrict__ in = p.region.in;
  double* __restrict__ out = p.region.out;
  // per-warp shared tile: outputs [32 steps][32 lanes], hit producers, miss list
  double* tile = smem + warp * (kLaneChunk * 32 + kLaneChunk * 32 / 8 + kLaneChunk * 32 / 4);
  signed char* hsrc = reinterpret_cast<signed char*>(tile + kLaneChunk * 32);          // [s][lane]
  short* mlist = reinterpret_cast<short*>(tile + kLaneChunk * 32 + kLaneChunk * 32 / 8);  // [<=1024]

  double tab[TS][kRecD];
  int sstep[TS];   // producing step of each slot
  double sval[TS]; // its price, once known (chunks before the current one)
#pragma unroll
  for (int k = 0; k < TS; ++k) {
    sstep[k] = -1;
    sval[k] = 0.0;
#pragma unroll
    for (int c = 0; c < kRecD; ++c) tab[k][c] = 0.0;
  }
  int rr = 0, occ = 0;
  unsigned c_total = 0, c_approx = 0, c_warp = 0, c_div = 0;
  bool touched = false, app_error = false;
  const int nsteps = (int)p.steps;

  for (int c0 = 0; c0 < nsteps; c0 += kLaneChunk) {
    const int cs = nsteps - c0 < kLaneChunk ? nsteps - c0 : kLaneChunk;
    unsigned act_m = 0, apx_m = 0, miss_m = 0;
    // ---- decisions: lookup (iact.hpp:58-110), vote, table insert
    double xn[kRecD];
    {
      const int64_t idx0 = tid + (int64_t)c0 * G;
      if (idx0 < p.n) {
#pragma unroll
        for (int c = 0; c < kRecD; ++c) xn[c] = __ldg(in + idx0 * kRecD + c);
      }
    }
    for (int s = 0; s < cs; ++s) {
      const int step = c0 + s;
      const int64_t idx = tid + (int64_t)step * G;
      const bool active = idx < p.n;
      double x[kRecD];
#pragma unroll
      for (int c = 0; c < kRecD; ++c) x[c] = xn[c];
      if (s + 1 < cs && idx + G < p.n) {  // next step's record in flight during this lookup
#pragma unroll
        for (int c = 0; c < kRecD; ++c) xn[c] = __ldg(in + (idx + G) * kRecD + c);
      }
      int near = -1;
      double near_q = dinf();
      double q[TS];
#pragma unroll
      for (int k = 0; k < TS; ++k) {
        double ssq = 0.0;
#pragma unroll
        for (int c = 0; c < kRecD; ++c) {
          const double df = __dsub_rn(tab[k][c], x[c]);
          ssq = __dadd_rn(ssq, __dmul_rn(df, df));
        }
        q[k] = ssq;
      }
#pragma unroll
      for (int k = 0; k < TS; ++k) {
        if (active && k < occ && q[k] < near_q) {
          bool take = true;
          if (near >= 0 && q[k] >= near_q * (1.0 - 0x1p-48))
            take = __dsqrt_rn(q[k]) < __dsqrt_rn(near_q);
          if (take) {
            near_q = q[k];
            near = k;
          }
        }
      }
      const bool pred = active && near >= 0 && near_q <= thr2;
      bool approx = pred;
      if (LEVEL == HPAC_LEVEL_WARP) {
        const unsigned bv = __ballot_sync(0xffffffffu, pred) & seg_mask;
        const unsigned ba = __ballot_sync(0xffffffffu, active) & seg_mask;
        approx = 2 * __popc(bv) > __popc(ba);
      }
      signed char hs = -1;
      if (active) {
        if (approx && near < 0) approx = false;  // empty table: accurate fallback
        if (approx) {
          // the slot's output (nearest slot when forced): a producer in this
          // chunk is resolved after pricing, an older one's price is known
          int ps = 0;
          double pv = 0.0;
#pragma unroll
          for (int k = 0; k < TS; ++k)
            if (k == near) {
              ps = sstep[k];
              pv = sval[k];
            }
          if (ps >= c0) hs = (signed char)(ps - c0);
          else tile[s * 32 + lane] = pv;
        } else {
          miss_m |= 1u << s;
          if (!pred) {  // writer (one lane per table): insert at the cursor
#pragma unroll
            for (int k = 0; k < TS; ++k)
              if (k == rr) {
#pragma unroll
                for (int c = 0; c < kRecD; ++c) tab[k][c] = x[c];
                sstep[k] = step;
              }
            rr = rr + 1 == TS ? 0 : rr + 1;
            occ = occ + 1 < TS ? occ + 1 : TS;
          }
        }
        act_m |= 1u << s;
        if (approx) apx_m |= 1u << s;
        if (p.paths) p.paths[idx] = approx ? 1 : 0;
      }
      hsrc[s * 32 + lane] = hs;
    }
    // ---- warp stats (cost.hpp:66-86)
    for (int s = 0; s < cs; ++s) {
      const unsigned ba = __ballot_sync(0xffffffffu, (act_m >> s) & 1u) & seg_mask;
      const unsigned bx = __ballot_sync(0xffffffffu, (apx_m >> s) & 1u) & seg_mask;
      if (sl == 0 && ba) {
        touched = true;
        c_warp += 1;
        if (bx != 0 && bx != ba) c_div += 1;
      }
    }
    c_total += __popc(act_m);
    c_approx += __popc(apx_m);
    // ---- the warp's misses, densely: exclusive scan of the per-lane counts
    const int mine = __popc(miss_m);
    int off = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, off, o);
      if (lane >= o) off += t;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= mine;
    for (unsigned m = miss_m; m; m &= m - 1) mlist[off++] = (short)((__ffs(m) - 1) * 32 + lane);
    __syncwarp();
    for (int i = lane; i < total; i += (HPAC_IACT_LANE_PAIR ? 64 : 32)) {
      const int j = HPAC_IACT_LANE_PAIR && i + 32 < total ? i + 32 : i;
      const int e0 = mlist[i], e1 = mlist[j];
      const int64_t t0 = tid - lane + (e0 & 31) + (int64_t)(c0 + (e0 >> 5)) * G;
      const int64_t t1 = tid - lane + (e1 & 31) + (int64_t)(c0 + (e1 >> 5)) * G;
      double a[kRecD], b[kRecD];
#pragma unroll
      for (int c = 0; c < kRecD; ++c) {
        a[c] = __ldg(in + t0 * kRecD + c);
        b[c] = __ldg(in + t1 * kRecD + c);
      }
      double v0, v1;
      const bool ok0 = bs_call(a[0], a[1], a[2], a[3], a[4], v0);
      const bool ok1 = HPAC_IACT_LANE_PAIR ? bs_call(b[0], b[1], b[2], b[3], b[4], v1) : true;
      if (!ok0 || !ok1) app_error = true;
      tile[(e0 >> 5) * 32 + (e0 & 31)] = v0;
      if (j != i) tile[(e1 >> 5) * 32 + (e1 & 31)] = v1;
    }
    __syncwarp();
    // ---- hits from producers in this chunk, remembered slot prices, store
    for (int s = 0; s < cs; ++s) {
      const int h = hsrc[s * 32 + lane];
      if (h >= 0) tile[s * 32 + lane] = tile[h * 32 + lane];
    }
#pragma unroll
    for (int k = 0; k < TS; ++k)
      if (sstep[k] >= c0) sval[k] = tile[(sstep[k] - c0) * 32 + lane];
    if (out)
      for (int s = 0; s < cs; ++s)
        if ((act_m >> s) & 1u) __stcs(out + tid + (int64_t)(c0 + s) * G, tile[s * 32 + lane]);
    __syncwarp();
  }

  const unsigned long long s_total = warp_sum(c_total);
  const unsigned long long s_approx = warp_sum(c_approx);
  const unsigned long long s_warp = warp_sum(c_warp);
  const unsigned long long s_div = warp_sum(c_div);
  const unsigned long long s_res = warp_sum((sl == 0 && touched) ? 1u : 0u);
  const unsigned any_err = __ballot_sync(0xffffffffu, app_error);
  if (lane == 0) {
    if (s_total) atomicAdd(&p.counters[kCntTotal], s_total);
    if (s_approx) atomicAdd(&p.counters[kCntApprox], s_approx);
    if (s_div) atomicAdd(&p.counters[kCntDivergent], s_div);
    if (s_warp) atomicAdd(&p.counters[kCntWarpSteps], s_warp);
    if (s_res) atomicAdd(&p.counters[kCntResidentWarps], s_res);
    if (any_err) atomicAdd(&p.counters[kCntAppError], 1ull);
  }
}

static bool bs_iact_lane_eligible(const EngineParams& p) {
  const char* e = getenv("HPAC_IACT_LANE");
  return !(e && strcmp(e, "0") == 0) && p.tpw == p.ws && p.level != HPAC_LEVEL_TEAM &&
         (p.tsize == 1 || p.tsize == 2 || p.tsize == 4 || p.tsize == 8);
}

static size_t bs_iact_lane_smem(const EngineParams& p) {
  return (size_t)(p.tpt / 32) * (kLaneChunk * 32 + kLaneChunk * 32 / 8 + kLaneChunk * 32 / 4) *
         sizeof(double);
}

bool engine_bs_iact_eligible(const EngineParams& p) {
  return p.region.app == HPAC_APP_BLACKSCHOLES && p.tech == HPAC_TECH_IACT && !p.per_team &&
         !p.has_enc && !p.barrier_eval && p.fast_ws && p.tpt % 32 == 0 && p.tpt <= kIactMaxT &&
         p.in_dims == kRecD && p.out_dims == 1 && p.steps < (1 << 23);
}

size_t engine_bs_iact_smem(EngineParams& p) {
  if (bs_iact_lane_eligible(p)) return bs_iact_lane_smem(p);
  p.q_steps = kQueueItems / p.tpt > 0 ? kQueueItems / p.tpt : 1;
  const IactLayout L = iact_layout(p.tpt, p.wpt * p.tpw, p.tsize, p.q_steps);
  return (size_t)L.total * sizeof(double);
}

template <int TS>
static auto bs_iact_pick(const EngineParams& p) {
  return p.voting ? (p.level == HPAC_LEVEL_WARP ? bs_iact_kernel<HPAC_LEVEL_WARP, TS>
                                                : bs_iact_kernel<HPAC_LEVEL_TEAM, TS>)
                  : bs_iact_kernel<HPAC_LEVEL_THREAD, TS>;
}

template <int TS>
static auto bs_iact_lane_pick(const EngineParams& p) {
  return p.level == HPAC_LEVEL_WARP && p.voting ? bs_iact_lane_kernel<HPAC_LEVEL_WARP, TS>
                                                : bs_iact_lane_kernel<HPAC_LEVEL_THREAD, TS>;
}

cudaError_t engine_bs_iact_launch(const EngineParams& p, int nblocks, size_t smem,
                                  cudaStream_t st) {
  if (bs_iact_lane_eligible(p)) {
    auto k = p.tsize == 1   ? bs_iact_lane_pick<1>(p)
             : p.tsize == 2 ? bs_iact_lane_pick<2>(p)
             : p.tsize == 4 ? bs_iact_lane_pick<4>(p)
                            : bs_iact_lane_pick<8>(p);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k<<<nblocks, p.tpt, smem, st>>>(p);
    return cudaGetLastError();
  }
  // table slots unrolled for the common sizes; the table's smem contents are
  // only read below occ, so unrolled reads past occ see stale but unused data
  auto k = p.tsize == 1   ? bs_iact_pick<1>(p)
           : p.tsize == 2 ? bs_iact_pick<2>(p)
           : p.tsize == 4 ? bs_iact_pick<4>(p)
           : p.tsize == 8 ? bs_iact_pick<8>(p)
                          : bs_iact_pick<0>(p);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<nblocks, p.tpt, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace hpac
