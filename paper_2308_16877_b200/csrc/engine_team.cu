// engine_team.cu — the approximate-region engine for the per-team work
// mapping (WorkMapping::kPerTeam, grid.hpp:14): every thread of a logical
// team works on the same item (engine.hpp:198, machine.hpp:77-80).
//
// Key property (verified there on the reference): under
// per-team mapping every lane of a team sees the same input, the same
// outputs and therefore the same technique state, so every predicate and
// every vote is team-uniform; iACT writer choice is the lowest lane and all
// of a team's tables hold identical entries. The engine therefore keeps ONE
// decision state per team (a team-shared iACT table, one TAF window, one
// perforation counter) and scales the lane-level statistics by the team
// shape: total/approx invocations x threads_per_team, warp steps x
// warps_per_team, zero divergence, uniform barrier arrivals. Results,
// decisions and stats equal the reference's lane-by-lane execution.
//
// Two kernels:
//  * engine_team_seq_kernel: apps whose evaluate is a scalar function
//    (TABLE / SYNTHETIC / BLACKSCHOLES); one CUDA thread runs one team.
//  * binomial_team_kernel: the CRR lattice (bench/binomial.hpp:16-50) is
//    evaluated cooperatively by a warp with a register-blocked, rebalanced
//    lattice; iACT / perforation decisions depend on inputs only, so the
//    team first decides a chunk of its items, then its warps evaluate the
//    misses in parallel and hits are resolved from the producing step.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "apps.cuh"
#include "fastmath.cuh"
#include "engine.h"
#include "hpac_device.cuh"

namespace hpac {

constexpr int kTechNoneT = 3;

namespace {

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void flush_stats(const EngineParams& p, unsigned long long tot,
                                            unsigned long long app, unsigned long long ws,
                                            unsigned long long res, bool err) {
  tot = warp_sum(tot);
  app = warp_sum(app);
  ws = warp_sum(ws);
  res = warp_sum(res);
  unsigned e = __ballot_sync(0xffffffffu, err);
  if ((threadIdx.x & 31) == 0) {
    if (tot) atomicAdd(&p.counters[kCntTotal], tot);
    if (app) atomicAdd(&p.counters[kCntApprox], app);
    if (ws) atomicAdd(&p.counters[kCntWarpSteps], ws);
    if (res) atomicAdd(&p.counters[kCntResidentWarps], res);
    if (e) atomicAdd(&p.counters[kCntAppError], 1ull);
  }
}

// Team-shared iACT lookup (MemoTable::lookup / nearest_slot, iact.hpp:93-122)
// over `occ` slots of a table stored as tab[(slot*D + c) * stride].
__device__ __forceinline__ void team_lookup(const double* tab, int stride, int D, int in_dims,
                                            const double* in, int occ, double thr, int& hit,
                                            int& near) {
  double hit_d = 0.0, near_d = dinf();
  hit = -1;
  near = -1;
  for (int s = 0; s < occ; ++s) {
    double ssq = 0.0;
    for (int c = 0; c < in_dims; ++c) {
      double df = __dsub_rn(tab[(s * D + c) * stride], in[c]);
      ssq = __dadd_rn(ssq, __dmul_rn(df, df));
    }
    double dd = __dsqrt_rn(ssq);
    if (dd <= thr && (hit < 0 || dd < hit_d)) {
      hit = s;
      hit_d = dd;
    }
    if (dd < near_d) {
      near_d = dd;
      near = s;
    }
  }
}

// team_lookup's hit for 5-dimensional records without square roots:
// sqrt_rn(ssq) <= thr  <=>  ssq <= thr2 (runtime.cu sqrt_threshold_square),
// and a later slot replaces the hit iff its rounded distance is strictly
// smaller: certain when its ssq is below the hit's by more than 2^-48
// relative (a 2^-49 gap in the root, far above rounding), decided on the
// rounded roots when the two ssq are that close.
__device__ __forceinline__ int team_hit5(const double* tab, const double* in, int occ, double thr2) {
  int hit = -1;
  double hq = 0.0;
  for (int s = 0; s < occ; ++s) {
    double ssq = 0.0;
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      const double df = __dsub_rn(tab[s * 5 + c], in[c]);
      ssq = __dadd_rn(ssq, __dmul_rn(df, df));
    }
    if (ssq <= thr2) {
      bool take = hit < 0 || ssq < hq * (1.0 - 0x1p-48);
      if (!take && ssq < hq) take = __dsqrt_rn(ssq) < __dsqrt_rn(hq);
      if (take) {
        hit = s;
        hq = ssq;
      }
    }
  }
  return hit;
}

}  // namespace

// Every lane of the team stores (engine.hpp:317,338); only an accumulating
// store is observable more than once, so repeat it threads_per_team times.
template <class App, class Out>
__device__ __forceinline__ void store_team(const EngineParams& p, int64_t idx, const Out& out) {
  const int reps = p.accumulate ? p.tpt : 1;
  for (int r = 0; r < reps; ++r) App::store(p, idx, out, r);
}

// ===========================================================================
// Scalar apps under per-team mapping: one CUDA thread = one logical team.
// ===========================================================================
template <class App, int TECH, int HREG>
__global__ void __launch_bounds__(128) engine_team_seq_kernel(const EngineParams p, int team_end) {
  extern __shared__ __align__(16) double smem[];
  constexpr int IN_MAX = App::IN_MAX;
  constexpr int OUT_MAX = App::OUT_MAX;
  const int team = p.team_begin + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  const bool live = team < team_end;
  const int stride_s = blockDim.x;
  double* ring = smem + p.smem_taf_off;  // [(d*h + slot) * blockDim + t]
  double* tab = smem + p.smem_tab_off;   // [(slot*D + c) * blockDim + t]
  ring += threadIdx.x;
  tab += threadIdx.x;
  const int D = p.in_dims + p.out_dims;

  int mode = kTafFilling, rem = 0, cnt = 0, head = 0;
  double win[HREG > 0 ? HREG : 1];
#pragma unroll
  for (int i = 0; i < (HREG > 0 ? HREG : 1); ++i) win[i] = 0.0;
  double last[OUT_MAX];
#pragma unroll
  for (int d = 0; d < OUT_MAX; ++d) last[d] = 0.0;
  int rr = 0, occ = 0;
  int64_t pcount = 0;
  int64_t trip = live ? trip_count(team, p.stride, p.n, p.steps) : 0;

  unsigned long long tot = 0, app = 0, wsteps = 0;
  bool touched = false, err = false;
  const unsigned long long tpt = (unsigned long long)p.tpt;
  const unsigned long long wpt = (unsigned long long)p.wpt;

  for (int64_t step = 0; live && step < trip; ++step) {
    const int64_t idx = team + step * p.stride;
    const int enc = p.has_enc ? App::encounters(p, idx) : 1;
    uint8_t pbits = 0;
    for (int round = 0; round < enc; ++round) {
      double in[IN_MAX];
      bool loaded = false, pred = false;
      int hit = -1, near = -1;
      if (TECH == HPAC_TECH_TAF) {
        pred = mode == kTafPredicting;
      } else if (TECH == HPAC_TECH_IACT) {
        App::load(p, idx, in);
        loaded = true;
        team_lookup(tab, stride_s, D, p.in_dims, in, occ, p.iact_thr, hit, near);
        pred = hit >= 0;
      } else if (TECH == HPAC_TECH_PERFO) {
        // per-thread and herded counters coincide under per-team mapping
        pred = perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, pcount,
                                 trip, team);
      }
      bool approx = pred;  // unanimous: every vote returns the predicate
      double out[OUT_MAX];
#pragma unroll
      for (int d = 0; d < OUT_MAX; ++d) out[d] = 0.0;
      if (approx) {
        if (TECH == HPAC_TECH_TAF) {
#pragma unroll
          for (int d = 0; d < OUT_MAX; ++d) out[d] = last[d];
          if (mode == kTafPredicting && --rem == 0) {
            cnt = 0;
            head = 0;
            mode = kTafFilling;
          }
          store_team<App>(p, idx, out);
        } else if (TECH == HPAC_TECH_IACT) {
#pragma unroll
          for (int d = 0; d < OUT_MAX; ++d)
            if (d < p.out_dims) out[d] = tab[(hit * D + p.in_dims + d) * stride_s];
          store_team<App>(p, idx, out);
        }
      } else {
        if (!loaded) App::load(p, idx, in);
        if (!App::eval(p, idx, in, out, nullptr, 0, round)) err = true;
        store_team<App>(p, idx, out);
        if (TECH == HPAC_TECH_TAF) {
          bool full;
          if (HREG > 0) {
#pragma unroll
            for (int i = 0; i + 1 < (HREG > 0 ? HREG : 1); ++i) win[i] = win[i + 1];
            win[(HREG > 0 ? HREG : 1) - 1] = out[0];
            if (cnt < HREG) ++cnt;
            full = cnt == HREG;
          } else {
            const int h = p.taf_h;
            int slot;
            if (cnt < h) {
              slot = head + cnt;
              if (slot >= h) slot -= h;
              ++cnt;
            } else {
              slot = head;
              head = head + 1 == h ? 0 : head + 1;
            }
            for (int d = 0; d < p.out_dims; ++d) ring[(d * h + slot) * stride_s] = out[d];
            full = cnt == h;
          }
#pragma unroll
          for (int d = 0; d < OUT_MAX; ++d) last[d] = out[d];
          if (mode == kTafPredicting) {
            if (--rem == 0) {
              cnt = 0;
              head = 0;
              mode = kTafFilling;
            }
          } else if ((mode == kTafFilling && full) || mode == kTafChecking) {
            bool pass = true;
            if (HREG > 0) {
              pass = taf_window_passes<(HREG > 0 ? HREG : 1)>(win, p.taf_thr);
            } else {
              for (int d = 0; d < p.out_dims && pass; ++d)
                pass = taf_ring_passes(ring + d * p.taf_h * stride_s, stride_s, p.taf_h, head,
                                       cnt, p.taf_thr);
            }
            if (pass) {
              rem = p.taf_p;
              mode = kTafPredicting;
            } else {
              mode = kTafChecking;
            }
          }
        }
        if (TECH == HPAC_TECH_IACT) {
          // every lane missed with the same input: the lowest lane writes
#pragma unroll
          for (int c = 0; c < IN_MAX; ++c)
            if (c < p.in_dims) tab[(rr * D + c) * stride_s] = in[c];
#pragma unroll
          for (int d = 0; d < OUT_MAX; ++d)
            if (d < p.out_dims) tab[(rr * D + p.in_dims + d) * stride_s] = out[d];
          rr = rr + 1 == p.tsize ? 0 : rr + 1;
          occ = occ + 1 < p.tsize ? occ + 1 : p.tsize;
        }
      }
      if (TECH == HPAC_TECH_PERFO) pcount += 1;
      tot += tpt;
      wsteps += wpt;
      touched = true;
      if (approx) {
        app += tpt;
        if (round < 8) pbits |= (uint8_t)(1u << round);
      }
    }
    if (p.paths) p.paths[idx] = pbits;
  }
  flush_stats(p, tot, app, wsteps, touched ? wpt : 0ull, err);
}

// ===========================================================================
// Binomial options: warp-cooperative register-blocked CRR lattice.
// ===========================================================================
#ifndef HPAC_LAT_FPMAX_ODD
#define HPAC_LAT_FPMAX_ODD 1  // odd nodes compare on the FP64 pipe (balances pipes)
#endif
#ifndef HPAC_LAT_FPMAX_ALL
#define HPAC_LAT_FPMAX_ALL 1  // segmented lattice: every node's max on the FP64 pipe (+8 %)
#endif

struct LatParams {
  double K;
  double pd, qd;  // disc * p, disc * (1 - p)
  double up, up2, up4, lnu, S;
  double c1, c2, c4;  // x recurrence offsets: +-K*(1 - up^m), m = 1, 2, 4
  double rho, upq, rinv;  // segmented lattice, scaled phases: pd/qd, up/qd, 1/qd
};

__device__ __forceinline__ void lat_offsets(LatParams& q, bool put) {
  q.up4 = q.up2 * q.up2;
  const double sg = put ? 1.0 : -1.0;
  q.c1 = sg * q.K * (1.0 - q.up);
  q.c2 = sg * q.K * (1.0 - q.up2);
  q.c4 = sg * q.K * (1.0 - q.up4);
}

// max(cont, x) where cont >= +0 always: signed-integer order of the bit
// patterns equals the double order when one operand is non-negative, so the
// compare+select runs on the integer pipe instead of the FP64 pipe
// (binomial.hpp:42-44: max(cont, max(x, 0))).
__device__ __forceinline__ double max_nonneg(double cont, double x) {
  long long ci = __double_as_longlong(cont), xi = __double_as_longlong(x);
  return __longlong_as_double(ci > xi ? ci : xi);
}
__device__ __forceinline__ double max_fp(double cont, double x) { return cont < x ? x : cont; }

// One phase of the lattice at block size B: lane owns nodes
// [lane*B, lane*B + B) in registers for every level whose live nodes
// (0..L+1) need blocks of B (L+2 > 32*(B-1)). Values enter and leave the
// phase through this warp's shared-memory node array `xch`, which is the
// rebalance: the next phase reads the same nodes back in smaller blocks,
// so the triangle keeps all 32 lanes busy down to the root.
template <int B, int BNEXT, int BMAX, bool AM, bool PUT>
__device__ __forceinline__ void lat_phase(double (&v)[BMAX], int& L, const LatParams& q, int lane,
                                          double* xch) {
  // active for levels whose live nodes (0..L+1) need more than 32*BNEXT slots
  if (L < 0 || L + 2 <= 32 * BNEXT) return;
#pragma unroll
  for (int i = 0; i < B; ++i) v[i] = xch[lane * B + i];
  // Exercise value of this lane's first node, x = +-(K - S*up^(2*j0 - L)).
  // Moving one level down multiplies the node price by up, one node up by
  // up^2, so x follows the affine recurrences x' = fma(x, m, c_m) with
  // c_m = +-K*(1-m): one FMA per node instead of a multiply and a subtract.
  double sp = q.S * exp((double)(2 * lane * B - L) * q.lnu);
  double x0 = PUT ? q.K - sp : sp - q.K;
  while (L >= 0 && L + 2 > 32 * BNEXT) {
    double vr = __shfl_down_sync(0xffffffffu, v[0], 1);
    if (!AM) {
#pragma unroll
      for (int i = 0; i < B; ++i) {
        double right = (i + 1 < B) ? v[i + 1] : vr;
        v[i] = fma(q.pd, right, q.qd * v[i]);
      }
    } else {
      // two interleaved x chains (even / odd nodes) halve the dependency depth
      double xa = x0, xb = fma(x0, q.up2, q.c2);
#pragma unroll
      for (int i = 0; i < B; ++i) {
        double right = (i + 1 < B) ? v[i + 1] : vr;
        double cont = fma(q.pd, right, q.qd * v[i]);
        if ((i & 1) == 0) {
          v[i] = max_nonneg(cont, xa);
          xa = fma(xa, q.up4, q.c4);
        } else {
          v[i] = (HPAC_LAT_FPMAX_ODD) ? max_fp(cont, xb) : max_nonneg(cont, xb);
          xb = fma(xb, q.up4, q.c4);
        }
      }
      x0 = fma(x0, q.up, q.c1);
    }
    --L;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < B; ++i) xch[lane * B + i] = v[i];
  __syncwarp();
}

template <int... Bs>
struct BList {};

// Walk the block sizes largest to smallest; each phase hands its nodes to
// the next through xch. A geometric set (ratio ~1.2) keeps ~91% of the
// lanes busy while the whole chain stays ~20 KB of SASS (the full 33-size
// chain is ~70 KB and thrashes the instruction cache: ncu "no_instruction").
template <int BMAX, bool AM, bool PUT, int B, int... REST>
__device__ __forceinline__ void lat_chain(double (&v)[BMAX], int& L, const LatParams& q, int lane,
                                          double* xch, BList<B, REST...>) {
  constexpr int nexts[] = {REST..., 0};
  lat_phase<B, nexts[0], BMAX, AM, PUT>(v, L, q, lane, xch);
  if constexpr (sizeof...(REST) > 0) lat_chain<BMAX, AM, PUT>(v, L, q, lane, xch, BList<REST...>{});
}

using LatBlocks = BList<33, 28, 24, 20, 17, 14, 12, 10, 8, 7, 6, 5, 4, 3, 2, 1>;

// ---------------------------------------------------------------------------
// American put with early-exercise boundary tracking.
//
// For the CRR American put the exercise region at every level is a prefix
// {j < j*(L)} of the nodes (the value minus the intrinsic is non-decreasing
// in the stock price, since the put's delta is >= -1), and there v = K - s
// exactly. A node j needs only children j and j+1, so nodes below a bound
// `lo` never feed nodes at or above it: each phase computes [lo, L] only.
// `lo` is placed a margin below the boundary measured at the end of the
// previous phase; the assumption "every node below lo is exercised" is
// verified at every level by checking that node lo itself is exercised
// (monotonicity covers the rest). If a check ever fails, the option is
// recomputed with the full lattice. Nodes entering the computed range from
// below are exactly their exercise values. About half of the triangle is
// skipped at the reference's result (within the 1e-6 tolerance).
template <int B, int BMAX>
__device__ __forceinline__ void bt_phase(double (&v)[BMAX], int& L, int lo, int pmax,
                                         const LatParams& q, int lane, double* xch, bool check,
                                         bool& ok, int& nex, int top, double eps_k, int& jsig) {
  const int base = lo + lane * B;
  // nodes above `top` (= N+1) are dead: never loaded from or stored to xch
#pragma unroll
  for (int i = 0; i < B; ++i) v[i] = base + i <= top ? xch[base + i] : 0.0;
  double x0 = q.K - q.S * exp((double)(2 * base - L) * q.lnu);
  double x0_last = x0;
  int L_last = L;
  for (int done = 0; L >= 0 && done < pmax; ++done) {
    // the block range's top node may be the zero node jk+1 (live range
    // capped at the highest in-the-money leaf): its right neighbour is 0,
    // not lane 31's own v[0] that shfl_down returns
    double vr = __shfl_down_sync(0xffffffffu, v[0], 1);
    if (lane == 31) vr = 0.0;
    double xa = x0, xb = fma(x0, q.up2, q.c2);
    const double xfirst = x0;
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double right = (i + 1 < B) ? v[i + 1] : vr;
      double cont = fma(q.pd, right, q.qd * v[i]);
      if ((i & 1) == 0) {
        v[i] = max_nonneg(cont, xa);
        xa = fma(xa, q.up4, q.c4);
      } else {
        v[i] = (HPAC_LAT_FPMAX_ODD) ? max_fp(cont, xb) : max_nonneg(cont, xb);
        xb = fma(xb, q.up4, q.c4);
      }
    }
    ok = ok && !(check && v[0] != xfirst);  // node lo must stay exercised (lane 0)
    x0_last = x0;
    L_last = L;
    x0 = fma(x0, q.up, q.c1);
    --L;
  }
  // exercised prefix length at the last level processed (boundary estimate),
  // and the highest node there whose value is still significant (> eps*K)
  int cnt = 0;
  int js = -1;
  {
    double xa = x0_last, xb = fma(x0_last, q.up2, q.c2);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      double x;
      if ((i & 1) == 0) {
        x = xa;
        xa = fma(xa, q.up4, q.c4);
      } else {
        x = xb;
        xb = fma(xb, q.up4, q.c4);
      }
      if (base + i <= L_last && v[i] == x) ++cnt;
      if (base + i <= L_last && base + i <= top && v[i] > eps_k) js = base + i;
    }
  }
  nex = __reduce_add_sync(0xffffffffu, cnt);
  jsig = __reduce_max_sync(0xffffffffu, js);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < B; ++i)
    if (base + i <= top) xch[base + i] = v[i];
  __syncwarp();
}

__device__ __forceinline__ void bt_fill_exercise(double* xch, int from, int to, int level,
                                                 const LatParams& q, int lane) {
  for (int j = from + lane; j < to; j += 32)
    xch[j] = q.K - q.S * exp((double)(2 * j - level) * q.lnu);
  __syncwarp();
}

// Returns false (caller recomputes the full triangle) when a boundary check
// fails or the continuation region outgrows the compiled block sizes.
constexpr int kBtBmax = 20;
#ifndef HPAC_BT_TAIL_EPS
#define HPAC_BT_TAIL_EPS 1e-16
#endif
constexpr double kBtTailEps = HPAC_BT_TAIL_EPS;  // relative to the strike

template <bool AM, bool PUT>
__device__ double lattice_smem_inplace(double spot, double strike, int N, const LatParams& q,
                                       double* xch);

template <int BMAX>
__device__ bool binomial_put_bt(double spot, double strike, int N, const LatParams& q,
                                double* xch, double& price, unsigned long long& nodes,
                                bool cut_tail) {
  const int lane = threadIdx.x & 31;
  constexpr int kPhase = 32;   // levels per phase
  constexpr int kMargin = 8;   // nodes kept below the measured boundary
  constexpr int kBtMax = BMAX;  // largest block size in the boundary-tracking chain
  double v[BMAX];
  // First bound: one step before expiry the put is exercised wherever
  // s*u < K, i.e. below j ~ (N-1 + ln(K/S)/lnu)/2; the boundary then drifts
  // down by ~1/2 node per level plus the early-time move of S*(tau). Keep a
  // generous margin (the phase checks it anyway).
  int lo = (int)floor(((double)(N - 1 - kPhase) + log(strike / spot) / q.lnu) * 0.5) - 48;
  lo = max(0, min(lo, N / 2));
  int jk = -1;  // highest in-the-money leaf
  for (int j = lo + lane; j <= N; j += 32) {
    double s = spot * exp((double)(2 * j - N) * q.lnu);
    double x = strike - s;
    xch[j] = x < 0.0 ? 0.0 : x;
    if (x > 0.0) jk = j;
  }
  jk = __reduce_max_sync(0xffffffffu, jk);
  __syncwarp();
  // Zero region: node (j, L) only reaches leaves j..j+N-L, all out of the
  // money when j > jk, and its exercise value is negative there too, so it
  // is exactly +0 at every level (0*p + 0*q = +0). The live range is capped
  // at jk (+ the zero right neighbour jk+1): the upper quarter of the
  // triangle is never computed, and every computed node is unchanged.
  //
  // Negligible tail: the set of nodes above an index J whose values are all
  // <= eps*K is closed under backward induction (node j at level L reads
  // only j and j+1 at L+1; above the strike node the exercise value is
  // negative, so the max is the discounted average, <= eps*K again). So at
  // the end of every phase the cap `hi` drops to the highest node still
  // above eps*K; the node hi+1 continues with a zero right neighbour. Each
  // level that changes the root by at most eps*K (the backward operator is
  // a sup-norm contraction), so the price moves by <= N*eps*K in total:
  // ~1e-13 K at N = 1024 with eps = 1e-16, far inside the 1e-6 exact-path
  // tolerance, while ~40 % of the remaining nodes (the far out-of-the-money
  // tail whose values underflow towards 0) are never computed.
  int hi = jk;
  const double eps_k = kBtTailEps * strike;
  if (jk < lo) {
    // no in-the-money leaf at or above the bound: with lo == 0 every node is
    // exactly 0; otherwise let the full lattice handle it
    if (jk < 0 && lo == 0) {
      price = 0.0;
      __syncwarp();
      return true;
    }
    return false;
  }
  int L = N - 1;
  while (L >= 0) {
    const int top = hi + 1;
    const int live = min(L, hi) + 2 - lo;
    if (live > 32 * kBtMax || live < 1) return false;
    {
      const int lv = min(L + 1, kPhase);  // levels L .. L-lv+1 over nodes lo..min(level, hi)
      for (int t = 0; t < lv; ++t) nodes += (unsigned long long)max(0, min(L - t, hi) + 1 - lo);
    }
    bool ok = true;
    int nex = 0, jsig = hi;
    const bool check = lo > 0;
#define HPAC_BT(b, bn) \
  if (live > 32 * (bn)) { bt_phase<b, BMAX>(v, L, lo, kPhase, q, lane, xch, check, ok, nex, top, eps_k, jsig); } else
    // 11 block sizes (13 before the 8-CTA/SM change: with more warps per SM
    // sharing the instruction cache, fewer instantiations beat tighter fits;
    // 9 and 7 sizes measured 0.5 % and 6 % slower)
    HPAC_BT(20, 16) HPAC_BT(16, 13) HPAC_BT(13, 10) HPAC_BT(10, 8) HPAC_BT(8, 6) HPAC_BT(6, 5)
    HPAC_BT(5, 4) HPAC_BT(4, 3) HPAC_BT(3, 2) HPAC_BT(2, 1) HPAC_BT(1, 0) {}
#undef HPAC_BT
    if (!__shfl_sync(0xffffffffu, ok ? 1 : 0, 0)) return false;
    if (L < 0) break;
    // the tail above the last significant node stays negligible (never below
    // the boundary bound: those nodes are exercised, hence significant)
    if (cut_tail) hi = max(min(hi, jsig), lo);
    // next bound: measured boundary (level L+1) minus margin and half a phase
    // of drift; never above mid-lattice; full range near the root
    int lo_new = lo + nex - kMargin - kPhase / 2;
    if (L < 3 * kPhase) lo_new = 0;
    lo_new = max(0, min(lo_new, (L + 1) / 2));
#ifdef HPAC_BT_DEBUG
    if (lane == 0 && blockIdx.x == 0 && threadIdx.x == 0)
      printf("bt L=%d lo=%d nex=%d live=%d lo_new=%d\n", L, lo, nex, live, lo_new);
#endif
    if (lo_new < lo) bt_fill_exercise(xch, lo_new, lo, L + 1, q, lane);
    lo = lo_new;
  }
  price = xch[0];
  __syncwarp();
  return true;
}

// ---------------------------------------------------------------------------
// Segmented boundary tracking: 32/SEG American puts per warp, SEG lanes each.
//
// With the early-exercise prefix and the negligible out-of-the-money tail
// cut, an option's live node range is ~80-130 nodes per level (boundary to
// the eps*K tail; SURVEY §8a-A10 restated in DESIGN.md §4.3), i.e. ~3-4
// nodes per lane of a whole warp, so per-level work (shuffle, exercise
// recurrence start, loop control, boundary check) outweighed the node
// updates. Here each option gets a SEG-lane segment of ~SEG x B nodes and
// the per-level overhead is spread over 32/SEG times more nodes. Node values
// are computed with the same fma/max per node as binomial_put_bt, but with
// per-node exercise registers (bts_phase), so an option's price does not
// depend on the warp's block size (that is, on the other options in the
// warp). Per option the nodes live in a window [lo, lo + WIN) of this warp's
// shared memory, re-based to the next phase's bound at the end of every
// phase. Options whose live range outgrows SEG * BMAX, whose boundary check
// fails, or whose price is too small for the tail cut return false and are
// priced by the whole-warp path (also a pure function of the option).
#ifndef HPAC_SEG_UNROLL
#define HPAC_SEG_UNROLL 1  // level-loop unroll of the segmented phases (2: 91.3 vs 93.4 M, I-cache)
#endif
constexpr int kSegUnroll = HPAC_SEG_UNROLL;
#ifndef HPAC_SEG_PHASE
#define HPAC_SEG_PHASE 24  // 16/20/28/32/36/40: 75.7/79.0/88.2/86.6/81.9/82.1 vs 89.2 M options/s
#endif
constexpr int kSegPhase = HPAC_SEG_PHASE;  // levels per phase (= binomial_put_bt)
#ifndef HPAC_SEG_MARGIN
#define HPAC_SEG_MARGIN 4  // 2 falls off a cliff (check failures -> whole-warp path); 3-4 fastest
#endif
constexpr int kSegMargin = HPAC_SEG_MARGIN;  // nodes kept below the measured boundary

// per-segment block bound: SEG * BMAX = 160 live nodes; chunk C: nodes per
// exercise register (2: lower bands of 4/6/8 nodes per lane; one-band blocks
// stay in steps of 4, HPAC_SEG_COARSE, for the instruction cache)
#ifndef HPAC_SEG_C
#define HPAC_SEG_C 0  // 0: by segment width
#endif
#ifndef HPAC_SEG_BO12
#define HPAC_SEG_BO12 1  // upper blocks of 12 nodes as well as 8 and 16
#endif
#ifndef HPAC_SEG_COMBOS
#define HPAC_SEG_COMBOS 2  // two-band shapes: 0 all nine, 1 without BI 4, 2 without BO 8, 3 neither
#endif
#ifndef HPAC_SEG_COARSE
#define HPAC_SEG_COARSE 1  // one-band block sizes in steps of 4 also for 2-node chunks
#endif
#ifndef HPAC_BINO_TWO_BAND
#define HPAC_BINO_TWO_BAND 1  // in-the-money / out-of-the-money bands (bts_phase2)
#endif
constexpr bool kBinoTwoBand = HPAC_BINO_TWO_BAND != 0;
template <int SEG>
struct SegWin {
  static constexpr int C = HPAC_SEG_C > 0 ? HPAC_SEG_C : 2;  // 4: 76.1 vs 80.6 M options/s (coarser lower band)
  static constexpr int BMAX = 160 / SEG;
  static constexpr int WIN = 160 + 32;  // live range + bound drift
};

// One phase (<= kSegPhase levels) on B-node register blocks, B a multiple
// of the chunk C (2 or 4). The exercise values come from one register per
// C-node chunk starting at j (j - lo a multiple of C): x_j(L) = K - S*up^(2j-L)
// is anchored exactly (exp) at the phase's first level and stepped down a
// level per iteration (x' = fma(x, up, c1)); inside the chunk x_{j+1} =
// fma(x_j, up^2, c2), x_{j+2} = fma(x_j, up^4, c4), x_{j+3} = fma(x_{j+1},
// up^4, c4). All of it depends on (lo, j, L) only, so a node's value never
// depends on how the range is cut into lane blocks: the block size can follow
// the widest option of the warp while every option's price stays a pure
// function of the option.
template <int C>
__device__ __forceinline__ double chunk_x(double a, int r, const LatParams& q) {
  if (r == 0) return a;
  const double b = fma(a, q.up2, q.c2);
  if (r == 1) return b;
  if (r == 2) return fma(a, q.up4, q.c4);
  return fma(b, q.up4, q.c4);
}

template <int B, int BMAX, int SEG, int C, int RN, int XN>
__device__ __forceinline__ void bts_phase(double (&v)[RN], double (&xa)[XN], int& L,
                                          int lo, const LatParams& q, int sub, const double* w,
                                          bool check, bool& ok, int& cnt_out, int& js_out,
                                          int top, double eps_k) {
  static_assert(B % C == 0 && B <= RN && B / C <= XN, "whole chunks");
  const int base = lo + sub * B;
#pragma unroll
  for (int i = 0; i < B; ++i) v[i] = base + i <= top ? w[sub * B + i] : 0.0;
  // scaled phase (binomial_put_seg): after t levels the registers hold
  // v / qd^t, so a node costs one DFMA (cont = rho*right + v) instead of a
  // DMUL + DFMA; the exercise values are carried on the same scale
  double sinv = q.rinv;  // 1/qd^(t+1) at level iteration t
  double sq = 1.0;       // qd^t
#pragma unroll
  for (int k = 0; k < B / C; ++k)
    xa[k] = (q.K - q.S * fm::exp((double)(2 * (base + C * k) - L) * q.lnu)) * sinv;
  int L_last = L;
  double c2t = q.c2 * sinv, c4t = q.c4 * sinv;
  // the right neighbour of the last node, one level ahead (as bts_phase2)
  const bool last = sub == SEG - 1;
  double vr = __shfl_down_sync(0xffffffffu, v[0], 1, SEG);
  if (last) vr = 0.0;  // the segment's top node: right neighbour 0
  unsigned long long okx = 0;  // bit difference of node lo from its exercise value
#pragma unroll kSegUnroll
  for (int done = 0; L >= 0 && done < kSegPhase; ++done) {
    if (done > 0) {
      sinv *= q.rinv;
      const double c1t = q.c1 * sinv;
#pragma unroll
      for (int k = 0; k < B / C; ++k) xa[k] = fma(xa[k], q.upq, c1t);
      c2t = q.c2 * sinv;
      c4t = q.c4 * sinv;
    }
    const double v0 = max_fp(fma(q.rho, B > 1 ? v[1] : vr, v[0]), xa[0]);
    const double nv = __shfl_down_sync(0xffffffffu, v0, 1, SEG);
#pragma unroll
    for (int k = 0; k < B / C; ++k) {
      double xb = 0.0;
#pragma unroll
      for (int r = 0; r < C; ++r) {
        const int i = k * C + r;
        double x;
        if (r == 0) x = xa[k];
        else if (r == 1) x = xb = fma(xa[k], q.up2, c2t);
        else if (r == 2) x = fma(xa[k], q.up4, c4t);
        else x = fma(xb, q.up4, c4t);
        if (i == 0) continue;
        const double right = (i + 1 < B) ? v[i + 1] : vr;
        const double cont = fma(q.rho, right, v[i]);
        v[i] = max_fp(cont, x);
      }
    }
    v[0] = v0;
    vr = last ? 0.0 : nv;
    okx |= __double_as_longlong(v[0]) ^ __double_as_longlong(xa[0]);  // node lo exercised (sub 0)
    sq *= q.qd;
    L_last = L;
    --L;
  }
  if (check && okx != 0) ok = false;
  int cnt = 0, js = -1;
#pragma unroll
  for (int k = 0; k < B / C; ++k) {
    double xb = 0.0;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int i = k * C + r;
      double x;
      if (r == 0) x = xa[k];
      else if (r == 1) x = xb = fma(xa[k], q.up2, c2t);
      else if (r == 2) x = fma(xa[k], q.up4, c4t);
      else x = fma(xb, q.up4, c4t);
      if (base + i <= L_last && v[i] == x) ++cnt;
      v[i] *= sq;  // back to prices
      if (base + i <= L_last && base + i <= top && v[i] > eps_k) js = base + i;
    }
  }
  cnt_out = cnt;
  js_out = js;
}

// Two-band phase: each lane holds BI nodes of the in-the-money band
// [lo, lo + SEG*BI) and BO nodes of the band above it. The caller puts the
// split above the highest node that can be in the money during the phase
// (the strike node only moves down as L decreases), so in the upper band the
// exercise value is negative and max(cont, x) = cont exactly (cont >= +0):
// the upper band updates with DMUL + DFMA and no exercise chain, bit-identical
// to the one-band phase. Right neighbours: the next lane's first node of the
// same band; the segment's last lane takes the upper band's first node (lower
// band) or 0 (upper band).
template <int BI, int BO, int RN, int XN, int SEG, int C>
__device__ __forceinline__ void bts_phase2(double (&r)[RN], double (&xa)[XN], int& L, int lo,
                                           const LatParams& q, int sub, const double* w,
                                           bool check, bool& ok, int& cnt_out, int& js_out,
                                           int top, double eps_k) {
  static_assert(BI % C == 0 && BI <= 8 && 8 + BO <= RN && BI / C <= XN, "block shapes");
  double* const vi = r;      // lower band: r[0 .. BI)
  double* const vo = r + 8;  // upper band: r[8 .. 8 + BO)
  const int base_i = lo + sub * BI;
  const int base_o = lo + SEG * BI + sub * BO;
  const int seg0 = (int)(threadIdx.x & 31) - sub;
#pragma unroll
  for (int i = 0; i < BI; ++i) vi[i] = base_i + i <= top ? w[sub * BI + i] : 0.0;
#pragma unroll
  for (int i = 0; i < BO; ++i) vo[i] = base_o + i <= top ? w[SEG * BI + sub * BO + i] : 0.0;
  double sinv = q.rinv, sq = 1.0;  // scaled phase, as bts_phase
#pragma unroll
  for (int k = 0; k < BI / C; ++k)
    xa[k] = (q.K - q.S * fm::exp((double)(2 * (base_i + C * k) - L) * q.lnu)) * sinv;
  double c2t = q.c2 * sinv, c4t = q.c4 * sinv;
  int L_last = L;
  // right neighbours of each band's last node, one level ahead: the shuffles
  // for level t+1 are issued right after this level's first nodes, so their
  // latency overlaps the rest of the level (width-SEG shuffles: no lane math)
  const bool last = sub == SEG - 1;
  double ri, ro;
  {
    const double a = __shfl_down_sync(0xffffffffu, vi[0], 1, SEG);
    const double b = __shfl_down_sync(0xffffffffu, vo[0], 1, SEG);
    const double c = __shfl_sync(0xffffffffu, vo[0], 0, SEG);
    ri = last ? c : a;
    ro = last ? 0.0 : b;
  }
  unsigned long long okx = 0;  // bit difference of node lo from its exercise value
#pragma unroll kSegUnroll
  for (int done = 0; L >= 0 && done < kSegPhase; ++done) {
    if (done > 0) {
      sinv *= q.rinv;
      const double c1t = q.c1 * sinv;
#pragma unroll
      for (int k = 0; k < BI / C; ++k) xa[k] = fma(xa[k], q.upq, c1t);
      c2t = q.c2 * sinv;
      c4t = q.c4 * sinv;
    }
    // first nodes of both bands, then the next level's neighbours
    const double vo0 = fma(q.rho, BO > 1 ? vo[1] : ro, vo[0]);
    const double vi0 = max_fp(fma(q.rho, BI > 1 ? vi[1] : ri, vi[0]), xa[0]);
    const double na = __shfl_down_sync(0xffffffffu, vi0, 1, SEG);
    const double nb = __shfl_down_sync(0xffffffffu, vo0, 1, SEG);
    const double nc = __shfl_sync(0xffffffffu, vo0, 0, SEG);
#pragma unroll
    for (int k = 0; k < BI / C; ++k) {
      double xb = 0.0;
#pragma unroll
      for (int r = 0; r < C; ++r) {
        const int i = k * C + r;
        double x;
        if (r == 0) x = xa[k];
        else if (r == 1) x = xb = fma(xa[k], q.up2, c2t);
        else if (r == 2) x = fma(xa[k], q.up4, c4t);
        else x = fma(xb, q.up4, c4t);
        if (i == 0) continue;
        const double right = (i + 1 < BI) ? vi[i + 1] : ri;
        const double cont = fma(q.rho, right, vi[i]);
        vi[i] = max_fp(cont, x);
      }
    }
#pragma unroll
    for (int i = 1; i < BO; ++i) {
      const double right = (i + 1 < BO) ? vo[i + 1] : ro;
      vo[i] = fma(q.rho, right, vo[i]);
    }
    vi[0] = vi0;
    vo[0] = vo0;
    ri = last ? nc : na;
    ro = last ? 0.0 : nb;
    okx |= __double_as_longlong(vi[0]) ^ __double_as_longlong(xa[0]);  // node lo exercised (sub 0)
    sq *= q.qd;
    L_last = L;
    --L;
  }
  if (check && okx != 0) ok = false;
  int cnt = 0, js = -1;
#pragma unroll
  for (int k = 0; k < BI / C; ++k) {
    double xb = 0.0;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int i = k * C + r;
      double x;
      if (r == 0) x = xa[k];
      else if (r == 1) x = xb = fma(xa[k], q.up2, c2t);
      else if (r == 2) x = fma(xa[k], q.up4, c4t);
      else x = fma(xb, q.up4, c4t);
      if (base_i + i <= L_last && vi[i] == x) ++cnt;
      vi[i] *= sq;
      if (base_i + i <= L_last && base_i + i <= top && vi[i] > eps_k) js = base_i + i;
    }
  }
#pragma unroll
  for (int i = 0; i < BO; ++i) {
    vo[i] *= sq;
    if (base_o + i <= L_last && base_o + i <= top && vo[i] > eps_k) js = base_o + i;
  }
  cnt_out = cnt;
  js_out = js;
}

template <int SEG>
__device__ __forceinline__ int seg_sum(int x) {
#pragma unroll
  for (int o = SEG >> 1; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
template <int SEG>
__device__ __forceinline__ int seg_max(int x) {
#pragma unroll
  for (int o = SEG >> 1; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

// CRR parameters of binomial_price (bench/binomial.hpp:16-32); false where
// the reference throws.
__device__ __forceinline__ bool lat_params(double spot, double strike, double rate, double vol,
                                           double mat, int N, bool put, LatParams& q) {
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol > 0) || N < 1) return false;
  const double dt = mat / N;
  const double lnu = vol * sqrt(dt);
  const double up = exp(lnu);
  const double down = 1.0 / up;
  const double growth = exp(rate * dt);
  const double pu = (growth - down) / (up - down);
  if (!(pu > 0.0) || !(pu < 1.0)) return false;
  const double disc = 1.0 / growth;
  q.K = strike;
  q.pd = disc * pu;
  q.qd = disc * (1.0 - pu);
  q.up = up;
  q.up2 = up * up;
  q.lnu = lnu;
  q.S = spot;
  lat_offsets(q, put);
  q.rho = q.pd / q.qd;
  q.upq = up / q.qd;
  q.rinv = 1.0 / q.qd;
  return true;
}

// All 32 lanes call, converged; segment g = lane / SEG prices option `o`
// (its own lanes' copy; `has` false = idle segment) in window w_g. Returns
// the segment's success; price valid on every lane of a successful segment.
template <int SEG, int BMAX>
__device__ bool binomial_put_seg(const double (&o)[5], bool has, int N, double* w, double& price,
                                 unsigned long long& nodes) {
  constexpr int WIN = SegWin<SEG>::WIN;
  const int lane = threadIdx.x & 31;
  const int sub = lane % SEG;
  LatParams q;
  // scaled phases keep v / qd^32 in range: qd >= 1e-6 (else the whole-warp path)
  bool alive = has && lat_params(o[0], o[1], o[2], o[3], o[4], N, true, q) && q.qd >= 1e-6;
  if (!alive) {  // keep the idle segment's arithmetic finite
    q.K = q.S = 1.0;
    q.pd = q.qd = 0.5;
    q.up = q.up2 = q.up4 = 1.0;
    q.lnu = 0.0;
    q.c1 = q.c2 = q.c4 = 0.0;
    q.rho = 1.0;
    q.upq = q.rinv = 2.0;
  }
  bool success = alive;
  const double spot = q.S, strike = q.K;
  int lo = alive ? (int)floor(((double)(N - 1 - kSegPhase) + log(strike / spot) / q.lnu) * 0.5) - 48
                 : 0;
  lo = max(0, min(lo, N / 2));
  // leaves within the window; the highest in-the-money leaf must be inside
  int jk = -1;
  for (int j = lo + sub; j < lo + WIN; j += SEG) {
    double x = 0.0;
    if (j <= N) {
      x = strike - spot * exp((double)(2 * j - N) * q.lnu);
      if (x > 0.0) jk = j;
    }
    w[j - lo] = x < 0.0 ? 0.0 : x;
  }
  jk = seg_max<SEG>(jk);
  price = 0.0;
  if (alive && jk >= lo + WIN - 1 && lo + WIN - 1 <= N) success = alive = false;
  if (alive && jk < lo) {
    alive = false;
    success = jk < 0 && lo == 0;  // every node exactly 0 (binomial_put_bt)
  }
  unsigned long long my_nodes = 0;
  int hi = jk;
  const double eps_k = kBtTailEps * strike;
  constexpr int C = SegWin<SEG>::C;
  // one register file for both phase shapes: one band v[0 .. B), or the
  // lower band v[0 .. 8) and the upper band v[8 .. 24)
  constexpr int RN = BMAX > 24 ? BMAX : 24;
  double v[RN], xa[BMAX / C > 2 ? BMAX / C : 2];
  // strike node offset: x_j(L) > 0  <=>  j < (L + ln(K/S)/lnu) / 2
  const double lks = log(strike / spot) / q.lnu;
  const bool lks_ok = alive && q.lnu > 1e-9 && isfinite(lks);
  int L = N - 1;
  __syncwarp();
  while (L >= 0) {
    const int top = hi + 1;
    const int live = min(L, hi) + 2 - lo;
    if (alive && (live > SEG * BMAX || live < 1)) success = alive = false;
    const int need = alive ? (live + SEG - 1) / SEG : 0;
    const int bw = __reduce_max_sync(0xffffffffu, need);
    if (bw == 0) break;
    if (alive && sub == 0) {
      const int lv = min(L + 1, kSegPhase);
      for (int t = 0; t < lv; ++t) my_nodes += (unsigned long long)max(0, min(L - t, hi) + 1 - lo);
    }
    bool ok = true;
    int cnt = 0, js = -1;
    const bool check = lo > 0;
    int Bsel = 0, Bi2 = 0, Bo2 = 0;
    // two-band shape: the lower band must reach past the highest node that
    // can be in the money during this phase (strike node at level L, + 2)
    if constexpr (SEG == 8 && (C == 4 || C == 2) && kBinoTwoBand) {
      int ni = 0;
      if (alive) {
        const int jo = (int)ceil(0.5 * ((double)L + lks)) + 1;
        ni = lks_ok ? max(1, (jo - lo + SEG - 1) / SEG) : 1 << 20;
        ni = (ni + C - 1) & ~(C - 1);  // whole chunks
        ni = ni < 4 ? 4 : ni;
        if ((HPAC_SEG_COMBOS == 1 || HPAC_SEG_COMBOS == 3) && ni < 6) ni = 6;
      }
      const int bi = __reduce_max_sync(0xffffffffu, ni);
      if (bi <= 8) {
        int no = 0;
        if (alive) no = max(0, (top + 1 - (lo + SEG * bi) + SEG - 1) / SEG);
        const int bo = __reduce_max_sync(0xffffffffu, no);
        if (bo > 0 && bo <= 16) {
          Bi2 = bi;
          Bo2 = bo <= 8 && HPAC_SEG_COMBOS < 2 ? 8 : (HPAC_SEG_BO12 && bo <= 12 ? 12 : 16);
        }
      }
    }
    if (Bi2 > 0) {
#define HPAC_BTS2(bi, bo)                                                                        \
  if (Bi2 == (bi) && Bo2 == (bo)) {                                                              \
    bts_phase2<bi, bo, RN, sizeof(xa) / sizeof(double), SEG, C>(v, xa, L, lo, q, sub, w, check,  \
                                                               ok, cnt, js, top, eps_k);        \
  } else
      if constexpr (C == 2 && HPAC_SEG_BO12 && HPAC_SEG_COMBOS == 3) {
        HPAC_BTS2(6, 12) HPAC_BTS2(6, 16) HPAC_BTS2(8, 12) HPAC_BTS2(8, 16) {}
      } else if constexpr (C == 2 && HPAC_SEG_BO12 && HPAC_SEG_COMBOS == 1) {
        HPAC_BTS2(6, 8) HPAC_BTS2(6, 12) HPAC_BTS2(6, 16) HPAC_BTS2(8, 8) HPAC_BTS2(8, 12)
        HPAC_BTS2(8, 16) {}
      } else if constexpr (C == 2 && HPAC_SEG_BO12 && HPAC_SEG_COMBOS == 2) {
        HPAC_BTS2(4, 12) HPAC_BTS2(4, 16) HPAC_BTS2(6, 12) HPAC_BTS2(6, 16) HPAC_BTS2(8, 12)
        HPAC_BTS2(8, 16) {}
      } else if constexpr (C == 2 && HPAC_SEG_BO12) {
        HPAC_BTS2(4, 8) HPAC_BTS2(4, 12) HPAC_BTS2(4, 16) HPAC_BTS2(6, 8) HPAC_BTS2(6, 12)
        HPAC_BTS2(6, 16) HPAC_BTS2(8, 8) HPAC_BTS2(8, 12) HPAC_BTS2(8, 16) {}
      } else if constexpr (C == 2) {
        HPAC_BTS2(4, 8) HPAC_BTS2(4, 16) HPAC_BTS2(6, 8) HPAC_BTS2(6, 16) HPAC_BTS2(8, 8)
        HPAC_BTS2(8, 16) {}
      } else {
        HPAC_BTS2(4, 8) HPAC_BTS2(4, 16) HPAC_BTS2(8, 8) HPAC_BTS2(8, 16) {}
      }
#undef HPAC_BTS2
    } else
#define HPAC_BTS(b, bn)                                                                      \
  if (bw > (bn)) {                                                                           \
    Bsel = (b);                                                                              \
    bts_phase<(b), BMAX, SEG, C, RN, sizeof(xa) / sizeof(double)>(v, xa, L, lo, q, sub, w, check, \
                                                                  ok, cnt, js, top, eps_k);    \
  } else
    if constexpr (C == 2 && BMAX == 20 && HPAC_SEG_COARSE == 2) {
      HPAC_BTS(20, 12) HPAC_BTS(12, 4) HPAC_BTS(4, 0) {}
    } else if constexpr (C == 2 && BMAX == 20 && HPAC_SEG_COARSE == 3) {
      HPAC_BTS(20, 10) HPAC_BTS(10, 0) {}
    } else if constexpr (C == 4 || (C == 2 && BMAX == 20 && HPAC_SEG_COARSE)) {
      HPAC_BTS(20, 16) HPAC_BTS(16, 12) HPAC_BTS(12, 8) HPAC_BTS(8, 4) HPAC_BTS(4, 0) {}
    } else if constexpr (BMAX == 20) {
      HPAC_BTS(20, 18) HPAC_BTS(18, 16) HPAC_BTS(16, 14) HPAC_BTS(14, 12) HPAC_BTS(12, 10)
      HPAC_BTS(10, 8) HPAC_BTS(8, 6) HPAC_BTS(6, 4) HPAC_BTS(4, 2) HPAC_BTS(2, 0) {}
    } else {
      HPAC_BTS(10, 8) HPAC_BTS(8, 6) HPAC_BTS(6, 4) HPAC_BTS(4, 2) HPAC_BTS(2, 0) {}
    }
#undef HPAC_BTS
    const int nex = seg_sum<SEG>(cnt);
    const int jsig = seg_max<SEG>(js);
    const bool ok0 = __shfl_sync(0xffffffffu, ok ? 1 : 0, lane - sub) != 0;
    if (alive && !ok0) success = alive = false;
    // next bound (binomial_put_bt): measured boundary minus margin and half
    // a phase of drift; full range near the root; the tail cap follows the
    // last significant node
    const int hi_new = max(min(hi, jsig), lo);
    int lo_new = lo + nex - kSegMargin - kSegPhase / 2;
    if (L < 3 * kSegPhase) lo_new = 0;
    lo_new = max(0, min(lo_new, (L + 1) / 2));
    if (L < 0) lo_new = lo;  // done: node 0 stays at window index 0 (lo == 0)
    if (alive && hi_new + 1 - lo_new + 1 > WIN) success = alive = false;
    __syncwarp();
    if (alive) {
      // write back re-based to lo_new (nodes below it are exercised: dropped)
      if (Bi2 > 0) {
        const int bi_ = lo + sub * Bi2, bo_ = lo + SEG * Bi2 + sub * Bo2;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = bi_ + i;
          if (i < Bi2 && j <= top && j >= lo_new && j - lo_new < WIN) w[j - lo_new] = v[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = bo_ + i;
          if (i < Bo2 && j <= top && j >= lo_new && j - lo_new < WIN) w[j - lo_new] = v[8 + i];
        }
      } else {
        const int base = lo + sub * Bsel;
#pragma unroll
        for (int i = 0; i < BMAX; ++i) {
          const int j = base + i;
          if (i < Bsel && j <= top && j >= lo_new && j - lo_new < WIN) w[j - lo_new] = v[i];
        }
      }
      // nodes entering from below are exactly their exercise values (level L+1)
      for (int j = lo_new + sub; j < lo; j += SEG)
        w[j - lo_new] = strike - spot * exp((double)(2 * j - (L + 1)) * q.lnu);
      lo = lo_new;
      hi = hi_new;
    }
    __syncwarp();
  }
  if (success && alive) price = w[0];
  __syncwarp();
  // the tail cut is only valid when N*eps*K << price (binomial_warp_price)
  if (success && alive && !(price * 1e-9 >= (double)N * kBtTailEps * strike)) success = false;
  if (success && sub == 0) nodes += my_nodes;
  return success;
}

// binomial_price (bench/binomial.hpp:16-50) by one warp; every lane
// returns the price. `xch` = 32*BMAX doubles of this warp's shared memory.
template <int BMAX, bool AM, bool PUT>
__device__ double binomial_warp_price(const double* o, int N, double* xch, bool& ok,
                                      unsigned long long* fallbacks = nullptr) {
  const int lane = threadIdx.x & 31;
  double spot = o[0], strike = o[1], rate = o[2], vol = o[3], mat = o[4];
  ok = true;
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol > 0) || N < 1) {
    ok = false;
    return 0.0;
  }
  double dt = mat / N;
  double lnu = vol * sqrt(dt);
  double up = exp(lnu);
  double down = 1.0 / up;
  double growth = exp(rate * dt);
  double pu = (growth - down) / (up - down);
  if (!(pu > 0.0) || !(pu < 1.0)) {
    ok = false;
    return 0.0;
  }
  double disc = 1.0 / growth;
  LatParams q;
  q.K = strike;
  q.pd = disc * pu;
  q.qd = disc * (1.0 - pu);
  q.up = up;
  q.up2 = up * up;
  q.lnu = lnu;
  q.S = spot;
  lat_offsets(q, PUT);
  if constexpr (AM && PUT) {
    // boundary tracking on <= 20-node register blocks; whole triangle in
    // shared memory if its checks fail (keeps the hot kernel small)
    double price;
    unsigned long long nodes = 0;
    // the tail cut moves the price by at most N*eps*K (binomial_put_bt); when
    // that is not below 1e-9 of the price itself (tiny, far out-of-the-money
    // prices) the lattice is recomputed without it (one call site: the hot
    // code is instantiated once)
    bool done = false;
    for (int pass = 0; pass < 2; ++pass) {
      done = binomial_put_bt<kBtBmax>(spot, strike, N, q, xch, price, nodes, pass == 0);
      if (!done || price * 1e-9 >= (double)N * kBtTailEps * strike) break;
    }
    if (done) {
      if (lane == 0 && fallbacks) atomicAdd(fallbacks + 1, nodes);
      return price;
    }
    if (lane == 0 && fallbacks) {
      atomicAdd(fallbacks, 1ull);
      atomicAdd(fallbacks + 1, (unsigned long long)N * (N + 1) / 2);
    }
    return lattice_smem_inplace<AM, PUT>(spot, strike, N, q, xch);
  }
  const int B0 = (N + 1 + 31) / 32;
  // leaves: intrinsic at S * up^(2j - N), j = 0..N (nodes beyond N are dead)
  for (int j = lane; j < 32 * B0; j += 32) {
    double s = spot * exp((double)(2 * j - N) * lnu);
    double x = PUT ? strike - s : s - strike;
    xch[j] = x < 0.0 ? 0.0 : x;
  }
  __syncwarp();
  double v[BMAX];
  int L = N - 1;
  lat_chain<BMAX, AM, PUT>(v, L, q, lane, xch, LatBlocks{});
  double r = xch[0];
  __syncwarp();
  return r;
}

// Whole-triangle lattice in this warp's shared node array, in place: each
// chunk of 32 nodes reads its right neighbours before anyone writes, and
// chunks go upward, so v_j(L) = f(v_j(L+1), v_{j+1}(L+1)) never reads a
// value already overwritten (cold fallback of the boundary-tracking path).
template <bool AM, bool PUT>
__device__ double lattice_smem_inplace(double spot, double strike, int N, const LatParams& q,
                                       double* xch) {
  const int lane = threadIdx.x & 31;
  for (int j = lane; j <= N; j += 32) {
    double s = spot * exp((double)(2 * j - N) * q.lnu);
    double x = PUT ? strike - s : s - strike;
    xch[j] = x < 0.0 ? 0.0 : x;
  }
  __syncwarp();
  for (int L = N - 1; L >= 0; --L) {
    for (int c = 0; c <= L; c += 32) {
      const int j = c + lane;
      double vl = 0.0, vr = 0.0;
      if (j <= L) {
        vl = xch[j];
        vr = xch[j + 1];
      }
      __syncwarp();
      if (j <= L) {
        double cont = fma(q.pd, vr, q.qd * vl);
        if (AM) {
          double s = spot * exp((double)(2 * j - L) * q.lnu);
          cont = max_nonneg(cont, PUT ? strike - s : s - strike);
        }
        xch[j] = cont;
      }
      __syncwarp();
    }
  }
  double r = xch[0];
  __syncwarp();
  return r;
}

// Lattices beyond the register bound (N+1 > 32*33): shared-memory values,
// warp-strided nodes, double-buffered levels (same arithmetic).
template <bool AM, bool PUT>
__device__ double binomial_warp_price_smem(const double* o, int N, double* buf, bool& ok) {
  const int lane = threadIdx.x & 31;
  double spot = o[0], strike = o[1], rate = o[2], vol = o[3], mat = o[4];
  ok = true;
  if (!(spot > 0) || !(strike > 0) || !(mat > 0) || !(vol > 0) || N < 1) {
    ok = false;
    return 0.0;
  }
  double dt = mat / N, lnu = vol * sqrt(dt), up = exp(lnu), down = 1.0 / up;
  double growth = exp(rate * dt);
  double pu = (growth - down) / (up - down);
  if (!(pu > 0.0) || !(pu < 1.0)) {
    ok = false;
    return 0.0;
  }
  double disc = 1.0 / growth;
  LatParams q;
  q.K = strike;
  q.pd = disc * pu;
  q.qd = disc * (1.0 - pu);
  q.up = up;
  q.up2 = up * up;
  q.lnu = lnu;
  q.S = spot;
  double* a = buf;
  double* b = buf + (N + 2);
  for (int j = lane; j <= N; j += 32) {
    double s = spot * exp((double)(2 * j - N) * lnu);
    double x = PUT ? strike - s : s - strike;
    a[j] = x < 0.0 ? 0.0 : x;
  }
  __syncwarp();
  for (int L = N - 1; L >= 0; --L) {
    for (int j = lane; j <= L; j += 32) {
      double s = spot * exp((double)(2 * j - L) * lnu);
      double cont = fma(q.pd, a[j + 1], q.qd * a[j]);
      b[j] = AM ? max_nonneg(cont, PUT ? strike - s : s - strike) : cont;
    }
    __syncwarp();
    double* t = a;
    a = b;
    b = t;
  }
  double r = a[0];
  __syncwarp();
  return r;
}

constexpr int kLatBmax = 33;  // register lattice up to N = 32*33 - 1 = 1055 steps
#ifndef HPAC_BINO_SEG
#define HPAC_BINO_SEG 8
#endif
constexpr int kBinoSeg = HPAC_BINO_SEG;  // lanes per American put (0 = whole warp)
constexpr int kBinoSegW = kBinoSeg > 0 ? kBinoSeg : 32;  // (keeps the disabled path well-formed)
constexpr int kBinoChunk = 256;
constexpr int kBinoWarps = 2;  // = threads_per_team / 32 at the default tpt 64
#ifndef HPAC_BINO_MIN_CTAS
#define HPAC_BINO_MIN_CTAS 8
#endif

// Decision codes in the chunk plan.
constexpr int kActSkip = -1;
constexpr int kActMiss = -2;
// >= 0: hit on a slot written in an earlier chunk -> (slot)         [kHitOld]
// <= -3: hit on a step s of this chunk -> -(3 + s)                    [kHitNew]

template <int TECH, bool AM, bool PUT>
__global__ void __launch_bounds__(kBinoWarps * 32, HPAC_BINO_MIN_CTAS) binomial_team_kernel(const EngineParams p) {
  extern __shared__ __align__(16) double smem[];
  const int team = p.team_begin + (int)blockIdx.x;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int N = p.region.binomial_steps;
  const bool big = N + 1 > 32 * kLatBmax;

  // shared-memory carve-up
  double* price = smem;                        // [kBinoChunk]
  double* slot_val = price + kBinoChunk;       // [tsize]
  double* tab = smem + p.smem_tab_off;         // [tsize * 5] team table inputs / TAF ring
  double* xch = smem + p.smem_scratch_off;     // [warps][32*BMAX or 2(N+2)]
  const int xch_per_warp = big ? 2 * (N + 2) : 32 * kLatBmax;
  xch += warp * xch_per_warp;
  int* act = reinterpret_cast<int*>(smem + p.smem_ctl_off);  // [kBinoChunk]
  int* miss = act + kBinoChunk;                              // [kBinoChunk]
  int* slot_src = miss + kBinoChunk;                         // [tsize] producing step
  int* nmiss_s = slot_src + (p.tsize > 0 ? p.tsize : 1);

  const int64_t trip = trip_count(team, p.stride, p.n, p.steps);
  int rr = 0, occ = 0;  // team table cursor (thread 0)
  unsigned long long tot = 0, app = 0, wsteps = 0;
  bool err = false;
  const unsigned long long tpt = (unsigned long long)p.tpt;
  const unsigned long long wpt = (unsigned long long)p.wpt;

  // TAF under per-team binomial: sequential, evaluated by warp 0 only.
  if (TECH == HPAC_TECH_TAF) {
    if (warp != 0) return;
    int mode = kTafFilling, rem = 0, cnt = 0, head = 0;
    double lastv = 0.0;
    double* ring = tab;  // h doubles (kept in smem; tiny)
    for (int64_t step = 0; step < trip; ++step) {
      const int64_t idx = team + step * p.stride;
      bool approx = mode == kTafPredicting;
      double outv;
      if (approx) {
        outv = lastv;
        if (--rem == 0) {
          cnt = 0;
          head = 0;
          mode = kTafFilling;
        }
      } else {
        double o[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) o[d] = p.region.in[idx * 5 + d];
        bool ok = true;
        bool priced = false;
        if constexpr (AM && PUT && kBinoSeg > 0) {
          // the exact path's pricing function (segment 0 of the warp)
          if (!big) {
            unsigned long long nodes = 0;
            double v;
            const bool okseg = binomial_put_seg<kBinoSegW, SegWin<kBinoSegW>::BMAX>(
                o, lane < kBinoSegW, N, xch + (lane / kBinoSegW) * SegWin<kBinoSegW>::WIN, v, nodes);
            priced = __shfl_sync(0xffffffffu, okseg ? 1 : 0, 0) != 0;
            outv = __shfl_sync(0xffffffffu, v, 0);
            if (priced && lane == 0) atomicAdd(&p.counters[kCntLatticeNodes], nodes);
          }
        }
        if (!priced)
          outv = big ? binomial_warp_price_smem<AM, PUT>(o, N, xch, ok)
                     : binomial_warp_price<kLatBmax, AM, PUT>(o, N, xch, ok, &p.counters[kCntLatticeFallback]);
        if (!ok) err = true;
        // TafState::observe_accurate (single output)
        const int h = p.taf_h;
        if (lane == 0) {
          int slot;
          if (cnt < h) {
            slot = head + cnt;
            if (slot >= h) slot -= h;
          } else {
            slot = head;
          }
          ring[slot] = outv;
        }
        __syncwarp();
        if (cnt < h) ++cnt; else head = head + 1 == h ? 0 : head + 1;
        lastv = outv;
        if (mode == kTafPredicting) {
          if (--rem == 0) {
            cnt = 0;
            head = 0;
            mode = kTafFilling;
          }
        } else if ((mode == kTafFilling && cnt == h) || mode == kTafChecking) {
          if (taf_ring_passes(ring, 1, h, head, cnt, p.taf_thr)) {
            rem = p.taf_p;
            mode = kTafPredicting;
          } else {
            mode = kTafChecking;
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        if (p.region.out) p.region.out[idx] = outv;
        if (p.paths) p.paths[idx] = approx ? 1 : 0;
      }
      tot += tpt;
      wsteps += wpt;
      if (approx) app += tpt;
    }
    if (lane != 0) tot = app = wsteps = 0;
    flush_stats(p, tot, app, wsteps, (lane == 0 && trip > 0) ? wpt : 0ull, err);
    return;
  }

  for (int64_t base = 0; base < trip; base += kBinoChunk) {
    const int cnt = (int)(trip - base < kBinoChunk ? trip - base : kBinoChunk);
    // ---- phase 1: decisions for the chunk (input-only; thread 0) ----------
    if (threadIdx.x == 0) {
      int nm = 0;
      for (int s = 0; s < cnt; ++s) {
        const int64_t step = base + s;
        const int64_t idx = team + step * p.stride;
        int a = kActMiss;
        if (TECH == HPAC_TECH_IACT) {
          double in[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) in[d] = p.region.in[idx * 5 + d];
          int hit, near;
          team_lookup(tab, 1, 5, 5, in, occ, p.iact_thr, hit, near);
          if (hit >= 0) {
            int src = slot_src[hit];
            a = src >= base ? -(3 + (int)(src - base)) : hit;
          } else {
            // miss: the (lowest) lane inserts at the round-robin cursor
#pragma unroll
            for (int d = 0; d < 5; ++d) tab[rr * 5 + d] = in[d];
            slot_src[rr] = (int)step;
            rr = rr + 1 == p.tsize ? 0 : rr + 1;
            occ = occ + 1 < p.tsize ? occ + 1 : p.tsize;
          }
        } else if (TECH == HPAC_TECH_PERFO) {
          if (perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step, trip,
                                team))
            a = kActSkip;
        }
        act[s] = a;
        if (a == kActMiss) miss[nm++] = s;
        tot += tpt;
        wsteps += wpt;
        if (a != kActMiss) app += tpt;
        if (p.paths) p.paths[idx] = a != kActMiss ? 1 : 0;
      }
      *nmiss_s = nm;
    }
    __syncthreads();
    // ---- phase 2: misses evaluated by the team's warps --------------------
    const int nm = *nmiss_s;
    if constexpr (AM && PUT && kBinoSeg > 0) {
      // American puts: 32/SEG options per warp (binomial_put_seg); options
      // it declines go through the whole-warp path below, one at a time
      if (!big) {
        constexpr int NSEG = 32 / kBinoSegW;
        const int g = lane / kBinoSegW;
        for (int m0 = warp * NSEG; m0 < nm; m0 += kBinoWarps * NSEG) {
          const int m = m0 + g;
          const bool has = m < nm;
          double o[5] = {100.0, 100.0, 0.05, 0.25, 1.0};
          if (has) {
            const int64_t idx = team + (base + miss[m]) * p.stride;
#pragma unroll
            for (int d = 0; d < 5; ++d) o[d] = __ldg(p.region.in + idx * 5 + d);
          }
          double v;
          unsigned long long nodes = 0;
          const bool okseg = binomial_put_seg<kBinoSegW, SegWin<kBinoSegW>::BMAX>(
              o, has, N, xch + g * SegWin<kBinoSegW>::WIN, v, nodes);
          if (has && okseg && (lane % kBinoSegW) == 0) {
            price[miss[m]] = v;
            atomicAdd(&p.counters[kCntLatticeNodes], nodes);
          }
          unsigned fb = __ballot_sync(0xffffffffu, has && !okseg && (lane % kBinoSegW) == 0);
          while (fb) {
            const int gg = (__ffs(fb) - 1) / kBinoSegW;
            fb &= fb - 1;
            const int sm = miss[m0 + gg];
            const int64_t idx = team + (base + sm) * p.stride;
            double oo[5];
#pragma unroll
            for (int d = 0; d < 5; ++d) oo[d] = __ldg(p.region.in + idx * 5 + d);
            bool ok;
            const double vv = binomial_warp_price<kLatBmax, AM, PUT>(oo, N, xch, ok,
                                                                     &p.counters[kCntLatticeFallback]);
            if (!ok) err = true;
            if (lane == 0) price[sm] = vv;
          }
        }
      }
    }
    for (int m = warp; m < nm; m += kBinoWarps) {
      if constexpr (AM && PUT && kBinoSeg > 0)
        if (!big) break;
      const int s = miss[m];
      const int64_t idx = team + (base + s) * p.stride;
      double o[5];
#pragma unroll
      for (int d = 0; d < 5; ++d) o[d] = __ldg(p.region.in + idx * 5 + d);
      bool ok;
      double v = big ? binomial_warp_price_smem<AM, PUT>(o, N, xch, ok)
                     : binomial_warp_price<kLatBmax, AM, PUT>(o, N, xch, ok, &p.counters[kCntLatticeFallback]);
      if (!ok) err = true;
      if (lane == 0) price[s] = v;
    }
    __syncthreads();
    // ---- phase 3: outputs (misses, hits from this or earlier chunks) -------
    for (int s = threadIdx.x; s < cnt; s += blockDim.x) {
      const int a = act[s];
      if (a == kActSkip) continue;
      double v;
      if (a == kActMiss)
        v = price[s];
      else if (a >= 0)
        v = slot_val[a];
      else
        v = price[-(a + 3)];
      if (p.region.out) p.region.out[team + (base + s) * p.stride] = v;
    }
    __syncthreads();
    // carry slot payloads produced in this chunk to the next one
    if (TECH == HPAC_TECH_IACT && threadIdx.x == 0) {
      for (int t = 0; t < occ; ++t)
        if (slot_src[t] >= base) slot_val[t] = price[slot_src[t] - base];
    }
    __syncthreads();
  }
  if (threadIdx.x != 0) tot = app = wsteps = 0;
  flush_stats(p, tot, app, wsteps, (threadIdx.x == 0 && trip > 0) ? wpt : 0ull, err);
}

// ---------------------------------------------------------------------------
// Binomial region without TAF: decide -> price -> resolve.
//
// Under the per-team mapping every lane of a team sees the same option, so
// iACT (one team-shared table) and perforation decide on the
// inputs alone, sequentially per team; the lattices are the cost, and they
// are independent of each other. So the launch is split:
//  1. binomial_decide_kernel: one warp per team walks the team's item stream
//     (inputs staged 32 steps at a time), runs the table / perforation
//     protocol on lane 0, and writes per item the producing step of a hit
//     (iACT), appends misses to a global list, and the stats / path bits;
//  2. binomial_price_kernel: persistent CTAs; each warp takes batches of
//     misses from an atomic counter (32/SEG American puts per batch through
//     binomial_put_seg, else one option per warp) and writes their prices —
//     no team's misses wait on another team's, no tail of uneven CTAs;
//  3. binomial_resolve_kernel: every hit copies its producer's price.
// Exact (spec NULL) launches price every item of the team range directly.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Binomial TAF for American puts: 8 teams per CTA, one per 8-lane segment.
// TAF decisions depend on the prices (taf.hpp:59-163), so each team's item
// stream is sequential; the teams are independent, so a warp runs four of
// them side by side: every step each segment either emits its team's last
// price (TafState::emit_approx) or prices its team's option in the shared
// binomial_put_seg call (idle segments skip the lattice), then runs the TAF
// state machine on its own shared-memory window ring. Prices are the exact
// path's (same function of the option), so decisions replay bit-exactly.
// ---------------------------------------------------------------------------
constexpr int kTafTeamsPerWarp = 32 / kBinoSegW;

__global__ void __launch_bounds__(kBinoWarps * 32, HPAC_BINO_MIN_CTAS)
    binomial_taf_seg_kernel(const EngineParams p, int team_end) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / kBinoSegW, sub = lane % kBinoSegW;
  const int N = p.region.binomial_steps;
  const int team = p.team_begin + ((int)blockIdx.x * kBinoWarps + warp) * kTafTeamsPerWarp + g;
  const bool mine = team < team_end;
  const int h = p.taf_h;
  double* xch = smem + warp * 32 * kLatBmax;  // 4 segment windows / whole-warp fallback
  double* ring = smem + kBinoWarps * 32 * kLatBmax + (warp * kTafTeamsPerWarp + g) * h;
  const int64_t G = p.stride;
  const int64_t trip = mine ? trip_count(team, G, p.n, p.steps) : 0;
  const unsigned long long tpt = (unsigned long long)p.tpt, wpt = (unsigned long long)p.wpt;
  int mode = kTafFilling, rem = 0, cnt = 0, head = 0;
  double lastv = 0.0;
  unsigned long long tot = 0, app = 0, ws = 0;
  bool err = false;
  // the warp walks the longest of its teams' streams
  int64_t tmax = trip;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t ot = __shfl_xor_sync(0xffffffffu, tmax, o);
    tmax = ot > tmax ? ot : tmax;
  }
  for (int64_t step = 0; step < tmax; ++step) {
    const bool active = step < trip;
    const int64_t idx = team + step * G;
    const bool approx = active && mode == kTafPredicting;
    const bool want = active && !approx;
    double o[5] = {100.0, 100.0, 0.05, 0.25, 1.0};
    if (want) {
#pragma unroll
      for (int d = 0; d < 5; ++d) o[d] = __ldg(p.region.in + idx * 5 + d);
    }
    double v = 0.0;
    unsigned long long nodes = 0;
    const bool okseg = binomial_put_seg<kBinoSegW, SegWin<kBinoSegW>::BMAX>(
        o, want, N, xch + g * SegWin<kBinoSegW>::WIN, v, nodes);
    if (want && okseg && sub == 0) atomicAdd(&p.counters[kCntLatticeNodes], nodes);
    // options the segment path declines: the whole-warp path, one at a time
    unsigned fb = __ballot_sync(0xffffffffu, want && !okseg && sub == 0);
    while (fb) {
      const int gg = (__ffs(fb) - 1) / kBinoSegW;
      fb &= fb - 1;
      const double oo[5] = {__shfl_sync(0xffffffffu, o[0], gg * kBinoSegW),
                            __shfl_sync(0xffffffffu, o[1], gg * kBinoSegW),
                            __shfl_sync(0xffffffffu, o[2], gg * kBinoSegW),
                            __shfl_sync(0xffffffffu, o[3], gg * kBinoSegW),
                            __shfl_sync(0xffffffffu, o[4], gg * kBinoSegW)};
      bool ok;
      const double vv = binomial_warp_price<kLatBmax, true, true>(oo, N, xch, ok,
                                                                  &p.counters[kCntLatticeFallback]);
      if (g == gg) {
        v = vv;
        if (!ok) err = true;
      }
    }
    double outv = 0.0;
    if (approx) {
      // TafState::emit_approx, taf.hpp:114-117
      outv = lastv;
      if (--rem == 0) {
        cnt = 0;
        head = 0;
        mode = kTafFilling;
      }
    } else if (want) {
      // TafState::observe_accurate, taf.hpp:94-108 (ring in shared memory)
      outv = v;
      if (sub == 0) {
        int slot;
        if (cnt < h) {
          slot = head + cnt;
          if (slot >= h) slot -= h;
        } else {
          slot = head;
        }
        ring[slot] = v;
      }
      if (cnt < h) ++cnt; else head = head + 1 == h ? 0 : head + 1;
      lastv = v;
    }
    __syncwarp();
    if (want) {
      if (mode == kTafPredicting) {
        if (--rem == 0) {
          cnt = 0;
          head = 0;
          mode = kTafFilling;
        }
      } else if ((mode == kTafFilling && cnt == h) || mode == kTafChecking) {
        if (taf_ring_passes(ring, 1, h, head, cnt, p.taf_thr)) {
          rem = p.taf_p;
          mode = kTafPredicting;
        } else {
          mode = kTafChecking;
        }
      }
    }
    if (active && sub == 0) {
      if (p.region.out) p.region.out[idx] = outv;
      if (p.paths) p.paths[idx] = approx ? 1 : 0;
      tot += tpt;
      ws += wpt;
      if (approx) app += tpt;
    }
    __syncwarp();
  }
  flush_stats(p, tot, app, ws, (sub == 0 && trip > 0) ? wpt : 0ull, err);
}

struct BinoWork {
  int* act;        // [n] producing step of a hit (>= 0), -1 priced, -2 skipped (iACT only)
  int* miss;       // [n] items to price (iACT / perforation)
  unsigned* ctr;   // [0] misses, [1] batch counter
};

__host__ __device__ inline int bino_decide_warp_doubles(int ts) {
  return 160 + 5 * ts + (ts + 32 + 1) / 2;  // staged inputs, table, producing steps, miss list
}

template <int TECH>
__global__ void __launch_bounds__(128) binomial_decide_kernel(const EngineParams p, int team_end,
                                                              BinoWork wk) {
  extern __shared__ __align__(16) double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int team = p.team_begin + (int)blockIdx.x * 4 + warp;
  if (team >= team_end) return;  // whole warp
  const int ts = p.tsize > 0 ? p.tsize : 1;
  double* inb = sm + warp * bino_decide_warp_doubles(ts);  // [32][5]
  double* tab = inb + 160;                                  // [ts][5]
  int* src = reinterpret_cast<int*>(tab + 5 * ts);          // [ts]
  int* ml = src + ts;                                       // [32]
  const int64_t G = p.stride;
  const int64_t trip = trip_count(team, G, p.n, p.steps);
  const unsigned long long tpt = (unsigned long long)p.tpt, wpt = (unsigned long long)p.wpt;
  unsigned long long app = 0;
  int rr = 0, occ = 0;
  // lane-parallel table (tsize <= 32): slot `lane` in registers
  const bool lane_tab = p.tsize <= 32;
  int width = 1;
  while (width < p.tsize && width < 32) width <<= 1;
  double ent[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  int sstep = -1;
  for (int64_t b0 = 0; b0 < trip; b0 += 32) {
    const int cnt = (int)(trip - b0 < 32 ? trip - b0 : 32);
    if (TECH == HPAC_TECH_IACT && lane < cnt) {
      const double* o = p.region.in + (team + (b0 + lane) * G) * 5;
#pragma unroll
      for (int d = 0; d < 5; ++d) inb[lane * 5 + d] = __ldg(o + d);
    }
    __syncwarp();
    int nm = 0, mbase = 0;
    if (TECH == HPAC_TECH_IACT && lane_tab) {
      // the team's table across the warp: lane e holds slot e (registers),
      // every slot's distance is computed at once, and the hit (smallest
      // rounded distance, lowest slot on ties: team_lookup's rule) comes
      // from a butterfly over the slots
      for (int s = 0; s < cnt; ++s) {
        const int64_t step = b0 + s;
        const int64_t item = team + step * G;
        double x[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) x[d] = inb[s * 5 + d];
        double q = 0.0;
        bool cand = false;
        if (lane < occ) {
#pragma unroll
          for (int d = 0; d < 5; ++d) {
            const double df = __dsub_rn(ent[d], x[d]);
            q = __dadd_rn(q, __dmul_rn(df, df));
          }
          cand = q <= p.iact_thr2;
        }
        int bi = lane;
        for (int o = 1; o < width; o <<= 1) {
          const double oq = __shfl_xor_sync(0xffffffffu, q, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          const bool oc = __shfl_xor_sync(0xffffffffu, cand, o);
          bool take_o;
          if (!oc) take_o = false;
          else if (!cand) take_o = true;
          else if (oq < q * (1.0 - 0x1p-48)) take_o = true;
          else if (q < oq * (1.0 - 0x1p-48)) take_o = false;
          else {
            const double da = __dsqrt_rn(q), db = __dsqrt_rn(oq);
            take_o = db < da || (db == da && oi < bi);
          }
          if (take_o) {
            q = oq;
            bi = oi;
            cand = true;
          }
        }
        // lanes past `width` reduced among themselves: lane 0 holds the answer
        cand = __shfl_sync(0xffffffffu, cand, 0);
        bi = __shfl_sync(0xffffffffu, bi, 0);
        const int hs = __shfl_sync(0xffffffffu, sstep, cand ? bi : 0);
        int a = -1;
        if (cand) {
          a = hs;
        } else {
          if (lane == rr) {
#pragma unroll
            for (int d = 0; d < 5; ++d) ent[d] = x[d];
            sstep = (int)step;
          }
          rr = rr + 1 == p.tsize ? 0 : rr + 1;
          occ = occ + 1 < p.tsize ? occ + 1 : p.tsize;
        }
        if (lane == 0) {
          wk.act[item] = a;
          if (a == -1) ml[nm] = (int)item;
          else app += tpt;
          if (p.paths) p.paths[item] = a != -1 ? 1 : 0;
        }
        if (a == -1) ++nm;
      }
      if (lane == 0 && nm) mbase = (int)atomicAdd(&wk.ctr[0], (unsigned)nm);
    } else if (lane == 0) {
      for (int s = 0; s < cnt; ++s) {
        const int64_t step = b0 + s;
        const int64_t item = team + step * G;
        int a = -1;
        if (TECH == HPAC_TECH_IACT) {
          // one team-shared MemoTable (iact.hpp:58-145): a hit emits the
          // slot's output, a miss is inserted at the round-robin cursor
          const int hit = team_hit5(tab, inb + s * 5, occ, p.iact_thr2);
          if (hit >= 0) {
            a = src[hit];
          } else {
#pragma unroll
            for (int d = 0; d < 5; ++d) tab[rr * 5 + d] = inb[s * 5 + d];
            src[rr] = (int)step;
            rr = rr + 1 == p.tsize ? 0 : rr + 1;
            occ = occ + 1 < p.tsize ? occ + 1 : p.tsize;
          }
          wk.act[item] = a;
        } else if (TECH == HPAC_TECH_PERFO) {
          if (perfo_should_skip(p.perfo_kind, p.perfo_mod, p.perfo_pct, p.perfo_seed, step, trip,
                                team))
            a = -2;
        }
        if (a == -1) ml[nm++] = (int)item;
        else app += tpt;
        if (p.paths) p.paths[item] = a != -1 ? 1 : 0;
      }
      if (nm) mbase = (int)atomicAdd(&wk.ctr[0], (unsigned)nm);
    }
    nm = __shfl_sync(0xffffffffu, nm, 0);
    mbase = __shfl_sync(0xffffffffu, mbase, 0);
    __syncwarp();
    for (int k = lane; k < nm; k += 32) wk.miss[mbase + k] = ml[k];
    __syncwarp();
  }
  if (lane == 0 && trip > 0) {
    atomicAdd(&p.counters[kCntTotal], (unsigned long long)trip * tpt);
    atomicAdd(&p.counters[kCntWarpSteps], (unsigned long long)trip * wpt);
    atomicAdd(&p.counters[kCntResidentWarps], wpt);
    if (app) atomicAdd(&p.counters[kCntApprox], app);
  }
}

// exact launches: stats and (zero) path bits of every item of the range
__global__ void binomial_exact_stats_kernel(const EngineParams p, int team_end) {
  const int64_t G = p.stride;
  const int nr = team_end - p.team_begin;
  const unsigned long long tpt = (unsigned long long)p.tpt, wpt = (unsigned long long)p.wpt;
  unsigned long long tot = 0, ws = 0, res = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nr; t += gridDim.x * blockDim.x) {
    const int team = p.team_begin + t;
    const int64_t trip = trip_count(team, G, p.n, p.steps);
    tot += trip * tpt;
    ws += trip * wpt;
    if (trip > 0) res += wpt;
    if (p.paths)
      for (int64_t s = 0; s < trip; ++s) p.paths[team + s * G] = 0;
  }
  flush_stats(p, tot, 0ull, ws, res, false);
}

#ifndef HPAC_BINO_PRICE_MIN_CTAS
#define HPAC_BINO_PRICE_MIN_CTAS 8  // 128 registers (ptxas picks 128 at 7 too; 6 = 168 registers: 4 % slower)
#endif
template <bool AM, bool PUT>
__global__ void __launch_bounds__(kBinoWarps * 32, HPAC_BINO_PRICE_MIN_CTAS)
    binomial_price_kernel(const EngineParams p, int team_end, BinoWork wk, int use_list) {
  extern __shared__ __align__(16) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = p.region.binomial_steps;
  const bool big = N + 1 > 32 * kLatBmax;
  const int xch_per_warp = big ? 2 * (N + 2) : 32 * kLatBmax;
  double* xch = smem + warp * xch_per_warp;
  const int64_t G = p.stride;
  const int nr = team_end - p.team_begin;
  // items to price: the miss list, or every (team, step) of the range
  const int64_t m_total = use_list ? (int64_t)*(volatile unsigned*)&wk.ctr[0] : (int64_t)nr * p.steps;
  auto item_of = [&](int64_t m) -> int64_t {
    if (use_list) return wk.miss[m];
    const int64_t it = p.team_begin + m % nr + (m / nr) * G;
    return it < p.n ? it : -1;
  };
  constexpr bool SEGD = AM && PUT && kBinoSeg > 0;
  const int NSEG = SEGD && !big ? 32 / kBinoSegW : 1;
  bool err = false;
  for (;;) {
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(&wk.ctr[1], 1u);
    b = __shfl_sync(0xffffffffu, b, 0);
    const int64_t m0 = (int64_t)b * NSEG;
    if (m0 >= m_total) break;
    bool done = false;
    if constexpr (SEGD) {
      if (!big) {
        done = true;
        const int g = lane / kBinoSegW;
        const int64_t m = m0 + g;
        const int64_t item = m < m_total ? item_of(m) : -1;
        const bool has = item >= 0;
        double o[5] = {100.0, 100.0, 0.05, 0.25, 1.0};
        if (has) {
#pragma unroll
          for (int d = 0; d < 5; ++d) o[d] = __ldg(p.region.in + item * 5 + d);
        }
        double v;
        unsigned long long nodes = 0;
        const bool okseg = binomial_put_seg<kBinoSegW, SegWin<kBinoSegW>::BMAX>(
            o, has, N, xch + g * SegWin<kBinoSegW>::WIN, v, nodes);
        if (has && okseg && (lane % kBinoSegW) == 0) {
          if (p.region.out) p.region.out[item] = v;
          atomicAdd(&p.counters[kCntLatticeNodes], nodes);
        }
        unsigned fb = __ballot_sync(0xffffffffu, has && !okseg && (lane % kBinoSegW) == 0);
        while (fb) {
          const int gg = (__ffs(fb) - 1) / kBinoSegW;
          fb &= fb - 1;
          const int64_t it = item_of(m0 + gg);
          double oo[5];
#pragma unroll
          for (int d = 0; d < 5; ++d) oo[d] = __ldg(p.region.in + it * 5 + d);
          bool ok;
          const double vv = binomial_warp_price<kLatBmax, AM, PUT>(oo, N, xch, ok,
                                                                   &p.counters[kCntLatticeFallback]);
          if (!ok) err = true;
          if (lane == 0 && p.region.out) p.region.out[it] = vv;
        }
      }
    }
    if (!done) {
      const int64_t item = item_of(m0);
      if (item >= 0) {
        double o[5];
#pragma unroll
        for (int d = 0; d < 5; ++d) o[d] = __ldg(p.region.in + item * 5 + d);
        bool ok;
        const double v = big ? binomial_warp_price_smem<AM, PUT>(o, N, xch, ok)
                             : binomial_warp_price<kLatBmax, AM, PUT>(o, N, xch, ok,
                                                                      &p.counters[kCntLatticeFallback]);
        if (!ok) err = true;
        if (lane == 0 && p.region.out) p.region.out[item] = v;
      }
    }
  }
  const unsigned e = __ballot_sync(0xffffffffu, err);
  if (lane == 0 && e) atomicAdd(&p.counters[kCntAppError], 1ull);
}

__global__ void binomial_resolve_kernel(const EngineParams p, int team_end, const int* act) {
  const int64_t G = p.stride;
  const int nr = team_end - p.team_begin;
  const int64_t total = (int64_t)nr * p.steps;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int team = p.team_begin + (int)(k % nr);
    const int64_t item = team + (k / nr) * G;
    if (item >= p.n) continue;
    const int a = act[item];
    if (a >= 0) p.region.out[item] = p.region.out[team + (int64_t)a * G];
  }
}

cudaMemPool_t bino_pool();

template <bool AM, bool PUT>
static cudaError_t launch_bino_pipeline(const EngineParams& p, int nblocks, cudaStream_t st) {
  const int team_end = p.team_begin + nblocks;
  const int N = p.region.binomial_steps;
  const bool big = N + 1 > 32 * kLatBmax;
  const bool iact = p.tech == HPAC_TECH_IACT, perfo = p.tech == HPAC_TECH_PERFO;
  const size_t n = (size_t)p.n;
  const size_t bytes = 16 + (iact ? n * sizeof(int) : 0) + ((iact || perfo) ? n * sizeof(int) : 0);
  char* ws = nullptr;
  cudaMemPool_t pool = bino_pool();
  cudaError_t e = pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ws), bytes, pool, st)
                       : cudaMallocAsync(reinterpret_cast<void**>(&ws), bytes, st);
  if (e != cudaSuccess) return e;
  BinoWork wk;
  wk.ctr = reinterpret_cast<unsigned*>(ws);
  wk.act = iact ? reinterpret_cast<int*>(ws + 16) : nullptr;
  wk.miss = (iact || perfo) ? reinterpret_cast<int*>(ws + 16 + (iact ? n * sizeof(int) : 0)) : nullptr;
  // every error path below releases the workspace
  auto fail_free = [&](cudaError_t err) {
    cudaFreeAsync(ws, st);
    return err;
  };
  if ((e = cudaMemsetAsync(ws, 0, 16, st)) != cudaSuccess) return fail_free(e);
  if (iact || perfo) {
    const int ts = p.tsize > 0 ? p.tsize : 1;
    const size_t dsm = 4 * (size_t)bino_decide_warp_doubles(ts) * sizeof(double);
    auto kd = iact ? binomial_decide_kernel<HPAC_TECH_IACT> : binomial_decide_kernel<HPAC_TECH_PERFO>;
    if (dsm > 48 * 1024 &&
        (e = cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm)) != cudaSuccess)
      return fail_free(e);
    kd<<<(nblocks + 3) / 4, 128, dsm, st>>>(p, team_end, wk);
  } else {
    binomial_exact_stats_kernel<<<(nblocks + 255) / 256 < 148 ? (nblocks + 255) / 256 : 148, 256, 0, st>>>(p, team_end);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_free(e);
  // persistent pricing grid: every resident CTA slot, at most one per batch
  auto kp = binomial_price_kernel<AM, PUT>;
  const size_t psm = (size_t)kBinoWarps * (big ? 2 * (N + 2) : 32 * kLatBmax) * sizeof(double);
  if (psm > 48 * 1024 &&
      (e = cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm)) != cudaSuccess)
    return fail_free(e);
  int per_sm = 0, dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, kBinoWarps * 32, psm)) != cudaSuccess)
    return fail_free(e);
  const long long items = (long long)nblocks * p.steps;
  const int nseg = (AM && PUT && kBinoSeg > 0 && !big) ? 32 / kBinoSegW : 1;
  long long grid = (long long)(per_sm > 0 ? per_sm : 1) * sms;
  const long long need = (items + (long long)nseg * kBinoWarps - 1) / ((long long)nseg * kBinoWarps);
  if (grid > need) grid = need > 0 ? need : 1;
  kp<<<(int)grid, kBinoWarps * 32, psm, st>>>(p, team_end, wk, (iact || perfo) ? 1 : 0);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_free(e);
  if (iact && p.region.out) {
    binomial_resolve_kernel<<<4 * sms, 256, 0, st>>>(p, team_end, wk.act);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail_free(e);
  }
  return cudaFreeAsync(ws, st);
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------
size_t binomial_team_smem(EngineParams& p) {
  const int N = p.region.binomial_steps;
  const bool big = N + 1 > 32 * kLatBmax;
  const int ts = p.tsize > 0 ? p.tsize : 1;
  size_t tabsz = 5 * (size_t)ts;
  if (p.tech == HPAC_TECH_TAF && (size_t)p.taf_h > tabsz) tabsz = p.taf_h;  // TAF ring
  p.smem_tab_off = kBinoChunk + ts;
  p.smem_scratch_off = (int)(p.smem_tab_off + tabsz);
  size_t dbl = p.smem_scratch_off + (size_t)kBinoWarps * (big ? 2 * (N + 2) : 32 * kLatBmax);
  p.smem_ctl_off = (int)dbl;
  size_t ints = 2 * kBinoChunk + ts + 2;
  return dbl * sizeof(double) + ints * sizeof(int);
}

size_t engine_team_seq_smem(EngineParams& p, int block) {
  size_t off = 0;
  p.smem_taf_off = 0;
  if (p.tech == HPAC_TECH_TAF && !(p.out_dims == 1 && p.taf_h <= 8)) {
    off += (size_t)p.out_dims * p.taf_h * block;
  }
  p.smem_tab_off = (int)off;
  if (p.tech == HPAC_TECH_IACT) off += (size_t)p.tsize * (p.in_dims + p.out_dims) * block;
  p.smem_ctl_off = (int)off;
  return off * sizeof(double) + 16;
}

template <class App, int TECH>
static cudaError_t launch_seq(const EngineParams& p, int team_end, int block, size_t smem,
                              cudaStream_t st) {
  int nteams = team_end - p.team_begin;
  int grid = (nteams + block - 1) / block;
  int hreg = (TECH == HPAC_TECH_TAF && p.out_dims == 1 && p.taf_h <= 8) ? p.taf_h : 0;
#define HPAC_SEQ(H)                                                                         \
  {                                                                                         \
    auto k = engine_team_seq_kernel<App, TECH, H>;                                          \
    if (smem > 48 * 1024) {                                                                 \
      cudaError_t e =                                                                       \
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
      if (e != cudaSuccess) return e;                                                       \
    }                                                                                       \
    k<<<grid, block, smem, st>>>(p, team_end);                                              \
    return cudaGetLastError();                                                              \
  }
  if (TECH == HPAC_TECH_TAF) {
    switch (hreg) {
      case 1: HPAC_SEQ(1);
      case 2: HPAC_SEQ(2);
      case 3: HPAC_SEQ(3);
      case 4: HPAC_SEQ(4);
      case 5: HPAC_SEQ(5);
      case 6: HPAC_SEQ(6);
      case 7: HPAC_SEQ(7);
      case 8: HPAC_SEQ(8);
      default: HPAC_SEQ(0);
    }
  }
  HPAC_SEQ(0);
#undef HPAC_SEQ
}

template <class App>
static cudaError_t launch_seq_app(const EngineParams& p, int team_end, int block, size_t smem,
                                  cudaStream_t st) {
  switch (p.tech) {
    case HPAC_TECH_TAF: return launch_seq<App, HPAC_TECH_TAF>(p, team_end, block, smem, st);
    case HPAC_TECH_IACT: return launch_seq<App, HPAC_TECH_IACT>(p, team_end, block, smem, st);
    case HPAC_TECH_PERFO: return launch_seq<App, HPAC_TECH_PERFO>(p, team_end, block, smem, st);
    default: return launch_seq<App, kTechNoneT>(p, team_end, block, smem, st);
  }
}

cudaError_t engine_team_seq_launch(const EngineParams& p, int team_end, int block, size_t smem,
                                   cudaStream_t st) {
  switch (p.region.app) {
    case HPAC_APP_TABLE: return launch_seq_app<AppTable>(p, team_end, block, smem, st);
    case HPAC_APP_SYNTHETIC: return launch_seq_app<AppSynthetic>(p, team_end, block, smem, st);
    case HPAC_APP_BLACKSCHOLES:
      return launch_seq_app<AppBlackScholes>(p, team_end, block, smem, st);
  }
  return cudaErrorInvalidValue;
}

template <int TECH, bool AM, bool PUT>
static cudaError_t launch_bino3(const EngineParams& p, int nblocks, size_t smem,
                                cudaStream_t st) {
  auto k = binomial_team_kernel<TECH, AM, PUT>;
  if (smem > 48 * 1024) {
    cudaError_t e =
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<nblocks, kBinoWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

template <int TECH>
static cudaError_t launch_bino2(const EngineParams& p, int nblocks, size_t smem,
                                cudaStream_t st) {
  const bool am = p.region.binomial_american != 0, put = p.region.binomial_put != 0;
  // decide -> price -> resolve for everything but TAF (whose decisions need
  // the prices); HPAC_BINO_PIPELINE=0 keeps the one-kernel chunked engine
  const char* pe = getenv("HPAC_BINO_PIPELINE");
  const int ts = p.tsize > 0 ? p.tsize : 1;
  if (TECH == HPAC_TECH_TAF && am && put && kBinoSeg > 0 &&
      p.region.binomial_steps + 1 <= 32 * kLatBmax && !(pe && strcmp(pe, "0") == 0)) {
    // 8 teams per CTA, one per 8-lane segment (binomial_taf_seg_kernel)
    const size_t tsm = ((size_t)kBinoWarps * 32 * kLatBmax +
                        (size_t)kBinoWarps * kTafTeamsPerWarp * (p.taf_h > 0 ? p.taf_h : 1)) *
                       sizeof(double);
    if (tsm > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(binomial_taf_seg_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      if (e != cudaSuccess) return e;
    }
    const int per = kBinoWarps * kTafTeamsPerWarp;
    binomial_taf_seg_kernel<<<(nblocks + per - 1) / per, kBinoWarps * 32, tsm, st>>>(
        p, p.team_begin + nblocks);
    return cudaGetLastError();
  }
  if (TECH != HPAC_TECH_TAF && !(pe && strcmp(pe, "0") == 0) && p.n < (1ll << 31) &&
      4 * (size_t)bino_decide_warp_doubles(ts) * sizeof(double) <= 200 * 1024) {
    if (am && put) return launch_bino_pipeline<true, true>(p, nblocks, st);
    if (am && !put) return launch_bino_pipeline<true, false>(p, nblocks, st);
    if (!am && put) return launch_bino_pipeline<false, true>(p, nblocks, st);
    return launch_bino_pipeline<false, false>(p, nblocks, st);
  }
  if (am && put) return launch_bino3<TECH, true, true>(p, nblocks, smem, st);
  if (am && !put) return launch_bino3<TECH, true, false>(p, nblocks, smem, st);
  if (!am && put) return launch_bino3<TECH, false, true>(p, nblocks, smem, st);
  return launch_bino3<TECH, false, false>(p, nblocks, smem, st);
}

cudaError_t binomial_team_launch(const EngineParams& p, int nblocks, size_t smem,
                                 cudaStream_t st) {
  switch (p.tech) {
    case HPAC_TECH_TAF: return launch_bino2<HPAC_TECH_TAF>(p, nblocks, smem, st);
    case HPAC_TECH_IACT: return launch_bino2<HPAC_TECH_IACT>(p, nblocks, smem, st);
    case HPAC_TECH_PERFO: return launch_bino2<HPAC_TECH_PERFO>(p, nblocks, smem, st);
    default: return launch_bino2<kTechNoneT>(p, nblocks, smem, st);
  }
}

}  // namespace hpac
