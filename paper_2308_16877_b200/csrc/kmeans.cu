// kmeans.cu — the K-Means Lloyd loop on the device (kmeans_benchmark,
// bench/kmeans.hpp:62-144), driving the approximate distance region once per
// iteration exactly like the reference: technique state is fresh every
// launch, convergence = no label changed, empty clusters keep their centroid.
//
// Labels-only equivalence: the reference stores all k
// distances per point and argmins them after the launch; a point the region
// skipped keeps its previous distances, hence its previous argmin. We keep
// that argmin ("dist label", initialised to 0 = argmin of the zero-filled
// distance matrix) instead of n*k doubles.
//
// Centroid update: running per-cluster sums and counts, changed by the
// points whose label changed this iteration (+x into the new cluster, -x out
// of the old one). One warp per contiguous chunk of points, lane = dimension
// (coalesced 256 B rows of the changed points only), per-warp private
// shared-memory accumulators (no atomics), then a fixed-order reduction
// (deterministic run to run). The packed [sum deltas | count deltas |
// changed] buffer is the only cross-GPU exchange; the caller's all-reduce
// hook (NCCL) runs between the partial sums and the centroid recompute.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "engine.h"
#include "hpac_offload.h"

#define HPAC_API extern "C" __attribute__((visibility("default")))

namespace hpac {

constexpr int kUpdWarps = 4;
constexpr int kMaxSubsPerWarp = 8;  // kmeans_update_partial: the pipelined stream's sub-chunk table

__global__ void kmeans_forgy(const double* pts, int64_t n, int dims, int k, double* cent) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k * dims; i += gridDim.x * blockDim.x) {
    int c = i / dims, d = i % dims;
    int64_t src = c < n - 1 ? c : n - 1;
    cent[i] = pts[src * dims + d];
  }
}

__global__ void kmeans_init_labels(int32_t* dist_label, int32_t* assign, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dist_label[i] = 0;
    assign[i] = -1;
  }
}

// The iteration's label changes, compacted per sub-chunk in point order
// (deterministic): sub-chunk g = points [g*sub, (g+1)*sub), one warp each,
// 4 batches of 32 labels in flight. Changed points are listed with their old
// assignment, and their assignment is updated (kmeans.hpp:122-127).
constexpr int kCompactU = 4;
__global__ void __launch_bounds__(256)
    kmeans_changed_compact(const int32_t* __restrict__ dist_label, int32_t* __restrict__ assign,
                           int64_t n, int64_t sub, int64_t nsub, int32_t* __restrict__ list,
                           int32_t* __restrict__ oldlab, int32_t* __restrict__ newlab,
                           int32_t* __restrict__ list_len) {
  const int lane = threadIdx.x & 31;
  const int64_t gs = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (gs >= nsub) return;
  const int64_t lo = gs * sub, hi = lo + sub < n ? lo + sub : n;
  int cnt = 0;
  for (int64_t b0 = lo; b0 < hi; b0 += 32 * kCompactU) {
    int nl[kCompactU], ol[kCompactU];
#pragma unroll
    for (int u = 0; u < kCompactU; ++u) {
      const int64_t i = b0 + u * 32 + lane;
      nl[u] = i < hi ? __ldcs(dist_label + i) : 0;
      ol[u] = i < hi ? assign[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kCompactU; ++u) {
      const int64_t i = b0 + u * 32 + lane;
      const bool ch = i < hi && nl[u] != ol[u];
      const unsigned m = __ballot_sync(0xffffffffu, ch);
      if (ch) {
        const int pos = cnt + __popc(m & ((1u << lane) - 1u));
        list[lo + pos] = (int32_t)(i - lo);
        oldlab[lo + pos] = ol[u];
        newlab[lo + pos] = nl[u];
        assign[i] = nl[u];
      }
      cnt += __popc(m);
    }
  }
  if (lane == 0) list_len[gs] = cnt;
}

// Per-CTA partials of the iteration's CHANGES: [k*dims sum deltas | k count
// deltas | changed] into part[cta][...]. Only points whose label changed
// move: + x into the new cluster, - x out of the old one (none on the first
// iteration, where every assignment is -1). The running sums (kmeans_accumulate)
// therefore always equal the sum of every point under its current label,
// the reference's full re-sum (kmeans.hpp:133-141) up to rounding, while an
// iteration reads the labels and assignments (8 B per point) plus the rows
// of the changed points only. Warp w walks the compacted lists of its
// sub-chunks in order, 32 entries at a time: lane j reads entry j (index,
// old and new label); the changed rows (lane = dimension, 256 B per row) of
// group g+1 are in flight while group g accumulates, in point order, into
// the warp's private shared-memory sums. Count deltas are integers.
constexpr int kBatch = 32;
__global__ void __launch_bounds__(kUpdWarps * 32, 2)
    kmeans_update_partial(const double* __restrict__ pts, const int32_t* __restrict__ dist_label,
                          const int32_t* __restrict__ list, const int32_t* __restrict__ oldlab,
                          const int32_t* __restrict__ newlab, const int32_t* __restrict__ list_len,
                          int64_t sub, int subs_per_warp, int64_t nsub, int dims, int k,
                          double* __restrict__ part) {
  extern __shared__ __align__(16) double acc[];  // [warps][k*dims] then int counts [warps][k]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int kd = k * dims;
  double* my = acc + (size_t)w * kd;
  int* cnts = reinterpret_cast<int*>(acc + (size_t)kUpdWarps * kd) + w * k;
  for (int i = lane; i < kd; i += 32) my[i] = 0.0;
  for (int i = lane; i < k; i += 32) cnts[i] = 0;
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * kUpdWarps + w;
  unsigned long long changed = 0;
  const bool dl = lane < dims;
  const int64_t gs0 = gw * subs_per_warp;
  const int S = gs0 >= nsub ? 0 : (int)(nsub - gs0 < subs_per_warp ? nsub - gs0 : subs_per_warp);
  if (dims <= 32 && subs_per_warp <= kMaxSubsPerWarp) {
    // The warp's sub-chunks as ONE stream of entries (sub order, then list
    // order: the same point order as sub by sub) in batches of 32, software
    // pipelined two batches deep: batch b+2's entries (index, old and new
    // label: coalesced loads, no dependent gather) and batch b+1's rows are
    // in flight while batch b accumulates, so a sub-chunk boundary costs no
    // memory round trip.
    const int mylen = lane < S ? list_len[gs0 + lane] : 0;
    int incl = mylen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int excl[kMaxSubsPerWarp];
#pragma unroll
    for (int t = 0; t < kMaxSubsPerWarp; ++t) excl[t] = __shfl_sync(0xffffffffu, incl - mylen, t);
    changed = total;
    // entry q of the stream: its sub-chunk and list position, its point
    auto entry = [&](int q, int64_t& pi, int& nl, int& ol) {
      if (q >= total) {
        pi = 0;
        nl = 0;
        ol = -1;
        return;
      }
      int t = 0, et = 0;  // excl[0] = 0 (registers only: no dynamic index)
#pragma unroll
      for (int u = 1; u < kMaxSubsPerWarp; ++u)
        if (u < S && excl[u] <= q) {
          t = u;
          et = excl[u];
        }
      const int64_t lo = (gs0 + t) * sub;
      const int64_t at = lo + (q - et);
      pi = lo + list[at];
      nl = newlab[at];
      ol = oldlab[at];
    };
    auto rows = [&](int q0, const int64_t pi, double (&x)[kBatch]) {
      const int c = total - q0 < kBatch ? total - q0 : kBatch;
#pragma unroll
      for (int j = 0; j < kBatch; ++j) {
        const int64_t pj = __shfl_sync(0xffffffffu, pi, j);
        x[j] = (j < c && dl) ? __ldcs(pts + pj * dims + lane) : 0.0;
      }
    };
    double xa[kBatch], xb[kBatch];
    int64_t p0 = 0, p1 = 0, p2 = 0;
    int n0 = 0, o0 = -1, n1 = 0, o1 = -1, n2 = 0, o2 = -1;
    if (total > 0) {
      entry(lane, p0, n0, o0);
      rows(0, p0, xa);
      entry(kBatch + lane, p1, n1, o1);
    }
    for (int q0 = 0; q0 < total; q0 += kBatch) {
      const int c = total - q0 < kBatch ? total - q0 : kBatch;
      if (q0 + kBatch < total) rows(q0 + kBatch, p1, xb);
      if (q0 + 2 * kBatch < total) entry(q0 + 2 * kBatch + lane, p2, n2, o2);
      if (lane < c) {
        atomicAdd(&cnts[n0], 1);
        if (o0 >= 0) atomicSub(&cnts[o0], 1);
      }
      // rows j and j+1 touching four different clusters (the common case)
      // read all their sums before writing any: two read-modify-write
      // chains in flight instead of one; a shared cluster keeps the order
#pragma unroll
      for (int j = 0; j < kBatch; j += 2) {
        if (j >= c) break;
        const int ca = __shfl_sync(0xffffffffu, n0, j), oa = __shfl_sync(0xffffffffu, o0, j);
        const int cb = __shfl_sync(0xffffffffu, n0, j + 1), ob = __shfl_sync(0xffffffffu, o0, j + 1);
        const bool two = j + 1 < c;
        const bool apart = two && cb != ca && cb != oa && (ob < 0 || (ob != ca && ob != oa));
        if (dl) {
          double* pa = my + (size_t)ca * dims + lane;
          double* qa = my + (size_t)(oa >= 0 ? oa : 0) * dims + lane;
          if (apart) {
            double* pb = my + (size_t)cb * dims + lane;
            double* qb = my + (size_t)(ob >= 0 ? ob : 0) * dims + lane;
            const double va = *pa, wa = oa >= 0 ? *qa : 0.0, vb = *pb, wb = ob >= 0 ? *qb : 0.0;
            *pa = va + xa[j];
            if (oa >= 0) *qa = wa - xa[j];
            *pb = vb + xa[j + 1];
            if (ob >= 0) *qb = wb - xa[j + 1];
          } else {
            *pa += xa[j];
            if (oa >= 0) *qa -= xa[j];
            if (two) {
              my[(size_t)cb * dims + lane] += xa[j + 1];
              if (ob >= 0) my[(size_t)ob * dims + lane] -= xa[j + 1];
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kBatch; ++j) xa[j] = xb[j];
      p0 = p1;
      n0 = n1;
      o0 = o1;
      p1 = p2;
      n1 = n2;
      o1 = o2;
    }
  } else {
    for (int64_t gs = gs0; gs < gs0 + S; ++gs) {
      const int64_t lo = gs * sub;
      const int len = list_len[gs];
      changed += len;
      for (int e0 = 0; e0 < len; e0 += 32) {
        const bool v = e0 + lane < len;
        const int64_t pi = v ? lo + list[lo + e0 + lane] : 0;
        const int nl = v ? newlab[lo + e0 + lane] : 0;
        const int ol = v ? oldlab[lo + e0 + lane] : -1;
        const int c = len - e0 < 32 ? len - e0 : 32;
        if (lane < c) {
          atomicAdd(&cnts[nl], 1);
          if (ol >= 0) atomicSub(&cnts[ol], 1);
        }
        for (int j = 0; j < c; ++j) {
          const int64_t pj = __shfl_sync(0xffffffffu, pi, j);
          const int cn = __shfl_sync(0xffffffffu, nl, j), co = __shfl_sync(0xffffffffu, ol, j);
          for (int d = lane; d < dims; d += 32) {
            const double x = __ldcs(pts + pj * dims + d);
            my[(size_t)cn * dims + d] += x;
            if (co >= 0) my[(size_t)co * dims + d] -= x;
          }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // fixed-order sum over the CTA's warps
  const int stride = kd + k;
  double* out = part + (size_t)blockIdx.x * (stride + 1);
  for (int j = threadIdx.x; j < kd; j += blockDim.x) {
    double s = 0.0;
    for (int v = 0; v < kUpdWarps; ++v) s += acc[(size_t)v * kd + j];
    out[j] = s;
  }
  const int* allc = reinterpret_cast<const int*>(acc + (size_t)kUpdWarps * kd);
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    long long s = 0;
    for (int v = 0; v < kUpdWarps; ++v) s += allc[v * k + j];
    out[kd + j] = (double)s;
  }
  __shared__ unsigned long long ch[kUpdWarps];
  if (lane == 0) ch[w] = changed;  // identical in every lane
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int v = 0; v < kUpdWarps; ++v) t += ch[v];
    out[stride] = (double)t;
  }
}

// Fixed-order sum over CTAs -> red[j] (deterministic).
__global__ void kmeans_reduce_partials(const double* part, int nparts, int width, double* red) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < width; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[(size_t)p * width + j];
    red[j] = s;
  }
}

// Running sums and counts += this iteration's (all-reduced) changes; an
// emptied cluster's sums restart from exact zero. One warp owns a cluster:
// every lane reads the old count before lane 0 overwrites it, so no thread
// can see a count another thread already updated (the sums and the count of
// a cluster are never touched by two warps).
__global__ void kmeans_accumulate(const double* red, int dims, int k, double* tot) {
  const int kd = k * dims;
  if (red[kd + k] == 0.0) return;  // converged: nothing moved
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < k; c += nwarps) {
    const double cnt = tot[kd + c] + red[kd + c];  // exact: integers below 2^53
    for (int d = lane; d < dims; d += 32) {
      const int i = c * dims + d;
      tot[i] = cnt > 0.0 ? tot[i] + red[i] : 0.0;
    }
    __syncwarp();
    if (lane == 0) tot[kd + c] = cnt;
  }
}

// centroids[c] = sums[c] / counts[c]; empty clusters keep theirs (kmeans.hpp:142-143)
__global__ void kmeans_recompute(const double* red, const double* tot, int dims, int k, double* cent) {
  const int kd = k * dims;
  if (red[kd + k] == 0.0) return;  // converged: centroids stay (kmeans.hpp:122-127)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kd; i += gridDim.x * blockDim.x) {
    const double cnt = tot[kd + i / dims];
    if (cnt > 0.0) cent[i] = tot[i] / cnt;
  }
}

// ---- captured Lloyd loop (one CUDA graph: a device-side while loop) -------
int region_prepare(const hpac_grid_t* g, int64_t n, int32_t mapping, const hpac_region_t* region,
                   const hpac_spec_t* spec, unsigned long long* d_counters,
                   const unsigned long long* seed_ptr, const double* km_aux, void** handle,
                   char* err, size_t el);
cudaError_t region_launch(const void* handle, cudaStream_t st);
void region_free(void* handle);
size_t kmeans_aux_bytes(int k);
}  // namespace hpac
cudaMemPool_t host_entry_pool();  // runtime.cu: retained pool of the host entries
namespace hpac {

// Device state of a captured run: the region counters accumulate across
// iterations; times are %globaltimer deltas (ns) between the marks.
struct LoopState {
  unsigned long long cnt[kNumCounters];
  unsigned long long seed;  // perforation seed of the next iteration
  int iter;                 // iterations run inside the graph
  int converged;
  unsigned long long t_mark, t_region, t_update;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void loop_init(LoopState* s, uint64_t seed) {
  for (int i = 0; i < kNumCounters; ++i) s->cnt[i] = i == kCntBarrierKey ? ~0ull : 0ull;
  s->seed = seed;
  s->iter = 0;
  s->converged = 0;
  s->t_mark = s->t_region = s->t_update = 0;
}
__global__ void loop_mark(LoopState* s) { s->t_mark = globaltimer(); }
__global__ void loop_after_region(LoopState* s) {
  const unsigned long long t = globaltimer();
  s->t_region += t - s->t_mark;
  s->t_mark = t;
}
// End of an iteration: count it, key the next seed, and continue while some
// label changed and iterations remain (kmeans.hpp:122-127)
__global__ void loop_cond(LoopState* s, const double* changed, int iters_left, uint64_t seed_next0,
                          cudaGraphConditionalHandle h) {
  s->t_update += globaltimer() - s->t_mark;
  const int it = ++s->iter;
  s->seed = seed_next0 + (uint64_t)it;
  bool more = true;
  if (*changed == 0.0) {
    s->converged = 1;
    more = false;
  } else if (it >= iters_left) {
    more = false;
  }
  cudaGraphSetConditional(h, more ? 1u : 0u);
}

}  // namespace hpac

namespace {
int kfail(char* err, size_t len, int code, const char* fmt, ...) {
  if (err && len) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, len, fmt, ap);
    va_end(ap);
  }
  return code;
}
}  // namespace

HPAC_API int hpac_kmeans_run(const hpac_grid_t* grid, const hpac_kmeans_problem_t* pb,
                             const hpac_spec_t* spec, void* stream, hpac_kmeans_result_t* res,
                             char* err, size_t el) {
  using namespace hpac;
  if (!grid || !pb || !res) return kfail(err, el, HPAC_ERR_CONFIG, "null argument");
  std::memset(res, 0, sizeof *res);
  const int64_t n = pb->n_points;
  const int dims = pb->dims, k = pb->k;
  if (n < 0 || dims < 1 || k < 1 || pb->max_iters < 0)
    return kfail(err, el, HPAC_ERR_CONFIG, "kmeans problem: bad sizes");
  const size_t stride = (size_t)k * dims + k;
  const size_t upd_smem = (size_t)kUpdWarps * ((size_t)k * dims * sizeof(double) + (size_t)k * sizeof(int)) + 16;
  if (upd_smem > 200 * 1024)
    return kfail(err, el, HPAC_ERR_UNSUPPORTED, "k*dims too large for the centroid update (%zu B)",
                 upd_smem);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  int32_t* dist_label = nullptr;
  double* part = nullptr;
  double* red = pb->reduce_buf;
  double* tot = nullptr;  // running [sums | counts] under the current labels
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nparts = sms * 2;
  const int64_t warps = (int64_t)nparts * kUpdWarps;
  // sub-chunks: kSubsPerWarp per update warp, one compaction warp each
  constexpr int kSubsPerWarp = 8;
  const int64_t nsub = warps * kSubsPerWarp;
  const int64_t sub = n > 0 ? (n + nsub - 1) / nsub : 1;
  int32_t *list = nullptr, *oldlab = nullptr, *newlab = nullptr, *list_len = nullptr;
  auto cleanup = [&]() {
    if (dist_label) cudaFreeAsync(dist_label, st);
    if (part) cudaFreeAsync(part, st);
    if (red && red != pb->reduce_buf) cudaFreeAsync(red, st);
    if (tot) cudaFreeAsync(tot, st);
    if (list) cudaFreeAsync(list, st);
    if (oldlab) cudaFreeAsync(oldlab, st);
    if (newlab) cudaFreeAsync(newlab, st);
    if (list_len) cudaFreeAsync(list_len, st);
  };
  // run-scoped buffers from the library's retained stream-ordered pool (no
  // re-mapping of ~200 MB of scratch on every run)
  cudaMemPool_t pool = host_entry_pool();
  auto palloc = [&](auto** ptr, size_t bytes) {
    return pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(ptr), bytes, pool, st)
                : cudaMallocAsync(reinterpret_cast<void**>(ptr), bytes, st);
  };
  const size_t nn = (size_t)(n > 0 ? n : 1);
  if ((e = palloc(&dist_label, sizeof(int32_t) * nn)) ||
      (e = palloc(&part, sizeof(double) * (stride + 1) * nparts)) ||
      (!red && (e = palloc(&red, sizeof(double) * (stride + 1)))) ||
      (e = palloc(&tot, sizeof(double) * stride)) || (e = palloc(&list, sizeof(int32_t) * nn)) ||
      (e = palloc(&oldlab, sizeof(int32_t) * nn)) ||
      (e = palloc(&newlab, sizeof(int32_t) * nn)) ||
      (e = palloc(&list_len, sizeof(int32_t) * (size_t)nsub)) ||
      (e = cudaMemsetAsync(tot, 0, sizeof(double) * stride, st))) {
    cleanup();
    return kfail(err, el, HPAC_ERR_CUDA, "kmeans alloc: %s", cudaGetErrorString(e));
  }
  if (upd_smem > 48 * 1024)
    cudaFuncSetAttribute(kmeans_update_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)upd_smem);
  if (!(pb->flags & HPAC_KMEANS_CENTROIDS_GIVEN) && n > 0)
    kmeans_forgy<<<(k * dims + 255) / 256, 256, 0, st>>>(pb->points, n, dims, k, pb->centroids);
  kmeans_init_labels<<<sms * 4, 256, 0, st>>>(dist_label, pb->assignments, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);

  hpac_region_t r{};
  r.app = HPAC_APP_KMEANS;
  r.kmeans_dims = dims;
  r.kmeans_k = k;
  r.flags = pb->flags & HPAC_REGION_KMEANS_FAST_MATH;
  r.in = pb->points;
  r.centroids = pb->centroids;
  r.labels = dist_label;
  hpac_spec_t sp{};
  if (spec) sp = *spec;
  hpac_launch_t L{};
  L.stream = st;
  L.synchronous = 1;

  // iterations first+1 .. max_iters inside one graph launch; returns
  // kGraphUnavailable (nothing ran) when the body cannot be captured or
  // instantiated, e.g. an all-reduce that is not stream-capturable
  constexpr int kGraphUnavailable = -1;
  auto run_graph = [&](int first) -> int {
    const int left = pb->max_iters - first;
    LoopState* ds = nullptr;
    double* aux = nullptr;
    void* hreg = nullptr;
    cudaStream_t cs = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int grc = HPAC_OK;
    LoopState hs{};
    auto done = [&](int code) {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      if (cs) cudaStreamDestroy(cs);
      if (hreg) region_free(hreg);
      if (ds) cudaFreeAsync(ds, st);
      if (aux) cudaFreeAsync(aux, st);
      return code;
    };
    cudaError_t ge;
    if ((ge = palloc(&ds, sizeof(LoopState))) != cudaSuccess ||
        (ge = palloc(&aux, kmeans_aux_bytes(k))) != cudaSuccess ||
        (loop_init<<<1, 1, 0, st>>>(ds, pb->perfo_seed_base + (uint64_t)first + 1),
         (ge = cudaGetLastError()) != cudaSuccess))
      return done(kfail(err, el, HPAC_ERR_CUDA, "kmeans graph alloc: %s", cudaGetErrorString(ge)));
    grc = region_prepare(grid, n, HPAC_MAP_PER_THREAD, &r, spec, ds->cnt, &ds->seed, aux, &hreg,
                         err, el);
    if (grc) return done(grc);
    cudaGraphConditionalHandle h;
    cudaGraphNodeParams cp{};
    cudaGraphNode_t node;
    if ((ge = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess ||
        (ge = cudaGraphCreate(&graph, 0)) != cudaSuccess ||
        (ge = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault)) !=
            cudaSuccess)
      return done(kGraphUnavailable);
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    if ((ge = cudaGraphAddNode(&node, graph, nullptr, 0, &cp)) != cudaSuccess)
      return done(kGraphUnavailable);
    // the loop body: one Lloyd iteration, captured
    if ((ge = cudaStreamBeginCaptureToGraph(cs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                            cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      return done(kGraphUnavailable);
    loop_mark<<<1, 1, 0, cs>>>(ds);
    ge = region_launch(hreg, cs);
    loop_after_region<<<1, 1, 0, cs>>>(ds);
    kmeans_changed_compact<<<(int)((nsub + 7) / 8), 256, 0, cs>>>(
        dist_label, pb->assignments, n, sub, nsub, list, oldlab, newlab, list_len);
    kmeans_update_partial<<<nparts, kUpdWarps * 32, upd_smem, cs>>>(
        pb->points, dist_label, list, oldlab, newlab, list_len, sub, kSubsPerWarp, nsub, dims, k, part);
    kmeans_reduce_partials<<<(int)((stride + 1 + 255) / 256), 256, 0, cs>>>(part, nparts,
                                                                              (int)(stride + 1), red);
    int hook_rc = pb->allreduce ? pb->allreduce(red, (int64_t)(stride + 1), pb->allreduce_user, cs)
                                : HPAC_OK;
    kmeans_accumulate<<<(k + 7) / 8, 256, 0, cs>>>(red, dims, k, tot);
    kmeans_recompute<<<(k * dims + 255) / 256, 256, 0, cs>>>(red, tot, dims, k, pb->centroids);
    loop_cond<<<1, 1, 0, cs>>>(ds, red + stride, left, pb->perfo_seed_base + (uint64_t)first + 1, h);
    cudaGraph_t body;
    cudaError_t ce = cudaStreamEndCapture(cs, &body);
    if (hook_rc != HPAC_OK) {
      cudaGetLastError();
      return done(kfail(err, el, HPAC_ERR_CUDA, "kmeans all-reduce hook failed (status %d)", hook_rc));
    }
    if (ge == cudaSuccess) ge = ce;
    if (ge == cudaSuccess) ge = cudaGetLastError();
    if (ge != cudaSuccess || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      cudaGetLastError();  // capture errors are not sticky: clear and fall back
      return done(kGraphUnavailable);
    }
    if ((ge = cudaGraphLaunch(exec, st)) != cudaSuccess ||
        (ge = cudaMemcpyAsync(&hs, ds, sizeof hs, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
        (ge = cudaStreamSynchronize(st)) != cudaSuccess)
      return done(kfail(err, el, HPAC_ERR_CUDA, "kmeans graph run: %s", cudaGetErrorString(ge)));
    if (pb->allreduce == hpac_nccl_allreduce && hpac_nccl_check(pb->allreduce_user) != HPAC_OK)
      return done(kfail(err, el, HPAC_ERR_CUDA, "kmeans all-reduce: NCCL communicator error"));
    res->iterations = first + hs.iter;
    res->converged = hs.converged;
    res->graph = 1;
    res->stats.total_invocations += hs.cnt[kCntTotal];
    res->stats.approx_invocations += hs.cnt[kCntApprox];
    res->stats.divergent_warp_steps += hs.cnt[kCntDivergent];
    res->stats.total_warp_steps += hs.cnt[kCntWarpSteps];
    if (hs.iter > 0) res->stats.resident_warps = (int32_t)(hs.cnt[kCntResidentWarps] / hs.iter);
    res->region_ms += hs.t_region * 1e-6;
    res->update_ms += hs.t_update * 1e-6;
    return done(HPAC_OK);
  };
  int rc = HPAC_OK;
  double h_changed = 0.0;
  // The whole loop runs as one CUDA graph (a conditional while node: no
  // host round trip per iteration) unless the caller's all-reduce hook is a
  // host callback (only no hook or the native NCCL hook are captured), or
  // HPAC_KMEANS_HOST_LOOP is set.
  // RANDOM perforation's exact first iteration runs on the host path.
  const bool random_perfo = spec && spec->technique == HPAC_TECH_PERFO &&
                            spec->perfo_kind == HPAC_PERFO_RANDOM;
  // (HPAC_KMEANS_HOST_LOOP=1 in the environment: for profilers, e.g. ncu does
  // not profile kernel nodes of graphs with conditional nodes)
  const char* hl = getenv("HPAC_KMEANS_HOST_LOOP");
  bool use_graph = (!pb->allreduce || pb->allreduce == hpac_nccl_allreduce) &&
                   !(pb->flags & HPAC_KMEANS_HOST_LOOP) && !(hl && strcmp(hl, "1") == 0) && n > 0;
  const int graph_start = random_perfo ? 2 : 1;
  for (int iter = 1; iter <= pb->max_iters; ++iter) {
    if (use_graph && iter == graph_start) {
      const int g = run_graph(iter - 1);
      if (g != kGraphUnavailable) {
        rc = g;
        break;
      }
      use_graph = false;  // not capturable here: the host drives the rest
    }
    if (spec && spec->technique == HPAC_TECH_PERFO && spec->perfo_kind == HPAC_PERFO_RANDOM)
      sp.perfo_seed = pb->perfo_seed_base + (uint64_t)iter;
    hpac_stats_t s{};
    // RANDOM extension: the first iteration is exact (a skipped point must
    // have a stale label to keep; the reference modes keep label 0)
    const bool exact_iter = spec && spec->technique == HPAC_TECH_PERFO &&
                            spec->perfo_kind == HPAC_PERFO_RANDOM && iter == 1;
    rc = hpac_run_region(grid, n, HPAC_MAP_PER_THREAD, &r, (spec && !exact_iter) ? &sp : nullptr,
                         &L, &s, err, el);
    if (rc) {
      res->stats.arena_required = s.arena_required;
      res->stats.arena_available = s.arena_available;
      break;
    }
    res->stats.total_invocations += s.total_invocations;
    res->stats.approx_invocations += s.approx_invocations;
    res->stats.divergent_warp_steps += s.divergent_warp_steps;
    res->stats.total_warp_steps += s.total_warp_steps;
    res->stats.resident_warps = s.resident_warps;
    res->region_ms += s.kernel_ms;
    res->iterations = iter;
    // labels -> assignments, change count, partial sums (every point, as the
    // reference sums all points in order, kmeans.hpp:135-141)
    cudaEventRecord(e0, st);
    kmeans_changed_compact<<<(int)((nsub + 7) / 8), 256, 0, st>>>(
        dist_label, pb->assignments, n, sub, nsub, list, oldlab, newlab, list_len);
    kmeans_update_partial<<<nparts, kUpdWarps * 32, upd_smem, st>>>(
        pb->points, dist_label, list, oldlab, newlab, list_len, sub, kSubsPerWarp, nsub, dims, k, part);
    kmeans_reduce_partials<<<(int)((stride + 1 + 255) / 256), 256, 0, st>>>(part, nparts,
                                                                              (int)(stride + 1), red);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      rc = kfail(err, el, HPAC_ERR_CUDA, "kmeans update: %s", cudaGetErrorString(e));
      break;
    }
    if (pb->allreduce) {
      const int hrc = pb->allreduce(red, (int64_t)(stride + 1), pb->allreduce_user, st);
      if (hrc != HPAC_OK) {
        rc = kfail(err, el, HPAC_ERR_CUDA, "kmeans all-reduce hook failed (status %d)", hrc);
        break;
      }
    }
    cudaMemcpyAsync(&h_changed, red + stride, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaEventRecord(e1, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
      rc = kfail(err, el, HPAC_ERR_CUDA, "kmeans iteration: %s", cudaGetErrorString(e));
      break;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    res->update_ms += ms;
    if (h_changed == 0.0) {  // no observation changed cluster (kmeans.hpp:122-127)
      res->converged = 1;
      break;
    }
    kmeans_accumulate<<<(k + 7) / 8, 256, 0, st>>>(red, dims, k, tot);
    kmeans_recompute<<<(k * dims + 255) / 256, 256, 0, st>>>(red, tot, dims, k, pb->centroids);
  }
  res->stats.kernel_ms = res->region_ms + res->update_ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cleanup();
  cudaError_t fe = cudaStreamSynchronize(st);
  if (rc == HPAC_OK && fe != cudaSuccess)
    rc = kfail(err, el, HPAC_ERR_CUDA, "kmeans: %s", cudaGetErrorString(fe));
  return rc;
}
