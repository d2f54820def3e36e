// ggnn_query.cu -- search kernels (query, greedy, descent, sym-check, top-k)
// and their C-ABI entry points (include/ggnn_b200.h).
//
// Launch shape: one warp per search, W warps per CTA, each warp owning a
// private shared-memory region (ring + visited ring + refcount table + query).
// Every search is independent, so the grid is simply ceil(m / W) CTAs and the
// hardware block scheduler balances the (very uneven) per-query work.
#include <atomic>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "ggnn_build.h"
#include "ggnn_capi_util.cuh"
#include "ggnn_p2p.h"
#include "ggnn_search.cuh"
#include "ggnn_shard.h"

namespace ggnn {

// tensor-core brute force (ggnn_bf_tc.cu)
bool bf_tc_eligible(const ggnn_vectors* X, const int32_t* d_rows, const ggnn_queries* Q, int k);
int bf_topk_tc(const ggnn_vectors* X, const ggnn_queries* Q, int k, int32_t* d_ids, double* d_dists,
               cudaStream_t st);
// tensor-core brute force for float tables (ggnn_bf_tf32.cu)
bool bf_tf32_eligible(const ggnn_vectors* X, const int32_t* d_rows, const ggnn_queries* Q, int k);
int bf_topk_tf32(const ggnn_vectors* X, const ggnn_queries* Q, int k, int32_t* d_ids, double* d_dists,
                 cudaStream_t st);
struct SearchArgs;
int exhaustive_warp(SearchArgs& a, const ggnn_vectors* X, const ggnn_queries* Q, const int32_t* d_rows, int64_t nrows,
                    int32_t* d_ids, double* d_dists, cudaStream_t st);

static thread_local std::string g_err;
// ggnn_search_accounting: (visited, steps) totals of the build-type searches
static thread_local unsigned long long* g_acc = nullptr;

__device__ __forceinline__ void account(unsigned long long* acc, long long visited, long long steps) {
  if (acc && lane_id() == 0) {
    atomicAdd(acc, (unsigned long long)visited);
    atomicAdd(acc + 1, (unsigned long long)steps);
  }
}
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

std::atomic<unsigned long long> g_kernel_launches{0};
void count_launch(int n) { g_kernel_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

DevInfo dev_info() {
  static DevInfo info{0, 0, 0};
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&info.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&info.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&info.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  });
  return info;
}

constexpr int MAX_LAYERS = 24;
// Search CTAs: up to 4 warps (one search each); 6 resident CTAs per SM caps
// registers at 80 per thread, so 24 searches share an SM (shared memory
// allows about as many for the default 266-entry ring + 512-entry visited
// ring + 1024-slot table).  Sym-check CTAs run 8 warps of small searches.
#ifndef GGNN_SEARCH_WARPS
#define GGNN_SEARCH_WARPS 1  // one-warp CTAs: no warp waits for slower CTA-mates
#endif
#ifndef GGNN_SEARCH_MIN_BLOCKS
#define GGNN_SEARCH_MIN_BLOCKS (28 / GGNN_SEARCH_WARPS)
#endif
#ifndef GGNN_PERSISTENT
#define GGNN_PERSISTENT 0  // persistent warps + work counter for the search kernels
#endif
constexpr int SEARCH_WARPS = GGNN_SEARCH_WARPS;
constexpr int SEARCH_THREADS = 32 * SEARCH_WARPS;
constexpr int SEARCH_MIN_BLOCKS = GGNN_SEARCH_MIN_BLOCKS;
// uint8 table + uint8 queries: the packed ring (no flag bytes) leaves 6.6 KB
// of shared memory per search, so more searches fit per SM when the register
// budget allows it
#ifndef GGNN_U8_MIN_BLOCKS
#define GGNN_U8_MIN_BLOCKS GGNN_SEARCH_MIN_BLOCKS
#endif
// resident CTAs per SM the intermediate resume round of a uint8 batch is
// compiled for (0: the default)
#ifndef GGNN_ROUND1_MIN_BLOCKS
#define GGNN_ROUND1_MIN_BLOCKS 32
#endif
template <typename TX, typename TQ>
constexpr int min_blocks() {
  return (sizeof(TX) == 1 && sizeof(TQ) == 1) ? GGNN_U8_MIN_BLOCKS / GGNN_SEARCH_WARPS : SEARCH_MIN_BLOCKS;
}
// the u8 query kernel fits 64 registers without spills (shared memory still
// limits it to 28 warps/SM); the staged variant is capped there so its extra
// load path does not change the search's code generation
#ifndef GGNN_QUERY_MIN_BLOCKS
#define GGNN_QUERY_MIN_BLOCKS (32 / GGNN_SEARCH_WARPS)
#endif
constexpr int QUERY_MIN_BLOCKS = GGNN_QUERY_MIN_BLOCKS;
#ifndef GGNN_STAGED_CAP
#define GGNN_STAGED_CAP 1
#endif
constexpr bool STAGED_CAP = GGNN_STAGED_CAP != 0;
#ifndef GGNN_SYM_PERSISTENT
#define GGNN_SYM_PERSISTENT 1
#endif
constexpr int SYM_THREADS = 256;
#ifndef GGNN_SYM_MIN_BLOCKS
#define GGNN_SYM_MIN_BLOCKS 4
#endif
constexpr int SYM_MIN_BLOCKS = GGNN_SYM_MIN_BLOCKS;

struct LayerDev {
  const int32_t* adj;
  const int32_t* to_row;
  const int32_t* down;
  int64_t node_count;
  int k;
  double slack;
};

struct SearchArgs {
  const void* X;
  int64_t n;
  int64_t d;
  int lpr;
  const void* Q;        // query table (TQ) or nullptr
  const int32_t* qrows; // rows of X used as queries, or nullptr
  int64_t m;
  SearchCfg c;
  size_t region;        // bytes per warp
  int32_t* ids;
  double* dists;
  int32_t* counters;
  uint32_t* ever;       // distinct_touched logs: m * ever_size entries, or nullptr
  uint32_t ever_size;   // log capacity per query
  int32_t* log_len;     // (m) entries logged per query, -1 when the log overflowed
  // query()
  const int32_t* top_rows;
  int64_t ntop;
  double dmax;
  LayerDev layer;
  // greedy
  const int32_t* seed_ids;
  const double* seed_dists;
  int nseeds;
  // descent
  LayerDev layers[MAX_LAYERS];
  int start, stop;
  const int32_t* seg_lo;
  const int32_t* seg_hi;
  // computed segments (construction): seg = (seg_of ? seg_of[i] : i) / seg_div,
  // rows [seg * seg_size, seg * seg_size + seg_size) of the start layer
  const int32_t* seg_of;
  int seg_div;
  int seg_size;
  int* work;  // persistent-warp item counter (nullptr: one item per warp)
  int chunk;  // items claimed per counter update
  // fused sharded exchange (ggnn_query_batch_push): block `push_rank` of
  // parity half `push_parity` of every receive allocation
  uint8_t* push_peers[GGNN_P2P_MAX_RANKS];
  int push_n, push_rank;
  size_t push_half, push_bb, push_doff, push_coff;
  const int32_t* push_gid;
  int64_t push_gid_size;
  // queries still arriving (ggnn_query_batch_staged): row qi is usable once
  // qflags[qi / qchunk] == qepoch; qconv: float rows narrowed to uint8 on load
  const uint32_t* qflags;
  int64_t qchunk;
  uint32_t qepoch;
  int qconv;
  int32_t* qstatus;
  unsigned long long* acc;  // build accounting (visited, steps) or nullptr
  // longest-first schedule (launch_query): pilot > 0 runs every search for at
  // most `pilot` expansions and parks the open ones (park_key: a predicted
  // length bucket, PARK_DONE when finished); the resume pass takes them in
  // park_order
  long long pilot;
  float park_a;  // weight of log2(pending work + 1) in the length prediction
  uint8_t* park;
  size_t park_slot;
  uint32_t* park_key;
  const int32_t* park_order;
  const int32_t* park_count;
};

constexpr uint32_t PARK_DONE = 0xffffffffu;
constexpr int PARK_BUCKETS = 1024;

// Predicted search length of a parked search, in eighth-octave buckets
// (larger = longer): log2 of its best distance so far plus park_a x log2 of
// its pending work (unexpanded ring entries within the stopping threshold).
// On C2 the best distance after 16-24 expansions ranks the remaining work
// with Spearman 0.5-0.6, the pending work after 32 with 0.87 (but coarsely);
// together they start most of the longest searches in the first wave
// (tools/drain_data.py).
__device__ __forceinline__ uint32_t park_bucket(double d1, int open, float wa) {
  const float v = (float)d1;
  float b = 0.0f;
  if (v > 0.0f) b = (log2f(v) + 64.0f) * 8.0f;
  b += wa * 8.0f * log2f((float)open + 1.0f);
  return b <= 0.0f ? 0u : (b >= (float)(PARK_BUCKETS - 1) ? (uint32_t)(PARK_BUCKETS - 1) : (uint32_t)b);
}

template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void park_search(WarpSearch<TX, TQ, LP>& s, const SearchArgs& a, int64_t qi) {
  using Key = typename VecTraits<TX, TQ>::Key;
  const int open = a.park_a != 0.0f ? s.open_work() : 0;
  s.park(a.park + (size_t)qi * a.park_slot, a.d * (int64_t)sizeof(TQ));
  if (lane_id() == 0) a.park_key[qi] = park_bucket(KeyOps<Key>::to_d(s.ring_key(0)), open, a.park_a);
}

// Persistent warps: with a work counter (zeroed before the launch) every warp
// takes the next items when it finishes one, so uneven search lengths never
// leave a warp idle until its CTA-mates finish; without one each warp runs
// its static item (one item per warp, grid covering all items).  Items are
// claimed WORK_CHUNK at a time: one atomic per item on a single counter cost
// more than the item itself for the many instant ones of a symmetrize pass
// (a pair already linked back, a request settled in an earlier round).
// The chunk shrinks to 1 when there are few items per resident warp (a late
// claim round's handful of re-checks must still spread over all SMs).
#ifndef GGNN_WORK_CHUNK
#define GGNN_WORK_CHUNK 8
#endif
struct WorkCursor {
  int64_t cur, end;
  int chunk;
};
__device__ __forceinline__ int64_t grab_chunk(int* work, WorkCursor& w) {
  int v = 0;
  if (lane_id() == 0) v = atomicAdd(work, w.chunk);
  w.cur = (int64_t)__shfl_sync(FULL, v, 0);
  w.end = w.cur + w.chunk;
  return w.cur;
}
__device__ __forceinline__ int64_t first_item(int* work, int chunk, WorkCursor& w) {
  if (!work) return (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  w.chunk = chunk;
  return grab_chunk(work, w);
}
__device__ __forceinline__ int64_t next_item(int* work, WorkCursor& w) {
  if (!work) return INT64_MAX;
  if (++w.cur < w.end) return w.cur;
  return grab_chunk(work, w);
}

// Staged queries: wait (bounded, ~50 ms) until the host's copy stream has
// published the chunk holding row qi; a timeout sets bit 1 of *qstatus.
// The flag is polled with relaxed volatile loads and the row is then read
// with ld.global.cv (from L2, where the copy landed before the flag): an
// acquire at system scope would invalidate the SM's L1 at every query start,
// throwing away the other searches' prefetched rows.
__device__ __forceinline__ void wait_query_chunk(const SearchArgs& a, int64_t qi) {
  if (!a.qflags) return;  // zero-copy: the rows are read straight from mapped host memory
  if (lane_id() == 0) {
    const volatile uint32_t* f = a.qflags + qi / a.qchunk;
    uint32_t v = *f;
    if (v != a.qepoch) {
      const long long t0 = clock64();
      do {
        __nanosleep(256);
        v = *f;
        if (clock64() - t0 > 100000000ll) {  // ~50 ms: the chunk was queued before the launch
          atomicOr(a.qstatus, 2);
          break;
        }
      } while (v != a.qepoch);
    }
  }
  __syncwarp();
}

template <typename TX, typename TQ, bool STAGED = false>
__device__ __forceinline__ void load_query(TQ* qs, const SearchArgs& a, int64_t qi) {
  const int lane = lane_id();
  if constexpr (STAGED) {
    wait_query_chunk(a, qi);
    if (sizeof(TQ) == 1 && a.qconv) {  // float32 row narrowed to uint8 (exact only for integers in [0, 255])
      const float* src = reinterpret_cast<const float*>(a.Q) + qi * a.d;
      bool bad = false;
      for (int64_t e = lane; e < a.d; e += 32) {
        const float f = __ldcv(src + e);
        const uint32_t u = (f >= 0.0f && f <= 255.0f) ? (uint32_t)f : 0u;
        bad |= (float)u != f;
        qs[e] = (TQ)u;
      }
      if (__any_sync(FULL, bad) && lane == 0) atomicOr(a.qstatus, 1);
      __syncwarp();
      return;
    }
  }
  const TQ* src;
  if (a.qrows) {
    src = reinterpret_cast<const TQ*>(a.X) + (int64_t)__ldg(a.qrows + qi) * a.d;
  } else {
    src = reinterpret_cast<const TQ*>(a.Q) + qi * a.d;
  }
  if constexpr (STAGED) {
    for (int64_t e = lane; e < a.d; e += 32) qs[e] = __ldcv(src + e);
  } else {
    for (int64_t e = lane; e < a.d; e += 32) qs[e] = src[e];
  }
  __syncwarp();
}

template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void init_search(WarpSearch<TX, TQ, LP>& s, const SearchArgs& a, uint8_t* region, int64_t qi) {
  s.X = reinterpret_cast<const TX*>(a.X);
  s.d = a.d;
  s.lpr = a.lpr;
  s.c = a.c;
  s.target = -1;
  s.carve(region);
  s.tlog = a.ever ? a.ever + (size_t)qi * a.ever_size : nullptr;
  s.log_cap = (int)a.ever_size;
  s.nlog = 0;
  s.log_tag = 0u;
}

// distinct_touched of a search: its log length for the counting pass (-1:
// overflowed), the counter column holding the part known without the log
template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void finish_log(const WarpSearch<TX, TQ, LP>& s, const SearchArgs& a, int64_t qi) {
  if (a.ever && lane_id() == 0) a.log_len[qi] = s.nlog <= s.log_cap ? s.nlog : -1;
}

template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void set_layer(WarpSearch<TX, TQ, LP>& s, const LayerDev& L) {
  s.adj = L.adj;
  s.k = L.k;
  s.to_row = L.to_row;
  s.dmax = L.slack;
}

// hits -> output rows (float keys optionally re-scored sequentially and
// re-sorted, WarpSearch::write_out) + the five counters.  distinct_touched is
// -1 when it was not computed (no GGNN_FLAG_DISTINCT) and when a compact
// distinct-set overflowed (the caller reruns those queries with exact tables).
template <typename TX, typename TQ, int LP>
__device__ void write_hits(WarpSearch<TX, TQ, LP>& s, const SearchArgs& a, int64_t qi, const int32_t* to_row,
                           int extra_visited, int extra_distinct) {
  const int k_out = a.c.k_out;
  s.write_out(to_row, (a.c.flags & FLAG_EXACT_DISTS) != 0, a.ids + qi * k_out, a.dists + qi * k_out);
#ifdef GGNN_DEBUG_OPEN
  extra_distinct = s.open_work();
#endif
  if (lane_id() == 0 && a.counters) {
    int32_t* c = a.counters + qi * 5;
    c[0] = s.visited + extra_visited;
    c[1] = s.steps;
    c[2] = s.term;
#ifdef GGNN_DEBUG_OPEN
    c[3] = extra_distinct;
#else
    c[3] = a.ever == nullptr ? -1 : extra_distinct;  // + the log's distinct ids (distinct_log_kernel)
#endif
    c[4] = s.forgotten;
  }
  finish_log(s, a, qi);
}

// Fused exchange: this query's row, ids globalized, into block push_rank of
// every receive allocation (NVLink stores to peer GPUs; the own one is local).
__device__ __forceinline__ void push_row(const SearchArgs& a, int64_t qi) {
  const int lane = lane_id();
  const int k = a.c.k_out;
  const int64_t base = (int64_t)a.push_rank * (int64_t)a.push_bb;
  for (int j = lane; j < k; j += 32) {
    const int32_t id = a.ids[qi * k + j];
    const double dv = a.dists[qi * k + j];
    const int32_t gid = (id >= 0 && id < a.push_gid_size) ? __ldg(a.push_gid + id) : -1;
    for (int g = 0; g < a.push_n; ++g) {
      uint8_t* blk = a.push_peers[g] + base;
      reinterpret_cast<int32_t*>(blk)[qi * k + j] = gid;
      reinterpret_cast<double*>(blk + a.push_doff)[qi * k + j] = dv;
    }
  }
  if (lane < 5 && a.counters) {
    const int32_t c = a.counters[qi * 5 + lane];
    for (int g = 0; g < a.push_n; ++g)
      reinterpret_cast<int32_t*>(a.push_peers[g] + base + a.push_coff)[qi * 5 + lane] = c;
  }
}

// ------------------------------------------------------------------ query()
template <typename TX, typename TQ, int LP, bool PUSH = false, bool STAGED = false>
__device__ __forceinline__ void query_kernel_one(const SearchArgs& a, uint8_t* smem_w, int* vring_lane, int64_t qi) {
  using Key = typename VecTraits<TX, TQ>::Key;
  const int lane = lane_id();
  WarpSearch<TX, TQ, LP> s;
  s.vr = vring_lane;
  init_search(s, a, smem_w, qi);
  load_query<TX, TQ, STAGED>(s.qs, a, qi);
  set_layer(s, a.layer);
  s.dmax = a.dmax;
  s.reset();
  // top_layer_seeds (search.py:100-112): exact top-min(k_out, ntop) over the
  // top layer, 32 ranks per pass (one pass unless k_out and the top layer
  // both exceed 32)
  const int kk = (int)min((int64_t)a.c.k_out, a.ntop);
  Key ak = 0;  // the previous pass's last (key, local index)
  int ai = -1;
  for (int b = 0; b < kk; b += 32) {
    const int kc = min(32, kk - b);
    Key bk;
    int bi;
    warp_topk_scan<TX, TQ, LP>(s.X, a.d, s.qs, a.lpr, a.top_rows, 0, (int)a.ntop, kc, s.crow, s.ckey, bk, bi, b > 0,
                               ak, ai);
    ak = KeyOps<Key>::shfl(bk, kc - 1);
    ai = __shfl_sync(FULL, bi, kc - 1);
    int sid = -1;
    if (lane < kc) sid = a.top_rows ? __ldg(a.top_rows + bi) : bi;
    s.seed(bk, sid, kc);
  }
  // one copy of the step loop (two inlined copies measured 2x slower: the
  // instruction cache holds one); target = -1, so run() == run_until(inf)
  const bool pilot = !PUSH && a.pilot > 0;
  if (s.run_until(pilot ? a.pilot : LLONG_MAX)) {
    park_search(s, a, qi);
    return;
  }
  if (pilot && lane == 0) a.park_key[qi] = PARK_DONE;
  // query() adds the top scan to the effort counters (search.py:134-136)
  write_hits(s, a, qi, a.layer.to_row, (int)a.ntop, (int)a.ntop - kk);
  if constexpr (PUSH) {
    __syncwarp();
    push_row(a, qi);
    __threadfence_system();  // the row is visible to the peers before this warp retires
  }
}

template <typename TX, typename TQ, int LP, bool PUSH = false, bool STAGED = false>
__global__ void __launch_bounds__(SEARCH_THREADS, (STAGED && STAGED_CAP && sizeof(TX) == 1) ? QUERY_MIN_BLOCKS
                                                                                              : min_blocks<TX, TQ>())
    query_kernel(const __grid_constant__ SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  int vring_lane[VR_SLOTS > 0 ? VR_SLOTS : 1];
  uint8_t* smem_w = smem + (size_t)(threadIdx.x >> 5) * a.region;
  if constexpr (GGNN_PERSISTENT != 0) {
    WorkCursor wc;
    for (int64_t qi = first_item(a.work, a.chunk, wc); qi < a.m; qi = next_item(a.work, wc))
      query_kernel_one<TX, TQ, LP, PUSH, STAGED>(a, smem_w, vring_lane, qi);
  } else {
    const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (qi < a.m) query_kernel_one<TX, TQ, LP, PUSH, STAGED>(a, smem_w, vring_lane, qi);
  }
}

// Resume pass of the longest-first schedule: warp w continues parked search
// park_order[w] to its end, or (pilot > 0: an intermediate round) up to
// `pilot` expansions in total and parks it again with a fresh prediction.
// MB > 0: this many resident CTAs per SM for the register budget (the
// intermediate round is throughput-bound: every search runs a bounded number
// of expansions, so more co-resident searches pay; the last round is bound by
// its longest searches and keeps the default)
template <typename TX, typename TQ, int LP, int MB = 0>
__global__ void __launch_bounds__(SEARCH_THREADS, MB > 0 ? MB : min_blocks<TX, TQ>())
    resume_kernel(const __grid_constant__ SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  int vring_lane[VR_SLOTS > 0 ? VR_SLOTS : 1];
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)*a.park_count) return;
  const int64_t qi = a.park_order[w];
  uint8_t* smem_w = smem + (size_t)(threadIdx.x >> 5) * a.region;
  WarpSearch<TX, TQ, LP> s;
  s.vr = vring_lane;
  init_search(s, a, smem_w, qi);
  set_layer(s, a.layer);
  s.dmax = a.dmax;
  s.reset();
  s.unpark(a.park + (size_t)qi * a.park_slot, a.d * (int64_t)sizeof(TQ));
  if (s.run_until(a.pilot > 0 ? a.pilot : LLONG_MAX)) {  // one copy of the step loop
    park_search(s, a, qi);
    return;
  }
  if (a.pilot > 0 && lane_id() == 0) a.park_key[qi] = PARK_DONE;
  const int kk = (int)min((int64_t)a.c.k_out, a.ntop);
  write_hits(s, a, qi, a.layer.to_row, (int)a.ntop, (int)a.ntop - kk);
}

// Parked searches in descending bucket order (one CTA; the order inside a
// bucket is arbitrary -- it only schedules, results do not depend on it).
__global__ void __launch_bounds__(PARK_BUCKETS) park_order_kernel(const uint32_t* key, int64_t m, int32_t* order,
                                                                  int32_t* count) {
  __shared__ int hist[PARK_BUCKETS];
  __shared__ int wsum[PARK_BUCKETS / 32];
  const int t = threadIdx.x;
  hist[t] = 0;
  __syncthreads();
  for (int64_t i = t; i < m; i += PARK_BUCKETS) {
    const uint32_t k = key[i];
    if (k != PARK_DONE) atomicAdd(&hist[k], 1);
  }
  __syncthreads();
  // exclusive scan over buckets from the highest down: thread t owns bucket
  // PARK_BUCKETS - 1 - t
  const int b = PARK_BUCKETS - 1 - t;
  const int v = hist[b];
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, x, o);
    if ((t & 31) >= o) x += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = x;
  __syncthreads();
  if (t < 32) {
    int z = wsum[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, z, o);
      if (t >= o) z += y;
    }
    wsum[t] = z;  // inclusive over warps
  }
  __syncthreads();
  const int excl = x - v + ((t >> 5) ? wsum[(t >> 5) - 1] : 0);
  __syncthreads();
  hist[b] = excl;
  if (t == PARK_BUCKETS - 1) *count = excl + v;
  __syncthreads();
  for (int64_t i = t; i < m; i += PARK_BUCKETS) {
    const uint32_t k = key[i];
    if (k != PARK_DONE) order[atomicAdd(&hist[k], 1)] = (int32_t)i;
  }
}

// ------------------------------------------------------------ greedy_search
template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void greedy_kernel_one(const SearchArgs& a, uint8_t* smem_w, int* vring_lane, int64_t qi) {
  using Key = typename VecTraits<TX, TQ>::Key;
  const int lane = lane_id();
  WarpSearch<TX, TQ, LP> s;
  s.vr = vring_lane;
  init_search(s, a, smem_w, qi);
  load_query<TX, TQ>(s.qs, a, qi);
  set_layer(s, a.layer);
  s.dmax = a.dmax;
  s.reset();
  for (int base = 0; base < a.nseeds; base += 32) {
    const int cnt = min(32, a.nseeds - base);
    int sid = -1;
    Key sk = KeyOps<Key>::max_key();
    if (lane < cnt) {
      sid = a.seed_ids[qi * a.nseeds + base + lane];
      sk = KeyOps<Key>::from_d(a.seed_dists[qi * a.nseeds + base + lane]);
    }
    s.seed(sk, sid, cnt);
  }
  s.run();
  account(a.acc, s.visited, s.steps);
  write_hits(s, a, qi, a.layer.to_row, 0, 0);
}

template <typename TX, typename TQ, int LP>
__global__ void __launch_bounds__(SEARCH_THREADS, min_blocks<TX, TQ>()) greedy_kernel(const __grid_constant__ SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  int vring_lane[VR_SLOTS > 0 ? VR_SLOTS : 1];
  uint8_t* smem_w = smem + (size_t)(threadIdx.x >> 5) * a.region;
  if constexpr (GGNN_PERSISTENT != 0) {
    WorkCursor wc;
    for (int64_t qi = first_item(a.work, a.chunk, wc); qi < a.m; qi = next_item(a.work, wc))
      greedy_kernel_one<TX, TQ, LP>(a, smem_w, vring_lane, qi);
  } else {
    const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (qi < a.m) greedy_kernel_one<TX, TQ, LP>(a, smem_w, vring_lane, qi);
  }
}

// ------------------------------------------------------- hierarchical_query
template <typename TX, typename TQ, int LP>
__device__ __forceinline__ void descent_kernel_one(const SearchArgs& a, uint8_t* smem_w, int* vring_lane, int64_t qi) {
  using Key = typename VecTraits<TX, TQ>::Key;
  const int lane = lane_id();
  WarpSearch<TX, TQ, LP> s;
  s.vr = vring_lane;
  init_search(s, a, smem_w, qi);
  load_query<TX, TQ>(s.qs, a, qi);
  const LayerDev& Ls = a.layers[a.start];
  int lo = a.seg_lo ? __ldg(a.seg_lo + qi) : 0;
  int hi = a.seg_hi ? __ldg(a.seg_hi + qi) : (int)Ls.node_count;
  if (a.seg_size > 0) {
    const int seg = (a.seg_of ? __ldg(a.seg_of + qi) : (int)qi) / a.seg_div;
    lo = seg * a.seg_size;
    hi = min(lo + a.seg_size, (int)Ls.node_count);
  }
  const int kk = min(a.c.k_out, hi - lo);
  // distinct_touched: the scanned rows not seeded, plus every layer search's
  // logged ids (tagged by layer) counted after the launch
  int visited = hi - lo, steps = 0, distinct = (hi - lo) - kk, forgotten = 0, term = TERM_EMPTY;
  if (a.c.k_out <= 32) {  // hits fit the lanes: carried between layers in registers
    Key bk;
    int bi;
    warp_topk_scan<TX, TQ, LP>(s.X, a.d, s.qs, a.lpr, Ls.to_row, lo, hi, kk, s.crow, s.ckey, bk, bi);
    int id = lane < kk ? bi + lo : -1;
    int nh = kk;
    for (int j = a.start - 1; j >= a.stop; --j) {
      const LayerDev& Lj = a.layers[j];
      const int sid = lane < nh ? __ldg(a.layers[j + 1].down + id) : -1;
      set_layer(s, Lj);
      s.reset();
      s.log_tag = (uint32_t)j << 27;
      s.seed(bk, sid, nh);
      s.run();
      visited += s.visited;
      steps += s.steps;
      forgotten += s.forgotten;
      term = s.term;
      nh = s.hits(bk, id);
    }
    if (a.start == a.stop) {  // no search ran: the segment's top-kk goes into the ring for write_out
      set_layer(s, Ls);
      s.reset();
      uint32_t* const tl = s.tlog;
      s.tlog = nullptr;  // placing the scan's result is not a search (counted in `distinct` above)
      s.seed(bk, id, nh);
      s.tlog = tl;
    }
  } else {
    // k_out > 32: the segment scan in passes of 32 ranks seeds the ring of
    // the start layer; between layers the hits wait at the top of the ring
    // (stash) while the next layer's search is seeded from them
    set_layer(s, Ls);
    s.reset();
    uint32_t* const tl = s.tlog;
    s.tlog = nullptr;  // placing the scan's result is not a search (counted in `distinct` above)
    Key ak = 0;
    int ai = -1;
    for (int b = 0; b < kk; b += 32) {
      const int kc = min(32, kk - b);
      Key bk;
      int bi;
      warp_topk_scan<TX, TQ, LP>(s.X, a.d, s.qs, a.lpr, Ls.to_row, lo, hi, kc, s.crow, s.ckey, bk, bi, b > 0, ak, ai);
      ak = KeyOps<Key>::shfl(bk, kc - 1);
      ai = __shfl_sync(FULL, bi, kc - 1);
      s.seed(bk, lane < kc ? bi + lo : -1, kc);
    }
    s.tlog = tl;
    for (int j = a.start - 1; j >= a.stop; --j) {
      const int nh = min(s.L, a.c.k_out);
      s.stash(nh);
      const int32_t* down = a.layers[j + 1].down;
      set_layer(s, a.layers[j]);
      s.reset();
      s.log_tag = (uint32_t)j << 27;
      for (int b = 0; b < nh; b += 32) {
        Key sk = KeyOps<Key>::max_key();
        int sid = -1;
        if (b + lane < nh) {
          s.stashed(nh, b + lane, sk, sid);
          sid = __ldg(down + sid);
        }
        __syncwarp();
        s.seed(sk, sid, min(32, nh - b));
      }
      s.run();
      visited += s.visited;
      steps += s.steps;
      forgotten += s.forgotten;
      term = s.term;
    }
  }
  account(a.acc, visited, steps);
  const int k_out = a.c.k_out;
  s.write_out(a.layers[a.stop].to_row, (a.c.flags & FLAG_EXACT_DISTS) != 0, a.ids + qi * k_out,
              a.dists + qi * k_out);
  if (lane == 0 && a.counters) {
    int32_t* c = a.counters + qi * 5;
    c[0] = visited;
    c[1] = steps;
    c[2] = term;
    c[3] = a.ever == nullptr ? -1 : distinct;  // + the log's distinct ids (distinct_log_kernel)
    c[4] = forgotten;
  }
  finish_log(s, a, qi);
}

template <typename TX, typename TQ, int LP>
__global__ void __launch_bounds__(SEARCH_THREADS, min_blocks<TX, TQ>()) descent_kernel(const __grid_constant__ SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  int vring_lane[VR_SLOTS > 0 ? VR_SLOTS : 1];
  uint8_t* smem_w = smem + (size_t)(threadIdx.x >> 5) * a.region;
  if constexpr (GGNN_PERSISTENT != 0) {
    WorkCursor wc;
    for (int64_t qi = first_item(a.work, a.chunk, wc); qi < a.m; qi = next_item(a.work, wc))
      descent_kernel_one<TX, TQ, LP>(a, smem_w, vring_lane, qi);
  } else {
    const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (qi < a.m) descent_kernel_one<TX, TQ, LP>(a, smem_w, vring_lane, qi);
  }
}

// ----------------------------------------------------------- sym_check_pair
// Request records of a symmetrize pass (int32, stride REQ_HDR + n_fallback):
//   {pair index p, x, z, d_xz low word, d_xz high word, fallback[n_fallback]}
constexpr int REQ_HDR = 5;

struct SymArgs {
  const void* X;
  int64_t d;
  int lpr;
  LayerDev layer;
  const int32_t* px;
  const int32_t* pz;
  const double* pd;
  int64_t npairs;
  SearchCfg c;
  double dmax;
  size_t region;
  int n_fallback;
  int32_t* verdict;
  int32_t* fallback;
  // layer-pairs mode (px == nullptr, recheck == false): pair p = x * per_node + t,
  // t < k_nn is direct slot t of x (adj / nnd), t >= k_nn the (t - k_nn)-th rescued entry
  const double* nnd;
  int k_nn;
  const int32_t* resc_id;
  const double* resc_d;
  int per_node;
  // verdict-2 output (append) / recheck input
  int32_t* req;
  int32_t* req_count;
  int64_t req_cap;
  // recheck mode: item i is request i; stage[i] < 0 means settled.  A request
  // that is no longer verdict 2 on the current graph is settled as -3, else
  // its fallbacks are refreshed from the new search.
  bool recheck;
  int32_t* stage;
  int32_t x_end;  // recheck only requests of nodes x < x_end
  const int32_t* idx;  // recheck: the request of item i is idx[i] (nullptr: i)
  int* work;      // persistent-warp item counter (nullptr: one item per warp)
  int chunk;      // items claimed per counter update
  unsigned long long* acc;  // build accounting (visited, steps) or nullptr
};

template <typename TX, int LP>
__device__ __forceinline__ void symcheck_kernel_one(const SymArgs& a, uint8_t* smem_w, int* vring_lane, int64_t pi) {
  using Key = typename VecTraits<TX, TX>::Key;
  const int lane = lane_id();
  const int rstride = REQ_HDR + a.n_fallback;
  int x, z;
  double dxz;
  int32_t* rec = nullptr;
  if (a.recheck) {
    if (a.idx) pi = a.idx[pi];
    if (a.stage[pi] < 0) return;
    rec = a.req + pi * rstride;
    x = rec[1];
    if (x >= a.x_end) return;
    z = rec[2];
    dxz = __hiloint2double(rec[4], rec[3]);
  } else if (a.px) {
    x = __ldg(a.px + pi);
    z = __ldg(a.pz + pi);
    dxz = a.pd[pi];
  } else {
    x = (int)(pi / a.per_node);
    const int t = (int)(pi - (int64_t)x * a.per_node);
    if (t < a.k_nn) {
      z = __ldg(a.layer.adj + (int64_t)x * a.layer.k + t);
      dxz = z >= 0 ? a.nnd[(int64_t)x * a.k_nn + t] : 0.0;
    } else {
      const int64_t r = (int64_t)x * (a.per_node - a.k_nn) + (t - a.k_nn);
      z = a.resc_id ? __ldg(a.resc_id + r) : -1;
      dxz = z >= 0 ? a.resc_d[r] : 0.0;
    }
  }
  int32_t* fb = a.fallback ? a.fallback + pi * a.n_fallback : nullptr;
  if (z < 0) {  // empty slot: nothing to check
    if (lane == 0 && a.verdict) a.verdict[pi] = -1;
    return;
  }
  // verdict 0: x already sits in one of z's slots (_core.pyx:405-408)
  int slot = lane < a.layer.k ? __ldg(a.layer.adj + (int64_t)z * a.layer.k + lane) : -1;
  const bool present = __any_sync(FULL, slot == x);
  int v = 0;
  int cand = -1;
  WarpSearch<TX, TX, LP> s;
  s.vr = vring_lane;
  if (!present) {
    s.X = reinterpret_cast<const TX*>(a.X);
    s.d = a.d;
    s.lpr = a.lpr;
    s.c = a.c;
    s.target = x;
    s.carve(smem_w);
    s.tlog = nullptr;
    s.log_cap = 0;
    s.nlog = 0;
    s.log_tag = 0u;
    set_layer(s, a.layer);
    s.dmax = a.dmax;
    const int xrow = a.layer.to_row ? __ldg(a.layer.to_row + x) : x;
    const TX* src = s.X + (int64_t)xrow * a.d;
    for (int64_t e = lane; e < a.d; e += 32) s.qs[e] = src[e];
    __syncwarp();
    s.reset();
    s.seed(KeyOps<Key>::from_d(dxz), lane == 0 ? z : -1, 1);
    s.run();
    account(a.acc, s.visited, s.steps);
    v = s.term ? 1 : 2;
    // fallbacks: closest explored ids excluding x and z (_core.pyx:420-426)
    const int nh = min(s.L, a.c.k_out);
    if (v == 2 && lane < nh) cand = s.ring_id(lane);
  }
  if (lane == 0 && a.verdict) a.verdict[pi] = v;
  const bool keep = cand >= 0 && cand != x && cand != z;
  const unsigned km = __ballot_sync(FULL, keep);
  const int rank = __popc(km & lanemask_lt());
  const int w = min(__popc(km), a.n_fallback);
  if (fb) {
    if (keep && rank < a.n_fallback) fb[rank] = cand;
    for (int j = w + lane; j < a.n_fallback; j += 32) fb[j] = -1;
  }
  if (a.recheck) {
    if (v != 2) {
      if (lane == 0) a.stage[pi] = -3;
      return;
    }
  } else if (v == 2 && a.req) {
    int slot_i = 0;
    if (lane == 0) slot_i = atomicAdd(a.req_count, 1);
    slot_i = __shfl_sync(FULL, slot_i, 0);
    if (slot_i >= a.req_cap) return;
    rec = a.req + (int64_t)slot_i * rstride;
    if (lane == 0) {
      rec[0] = (int32_t)pi;
      rec[1] = x;
      rec[2] = z;
      rec[3] = __double2loint(dxz);
      rec[4] = __double2hiint(dxz);
    }
  } else {
    return;
  }
  if (keep && rank < a.n_fallback) rec[REQ_HDR + rank] = cand;
  for (int j = w + lane; j < a.n_fallback; j += 32) rec[REQ_HDR + j] = -1;
}

template <typename TX, int LP>
__global__ void __launch_bounds__(SYM_THREADS, SYM_MIN_BLOCKS) symcheck_kernel(const __grid_constant__ SymArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  int vring_lane[VR_SLOTS > 0 ? VR_SLOTS : 1];
  uint8_t* smem_w = smem + (size_t)(threadIdx.x >> 5) * a.region;
  if constexpr (GGNN_SYM_PERSISTENT != 0) {
    WorkCursor wc;
    for (int64_t pi = first_item(a.work, a.chunk, wc); pi < a.npairs; pi = next_item(a.work, wc))
      symcheck_kernel_one<TX, LP>(a, smem_w, vring_lane, pi);
  } else {
    const int64_t pi = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (pi < a.npairs) symcheck_kernel_one<TX, LP>(a, smem_w, vring_lane, pi);
  }
}

// ----------------------------------------------------------- exhaustive_topk
template <typename TX, typename TQ, int LP>
__global__ void __launch_bounds__(256) topk_kernel(const __grid_constant__ SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  using Key = typename VecTraits<TX, TQ>::Key;
  const int wib = threadIdx.x >> 5;
  const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (qi >= a.m) return;
  const int lane = lane_id();
  uint8_t* base = smem + (size_t)wib * a.region;
  int* crow = reinterpret_cast<int*>(base);
  Key* ckey = reinterpret_cast<Key*>(base + 128);
  TQ* qs = reinterpret_cast<TQ*>(base + 128 + align16(32 * sizeof(Key)));
  load_query<TX, TQ>(qs, a, qi);
  // k_out = the requested k (any size): ranks [b, b + 32) per pass
  const int k_out = a.c.k_out;
  const int kk = (int)min((int64_t)k_out, a.ntop);
  Key ak = 0;
  int ai = -1;
  for (int b = 0; b < k_out; b += 32) {
    const int kc = max(0, min(32, kk - b));
    double dv = __longlong_as_double(0x7ff0000000000000ll);
    int id = INT_MAX;
    if (kc > 0) {
      Key bk;
      int bi;
      warp_topk_scan<TX, TQ, LP>(reinterpret_cast<const TX*>(a.X), a.d, qs, a.lpr, a.top_rows, 0, (int)a.ntop, kc,
                                 crow, ckey, bk, bi, b > 0, ak, ai);
      ak = KeyOps<Key>::shfl(bk, kc - 1);
      ai = __shfl_sync(FULL, bi, kc - 1);
      if (lane < kc) {
        id = bi;
        dv = KeyOps<Key>::to_d(bk);
        if constexpr (sizeof(Key) == 8) {  // exact sequential FP64, then the (exact, row) order
          int row = a.top_rows ? __ldg(a.top_rows + bi) : bi;
          dv = seq_sqdist<TX, TQ>(reinterpret_cast<const TX*>(a.X) + (int64_t)row * a.d, qs, a.d);
        }
      }
      if constexpr (sizeof(Key) == 8) warp_sort(dv, id);
    }
    const int o = b + lane;
    if (o < k_out) {
      a.ids[qi * k_out + o] = lane < kc ? id : -1;
      a.dists[qi * k_out + o] = dv;
    }
  }
}

// --------------------------------------------------------- squared_l2_many
template <typename TX, typename TQ>
__global__ void sqdist_kernel(const TX* X, int64_t d, const TQ* Q, const int32_t* qrows, const int32_t* rows,
                              int per_query, int64_t total, double* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int64_t qi = i / per_query;
  const TQ* q = qrows ? reinterpret_cast<const TQ*>(X) + (int64_t)qrows[qi] * d : Q + qi * d;
  out[i] = seq_sqdist<TX, TQ>(X + (int64_t)rows[i] * d, q, d);
}

// ----------------------------------------------------------------- helpers
__global__ void sanitize_kernel(const int32_t* adj, const int32_t* symc, int64_t n, int k, int k_nn, int32_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * k) return;
  int64_t node = i / k;
  int j = (int)(i - node * k);
  int32_t v = adj[i];
  bool keep = j < k_nn ? v >= 0 : (j < k_nn + (symc ? symc[node] : 0));
  out[i] = keep ? v : -1;
}

__global__ void f32_to_u8_kernel(const float* src, int64_t count, uint8_t* dst, int32_t* flag) {
  int ok = 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    float v = src[i];
    bool good = v >= 0.0f && v <= 255.0f && v == rintf(v);
    ok &= good ? 1 : 0;
    if (dst) dst[i] = good ? (uint8_t)v : 0;
  }
  if (!__all_sync(FULL, ok) && (threadIdx.x & 31) == 0) atomicAnd(flag, 0);
}

}  // namespace ggnn

using namespace ggnn;

// ========================================================================= C ABI
namespace {

LayerDev to_dev(const ggnn_layer& l) {
  LayerDev d;
  d.adj = l.d_adj;
  d.to_row = l.d_to_row;
  d.down = l.d_down;
  d.node_count = l.node_count;
  d.k = l.k;
  d.slack = l.slack;
  return d;
}

int validate_params(const ggnn_search_params* p) {
  GGNN_CHECK_ARG(p != nullptr, "null search params");
  GGNN_CHECK_ARG(p->k_out >= 1, "k_out must be >= 1 (got %d)", p->k_out);
  GGNN_CHECK_ARG(p->prioq_size >= 1 && p->visited_size >= 1, "cache geometry values must be >= 1");
  // more than 32 hits are carried between passes at the top of the ring
  // (WarpSearch::stash), which needs ring capacity k_out + prioq >= 2 * k_out
  GGNN_CHECK_ARG(p->k_out <= 32 || p->prioq_size >= p->k_out,
                 "k_out > 32 needs prioq_size >= k_out (got k_out=%d, prioq_size=%d)", p->k_out, p->prioq_size);
  GGNN_CHECK_ARG(p->max_iterations >= 0, "max_iterations must be >= 0");
  return GGNN_OK;
}

SearchCfg make_cfg(const ggnn_search_params* p) {
  SearchCfg c;
  c.k_out = p->k_out;
  c.cap = p->k_out + p->prioq_size;
  c.vsz = p->visited_size;
  c.hlog = table_log2(c.cap, c.vsz);
  c.tau = p->tau;
  c.max_steps = p->max_iterations;
  c.flags = p->flags;
  return c;
}

// extra shared memory per CTA (occupancy experiments only: fewer resident
// searches per SM leave more of the unified L1/shared array to the L1)
#ifndef GGNN_SMEM_PAD
#define GGNN_SMEM_PAD 0
#endif

// choose warps per CTA so that the CTA fits in shared memory
int pick_warps(size_t region, int want) {
  DevInfo di = dev_info();
  size_t limit = di.smem_optin > 0 ? (size_t)di.smem_optin : (size_t)48 * 1024;
  int w = want;
  while (w > 1 && (size_t)w * region > limit) --w;
  return ((size_t)w * region > limit) ? 0 : w;
}

// Work counters for persistent launches: a per-device pool of ints, one slot
// per launch (round robin, zeroed on the launch's stream), so concurrent
// launches on different streams never share a counter.
constexpr int WORK_SLOTS = 4096;
int* work_counter(cudaStream_t st) {
  static std::mutex mu;
  static int* pools[64] = {nullptr};
  static unsigned next[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev] && cudaMalloc(&pools[dev], WORK_SLOTS * sizeof(int)) != cudaSuccess) {
    pools[dev] = nullptr;
    return nullptr;
  }
  int* slot = pools[dev] + (next[dev]++ % WORK_SLOTS);
  if (cudaMemsetAsync(slot, 0, sizeof(int), st) != cudaSuccess) return nullptr;
  return slot;
}

// Persistent grid: as many CTAs as fit on the device at once (never more
// than the items need); items are handed out through a work counter.
template <typename Kern>
int64_t persistent_grid(Kern kern, int threads, size_t smem, int64_t items_per_cta_max) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t resident = (int64_t)std::max(dev_info().sm_count, 1) * per_sm;
  return std::min(resident, items_per_cta_max);
}

template <typename Kern, typename Args>
int launch_items(Kern kern, Args a, int64_t items, size_t region, cudaStream_t st, int want, bool persistent = true,
                 int occ_cap = 0) {
  if (items <= 0) return GGNN_OK;
  int W = pick_warps(region, want);
  GGNN_CHECK_ARG(W > 0, "search state of %zu bytes does not fit in shared memory", region);
  size_t smem = (size_t)W * region + GGNN_SMEM_PAD;
  if (occ_cap > 0) {  // at most occ_cap CTAs per SM: pad the dynamic shared memory
    const size_t per_cta = (size_t)dev_info().smem_per_sm / (size_t)occ_cap;
    if (per_cta > smem + 1024) smem = std::min(per_cta - 1024, (size_t)dev_info().smem_optin);
  }
  GGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t grid = (items + W - 1) / W;
  a.work = persistent ? work_counter(st) : nullptr;
  a.chunk = 1;
  if (a.work) {
    grid = persistent_grid(kern, W * 32, smem, grid);
    a.chunk = (int)std::max<int64_t>(1, std::min<int64_t>(GGNN_WORK_CHUNK, items / (grid * W * 16)));
  }
  kern<<<(unsigned)grid, W * 32, smem, st>>>(a);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

template <typename Kern>
int launch_warps(Kern kern, const SearchArgs& a, int64_t items, size_t region, cudaStream_t st,
                 int want = SEARCH_WARPS) {
  return launch_items(kern, a, items, region, st, want, GGNN_PERSISTENT != 0);
}
// one item per warp (kernels without a work loop)
template <typename Kern>
int launch_static(Kern kern, const SearchArgs& a, int64_t items, size_t region, cudaStream_t st, int want,
                  int occ_cap = 0) {
  return launch_items(kern, a, items, region, st, want, false, occ_cap);
}

// ---- longest-first schedule of a query batch --------------------------------
// A batch of m searches on R resident warps runs in m / R waves; the launch
// ends when its longest searches do, and under FIFO some of those start in the
// last wave (C2: 1.88 ms per 10k queries against 1.22 ms when the same batch is
// launched longest-first).  So every search first runs a pilot of P
// expansions (GGNN_PILOT, default 8; 0 disables), the open ones are parked
// with a predicted-length bucket and sorted by one CTA; a second round runs
// them longest-predicted first up to GGNN_PILOT2 (default 32) expansions and
// parks the still-open ones again with a sharper prediction; the last round
// runs them to their ends, longest-predicted first (C2: 1.83 -> 1.53 ms).  Used for batches of at least 1.5 waves that need
// no distinct_touched logs; results are step-by-step those of the plain launch.
constexpr size_t PARK_MAX_BYTES = size_t(4) << 30;

long long g_pilot = -1;        // < 0: GGNN_PILOT or the default
double g_min_waves = 1.5;       // batches of fewer waves launch plainly
// uint8 batches of at least this many waves (of default residency) are
// throughput-bound rather than bound by their longest searches: their second
// round runs to GGNN_PILOT2_LARGE expansions and their last round is compiled
// for 32 CTAs per SM (ggnn_query_schedule_large; <= 0 disables)
double g_large_waves = 3.5;

long long pilot_steps() {
  if (g_pilot >= 0) return g_pilot;
  static const long long P = [] {
    const char* e = getenv("GGNN_PILOT");
    return e ? atoll(e) : 8LL;
  }();
  return P;
}
// second round: searches still open after the pilot run up to this many
// expansions in total and are parked again with a better prediction (the
// pending work is a sharper predictor later in the search); 0 = one round
long long pilot2_steps() {
  static const long long P = [] {
    const char* e = getenv("GGNN_PILOT2");
    return e ? atoll(e) : 32LL;
  }();
  return P;
}
long long pilot2_large_steps() {
  static const long long P = [] {
    const char* e = getenv("GGNN_PILOT2_LARGE");
    return e ? atoll(e) : 40LL;
  }();
  return P;
}
float pilot_weight() {
  static const float A = [] {
    const char* e = getenv("GGNN_PILOT_A");
    return e ? (float)atof(e) : 0.5f;
  }();
  return A;
}

// stream-ordered park buffers stay in the device's default pool between
// batches instead of being returned to the driver at every synchronisation
void keep_default_pool() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

template <typename Kern>
int64_t resident_searches(Kern kern, size_t region) {
  const int W = pick_warps(region, SEARCH_WARPS);
  if (W <= 0) return 0;
  const size_t smem = (size_t)W * region + GGNN_SMEM_PAD;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem) != cudaSuccess) return 0;
  return (int64_t)per_sm * W * std::max(dev_info().sm_count, 1);
}

template <typename TX, typename TQ, int LP, bool STAGED>
int launch_query(SearchArgs a, cudaStream_t st) {
  auto qk = query_kernel<TX, TQ, LP, false, STAGED>;
  const long long P = pilot_steps();
  const size_t slot = WarpSearch<TX, TQ, LP>::park_bytes(a.c, a.d * (int64_t)sizeof(TQ));
  const size_t bytes = (size_t)a.m * (slot + 8) + 16;
  bool sched = P > 0 && !a.ever && a.m > 0 && bytes <= PARK_MAX_BYTES && a.c.max_steps > P;
  bool large = false;
  if (sched) {
    const int64_t res = resident_searches(qk, a.region);
    sched = res > 0 && (double)a.m >= g_min_waves * (double)res;
    large = sched && sizeof(TX) == 1 && sizeof(TQ) == 1 && g_large_waves > 0.0 &&
            (double)a.m >= g_large_waves * (double)res;
  }
  if (!sched) return launch_warps(qk, a, a.m, a.region, st);
  keep_default_pool();
  uint8_t* buf = nullptr;
  GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st));
  a.pilot = P;
  a.park_a = pilot_weight();
  a.park = buf;
  a.park_slot = slot;
  a.park_key = reinterpret_cast<uint32_t*>(buf + (size_t)a.m * slot);
  int32_t* order = reinterpret_cast<int32_t*>(buf + (size_t)a.m * (slot + 4));
  int32_t* count = reinterpret_cast<int32_t*>(buf + (size_t)a.m * (slot + 8));
  int rc = launch_warps(qk, a, a.m, a.region, st);
  if (rc == GGNN_OK) {
    park_order_kernel<<<1, PARK_BUCKETS, 0, st>>>(a.park_key, a.m, order, count);
    count_launch();
    rc = cudaGetLastError() == cudaSuccess ? GGNN_OK : GGNN_E_CUDA;
    if (rc) set_error("park_order_kernel launch failed");
  }
  const long long P2 = large ? pilot2_large_steps() : pilot2_steps();
  SearchArgs b = a;
  b.park_order = order;
  b.park_count = count;
  if (rc == GGNN_OK && P2 > P && a.c.max_steps > P2) {
    b.pilot = P2;
    constexpr int MB1 = (sizeof(TX) == 1 && sizeof(TQ) == 1) ? GGNN_ROUND1_MIN_BLOCKS : 0;
    rc = launch_static(resume_kernel<TX, TQ, LP, MB1>, b, a.m, a.region, st, SEARCH_WARPS);
    if (rc == GGNN_OK) {
      park_order_kernel<<<1, PARK_BUCKETS, 0, st>>>(a.park_key, a.m, order, count);
      count_launch();
      rc = cudaGetLastError() == cudaSuccess ? GGNN_OK : GGNN_E_CUDA;
      if (rc) set_error("park_order_kernel launch failed");
    }
  }
  if (rc == GGNN_OK) {
    b.pilot = 0;
    static const int occ = [] {
      const char* e = getenv("GGNN_OCC_CAP");
      return e ? atoi(e) : 0;
    }();
    constexpr int MB1 = (sizeof(TX) == 1 && sizeof(TQ) == 1) ? GGNN_ROUND1_MIN_BLOCKS : 0;
    if (large) rc = launch_static(resume_kernel<TX, TQ, LP, MB1>, b, a.m, a.region, st, SEARCH_WARPS, occ);
    else rc = launch_static(resume_kernel<TX, TQ, LP>, b, a.m, a.region, st, SEARCH_WARPS, occ);
  }
  cudaFreeAsync(buf, st);
  return rc;
}

template <bool STAGED>
int launch_query_combo(const SearchArgs& a, int cmb, cudaStream_t st) {
  switch (cmb) {
    case 0:
      if (a.lpr == 8) return launch_query<float, float, 8, STAGED>(a, st);
      if (a.lpr == 32) return launch_query<float, float, 32, STAGED>(a, st);
      return launch_query<float, float, 0, STAGED>(a, st);
    case 1:
      if (a.lpr == 8) return launch_query<uint8_t, uint8_t, 8, STAGED>(a, st);
      if (a.lpr == 32) return launch_query<uint8_t, uint8_t, 32, STAGED>(a, st);
      return launch_query<uint8_t, uint8_t, 0, STAGED>(a, st);
    default:
      return launch_query<uint8_t, float, 0, STAGED>(a, st);
  }
}

// Launch the LP-specialised instantiation matching a.lpr (see warp_dists_t).
#define GGNN_LAUNCH_LP(KER, TX, TQ, ...)                                          \
  (a.lpr == 8    ? launch_warps(KER<TX, TQ, 8>, __VA_ARGS__)                     \
   : a.lpr == 32 ? launch_warps(KER<TX, TQ, 32>, __VA_ARGS__)                    \
                 : launch_warps(KER<TX, TQ, 0>, __VA_ARGS__))

template <typename TX>
int launch_sym(const SymArgs& a, int64_t items, cudaStream_t st) {
  const bool pers = GGNN_SYM_PERSISTENT != 0;
  if (a.lpr == 8) return launch_items(symcheck_kernel<TX, 8>, a, items, a.region, st, SYM_THREADS / 32, pers);
  if (a.lpr == 32) return launch_items(symcheck_kernel<TX, 32>, a, items, a.region, st, SYM_THREADS / 32, pers);
  return launch_items(symcheck_kernel<TX, 0>, a, items, a.region, st, SYM_THREADS / 32, pers);
}

int qelem_of(int dtype) { return dtype == GGNN_U8 ? 1 : 4; }

int fill_common(SearchArgs& a, const ggnn_vectors* X, const ggnn_queries* Q, const ggnn_search_params* p) {
  GGNN_CHECK_ARG(X && X->d_data && X->d > 0 && X->n > 0, "invalid vector table");
  GGNN_CHECK_ARG(X->dtype == GGNN_F32 || X->dtype == GGNN_U8, "unknown vector dtype %d", X->dtype);
  GGNN_CHECK_ARG(Q && (Q->d_data || Q->d_rows) && Q->m >= 0, "invalid queries");
  int qd = Q->d_rows ? X->dtype : Q->dtype;
  GGNN_CHECK_ARG(qd == GGNN_F32 || qd == GGNN_U8, "unknown query dtype %d", qd);
  GGNN_CHECK_ARG(!(X->dtype == GGNN_F32 && qd == GGNN_U8), "uint8 queries need uint8 vectors");
  int rc = validate_params(p);
  if (rc) return rc;
  memset(&a, 0, sizeof(a));
  a.acc = g_acc;
  a.X = X->d_data;
  a.n = X->n;
  a.d = X->d;
  a.lpr = choose_lpr(X->d, X->dtype, qd, reinterpret_cast<uintptr_t>(X->d_data));
  a.Q = Q->d_rows ? nullptr : Q->d_data;
  a.qrows = Q->d_rows;
  a.m = Q->m;
  a.c = make_cfg(p);
  int keysize = (X->dtype == GGNN_U8 && qd == GGNN_U8) ? 4 : 8;
  a.region = set_layout(a.c, X->d, qelem_of(qd), keysize);
  return GGNN_OK;
}

int combo(const ggnn_vectors* X, const ggnn_queries* Q) {
  int qd = Q->d_rows ? X->dtype : Q->dtype;
  if (X->dtype == GGNN_F32) return 0;          // f32 / f32
  return qd == GGNN_U8 ? 1 : 2;                // u8 / u8, u8 / f32
}

// Exact distinct_touched: each search appends every id it inserts to a
// per-query log in the workspace (no atomics, nothing on the search's
// critical path waits on it) and distinct_log_kernel counts the distinct
// entries after the launch.  ggnn_search_workspace_bytes asks for COMPACT_LOG
// entries per query (typical searches log ~1-2 k); a longer log reports
// distinct_touched = -1 and the caller reruns those queries with a workspace
// of the exact size (attach_ever takes whatever capacity the workspace holds).
constexpr uint32_t COMPACT_LOG = 4096;
constexpr uint32_t LOG_SMEM_SLOTS = 32768;  // counting table in shared memory up to this size

uint32_t log_entries_for(const ggnn_search_params* p, int32_t max_seeds, int k) {
  // one layer's search inserts at most its seeds plus k ids per step; twice
  // that also covers a descent's coarse layers (a longer log reports -1)
  const uint64_t one = (uint64_t)std::max(max_seeds, 0) + (uint64_t)std::max<int64_t>(p->max_iterations, 1) * k;
  return (uint32_t)std::min<uint64_t>(2 * one + 64, 1u << 28);
}

size_t log_bytes(int64_t m, uint32_t cap) { return (size_t)m * cap * 4 + (size_t)m * 4; }

int attach_ever(SearchArgs& a, const ggnn_search_params* p, int32_t max_seeds, int k, void* ws, size_t wsb) {
  if (!(p->flags & GGNN_FLAG_DISTINCT) || a.m <= 0) return GGNN_OK;
  const uint32_t full = log_entries_for(p, max_seeds, k);
  const uint32_t small = std::min(full, COMPACT_LOG);
  GGNN_CHECK_ARG(ws != nullptr && wsb >= log_bytes(a.m, small),
                 "GGNN_FLAG_DISTINCT needs %zu bytes of workspace (exact: %zu)", log_bytes(a.m, small),
                 log_bytes(a.m, full));
  const size_t per = (wsb - (size_t)a.m * 4) / ((size_t)a.m * 4);
  a.ever = reinterpret_cast<uint32_t*>(ws);
  a.ever_size = (uint32_t)std::min<size_t>(per, full);
  a.log_len = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ws) + (size_t)a.m * a.ever_size * 4);
  return GGNN_OK;
}

// One CTA per query: insert its logged ids into an open-addressing set (shared
// memory, or global scratch for very long logs) and add the number of new
// ones to counter column 3; an overflowed log gives -1.
__global__ void __launch_bounds__(256) distinct_log_kernel(const uint32_t* logs, const int32_t* len, uint32_t cap,
                                                           int32_t* counters, uint32_t slots, uint32_t* gtab) {
  extern __shared__ uint32_t tab_s[];
  __shared__ int total;
  const int64_t qi = blockIdx.x;
  const int n = len[qi];
  if (n < 0) {
    if (threadIdx.x == 0) counters[qi * 5 + 3] = -1;
    return;
  }
  uint32_t* tab = gtab ? gtab + (size_t)qi * slots : tab_s;
  for (uint32_t i = threadIdx.x; i < slots; i += blockDim.x) tab[i] = 0u;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  const uint32_t* lg = logs + (size_t)qi * cap;
  const uint32_t mask = slots - 1u;
  int fresh = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t key = lg[i] + 1u;
    uint32_t h = (key * 2654435761u) & mask;
    for (;;) {
      const uint32_t o = atomicCAS(&tab[h], 0u, key);
      if (o == 0u) {
        ++fresh;
        break;
      }
      if (o == key) break;
      h = (h + 1u) & mask;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fresh += __shfl_xor_sync(FULL, fresh, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&total, fresh);
  __syncthreads();
  if (threadIdx.x == 0) counters[qi * 5 + 3] += total;
}

int count_distinct(const SearchArgs& a, cudaStream_t st) {
  if (!a.ever || !a.counters || a.m <= 0) return GGNN_OK;
  uint32_t slots = 64;
  while ((uint64_t)slots * 3 < (uint64_t)a.ever_size * 4) slots <<= 1;  // load <= 3/4
  uint32_t* g = nullptr;
  size_t smem = (size_t)slots * 4;
  if (slots > LOG_SMEM_SLOTS) {
    GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&g), (size_t)a.m * slots * 4, st));
    smem = 0;
  } else {
    GGNN_CUDA_TRY(cudaFuncSetAttribute(distinct_log_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  distinct_log_kernel<<<(unsigned)a.m, 256, smem, st>>>(a.ever, a.log_len, a.ever_size, a.counters, slots, g);
  count_launch();
  GGNN_LAUNCH_CHECK();
  if (g) GGNN_CUDA_TRY(cudaFreeAsync(g, st));
  return GGNN_OK;
}

}  // namespace

extern "C" {

const char* ggnn_last_error(void) { return g_err.c_str(); }

int ggnn_search_accounting(unsigned long long* d_acc) {
  g_acc = d_acc;
  return GGNN_OK;
}
unsigned long long ggnn_kernel_launches(void) { return ggnn::g_kernel_launches.load(); }

int ggnn_query_schedule_large(double large_waves) {
  g_large_waves = large_waves;
  return GGNN_OK;
}

int ggnn_query_schedule(long long pilot_steps, double min_waves) {
  GGNN_CHECK_ARG(min_waves >= 0.0, "min_waves must be >= 0");
  g_pilot = pilot_steps;
  g_min_waves = min_waves;
  return GGNN_OK;
}

int ggnn_version(void) { return 100; }

int ggnn_device_info(int* sm_count, int* smem_per_block) {
  DevInfo di = dev_info();
  if (sm_count) *sm_count = di.sm_count;
  if (smem_per_block) *smem_per_block = di.smem_optin;
  return di.sm_count > 0 ? GGNN_OK : GGNN_E_CUDA;
}

size_t ggnn_search_workspace_bytes(int64_t m, const ggnn_search_params* p, int32_t max_seeds) {
  if (!p || !(p->flags & GGNN_FLAG_DISTINCT)) return 0;
  // max_seeds < 0: room for the exact log of every query (any seed count <= max(32, k_out))
  const uint32_t full = log_entries_for(p, max_seeds < 0 ? std::max(32, p->k_out) : max_seeds, MAX_K);
  if (max_seeds < 0) return log_bytes(m, full);
  return log_bytes(m, std::min(full, COMPACT_LOG));
}

__global__ void rows_unique_kernel(const int32_t* adj, int64_t node_count, int k, int32_t* result) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= node_count) return;
  const int lane = lane_id();
  const int32_t v = lane < k ? adj[row * k + lane] : -1;
  const unsigned same = __match_any_sync(FULL, v >= 0 ? (unsigned)v : (0x80000000u | (unsigned)lane));
  if (v >= 0 && (same & ~(1u << lane))) *result = 0;
}

int ggnn_rows_unique(const int32_t* d_adj, int64_t node_count, int32_t k, int32_t* d_result, void* stream) {
  GGNN_CHECK_ARG(d_adj && d_result && node_count >= 0 && k >= 1 && k <= 32, "invalid arguments");
  cudaStream_t st = as_stream(stream);
  const int32_t one = 1;
  GGNN_CUDA_TRY(cudaMemcpyAsync(d_result, &one, sizeof(one), cudaMemcpyHostToDevice, st));
  if (node_count == 0) return GGNN_OK;
  rows_unique_kernel<<<(unsigned)((node_count + 7) / 8), 256, 0, st>>>(d_adj, node_count, k, d_result);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

int ggnn_sanitize_layer(const int32_t* d_adj, const int32_t* d_sym_count, int64_t node_count, int32_t k,
                        int32_t k_nn, int32_t* d_out, void* stream) {
  GGNN_CHECK_ARG(d_adj && d_out && node_count >= 0 && k >= 1 && k <= MAX_K && k_nn >= 1 && k_nn <= k,
                 "invalid layer geometry (k=%d, k_nn=%d; k <= %d supported)", k, k_nn, MAX_K);
  int64_t total = node_count * k;
  if (total == 0) return GGNN_OK;
  sanitize_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(d_adj, d_sym_count, node_count, k,
                                                                                   k_nn, d_out);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

int ggnn_query_batch(const ggnn_vectors* X, const ggnn_layer* bottom, const int32_t* d_top_rows, int64_t ntop,
                     const ggnn_queries* Q, const ggnn_search_params* p, double d_nn1_max, int32_t* d_ids,
                     double* d_dists, int32_t* d_counters, void* d_workspace, size_t workspace_bytes,
                     void* stream) {
  SearchArgs a;
  int rc = fill_common(a, X, Q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(bottom && bottom->d_adj && bottom->k >= 1 && bottom->k <= MAX_K, "invalid bottom layer");
  GGNN_CHECK_ARG(ntop >= 1, "the top layer is empty");
  GGNN_CHECK_ARG(d_ids && d_dists, "null outputs");
  a.layer = to_dev(*bottom);
  a.top_rows = d_top_rows;
  a.ntop = ntop;
  a.dmax = d_nn1_max;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  rc = attach_ever(a, p, p->k_out, bottom->k, d_workspace, workspace_bytes);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  rc = launch_query_combo<false>(a, combo(X, Q), st);
  return rc ? rc : count_distinct(a, st);
}

int ggnn_query_batch_push(const ggnn_vectors* X, const ggnn_layer* bottom, const int32_t* d_top_rows, int64_t ntop,
                          const ggnn_queries* Q, const ggnn_search_params* p, double d_nn1_max, int32_t* d_ids,
                          double* d_dists, int32_t* d_counters, const ggnn_push* push, void* stream) {
  SearchArgs a;
  int rc = fill_common(a, X, Q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(!(p->flags & GGNN_FLAG_DISTINCT), "the push search does not track distinct_touched");
  GGNN_CHECK_ARG(bottom && bottom->d_adj && bottom->k >= 1 && bottom->k <= MAX_K, "invalid bottom layer");
  GGNN_CHECK_ARG(ntop >= 1, "the top layer is empty");
  GGNN_CHECK_ARG(d_ids && d_dists && d_counters, "null outputs");
  GGNN_CHECK_ARG(push && push->nranks >= 1 && push->nranks <= GGNN_P2P_MAX_RANKS && push->rank >= 0 &&
                     push->rank < push->nranks && (push->parity == 0 || push->parity == 1) && push->d_gid_of_local,
                 "invalid push descriptor");
  a.layer = to_dev(*bottom);
  a.top_rows = d_top_rows;
  a.ntop = ntop;
  a.dmax = d_nn1_max;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  const size_t bb = ggnn_shard_block_bytes(a.m, p->k_out);
  const size_t half = (size_t)push->nranks * bb + (((size_t)push->nranks * 4 + 255) & ~size_t(255));
  for (int g = 0; g < push->nranks; ++g) {
    GGNN_CHECK_ARG(push->d_peers[g] != nullptr, "push: receive allocation %d missing", g);
    a.push_peers[g] = static_cast<uint8_t*>(push->d_peers[g]) + (size_t)push->parity * half;
  }
  a.push_n = push->nranks;
  a.push_rank = push->rank;
  a.push_half = half;
  a.push_bb = bb;
  a.push_doff = ggnn_shard_block_dists_offset(a.m, p->k_out);
  a.push_coff = ggnn_shard_block_counters_offset(a.m, p->k_out);
  a.push_gid = push->d_gid_of_local;
  a.push_gid_size = push->gid_size;
  cudaStream_t st = as_stream(stream);
  switch (combo(X, Q)) {
    case 0:
      if (a.lpr == 32) return launch_warps(query_kernel<float, float, 32, true>, a, a.m, a.region, st);
      if (a.lpr == 8) return launch_warps(query_kernel<float, float, 8, true>, a, a.m, a.region, st);
      return launch_warps(query_kernel<float, float, 0, true>, a, a.m, a.region, st);
    case 1:
      if (a.lpr == 32) return launch_warps(query_kernel<uint8_t, uint8_t, 32, true>, a, a.m, a.region, st);
      if (a.lpr == 8) return launch_warps(query_kernel<uint8_t, uint8_t, 8, true>, a, a.m, a.region, st);
      return launch_warps(query_kernel<uint8_t, uint8_t, 0, true>, a, a.m, a.region, st);
    default: return launch_warps(query_kernel<uint8_t, float, 0, true>, a, a.m, a.region, st);
  }
}

int ggnn_query_batch_staged(const ggnn_vectors* X, const ggnn_layer* bottom, const int32_t* d_top_rows, int64_t ntop,
                            const float* d_q_f32, int64_t m, const ggnn_search_params* p, double d_nn1_max,
                            const uint32_t* d_chunk_flags, int64_t chunk_rows, uint32_t epoch, int32_t narrow,
                            int32_t* d_ids, double* d_dists, int32_t* d_counters, int32_t* d_status, void* stream) {
  GGNN_CHECK_ARG(X && d_q_f32 && (!d_chunk_flags || chunk_rows >= 1) && d_status, "invalid staged query arguments");
  GGNN_CHECK_ARG(!narrow || X->dtype == GGNN_U8, "narrowing needs a uint8 table");
  ggnn_queries Q;
  Q.d_data = d_q_f32;
  Q.d_rows = nullptr;
  Q.m = m;
  Q.dtype = narrow ? GGNN_U8 : GGNN_F32;
  Q.pad_ = 0;
  SearchArgs a;
  int rc = fill_common(a, X, &Q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(!(p->flags & GGNN_FLAG_DISTINCT), "the staged search does not track distinct_touched");
  GGNN_CHECK_ARG(bottom && bottom->d_adj && bottom->k >= 1 && bottom->k <= MAX_K, "invalid bottom layer");
  GGNN_CHECK_ARG(ntop >= 1, "the top layer is empty");
  GGNN_CHECK_ARG(d_ids && d_dists && d_counters, "null outputs");
  a.layer = to_dev(*bottom);
  a.top_rows = d_top_rows;
  a.ntop = ntop;
  a.dmax = d_nn1_max;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  a.qflags = d_chunk_flags;
  a.qchunk = chunk_rows;
  a.qepoch = epoch;
  a.qconv = narrow ? 1 : 0;
  a.qstatus = d_status;
  cudaStream_t st = as_stream(stream);
  return launch_query_combo<true>(a, combo(X, &Q), st);
}

// Device address of a page-locked host buffer, or nullptr for pageable memory.
static void* mapped_host(const void* h) {
  cudaPointerAttributes pa;
  if (cudaPointerGetAttributes(&pa, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return pa.type == cudaMemoryTypeHost ? pa.devicePointer : nullptr;
}

static bool zero_copy_enabled() {
  static const bool on = [] {
    const char* e = getenv("GGNN_ZERO_COPY");
    return !(e && e[0] == '0');
  }();
  return on;
}

int ggnn_query_batch_host(const ggnn_vectors* X, const ggnn_layer* bottom, const int32_t* d_top_rows, int64_t ntop,
                          const float* h_q, int64_t m, const ggnn_search_params* p, double d_nn1_max, float* d_q_stage,
                          uint32_t* d_chunk_flags, const uint32_t* h_epoch, int32_t nchunks, int32_t narrow,
                          int32_t* d_ids, double* d_dists, int32_t* d_counters, int32_t* d_status, int32_t* h_ids,
                          double* h_dists, int32_t* h_counters, int32_t* h_status, void* search_stream,
                          void* copy_stream) {
  GGNN_CHECK_ARG(X && h_q && d_q_stage && d_chunk_flags && h_epoch && nchunks >= 1 && m >= 1 && h_ids && h_dists &&
                     h_counters && h_status,
                 "invalid host query arguments");
  cudaStream_t ss = as_stream(search_stream), cs = as_stream(copy_stream);
  const int64_t d = X->d;
  const int64_t rows = (m + nchunks - 1) / nchunks;
  const int k = p ? p->k_out : 0;
  auto upload = [&](int64_t c) -> int {
    const int64_t lo = c * rows, hi = std::min(m, lo + rows);
    if (lo >= hi) return GGNN_OK;
    GGNN_CUDA_TRY(cudaMemcpyAsync(d_q_stage + lo * d, h_q + lo * d, (size_t)(hi - lo) * d * sizeof(float),
                                  cudaMemcpyHostToDevice, cs));
    GGNN_CUDA_TRY(cudaMemcpyAsync(d_chunk_flags + c, h_epoch, sizeof(uint32_t), cudaMemcpyHostToDevice, cs));
    return GGNN_OK;
  };
  GGNN_CUDA_TRY(cudaMemsetAsync(d_status, 0, sizeof(int32_t), ss));
  // Zero copy: when the query rows and the three result arrays are pinned
  // (page-locked host memory is mapped into the device's address space) the
  // search reads each query row over PCIe as its warp starts it and writes
  // its hits back as it finishes: no upload chunks, no flags and no trailing
  // device-to-host copies -- the transfers hide under the search itself.
  const void* zq = mapped_host(h_q);
  void* zi = mapped_host(h_ids);
  void* zd = mapped_host(h_dists);
  void* zc = mapped_host(h_counters);
  if (zq && zi && zd && zc && zero_copy_enabled()) {
    int rc = ggnn_query_batch_staged(X, bottom, d_top_rows, ntop, static_cast<const float*>(zq), m, p, d_nn1_max,
                                     nullptr, 1, 0, narrow, static_cast<int32_t*>(zi), static_cast<double*>(zd),
                                     static_cast<int32_t*>(zc), d_status, search_stream);
    if (rc) return rc;
    GGNN_CUDA_TRY(cudaMemcpyAsync(h_status, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, ss));
    return GGNN_OK;
  }
  // Every upload is queued before the search is launched: from pinned memory
  // the queueing is asynchronous, so the search still starts while the
  // chunks are in flight, and when the two streams cannot overlap (a
  // profiler serialising work, CUDA_LAUNCH_BLOCKING) the chunks are already
  // there instead of being queued behind a search that waits for them.
  for (int64_t c = 0; c < nchunks; ++c) {
    int rc = upload(c);
    if (rc) return rc;
  }
  int rc = ggnn_query_batch_staged(X, bottom, d_top_rows, ntop, d_q_stage, m, p, d_nn1_max, d_chunk_flags, rows,
                                   *h_epoch, narrow, d_ids, d_dists, d_counters, d_status, search_stream);
  if (rc) return rc;
  GGNN_CUDA_TRY(cudaMemcpyAsync(h_ids, d_ids, (size_t)m * k * sizeof(int32_t), cudaMemcpyDeviceToHost, ss));
  GGNN_CUDA_TRY(cudaMemcpyAsync(h_dists, d_dists, (size_t)m * k * sizeof(double), cudaMemcpyDeviceToHost, ss));
  GGNN_CUDA_TRY(cudaMemcpyAsync(h_counters, d_counters, (size_t)m * 5 * sizeof(int32_t), cudaMemcpyDeviceToHost, ss));
  GGNN_CUDA_TRY(cudaMemcpyAsync(h_status, d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, ss));
  return GGNN_OK;
}

int ggnn_greedy_batch(const ggnn_vectors* X, const ggnn_layer* layer, const ggnn_queries* Q,
                      const int32_t* d_seed_ids, const double* d_seed_dists, int32_t nseeds,
                      const ggnn_search_params* p, double d_nn1_max, int32_t* d_ids, double* d_dists,
                      int32_t* d_counters, void* d_workspace, size_t workspace_bytes, void* stream) {
  SearchArgs a;
  int rc = fill_common(a, X, Q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(layer && layer->d_adj && layer->k >= 1 && layer->k <= MAX_K, "invalid layer");
  GGNN_CHECK_ARG(nseeds >= 1 && d_seed_ids && d_seed_dists, "greedy search needs at least one seed");
  GGNN_CHECK_ARG(nseeds <= a.c.cap, "more seeds (%d) than cache capacity (%d)", nseeds, a.c.cap);
  a.layer = to_dev(*layer);
  a.dmax = d_nn1_max;
  a.seed_ids = d_seed_ids;
  a.seed_dists = d_seed_dists;
  a.nseeds = nseeds;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  rc = attach_ever(a, p, nseeds, layer->k, d_workspace, workspace_bytes);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  switch (combo(X, Q)) {
    case 0: rc = GGNN_LAUNCH_LP(greedy_kernel, float, float, a, a.m, a.region, st); break;
    case 1: rc = GGNN_LAUNCH_LP(greedy_kernel, uint8_t, uint8_t, a, a.m, a.region, st); break;
    default: rc = launch_warps(greedy_kernel<uint8_t, float, 0>, a, a.m, a.region, st); break;
  }
  return rc ? rc : count_distinct(a, st);
}

int ggnn_descent_batch(const ggnn_vectors* X, const ggnn_layer* layers, int32_t num_layers, int32_t start,
                       int32_t stop, const ggnn_queries* Q, const int32_t* d_seg_lo, const int32_t* d_seg_hi,
                       const ggnn_search_params* p, int32_t* d_ids, double* d_dists, int32_t* d_counters,
                       void* d_workspace, size_t workspace_bytes, void* stream) {
  SearchArgs a;
  int rc = fill_common(a, X, Q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(layers && num_layers >= 1 && num_layers <= MAX_LAYERS, "1..%d layers supported", MAX_LAYERS);
  GGNN_CHECK_ARG(0 <= stop && stop <= start && start < num_layers, "invalid layer range %d..%d for %d layers",
                 start, stop, num_layers);
  for (int j = 0; j < num_layers; ++j) {
    GGNN_CHECK_ARG(layers[j].k >= 1 && layers[j].k <= MAX_K, "invalid layer %d", j);
    if (j > stop && j <= start) GGNN_CHECK_ARG(layers[j].d_down != nullptr, "layer %d needs a down map", j);
    a.layers[j] = to_dev(layers[j]);
  }
  if (p->flags & GGNN_FLAG_DISTINCT)  // distinct_touched logs tag ids with their layer (bits 27..31)
    for (int j = stop; j <= start; ++j)
      GGNN_CHECK_ARG(layers[j].node_count < (1 << 27), "distinct_touched on descents needs layers below 2^27 nodes");
  a.start = start;
  a.stop = stop;
  a.seg_lo = d_seg_lo;
  a.seg_hi = d_seg_hi;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  rc = attach_ever(a, p, p->k_out, MAX_K, d_workspace, workspace_bytes);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  switch (combo(X, Q)) {
    case 0: rc = GGNN_LAUNCH_LP(descent_kernel, float, float, a, a.m, a.region, st); break;
    case 1: rc = GGNN_LAUNCH_LP(descent_kernel, uint8_t, uint8_t, a, a.m, a.region, st); break;
    default: rc = launch_warps(descent_kernel<uint8_t, float, 0>, a, a.m, a.region, st); break;
  }
  return rc ? rc : count_distinct(a, st);
}

int ggnn_merge_descent(const ggnn_vectors* X, const ggnn_layer* layers, int32_t num_layers, int32_t start,
                       int32_t stop, const int32_t* d_query_rows, int64_t m, const int32_t* d_seg_of, int32_t seg_div,
                       int32_t seg_size, const ggnn_search_params* p, int32_t* d_ids, double* d_dists,
                       int32_t* d_counters, void* stream) {
  GGNN_CHECK_ARG(d_query_rows && seg_div >= 1 && seg_size >= 1, "invalid merge descent arguments");
  ggnn_queries q{nullptr, d_query_rows, m, X ? X->dtype : 0, 0};
  SearchArgs a;
  int rc = fill_common(a, X, &q, p);
  if (rc) return rc;
  GGNN_CHECK_ARG(layers && num_layers >= 1 && num_layers <= MAX_LAYERS, "1..%d layers supported", MAX_LAYERS);
  GGNN_CHECK_ARG(0 <= stop && stop <= start && start < num_layers, "invalid layer range");
  for (int j = 0; j < num_layers; ++j) {
    GGNN_CHECK_ARG(layers[j].k >= 1 && layers[j].k <= MAX_K, "invalid layer %d", j);
    if (j > stop && j <= start) GGNN_CHECK_ARG(layers[j].d_down != nullptr, "layer %d needs a down map", j);
    a.layers[j] = to_dev(layers[j]);
  }
  a.start = start;
  a.stop = stop;
  a.seg_of = d_seg_of;
  a.seg_div = seg_div;
  a.seg_size = seg_size;
  a.ids = d_ids;
  a.dists = d_dists;
  a.counters = d_counters;
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_F32) return GGNN_LAUNCH_LP(descent_kernel, float, float, a, a.m, a.region, st);
  return GGNN_LAUNCH_LP(descent_kernel, uint8_t, uint8_t, a, a.m, a.region, st);
}

int ggnn_sym_check_layer(const ggnn_vectors* X, const ggnn_layer* layer, const double* d_nnd,
                         const int32_t* d_resc_id, const double* d_resc_d, int32_t per_node, double tau,
                         double d_nn1_max, int32_t budget, int32_t k_out, int32_t prioq_size, int32_t visited_size,
                         int32_t n_fallback, int32_t* d_req, int32_t* d_req_count, int64_t req_cap, void* stream) {
  GGNN_CHECK_ARG(X && X->d_data && layer && layer->d_adj && d_nnd && d_req && d_req_count, "invalid arguments");
  GGNN_CHECK_ARG(layer->k >= 1 && layer->k <= MAX_K && per_node >= layer->k_nn, "invalid layer geometry");
  GGNN_CHECK_ARG(k_out >= 1 && k_out <= 32 && n_fallback >= 0 && n_fallback <= 32, "k_out / n_fallback in [1, 32]");
  int64_t npairs = layer->node_count * per_node;
  if (npairs <= 0) return GGNN_OK;
  SymArgs a;
  memset(&a, 0, sizeof(a));
  a.acc = g_acc;
  a.X = X->d_data;
  a.d = X->d;
  a.lpr = choose_lpr(X->d, X->dtype, X->dtype, reinterpret_cast<uintptr_t>(X->d_data));
  a.layer = to_dev(*layer);
  a.npairs = npairs;
  ggnn_search_params p{k_out, prioq_size, visited_size, 0, tau, budget};
  a.c = make_cfg(&p);
  a.dmax = d_nn1_max;
  a.n_fallback = n_fallback;
  a.nnd = d_nnd;
  a.k_nn = layer->k_nn;
  a.resc_id = d_resc_id;
  a.resc_d = d_resc_d;
  a.per_node = per_node;
  a.req = d_req;
  a.req_count = d_req_count;
  a.req_cap = req_cap;
  int keysize = X->dtype == GGNN_U8 ? 4 : 8;
  a.region = set_layout(a.c, X->d, qelem_of(X->dtype), keysize);
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_U8) return launch_sym<uint8_t>(a, npairs, st);
  return launch_sym<float>(a, npairs, st);
}

int ggnn_sym_recheck(const ggnn_vectors* X, const ggnn_layer* layer, int32_t* d_req, int64_t nreq,
                      int32_t* d_stage, int32_t x_end, double tau, double d_nn1_max, int32_t budget, int32_t k_out,
                      int32_t prioq_size, int32_t visited_size, int32_t n_fallback, const int32_t* d_idx,
                      void* stream) {
  GGNN_CHECK_ARG(X && X->d_data && layer && layer->d_adj && d_req && d_stage, "invalid arguments");
  GGNN_CHECK_ARG(layer->k >= 1 && layer->k <= MAX_K, "invalid layer geometry");
  GGNN_CHECK_ARG(k_out >= 1 && k_out <= 32 && n_fallback >= 0 && n_fallback <= 32, "k_out / n_fallback in [1, 32]");
  if (nreq <= 0) return GGNN_OK;
  SymArgs a;
  memset(&a, 0, sizeof(a));
  a.acc = g_acc;
  a.X = X->d_data;
  a.d = X->d;
  a.lpr = choose_lpr(X->d, X->dtype, X->dtype, reinterpret_cast<uintptr_t>(X->d_data));
  a.layer = to_dev(*layer);
  a.npairs = nreq;
  ggnn_search_params p{k_out, prioq_size, visited_size, 0, tau, budget};
  a.c = make_cfg(&p);
  a.dmax = d_nn1_max;
  a.n_fallback = n_fallback;
  a.req = d_req;
  a.recheck = true;
  a.stage = d_stage;
  a.x_end = x_end;
  a.idx = d_idx;
  int keysize = X->dtype == GGNN_U8 ? 4 : 8;
  a.region = set_layout(a.c, X->d, qelem_of(X->dtype), keysize);
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_U8) return launch_sym<uint8_t>(a, nreq, st);
  return launch_sym<float>(a, nreq, st);
}

int ggnn_sym_check_batch(const ggnn_vectors* X, const ggnn_layer* layer, const int32_t* d_x, const int32_t* d_z,
                         const double* d_dxz, int64_t npairs, double tau, double d_nn1_max, int32_t budget,
                         int32_t k_out, int32_t prioq_size, int32_t visited_size, int32_t n_fallback,
                         int32_t* d_verdict, int32_t* d_fallback, void* stream) {
  GGNN_CHECK_ARG(X && X->d_data && layer && layer->d_adj, "invalid arguments");
  GGNN_CHECK_ARG(layer->k >= 1 && layer->k <= MAX_K, "k <= %d supported", MAX_K);
  GGNN_CHECK_ARG(k_out >= 1 && k_out <= 32 && n_fallback >= 0 && n_fallback <= 32, "k_out / n_fallback in [1, 32]");
  if (npairs <= 0) return GGNN_OK;
  SymArgs a;
  memset(&a, 0, sizeof(a));
  a.acc = g_acc;
  a.X = X->d_data;
  a.d = X->d;
  a.lpr = choose_lpr(X->d, X->dtype, X->dtype, reinterpret_cast<uintptr_t>(X->d_data));
  a.layer = to_dev(*layer);
  a.px = d_x;
  a.pz = d_z;
  a.pd = d_dxz;
  a.npairs = npairs;
  ggnn_search_params p{k_out, prioq_size, visited_size, 0, tau, budget};
  a.c = make_cfg(&p);
  a.dmax = d_nn1_max;
  a.n_fallback = n_fallback;
  a.verdict = d_verdict;
  a.fallback = d_fallback;
  int keysize = X->dtype == GGNN_U8 ? 4 : 8;
  a.region = set_layout(a.c, X->d, qelem_of(X->dtype), keysize);
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_U8) return launch_sym<uint8_t>(a, npairs, st);
  return launch_sym<float>(a, npairs, st);
}

int ggnn_exhaustive_topk(const ggnn_vectors* X, const int32_t* d_rows, int64_t nrows, const ggnn_queries* Q,
                         int32_t k, int32_t* d_ids, double* d_dists, void* stream) {
  GGNN_CHECK_ARG(k >= 1, "k must be >= 1 (got %d)", k);
  ggnn_search_params p{k, k, 1, 0, 0.0, 0};
  SearchArgs a;
  int rc = fill_common(a, X, Q, &p);
  if (rc) return rc;
  GGNN_CHECK_ARG(nrows >= 1 && nrows <= INT32_MAX, "invalid row count");
  // whole-table scans at least one X tile per split long: tensor cores
  // (kind::i8 for uint8 tables, 3xTF32 + exact re-score for float tables)
  if (bf_tc_eligible(X, d_rows, Q, k) && nrows == X->n && X->n >= 4096)
    return bf_topk_tc(X, Q, k, d_ids, d_dists, as_stream(stream));
  if (bf_tf32_eligible(X, d_rows, Q, k) && nrows == X->n)
    return bf_topk_tf32(X, Q, k, d_ids, d_dists, as_stream(stream));
  return exhaustive_warp(a, X, Q, d_rows, nrows, d_ids, d_dists, as_stream(stream));
}

}  // extern "C"

namespace ggnn {
// the CUDA-core scan (any k, ceil(k / 32) passes over the rows)
int exhaustive_warp(SearchArgs& a, const ggnn_vectors* X, const ggnn_queries* Q, const int32_t* d_rows, int64_t nrows,
                    int32_t* d_ids, double* d_dists, cudaStream_t st) {
  a.top_rows = d_rows;
  a.ntop = nrows;
  a.ids = d_ids;
  a.dists = d_dists;
  int qd = Q->d_rows ? X->dtype : Q->dtype;
  int keysize = (X->dtype == GGNN_U8 && qd == GGNN_U8) ? 4 : 8;
  a.region = 128 + align16(32 * (size_t)keysize) + align16((size_t)X->d * qelem_of(qd));
  switch (combo(X, Q)) {
    case 0:
      if (a.lpr == 32) return launch_static(topk_kernel<float, float, 32>, a, a.m, a.region, st, 8);
      if (a.lpr == 8) return launch_static(topk_kernel<float, float, 8>, a, a.m, a.region, st, 8);
      return launch_static(topk_kernel<float, float, 0>, a, a.m, a.region, st, 8);
    case 1:
      if (a.lpr == 32) return launch_static(topk_kernel<uint8_t, uint8_t, 32>, a, a.m, a.region, st, 8);
      if (a.lpr == 8) return launch_static(topk_kernel<uint8_t, uint8_t, 8>, a, a.m, a.region, st, 8);
      return launch_static(topk_kernel<uint8_t, uint8_t, 0>, a, a.m, a.region, st, 8);
    default: return launch_static(topk_kernel<uint8_t, float, 0>, a, a.m, a.region, st, 8);
  }
}

int topk_scan_subset(const ggnn_vectors* X, const float* Qsub, int64_t cnt, int k, int32_t* ids, double* dists,
                     cudaStream_t st) {
  ggnn_queries q{Qsub, nullptr, cnt, GGNN_F32, 0};
  ggnn_search_params p{k, k, 1, 0, 0.0, 0};
  SearchArgs a;
  int rc = fill_common(a, X, &q, &p);
  if (rc) return rc;
  return exhaustive_warp(a, X, &q, nullptr, X->n, ids, dists, st);
}
}  // namespace ggnn

extern "C" {

int ggnn_exhaustive_topk_tc(const ggnn_vectors* X, const ggnn_queries* Q, int32_t k, int32_t* d_ids,
                            double* d_dists, void* stream) {
  GGNN_CHECK_ARG(k >= 1, "k must be >= 1 (got %d)", k);
  ggnn_search_params p{k, k, 1, 0, 0.0, 0};
  SearchArgs a;
  int rc = fill_common(a, X, Q, &p);
  if (rc) return rc;
  GGNN_CHECK_ARG(bf_tc_eligible(X, nullptr, Q, k),
                 "the tensor-core scan needs uint8 table and queries, d %% 32 == 0, and k <= 32 with d <= 224 "
                 "or k <= 128 with d <= 128");
  return bf_topk_tc(X, Q, k, d_ids, d_dists, as_stream(stream));
}

int ggnn_squared_l2_many(const ggnn_vectors* X, const ggnn_queries* Q, const int32_t* d_rows, int32_t per_query,
                         double* d_out, void* stream) {
  GGNN_CHECK_ARG(X && X->d_data && Q && d_rows && d_out && per_query >= 0, "invalid arguments");
  int64_t total = Q->m * (int64_t)per_query;
  if (total == 0) return GGNN_OK;
  int qd = Q->d_rows ? X->dtype : Q->dtype;
  unsigned grid = (unsigned)((total + 127) / 128);
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_F32) {
    sqdist_kernel<float, float><<<grid, 128, 0, st>>>((const float*)X->d_data, X->d, (const float*)Q->d_data,
                                                      Q->d_rows, d_rows, per_query, total, d_out);
    count_launch();
  } else if (qd == GGNN_U8) {
    sqdist_kernel<uint8_t, uint8_t><<<grid, 128, 0, st>>>((const uint8_t*)X->d_data, X->d,
                                                          (const uint8_t*)Q->d_data, Q->d_rows, d_rows, per_query,
                                                          total, d_out);
    count_launch();
  } else {
    sqdist_kernel<uint8_t, float><<<grid, 128, 0, st>>>((const uint8_t*)X->d_data, X->d, (const float*)Q->d_data,
                                                        Q->d_rows, d_rows, per_query, total, d_out);
    count_launch();
  }
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

int ggnn_f32_to_u8(const float* d_src, int64_t count, uint8_t* d_u8, int32_t* d_flag, void* stream) {
  GGNN_CHECK_ARG(d_src && d_flag && count >= 0, "invalid arguments");
  if (count == 0) return GGNN_OK;
  DevInfo di = dev_info();
  int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)std::max(di.sm_count, 1) * 8);
  f32_to_u8_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(d_src, count, d_u8, d_flag);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

}  // extern "C"
