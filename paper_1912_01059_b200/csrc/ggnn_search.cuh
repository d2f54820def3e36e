// ggnn_search.cuh -- one-warp-per-search best-first graph search.
//
// Restates the reference's `_greedy_core` (_core.pyx:190-311) with its search
// cache (_core.pyx:135-176, cache.py:25-141) so that, on exact keys (uint8
// data), ids / distances / visited_count / steps / terminated_by / forgotten
// match the reference bit for bit.  The cache lives in
// shared memory, one private region per warp:
//
//   rk[cap], rid[cap], rvis[cap]  the sorted ring (best-list + priority queue);
//                                 uint32 keys: one u64 word per entry,
//                                 key << 32 | id << 1 | visited
//   vring[vsz]                    the visited ring (FIFO of expanded ids)
//   ht[H]                         exact refcount table over ring u vring
//   crow/cid/ckey[32]             per-step candidate scratch
//   qs[d]                         the query vector
//
// One expansion step is executed warp-wide:
//   head scan (ballot over visited bytes) -> threshold in FP64 -> adjacency row
//   load (one coalesced 96-byte read for k=24) -> parallel refcount lookups +
//   __match_any dedupe -> warp-cooperative 16-byte-vector distance gathers ->
//   bitonic sort of the candidates -> threshold admission -> parallel merge
//   into the ring (binary-search ranks, chunked right shift) with the exact
//   eviction / visited-ring / refcount sequence of the sequential reference.
#pragma once
#include <climits>
#include "ggnn_common.cuh"

namespace ggnn {

struct SearchCfg {
  int k_out;
  int cap;  // k_out + prioq_size
  int vsz;  // visited ring size
  int hlog; // log2 of the refcount table size
  double tau;
  long long max_steps;  // max_iterations, or the budget in found-target mode
  int flags;
  // byte offsets of the per-warp shared region (set_layout); the ring starts at 0
  uint32_t o_rvis, o_vring, o_ht, o_crow, o_cid, o_ckey, o_qs;
};

constexpr int FLAG_DISTINCT = 1;     // exact distinct_touched via a global set
constexpr int FLAG_EXACT_DISTS = 2;  // re-score returned hits sequentially (bitwise _sqdist)
constexpr int FLAG_UNIQUE_ROWS = 4;  // rows never repeat a neighbour: no duplicate filter

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Visited rings of up to 32 * VR_SLOTS entries live in per-lane local memory
// (entry i in lane i & 31, slot i >> 5): the ring is written once per
// expansion and read back only when it wraps, so it needs no shared memory.
// 4096 entries: the large query caches C4 needs at R@10 >= 0.99 (visited
// 2048-4096) keep their shared memory for the ring and the refcount table,
// 22 % faster at visited 2048 than a shared-memory visited ring; the default
// 512-entry ring touches the same 16 slots per lane as before.
#ifndef GGNN_VR_SLOTS
#define GGNN_VR_SLOTS 128
#endif
constexpr int VR_SLOTS = GGNN_VR_SLOTS;
__host__ __device__ inline bool vring_local(int vsz) { return vsz <= 32 * VR_SLOTS; }

// Each search kernel declares its lane's slice of the visited ring outside the
// WarpSearch object (an indexed array member would push the whole object --
// counters included -- to the stack):  VRING_DECL(s);
#define VRING_DECL(s)                      \
  int vring_lane_[VR_SLOTS > 0 ? VR_SLOTS : 1]; \
  (s).vr = vring_lane_

// Lay out one warp's shared region (offsets into c, computed once on the
// host so the kernels address every array as base + constant) and return its
// byte size: ring keys + ids (packed u64 words for 4-byte keys, whose low
// bit is the visited flag), visited flags otherwise (padded for 4-byte
// scans), the shared visited ring when it is too
// large for the lanes, the refcount table, candidate rows / ids / keys and
// the query.
inline size_t set_layout(SearchCfg& c, int64_t d, int qelem, int keysize) {
  size_t b = align16((size_t)c.cap * keysize) + align16((size_t)c.cap * 4);
  c.o_rvis = (uint32_t)b;
  if (keysize != 4) b += align16((size_t)((c.cap + 127) / 128) * 128);
  c.o_vring = (uint32_t)b;
  if (!vring_local(c.vsz)) b += align16((size_t)c.vsz * 4);
  c.o_ht = (uint32_t)b;
  b += align16((size_t)(1u << c.hlog) * 4);
  c.o_crow = (uint32_t)b;
  c.o_cid = (uint32_t)(b + 32 * 4);
  c.o_ckey = (uint32_t)(b + 64 * 4);
  b += 64 * 4 + align16(32 * (size_t)keysize);
  c.o_qs = (uint32_t)b;
  b += align16((size_t)d * qelem);
  return b;
}

// Refcount table size: at most cap + vsz ids are live at once (ring u visited
// ring); the table keeps >= 64 + cap / 8 spare slots beyond that so probing
// always meets an empty slot (tombstones are purged by rebuild(), see merge()).
inline int table_log2(int cap, int vsz) {
  int need = cap + vsz + 64 + cap / 8;
  int lg = 6;
  while ((1 << lg) < need) ++lg;
  return lg;
}

// Refcount-table purge threshold in sixteenths of the table: linear probing
// counts tombstones as occupied, so a miss costs ~(1 + 1/(1-a)^2)/2 probes at
// occupancy a; purging earlier trades rebuilds for shorter probe chains.
#ifndef GGNN_HT_FILL
#define GGNN_HT_FILL 12
#endif
constexpr int HT_FILL = GGNN_HT_FILL;

// 128-byte lines of each neighbour row prefetched into L1 at the start of an
// expansion (0 disables; rows longer than this are only partly prefetched)
#ifndef GGNN_PREFETCH_LINES
#define GGNN_PREFETCH_LINES 1
#endif
constexpr int PREFETCH_LINES = GGNN_PREFETCH_LINES;
// prefetch into L2 only (the L1 left beside 28 searches' shared memory is
// small: ncu measures a 2 % L1 hit rate for the row gathers)
#ifndef GGNN_PREFETCH_L2
#define GGNN_PREFETCH_L2 0
#endif

template <typename Key>
__device__ void warp_sorted_out(const Key* keys, const int* ids, int n, int K, int32_t* out_ids, double* out_d);

template <typename TX, typename TQ, int LP = 0>
struct WarpSearch {
  using Key = typename VecTraits<TX, TQ>::Key;
  using KO = KeyOps<Key>;

  // data
  const TX* X;
  int64_t d;
  int lpr;
  TQ* qs;
  // layer
  const int32_t* adj;
  int k;
  const int32_t* to_row;  // nullptr = identity
  double dmax;
  // config
  SearchCfg c;
  int target;  // -1: normal mode
  // shared memory: the ring as packed (key << 32 | id) words for exact
  // integer keys (PACK), as separate key / id arrays otherwise
  static constexpr bool PACK = sizeof(Key) == 4;
  uint64_t* re;
  Key* rk;
  int* rid;
  uint8_t* rvis;
  int* vring;  // shared visited ring (vsz > 32 * VR_SLOTS only)
  int* vr;  // local visited ring (the kernel's per-lane array, see VRING_DECL)
  RefTable ht;
  int* crow;
  int* cid;
  Key* ckey;
  // distinct_touched log (FLAG_DISTINCT): every id the search inserts --
  // seeds and computed candidates -- is appended to a per-query list in
  // global memory with plain stores that nothing waits on; a pass after the
  // search counts the distinct entries (distinct_log_kernel).  log_tag keeps
  // the ids of different layers apart (descents: layer << 27).
  uint32_t* tlog;
  int log_cap;
  int nlog;
  uint32_t log_tag;
  // warp-uniform state
  int L, vlen, vpos, used, rebuild_at;
  // adjacency row of the predicted next expansion, loaded while the current
  // step merges (pf_nb: this lane's slot of row pf_node)
  int pf_node, pf_nb;
  // ring position of the next expansion when known from the last merge
  // (-1: none left), -2 when head() must scan
  int next_head;
  int visited, steps, distinct, forgotten, term;
  bool found_target;
  // the stopping threshold, recomputed only after a merge placed a candidate
  // among the first k_out ring entries (the only entries it depends on):
  // integer keys keep floor(thr) (key <= thr <=> key <= floor(thr), thr >= 0)
  bool thr_dirty;
  uint32_t thr_u;
  double thr_d;

  __device__ __forceinline__ Key ring_key(int i) const {
    if constexpr (PACK) return (Key)(re[i] >> 32);
    else return rk[i];
  }
  __device__ __forceinline__ int ring_id(int i) const {
    if constexpr (PACK) return (int)((uint32_t)re[i] >> 1);
    else return rid[i];
  }
  // packed ring word: key << 32 | id << 1 | visited.  The flag below the id
  // keeps the (key, id) order of the words (ids are distinct, < 2^31).
  static __device__ __forceinline__ uint64_t ring_word(uint32_t key, int id) {
    return ((uint64_t)key << 32) | ((uint64_t)(uint32_t)id << 1);
  }
  __device__ __forceinline__ bool ring_vis(int i) const {
    if constexpr (PACK) return (reinterpret_cast<const uint32_t*>(re)[2 * i] & 1u) != 0u;
    else return rvis[i] != 0;
  }

  __device__ void carve(uint8_t* base) {
    if constexpr (PACK) {
      re = reinterpret_cast<uint64_t*>(base);
    } else {
      rk = reinterpret_cast<Key*>(base);
      rid = reinterpret_cast<int*>(base + align16((size_t)c.cap * sizeof(Key)));
    }
    rvis = base + c.o_rvis;
    vring = vring_local(c.vsz) ? nullptr : reinterpret_cast<int*>(base + c.o_vring);
    ht.t = reinterpret_cast<uint32_t*>(base + c.o_ht);
    ht.mask = (1u << c.hlog) - 1u;
    ht.shift = 32 - c.hlog;
    crow = reinterpret_cast<int*>(base + c.o_crow);
    cid = reinterpret_cast<int*>(base + c.o_cid);
    ckey = reinterpret_cast<Key*>(base + c.o_ckey);
    qs = reinterpret_cast<TQ*>(base + c.o_qs);
  }

  __device__ void reset() {
    ht.clear();
    L = vlen = vpos = used = 0;
    rebuild_at = (int)((ht.mask + 1) * HT_FILL / 16);
    pf_node = -1;
    pf_nb = -1;
    next_head = -2;
    visited = steps = distinct = forgotten = 0;
    term = TERM_EMPTY;
    found_target = false;
    thr_dirty = true;
  }

  // append lanes [0, n) with valid[lane] to the log (in lane order)
  __device__ __forceinline__ void log_lanes(bool valid, int id) {
    const unsigned vm = __ballot_sync(FULL, valid);
    const int pos = nlog + __popc(vm & lanemask_lt());
    if (valid && pos < log_cap) tlog[pos] = log_tag | (uint32_t)id;
    nlog += __popc(vm);
  }

  __device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
  }

  __device__ void rebuild() {
    const int lane = lane_id();
    ht.clear();
    int u = 0;
    for (int i = lane; i < L; i += 32) u += ht.add_one((uint32_t)ring_id(i));
    for (int i = lane; i < vlen; i += 32) u += ht.add_one((uint32_t)(vring ? vring[i] : vr[i >> 5]));
    used = warp_sum(u);
    // next purge once the occupied slots (live + tombstones) pass HT_FILL / 16
    // of the table or tombstones fill an eighth of it, never so late that
    // fewer than 40 slots stay empty (one merge adds at most 32)
    const int size = (int)ht.mask + 1;
    rebuild_at = min(max(size * HT_FILL / 16, used + size / 8), size - 40);
    __syncwarp();
  }

  // ring position of the first unvisited entry, -1 if none
  __device__ int head() const { return head_from(0); }

  // first unvisited ring position >= start (start a multiple of 4 or not), -1 if none
  __device__ int head_from(int start) const {
    const int lane = lane_id();
    if constexpr (PACK) {
      const uint32_t* lo = reinterpret_cast<const uint32_t*>(re);  // low words: id << 1 | visited
      for (int base = start; base < L; base += 32) {
        const int p = base + lane;
        const unsigned bal = __ballot_sync(FULL, p < L && (lo[2 * p] & 1u) == 0u);
        if (bal) return base + __ffs(bal) - 1;
      }
      return -1;
    }
    for (int base = start & ~3; base < L; base += 128) {
      const int p0 = base + 4 * lane;
      const uint32_t w = *reinterpret_cast<const uint32_t*>(rvis + p0);
      // visited flags are 0 / 1 bytes: bit 8b of z is set iff byte b is 0;
      // keep the bytes at positions [start, L)
      uint32_t z = ~w & 0x01010101u;
      const int lo = start - p0, hi = L - p0;
      if (lo > 0) z = lo >= 4 ? 0u : z & (0xffffffffu << (8 * lo));
      if (hi < 4) z = hi <= 0 ? 0u : z & (0xffffffffu >> (32 - 8 * hi));
      const unsigned bal = __ballot_sync(FULL, z != 0u);
      if (bal) {
        const int src = __ffs(bal) - 1;
        return base + 4 * src + (__shfl_sync(FULL, __ffs(z), src) >> 3);
      }
    }
    return -1;
  }

  __device__ void vring_push(int node) {
    const int lane = lane_id();
    if (vlen == c.vsz) {
      int old;
      if (vring) {
        old = vring[vpos];
        __syncwarp();
        if (lane == 0) vring[vpos] = node;
      } else {
        int o = 0;
        if (lane == (vpos & 31)) {
          o = vr[vpos >> 5];
          vr[vpos >> 5] = node;
        }
        old = __shfl_sync(FULL, o, vpos & 31);
      }
      if (ht.dec((uint32_t)old)) forgotten++;
      vpos = (vpos + 1 == c.vsz) ? 0 : vpos + 1;
    } else {
      if (vring) {
        if (lane == 0) vring[vlen] = node;
      } else if (lane == (vlen & 31)) {
        vr[vlen >> 5] = node;
      }
      vlen++;
    }
    __syncwarp();
  }

  // Drop the E (<= 32) largest ring entries, largest first (_core.pyx:161-166).
  // Unvisited ones have refcount exactly 1 and vanish (forgotten); their table
  // slots are tombstoned lane-parallel.  Visited ones go to the visited ring
  // in eviction order (their +1 there and -1 here cancel).
  __device__ __forceinline__ void evict(int E) {
    const int lane = lane_id();
    const bool in = lane < E;
    const int r = L - 1 - lane;
    const int t = in ? ring_id(r) : -1;
    const bool vis = in && ring_vis(r);
    const bool gone = in && !vis;
    if (gone) ht.tomb_lane((uint32_t)t);
    forgotten += __popc(__ballot_sync(FULL, gone));
    __syncwarp();
    unsigned vm = __ballot_sync(FULL, vis);
    while (vm) {
      const int e = __ffs(vm) - 1;
      vm &= vm - 1;
      vring_push(__shfl_sync(FULL, t, e));
    }
  }

  // Lanes [0, m) hold ascending, distinct, currently-unknown (key, id) pairs.
  // Equivalent to calling the reference's _ring_insert on each in order.
  // Returns the first unvisited ring position after the merge, given q = the
  // first unvisited position before it (-1 if none; q == -2: unknown).
  __device__ int merge(Key key, int id, int m, int q = -2) {
    const int lane = lane_id();
    int rank = 0;
    if (lane < m) {
      int lo = 0, hi = L;
      if constexpr (PACK) {
        const uint64_t pk = ring_word((uint32_t)key, id);
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (re[mid] <= pk)
            lo = mid + 1;
          else
            hi = mid;
        }
      } else {
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          const Key km = rk[mid];
          if (km < key || (km == key && rid[mid] <= id))
            lo = mid + 1;
          else
            hi = mid;
        }
      }
      rank = lo;
    }
    const int p = rank + lane;
    const bool ok = lane < m && p < c.cap;
    const int madm = __popc(__ballot_sync(FULL, ok));
    forgotten += m - madm;  // worse than the tail of a full ring
    if (madm == 0) return q;
    const int newL = min(c.cap, L + madm);
    const int E = L + madm - newL;
    // next expansion: the first admitted candidate or the old q, shifted by
    // the candidates placed before it (q is gone if it was evicted)
    int nh = -2;
    if (q != -2) {
      nh = __shfl_sync(FULL, p, 0);
      if (q >= 0 && q < L - E) nh = min(nh, q + __popc(__ballot_sync(FULL, ok && rank <= q)));
    }
    if (E > 0) evict(E);
    // Scatter the merged sequence in place, top chunk first: output position
    // o holds the candidate whose slot is o, else ring entry o - #{candidates
    // placed below o}.  Every source index is <= its destination and chunks
    // go downwards, so nothing is overwritten before it is read.
    const int p0 = __shfl_sync(FULL, p, 0);
    if (p0 < c.k_out) thr_dirty = true;
    // chunks wholly above the last candidate's slot only move up by madm
    // (every candidate lies below them): a plain copy, no candidate masks
    const int pl = __shfl_sync(FULL, p, madm - 1);  // admitted lanes are the prefix [0, madm)
    int hi = newL;
    for (; hi - 32 > pl; hi -= 32) {
      const int o = hi - 32 + lane;
      if constexpr (PACK) {
        const uint64_t ee = re[o - madm];
        __syncwarp();
        re[o] = ee;
      } else {
        const Key kk = rk[o - madm];
        const int ii = rid[o - madm];
        const uint8_t vv = rvis[o - madm];
        __syncwarp();
        rk[o] = kk;
        rid[o] = ii;
        rvis[o] = vv;
      }
      __syncwarp();
    }
    for (; hi > p0; hi -= 32) {
      const int cb = hi - 32;
      const int o = cb + lane;
      const bool act = o >= p0;
      const unsigned bit = (ok && p >= cb && p < hi) ? (1u << (p - cb)) : 0u;
      const unsigned cmask = __reduce_or_sync(FULL, bit);
      const int below = __popc(__ballot_sync(FULL, ok && p < cb)) + __popc(cmask & lanemask_lt());
      const bool is_c = (cmask >> lane) & 1u;
      if constexpr (PACK) {
        uint64_t ee = __shfl_sync(FULL, ring_word((uint32_t)key, id), below & 31);
        if (act && !is_c) ee = re[o - below];
        __syncwarp();
        if (act) re[o] = ee;
      } else {
        const Key ck = KO::shfl(key, below & 31);
        const int ci = __shfl_sync(FULL, id, below & 31);
        Key kk = ck;
        int ii = ci;
        uint8_t vv = 0;
        if (act && !is_c) {
          const int r = o - below;
          kk = rk[r];
          ii = rid[r];
          vv = rvis[r];
        }
        __syncwarp();
        if (act) {
          rk[o] = kk;
          rid[o] = ii;
          rvis[o] = vv;
        }
      }
      __syncwarp();
    }
    int took = ok ? ht.insert_new((uint32_t)id) : 0;
    used += __popc(__ballot_sync(FULL, took != 0));
    L = newL;
    __syncwarp();
    if (used > rebuild_at) rebuild();
    return nh;
  }

  // Seeds: lanes [0, n) hold (key, id) in the caller's order; duplicates and
  // already-known ids are skipped (first occurrence wins), _core.pyx:219-229.
  __device__ void seed(Key key, int id, int n) {
    const int lane = lane_id();
    bool v = lane < n && id >= 0;
    if (v) v = ht.count((uint32_t)id) == 0u;
    unsigned same = __match_any_sync(FULL, v ? (unsigned)id : (0x80000000u | (unsigned)lane));
    v = v && ((same & lanemask_lt()) == 0u);
    if (!v) {
      key = KO::max_key();
      id = INT_MAX;
    }
    const int cnt = __popc(__ballot_sync(FULL, v));
    if (tlog) log_lanes(v, id);
    distinct += cnt;
    warp_sort_n(key, id, n);  // valid seeds sit anywhere in lanes [0, n): bitonic
    if (cnt) merge(key, id, cnt);
    next_head = -2;
  }

  // One expansion.  Returns false when the search has terminated.
  __device__ bool step() {
    const int lane = lane_id();
    const int pos = next_head != -2 ? next_head : head();
    if (pos < 0) {
      term = TERM_EMPTY;
      return false;
    }
    if (thr_dirty) {
      // FP64, rounded exactly like the reference (no FMA contraction):
      // thr = ring[k_out-1] + tau * min(d_nn1_max, ring[0])   (_core.pyx:241-244)
      double thr = __longlong_as_double(0x7ff0000000000000ll);
      if (L >= c.k_out)
        thr = __dadd_rn(KO::to_d(ring_key(c.k_out - 1)), __dmul_rn(c.tau, fmin(dmax, KO::to_d(ring_key(0)))));
      if constexpr (PACK) thr_u = thr < 4294967295.0 ? (uint32_t)thr : 0xffffffffu;
      else thr_d = thr;
      thr_dirty = false;
    }
    bool stop;
    if constexpr (PACK) stop = (uint32_t)ring_key(pos) > thr_u;
    else stop = KO::to_d(ring_key(pos)) > thr_d;
    if (stop) {
      term = TERM_STOP;
      return false;
    }
    if ((long long)steps >= c.max_steps) {
      term = TERM_CAP;
      return false;
    }
    const int node = ring_id(pos);
    __syncwarp();
    if (lane == 0) {
      if constexpr (PACK) reinterpret_cast<uint32_t*>(re)[2 * pos] |= 1u;
      else rvis[pos] = 1;
    }
    vring_push(node);
    // ht.inc(node) and the scan for the next unvisited entry do not depend on
    // this step's candidates: they run while the row gathers are in flight
    // (node's count only matters to later lookups; it is in the ring already)

    int nb = -1;
    if (node == pf_node) {
      nb = pf_nb;
    } else if (lane < k) {
      nb = __ldg(adj + (int64_t)node * k + lane);
    }
    pf_node = -1;
    // start pulling every neighbour's row towards L1 now; the membership
    // filter below usually keeps about half of them
    int nrow = -1;
    if (nb >= 0) {
      nrow = to_row ? __ldg(to_row + nb) : nb;
      if (PREFETCH_LINES > 0) {
        const char* rp = reinterpret_cast<const char*>(X + (int64_t)nrow * d);
#pragma unroll
        for (int l = 0; l < PREFETCH_LINES; ++l)
          if (l * 128 < d * (int64_t)sizeof(TX)) {
            if (GGNN_PREFETCH_L2) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + l * 128));
            else asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + l * 128));
          }
      }
    }
    bool cand = nb >= 0;
    if (cand) cand = ht.count((uint32_t)nb) == 0u;
    if (!(c.flags & FLAG_UNIQUE_ROWS)) {  // "nb in cands" (_core.pyx:268-272)
      unsigned same = __match_any_sync(FULL, cand ? (unsigned)nb : (0x80000000u | (unsigned)lane));
      cand = cand && ((same & lanemask_lt()) == 0u);
    }
    const unsigned cm = __ballot_sync(FULL, cand);
    const int nc = __popc(cm);
    bool found = false;
    if (nc) {
      const int ci = __popc(cm & lanemask_lt());
      if (cand) {
        crow[ci] = nrow;
        cid[ci] = nb;
      }
      __syncwarp();
      int q = -1;
      warp_dists_t<TX, TQ, LP>(X, d, qs, crow, nc, ckey, lpr, [&]() {
        ht.inc_present((uint32_t)node);
        q = head_from(pos + 1);
      });
      __syncwarp();
      Key key = KO::max_key();
      int id = INT_MAX;
      if (lane < nc) {
        key = ckey[lane];
        id = cid[lane];
      }
      __syncwarp();
      visited += nc;
      if (tlog) log_lanes(lane < nc, id);
      int m;
      if (PACK && d <= 33000) {  // u8 keys (d * 255^2) stay below 2^31
        // admission first, then rank only what is admitted: every rejected
        // key exceeds thr >= every admitted key, so counting smaller keys
        // over all nc candidates already ranks the admitted ones among
        // themselves.  Keys < 2^31: (kj - key) >> 31 == (kj < key).
        // integer keys: key <= thr  <=>  key <= floor(thr) (thr >= 0), one
        // conversion per step instead of one FP64 compare per lane
        const bool adm = lane < nc && (uint32_t)key <= thr_u;
        const unsigned am = __ballot_sync(FULL, adm);
        m = __popc(am);
        forgotten += nc - m;
        if (target >= 0) found = __any_sync(FULL, adm && id == target);
        if (m) {
          uint32_t* ck = reinterpret_cast<uint32_t*>(ckey);
          if (lane >= nc && lane < ((nc + 3) & ~3)) ck[lane] = 0x7fffffffu;  // never below a real key
          __syncwarp();
          int rank = 0;
          const uint32_t kk = (uint32_t)key;
          if (adm) {
            const uint4* k4 = reinterpret_cast<const uint4*>(ck);
            for (int j = 0; j < nc; j += 4) {
              const uint4 w = k4[j >> 2];
              rank += (int)((w.x - kk) >> 31) + (int)((w.y - kk) >> 31) + (int)((w.z - kk) >> 31) +
                      (int)((w.w - kk) >> 31);
            }
          }
          __syncwarp();
          uint64_t* sc = reinterpret_cast<uint64_t*>(crow);  // crow + cid: 32 words
          const uint64_t mine = pack_ki(kk, id);
          if (adm) sc[rank] = mine;
          __syncwarp();
          // equal keys (only admitted ones can equal an admitted key) share a
          // count and collide in sc: rank them by id, the (key, id) order of
          // the ring (rare; candidate j's key / id sit in lane j)
          if (__any_sync(FULL, adm && sc[rank] != mine)) {
            for (int j = 0; j < nc; ++j) {
              const uint32_t kj = __shfl_sync(FULL, kk, j);
              const int ij = __shfl_sync(FULL, id, j);
              rank += (adm && kj == kk && ij < id) ? 1 : 0;
            }
            __syncwarp();
            if (adm) sc[rank] = mine;
            __syncwarp();
          }
          if (lane < m) {
            const uint64_t v = sc[lane];
            key = (Key)(v >> 32);
            id = (int)(uint32_t)v;
          } else {
            key = KO::max_key();
            id = INT_MAX;
          }
          __syncwarp();
        }
      } else {
        // candidates are compacted into lanes [0, nc); crow / cid are free now
        warp_sort_n(key, id, nc, reinterpret_cast<uint64_t*>(crow));
        bool adm = lane < nc;
        if constexpr (PACK) adm = adm && (uint32_t)key <= thr_u;
        else adm = adm && KO::to_d(key) <= thr_d;
        m = __popc(__ballot_sync(FULL, adm));
        forgotten += nc - m;
        if (target >= 0) found = __any_sync(FULL, adm && id == target);
      }
      // predict the next expansion -- the smaller of the next unvisited ring
      // entry q and the best admitted candidate -- and load its adjacency row
      // while the merge runs (checked against the real head next step)
      if (!found) prefetch_next(q, m > 0, KO::shfl(key, 0), __shfl_sync(FULL, id, 0));
      next_head = m ? merge(key, id, m, q) : q;
    } else {
      ht.inc_present((uint32_t)node);
      const int q = head_from(pos + 1);
      prefetch_next(q, false, KO::max_key(), INT_MAX);
      next_head = q;
    }
    steps++;
    if (found) {
      found_target = true;  // _core.pyx:309-311 returns here with term = 1
      term = 1;
      return false;
    }
    return true;
  }

  // q = first unvisited ring position after the one being expanded (-1: none)
  __device__ __forceinline__ void prefetch_next(int q, bool have_cand, Key kc, int ic) {
    Key ko = KO::max_key();
    int io = INT_MAX;
    if (q >= 0) {
      ko = ring_key(q);
      io = ring_id(q);
    }
    int pred = io;
    if (have_cand && key_less(kc, ic, ko, io)) pred = ic;
    if (pred != INT_MAX) {
      pf_node = pred;
      pf_nb = lane_id() < k ? __ldg(adj + (int64_t)pred * k + lane_id()) : -1;
    }
  }

  // unexpanded ring entries within the stopping threshold: the pending work
  // of a search cut off by a step limit (longest-first schedule)
  __device__ int open_work() {
    double thr = __longlong_as_double(0x7ff0000000000000ll);
    if (L >= c.k_out)
      thr = __dadd_rn(KO::to_d(ring_key(c.k_out - 1)), __dmul_rn(c.tau, fmin(dmax, KO::to_d(ring_key(0)))));
    int n = 0;
    for (int i = lane_id(); i < L; i += 32) n += (!ring_vis(i) && KO::to_d(ring_key(i)) <= thr) ? 1 : 0;
    return warp_sum(n);
  }

  // Run at most `limit` expansions in total; true while the search is still
  // open (the pilot pass of the longest-first schedule, see park()).
  __device__ __forceinline__ bool run_until(long long limit) {
    while ((long long)steps < limit)
      if (!step()) return false;
    return true;
  }

  // Park / unpark an open search (the longest-first schedule of the query
  // batch: every search first runs a short pilot, the open ones are parked
  // and resumed longest-predicted first).  Parked: the ring and its visited
  // flags (and a shared visited ring) -- the region's bytes below the
  // refcount table --, the query row, the lane-held visited ring and the
  // scalars.  The refcount table is rebuilt from the ring and the visited
  // ring on unpark: its counts are exact functions of the two, tombstones
  // only affect probing speed.  Step-by-step identical to an uninterrupted
  // search.
  static __host__ __device__ size_t park_bytes(const SearchCfg& c, int64_t qbytes) {
    return 64 + (size_t)c.o_ht + align16((size_t)qbytes) + (vring_local(c.vsz) ? align16((size_t)c.vsz * 4) : 0);
  }
  __device__ __forceinline__ uint8_t* region_base() const {
    if constexpr (PACK) return reinterpret_cast<uint8_t*>(re);
    else return reinterpret_cast<uint8_t*>(rk);
  }
  __device__ void park(uint8_t* dst, int64_t qbytes) {
    const int lane = lane_id();
    __syncwarp();
    if (lane == 0) {
      int* h = reinterpret_cast<int*>(dst);
      h[0] = L;
      h[1] = vlen;
      h[2] = vpos;
      h[3] = visited;
      h[4] = steps;
      h[5] = distinct;
      h[6] = forgotten;
    }
    const uint4* src = reinterpret_cast<const uint4*>(region_base());
    uint4* o = reinterpret_cast<uint4*>(dst + 64);
    for (int i = lane; i < (int)(c.o_ht / 16); i += 32) o[i] = src[i];
    uint8_t* oq = dst + 64 + c.o_ht;
    const uint8_t* q = reinterpret_cast<const uint8_t*>(qs);
    for (int64_t i = lane * 4; i < qbytes; i += 128)
      *reinterpret_cast<uint32_t*>(oq + i) = *reinterpret_cast<const uint32_t*>(q + i);
    if (!vring) {
      int* ov = reinterpret_cast<int*>(oq + align16((size_t)qbytes));
      for (int j = 0; j < ((vlen + 31) >> 5); ++j) ov[j * 32 + lane] = vr[j];
    }
  }
  // (after carve + set_layer + reset)
  __device__ void unpark(const uint8_t* srcp, int64_t qbytes) {
    const int lane = lane_id();
    const int* h = reinterpret_cast<const int*>(srcp);
    L = h[0];
    vlen = h[1];
    vpos = h[2];
    visited = h[3];
    steps = h[4];
    distinct = h[5];
    forgotten = h[6];
    const uint4* src = reinterpret_cast<const uint4*>(srcp + 64);
    uint4* o = reinterpret_cast<uint4*>(region_base());
    for (int i = lane; i < (int)(c.o_ht / 16); i += 32) o[i] = src[i];
    const uint8_t* sq = srcp + 64 + c.o_ht;
    uint8_t* q = reinterpret_cast<uint8_t*>(qs);
    for (int64_t i = lane * 4; i < qbytes; i += 128)
      *reinterpret_cast<uint32_t*>(q + i) = *reinterpret_cast<const uint32_t*>(sq + i);
    if (!vring) {
      const int* sv = reinterpret_cast<const int*>(sq + align16((size_t)qbytes));
      for (int j = 0; j < ((vlen + 31) >> 5); ++j) vr[j] = sv[j * 32 + lane];
    }
    __syncwarp();
    rebuild();
  }

  __device__ void run() {
    while (step()) {
    }
    if (target >= 0) term = found_target ? 1 : 0;  // _core.pyx:311-312
  }

  // first min(L, k_out) ring entries -> ids / keys in lanes (k_out <= 32)
  __device__ int hits(Key& key, int& id) const {
    const int lane = lane_id();
    const int nh = min(L, c.k_out);
    key = KO::max_key();
    id = -1;
    if (lane < nh) {
      key = ring_key(lane);
      id = ring_id(lane);
    }
    return nh;
  }

  // Copy the first nh ring entries to the top of the ring array, positions
  // [cap - nh, cap), where seeding the next search (which fills [0, nh))
  // cannot reach them while cap >= 2 * nh: hits of more than 32 entries
  // carried from one layer's search to the next (descent).
  __device__ void stash(int nh) {
    const int base = c.cap - nh;
    for (int i = lane_id(); i < nh; i += 32) {
      if constexpr (PACK) {
        re[base + i] = re[i];
      } else {
        rk[base + i] = rk[i];
        rid[base + i] = rid[i];
      }
    }
    __syncwarp();
  }
  __device__ __forceinline__ void stashed(int nh, int i, Key& key, int& id) const {
    key = ring_key(c.cap - nh + i);
    id = ring_id(c.cap - nh + i);
  }

  // The first min(L, k_out) ring entries -> out_ids / out_d[0, k_out), -1 /
  // +inf padded.  With `rescore` (float keys: FP32-partial or lane-parallel
  // sums drove the search) each hit's distance is recomputed with the
  // reference's sequential FP64 _sqdist and the hits are re-sorted by
  // (exact distance, id), the order the reference's ring would hold them in.
  // to_row_map: layer id -> dataset row (nullptr = identity).
  __device__ void write_out(const int32_t* to_row_map, bool rescore, int32_t* out_ids, double* out_d) {
    const int lane = lane_id();
    const int nh = min(L, c.k_out);
    if constexpr (!PACK) {
      if (rescore) {
        for (int i = lane; i < nh; i += 32) {
          const int id = rid[i];
          const int row = to_row_map ? __ldg(to_row_map + id) : id;
          rk[i] = seq_sqdist<TX, TQ>(X + (int64_t)row * d, qs, d);
        }
        __syncwarp();
        warp_sorted_out<Key>(rk, rid, nh, c.k_out, out_ids, out_d);
        return;
      }
    }
    for (int i = lane; i < c.k_out; i += 32) {
      const bool ok = i < nh;
      out_ids[i] = ok ? ring_id(i) : -1;
      out_d[i] = ok ? KO::to_d(ring_key(i)) : __longlong_as_double(0x7ff0000000000000ll);
    }
  }
};

// Merge one unsorted chunk (ck, cx) (one pair per lane, invalid lanes hold
// (max, INT_MAX)) into the running ascending top list (bk, bi), keeping the kk
// smallest (kk <= 32).  The 32 smallest of two ascending lists is the
// elementwise min against the reversed chunk (a bitonic sequence), which the
// half-cleaners then sort.
template <typename Key>
__device__ __forceinline__ void topk_merge_chunk(Key& bk, int& bi, Key ck, int cx, int kk) {
  using KO = KeyOps<Key>;
  const int lane = lane_id();
  warp_sort(ck, cx);
  Key rk2 = KO::shfl(ck, 31 - lane);
  int ri2 = __shfl_sync(FULL, cx, 31 - lane);
  if (key_less(rk2, ri2, bk, bi)) {
    bk = rk2;
    bi = ri2;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
    Key ok = KO::shfl_xor(bk, stride);
    int oi = __shfl_xor_sync(FULL, bi, stride);
    bool lower = (lane & stride) == 0;
    if (lower ? key_less(ok, oi, bk, bi) : key_less(bk, bi, ok, oi)) {
      bk = ok;
      bi = oi;
    }
  }
  if (lane >= kk) {
    bk = KO::max_key();
    bi = INT_MAX;
  }
}

// Exhaustive top-kk (kk <= 32) over rows[lo..hi) (or the index range itself
// when rows is null), ties by local index; the result sits in lanes [0, kk)
// as (key, local index) -- the reference's exhaustive_topk (_core.pyx:86-104).
// With `after`, only pairs ordered strictly after (ak, ai) compete: pass p of
// a top-K with K > 32 selects ranks [32p, 32p + 32) this way.
template <typename TX, typename TQ, int LP = 0>
__device__ void warp_topk_scan(const TX* X, int64_t d, const TQ* qs, int lpr, const int32_t* rows, int lo, int hi,
                               int kk, int* crow, typename VecTraits<TX, TQ>::Key* ckey,
                               typename VecTraits<TX, TQ>::Key& bk, int& bi, bool after = false,
                               typename VecTraits<TX, TQ>::Key ak = 0, int ai = -1) {
  using Key = typename VecTraits<TX, TQ>::Key;
  using KO = KeyOps<Key>;
  const int lane = lane_id();
  bk = KO::max_key();
  bi = INT_MAX;
  for (int base = lo; base < hi; base += 32) {
    const int cnt = min(32, hi - base);
    if (lane < cnt) crow[lane] = rows ? __ldg(rows + base + lane) : base + lane;
    __syncwarp();
    warp_dists_t<TX, TQ, LP>(X, d, qs, crow, cnt, ckey, lpr);
    __syncwarp();
    Key ck = KO::max_key();
    int cx = INT_MAX;
    if (lane < cnt) {
      ck = ckey[lane];
      cx = base + lane - lo;
      if (after && !key_less(ak, ai, ck, cx)) {
        ck = KO::max_key();
        cx = INT_MAX;
      }
    }
    __syncwarp();
    topk_merge_chunk(bk, bi, ck, cx, kk);
  }
}

// Top-K (any K) of n (key, id) pairs held in shared memory (keys[i], ids[i],
// distinct ids), written ascending by (key, id) to out_ids / out_d[0, K):
// ceil(K / 32) passes of the warp top-32, pass p keeping the pairs after the
// last one pass p - 1 emitted.  Positions >= n are padded (-1, +inf).
template <typename Key>
__device__ void warp_sorted_out(const Key* keys, const int* ids, int n, int K, int32_t* out_ids, double* out_d) {
  using KO = KeyOps<Key>;
  const int lane = lane_id();
  Key ak = 0;
  int ai = -1;
  for (int b = 0; b < K; b += 32) {
    Key bk = KO::max_key();
    int bi = INT_MAX;
    if (b < n) {
      for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        Key ck = KO::max_key();
        int cx = INT_MAX;
        if (i < n) {
          ck = keys[i];
          cx = ids[i];
          if (b > 0 && !key_less(ak, ai, ck, cx)) {
            ck = KO::max_key();
            cx = INT_MAX;
          }
        }
        topk_merge_chunk(bk, bi, ck, cx, 32);
      }
      ak = KO::shfl(bk, 31);
      ai = __shfl_sync(FULL, bi, 31);
    }
    const int o = b + lane;
    if (o < K) {
      const bool ok = o < n;
      out_ids[o] = ok ? bi : -1;
      out_d[o] = ok ? KO::to_d(bk) : __longlong_as_double(0x7ff0000000000000ll);
    }
  }
  __syncwarp();
}

}  // namespace ggnn
