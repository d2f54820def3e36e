// ggnn_common.cuh -- shared device building blocks for the GGNN sm_100a kernels.
//
// Layout conventions:
//   vectors  : row-major (n, d), either float32 or uint8 (lossless copy of
//              integer-valued data in [0, 255]); rows are 16-byte aligned when
//              d * elem_size is a multiple of 16.
//   adjacency: row-major int32 (node_count, k), "sanitized": every slot the
//              reference would skip is -1 (direct slots holding -1, sym slots at
//              or beyond sym_count), so the kernels need no sym_count array.
//   keys     : distances are carried as exact uint32 for uint8 data (the sum of
//              squared byte differences) and as double for float data, matching
//              the reference's float64 accumulation (_core.pyx:30-37).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

namespace ggnn {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARP = 32;
constexpr int MAX_K = 32;  // slots per adjacency row handled by one warp

enum Term : int { TERM_STOP = 0, TERM_EMPTY = 1, TERM_CAP = 2 };

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- key types
template <typename K> struct KeyOps;
template <> struct KeyOps<uint32_t> {
  static __device__ __forceinline__ uint32_t max_key() { return 0xffffffffu; }
  static __device__ __forceinline__ double to_d(uint32_t k) { return (double)k; }
  static __device__ __forceinline__ uint32_t from_d(double v) { return (uint32_t)v; }
  static __device__ __forceinline__ uint32_t shfl(uint32_t v, int src) { return __shfl_sync(FULL, v, src); }
  static __device__ __forceinline__ uint32_t shfl_xor(uint32_t v, int m) { return __shfl_xor_sync(FULL, v, m); }
};
template <> struct KeyOps<double> {
  static __device__ __forceinline__ double max_key() { return __longlong_as_double(0x7ff0000000000000ll); }
  static __device__ __forceinline__ double to_d(double k) { return k; }
  static __device__ __forceinline__ double from_d(double v) { return v; }
  static __device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(FULL, v, src); }
  static __device__ __forceinline__ double shfl_xor(double v, int m) { return __shfl_xor_sync(FULL, v, m); }
};

template <typename K>
__device__ __forceinline__ bool key_less(K ka, int ia, K kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// Bitonic sort of one (key, id) pair per lane, ascending by (key, id).
template <typename K>
__device__ __forceinline__ void warp_sort(K& key, int& id) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      K ok = KeyOps<K>::shfl_xor(key, stride);
      int oi = __shfl_xor_sync(FULL, id, stride);
      bool up = ((lane & size) == 0);       // ascending block
      bool lower = ((lane & stride) == 0);  // I hold the lower index of the pair
      bool other_less = key_less(ok, oi, key, id);
      // lower lane keeps the min in an ascending block, the max otherwise
      bool take = (lower == up) ? other_less : !other_less && !(ok == key && oi == id);
      if (take) {
        key = ok;
        id = oi;
      }
    }
  }
}

// Exact integer keys pack with their id into one u64 whose unsigned order is
// the (key, id) order (ids are >= 0, padding uses INT_MAX): one compare and
// one 64-bit exchange per network stage.
__device__ __forceinline__ uint64_t pack_ki(uint32_t key, int id) {
  return ((uint64_t)key << 32) | (uint64_t)(uint32_t)id;
}

// Bitonic sort of the first W (16 or 32) lanes, ascending, fully unrolled;
// for W = 16 lanes 16..31 must hold values >= every lane below (padding).
template <int W>
__device__ __forceinline__ void warp_sort_u64(uint64_t& v) {
  const int lane = lane_id();
#pragma unroll
  for (int size = 2; size <= W; size <<= 1) {
    const bool up = ((lane & size) == 0);
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint64_t o = __shfl_xor_sync(FULL, v, stride);
      const bool lower = ((lane & stride) == 0);
      // lower lane of an ascending pair keeps the min, of a descending pair the max
      const bool take = (lower == up) ? (o < v) : (o > v);
      v = take ? o : v;
    }
  }
}

// Rank sort of distinct packed words: lanes [0, n) hold the values (lanes >= n
// padding that is never smaller); every valid lane counts the smaller values
// with n independent broadcasts (no dependent chain, unlike a bitonic
// network) and scatters itself through `scratch` (32 u64, shared).
__device__ __forceinline__ void warp_rank_sort_u64(uint64_t& v, int n, uint64_t* scratch) {
  const int lane = lane_id();
  int rank = 0;
  for (int j = 0; j < n; ++j) rank += (__shfl_sync(FULL, v, j) < v) ? 1 : 0;
  __syncwarp();
  if (lane < n) scratch[rank] = v;
  __syncwarp();
  if (lane < n) v = scratch[lane];
  __syncwarp();
}

// Sort of the first n (<= 32) (key, id) lanes, padding (max, INT_MAX) above n.
// With a scratch buffer, exact integer keys use the rank sort above.
template <typename K>
__device__ __forceinline__ void warp_sort_n(K& key, int& id, int n, uint64_t* scratch = nullptr) {
  if constexpr (sizeof(K) == 4) {
    if (scratch) {
      uint64_t v = pack_ki(key, id);
      warp_rank_sort_u64(v, n, scratch);
      key = (K)(v >> 32);
      id = (int)(uint32_t)v;
      return;
    }
    uint64_t v = pack_ki(key, id);
    if (n <= 16)
      warp_sort_u64<16>(v);
    else
      warp_sort_u64<32>(v);
    key = (K)(v >> 32);
    id = (int)(uint32_t)v;
  } else {
    warp_sort(key, id);
  }
}

// ---------------------------------------------------------------- vectors
// Query storage: float queries are kept as float in shared memory, uint8
// queries as uint8.  Distances:
//   float data / float query : double accumulation of ((double)x - (double)q)^2
//   uint8 data / uint8 query : exact uint32 sum of squared byte differences
//   uint8 data / float query : double accumulation (non-integral queries)
template <typename TX, typename TQ> struct VecTraits;
template <> struct VecTraits<float, float> { using Key = double; };
template <> struct VecTraits<uint8_t, uint8_t> { using Key = uint32_t; };
template <> struct VecTraits<uint8_t, float> { using Key = double; };

// Partial distance of the elements [e0, e0+CH) handled by one lane.
// FP32 partial: the lane's share of a float row summed in single precision
// (rounding ~1e-7 relative, far inside the north star's 1e-5 near-tie band);
// the group reduction and everything after it stay FP64, and returned hits
// are re-scored with the exact sequential FP64 sum (FLAG_EXACT_DISTS).
__device__ __forceinline__ float part_f32_sp(const float4 a, const float* q) {
  const float d0 = a.x - q[0], d1 = a.y - q[1], d2 = a.z - q[2], d3 = a.w - q[3];
  return fmaf(d3, d3, fmaf(d2, d2, fmaf(d1, d1, d0 * d0)));
}
#ifndef GGNN_F32_PARTIALS
#define GGNN_F32_PARTIALS 1
#endif
#ifndef GGNN_F32_UNR
#define GGNN_F32_UNR 4  // float rows in flight per lane group
#endif

__device__ __forceinline__ double part_f32(const float4 a, const float* q) {
  double d0 = (double)a.x - (double)q[0], d1 = (double)a.y - (double)q[1];
  double d2 = (double)a.z - (double)q[2], d3 = (double)a.w - (double)q[3];
  double s = d0 * d0;
  s = fma(d1, d1, s);
  s = fma(d2, d2, s);
  return fma(d3, d3, s);
}
__device__ __forceinline__ uint32_t sad_sq4(uint32_t a, uint32_t b, uint32_t acc) {
  uint32_t ad = __vabsdiffu4(a, b);
  return __dp4a(ad, ad, acc);
}
__device__ __forceinline__ uint32_t part_u8(const uint4 a, const uint4 q) {
  uint32_t s = sad_sq4(a.x, q.x, 0u);
  s = sad_sq4(a.y, q.y, s);
  s = sad_sq4(a.z, q.z, s);
  return sad_sq4(a.w, q.w, s);
}

// Distances of `cnt` compacted candidate rows (rows[c], c < cnt, in shared
// memory) to the query qs (shared memory); results go to kout[c] (shared).
// Rows are read with 16-byte vector loads; LPR lanes cooperate on one row
// (LPR = power of two >= 16-byte chunks per row, at most 32), so one load
// instruction covers 32/LPR rows, and UNR row groups are issued before any
// is consumed so their latencies overlap.  Callers __syncwarp() afterwards.
template <int LPR, typename Acc>
__device__ __forceinline__ Acc group_reduce(Acc v) {
#pragma unroll
  for (int o = LPR >> 1; o > 0; o >>= 1) v += KeyOps<Acc>::shfl_xor(v, o);
  return v;
}

// `hook` (warp-collective, independent of the distances) runs once while the
// first row gathers are in flight: the caller's bookkeeping leaves the
// dependent chain of the step.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

template <int LPR, int UNR, typename Hook = NoHook>
__device__ __forceinline__ void dists_f32_vec(const float* X, int64_t d, const float* qs, const int* rows, int cnt,
                                              double* kout, Hook&& hook = Hook()) {
  const int lane = lane_id();
  const int nch = (int)(d >> 2);
  constexpr int RPP = 32 / LPR;
  const int sub = lane & (LPR - 1);
  const int grp = lane / LPR;
  for (int base = 0; base < cnt; base += RPP * UNR) {
    double acc[UNR];
    const float4* rp[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int ci = base + u * RPP + grp;
      int r = ci < cnt ? rows[ci] : -1;
      rp[u] = r >= 0 ? reinterpret_cast<const float4*>(X + (int64_t)r * d) : nullptr;
      acc[u] = 0.0;
    }
    float accf[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) accf[u] = 0.0f;
    // first chunk's loads, then the hook (every lane, also those without a
    // chunk: it is warp-collective), then the chunk loop (LPR < 32: at most
    // one chunk per lane, see dists_u8_vec)
    int c = sub;
    bool have = c < nch;
    float4 v[UNR];
    if (have) {
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (rp[u]) v[u] = __ldg(rp[u] + c);
    }
    if (base == 0) hook();
    while (have) {
      const float* qc = qs + 4 * c;
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (!rp[u]) continue;
        if constexpr (GGNN_F32_PARTIALS) accf[u] += part_f32_sp(v[u], qc);
        else acc[u] += part_f32(v[u], qc);
      }
      c += LPR;
      have = LPR == 32 && c < nch;
      if (have) {
#pragma unroll
        for (int u = 0; u < UNR; ++u)
          if (rp[u]) v[u] = __ldg(rp[u] + c);
      }
    }
    if constexpr (GGNN_F32_PARTIALS) {
#pragma unroll
      for (int u = 0; u < UNR; ++u) acc[u] = (double)accf[u];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      double t = group_reduce<LPR, double>(acc[u]);
      int ci = base + u * RPP + grp;
      if (sub == 0 && ci < cnt) kout[ci] = t;
    }
  }
}

// row gathers through L2 only (ld.global.cg) instead of the read-only L1 path
#ifndef GGNN_GATHER_CG
#define GGNN_GATHER_CG 0
#endif
template <int LPR, int UNR>
__device__ __forceinline__ void dists_u8_vec(const uint8_t* X, int64_t d, const uint8_t* qs, const int* rows,
                                             int cnt, uint32_t* kout) {
  const int lane = lane_id();
  const int nch = (int)(d >> 4);
  constexpr int RPP = 32 / LPR;
  const int sub = lane & (LPR - 1);
  const int grp = lane / LPR;
  for (int base = 0; base < cnt; base += RPP * UNR) {
    uint32_t acc[UNR];
    const uint4* rp[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int ci = base + u * RPP + grp;
      int r = ci < cnt ? rows[ci] : -1;
      rp[u] = r >= 0 ? reinterpret_cast<const uint4*>(X + (int64_t)r * d) : nullptr;
      acc[u] = 0u;
    }
    // choose_lpr picks the smallest power of two >= the chunk count (capped
    // at 32), so below 32 lanes per row every lane owns at most one chunk
    for (int c = sub; c < nch; c += LPR) {
      uint4 v[UNR];
      const uint4 qv = reinterpret_cast<const uint4*>(qs)[c];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (rp[u]) v[u] = GGNN_GATHER_CG ? __ldcg(rp[u] + c) : __ldg(rp[u] + c);
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (rp[u]) acc[u] += part_u8(v[u], qv);
      if constexpr (LPR < 32) break;
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      uint32_t t = group_reduce<LPR, uint32_t>(acc[u]);
      int ci = base + u * RPP + grp;
      if (sub == 0 && ci < cnt) kout[ci] = t;
    }
  }
}

// The LP = 8 uint8 case of dists_u8_vec (rows of 5-8 16-byte chunks: the C2 /
// C5 shapes) with its per-step overhead removed: every lane owns at most one
// chunk, so the query chunk is loaded once, row addresses are one 32-bit
// offset per group into a uint4 view of the table (no 64-bit pointer selects,
// no null checks), and lanes past the row's last chunk load nothing.
#ifndef GGNN_DISTS_V2
#define GGNN_DISTS_V2 1
#endif
template <int UNR, typename Hook>
__device__ __forceinline__ void dists_u8_lp8(const uint8_t* X, int64_t d, const uint8_t* qs, const int* rows, int cnt,
                                             uint32_t* kout, Hook& hook) {
  constexpr int LPR = 8, RPP = 32 / LPR;
  const int lane = lane_id();
  const int sub = lane & (LPR - 1);
  const int grp = lane >> 3;
  const uint32_t nch = (uint32_t)(d >> 4);
  const bool mine = (uint32_t)sub < nch;
  const uint4* X4 = reinterpret_cast<const uint4*>(X) + sub;
  const uint4 qv = mine ? reinterpret_cast<const uint4*>(qs)[sub] : make_uint4(0u, 0u, 0u, 0u);
  if constexpr (UNR == 4) {
    // group g owns candidates base + 4g .. base + 4g + 3 (one 16-byte read of
    // their rows; rows / kout are 16-byte aligned 32-entry arrays), and the
    // four sums are reduced transposed: 4 shuffles instead of 12, after which
    // lane sub (even) of the group holds the sum of candidate 2 (sub & 4) / 4 + (sub & 2) / 2
    for (int base = 0; base < cnt; base += 16) {
      const int c0 = base + 4 * grp;
      const int4 r4 = *reinterpret_cast<const int4*>(rows + c0);
      const int rr[4] = {r4.x, r4.y, r4.z, r4.w};
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        v[u] = make_uint4(0u, 0u, 0u, 0u);
        if (mine && c0 + u < cnt) v[u] = __ldg(X4 + (size_t)(uint32_t)rr[u] * nch);
      }
      if (base == 0) hook();
      uint32_t a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = part_u8(v[u], qv);
      const bool b2 = (sub & 4) != 0, b1 = (sub & 2) != 0;
      uint32_t x0 = b2 ? a[2] : a[0], x1 = b2 ? a[3] : a[1];
      const uint32_t y0 = b2 ? a[0] : a[2], y1 = b2 ? a[1] : a[3];
      x0 += __shfl_xor_sync(FULL, y0, 4);
      x1 += __shfl_xor_sync(FULL, y1, 4);
      uint32_t z = b1 ? x1 : x0;
      const uint32_t w = b1 ? x0 : x1;
      z += __shfl_xor_sync(FULL, w, 2);
      z += __shfl_xor_sync(FULL, z, 1);
      const int ci = c0 + (b2 ? 2 : 0) + (b1 ? 1 : 0);
      if ((sub & 1) == 0 && ci < cnt) kout[ci] = z;
    }
  } else {
    for (int base = 0; base < cnt; base += RPP * UNR) {
      uint4 v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int ci = base + u * RPP + grp;
        v[u] = make_uint4(0u, 0u, 0u, 0u);
        if (mine && ci < cnt) v[u] = __ldg(X4 + (size_t)(uint32_t)rows[ci] * nch);
      }
      if (base == 0) hook();
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const uint32_t t = group_reduce<LPR, uint32_t>(part_u8(v[u], qv));
        const int ci = base + u * RPP + grp;
        if (sub == 0 && ci < cnt) kout[ci] = t;
      }
    }
  }
}

// scalar fallbacks (any d, any alignment): one row at a time, lanes stride d
template <typename TX, typename TQ, typename Key>
__device__ __forceinline__ void dists_scalar(const TX* X, int64_t d, const TQ* qs, const int* rows, int cnt,
                                             Key* kout) {
  const int lane = lane_id();
  for (int c = 0; c < cnt; ++c) {
    const TX* xr = X + (int64_t)rows[c] * d;
    Key s = 0;
    for (int64_t e = lane; e < d; e += 32) {
      if constexpr (sizeof(Key) == 4) {
        int df = (int)xr[e] - (int)qs[e];
        s += (Key)(df * df);
      } else {
        double df = (double)xr[e] - (double)qs[e];
        s = fma(df, df, s);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += KeyOps<Key>::shfl_xor(s, o);
    if (lane == 0) kout[c] = s;
  }
}

template <typename TX, typename TQ>
__device__ __forceinline__ void warp_dists(const TX* X, int64_t d, const TQ* qs, const int* rows, int cnt,
                                           typename VecTraits<TX, TQ>::Key* kout, int lpr) {
  if constexpr (std::is_same<TX, float>::value && std::is_same<TQ, float>::value) {
    switch (lpr) {
      case 32: dists_f32_vec<32, 8>(X, d, qs, rows, cnt, kout); return;
      case 16: dists_f32_vec<16, 4>(X, d, qs, rows, cnt, kout); return;
      case 8: dists_f32_vec<8, 4>(X, d, qs, rows, cnt, kout); return;
      case 4: dists_f32_vec<4, 2>(X, d, qs, rows, cnt, kout); return;
      case 2: dists_f32_vec<2, 2>(X, d, qs, rows, cnt, kout); return;
      case 1: dists_f32_vec<1, 1>(X, d, qs, rows, cnt, kout); return;
      default: break;
    }
  } else if constexpr (std::is_same<TX, uint8_t>::value && std::is_same<TQ, uint8_t>::value) {
    switch (lpr) {
      case 32: dists_u8_vec<32, 4>(X, d, qs, rows, cnt, kout); return;
      case 16: dists_u8_vec<16, 4>(X, d, qs, rows, cnt, kout); return;
      case 8: dists_u8_vec<8, 8>(X, d, qs, rows, cnt, kout); return;
      case 4: dists_u8_vec<4, 4>(X, d, qs, rows, cnt, kout); return;
      case 2: dists_u8_vec<2, 2>(X, d, qs, rows, cnt, kout); return;
      case 1: dists_u8_vec<1, 1>(X, d, qs, rows, cnt, kout); return;
      default: break;
    }
  }
  dists_scalar<TX, TQ>(X, d, qs, rows, cnt, kout);
}

// Compile-time lanes-per-row dispatch: LP > 0 selects one vectorised variant
// (so a kernel instantiated for LP carries only that variant's registers),
// LP == 0 keeps the runtime switch above.  LP must equal choose_lpr(...) of
// the launch; mixed u8-data / float-query searches always use LP == 0.
#ifndef GGNN_U8_UNR
#define GGNN_U8_UNR 4  // row groups in flight for 128-byte uint8 rows (dists_u8_lp8: 16 rows; 3 and 6 measured slower)
#endif
template <typename TX, typename TQ, int LP, typename Hook = NoHook>
__device__ __forceinline__ void warp_dists_t(const TX* X, int64_t d, const TQ* qs, const int* rows, int cnt,
                                             typename VecTraits<TX, TQ>::Key* kout, int lpr, Hook hook = Hook()) {
  if constexpr (LP == 8 && std::is_same<TX, uint8_t>::value && std::is_same<TQ, uint8_t>::value &&
                GGNN_DISTS_V2 != 0) {
    if (cnt > 0) dists_u8_lp8<GGNN_U8_UNR>(X, d, qs, rows, cnt, kout, hook);
    else hook();
    return;
  }
  if constexpr ((LP == 8 || LP == 32) && std::is_same<TX, float>::value && std::is_same<TQ, float>::value) {
    // (every lane owns a chunk of a float row: d / 4 >= LP, see choose_lpr)
    if (cnt > 0) {
      if constexpr (LP == 8) dists_f32_vec<8, 4>(X, d, qs, rows, cnt, kout, hook);
      else dists_f32_vec<32, GGNN_F32_UNR>(X, d, qs, rows, cnt, kout, hook);
    } else {
      hook();
    }
    return;
  }
  hook();
  if constexpr (LP == 8 && std::is_same<TX, uint8_t>::value && std::is_same<TQ, uint8_t>::value) {
    dists_u8_vec<8, GGNN_U8_UNR>(X, d, qs, rows, cnt, kout);
  } else if constexpr (LP == 32 && std::is_same<TX, uint8_t>::value && std::is_same<TQ, uint8_t>::value) {
    dists_u8_vec<32, 4>(X, d, qs, rows, cnt, kout);
  } else if constexpr (LP == 8 && std::is_same<TX, float>::value && std::is_same<TQ, float>::value) {
    dists_f32_vec<8, 4>(X, d, qs, rows, cnt, kout);
  } else if constexpr (LP == 32 && std::is_same<TX, float>::value && std::is_same<TQ, float>::value) {
    dists_f32_vec<32, GGNN_F32_UNR>(X, d, qs, rows, cnt, kout);
  } else {
    warp_dists<TX, TQ>(X, d, qs, rows, cnt, kout, lpr);
  }
}

// Lanes-per-row code for the vectorised paths (0 = scalar fallback).
inline int choose_lpr(int64_t d, int dtype_x, int dtype_q, uintptr_t base) {
  int chunk = 0;
  if (dtype_x == 0 && dtype_q == 0) chunk = 4;
  if (dtype_x == 1 && dtype_q == 1) chunk = 16;
  if (!chunk || d % chunk != 0 || (base & 15)) return 0;
  int64_t nch = d / chunk;
  int lpr = 1;
  while (lpr < nch && lpr < 32) lpr <<= 1;
  return lpr;
}

// Exact sequential float64 squared distance, the reference's _sqdist
// (_core.pyx:30-37) operation for operation: no FMA contraction.
template <typename TX, typename TQ>
__device__ __forceinline__ double seq_sqdist(const TX* xr, const TQ* q, int64_t d) {
  double acc = 0.0;
  for (int64_t i = 0; i < d; ++i) {
    double df = __dsub_rn((double)xr[i], (double)q[i]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return acc;
}

// ---------------------------------------------------------------- membership
// Open-addressing refcount table in shared memory (one per warp).
//   slot == 0          : empty
//   slot == 0xffffffff : tombstone
//   otherwise          : (count << 30) | node, count in 1..3, node < 2^30 - 1
struct RefTable {
  uint32_t* t;
  uint32_t mask;
  int shift;
  static constexpr uint32_t EMPTY = 0u, TOMB = 0xffffffffu, KMASK = (1u << 30) - 1u, ONE = 1u << 30;

  __device__ __forceinline__ uint32_t home(uint32_t key) const { return (key * 2654435761u) >> shift; }

  // per-lane lookup: count of `key` (0 if absent)
  __device__ __forceinline__ uint32_t count(uint32_t key) const {
    uint32_t s = home(key);
    for (;;) {
      uint32_t v = t[s];
      if (v == EMPTY) return 0u;
      if (v != TOMB && (v & KMASK) == key) return v >> 30;
      s = (s + 1) & mask;
    }
  }
  // per-lane insert of an absent key with count 1; returns 1 if an empty slot was consumed
  __device__ __forceinline__ int insert_new(uint32_t key) {
    uint32_t s = home(key);
    for (;;) {
      uint32_t v = t[s];
      if (v == EMPTY || v == TOMB) {
        uint32_t old = atomicCAS(&t[s], v, ONE | key);
        if (old == v) return v == EMPTY ? 1 : 0;
        continue;  // lost the race, re-read this slot
      }
      s = (s + 1) & mask;
    }
  }
  // per-lane insert-or-increment (used by rebuild; no tombstones present)
  __device__ __forceinline__ int add_one(uint32_t key) {
    uint32_t s = home(key);
    for (;;) {
      uint32_t v = t[s];
      if (v == EMPTY) {
        uint32_t old = atomicCAS(&t[s], EMPTY, ONE | key);
        if (old == EMPTY) return 1;
        continue;
      }
      if ((v & KMASK) == key) {
        atomicAdd(&t[s], ONE);
        return 0;
      }
      s = (s + 1) & mask;
    }
  }
  // warp-cooperative location of a live key (uniform result, -1 if absent)
  __device__ __forceinline__ int find_slot(uint32_t key) const {
    const int lane = lane_id();
    uint32_t s0 = home(key);
    for (uint32_t off = 0;; off += 32) {
      uint32_t s = (s0 + off + lane) & mask;
      uint32_t v = t[s];
      unsigned hit = __ballot_sync(FULL, v != TOMB && v != EMPTY && (v & KMASK) == key);
      unsigned emp = __ballot_sync(FULL, v == EMPTY);
      if (hit && (!emp || __ffs(hit) < __ffs(emp))) return (int)((s0 + off + __ffs(hit) - 1) & mask);
      if (emp) return -1;
    }
  }
  // decrement (warp-uniform call); returns true when the count reached zero
  __device__ __forceinline__ bool dec(uint32_t key) {
    int s = find_slot(key);
    bool zero = false;
    if (s >= 0) {
      uint32_t v = t[s];
      zero = (v >> 30) == 1u;
      __syncwarp();
      if (lane_id() == 0) t[s] = zero ? TOMB : v - ONE;
    }
    __syncwarp();
    return zero;
  }
  __device__ __forceinline__ void inc(uint32_t key) {
    int s = find_slot(key);
    if (s >= 0) {
      uint32_t v = t[s];
      __syncwarp();
      if (lane_id() == 0) t[s] = v + ONE;
    }
    __syncwarp();
  }
  // increment of a key known to be present: one lane probes (the key sits
  // within a slot or two of its home), no warp-wide ballots
  __device__ __forceinline__ void inc_present(uint32_t key) {
    if (lane_id() == 0) {
      uint32_t s = home(key);
      for (;;) {
        const uint32_t v = t[s];
        if (v != TOMB && v != EMPTY && (v & KMASK) == key) {
          t[s] = v + ONE;
          break;
        }
        if (v == EMPTY) break;  // absent: nothing to count (as inc)
        s = (s + 1) & mask;
      }
    }
    __syncwarp();
  }
  __device__ __forceinline__ void tomb(uint32_t key) {
    int s = find_slot(key);
    __syncwarp();
    if (s >= 0 && lane_id() == 0) t[s] = TOMB;
    __syncwarp();
  }
  // per-lane tombstoning of a live key with count 1 (distinct keys per lane).
  // A lane probing past another lane's slot may read it before or after that
  // lane writes TOMB; either value is "occupied, not my key", so the probe
  // continues the same way (racecheck reports this as a benign WAR warning).
  __device__ __forceinline__ void tomb_lane(uint32_t key) {
    uint32_t s = home(key);
    for (;;) {
      const uint32_t v = t[s];
      if (v != TOMB && v != EMPTY && (v & KMASK) == key) {
        t[s] = TOMB;
        return;
      }
      s = (s + 1) & mask;
    }
  }
  __device__ __forceinline__ void clear() {  // (tables of >= 64 slots, 16-byte aligned)
    for (uint32_t i = 4u * lane_id(); i <= mask; i += 128u) *reinterpret_cast<uint4*>(t + i) = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
  }
};

}  // namespace ggnn
