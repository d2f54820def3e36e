// ggnn_bf_tc.cu -- exact brute-force top-k on the tcgen05 tensor cores for
// uint8 tables: the reference's exhaustive_topk (_core.pyx:86-104) as used by
// brute_force_oracle (evaluate.py:32-57), for a whole query batch at once.
//
// D = Q X^T runs as tcgen05.mma kind::i8 (u8 x u8 -> s32, exact) with a
// 128-query A tile resident in shared memory and 256-row X tiles streamed
// through two cp.async stages; each X tile's products land in one of two
// 256-column TMEM accumulators, so the MMA of tile t overlaps the top-k
// epilogue of tile t-1.  The epilogue turns products into exact squared
// distances ||q||^2 + ||x||^2 - 2 q.x and keeps, per (query, column half), a
// sorted top-k of packed (distance << 32 | row) words -- ties by ascending
// row, as the reference.  CTAs split X into ranges; the 2 x splits partial
// lists per query are merged by ggnn_shard_merge.
#include <algorithm>
#include <climits>
#include <cstring>

#include "ggnn_capi_util.cuh"
#include "ggnn_common.cuh"
#include "ggnn_shard.h"
#include "ggnn_tc.cuh"

namespace ggnn {

__device__ int g_bf_timeouts = 0;

namespace {

constexpr int BF_M = 128;        // queries per CTA (TMEM lanes)
constexpr int BF_N = 256;        // X rows per tile (accumulator columns)
// k <= 32: 8 warps, lane quarter = warp & 3, column half = warp >> 2 (two
// partial lists per query); 32 < k <= 128: 4 warps, one list per query
// (the per-thread lists of k packed words then fill the shared memory).
constexpr int BF_K_SMALL = 32;
constexpr int BF_K_MAX = 128;

struct BfArgs {
  const uint8_t* X;
  int64_t n;
  int d;
  const uint8_t* Q;
  const int32_t* qrows;
  int64_t m;
  const uint32_t* xnorm;
  int k;
  int64_t tiles;             // ceil(n / BF_N)
  int64_t tiles_per_split;
  int splits;
  uint8_t* blocks;           // 2 * splits shard blocks of (m, k)
  size_t block_bytes, dists_off;
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void sqnorm_u8_kernel(const uint8_t* X, int64_t n, int d, uint32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4* r = reinterpret_cast<const uint4*>(X + i * d);
  uint32_t s = 0;
  for (int c = 0; c < (d >> 4); ++c) {
    const uint4 v = __ldg(r + c);
    s = __dp4a(v.x, v.x, s);
    s = __dp4a(v.y, v.y, s);
    s = __dp4a(v.z, v.z, s);
    s = __dp4a(v.w, v.w, s);
  }
  out[i] = s;
}

inline size_t bf_smem(int d, int k, int threads) {
  return (size_t)BF_M * d + 2 * (size_t)BF_N * d + 3 * BF_N * 4 + BF_M * 4 + (size_t)threads * (k + 1) * 8 + 32;
}

template <int HALVES>
__global__ void __launch_bounds__(128 * HALVES, 1) bf_tc_kernel(const __grid_constant__ BfArgs a) {
  constexpr int THREADS = 128 * HALVES;
  constexpr int COLS = BF_N / HALVES;  // columns scanned per thread and tile
  extern __shared__ __align__(16) uint8_t smem_bf[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.d, nch = K >> 4;
  const int64_t qt = blockIdx.x / a.splits, sp = blockIdx.x % a.splits;
  const int64_t q0 = qt * BF_M;
  const int64_t t_begin = sp * a.tiles_per_split;
  const int64_t t_end = min(a.tiles, t_begin + a.tiles_per_split);
  uint8_t* A = smem_bf;
  uint8_t* B = A + (size_t)BF_M * K;  // two stages of BF_N * K
  uint32_t* xn = reinterpret_cast<uint32_t*>(B + 2 * (size_t)BF_N * K);  // three stages of BF_N
  uint32_t* qn = xn + 3 * BF_N;
  uint64_t* top = reinterpret_cast<uint64_t*>(qn + BF_M);
  const int tstride = a.k + 1;
  uint64_t* mbar = top + (size_t)THREADS * tstride;
  uint32_t* taddr = reinterpret_cast<uint32_t*>(mbar + 2);

  if (warp == 0) tc::tmem_alloc<512>(taddr);
  if (tid == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
  }
  // query tile (rows past m are zero) and its norms
  for (int t = tid; t < BF_M * nch; t += THREADS) {
    const int r = t / nch, c = t - r * nch;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (q0 + r < a.m) {
      const uint8_t* src = a.qrows ? a.X + (int64_t)__ldg(a.qrows + q0 + r) * K : a.Q + (q0 + r) * K;
      v = __ldg(reinterpret_cast<const uint4*>(src) + c);
    }
    *reinterpret_cast<uint4*>(A + tc::il_offset(r, c * 16, K)) = v;
  }
  uint64_t* mytop = top + (size_t)tid * tstride;
  for (int j = 0; j < a.k; ++j) mytop[j] = ~0ull;
  uint64_t kth = ~0ull;

  auto load_tile = [&](int64_t t, int stage) {
    const uint32_t bs = tc::smem_u32(B + (size_t)stage * BF_N * K);
    const int64_t r0 = t * BF_N;
    for (int e = tid; e < BF_N * nch; e += THREADS) {
      const int r = e / nch, c = e - r * nch;
      const bool valid = r0 + r < a.n;
      const uint8_t* src = a.X + (valid ? (r0 + r) : 0) * (int64_t)K + c * 16;
      cp_async16(bs + tc::il_offset(r, c * 16, K), src, valid);
    }
    const uint32_t ns = tc::smem_u32(xn + (t % 3) * BF_N);
    for (int r = tid; r < BF_N / 4; r += THREADS) {
      const bool valid = r0 + 4 * r + 3 < a.n;
      if (valid) {
        cp_async16(ns + r * 16, a.xnorm + r0 + 4 * r, true);
      } else {
        for (int q = 0; q < 4; ++q) xn[(t % 3) * BF_N + 4 * r + q] = r0 + 4 * r + q < a.n ? a.xnorm[r0 + 4 * r + q] : 0u;
      }
    }
    cp_async_commit();
  };

  if (t_begin < t_end) load_tile(t_begin, 0);
  cp_async_wait_all();
  tc::fence_async_smem();
  __syncthreads();
  if (tid < BF_M) {
    uint32_t s = 0;
    for (int c = 0; c < nch; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(A + tc::il_offset(tid, c * 16, K));
      s = __dp4a(v.x, v.x, s);
      s = __dp4a(v.y, v.y, s);
      s = __dp4a(v.z, v.z, s);
      s = __dp4a(v.w, v.w, s);
    }
    qn[tid] = s;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *taddr;
  const uint32_t idesc = tc::idesc_u8(BF_M, BF_N);
  const uint32_t sbo = (uint32_t)nch * 128u;
  const int wq = warp & 3, half = HALVES == 2 ? (warp >> 2) : 0;
  const int row = wq * 32 + lane;
  const uint32_t qnr = qn[row];
  uint32_t phase[2] = {0u, 0u};

  auto epilogue = [&](int64_t t, int stage) {
    const uint32_t* xs = xn + (t % 3) * BF_N;
    const int64_t r0 = t * BF_N;
    const uint32_t base = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(stage * BF_N + half * COLS);
    for (int c0 = 0; c0 < COLS; c0 += 16) {
      uint32_t v[16];
      tc::tmem_ld16(base + (uint32_t)c0, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = half * COLS + c0 + j;
        const int64_t id = r0 + col;
        const uint32_t dist = qnr + xs[col] - 2u * v[j];
        const uint64_t pk = ((uint64_t)dist << 32) | (uint64_t)(uint32_t)id;
        if (id < a.n && pk < kth) {
          int p = a.k - 1;
          while (p > 0 && mytop[p - 1] > pk) {
            mytop[p] = mytop[p - 1];
            --p;
          }
          mytop[p] = pk;
          kth = mytop[a.k - 1];
        }
      }
    }
  };

  bool ok = true;
  for (int64_t t = t_begin; t < t_end; ++t) {
    const int stage = (int)((t - t_begin) & 1);
    if (tid == 0) {
      const uint32_t abase = tc::smem_u32(A);
      const uint32_t bbase = tc::smem_u32(B + (size_t)stage * BF_N * K);
      for (int s = 0; s < (K >> 5); ++s)
        tc::mma_u8(tmem + (uint32_t)(stage * BF_N), tc::smem_desc(abase + (uint32_t)s * 256u, 128u, sbo),
                   tc::smem_desc(bbase + (uint32_t)s * 256u, 128u, sbo), idesc, s > 0 ? 1u : 0u);
      tc::commit(&mbar[stage]);
    }
    __syncwarp();
    if (t > t_begin) {
      const int ps = stage ^ 1;
      ok &= tc::mbar_wait(&mbar[ps], phase[ps]);
      phase[ps] ^= 1u;
      tc::fence_after_sync();
      if (t + 1 < t_end) load_tile(t + 1, ps);  // stage ps is free: its MMA is done
      epilogue(t - 1, ps);
    } else if (t + 1 < t_end) {
      load_tile(t + 1, stage ^ 1);
    }
    cp_async_wait_all();
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  if (t_begin < t_end) {
    const int ls = (int)((t_end - 1 - t_begin) & 1);
    ok &= tc::mbar_wait(&mbar[ls], phase[ls]);
    tc::fence_after_sync();
    epilogue(t_end - 1, ls);
  }
  if (!ok && lane == 0) atomicAdd(&g_bf_timeouts, 1);
  // this thread's partial top-k -> block (HALVES * sp + half)
  if (q0 + row < a.m) {
    uint8_t* blk = a.blocks + (size_t)(HALVES * sp + half) * a.block_bytes;
    int32_t* ids = reinterpret_cast<int32_t*>(blk) + (q0 + row) * a.k;
    double* ds = reinterpret_cast<double*>(blk + a.dists_off) + (q0 + row) * a.k;
    for (int j = 0; j < a.k; ++j) {
      const uint64_t v = mytop[j];
      ids[j] = v == ~0ull ? -1 : (int32_t)(uint32_t)v;
      ds[j] = v == ~0ull ? __longlong_as_double(0x7ff0000000000000ll) : (double)(uint32_t)(v >> 32);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_free<512>(tmem);
}

// k-way merge of G ascending (dist, id) lists per query (k > 32 path of the
// brute force; ggnn_shard_merge covers k <= 32).  One thread per query.
__global__ void merge_lists_kernel(const uint8_t* blocks, size_t block_bytes, size_t dists_off, int G, int64_t m,
                                   int k, int32_t* out_ids, double* out_dists) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= m) return;
  int head[16];
  for (int g = 0; g < G; ++g) head[g] = 0;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    double bd = 0.0;
    int bi = INT_MAX;
    for (int g = 0; g < G; ++g) {
      if (head[g] >= k) continue;
      const uint8_t* blk = blocks + (size_t)g * block_bytes;
      const int32_t id = reinterpret_cast<const int32_t*>(blk)[q * k + head[g]];
      if (id < 0) continue;
      const double dd = reinterpret_cast<const double*>(blk + dists_off)[q * k + head[g]];
      if (best < 0 || dd < bd || (dd == bd && id < bi)) {
        best = g;
        bd = dd;
        bi = id;
      }
    }
    out_ids[q * k + j] = best < 0 ? -1 : bi;
    out_dists[q * k + j] = best < 0 ? __longlong_as_double(0x7ff0000000000000ll) : bd;
    if (best >= 0) ++head[best];
  }
}

}  // namespace

// true when the tensor-core path applies to this scan
bool bf_tc_eligible(const ggnn_vectors* X, const int32_t* d_rows, const ggnn_queries* Q, int k) {
  const int qd = Q->d_rows ? X->dtype : Q->dtype;
  const int dmax = k <= BF_K_SMALL ? 224 : 128;
  return X->dtype == GGNN_U8 && qd == GGNN_U8 && d_rows == nullptr && k >= 1 && k <= BF_K_MAX && X->d % 32 == 0 &&
         X->d <= dmax && X->n < INT32_MAX && (reinterpret_cast<uintptr_t>(X->d_data) & 15) == 0 &&
         (Q->d_rows || (reinterpret_cast<uintptr_t>(Q->d_data) & 15) == 0);
}

int bf_topk_tc(const ggnn_vectors* X, const ggnn_queries* Q, int k, int32_t* d_ids, double* d_dists,
               cudaStream_t st) {
  const int64_t m = Q->m, n = X->n;
  if (m == 0) return GGNN_OK;
  DevInfo di = dev_info();
  const int64_t qtiles = (m + BF_M - 1) / BF_M;
  const int64_t tiles = (n + BF_N - 1) / BF_N;
  const int halves = k <= BF_K_SMALL ? 2 : 1;
  int64_t splits = std::max<int64_t>(1, (2 * (int64_t)std::max(di.sm_count, 1) + qtiles - 1) / qtiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, tiles / 4));
  if (halves == 1) splits = std::min<int64_t>(splits, 16);  // merge_lists_kernel keeps 16 list heads
  const int64_t per = (tiles + splits - 1) / splits;
  splits = (tiles + per - 1) / per;
  const size_t bb = ggnn_shard_block_bytes(m, k);
  uint8_t* blocks = nullptr;
  uint32_t* xnorm = nullptr;
  GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&blocks), bb * halves * splits, st));
  GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&xnorm), (size_t)n * 4, st));
  GGNN_CUDA_TRY(cudaMemsetAsync(blocks, 0, bb * halves * splits, st));
  const uint8_t* Xd = static_cast<const uint8_t*>(X->d_data);
  sqnorm_u8_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Xd, n, X->d, xnorm);
  count_launch();
  GGNN_LAUNCH_CHECK();
  BfArgs a;
  a.X = Xd;
  a.n = n;
  a.d = X->d;
  a.Q = static_cast<const uint8_t*>(Q->d_data);
  a.qrows = Q->d_rows;
  a.m = m;
  a.xnorm = xnorm;
  a.k = k;
  a.tiles = tiles;
  a.tiles_per_split = per;
  a.splits = (int)splits;
  a.blocks = blocks;
  a.block_bytes = bb;
  a.dists_off = ggnn_shard_block_dists_offset(m, k);
  const size_t smem = bf_smem(X->d, k, 128 * halves);
  int rc = GGNN_OK;
  if (halves == 2) {
    GGNN_CUDA_TRY(cudaFuncSetAttribute(bf_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bf_tc_kernel<2><<<(unsigned)(qtiles * splits), 256, smem, st>>>(a);
    count_launch();
    GGNN_LAUNCH_CHECK();
    rc = ggnn_shard_merge(blocks, (int32_t)(2 * splits), m, k, k, d_ids, d_dists, nullptr, st);
  } else {
    GGNN_CUDA_TRY(cudaFuncSetAttribute(bf_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bf_tc_kernel<1><<<(unsigned)(qtiles * splits), 128, smem, st>>>(a);
    count_launch();
    GGNN_LAUNCH_CHECK();
    merge_lists_kernel<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(blocks, bb, a.dists_off, (int)splits, m, k,
                                                                     d_ids, d_dists);
    count_launch();
    GGNN_LAUNCH_CHECK();
  }
  cudaFreeAsync(blocks, st);
  cudaFreeAsync(xnorm, st);
  return rc;
}

}  // namespace ggnn

namespace ggnn {
int bf_tf32_timeouts();  // ggnn_bf_tf32.cu
}

extern "C" int ggnn_bf_timeouts(void) {
  int v = 0;
  if (cudaMemcpyFromSymbol(&v, ggnn::g_bf_timeouts, sizeof(int)) != cudaSuccess) return -1;
  const int w = ggnn::bf_tf32_timeouts();
  return w < 0 ? -1 : v + w;
}
