// ggnn_shard.cu -- id globalization and the exact G-way merge of per-shard
// top-k lists (the reference's _merge_shard_results, shard.py:91-110).
//
// One warp per query: the G * k_in candidates of the query are streamed
// through the warp 32 at a time and folded into a running ascending top-32
// by the bitonic merge of search.cuh (topk_merge_chunk), keyed by
// (distance f64, dataset id) -- the reference's sort key (shard.py:106).
// The shard whose list holds the overall best hit (ids of different shards
// are disjoint) gives terminated_by (shard.py:108).
#include <climits>
#include "ggnn_capi_util.cuh"
#include "ggnn_p2p.h"
#include "ggnn_search.cuh"
#include "ggnn_shard.h"

namespace ggnn {
namespace {

__host__ __device__ inline size_t block_dists_off(int64_t m, int k_in) {
  return (((size_t)m * k_in * 4) + 15) & ~size_t(15);
}
__host__ __device__ inline size_t block_cnt_off(int64_t m, int k_in) {
  return block_dists_off(m, k_in) + (size_t)m * k_in * 8;
}
__host__ __device__ inline size_t block_bytes(int64_t m, int k_in) {
  return (block_cnt_off(m, k_in) + (size_t)m * 5 * 4 + 255) & ~size_t(255);
}

__global__ void globalize_kernel(int32_t* ids, int64_t count, const int32_t* gid, int64_t size) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = ids[i];
    if (v >= 0 && v < size) ids[i] = __ldg(gid + v);
  }
}

struct MergeShardArgs {
  const uint8_t* blocks;
  size_t block_bytes, dists_off, cnt_off;
  int G;
  int64_t m;
  int k_in, k_out;
  int32_t* out_ids;
  double* out_dists;
  int32_t* out_cnt;
  // fused exchange: wait until every flags[g] == epoch (nullptr: no wait)
  const uint32_t* flags;
  uint32_t epoch;
  int32_t* error;
};

// Bounded acquire-spin of one thread on G peer-written flags (~10 s at
// 2 GHz, then *error = 1 and the merge proceeds on whatever arrived).
__device__ void wait_flags(const uint32_t* flags, int G, uint32_t epoch, int32_t* error) {
  const long long t0 = clock64();
  for (int g = 0; g < G; ++g) {
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + g) : "memory");
      if (v == epoch) break;
      if (clock64() - t0 > 20000000000ll) {
        if (error) atomicExch(error, 1);
        return;
      }
      __nanosleep(200);
    }
  }
  __threadfence();
}

__global__ void __launch_bounds__(256) shard_merge_kernel(const __grid_constant__ MergeShardArgs a) {
  if (a.flags) {
    if (threadIdx.x == 0) wait_flags(a.flags, a.G, a.epoch, a.error);
    __syncthreads();
  }
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= a.m) return;
  const int lane = lane_id();
  using KO = KeyOps<double>;
  const int total = a.G * a.k_in;
  long long vsum = 0, tsum = 0;
  // ranks [b, b + 32) of the merged list per pass: pass b keeps the pairs
  // ordered after the last one of pass b - 32 (one pass for k_out <= 32)
  int best = INT_MAX;
  double ak = 0.0;
  int ai = -1;
  for (int b = 0; b < a.k_out; b += 32) {
    const int kk = min(32, a.k_out - b);
    double bk = KO::max_key();
    int bi = INT_MAX;
    if (b == 0 || ai != INT_MAX) {
      for (int base = 0; base < total; base += 32) {
        const int e = base + lane;
        double ck = KO::max_key();
        int cx = INT_MAX;
        if (e < total) {
          const int g = e / a.k_in, j = e - g * a.k_in;
          const uint8_t* blk = a.blocks + (size_t)g * a.block_bytes;
          const int32_t id = reinterpret_cast<const int32_t*>(blk)[q * a.k_in + j];
          if (id >= 0) {
            ck = reinterpret_cast<const double*>(blk + a.dists_off)[q * a.k_in + j];
            cx = id;
            if (b > 0 && !key_less(ak, ai, ck, cx)) {
              ck = KO::max_key();
              cx = INT_MAX;
            }
          }
        }
        topk_merge_chunk(bk, bi, ck, cx, kk);
      }
    }
    if (b == 0) best = __shfl_sync(FULL, bi, 0);
    ak = KO::shfl(bk, 31);
    ai = __shfl_sync(FULL, bi, 31);
    if (lane < kk) {
      const bool ok = bi != INT_MAX;
      a.out_ids[q * a.k_out + b + lane] = ok ? bi : -1;
      a.out_dists[q * a.k_out + b + lane] = ok ? bk : KO::max_key();
    }
  }
  if (a.out_cnt) {
    for (int g = lane; g < a.G; g += 32) {
      const int32_t* c = reinterpret_cast<const int32_t*>(a.blocks + (size_t)g * a.block_bytes + a.cnt_off) + q * 5;
      vsum += c[0];
      tsum += c[1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      vsum += __shfl_xor_sync(FULL, vsum, o);
      tsum += __shfl_xor_sync(FULL, tsum, o);
    }
  }
  if (a.out_cnt) {
    int term = TERM_EMPTY;  // shard.py:108 "queue-empty" when nothing was found
    if (best != INT_MAX) {
      // exactly one shard list holds `best` (shard ids are disjoint).  It is
      // not necessarily that list's first entry: a shard orders its hits by
      // (dist, LOCAL id), and a permutation can reverse two tied hits, so
      // every entry is searched, not position 0 alone.
      int src = -1;
      for (int base = 0; base < total && src < 0; base += 32) {
        const int e = base + lane;
        bool hit = false;
        if (e < total) {
          const int g = e / a.k_in, j = e - g * a.k_in;
          hit = reinterpret_cast<const int32_t*>(a.blocks + (size_t)g * a.block_bytes)[q * a.k_in + j] == best;
        }
        const unsigned bal = __ballot_sync(FULL, hit);
        if (bal) src = (base + __ffs(bal) - 1) / a.k_in;
      }
      if (src >= 0)
        term = reinterpret_cast<const int32_t*>(a.blocks + (size_t)src * a.block_bytes + a.cnt_off)[q * 5 + 2];
    }
    if (lane == 0) {
      int32_t* c = a.out_cnt + q * 5;
      c[0] = (int32_t)vsum;
      c[1] = (int32_t)tsum;
      c[2] = term;
      c[3] = 0;
      c[4] = 0;
    }
  }
}

struct SignalArgs {
  uint32_t* flags[GGNN_P2P_MAX_RANKS];  // flag `rank` of every receive allocation (parity half)
  int G;
  uint32_t epoch;
};

__global__ void p2p_signal_kernel(const __grid_constant__ SignalArgs a) {
  const int g = threadIdx.x;
  if (g >= a.G) return;
  __threadfence_system();  // this rank's pushed rows are visible system-wide first
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flags[g]), "r"(a.epoch) : "memory");
}

inline size_t p2p_half(int G, int64_t m, int k) {
  return (size_t)G * block_bytes(m, k) + (((size_t)G * 4 + 255) & ~size_t(255));
}

}  // namespace
}  // namespace ggnn

using namespace ggnn;

extern "C" size_t ggnn_p2p_bytes(int32_t G, int64_t m, int32_t k) { return 2 * p2p_half(G, m, k); }

extern "C" int ggnn_p2p_alloc(size_t bytes, void** d_ptr, void* ipc_handle_out) {
  GGNN_CHECK_ARG(d_ptr && ipc_handle_out && bytes > 0, "ggnn_p2p_alloc: invalid arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == GGNN_IPC_HANDLE_BYTES, "IPC handle size");
  void* p = nullptr;
  GGNN_CUDA_TRY(cudaMalloc(&p, bytes));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);  // no leak on the error path
    ::ggnn::set_error("ggnn_p2p_alloc: %s", cudaGetErrorString(e));
    return GGNN_E_CUDA;
  }
  memcpy(ipc_handle_out, &h, sizeof(h));
  *d_ptr = p;
  return GGNN_OK;
}

extern "C" int ggnn_p2p_open(const void* ipc_handle, void** d_peer_ptr) {
  GGNN_CHECK_ARG(ipc_handle && d_peer_ptr, "ggnn_p2p_open: invalid arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  GGNN_CUDA_TRY(cudaIpcOpenMemHandle(d_peer_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return GGNN_OK;
}

extern "C" int ggnn_p2p_close(void* d_peer_ptr) {
  GGNN_CUDA_TRY(cudaIpcCloseMemHandle(d_peer_ptr));
  return GGNN_OK;
}

extern "C" int ggnn_p2p_free(void* d_ptr) {
  GGNN_CUDA_TRY(cudaFree(d_ptr));
  return GGNN_OK;
}

extern "C" int ggnn_p2p_signal(const ggnn_push* push, int64_t m, int32_t k, uint32_t epoch, void* stream) {
  GGNN_CHECK_ARG(push && push->nranks >= 1 && push->nranks <= GGNN_P2P_MAX_RANKS && push->rank >= 0 &&
                     push->rank < push->nranks && (push->parity == 0 || push->parity == 1),
                 "invalid push descriptor");
  const size_t half = p2p_half(push->nranks, m, k);
  SignalArgs a;
  a.G = push->nranks;
  a.epoch = epoch;
  for (int g = 0; g < push->nranks; ++g)
    a.flags[g] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(push->d_peers[g]) + (size_t)push->parity * half +
                                             (size_t)push->nranks * block_bytes(m, k)) + push->rank;
  p2p_signal_kernel<<<1, 32, 0, as_stream(stream)>>>(a);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

extern "C" size_t ggnn_shard_block_bytes(int64_t m, int32_t k_in) { return block_bytes(m, k_in); }
extern "C" size_t ggnn_shard_block_dists_offset(int64_t m, int32_t k_in) { return block_dists_off(m, k_in); }
extern "C" size_t ggnn_shard_block_counters_offset(int64_t m, int32_t k_in) { return block_cnt_off(m, k_in); }

extern "C" int ggnn_shard_globalize(int32_t* d_ids, int64_t count, const int32_t* d_gid_of_local, int64_t size,
                                    void* stream) {
  GGNN_CHECK_ARG(count >= 0 && size >= 0, "ggnn_shard_globalize: negative size");
  if (count == 0) return GGNN_OK;
  GGNN_CHECK_ARG(d_ids && d_gid_of_local, "ggnn_shard_globalize: null pointer");
  const int threads = 256;
  const int64_t want = (count + threads - 1) / threads;
  const int blocks = (int)(want < 148 * 8 ? want : 148 * 8);
  globalize_kernel<<<blocks, threads, 0, as_stream(stream)>>>(d_ids, count, d_gid_of_local, size);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

static int shard_merge_impl(const void* d_blocks, int32_t G, int64_t m, int32_t k_in, int32_t k_out,
                            int32_t* d_out_ids, double* d_out_dists, int32_t* d_out_counters, const uint32_t* flags,
                            uint32_t epoch, int32_t* error, void* stream);

extern "C" int ggnn_shard_merge(const void* d_blocks, int32_t G, int64_t m, int32_t k_in, int32_t k_out,
                                int32_t* d_out_ids, double* d_out_dists, int32_t* d_out_counters, void* stream) {
  return shard_merge_impl(d_blocks, G, m, k_in, k_out, d_out_ids, d_out_dists, d_out_counters, nullptr, 0u, nullptr,
                          stream);
}

extern "C" int ggnn_shard_merge_wait(const void* d_recv, int32_t parity, uint32_t epoch, int32_t G, int64_t m,
                                     int32_t k, int32_t k_out, int32_t* d_out_ids, double* d_out_dists,
                                     int32_t* d_out_counters, int32_t* d_error, void* stream) {
  GGNN_CHECK_ARG(d_recv && (parity == 0 || parity == 1) && G >= 1 && G <= GGNN_P2P_MAX_RANKS,
                 "ggnn_shard_merge_wait: invalid arguments");
  const uint8_t* half = static_cast<const uint8_t*>(d_recv) + (size_t)parity * p2p_half(G, m, k);
  const uint32_t* flags = reinterpret_cast<const uint32_t*>(half + (size_t)G * block_bytes(m, k));
  return shard_merge_impl(half, G, m, k, k_out, d_out_ids, d_out_dists, d_out_counters, flags, epoch, d_error,
                          stream);
}

static int shard_merge_impl(const void* d_blocks, int32_t G, int64_t m, int32_t k_in, int32_t k_out,
                            int32_t* d_out_ids, double* d_out_dists, int32_t* d_out_counters, const uint32_t* flags,
                            uint32_t epoch, int32_t* error, void* stream) {
  GGNN_CHECK_ARG(G >= 1 && m >= 0 && k_in >= 1, "ggnn_shard_merge: bad shape G=%d m=%lld k_in=%d", G, (long long)m,
                 k_in);
  GGNN_CHECK_ARG(k_out >= 1, "ggnn_shard_merge: k_out must be >= 1, got %d", k_out);
  if (m == 0) return GGNN_OK;
  GGNN_CHECK_ARG(d_blocks && d_out_ids && d_out_dists, "ggnn_shard_merge: null pointer");
  MergeShardArgs a;
  a.blocks = static_cast<const uint8_t*>(d_blocks);
  a.block_bytes = block_bytes(m, k_in);
  a.dists_off = block_dists_off(m, k_in);
  a.cnt_off = block_cnt_off(m, k_in);
  a.G = G;
  a.m = m;
  a.k_in = k_in;
  a.k_out = k_out;
  a.out_ids = d_out_ids;
  a.out_dists = d_out_dists;
  a.out_cnt = d_out_counters;
  a.flags = flags;
  a.epoch = epoch;
  a.error = error;
  const int wpb = 8;
  const int64_t blocks = (m + wpb - 1) / wpb;
  shard_merge_kernel<<<(unsigned)blocks, wpb * 32, 0, as_stream(stream)>>>(a);
  count_launch();
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}
