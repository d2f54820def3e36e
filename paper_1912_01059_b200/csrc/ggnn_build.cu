// ggnn_build.cu -- construction kernels: within-batch exact kNN (leaf and
// coarse-segment brute force), merge of descent hits into direct slots,
// inverse-link claims, and layer statistics.  C-ABI entry points are declared
// in include/ggnn_build.h.
#include <algorithm>
#include <climits>
#include <cstring>

#include "ggnn_build.h"
#include "ggnn_capi_util.cuh"
#include "ggnn_search.cuh"

namespace ggnn {

// ---------------------------------------------------------------- leaf kNN
// One CTA per batch.  The batch's vectors are staged in shared memory with a
// one-word row pad (conflict-free column reads), then each warp takes rows i
// and scores all j in chunks of 32 (one j per lane), merging each chunk into a
// running top-k_nn by (distance, position) -- the reference's
// batch_bruteforce (_core.pyx:107-130).  Float data uses the sequential FP64
// sum per pair, i.e. the reference's exact _sqdist; uint8 data exact integers.
struct LeafArgs {
  const void* X;
  int64_t d;
  const int32_t* nodes;    // layer-local ids of batch members (concatenated)
  const int32_t* rows;     // dataset rows of the members (nullptr = nodes)
  const int64_t* offsets;  // nbatches + 1
  int k_nn;
  int32_t* pos;            // (total, k_nn) or nullptr
  double* dist;            // (total, k_nn) or nullptr
  int32_t* adj;            // layer outputs (optional)
  int k;
  double* nnd;
  double* dnn1;
  int32_t* reduced;
  size_t smem_limit;
};

template <typename TX>
struct LeafRowAccess;

template <>
struct LeafRowAccess<float> {
  // sequential FP64, operation for operation the reference's _sqdist
  static __device__ __forceinline__ double dist(const float* a, const float* b, int64_t d) {
    double acc = 0.0;
    for (int64_t e = 0; e < d; ++e) {
      double df = __dsub_rn((double)a[e], (double)b[e]);
      acc = __dadd_rn(acc, __dmul_rn(df, df));
    }
    return acc;
  }
  static constexpr int PAD_ELEMS = 1;
};

template <>
struct LeafRowAccess<uint8_t> {
  static __device__ __forceinline__ double dist(const uint8_t* a, const uint8_t* b, int64_t d) {
    uint32_t acc = 0;
    if ((d & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 3) == 0) {
      const uint32_t* aw = reinterpret_cast<const uint32_t*>(a);
      const uint32_t* bw = reinterpret_cast<const uint32_t*>(b);
      for (int64_t e = 0; e < (d >> 2); ++e) acc = sad_sq4(aw[e], bw[e], acc);
    } else {
      for (int64_t e = 0; e < d; ++e) {
        int df = (int)a[e] - (int)b[e];
        acc += (uint32_t)(df * df);
      }
    }
    return (double)acc;
  }
  static constexpr int PAD_ELEMS = 4;
};

template <typename TX>
__global__ void __launch_bounds__(256) leaf_knn_kernel(const __grid_constant__ LeafArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int b = blockIdx.x;
  const int64_t off = a.offsets[b];
  const int m = (int)(a.offsets[b + 1] - off);
  const int lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const TX* X = reinterpret_cast<const TX*>(a.X);
  const int64_t stride = a.d + LeafRowAccess<TX>::PAD_ELEMS;
  const bool staged = (size_t)m * stride * sizeof(TX) <= a.smem_limit;
  TX* S = reinterpret_cast<TX*>(smem);
  if (staged) {
    for (int64_t t = threadIdx.x; t < (int64_t)m * a.d; t += blockDim.x) {
      int64_t r = t / a.d, e = t - r * a.d;
      int32_t node = a.nodes[off + r];
      int32_t row = a.rows ? a.rows[off + r] : node;
      S[r * stride + e] = X[(int64_t)row * a.d + e];
    }
  }
  __syncthreads();
  const int k_eff = min(a.k_nn, m - 1);
  if (k_eff < a.k_nn && threadIdx.x == 0 && a.reduced) atomicAdd(a.reduced, 1);
  auto rowp = [&](int r) -> const TX* {
    if (staged) return S + (int64_t)r * stride;
    int32_t node = a.nodes[off + r];
    int32_t row = a.rows ? a.rows[off + r] : node;
    return X + (int64_t)row * a.d;
  };
  for (int i = warp; i < m; i += nw) {
    double bk = KeyOps<double>::max_key();
    int bi = INT_MAX;
    const TX* xi = rowp(i);
    if (k_eff > 0) {
      for (int jb = 0; jb < m; jb += 32) {
        const int j = jb + lane;
        double dv = KeyOps<double>::max_key();
        int jj = INT_MAX;
        if (j < m && j != i) {
          dv = LeafRowAccess<TX>::dist(xi, rowp(j), a.d);
          jj = j;
        }
        topk_merge_chunk(bk, bi, dv, jj, k_eff);
      }
    }
    const int64_t gi = off + i;
    if (lane < a.k_nn) {
      const bool v = lane < k_eff;
      if (a.pos) a.pos[gi * a.k_nn + lane] = v ? bi : -1;
      if (a.dist) a.dist[gi * a.k_nn + lane] = v ? bk : KeyOps<double>::max_key();
      if (a.adj && v) {
        const int32_t node = a.nodes[gi];
        a.adj[(int64_t)node * a.k + lane] = a.nodes[off + bi];
        a.nnd[(int64_t)node * a.k_nn + lane] = bk;
      }
    }
    if (a.dnn1 && lane == 0) a.dnn1[a.nodes[gi]] = k_eff > 0 ? bk : KeyOps<double>::max_key();
  }
}

}  // namespace ggnn

using namespace ggnn;

extern "C" {

int ggnn_leaf_knn(const ggnn_vectors* X, const int32_t* d_nodes, const int32_t* d_rows, const int64_t* d_offsets,
                  int64_t nbatches, int64_t max_batch, int32_t k_nn, int32_t* d_pos, double* d_dist, int32_t* d_adj,
                  int32_t k, double* d_nnd, double* d_dnn1, int32_t* d_reduced, void* stream) {
  GGNN_CHECK_ARG(X && X->d_data && d_nodes && d_offsets && nbatches >= 0, "invalid arguments");
  GGNN_CHECK_ARG(k_nn >= 1 && k_nn <= 32, "k_nn must be in [1, 32] on the GPU path");
  GGNN_CHECK_ARG(!d_adj || (d_nnd && d_dnn1 && k >= k_nn && k <= MAX_K), "layer outputs need nn_dists and d_nn1");
  if (nbatches == 0) return GGNN_OK;
  LeafArgs a;
  memset(&a, 0, sizeof(a));
  a.X = X->d_data;
  a.d = X->d;
  a.nodes = d_nodes;
  a.rows = d_rows;
  a.offsets = d_offsets;
  a.k_nn = k_nn;
  a.pos = d_pos;
  a.dist = d_dist;
  a.adj = d_adj;
  a.k = k;
  a.nnd = d_nnd;
  a.dnn1 = d_dnn1;
  a.reduced = d_reduced;
  const size_t esz = X->dtype == GGNN_U8 ? 1 : 4;
  const size_t pad = X->dtype == GGNN_U8 ? 4 : 1;
  size_t want = (size_t)max_batch * (size_t)(X->d + pad) * esz;
  DevInfo di = dev_info();
  size_t cap = std::min<size_t>((size_t)di.smem_optin, 160 * 1024);
  size_t smem = want <= cap ? want : 0;
  a.smem_limit = smem;
  cudaStream_t st = as_stream(stream);
  if (X->dtype == GGNN_U8) {
    GGNN_CUDA_TRY(cudaFuncSetAttribute(leaf_knn_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    leaf_knn_kernel<uint8_t><<<(unsigned)nbatches, 256, smem, st>>>(a);
  } else {
    GGNN_CUDA_TRY(cudaFuncSetAttribute(leaf_knn_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    leaf_knn_kernel<float><<<(unsigned)nbatches, 256, smem, st>>>(a);
  }
  GGNN_LAUNCH_CHECK();
  return GGNN_OK;
}

}  // extern "C"
