// ggnn_bf_tf32.cu -- exact brute-force top-k for FLOAT tables on the tcgen05
// tensor cores: the reference's exhaustive_topk (_core.pyx:86-104) as used by
// brute_force_oracle (evaluate.py:32-57), whole query batches at once.
//
// Rows and queries are centred on the table's column mean mu (x' = fl(x - mu))
// and split x' = hi + lo into tf32 halves; D = Q' X'^T runs as 3xTF32
// (hi.hi + hi.lo + lo.hi, tcgen05.mma kind::tf32, F32 accumulators in TMEM)
// over 128-query x 128-row tiles, K staged in chunks of 32 elements.  From D
// each query keeps the TF_L smallest APPROXIMATE distances
//   a_qx = |q'|^2 + |x'|^2 - 2 D_qx        (FP64 from the FP64 norms)
// per X split.  With beta_q = (8 d 2^-23 + 2^-18)(|q'| + max_x |x'|)^2 a
// rigorous bound on |a_qx - r_qx| (r = the reference's sequential FP64
// _sqdist; see leaf_knn_tf32_kernel for the derivation), every x with
// a_qx <= A_k + 2 beta_q (A_k: the query's k-th smallest a) is re-scored with
// the sequential FP64 sum and the top-k is taken by (r, row) -- bit for bit
// the reference's answer.  Any x outside the candidates has
// r > A_k + beta_q >= r of k candidates, so it cannot belong.  A query whose
// kept lists might have cut a candidate (a full list whose last key is <= the
// limit) is answered by the CUDA-core scan instead.
#include <algorithm>
#include <climits>
#include <cstring>

#include "ggnn_b200.h"
#include "ggnn_capi_util.cuh"
#include "ggnn_search.cuh"
#include "ggnn_tc.cuh"

namespace ggnn {

// this translation unit's MMA-wait timeouts (device symbols are per unit
// without -rdc); ggnn_bf_timeouts() adds them to the uint8 kernel's
__device__ int g_bf32_timeouts = 0;

int bf_tf32_timeouts() {
  int v = 0;
  if (cudaMemcpyFromSymbol(&v, g_bf32_timeouts, sizeof(int)) != cudaSuccess) return -1;
  return v;
}

namespace {

constexpr int TB_M = 128;   // queries per CTA (TMEM lanes)
constexpr int TB_N = 128;   // table rows per tile (accumulator columns)
constexpr int TB_KC = 32;   // tf32 elements per staged K chunk
constexpr int TF_L = 48;    // approximate candidates kept per (query, split)
constexpr int TB_KMAX = 32; // k served by this path

struct Tf32Args {
  const float* X;
  int64_t n;
  int d;
  const float* Q;
  const int32_t* qrows;
  int64_t m;
  const float* mu;
  const double* xn;       // |x'|^2 per row
  int64_t tiles, tiles_per_split;
  int splits;
  double* lk;             // (m, splits, TF_L) approximate keys
  int32_t* li;            // (m, splits, TF_L) rows
};

inline size_t tf32_smem() {
  return 4 * (size_t)TB_M * TB_KC * 4                  // A hi / lo, B hi / lo chunks
         + (size_t)TB_M * 8                            // query norms
         + (size_t)TB_M * TF_L * 12 + 64;              // per-query lists + barrier
}

__global__ void col_sum_kernel(const float* X, int64_t n, int d, double* sums) {
  // each block: a contiguous row range; each thread: columns tid, tid + 256, ...
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(n, r0 + per);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    double s = 0.0;
    for (int64_t r = r0; r < r1; ++r) s += (double)__ldg(X + r * d + e);
    atomicAdd(sums + e, s);
  }
}

__global__ void mean_kernel(const double* sums, int64_t n, int d, float* mu) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < d) mu[e] = (float)(sums[e] / (double)n);
}

// |fl(x - mu)|^2 in FP64 per row, and the largest one (as ordered bits)
__global__ void row_norm_kernel(const float* X, int64_t n, int d, const float* mu, double* xn,
                                unsigned long long* xmax) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  const int lane = lane_id();
  double s = 0.0;
  for (int e = lane; e < d; e += 32) {
    const float v = __ldg(X + r * d + e) - mu[e];
    s += (double)v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if (lane == 0) {
    xn[r] = s;
    atomicMax(xmax, (unsigned long long)__double_as_longlong(s));
  }
}

// stage `rows` rows (thread t: row t) of a K chunk, centred and split
__device__ __forceinline__ void stage_chunk(const float* src, bool valid, const float* mu, int c0, int kc, float* hi,
                                            float* lo, double* norm) {
  const int t = threadIdx.x;
#pragma unroll
  for (int e = 0; e < TB_KC; e += 4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid && e < kc) {
      v = __ldg(reinterpret_cast<const float4*>(src + c0 + e));
      v.x -= __ldg(mu + c0 + e);
      v.y -= __ldg(mu + c0 + e + 1);
      v.z -= __ldg(mu + c0 + e + 2);
      v.w -= __ldg(mu + c0 + e + 3);
      if (norm) *norm += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
    float4 h, l;
    h.x = tc::to_tf32(v.x);
    h.y = tc::to_tf32(v.y);
    h.z = tc::to_tf32(v.z);
    h.w = tc::to_tf32(v.w);
    l.x = tc::to_tf32(v.x - h.x);
    l.y = tc::to_tf32(v.y - h.y);
    l.z = tc::to_tf32(v.z - h.z);
    l.w = tc::to_tf32(v.w - h.w);
    const uint32_t o = tc::il_offset(t, e * 4, TB_KC * 4);
    *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(hi) + o) = h;
    *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(lo) + o) = l;
  }
}

__global__ void __launch_bounds__(128, 1) bf_tf32_kernel(const __grid_constant__ Tf32Args a) {
  extern __shared__ __align__(16) uint8_t smem_t[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t qt = blockIdx.x / a.splits, sp = blockIdx.x % a.splits;
  const int64_t q0 = qt * TB_M;
  const int64_t t_begin = sp * a.tiles_per_split;
  const int64_t t_end = min(a.tiles, t_begin + a.tiles_per_split);
  float* Ah = reinterpret_cast<float*>(smem_t);
  float* Al = Ah + TB_M * TB_KC;
  float* Bh = Al + TB_M * TB_KC;
  float* Bl = Bh + TB_N * TB_KC;
  double* qn = reinterpret_cast<double*>(Bl + TB_N * TB_KC);
  double* lk = qn + TB_M;
  int32_t* li = reinterpret_cast<int32_t*>(lk + TB_M * TF_L);
  uint64_t* mbar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(li + TB_M * TF_L) + 15) & ~uintptr_t(15));
  uint32_t* taddr = reinterpret_cast<uint32_t*>(mbar + 1);
  if (warp == 0) tc::tmem_alloc<128>(taddr);
  if (tid == 0) tc::mbar_init(mbar, 1);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *taddr;
  const int64_t qi = q0 + tid;
  const bool qvalid = qi < a.m;
  const float* qsrc = qvalid ? (a.qrows ? a.X + (int64_t)__ldg(a.qrows + qi) * a.d : a.Q + qi * a.d) : a.X;
  double* mk = lk + tid * TF_L;
  int32_t* mi = li + tid * TF_L;
  for (int j = 0; j < TF_L; ++j) {
    mk[j] = KeyOps<double>::max_key();
    mi[j] = -1;
  }
  double qnorm = 0.0;
  const uint32_t idesc = tc::idesc_tf32(TB_M, TB_N);
  const uint32_t sbo = (uint32_t)(TB_KC * 4 / 16) * 128u;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  uint32_t phase = 0;
  bool ok = true;
  for (int64_t t = t_begin; t < t_end; ++t) {
    const int64_t r0 = t * TB_N;
    const bool xvalid = r0 + tid < a.n;
    const float* xsrc = a.X + (xvalid ? r0 + tid : 0) * a.d;
    for (int c0 = 0; c0 < a.d; c0 += TB_KC) {
      const int kc = min(TB_KC, a.d - c0);  // a multiple of 8
      stage_chunk(qsrc, qvalid, a.mu, c0, kc, Ah, Al, t == t_begin ? &qnorm : nullptr);
      stage_chunk(xsrc, xvalid, a.mu, c0, kc, Bh, Bl, nullptr);
      tc::fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t ah = tc::smem_u32(Ah), al = tc::smem_u32(Al), bh = tc::smem_u32(Bh), bl = tc::smem_u32(Bl);
        for (int s = 0; s < (kc >> 3); ++s) {
          const uint32_t so = (uint32_t)s * 256u;
          const uint64_t dah = tc::smem_desc(ah + so, 128u, sbo), dal = tc::smem_desc(al + so, 128u, sbo);
          const uint64_t dbh = tc::smem_desc(bh + so, 128u, sbo), dbl = tc::smem_desc(bl + so, 128u, sbo);
          tc::mma_tf32(tmem, dah, dbh, idesc, (c0 > 0 || s > 0) ? 1u : 0u);
          tc::mma_tf32(tmem, dah, dbl, idesc, 1u);
          tc::mma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        tc::commit(mbar);
      }
      __syncwarp();
      ok &= tc::mbar_wait(mbar, phase);
      phase ^= 1u;
      tc::fence_after_sync();
      __syncthreads();  // chunk buffers free
    }
    if (t == t_begin) qn[tid] = qnorm;
    // epilogue: this query's approximate distances to the tile's rows
    for (int c = 0; c < TB_N; c += 16) {
      uint32_t v[16];
      tc::tmem_ld16(tmem + lane_base + (uint32_t)c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t row = r0 + c + j;
        if (qvalid && row < a.n) {
          const double ap = qnorm + __ldg(a.xn + row) - 2.0 * (double)__uint_as_float(v[j]);
          if (ap < mk[TF_L - 1] || (ap == mk[TF_L - 1] && row < mi[TF_L - 1])) {
            int p = TF_L - 1;
            while (p > 0 && (mk[p - 1] > ap || (mk[p - 1] == ap && mi[p - 1] > row))) {
              mk[p] = mk[p - 1];
              mi[p] = mi[p - 1];
              --p;
            }
            mk[p] = ap;
            mi[p] = (int32_t)row;
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();  // TMEM reads done before the next tile's MMA
    tc::fence_after_sync();
  }
  if (!ok && lane == 0) atomicAdd(&g_bf32_timeouts, 1);
  if (qvalid) {
    double* ok_ = a.lk + ((size_t)qi * a.splits + sp) * TF_L;
    int32_t* oi = a.li + ((size_t)qi * a.splits + sp) * TF_L;
    for (int j = 0; j < TF_L; ++j) {
      ok_[j] = mk[j];
      oi[j] = mi[j];
    }
  }
  if (warp == 0) tc::tmem_free<128>(tmem);
}

// One warp per query: the k-th approximate key over all splits' lists, the
// candidate limit, sequential FP64 re-score of the candidates, top-k by
// (distance, row).  flag[q] = 1 when a list may have cut a candidate.
__global__ void __launch_bounds__(256) bf_tf32_finalize(const Tf32Args a, const float* Qf, const double* qn_all,
                                                       const unsigned long long* xmax_bits, int k, int32_t* out_ids,
                                                       double* out_d, int32_t* flag, int32_t* nflag) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= a.m) return;
  const int lane = lane_id();
  using KO = KeyOps<double>;
  const double* lk = a.lk + (size_t)q * a.splits * TF_L;
  const int32_t* li = a.li + (size_t)q * a.splits * TF_L;
  const int total = a.splits * TF_L;
  // k-th smallest approximate key
  double bk = KO::max_key();
  int bi = INT_MAX;
  for (int base = 0; base < total; base += 32) {
    const int e = base + lane;
    double ck = KO::max_key();
    int cx = INT_MAX;
    if (e < total && li[e] >= 0) {
      ck = lk[e];
      cx = li[e];
    }
    topk_merge_chunk(bk, bi, ck, cx, k);
  }
  const double ak = KO::shfl(bk, k - 1);
  const double qn = qn_all[q];
  const double nrm = sqrt(qn) + sqrt(__longlong_as_double((long long)*xmax_bits));
  const double lim = ak + 2.0 * (8.0 * a.d * 0x1p-23 + 0x1p-18) * nrm * nrm;
  // a full split list whose last key is within the limit may have dropped one
  bool unsafe = false;
  for (int s = lane; s < a.splits; s += 32)
    unsafe |= li[(size_t)s * TF_L + TF_L - 1] >= 0 && lk[(size_t)s * TF_L + TF_L - 1] <= lim;
  if (__any_sync(FULL, unsafe)) {
    if (lane == 0) {
      flag[q] = 1;
      atomicAdd(nflag, 1);
    }
    return;
  }
  const float* qv = a.qrows ? a.X + (int64_t)__ldg(a.qrows + q) * a.d : Qf + q * a.d;
  bk = KO::max_key();
  bi = INT_MAX;
  for (int base = 0; base < total; base += 32) {
    const int e = base + lane;
    double ck = KO::max_key();
    int cx = INT_MAX;
    if (e < total && li[e] >= 0 && lk[e] <= lim) {
      cx = li[e];
      ck = seq_sqdist<float, float>(a.X + (int64_t)cx * a.d, qv, a.d);
    }
    topk_merge_chunk(bk, bi, ck, cx, k);
  }
  if (lane < k) {
    const bool v = bi != INT_MAX;
    out_ids[q * k + lane] = v ? bi : -1;
    out_d[q * k + lane] = v ? bk : KO::max_key();
  }
  if (lane == 0) flag[q] = 0;
}

__global__ void query_norm_kernel(const float* X, const float* Q, const int32_t* qrows, int64_t m, int d,
                                  const float* mu, double* qn) {
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= m) return;
  const float* src = qrows ? X + (int64_t)qrows[q] * d : Q + q * d;
  double s = 0.0;
  for (int e = lane_id(); e < d; e += 32) {
    const float v = __ldg(src + e) - mu[e];
    s += (double)v * v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  if (lane_id() == 0) qn[q] = s;
}

__global__ void gather_rows_kernel(const float* X, const float* Q, const int32_t* qrows, const int32_t* sel, int64_t cnt,
                                   int d, float* out) {
  const int64_t i = blockIdx.x;
  if (i >= cnt) return;
  const int64_t q = sel[i];
  const float* src = qrows ? X + (int64_t)qrows[q] * d : Q + q * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) out[i * d + e] = src[e];
}

__global__ void scatter_rows_kernel(const int32_t* sel, int64_t cnt, int k, const int32_t* ids, const double* dists,
                                    int32_t* out_ids, double* out_d) {
  const int64_t i = blockIdx.x;
  if (i >= cnt) return;
  const int64_t q = sel[i];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    out_ids[q * k + j] = ids[i * k + j];
    out_d[q * k + j] = dists[i * k + j];
  }
}

__global__ void flagged_kernel(const int32_t* flag, int64_t m, int32_t* sel, int32_t* cnt) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < m && flag[q]) sel[atomicAdd(cnt, 1)] = (int32_t)q;
}

}  // namespace

bool bf_tf32_eligible(const ggnn_vectors* X, const int32_t* d_rows, const ggnn_queries* Q, int k) {
  const int qd = Q->d_rows ? X->dtype : Q->dtype;
  return X->dtype == GGNN_F32 && qd == GGNN_F32 && d_rows == nullptr && k >= 1 && k <= TB_KMAX && X->d % 8 == 0 &&
         X->n >= 4096 && X->n < INT32_MAX && (reinterpret_cast<uintptr_t>(X->d_data) & 15) == 0 &&
         (Q->d_rows || (reinterpret_cast<uintptr_t>(Q->d_data) & 15) == 0);
}

// the CUDA-core scan of queries `sel` (ggnn_exhaustive_topk's warp path)
int topk_scan_subset(const ggnn_vectors* X, const float* Qsub, int64_t cnt, int k, int32_t* ids, double* dists,
                     cudaStream_t st);

int bf_topk_tf32(const ggnn_vectors* X, const ggnn_queries* Q, int k, int32_t* d_ids, double* d_dists,
                 cudaStream_t st) {
  const int64_t m = Q->m, n = X->n;
  const int d = (int)X->d;
  if (m == 0) return GGNN_OK;
  DevInfo di = dev_info();
  const float* Xd = static_cast<const float*>(X->d_data);
  const int64_t qtiles = (m + TB_M - 1) / TB_M;
  const int64_t tiles = (n + TB_N - 1) / TB_N;
  int64_t splits = std::max<int64_t>(1, (2 * (int64_t)std::max(di.sm_count, 1) + qtiles - 1) / qtiles);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, tiles / 4));
  const int64_t per = (tiles + splits - 1) / splits;
  splits = (tiles + per - 1) / per;
  // scratch: column sums, mean, row / query norms, max, lists, flags
  const size_t lists = (size_t)m * splits * TF_L;
  size_t bytes = (size_t)d * 8 + (size_t)d * 4 + (size_t)n * 8 + (size_t)m * 8 + 64 + lists * 12 + (size_t)m * 8 + 64;
  uint8_t* buf = nullptr;
  GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st));
  double* sums = reinterpret_cast<double*>(buf);
  float* mu = reinterpret_cast<float*>(sums + d);
  double* xn = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(buf) + (((size_t)d * 12 + 15) & ~size_t(15)));
  double* qn = xn + n;
  unsigned long long* xmax = reinterpret_cast<unsigned long long*>(qn + m);
  int32_t* nflag = reinterpret_cast<int32_t*>(xmax + 1);
  double* lk = reinterpret_cast<double*>(xmax + 8);
  int32_t* li = reinterpret_cast<int32_t*>(lk + lists);
  int32_t* flag = li + lists;
  int32_t* sel = flag + m;
  GGNN_CUDA_TRY(cudaMemsetAsync(sums, 0, (size_t)d * 8, st));
  GGNN_CUDA_TRY(cudaMemsetAsync(xmax, 0, 64, st));
  col_sum_kernel<<<(unsigned)std::min<int64_t>(std::max(di.sm_count, 1) * 8, std::max<int64_t>(1, n / 64)), 256, 0,
                   st>>>(Xd, n, d, sums);
  count_launch();
  mean_kernel<<<(d + 255) / 256, 256, 0, st>>>(sums, n, d, mu);
  count_launch();
  row_norm_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(Xd, n, d, mu, xn, xmax);
  count_launch();
  const float* Qf = static_cast<const float*>(Q->d_data);
  query_norm_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(Xd, Qf, Q->d_rows, m, d, mu, qn);
  count_launch();
  GGNN_LAUNCH_CHECK();
  Tf32Args a;
  a.X = Xd;
  a.n = n;
  a.d = d;
  a.Q = Qf;
  a.qrows = Q->d_rows;
  a.m = m;
  a.mu = mu;
  a.xn = xn;
  a.tiles = tiles;
  a.tiles_per_split = per;
  a.splits = (int)splits;
  a.lk = lk;
  a.li = li;
  const size_t smem = tf32_smem();
  GGNN_CUDA_TRY(cudaFuncSetAttribute(bf_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  bf_tf32_kernel<<<(unsigned)(qtiles * splits), TB_M, smem, st>>>(a);
  count_launch();
  GGNN_LAUNCH_CHECK();
  bf_tf32_finalize<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(a, Qf, qn, xmax, k, d_ids, d_dists, flag, nflag);
  count_launch();
  GGNN_LAUNCH_CHECK();
  // the one host synchronisation of this path: how many queries need the
  // CUDA-core scan (almost always none)
  int32_t nf = 0;
  GGNN_CUDA_TRY(cudaMemcpyAsync(&nf, nflag, 4, cudaMemcpyDeviceToHost, st));
  GGNN_CUDA_TRY(cudaStreamSynchronize(st));
  int rc = GGNN_OK;
  if (nf > 0) {  // the few queries whose candidate lists may be cut: CUDA-core scan
    GGNN_CUDA_TRY(cudaMemsetAsync(nflag, 0, 4, st));
    flagged_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(flag, m, sel, nflag);
    count_launch();
    float* qsub = nullptr;
    int32_t* ids2 = nullptr;
    double* d2 = nullptr;
    GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&qsub), (size_t)nf * d * 4, st));
    GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&ids2), (size_t)nf * k * 4, st));
    GGNN_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d2), (size_t)nf * k * 8, st));
    gather_rows_kernel<<<(unsigned)nf, 128, 0, st>>>(Xd, Qf, Q->d_rows, sel, nf, d, qsub);
    count_launch();
    rc = topk_scan_subset(X, qsub, nf, k, ids2, d2, st);
    if (rc == GGNN_OK) {
      scatter_rows_kernel<<<(unsigned)nf, 32, 0, st>>>(sel, nf, k, ids2, d2, d_ids, d_dists);
      count_launch();
    }
    cudaFreeAsync(qsub, st);
    cudaFreeAsync(ids2, st);
    cudaFreeAsync(d2, st);
  }
  cudaFreeAsync(buf, st);
  GGNN_LAUNCH_CHECK();
  return rc;
}

}  // namespace ggnn
