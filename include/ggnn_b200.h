/*
 * ggnn_b200.h -- C ABI of libggnn_b200.so, the B200 (sm_100a) GGNN hot path.
 *
 * This is the drop-in boundary for the reference's kernel seam: the module
 * object `graphann.backend.impl` (/root/reference/pkg/src/graphann/backend.py:17-29)
 * whose functions are defined in _core.pyx.  The reference crosses that seam
 * once per query / per (x, z) pair; these entry points are batch-granular
 * (one launch per batch) and otherwise keep the reference's argument meaning.
 * INTEGRATION.md shows the ctypes binding a graphann maintainer would add.
 *
 * Conventions
 *  - Every pointer argument named d_* is DEVICE memory; h_* is host memory.
 *  - All calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) unless the name ends in _host (those synchronize).
 *  - Return 0 on success or a negative GGNN_E* code; ggnn_last_error()
 *    returns a thread-local message for the last failure.
 *  - ids are int32; distances are returned as float64 (the reference's dtype),
 *    computed exactly for uint8 data and in FP64 for float data.
 *  - Vector dtype: GGNN_F32 (float32 rows) or GGNN_U8 (uint8 rows, the
 *    lossless device copy of integer-valued data in [0, 255]).
 */
#ifndef GGNN_B200_H
#define GGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GGNN_OK 0
#define GGNN_E_INVALID (-1) /* bad argument (reference: ValueError)           */
#define GGNN_E_CUDA (-2)    /* CUDA runtime / launch failure                    */
#define GGNN_E_UNSUPPORTED (-3)
#define GGNN_E_NOMEM (-4)

#define GGNN_F32 0
#define GGNN_U8 1

/* search flags */
#define GGNN_FLAG_DISTINCT 1    /* exact distinct_touched (diagnostic; needs workspace) */
#define GGNN_FLAG_EXACT_DISTS 2 /* re-score returned hits with the sequential FP64 sum  */
#define GGNN_FLAG_UNIQUE_ROWS 4 /* caller asserts (ggnn_rows_unique) that no adjacency row of the
                                   searched layer repeats a neighbour: the per-step duplicate
                                   filter (_core.pyx:268-272) is skipped */

/* Termination codes, _core.pyx:21-23 */
#define GGNN_TERM_STOPPING 0
#define GGNN_TERM_QUEUE_EMPTY 1
#define GGNN_TERM_ITERATION_CAP 2

/* A dense (n, d) vector table. */
typedef struct ggnn_vectors {
    const void *d_data;
    int64_t n;
    int32_t d;
    int32_t dtype; /* GGNN_F32 | GGNN_U8 */
} ggnn_vectors;

/* Query rows: either their own table (d_data, dtype) or, when d_rows is not
 * NULL, rows d_rows[i] of the base table (build-time self queries). */
typedef struct ggnn_queries {
    const void *d_data;
    const int32_t *d_rows;
    int64_t m;
    int32_t dtype;
    int32_t pad_;
} ggnn_queries;

/* One graph layer (graph.py:37-199 AdjacencyLayer) in device layout:
 * adjacency is "sanitized" (see ggnn_sanitize_layer), to_row maps layer-local
 * ids to base rows (NULL = identity, the bottom layer), down maps local ids to
 * local ids of the next finer layer (NULL for the bottom), slack is the
 * layer's d_nn1_max bound used by the stopping rule. */
typedef struct ggnn_layer {
    const int32_t *d_adj;
    const int32_t *d_to_row;
    const int32_t *d_down;
    int64_t node_count;
    int32_t k;
    int32_t k_nn;
    double slack;
} ggnn_layer;

/* QueryConfig (config.py:56-78) plus flags. */
typedef struct ggnn_search_params {
    int32_t k_out;
    int32_t prioq_size;
    int32_t visited_size;
    int32_t flags;
    double tau;
    int64_t max_iterations;
} ggnn_search_params;

const char *ggnn_last_error(void);
int ggnn_version(void);
/* Device properties used for sizing (SM count, smem per block). */
int ggnn_device_info(int *sm_count, int *smem_per_block);

/* Bytes of device workspace a search batch needs for the given flags.  With
 * GGNN_FLAG_DISTINCT the default is a compact per-query set: a query that
 * touches more ids than it holds reports distinct_touched = -1 and is rerun
 * by the caller with the exact size, which max_seeds < 0 returns (a workspace
 * that large always gets exact tables). */
size_t ggnn_search_workspace_bytes(int64_t m, const ggnn_search_params *p, int32_t max_seeds);

/* Replaces: AdjacencyLayer storage semantics read by _greedy_core
 * (_core.pyx:259-264): writes d_out (node_count, k) where slot j keeps
 * d_adj[j] iff (j < k_nn and d_adj[j] >= 0) or (k_nn <= j < k_nn + sym_count),
 * else -1. */
int ggnn_sanitize_layer(const int32_t *d_adj, const int32_t *d_sym_count, int64_t node_count, int32_t k,
                        int32_t k_nn, int32_t *d_out, void *stream);

/* *d_result = 1 if no row of the (sanitized) adjacency holds the same
 * neighbour twice, else 0 (for GGNN_FLAG_UNIQUE_ROWS). */
int ggnn_rows_unique(const int32_t *d_adj, int64_t node_count, int32_t k, int32_t *d_result, void *stream);

/* Replaces: search.query (search.py:115-137) = top_layer_seeds
 * (search.py:100-112, exhaustive_topk _core.pyx:86-104 over the top layer)
 * followed by greedy_search on the bottom layer (_core.pyx:314-353).
 * Outputs: d_ids / d_dists (m, k_out) -1 / +inf padded; d_counters (m, 5)
 * int32 = [visited_count, steps, term, distinct_touched, forgotten] with the
 * query() adjustments of search.py:134-136 applied.  distinct_touched is exact
 * only with GGNN_FLAG_DISTINCT. */
int ggnn_query_batch(const ggnn_vectors *X, const ggnn_layer *bottom, const int32_t *d_top_rows, int64_t ntop,
                     const ggnn_queries *Q, const ggnn_search_params *p, double d_nn1_max, int32_t *d_ids,
                     double *d_dists, int32_t *d_counters, void *d_workspace, size_t workspace_bytes,
                     void *stream);

/* Scheduling of the query batch launches (ggnn_query_batch and the staged /
 * host variants; no reference counterpart -- results never depend on it):
 * a batch of at least min_waves waves of resident searches first runs every
 * search for pilot_steps expansions, parks the open ones and resumes them
 * longest-predicted first (a second round up to GGNN_PILOT2 = 32 expansions
 * re-parks them with a sharper prediction).  pilot_steps < 0 restores the
 * default (GGNN_PILOT, else 8), 0 disables; min_waves defaults to 1.5.
 * Process-wide. */
int ggnn_query_schedule(long long pilot_steps, double min_waves);

/* Large batches (no reference counterpart -- results never depend on it):
 * uint8 batches of at least large_waves waves of resident searches (default
 * 3.5) are throughput-bound, so their second round runs up to
 * GGNN_PILOT2_LARGE = 40 expansions and their last round uses a kernel
 * compiled for 32 CTAs per SM.  large_waves <= 0 disables.  Process-wide. */
int ggnn_query_schedule_large(double large_waves);

/* Number of kernels this library has launched in this process (all entry
 * points; no reference counterpart): the bench reads it around its timed
 * region to report gpu_launches. */
unsigned long long ggnn_kernel_launches(void);

/* Replaces: query (search.py:115-137) for a batch, like ggnn_query_batch,
 * over float32 queries that are still being uploaded (the
 * host-to-host path overlaps the upload with the search): rows
 * [c * chunk_rows, (c + 1) * chunk_rows) of d_q_f32 may be read once
 * d_chunk_flags[c] == epoch, which the caller's copy stream writes after the
 * rows; d_chunk_flags == NULL means every row is already readable (e.g. the
 * device address of pinned host memory).  narrow != 0 (uint8 tables): rows are narrowed to uint8 on load and a
 * value that is not an integer in [0, 255] sets bit 0 of *d_status; a chunk
 * that does not arrive within ~50 ms sets bit 1.  Either bit voids the
 * results (the caller reruns).  distinct_touched is not tracked. */
int ggnn_query_batch_staged(const ggnn_vectors *X, const ggnn_layer *bottom, const int32_t *d_top_rows, int64_t ntop,
                            const float *d_q_f32, int64_t m, const ggnn_search_params *p, double d_nn1_max,
                            const uint32_t *d_chunk_flags, int64_t chunk_rows, uint32_t epoch, int32_t narrow,
                            int32_t *d_ids, double *d_dists, int32_t *d_counters, int32_t *d_status, void *stream);

/* Replaces: batch_query (search.py:213-226) called with host arrays, as one
 * asynchronous native call.  The whole host-to-host query: host float32 queries h_q
 * (pinned for a true async upload) go to d_q_stage in nchunks chunks on
 * copy_stream, each followed by its flag (the epoch, read from pinned
 * *h_epoch), all queued before ggnn_query_batch_staged is launched on
 * search_stream (which then overlaps the chunks still in flight); the
 * results (and status, see above) are copied back into the pinned h_*
 * buffers on search_stream.  When h_q and h_ids / h_dists / h_counters are
 * all page-locked, the search instead reads the rows and writes the results
 * through their mapped device addresses (zero copy; GGNN_ZERO_COPY=0 turns it
 * off) and d_q_stage / d_chunk_flags are unused.  Asynchronous: the caller synchronises both
 * streams, checks *h_status == 0, and must not change *h_epoch or reuse the
 * staging buffers before that. */
int ggnn_query_batch_host(const ggnn_vectors *X, const ggnn_layer *bottom, const int32_t *d_top_rows, int64_t ntop,
                          const float *h_q, int64_t m, const ggnn_search_params *p, double d_nn1_max, float *d_q_stage,
                          uint32_t *d_chunk_flags, const uint32_t *h_epoch, int32_t nchunks, int32_t narrow,
                          int32_t *d_ids, double *d_dists, int32_t *d_counters, int32_t *d_status, int32_t *h_ids,
                          double *h_dists, int32_t *h_counters, int32_t *h_status, void *search_stream,
                          void *copy_stream);

/* Replaces: greedy_search (_core.pyx:314-353) for a batch of queries with
 * explicit seeds d_seed_ids / d_seed_dists (m, nseeds; -1 ids skipped). */
int ggnn_greedy_batch(const ggnn_vectors *X, const ggnn_layer *layer, const ggnn_queries *Q,
                      const int32_t *d_seed_ids, const double *d_seed_dists, int32_t nseeds,
                      const ggnn_search_params *p, double d_nn1_max, int32_t *d_ids, double *d_dists,
                      int32_t *d_counters, void *d_workspace, size_t workspace_bytes, void *stream);

/* Replaces: hierarchical_query (search.py:140-210): brute-force the segment
 * [d_seg_lo[i], d_seg_hi[i]) of layer `start` (NULL = whole layer), then
 * descend layer by layer to `stop`, each layer's greedy search seeded with the
 * previous layer's k_out hits.  layers[] is indexed by layer number and each
 * layer's `slack` is its d_nn1_max bound.  Output ids are stop-layer local. */
int ggnn_descent_batch(const ggnn_vectors *X, const ggnn_layer *layers, int32_t num_layers, int32_t start,
                       int32_t stop, const ggnn_queries *Q, const int32_t *d_seg_lo, const int32_t *d_seg_hi,
                       const ggnn_search_params *p, int32_t *d_ids, double *d_dists, int32_t *d_counters,
                       void *d_workspace, size_t workspace_bytes, void *stream);

/* Replaces: sym_check_pair (_core.pyx:375-435) for a batch of (x, z, d_xz)
 * checks on one layer.  d_verdict[i] in {0, 1, 2}; d_fallback (npairs,
 * n_fallback) -1 padded, filled for verdict 2. */
int ggnn_sym_check_batch(const ggnn_vectors *X, const ggnn_layer *layer, const int32_t *d_x, const int32_t *d_z,
                         const double *d_dxz, int64_t npairs, double tau, double d_nn1_max, int32_t budget,
                         int32_t k_out, int32_t prioq_size, int32_t visited_size, int32_t n_fallback,
                         int32_t *d_verdict, int32_t *d_fallback, void *stream);

/* Replaces: exhaustive_topk (_core.pyx:86-104), batched over queries, over
 * rows d_rows[0..nrows) of X (NULL = all rows), any k >= 1; ties by row
 * index; distances are the reference's sequential FP64 _sqdist values.
 * Whole-table scans of at least 4096 rows run on the tensor cores: uint8
 * tables as exact kind::i8, float tables (d % 8 == 0, k <= 32) as 3xTF32
 * with a rigorous error bound and an exact re-score of every candidate.
 * The float tensor-core path synchronizes the stream once (to send the rare
 * query whose candidate list may be cut to the CUDA-core scan). */
int ggnn_exhaustive_topk(const ggnn_vectors *X, const int32_t *d_rows, int64_t nrows, const ggnn_queries *Q,
                         int32_t k, int32_t *d_ids, double *d_dists, void *stream);

/* Same contract as ggnn_exhaustive_topk over the whole table, forced onto the
 * tcgen05 path (kind::i8 MMA of 128-query tiles against streamed 256-row
 * tiles, exact integer distances, top-k epilogue from TMEM); GGNN_E_INVALID
 * unless X and Q are uint8, d % 32 == 0, and 1 <= k <= 32 with d <= 224 or
 * 32 < k <= 128 with d <= 128.  ggnn_exhaustive_topk takes this path by
 * itself for such whole-table scans of at least 4096 rows (and is limited to
 * k <= 32 otherwise). */
int ggnn_exhaustive_topk_tc(const ggnn_vectors *X, const ggnn_queries *Q, int32_t k, int32_t *d_ids,
                            double *d_dists, void *stream);

/* Tensor-core brute-force tiles whose MMA wait timed out since load (0 when healthy). */
int ggnn_bf_timeouts(void);

/* Replaces: squared_l2_many (_core.pyx:47-55): exact sequential FP64
 * distances of query i to rows d_rows[i*per_query + j]. */
int ggnn_squared_l2_many(const ggnn_vectors *X, const ggnn_queries *Q, const int32_t *d_rows, int32_t per_query,
                         double *d_out, void *stream);

/* Replaces: the integrality check implied by the uint8 device copy: sets
 * *d_flag = 1 iff every value of the float table is an integer in [0, 255]
 * (d_flag must be pre-set to 1), and writes the uint8 copy to d_u8 if not NULL. */
int ggnn_f32_to_u8(const float *d_src, int64_t count, uint8_t *d_u8, int32_t *d_flag, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GGNN_B200_H */
