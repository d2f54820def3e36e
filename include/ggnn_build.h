/*
 * ggnn_build.h -- C ABI of the construction kernels in libggnn_b200.so.
 * Conventions as in ggnn_b200.h (device pointers d_*, async on `stream`,
 * 0 / negative GGNN_E* return codes).
 */
#ifndef GGNN_BUILD_H
#define GGNN_BUILD_H

#include "ggnn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Replaces: batch_bruteforce (_core.pyx:107-130) as driven by build_base
 * (build.py:78-94), for nbatches batches in one launch.  Batch b's members are
 * d_nodes[off_b .. off_{b+1}) (layer-local ids; d_offsets int64, nbatches+1),
 * whose vectors are rows d_rows[...] of X (NULL: rows == nodes).  max_batch is
 * the largest batch size.  Outputs (each optional):
 *   d_pos / d_dist (total, k_nn): positions within the batch (-1 padded) and
 *     squared distances (+inf padded), ties broken by position;
 *   d_adj (node_count, k) / d_nnd (node_count, k_nn) / d_dnn1 (node_count):
 *     build_base's writes (slots [0, k_eff) of each member, d_nn1 = slot 0);
 *   d_reduced: incremented once per batch with fewer than k_nn + 1 members. */
int ggnn_leaf_knn(const ggnn_vectors *X, const int32_t *d_nodes, const int32_t *d_rows, const int64_t *d_offsets,
                  int64_t nbatches, int64_t max_batch, int32_t k_nn, int32_t *d_pos, double *d_dist, int32_t *d_adj,
                  int32_t k, double *d_nnd, double *d_dnn1, int32_t *d_reduced, void *stream);

/* Same contract as ggnn_leaf_knn, forced onto the tcgen05 tensor-core path
 * (kind::i8 MMA of the staged batch against itself, exact integer distances);
 * GGNN_E_INVALID unless X is uint8 with d % 32 == 0, d <= 512 and every batch
 * has 2..128 rows.  ggnn_leaf_knn takes this path automatically when eligible. */
int ggnn_leaf_knn_tc(const ggnn_vectors *X, const int32_t *d_nodes, const int32_t *d_rows, const int64_t *d_offsets,
                     int64_t nbatches, int64_t max_batch, int32_t k_nn, int32_t *d_pos, double *d_dist,
                     int32_t *d_adj, int32_t k, double *d_nnd, double *d_dnn1, int32_t *d_reduced, void *stream);

/* Number of tensor-core tiles whose MMA completion wait timed out since the
 * library was loaded (0 in a healthy run; synchronizes). */
int ggnn_tc_timeouts(void);

/* Build accounting: while d_acc != NULL, every search launched
 * from this host thread by ggnn_merge_descent, ggnn_descent_batch,
 * ggnn_greedy_batch and the sym-check entry points adds its visited count to
 * d_acc[0] and its steps to d_acc[1] (device uint64, caller-zeroed), so the
 * algorithmic bytes of a phase are d_acc[0] * d * e + d_acc[1] * (4k + 4).
 * NULL switches it off (the default; the query kernel is never counted).
 * No reference counterpart (the reference reports no such totals). */
int ggnn_search_accounting(unsigned long long *d_acc);

/* Replaces: the per-node hierarchical_query calls of merge_layer
 * (build.py:146-197, search.py:140-210) for all m nodes of layer `stop` at
 * once.  Query i is base row d_query_rows[i]; it brute-forces the segment
 * seg = (d_seg_of ? d_seg_of[i] : i) / seg_div, i.e. rows
 * [seg * seg_size, (seg + 1) * seg_size) of layer `start`, then descends to
 * `stop` (each layer's slack = its frozen live_d_nn1_max).  Outputs are
 * stop-layer local ids / distances (m, k_out) and optional counters (m, 5). */
int ggnn_merge_descent(const ggnn_vectors *X, const ggnn_layer *layers, int32_t num_layers, int32_t start,
                       int32_t stop, const int32_t *d_query_rows, int64_t m, const int32_t *d_seg_of, int32_t seg_div,
                       int32_t seg_size, const ggnn_search_params *p, int32_t *d_ids, double *d_dists,
                       int32_t *d_counters, void *stream);

/* Replaces: AdjacencyLayer.merge_hits (graph.py:121-165) applied to every
 * node of a layer: d_hit_ids / d_hit_dists (node_count, hits_per_node) are the
 * node's descent results (its own id and -1 entries are ignored).  Rescued
 * (displaced) neighbours go to d_resc_ids / d_resc_dists (node_count, k_nn),
 * -1 padded, in their former slot order.  d_changed (optional) counts the rows
 * whose direct set changed. */
int ggnn_merge_rows(int64_t node_count, int32_t k, int32_t k_nn, int32_t *d_adj, double *d_nnd, int32_t *d_sym_count,
                    double *d_dnn1, const int32_t *d_hit_ids, const double *d_hit_dists, int32_t hits_per_node,
                    int32_t *d_resc_ids, double *d_resc_dists, int32_t *d_changed, void *stream);

/* ggnn_merge_rows for nodes node_begin .. node_begin + count - 1 only: hit
 * and rescued rows are indexed from 0 (row i belongs to node node_begin + i).
 * merge_layer applies its merges window by window with this (see build.py). */
int ggnn_merge_rows_range(int64_t node_begin, int64_t count, int32_t k, int32_t k_nn, int32_t *d_adj, double *d_nnd,
                          int32_t *d_sym_count, double *d_dnn1, const int32_t *d_hit_ids, const double *d_hit_dists,
                          int32_t hits_per_node, int32_t *d_resc_ids, double *d_resc_dists, int32_t *d_changed,
                          void *stream);

/* Replaces: the check half of symmetrize (build.py:200-266 with
 * sym_check_pair, _core.pyx:375-435) for every (x, z) of a layer: pair
 * p = x * per_node + t checks direct slot t < k_nn of x, or rescued entry
 * t - k_nn (d_resc_ids (node_count, per_node - k_nn), may be NULL).  Pairs
 * with verdict 2 are appended to d_req as {p, x, z, d_xz lo, d_xz hi,
 * fallback[n_fallback]} (int32, stride 5 + n_fallback); *d_req_count counts them (it may exceed
 * req_cap, in which case the surplus was not stored). */
int ggnn_sym_check_layer(const ggnn_vectors *X, const ggnn_layer *layer, const double *d_nnd,
                         const int32_t *d_resc_id, const double *d_resc_d, int32_t per_node, double tau,
                         double d_nn1_max, int32_t budget, int32_t k_out, int32_t prioq_size, int32_t visited_size,
                         int32_t n_fallback, int32_t *d_req, int32_t *d_req_count, int64_t req_cap, void *stream);

/* Replaces: the claim half of symmetrize (reserve_sym_slot, graph.py:167-191,
 * and the fallback loop of build.py:237-244) -- one round.  Requests are the
 * records written by ggnn_sym_check_layer ({p, x, z, d_xz lo, d_xz hi,
 * fallback[n_fallback]}); d_stage[r] >= 0 is the index of the request's
 * current target (0 = z, s = fallback s-1), < 0 settled (-1 claimed,
 * -2 dropped, -3 resolved by a re-check).  Each open request proposes to its
 * current target (skipping full targets and targets that already hold x);
 * every target accepts the proposal with the smallest pair index.
 * d_best_scratch (node_count int32) must hold INT32_MAX and d_tgt_scratch
 * (nreq int32) -1 on entry; both are restored.  *d_pending = open requests
 * after the round, *d_dropped += requests that ran out of targets.  Only
 * requests of nodes x < x_end take part (the reference visits x ascending),
 * and per x only its lowest open pair index proposes (d_first_scratch:
 * node_count int32 holding INT32_MAX, restored). */
int ggnn_sym_claim_round(const int32_t *d_req, int64_t nreq, int32_t n_fallback, int32_t *d_adj,
                         int32_t *d_sym_count, int32_t k, int32_t k_nn, int32_t *d_best_scratch, int32_t *d_stage,
                         int32_t *d_tgt_scratch, int32_t *d_dropped, int32_t *d_pending, int32_t x_end,
                         int32_t *d_first_scratch, const int32_t *d_idx, void *stream);

/* The still-open requests (d_stage[r] >= 0) among d_idx_in[0 .. n_in) (NULL:
 * requests 0 .. n_in - 1) -> d_idx_out, their count -> *d_n_out.  Rounds late
 * in a pass then touch only the requests that are still open (d_idx of
 * ggnn_sym_claim_round / ggnn_sym_recheck, nreq = the count).  No reference
 * counterpart (the reference walks its requests sequentially). */
int ggnn_sym_compact(const int32_t *d_stage, const int32_t *d_idx_in, int64_t n_in, int32_t *d_idx_out,
                     int32_t *d_n_out, void *stream);

/* Re-check of open requests on the current graph (between claim rounds):
 * for every r with d_stage[r] >= 0, re-runs the reachability search of
 * sym_check_pair (_core.pyx:375-435) for (x, z, d_xz) of record r; settles it
 * (d_stage[r] = -3) if the verdict is no longer 2, else refreshes its
 * fallbacks in place.  Requests of nodes x >= x_end are skipped. */
int ggnn_sym_recheck(const ggnn_vectors *X, const ggnn_layer *layer, int32_t *d_req, int64_t nreq, int32_t *d_stage,
                     int32_t x_end, double tau, double d_nn1_max, int32_t budget, int32_t k_out, int32_t prioq_size,
                     int32_t visited_size, int32_t n_fallback, const int32_t *d_idx, void *stream);

/* Replaces: compute_stats (build.py:275-280) / live_d_nn1_max
 * (graph.py:196-199): d_out[4] = {max of finite values (0 if none), sum of
 * finite values, count of finite values, count of non-finite values}. */
int ggnn_layer_stats(const double *d_values, int64_t n, double *d_scratch, double *d_out, void *stream);
size_t ggnn_layer_stats_scratch_bytes(void);

#ifdef __cplusplus
}
#endif
#endif /* GGNN_BUILD_H */
