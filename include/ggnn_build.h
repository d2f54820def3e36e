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

#ifdef __cplusplus
}
#endif
#endif /* GGNN_BUILD_H */
