/*
 * ggnn_shard.h -- C ABI of the sharded-search kernels in libggnn_b200.so.
 * Conventions as in ggnn_b200.h (device pointers d_*, async on `stream`,
 * 0 / negative GGNN_E* return codes).
 *
 * A sharded query (shard.py:91-128 in the reference) is: every shard answers
 * the query batch on its own hierarchy, the local ids are mapped to dataset
 * ids through the shard's slice of the global permutation, and the G lists
 * of every query are merged by (distance, dataset id).  On the device the
 * per-shard results of one batch live in a "shard block":
 *
 *     ids      int32  (m, k_in)   at byte 0
 *     dists    f64    (m, k_in)   at ggnn_shard_block_dists_offset(m, k_in)
 *     counters int32  (m, 5)      at ggnn_shard_block_counters_offset(m, k_in)
 *
 * and G blocks sit back to back (block g at g * ggnn_shard_block_bytes).  The
 * query kernel writes straight into a block (ggnn_query_batch takes the three
 * pointers), so with G ranks the blocks are exactly the NCCL all-gather
 * send / receive buffers and no copy is needed before or after the exchange.
 */
#ifndef GGNN_SHARD_H
#define GGNN_SHARD_H

#include "ggnn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

size_t ggnn_shard_block_bytes(int64_t m, int32_t k_in);
size_t ggnn_shard_block_dists_offset(int64_t m, int32_t k_in);
size_t ggnn_shard_block_counters_offset(int64_t m, int32_t k_in);

/* Replaces: the id globalization of _merge_shard_results
 * (shard.py:100: gid = permutation[offset + local]).  Rewrites the count ids
 * of d_ids in place: id >= 0 becomes d_gid_of_local[id], -1 stays -1.
 * d_gid_of_local is the shard's slice permutation[offset : offset + size]. */
int ggnn_shard_globalize(int32_t *d_ids, int64_t count, const int32_t *d_gid_of_local, int64_t size,
                         void *stream);

/* Replaces: _merge_shard_results (shard.py:91-110) for m queries at once.
 * d_blocks holds G shard blocks (layout above) whose ids are already global.
 * Output: d_out_ids / d_out_dists (m, k_out), the k_out smallest (dist, id)
 * pairs over all G lists, ascending, -1 / +inf padded; d_out_counters (m, 5)
 * (optional) = [sum of visited_count, sum of steps, terminated_by of the
 * shard holding the best hit (queue-empty = 1 when there is none), 0, 0] --
 * the reference's merged QueryResult leaves distinct_touched and forgotten
 * at their defaults (0). */
int ggnn_shard_merge(const void *d_blocks, int32_t G, int64_t m, int32_t k_in, int32_t k_out, int32_t *d_out_ids,
                     double *d_out_dists, int32_t *d_out_counters, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GGNN_SHARD_H */
