/*
 * ggnn_p2p.h -- fused sharded exchange over peer memory (NVLink / NVSwitch).
 *
 * The NCCL path (ggnn_shard.h + all_gather_into_tensor) moves each rank's
 * shard block after its search finishes.  This path fuses the exchange into
 * the search: every warp of ggnn_query_batch_push, as it finishes a query,
 * stores that query's globalized (ids, dists, counters) row straight into
 * block `rank` of EVERY rank's receive buffer (peer pointers from CUDA IPC),
 * so the transfer overlaps the search query by query; ggnn_p2p_signal then
 * publishes the epoch to every peer and ggnn_shard_merge_wait merges once all
 * G flags show it.  Receive buffers are double-buffered by epoch parity.
 *
 * Layout of one receive allocation (ggnn_p2p_bytes): two halves (parity 0 / 1),
 * each G shard blocks (ggnn_shard.h layout) followed by G uint32 flags.
 */
#ifndef GGNN_P2P_H
#define GGNN_P2P_H

#include "ggnn_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define GGNN_P2P_MAX_RANKS 8
#define GGNN_IPC_HANDLE_BYTES 64

size_t ggnn_p2p_bytes(int32_t G, int64_t m, int32_t k);
/* cudaMalloc'd, zeroed receive allocation and its CUDA IPC handle (64 bytes). */
int ggnn_p2p_alloc(size_t bytes, void **d_ptr, void *ipc_handle_out);
/* Map a peer's receive allocation (lazy peer access); same-device handles work too. */
int ggnn_p2p_open(const void *ipc_handle, void **d_peer_ptr);
int ggnn_p2p_close(void *d_peer_ptr);
int ggnn_p2p_free(void *d_ptr);

/* Where the search stores its rows: d_peers[g] = rank g's receive allocation
 * (own one included), this rank's index, the epoch parity to use, and the
 * shard's local -> dataset id table (shard.py:100). */
typedef struct ggnn_push {
    void *d_peers[GGNN_P2P_MAX_RANKS];
    int32_t nranks;
    int32_t rank;
    int32_t parity;
    int32_t pad_;
    const int32_t *d_gid_of_local;
    int64_t gid_size;
} ggnn_push;

/* ggnn_query_batch whose epilogue also writes every query's globalized row
 * into block `rank` of all receive allocations (d_ids / d_dists / d_counters
 * still receive the local, shard-local-id results). */
int ggnn_query_batch_push(const ggnn_vectors *X, const ggnn_layer *bottom, const int32_t *d_top_rows, int64_t ntop,
                          const ggnn_queries *Q, const ggnn_search_params *p, double d_nn1_max, int32_t *d_ids,
                          double *d_dists, int32_t *d_counters, const ggnn_push *push, void *stream);

/* After the push search on the same stream: system-scope fence, then store
 * `epoch` into flag `rank` of every receive allocation (parity half). */
int ggnn_p2p_signal(const ggnn_push *push, int64_t m, int32_t k, uint32_t epoch, void *stream);

/* Wait (bounded: ~10 s, then *d_error = 1) until all G flags of the parity
 * half of d_recv show `epoch`, then ggnn_shard_merge of its G blocks. */
int ggnn_shard_merge_wait(const void *d_recv, int32_t parity, uint32_t epoch, int32_t G, int64_t m, int32_t k,
                          int32_t k_out, int32_t *d_out_ids, double *d_out_dists, int32_t *d_out_counters,
                          int32_t *d_error, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GGNN_P2P_H */
