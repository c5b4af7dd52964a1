// abi_internal.cuh — pieces of the C ABI shared between attncache.cu (local calls) and collective.cu.
#pragma once
#include "kernels.cuh"

namespace ac {

// K1 on this shard: keys[b] = packed top-1 key of queries[b] over the local entries (0 for an empty shard).
attncache_status search_keys_impl(attncache_db *db, const void *queries, int64_t n, uint64_t *keys, cudaStream_t st);

// Validated local A.V (rows whose entry lies in this shard; others are skipped and reported by ctx_sync).
attncache_status apply_local_impl(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                  int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t n_kv_heads,
                                  int32_t act_dtype, const void *V, void *O, cudaStream_t st);

// collective.cu
attncache_status comm_check(attncache_ctx *ctx);          // polls the async error; aborts the comm on one
attncache_status comm_failed_status();                    // ERR_NCCL: the comm was aborted (see comm_check)
// Host wait for `st` (marked_only: for the last collective work recorded, if any) polling the async NCCL error.
attncache_status comm_wait(attncache_ctx *ctx, cudaStream_t st, bool marked_only);
attncache_status db_load_collective(attncache_db *db);
attncache_status search_collective(attncache_db *db, const void *q, int64_t n_home, float tau, bool all, int64_t *idx,
                                   float *score, uint8_t *hit, cudaStream_t st);
attncache_status apply_routed(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_home,
                              int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t n_kv_heads,
                              int32_t act_dtype, const void *V, void *O, cudaStream_t st);

}  // namespace ac
