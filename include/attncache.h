/*
 * attncache.h — C ABI of the B200-native AttnCache hot path (arXiv 2510.25979).
 *
 * The library implements the data-parallel hot path of AttnCache: Alg. 1's
 * "VecDB.search" + threshold gate and Alg. 2's attention
 * step — on a hit, O = attn_map . V with the cached maps
 * (Alg. 2 l.373-375); on a miss, the causal softmax(QK^T/sqrt(d_k)) . V of
 * Eq. 5.  Readings of the paper that the library fixes
 * are listed in DESIGN.md §Readings (R1..R25).
 *
 * Conventions (apply to every call):
 *  - Every call returns attncache_status; ATTNCACHE_OK == 0.  No exception or
 *    C++ type crosses the ABI.  attncache_last_error() gives a thread-local
 *    human-readable detail of the last non-OK status.
 *  - All data pointers are DEVICE pointers owned by the caller (e.g. torch
 *    tensors' data_ptr()); host pointers are rejected with
 *    ATTNCACHE_ERR_INVALID_ARGUMENT when the driver can tell.  Scalars and
 *    descriptor structs are host memory.
 *  - Calls are asynchronous on the given stream (a cudaStream_t passed as
 *    void*; NULL = the legacy default stream); outputs are valid after the
 *    stream is synchronised.  No steady-state call allocates device memory
 *    except the first time a larger batch is seen (scratch growth).
 *  - Errors found by device code (an index outside the database) are
 *    deferred: the offending rows are skipped and the next
 *    attncache_ctx_sync() returns the status.
 *  - All arrays are dense row-major with the innermost dimension contiguous.
 *  - A ctx is used by one host thread at a time.  A db is immutable after
 *    load and may be read concurrently.
 *  - Scratch is per (ctx, stream) and stream-ordered (cudaMallocAsync/cudaFreeAsync on the call's
 *    stream): growing it never synchronises the device, and calls on two streams never share a buffer.
 *    A call captured into a CUDA graph gets scratch of its own that lives as long as the ctx.
 *  - COLLECTIVE calls (marked below) run on a ctx created with a communicator (rank, world, uid):
 *    every rank calls them in the same order with the same tau / layer range (NCCL semantics);
 *    the NCCL operations are enqueued on the caller's stream.  Host round trips inside a collective
 *    call are listed with the call.  On a ctx without a communicator they are the local calls.
 */
#ifndef ATTNCACHE_H_
#define ATTNCACHE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ATTNCACHE_OK = 0,
    ATTNCACHE_ERR_INVALID_ARGUMENT = 1, /* null pointer, NaN tau, bad range, host pointer     */
    ATTNCACHE_ERR_SHAPE = 2,            /* S/L/H/d/D disagree with the database  */
    ATTNCACHE_ERR_DTYPE = 3,            /* unsupported dtype or dtype combination             */
    ATTNCACHE_ERR_ALIGNMENT = 4,        /* base pointer or row pitch not 16-byte aligned      */
    ATTNCACHE_ERR_NOT_FOUND = 5,        /* an index outside the database (deferred)           */
    ATTNCACHE_ERR_EMPTY = 6,            /* search against a database with no entries          */
    ATTNCACHE_ERR_OUT_OF_MEMORY = 7,
    ATTNCACHE_ERR_CUDA = 8,             /* a CUDA runtime/driver error (sticky errors too)    */
    ATTNCACHE_ERR_STATE = 9,            /* wrong device / destroyed handle                    */
    ATTNCACHE_ERR_UNSUPPORTED = 10,     /* e.g. no sm_100 device                              */
    ATTNCACHE_ERR_NCCL = 11             /* NCCL missing or an NCCL call failed (also async)   */
} attncache_status;

typedef enum { ATTNCACHE_F32 = 0, ATTNCACHE_F16 = 1, ATTNCACHE_BF16 = 2 } attncache_dtype;

/* Storage layout of one S x S causal map (see attncache_db_desc):
 *  DENSE  — the full square, row-major, exact +0.0 above the diagonal (S*S elements).
 *  PACKED — the lower triangle only, row-major, row i holding its first 8*(i/8 + 1) elements
 *           (whole 16-byte pieces; entries j > i inside the last piece are the dense map's
 *           +0.0), rows back to back:  row i starts at element 8*(4q(q+1) + r(q+1)) with
 *           q = i / 8, r = i % 8, and a map occupies attncache_packed_map_elems(S) elements.
 *           Requires S % 8 == 0.  It holds exactly the bytes A.V reads (about half of DENSE), so
 *           HBM traffic and DB capacity both halve; attncache_pack_maps builds it (DB building,
 *           Fig. 4 step 3 "store"). */
typedef enum { ATTNCACHE_MAPS_DENSE = 0, ATTNCACHE_MAPS_PACKED = 1 } attncache_map_layout;

typedef struct attncache_ctx attncache_ctx; /* per process and device: scratch + deferred errors */
typedef struct attncache_db attncache_db;   /* this rank's shard view of the memoization database */

const char *attncache_status_string(attncache_status s);
const char *attncache_last_error(void);
/* Library version, e.g. 100 for 0.1.0. */
int32_t attncache_version(void);
/* Number of device kernels this library has launched in this process (all devices, all
 * streams; a monotone counter used to report gpu_launches).  Library-internal memsets are
 * not counted. */
uint64_t attncache_launch_count(void);

/* ---- lifecycle --------------------------------------------------------- */

/* A 128-byte NCCL unique id (ncclGetUniqueId) for attncache_ctx_create: rank 0 creates it and the caller
 * broadcasts it to the other ranks by any means (torch.distributed, a file, MPI).  NCCL is loaded with
 * dlopen ($ATTNCACHE_NCCL_LIB when set, else the copy already in the process, else libnccl.so.2).
 * Errors: NCCL (library not found or call failed), INVALID_ARGUMENT (out NULL). */
attncache_status attncache_get_unique_id(uint8_t out[128]);

/* Creates a context bound to CUDA device `device` (the caller's current device is not changed
 * permanently).  Requires compute capability 10.0 (sm_100a); else ATTNCACHE_ERR_UNSUPPORTED.
 * uid == NULL (world must be 1): a local ctx, no communicator.  uid != NULL: COLLECTIVE — every rank r of
 * [0, world) calls it with the same uid and world, and the ctx owns an NCCL communicator (one process per
 * GPU; north_star: the DB shards by entry across the GPUs of one box).  A world-1 ctx with a uid runs the
 * collective code paths over a one-rank communicator.
 * Errors: INVALID_ARGUMENT (rank outside [0, world), world > 1 without uid), UNSUPPORTED, NCCL, CUDA. */
attncache_status attncache_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t *uid,
                                      attncache_ctx **out);
/* rank / world of the ctx (0 / 1 for a local ctx); either pointer may be NULL. */
attncache_status attncache_ctx_info(const attncache_ctx *ctx, int32_t *rank, int32_t *world);
/* SM budget of the ctx's kernels (no paper passage: a B200 scheduling control for the pipelined multi-GPU
 * step).  compute_sms caps the CTAs of the persistent layer kernels (apply_cached / _local,
 * attend_full, capture_maps, linear), aux_sms the CTAs of the search, projector, placement and row-copy
 * kernels.  Both default to the device's SM count.  A caller that runs the next batch's search, placement
 * and relocation on other streams beside this batch's layers sets compute_sms + aux_sms <= the SM count,
 * so those kernels (and NCCL's) find free SMs instead of queueing behind the persistent kernels (at world 1
 * every reserve measured slower: the HBM-bound A.V needs every SM).  Results do not depend on
 * the budget (the kernels' outputs are independent of their CTA counts).
 * Errors: INVALID_ARGUMENT (NULL ctx, a value < 1 or above the SM count). */
attncache_status attncache_ctx_set_sm_budget(attncache_ctx *ctx, int32_t compute_sms, int32_t aux_sms);
attncache_status attncache_ctx_destroy(attncache_ctx *ctx);
/* Synchronises the device and returns (then clears) any deferred error: ERR_NOT_FOUND when an
 * apply call met an index outside its shard, ERR_CUDA on an asynchronous CUDA fault, ERR_NCCL on an
 * asynchronous communicator error (ncclCommGetAsyncError).  On such an error the library aborts its
 * communicator (ncclCommAbort: no barrier with peers that may be gone) and the ctx stays failed: every
 * later collective call (search, apply_cached, relocate_rows, db_load) and ctx_sync return ERR_NCCL; the
 * caller destroys the ctx (and its dbs) and creates a new one.  Every host wait on collective work (this
 * call, and the count exchanges inside search / apply_cached / db_load) polls that error while it waits, so a
 * peer that died turns into ERR_NCCL instead of a wait that never ends.  SURVEY.md §5 failure detection. */
attncache_status attncache_ctx_sync(attncache_ctx *ctx);

/* The home batch size of every rank for the following collective calls (home_counts: host int64 [world];
 * NULL clears it).  With a layout, collective search needs no host round trip (CUDA-graph capturable);
 * without one it all-gathers the counts and synchronises the stream once per call.  A collective call
 * whose n_home differs from home_counts[rank] returns ERR_STATE. */
attncache_status attncache_set_batch_layout(attncache_ctx *ctx, const int64_t *home_counts, int32_t world);

/* ---- database (Fig. 4: "Both databases share the same index") ----
 *
 * The feature-vector DB (key = vector, value = index) and the attention-map DB (key = index,
 * value = maps) share one index space [0, n_global).  This rank holds the contiguous slice
 * [shard_begin, shard_begin + shard_count).  db_load BORROWS `feats` and `maps`: the caller
 * keeps them alive and unmodified until attncache_db_free.
 *   feats: [shard_count][feat_dim] in feat_dtype (F32 or BF16), rows L2-normalised by the
 *          producer (reading R2: the library never renormalises).
 *   maps : [shard_count][n_layers][n_heads][map] in map_dtype (F16 or BF16) where each map is
 *          one post-softmax causal S x S map in `map_layout` (DENSE: S*S elements, exact +0.0
 *          above the diagonal, reading R11; PACKED: see attncache_map_layout) — layer-
 *          contiguous per entry and head-major inside a layer.  May be NULL
 *          for a search-only database (n_layers = n_heads = seq_len = 0).
 * COLLECTIVE on a ctx with a communicator: the ranks' descriptors must agree on every global field
 * (n_global, feat_dim/dtype, L, H, S, map dtype/layout) and their shards must tile [0, n_global) in rank
 * order (rank r's shard_begin = the sum of the lower ranks' shard_count); one host round trip.
 * Errors: INVALID_ARGUMENT (ranges, null feats with shard_count > 0, n_global >= 2^32, PACKED
 * non-causal maps, shards not tiling), SHAPE (ranks disagree), DTYPE, ALIGNMENT (feats/maps base or row
 * pitch not a multiple of 16 bytes), NCCL. */
typedef struct {
    int64_t n_global;
    int64_t shard_begin;
    int64_t shard_count;
    int32_t feat_dim;
    int32_t feat_dtype; /* attncache_dtype */
    const void *feats;
    int32_t n_layers;
    int32_t n_heads;
    int32_t seq_len;
    int32_t map_dtype; /* attncache_dtype */
    const void *maps;
    int32_t map_layout;     /* attncache_map_layout */
    int32_t maps_noncausal; /* 0: causal decoder maps (R11); 1: full encoder maps (bidirectional
                               models; f3) — A.V reads every column; DENSE only */
} attncache_db_desc;

attncache_status attncache_db_load(attncache_ctx *ctx, const attncache_db_desc *desc, attncache_db **out);
/* Frees the db handle (never the borrowed tensors).  May run after its ctx is destroyed; every other call
 * on a db needs its ctx alive. */
attncache_status attncache_db_free(attncache_db *db);

/* ---- Alg. 1: VecDB.search + theta gate -----------
 *
 * attncache_search — the top-1 of this rank's n_queries HOME queries over the WHOLE database.
 *   Local ctx: the shard must cover the whole DB (shard_count == n_global; for shards on one process use
 *   search_keys + keys_decode).  COLLECTIVE ctx (north_star's sharded search):
 *   C1 the query batch is gathered on every rank (an NCCL all-gather when every home block has the same
 *   size, else grouped send/recv), K1 every rank takes its shard's top-1 key of every query, C2 one NCCL
 *   u64 max-all-reduce of the keys (= the global top-1 with the lowest-index tie-break, reading R3), K2
 *   decode + tau gate of the home block.  Host round trip: the home counts exchange when no batch layout
 *   is set (attncache_set_batch_layout).  n_queries may be 0 on some ranks.
 *   queries: [n_queries][feat_dim] in the DB's feat_dtype (no silent casts; reading R10).
 *   idx[b]  : global index of the top-1 entry by inner product s = q . x (fp32 accumulation),
 *             the LOWEST index among equal scores (reading R3); always set, also on a miss.
 *   score[b]: that fp32 inner product.   hit[b]: 1 iff score[b] >= tau (inclusive).
 * tau may be any non-NaN float (tau > 1: every query misses).  n_queries may be 0.
 * Errors: EMPTY (n_global == 0), INVALID_ARGUMENT (NaN tau, null pointers with n > 0), STATE (a partial
 * shard on a local ctx; n_queries disagreeing with the batch layout), NCCL. */
attncache_status attncache_search(attncache_db *db, const void *queries, int64_t n_queries, float tau,
                                  int64_t *idx, float *score, uint8_t *hit, void *stream);
/* The same search, writing the decisions of the WHOLE batch (every rank's home block in rank order,
 * sum of the home counts rows) on every rank — what the owner-affinity placement needs.
 * COLLECTIVE on a ctx with a communicator; on a local ctx the same as attncache_search. */
attncache_status attncache_search_all(attncache_db *db, const void *queries, int64_t n_queries, float tau,
                                      int64_t *idx, float *score, uint8_t *hit, void *stream);

/* Sharded halves of the same search (C1/C2 of SURVEY.md §2.4).  search_keys writes, per query,
 * the packed key of this shard's top-1:  key = ord(score) << 32 | (0xFFFFFFFF - global_index),
 * an unsigned 64-bit value where ord() maps fp32 bits to an order-preserving u32 (-0.0
 * canonicalised to +0.0).  The maximum key over shards is the global top-1 with the
 * lowest-index tie-break, in any reduction order (reading R3).  An empty shard writes 0 (the
 * neutral element).  keys: [n_queries] uint64 on the device (callers may move them as int64 bit
 * patterns, e.g. with an all-gather).
 * keys_decode reduces keys [n_shards][n_queries] by unsigned max over shards (the cross-shard
 * top-1 of north_star) and decodes idx/score/hit exactly as attncache_search does; a query whose
 * keys are all 0 gets idx = -1, score = -inf, hit = 0. */
attncache_status attncache_search_keys(attncache_db *db, const void *queries, int64_t n_queries,
                                       uint64_t *keys, void *stream);
attncache_status attncache_keys_decode(const uint64_t *keys, int32_t n_shards, int64_t n_queries, float tau,
                                       int64_t *idx, float *score, uint8_t *hit, void *stream);

/* ---- Alg. 2 hit branch: O = attn_map . V ---------------
 *
 * For every row b in [0, n_rows) that is selected — hit[b] != 0 when `hit` is non-NULL, else
 * idx[b] >= 0 — and for every layer l in [layer_begin, layer_end) and head h (idx: GLOBAL entry indices):
 *     O[b][l-layer_begin][h] (S x d) = maps[idx[b] - shard_begin][l][h] (S x S) . V[b][l-layer_begin][h] (S x d)
 * accumulated in fp32 and rounded once to act_dtype.  Unselected rows of O are left untouched.
 * V, O: [n_rows][layer_end-layer_begin][n_heads][seq_len][head_dim] in act_dtype.
 * The maps are read in place from the DB (no "attention cache" copy; reading R18); tiles above
 * the diagonal are never read.  A selected idx outside this shard is skipped and reported by the
 * next attncache_ctx_sync() as ERR_NOT_FOUND.  Supported: act_dtype == map_dtype (tensor cores),
 * or act_dtype F32 with any map dtype (CUDA cores).
 * COLLECTIVE ctx (north_star: "Hit queries are then routed to the owning GPU, whose A.V output returns
 * to the query's home GPU by NCCL send/recv"): K3 buckets the selected home rows by the rank owning their
 * entry, C3 exchanges the per-peer counts (one host round trip sizes the transfers), C4 ships the V rows
 * and entry indices to the owners (grouped ncclSend/ncclRecv), K4 runs A.V there on the local maps, C5
 * returns the O rows, K3 scatters them into O.  Scratch for the transfers is stream-ordered.
 * Errors: SHAPE (layer range outside [0, n_layers), head_dim <= 0), DTYPE, ALIGNMENT, STATE
 * (db has no maps), NCCL. */
attncache_status attncache_apply_cached(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                        int32_t layer_begin, int32_t layer_end, int32_t head_dim,
                                        int32_t act_dtype, const void *V, void *O, void *stream);

/* The LOCAL A.V of the rows whose entry lies in this rank's shard (no communication, never routes; the
 * owner-affinity placement runs every hit on its owner): the same as attncache_apply_cached
 * on a local ctx, with GQA head counts as attncache_apply_cached_gqa.  A selected idx outside this shard is
 * skipped and reported by the next ctx_sync as ERR_NOT_FOUND. */
attncache_status attncache_apply_cached_local(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                              int32_t layer_begin, int32_t layer_end, int32_t head_dim,
                                              int32_t n_kv_heads, int32_t act_dtype, const void *V, void *O,
                                              void *stream);

/* Grouped-query attention (GQA; SURVEY.md §8(f) f3 "optional GQA n_kv_heads"; Llama-3 models keep fewer
 * K/V heads than query heads): the same as attncache_apply_cached with V: [n_rows][layer_end-layer_begin]
 * [n_kv_heads][seq_len][head_dim] and O: [n_rows][layer_end-layer_begin][n_heads][seq_len][head_dim]; the map
 * of query head h multiplies V head h / (n_heads / n_kv_heads).  n_kv_heads == n_heads is exactly
 * attncache_apply_cached.  Errors as apply_cached, plus SHAPE when n_kv_heads does not divide n_heads. */
attncache_status attncache_apply_cached_gqa(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                            int32_t layer_begin, int32_t layer_end, int32_t head_dim,
                                            int32_t n_kv_heads, int32_t act_dtype, const void *V, void *O,
                                            void *stream);

/* ---- Alg. 2 miss branch core (Eq. 5) -------
 *
 * O = softmax(Q K^T * scale with keys j > i masked) . V for every selected row b (skip == NULL
 * or skip[b] == 0), layer and head.  Q and K arrive post-RoPE (RoPE is outside the path;
 * reading R16).  scale <= 0 means 1/sqrt(head_dim).  Q, K, V, O:
 * [batch][n_layers][n_heads][seq_len][head_dim] in act_dtype; fp32 softmax statistics.
 * Local to the calling device. */
attncache_status attncache_attend_full(attncache_ctx *ctx, int64_t batch, int32_t n_layers, int32_t n_heads,
                                       int32_t seq_len, int32_t head_dim, int32_t act_dtype, const void *Q,
                                       const void *K, const void *V, float scale, const uint8_t *skip, void *O,
                                       void *stream);

/* GQA variant: Q, O: [batch][n_layers][n_heads][seq_len][head_dim]; K, V: [batch][n_layers][n_kv_heads]
 * [seq_len][head_dim]; query head h attends with K/V head h / (n_heads / n_kv_heads).  n_kv_heads == n_heads is
 * exactly attncache_attend_full.  Errors as attend_full, plus SHAPE when n_kv_heads does not divide n_heads. */
attncache_status attncache_attend_full_gqa(attncache_ctx *ctx, int64_t batch, int32_t n_layers, int32_t n_heads,
                                           int32_t n_kv_heads, int32_t seq_len, int32_t head_dim, int32_t act_dtype,
                                           const void *Q, const void *K, const void *V, float scale,
                                           const uint8_t *skip, void *O, void *stream);

/* ---- the whole single-rank step from HOST buffers (the end-to-end call) ----------------------
 * Alg. 1 then Alg. 2 for every layer of the DB, with the host<->device copies inside the call: H2D of the
 * queries, search (idx/score/hit as attncache_search), D2H of the decisions (one host sync: Alg. 2 computes
 * q and k only on a miss, so only the misses' Q and K cross PCIe), then chunks of `chunk`
 * rows through a ring of `depth` device slots on three library streams (copy-in, compute, copy-out):
 * H2D of V (every row) and Q, K (miss rows), attncache_apply_cached on the hits and attncache_attend_full on
 * the misses, D2H of O.  Synchronous: returns when O and idx/score/hit are in host memory.
 *   q: [n][feat_dim] feat dtype; Q, K, V, O: [n][n_layers][n_heads][seq_len][head_dim] act_dtype;
 *   idx int64 / score fp32 / hit uint8: [n].  Every pointer must be PAGE-LOCKED HOST memory
 *   (cudaHostAlloc / cudaHostRegister).  Device staging is ctx scratch.  A local db holding every entry.
 *   chunk: rows per pipeline step; ~100-300 MB of V per chunk keeps the copy engines busy with a short ring
 *   fill / drain (the Python binding's default: ~192 MB, at most 16 rows).
 * Errors: INVALID_ARGUMENT (pageable or device pointers, chunk <= 0, depth outside [2, 8], NaN tau), STATE
 * (a shard / a collective ctx of world > 1 / no maps), EMPTY, DTYPE, ALIGNMENT, CUDA. */
attncache_status attncache_prefill_host(attncache_db *db, const void *q, int64_t n, float tau, const void *Q,
                                        const void *K, const void *V, int32_t head_dim, int32_t act_dtype, void *O,
                                        int64_t *idx, float *score, uint8_t *hit, int32_t chunk, int32_t depth);

/* ---- DB building, capture (Fig. 4 step 1; "collect
 * the input hidden states and their corresponding attention maps at each layer") --------------
 * maps_out[b][l][h] = softmax(Q K^T * scale with keys j > i masked), rounded once to map_dtype (the
 * post-softmax probabilities of the miss branch; reading R12), for every selected row b (skip == NULL
 * or skip[b] == 0), stored in `map_layout` exactly as a DB entry [n_layers][n_heads][map] (DENSE:
 * +0.0 above the diagonal); unselected rows untouched.  Q, K: [batch][L][H][S][d] in act_dtype;
 * scale <= 0 means 1/sqrt(head_dim).  maps_out rows can be handed to attncache_db_load as entries.
 * Errors: SHAPE (S % 8 != 0 for 16-byte map rows), DTYPE (map_dtype not F16/BF16), ALIGNMENT. */
attncache_status attncache_capture_maps(attncache_ctx *ctx, int64_t batch, int32_t n_layers, int32_t n_heads,
                                        int32_t seq_len, int32_t head_dim, int32_t act_dtype, const void *Q,
                                        const void *K, float scale, const uint8_t *skip, int32_t map_dtype,
                                        int32_t map_layout, void *maps_out, void *stream);

/* ---- feature projector (Alg. 1 l.254 "f <- feature_projector(h)", PAPER.md:254;
 * PAPER.md:278 "two layers of Multi-Layer Perceptron ... maps the input embedding to a feature vector") ----
 * For every row b of h (readings R30-R32):
 *     z = relu(W1 h[b] + b1)        W1: [hidden_dim][in_dim]  (nn.Linear layout), b1: [hidden_dim] fp32
 *     y = W2 z + b2                 W2: [feat_dim][hidden_dim],                   b2: [feat_dim] fp32
 *     features[b] = y / ||y||_2     (0 if y = 0), rounded once to feat_dtype
 * h: [n][in_dim], W1, W2 in act_dtype (BF16/F16: tensor cores when in_dim, hidden_dim and feat_dim are
 * multiples of 64; F32 or other shapes: CUDA cores); fp32 accumulation; z is rounded once to act_dtype
 * (the second layer's operand) and y kept in fp32.  features: [n][feat_dim] in feat_dtype, ready to be
 * searched (attncache_search) or stored as DB rows (Fig. 4 step 2).  Device pointers;
 * scratch (z, y) is owned by ctx.  Errors: SHAPE (non-positive dims), DTYPE, ALIGNMENT (bases, or rows
 * of in_dim / hidden_dim elements, not 16-byte aligned), INVALID_ARGUMENT (NULL or host pointers). */
attncache_status attncache_project_features(attncache_ctx *ctx, const void *h, int64_t n, int32_t in_dim,
                                            int32_t act_dtype, const void *W1, const float *b1, int32_t hidden_dim,
                                            const void *W2, const float *b2, int32_t feat_dim, int32_t feat_dtype,
                                            void *features, void *stream);

/* GQA variant of attncache_capture_maps: K: [batch][L][n_kv_heads][S][d], one map per query head (query head h
 * uses K head h / (n_heads / n_kv_heads)).  Errors as capture_maps, plus SHAPE (n_kv_heads not dividing n_heads). */
attncache_status attncache_capture_maps_gqa(attncache_ctx *ctx, int64_t batch, int32_t n_layers, int32_t n_heads,
                                            int32_t n_kv_heads, int32_t seq_len, int32_t head_dim, int32_t act_dtype,
                                            const void *Q, const void *K, float scale, const uint8_t *skip,
                                            int32_t map_dtype, int32_t map_layout, void *maps_out, void *stream);

/* ---- projection GEMM for the Eq. 5 block-level comparison (Alg. 2 l.372 "v = V(h)",
 * l.377-378 "q = Q(h)", "k = K(h)"; Eq. 5) ----------------------------------------
 * Y = X W^T (+ bias): X [M][K] with M = B * seq_len rows (row m = sequence b, position s), W [N][K] (the
 * nn.Linear layout), N = n_heads * head_dim; the result is stored HEAD-MAJOR, Y [B][n_heads][seq_len][head_dim]
 * (the layout attncache_attend_full / attncache_apply_cached read, so no permute pass follows).  dtype for X, W
 * and Y; fp32 accumulation, one rounding; bias: NULL or device fp32 [N].  BF16/F16 with K % 64 == 0,
 * N % 64 == 0 and head_dim % 32 == 0: tcgen05 GEMM; other shapes / F32: CUDA cores.
 * Errors: SHAPE (M not whole sequences, N not whole heads), DTYPE, ALIGNMENT, INVALID_ARGUMENT. */
attncache_status attncache_linear(attncache_ctx *ctx, const void *X, int64_t M, int32_t K, const void *W, int32_t N,
                                  int32_t dtype, const float *bias, int32_t seq_len, int32_t head_dim, void *Y,
                                  void *stream);

/* ---- RoPE for the Eq. 5 block-level comparison (Alg. 2 l.379) ----------
 * In place on X [n_units][S][d] (act_dtype): for i < d/2 the pair (x_i, x_{i+d/2}) at position p
 * (= row index) is rotated by the angle p * base^(-2i/d) (rotate-half convention; reading R29),
 * computed in fp32 and rounded once.  Errors: SHAPE (d odd), DTYPE, ALIGNMENT. */
attncache_status attncache_rope(void *X, int64_t n_units, int32_t seq_len, int32_t head_dim, int32_t act_dtype,
                                float base, void *stream);

/* ---- routing helpers for the multi-GPU path (north_star: hits go to the owning GPU) ----
 *
 * route_plan: for rows b in [0, n_rows) with hit[b] != 0, owner[b] = the rank r with
 * shard_begins[r] <= idx[b] < shard_begins[r+1] (shard_begins: device int64[world+1]);
 * owner[b] = -1 for misses.  counts[r] = number of rows owned by r; order = the selected rows
 * grouped by owner (ascending rank, ascending b inside a rank), n = sum(counts) entries used.
 * Deterministic.  gather_rows: dst[k] = src[rows[k]]; scatter_rows: dst[rows[k]] = src[k];
 * rows are int64 row numbers and rows are row_bytes long (a multiple of 8; 16 is faster).
 * route_plan with hit == NULL selects the rows with idx[b] >= 0. */
attncache_status attncache_route_plan(const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                      const int64_t *shard_begins, int32_t world, int32_t *owner, int32_t *counts,
                                      int64_t *order, void *stream);
attncache_status attncache_gather_rows(const void *src, const int64_t *rows, int64_t n_rows, int64_t row_bytes,
                                       void *dst, void *stream);
attncache_status attncache_scatter_rows(const void *src, const int64_t *rows, int64_t n_rows, int64_t row_bytes,
                                        void *dst, void *stream);

/* ---- owner-affinity placement (the scalable multi-GPU variant) ----
 * HOST function: plain host pointers, no device work, callable without a GPU.  Decides once per batch,
 * before the layer loop, which rank processes each query, so that no per-layer V or O crosses NVLink
 * (the prescribed V -> owner / O -> home routing moves both for every layer):
 *   - a hit row b goes to the rank r owning its entry, shard_begins[r] <= idx[b] < shard_begins[r+1],
 *     where the maps are local (north_star: "routed to the owning GPU");
 *   - then every miss row, in ascending b, goes to the rank with the smallest accumulated cost (the
 *     lowest rank on ties); a hit adds hit_cost to its rank and a miss miss_cost (callers pass the
 *     per-query algorithmic HBM bytes of one A.V / one attention, which set the kernel times).
 * Placing equal-cost misses one at a time on the least-loaded rank, on top of the fixed hit loads,
 * minimises the maximum load (tested against brute force).  idx, hit: [n_rows] for the whole batch
 * (every rank computes the same plan from the same inputs).  Outputs: assign[b] = the processing rank;
 * load[r] (optional, may be NULL; [world]) = the accumulated cost on rank r.  Deterministic.
 * Errors: INVALID_ARGUMENT (n_rows < 0, world outside [1, 1024], NULL arrays, shard_begins not
 * non-decreasing, NaN or negative costs, a hit idx outside [shard_begins[0], shard_begins[world])). */
attncache_status attncache_affinity_plan(const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                         const int64_t *shard_begins, int32_t world, double hit_cost,
                                         double miss_cost, int32_t *assign, double *load);

/* The same plan on the DEVICE, plus one rank's relocation lists, so the placement costs no host round
 * trip beyond the counts NCCL's all_to_all needs (one kernel launch of one CTA on `stream`).  assign and
 * load are bitwise those of attncache_affinity_plan (the per-rank loads are the same sequential sums).
 * Inputs: idx, hit: device [n_rows] (the whole batch; every rank passes the same); shard_begins,
 * home_begins: HOST [world + 1] (home_begins: the batch positions of each rank's home block, 0 .. n_rows);
 * world in [1, 32]; rank: this rank.  Outputs (device, caller-allocated): assign int32 [n_rows];
 * load double [world]; loc int64 [n_rows] (the positions placed on `rank`, ascending: the first n_loc
 * entries); idx_loc int64 / hit_loc uint8 [n_rows] (their idx, 0 for misses, and hit flags); send_order
 * int64 [home size] (this rank's home rows, home-relative, stably sorted by destination rank);
 * counts int32 [2 world + 1] = send_n[world] | recv_n[world] | n_loc.  A hit idx outside
 * [shard_begins[0], shard_begins[world]) is placed on rank 0 or world - 1 (the host function rejects it).
 * Scratch: n_rows int64 from ctx.  Errors: INVALID_ARGUMENT (world outside [1, 32], rank outside
 * [0, world), NULL arrays, begins not non-decreasing, home_begins not spanning [0, n_rows], NaN or
 * negative costs), OUT_OF_MEMORY, CUDA. */
attncache_status attncache_affinity_plan_device(attncache_ctx *ctx, const int64_t *idx, const uint8_t *hit,
                                                int64_t n_rows, const int64_t *shard_begins, int32_t world,
                                                double hit_cost, double miss_cost, int32_t rank,
                                                const int64_t *home_begins, int32_t *assign, double *load,
                                                int64_t *loc, int64_t *idx_loc, uint8_t *hit_loc,
                                                int64_t *send_order, int32_t *counts, void *stream);

/* Moves request state to the ranks the placement chose (COLLECTIVE; SURVEY.md §8(e) owner-affinity: "the
 * request's hidden state moves once").  Sends this rank's home rows src[send_order[k]] (k < n_home) to the
 * ranks in the order of `counts` (host int32 [2 world + 1] as attncache_affinity_plan_device returns it:
 * send_n[world] | recv_n[world] | n_loc; send_n sums to n_home) and writes the rows received from ranks
 * 0..world-1, in rank order, to dst [sum recv_n rows].  Rows are row_bytes long (a multiple of 8).  One
 * NCCL group of send/recv pairs; on a local ctx a device copy.  Errors: INVALID_ARGUMENT, NCCL, CUDA. */
attncache_status attncache_relocate_rows(attncache_ctx *ctx, const void *src, int64_t n_home, int64_t row_bytes,
                                         const int64_t *send_order, const int32_t *counts, void *dst, void *stream);

/* ---- DB building: packed map layout (Fig. 4 step 3) -----------
 * Number of elements one PACKED S x S map occupies (0 if S % 8 != 0). */
int64_t attncache_packed_map_elems(int32_t seq_len);
/* Converts n_maps DENSE S x S maps (16-bit elements, device) into the PACKED layout (device,
 * n_maps * attncache_packed_map_elems(S) elements).  Pure data movement: the packed map holds the
 * dense map's bytes for every j <= i.  Errors: SHAPE (S % 8 != 0), ALIGNMENT. */
attncache_status attncache_pack_maps(const void *dense, int64_t n_maps, int32_t seq_len, void *packed, void *stream);

/* ---- test/debug: literal AttnMapsDB.get(idx, n) (Alg. 1 l.259) ------------
 * Writes maps[idx - shard_begin][layer_begin:layer_end] of a LOCAL entry to `out` (device) as
 * DENSE [layers][H][S][S] maps whatever the DB layout (a PACKED DB is expanded, +0.0 above the
 * diagonal).  Errors: NOT_FOUND (idx outside this shard), SHAPE. */
attncache_status attncache_fetch_maps(attncache_db *db, int64_t idx, int32_t layer_begin, int32_t layer_end,
                                      void *out, void *stream);

/* ---- introspection: kernel variant chosen for a call (for tests/bench) ----
 * kind: 0 = search, 1 = apply, 2 = attend, 3 = capture, 4 = one projector layer (seq_len = its K, head_dim =
 * its output width).  Returns a static string such as "tc" (tcgen05) or "ffma" for the arguments given
 * (no launch). */
const char *attncache_variant(int32_t kind, int32_t dtype, int32_t seq_len, int32_t head_dim);

#ifdef __cplusplus
}
#endif
#endif /* ATTNCACHE_H_ */
