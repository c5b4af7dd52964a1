// attncache.cu — the C ABI (include/attncache.h): validation, scratch management, dispatch.
// Every step of the hot path runs in the kernels launched from here; nothing computes on the host.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <cmath>

#include "abi_internal.cuh"

namespace ac {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

attncache_status fail(attncache_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

attncache_status cuda_status(cudaError_t e, const char *what) {
    if (e == cudaErrorMemoryAllocation) return fail(ATTNCACHE_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(ATTNCACHE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Row selection fused into the layer kernels (one launch fewer) on a local ctx only: a collective ctx runs the
// next batch's search / placement / relocation on side streams beside its layer kernels, and the select launch
// between A.V and attention is the window in which those kernels get SMs (world-1 pipelined step: 1.17 ms fused
// against 1.10-1.15 with the select launches; DESIGN.md §7 K3).  AC_NO_FUSED_SELECT=1 turns it off everywhere.
bool fused_select_ok(const attncache_ctx *ctx) { return ctx->comm == nullptr && !getenv("AC_NO_FUSED_SELECT"); }

attncache_status scratch(attncache_ctx *ctx, cudaStream_t st, int kind, size_t bytes, void **out, bool *fresh) {
    *out = nullptr;
    if (fresh) *fresh = false;
    if (bytes == 0) bytes = 16;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    AC_CUDA(cudaStreamIsCapturing(st, &cs));
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (cs == cudaStreamCaptureStatusActive) {
        // a graph keeps its scratch for its whole life: a buffer of its own, allocated outside the capture
        // (relaxed mode: cudaMalloc does not touch the captured stream) and freed with the ctx
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        AC_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, bytes);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (e != cudaSuccess) return cuda_status(e, "scratch (graph capture)");
        ctx->graph_owned.push_back(p);
        *out = p;
        if (fresh) *fresh = true;
        return ATTNCACHE_OK;
    }
    Scratch &s = ctx->scratch[st].s[kind];
    if (s.bytes < bytes) {
        // stream-ordered: the old buffer is released after the work already queued on this stream
        if (s.ptr) AC_CUDA(cudaFreeAsync(s.ptr, st));
        s.ptr = nullptr;
        s.bytes = 0;
        const size_t cap = bytes < 4096 ? 4096 : bytes + bytes / 4;
        AC_CUDA(cudaMallocAsync(&s.ptr, cap, st));
        s.bytes = cap;
        if (fresh) *fresh = true;
    }
    *out = s.ptr;
    return ATTNCACHE_OK;
}

}  // namespace ac

using namespace ac;

extern "C" {

const char *attncache_status_string(attncache_status s) {
    switch (s) {
    case ATTNCACHE_OK: return "ATTNCACHE_OK";
    case ATTNCACHE_ERR_INVALID_ARGUMENT: return "ATTNCACHE_ERR_INVALID_ARGUMENT";
    case ATTNCACHE_ERR_SHAPE: return "ATTNCACHE_ERR_SHAPE";
    case ATTNCACHE_ERR_DTYPE: return "ATTNCACHE_ERR_DTYPE";
    case ATTNCACHE_ERR_ALIGNMENT: return "ATTNCACHE_ERR_ALIGNMENT";
    case ATTNCACHE_ERR_NOT_FOUND: return "ATTNCACHE_ERR_NOT_FOUND";
    case ATTNCACHE_ERR_EMPTY: return "ATTNCACHE_ERR_EMPTY";
    case ATTNCACHE_ERR_OUT_OF_MEMORY: return "ATTNCACHE_ERR_OUT_OF_MEMORY";
    case ATTNCACHE_ERR_CUDA: return "ATTNCACHE_ERR_CUDA";
    case ATTNCACHE_ERR_STATE: return "ATTNCACHE_ERR_STATE";
    case ATTNCACHE_ERR_UNSUPPORTED: return "ATTNCACHE_ERR_UNSUPPORTED";
    case ATTNCACHE_ERR_NCCL: return "ATTNCACHE_ERR_NCCL";
    }
    return "ATTNCACHE_ERR_UNKNOWN";
}

const char *attncache_last_error(void) { return g_err; }

int32_t attncache_version(void) { return 200; }

uint64_t attncache_launch_count(void) { return ac::launch_count(); }

const char *attncache_variant(int32_t kind, int32_t dtype, int32_t seq_len, int32_t head_dim) {
    if (kind == 4) return linear_tc_supported(dtype, seq_len, head_dim) ? "tc" : "ffma";
    switch (kind) {
    case 0: return search_tc_supported(dtype, head_dim) ? "tc" : "ffma";  // head_dim = feat_dim here
    case 1: return apply_tc_supported(dtype, dtype, seq_len, head_dim) ? "tc" : "ffma";
    case 2: return attend_tc_supported(dtype, seq_len, head_dim) ? "tc" : "ffma";
    case 3: return capture_tc_supported(dtype, seq_len, head_dim) ? "tc" : "ffma";
    }
    return "none";
}

// ---- lifecycle ------------------------------------------------------------------------------

attncache_status attncache_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t *uid,
                                      attncache_ctx **out) {
    if (!out) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_create: out is NULL");
    *out = nullptr;
    if (world < 1 || world > 1024 || rank < 0 || rank >= world)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_create: rank %d of world %d", rank, world);
    if (world > 1 && !uid) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_create: world %d needs a unique id", world);
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(ATTNCACHE_ERR_UNSUPPORTED, "ctx_create: no CUDA device (%s)", cudaGetErrorString(e));
    }
    if (device < 0 || device >= n) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_create: device %d of %d", device, n);
    cudaDeviceProp prop;
    AC_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(ATTNCACHE_ERR_UNSUPPORTED, "ctx_create: device %d is sm_%d%d; this library is built for sm_100a",
                    device, prop.major, prop.minor);
    DeviceGuard g(device);
    attncache_ctx *c = new attncache_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    c->compute_sms = c->aux_sms = c->sm_count;
    const char *fr = getenv("ATTNCACHE_FORCE_ROUTE");
    c->force_route = fr && *fr == '1';
    e = cudaMalloc(&c->d_error, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(c->d_error, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&c->d_small, sizeof(int64_t) * kPinnedInts);
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_pinned, sizeof(int64_t) * kPinnedInts);
    if (e != cudaSuccess) {
        attncache_ctx_destroy(c);
        return cuda_status(e, "ctx_create: scratch");
    }
    if (uid) {  // COLLECTIVE: every rank of the world calls ctx_create with the same uid
        attncache_status s = comm_init(c, rank, world, uid);
        if (s) {
            attncache_ctx_destroy(c);
            return s;
        }
    }
    *out = c;
    return ATTNCACHE_OK;
}

attncache_status attncache_ctx_info(const attncache_ctx *ctx, int32_t *rank, int32_t *world) {
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_info: ctx is NULL");
    if (rank) *rank = ctx->rank;
    if (world) *world = ctx->world;
    return ATTNCACHE_OK;
}

attncache_status attncache_ctx_set_sm_budget(attncache_ctx *ctx, int32_t compute_sms, int32_t aux_sms) {
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_set_sm_budget: ctx is NULL");
    if (compute_sms < 1 || compute_sms > ctx->sm_count || aux_sms < 1 || aux_sms > ctx->sm_count)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_set_sm_budget: compute_sms %d / aux_sms %d outside [1, %d]",
                    compute_sms, aux_sms, ctx->sm_count);
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->compute_sms = compute_sms;
    ctx->aux_sms = aux_sms;
    return ATTNCACHE_OK;
}

attncache_status attncache_ctx_destroy(attncache_ctx *ctx) {
    if (!ctx) return ATTNCACHE_OK;
    DeviceGuard g(ctx->device);
    cudaDeviceSynchronize();
    comm_destroy(ctx);
    cudaFree(ctx->d_error);
    cudaFree(ctx->d_small);
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    for (auto &kv : ctx->scratch)
        for (auto &sc : kv.second.s)
            if (sc.ptr) cudaFree(sc.ptr);
    for (void *p : ctx->graph_owned) cudaFree(p);
    for (int i = 0; i < 3; ++i)
        if (ctx->io_stream[i]) cudaStreamDestroy(ctx->io_stream[i]);
    if (ctx->comm_ev) cudaEventDestroy(ctx->comm_ev);
    delete ctx;
    return ATTNCACHE_OK;
}

attncache_status attncache_ctx_sync(attncache_ctx *ctx) {
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "ctx_sync: ctx is NULL");
    DeviceGuard g(ctx->device);
    // the last collective work first, polling the communicator's async error (a dead peer would otherwise
    // leave cudaDeviceSynchronize waiting forever)
    attncache_status s = comm_wait(ctx, nullptr, true);
    if (s) return s;
    AC_CUDA(cudaDeviceSynchronize());
    if ((s = comm_check(ctx))) return s;
    int flags = 0;
    AC_CUDA(cudaMemcpy(&flags, ctx->d_error, sizeof(int), cudaMemcpyDeviceToHost));
    if (flags) {
        AC_CUDA(cudaMemset(ctx->d_error, 0, sizeof(int)));
        if (flags & 1) return fail(ATTNCACHE_ERR_NOT_FOUND, "apply_cached: an index outside this shard was skipped");
    }
    return ATTNCACHE_OK;
}

// ---- database -------------------------------------------------------------------------------

attncache_status attncache_db_load(attncache_ctx *ctx, const attncache_db_desc *d, attncache_db **out) {
    if (!ctx || !d || !out) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: NULL argument");
    *out = nullptr;
    if (d->n_global < 0 || d->shard_begin < 0 || d->shard_count < 0 || d->shard_begin + d->shard_count > d->n_global)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: shard [%lld, +%lld) outside [0, %lld)",
                    (long long)d->shard_begin, (long long)d->shard_count, (long long)d->n_global);
    if (d->n_global >= (int64_t)0xFFFFFFFFll)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: n_global must be < 2^32 - 1 (packed keys)");
    if (d->feat_dim <= 0) return fail(ATTNCACHE_ERR_SHAPE, "db_load: feat_dim %d", d->feat_dim);
    if (d->feat_dtype != ATTNCACHE_F32 && d->feat_dtype != ATTNCACHE_BF16)
        return fail(ATTNCACHE_ERR_DTYPE, "db_load: feat_dtype must be F32 or BF16");
    DeviceGuard g(ctx->device);
    if (d->shard_count > 0) {
        if (!d->feats) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: feats is NULL");
        if (!is_device_ptr(d->feats)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: feats is not device memory");
        if (!aligned16(d->feats) || ((int64_t)d->feat_dim * dtype_size(d->feat_dtype)) % 16)
            return fail(ATTNCACHE_ERR_ALIGNMENT, "db_load: feats base / row pitch not 16-byte aligned");
    }
    const bool has_maps = d->n_layers > 0 || d->n_heads > 0 || d->seq_len > 0 || d->maps;
    if (has_maps) {
        if (d->n_layers <= 0 || d->n_heads <= 0 || d->seq_len <= 0)
            return fail(ATTNCACHE_ERR_SHAPE, "db_load: L=%d H=%d S=%d", d->n_layers, d->n_heads, d->seq_len);
        if (d->map_dtype != ATTNCACHE_F16 && d->map_dtype != ATTNCACHE_BF16)
            return fail(ATTNCACHE_ERR_DTYPE, "db_load: map_dtype must be F16 or BF16");
        if (d->map_layout != ATTNCACHE_MAPS_DENSE && d->map_layout != ATTNCACHE_MAPS_PACKED)
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: map_layout %d", d->map_layout);
        if (d->maps_noncausal && d->map_layout == ATTNCACHE_MAPS_PACKED)
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: non-causal maps need the DENSE layout");
        if (d->seq_len % 8)
            return fail(ATTNCACHE_ERR_ALIGNMENT, "db_load: seq_len %d: map rows (S*2 bytes) must be 16-byte aligned",
                        d->seq_len);
        if (d->shard_count > 0) {
            if (!d->maps) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: maps is NULL");
            if (!is_device_ptr(d->maps)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: maps is not device memory");
            if (!aligned16(d->maps)) return fail(ATTNCACHE_ERR_ALIGNMENT, "db_load: maps base not 16-byte aligned");
        }
    }
    attncache_db *db = new attncache_db();
    db->ctx = ctx;
    db->device = ctx->device;
    db->d = *d;
    if (!has_maps) db->d.maps = nullptr;
    attncache_status s = db_load_collective(db);  // COLLECTIVE with a communicator: checks the shard tiling
    if (s) {
        attncache_db_free(db);
        return s;
    }
    *out = db;
    return ATTNCACHE_OK;
}

attncache_status attncache_db_free(attncache_db *db) {
    if (!db) return ATTNCACHE_OK;
    if (db->d_shard_begins) {  // db-local state only: the ctx may already be destroyed
        DeviceGuard g(db->device);
        cudaFree(db->d_shard_begins);
    }
    delete db;
    return ATTNCACHE_OK;
}

// ---- search ---------------------------------------------------------------------------------

}  // extern "C"

attncache_status ac::search_keys_impl(attncache_db *db, const void *queries, int64_t n, uint64_t *keys,
                                      cudaStream_t st) {
    const attncache_db_desc &d = db->d;
    AC_CUDA(cudaMemsetAsync(keys, 0, sizeof(uint64_t) * (size_t)n, st));
    if (d.shard_count == 0 || n == 0) return ATTNCACHE_OK;
    if (search_tc_supported(d.feat_dtype, d.feat_dim)) {
        AC_CUDA(launch_search_tc(queries, d.feats, n, d.shard_count, d.feat_dim, d.shard_begin, keys,
                                 db->ctx->aux_sms, st));
    } else {
        if (d.feat_dim > kSimtMaxLen)
            return fail(ATTNCACHE_ERR_SHAPE, "search: feat_dim %d of dtype %d takes the CUDA-core kernel, which holds "
                        "at most %d elements per query", d.feat_dim, d.feat_dtype, kSimtMaxLen);
        AC_CUDA(launch_search_ffma(d.feat_dtype, queries, d.feats, n, d.shard_count, d.feat_dim, d.shard_begin, keys, st));
    }
    return ATTNCACHE_OK;
}

extern "C" {

static attncache_status check_queries(attncache_db *db, const void *queries, int64_t n) {
    if (!db) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: db is NULL");
    if (n < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: n_queries < 0");
    if (n > 0) {
        if (!queries) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: queries is NULL");
        if (!is_device_ptr(queries)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: queries is not device memory");
        if (!aligned16(queries)) return fail(ATTNCACHE_ERR_ALIGNMENT, "search: queries not 16-byte aligned");
    }
    return ATTNCACHE_OK;
}

attncache_status attncache_search_keys(attncache_db *db, const void *queries, int64_t n, uint64_t *keys, void *stream) {
    AC_NVTX("attncache_search_keys");
    attncache_status s = check_queries(db, queries, n);
    if (s) return s;
    if (n > 0 && !keys) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search_keys: keys is NULL");
    DeviceGuard g(db->ctx->device);
    return search_keys_impl(db, queries, n, keys, (cudaStream_t)stream);
}

attncache_status attncache_keys_decode(const uint64_t *keys, int32_t n_shards, int64_t n, float tau, int64_t *idx,
                                       float *score, uint8_t *hit, void *stream) {
    if (std::isnan(tau)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "keys_decode: tau is NaN");
    if (n < 0 || n_shards <= 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "keys_decode: n=%lld n_shards=%d", (long long)n, n_shards);
    if (n > 0 && (!keys || !idx || !score || !hit)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "keys_decode: NULL output");
    AC_CUDA(launch_keys_decode(keys, n_shards, n, tau, idx, score, hit, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

static attncache_status search_common(attncache_db *db, const void *queries, int64_t n, float tau, int64_t *idx,
                                      float *score, uint8_t *hit, bool all, void *stream) {
    AC_NVTX("attncache_search");
    attncache_status s = check_queries(db, queries, n);
    if (s) return s;
    if (std::isnan(tau)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: tau is NaN");
    if (db->d.n_global == 0) return fail(ATTNCACHE_ERR_EMPTY, "search: the database has no entries");
    if (db->ctx->comm_failed) return comm_failed_status();
    DeviceGuard g(db->ctx->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (db->ctx->comm) {  // COLLECTIVE: C1 query all-gather, K1, C2 key max-all-reduce, K2
        if (n > 0 && !all && (!idx || !score || !hit)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: NULL output");
        return search_collective(db, queries, n, tau, all, idx, score, hit, st);
    }
    if (db->d.shard_count != db->d.n_global)
        return fail(ATTNCACHE_ERR_STATE, "search: this db is one shard of %lld and the ctx has no communicator; use "
                    "search_keys + keys_decode, or a ctx created with rank/world/uid", (long long)db->d.n_global);
    if (n == 0) return ATTNCACHE_OK;
    if (!idx || !score || !hit) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search: NULL output");
    if (search_tc_supported(db->d.feat_dtype, db->d.feat_dim)) {
        // K1 with K2 fused: the search kernel's last CTA to finish applies the gate and re-zeroes the keys for the
        // next call (no memset and no decode launch per call; a fresh buffer is zeroed once)
        void *buf = nullptr;
        bool fresh = false;
        if ((s = scratch(db->ctx, st, kScSearchFused, 16 + sizeof(uint64_t) * (size_t)n, &buf, &fresh))) return s;
        if (fresh) AC_CUDA(cudaMemsetAsync(buf, 0, 16 + sizeof(uint64_t) * (size_t)n, st));
        const SearchDecode dec{idx, score, hit, tau, (unsigned int *)buf};
        AC_CUDA(launch_search_tc(queries, db->d.feats, n, db->d.shard_count, db->d.feat_dim, db->d.shard_begin,
                                 (uint64_t *)((char *)buf + 16), db->ctx->aux_sms, st, &dec));
        return ATTNCACHE_OK;
    }
    void *keys = nullptr;
    if ((s = scratch(db->ctx, st, kScSearchKeys, sizeof(uint64_t) * (size_t)n, &keys))) return s;
    if ((s = search_keys_impl(db, queries, n, (uint64_t *)keys, st))) return s;
    AC_CUDA(launch_keys_decode((const uint64_t *)keys, 1, n, tau, idx, score, hit, st));
    return ATTNCACHE_OK;
}

attncache_status attncache_search(attncache_db *db, const void *queries, int64_t n, float tau, int64_t *idx,
                                  float *score, uint8_t *hit, void *stream) {
    return search_common(db, queries, n, tau, idx, score, hit, false, stream);
}

attncache_status attncache_search_all(attncache_db *db, const void *queries, int64_t n, float tau, int64_t *idx,
                                      float *score, uint8_t *hit, void *stream) {
    if (n > 0 && (!idx || !score || !hit)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "search_all: NULL output");
    return search_common(db, queries, n, tau, idx, score, hit, true, stream);
}

// ---- apply ----------------------------------------------------------------------------------

#if defined(SM_EXPERIMENT)  // experiment: per-call CTA counts from the environment
static int sm_override(const char *name, int def) {
    const char *v = getenv(name);
    return v && atoi(v) > 0 ? atoi(v) : def;
}
#else
static inline int sm_override(const char *, int def) { return def; }
#endif

static attncache_status apply_check(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                    int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t n_kv_heads,
                                    int32_t act_dtype, const void *V, void *O) {
    if (!db) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: db is NULL");
    const attncache_db_desc &d = db->d;
    if (d.n_layers <= 0) return fail(ATTNCACHE_ERR_STATE, "apply_cached: this database holds no maps");
    if (n_kv_heads <= 0 || d.n_heads % n_kv_heads)
        return fail(ATTNCACHE_ERR_SHAPE, "apply_cached: n_kv_heads %d does not divide n_heads %d", n_kv_heads, d.n_heads);
    if (n_rows < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: n_rows < 0");
    if (layer_begin < 0 || layer_end > d.n_layers || layer_begin >= layer_end)
        return fail(ATTNCACHE_ERR_SHAPE, "apply_cached: layers [%d, %d) outside [0, %d)", layer_begin, layer_end, d.n_layers);
    if (head_dim <= 0) return fail(ATTNCACHE_ERR_SHAPE, "apply_cached: head_dim %d", head_dim);
    if (!dtype_valid(act_dtype)) return fail(ATTNCACHE_ERR_DTYPE, "apply_cached: act_dtype %d", act_dtype);
    if (!(act_dtype == ATTNCACHE_F32 || act_dtype == d.map_dtype))
        return fail(ATTNCACHE_ERR_DTYPE, "apply_cached: act_dtype must equal the map dtype or be F32");
    if (n_rows == 0) return ATTNCACHE_OK;
    if (!idx || !V || !O) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: NULL idx/V/O");
    if (!is_device_ptr(idx) || !is_device_ptr(V) || !is_device_ptr(O) || (hit && !is_device_ptr(hit)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: idx/hit/V/O must be device memory");
    if (!aligned16(V) || !aligned16(O) || ((int64_t)head_dim * dtype_size(act_dtype)) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "apply_cached: V/O base or row pitch (head_dim*elem) not 16-byte aligned");
    return ATTNCACHE_OK;
}

}  // extern "C"

attncache_status ac::apply_local_impl(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                      int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t n_kv_heads,
                                      int32_t act_dtype, const void *V, void *O, cudaStream_t st) {
    attncache_status s = apply_check(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, V, O);
    if (s || n_rows == 0) return s;
    const attncache_db_desc &d = db->d;
    DeviceGuard g(db->ctx->device);
    void *list = nullptr;
    if ((s = scratch(db->ctx, st, kScApplyList, rowlist_bytes(n_rows), &list))) return s;
    ApplyArgs a;
    a.maps = d.maps;
    a.L = d.n_layers;
    a.H = d.n_heads;
    a.S = d.seq_len;
    a.d = head_dim;
    a.layer_begin = layer_begin;
    a.n_lay = layer_end - layer_begin;
    a.map_dt = d.map_dtype;
    a.act_dt = act_dtype;
    a.map_layout = d.map_layout;
    a.map_stride = map_elems(d.seq_len, d.map_layout);
    a.causal = d.maps_noncausal ? 0 : 1;
    a.Hkv = n_kv_heads;
    a.V = V;
    a.O = O;
    a.list = rowlist_view(list, n_rows);
    a.max_rows = n_rows;
    if (apply_tc_fused_select(a, n_rows) && fused_select_ok(db->ctx)) {
        // the A.V kernel selects the rows in its prologue (one launch fewer; the same order-preserving list)
        a.sel.idx = idx;
        a.sel.mask = hit;
        a.sel.n = n_rows;
        a.sel.shard_begin = d.shard_begin;
        a.sel.shard_count = d.shard_count;
        a.sel.err = db->ctx->d_error;
        AC_CUDA(launch_apply_tc(a, sm_override("AC_APPLY_SMS", db->ctx->compute_sms), st));
        return ATTNCACHE_OK;
    }
    AC_CUDA(launch_select_apply(idx, hit, n_rows, d.shard_begin, d.shard_count, a.list, db->ctx->d_error, st));
    if (apply_tc_supported(d.map_dtype, act_dtype, d.seq_len, head_dim)) {
        AC_CUDA(launch_apply_tc(a, sm_override("AC_APPLY_SMS", db->ctx->compute_sms), st));
    } else {
        AC_CUDA(launch_apply_ffma(a, db->ctx->compute_sms, st));
    }
    return ATTNCACHE_OK;
}

extern "C" {

attncache_status attncache_apply_cached_local(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                              int32_t layer_begin, int32_t layer_end, int32_t head_dim,
                                              int32_t n_kv_heads, int32_t act_dtype, const void *V, void *O,
                                              void *stream) {
    AC_NVTX("attncache_apply_cached_local");
    return apply_local_impl(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, V, O,
                            (cudaStream_t)stream);
}

attncache_status attncache_apply_cached_gqa(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                            int32_t layer_begin, int32_t layer_end, int32_t head_dim,
                                            int32_t n_kv_heads, int32_t act_dtype, const void *V, void *O,
                                            void *stream) {
    AC_NVTX("attncache_apply_cached");
    attncache_status s = apply_check(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, V, O);
    if (s) return s;
    attncache_ctx *ctx = db->ctx;
    if (ctx->comm_failed) return comm_failed_status();
    if (ctx->comm && (ctx->world > 1 || ctx->force_route)) {  // COLLECTIVE: route hits to the owner and O back
        if (n_rows && hit && !is_device_ptr(hit))
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: hit must be device memory");
        DeviceGuard g(ctx->device);
        return apply_routed(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, V, O,
                            (cudaStream_t)stream);
    }
    return apply_local_impl(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, V, O,
                            (cudaStream_t)stream);
}

attncache_status attncache_apply_cached(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_rows,
                                        int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t act_dtype,
                                        const void *V, void *O, void *stream) {
    if (!db) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "apply_cached: db is NULL");
    return attncache_apply_cached_gqa(db, idx, hit, n_rows, layer_begin, layer_end, head_dim, db->d.n_heads, act_dtype,
                                      V, O, stream);
}

// ---- attend ---------------------------------------------------------------------------------

attncache_status attncache_attend_full(attncache_ctx *ctx, int64_t batch, int32_t L, int32_t H, int32_t S, int32_t dd,
                                       int32_t act_dtype, const void *Q, const void *K, const void *V, float scale,
                                       const uint8_t *skip, void *O, void *stream) {
    return attncache_attend_full_gqa(ctx, batch, L, H, H, S, dd, act_dtype, Q, K, V, scale, skip, O, stream);
}

attncache_status attncache_attend_full_gqa(attncache_ctx *ctx, int64_t batch, int32_t L, int32_t H, int32_t n_kv_heads,
                                           int32_t S, int32_t dd, int32_t act_dtype, const void *Q, const void *K,
                                           const void *V, float scale, const uint8_t *skip, void *O, void *stream) {
    AC_NVTX("attncache_attend_full");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "attend_full: ctx is NULL");
    if (H > 0 && (n_kv_heads <= 0 || H % n_kv_heads))
        return fail(ATTNCACHE_ERR_SHAPE, "attend_full: n_kv_heads %d does not divide n_heads %d", n_kv_heads, H);
    if (batch < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "attend_full: batch < 0");
    if (L <= 0 || H <= 0 || S <= 0 || dd <= 0) return fail(ATTNCACHE_ERR_SHAPE, "attend_full: L=%d H=%d S=%d d=%d", L, H, S, dd);
    if (S > 8192) return fail(ATTNCACHE_ERR_SHAPE, "attend_full: seq_len %d > 8192", S);
    if (!dtype_valid(act_dtype)) return fail(ATTNCACHE_ERR_DTYPE, "attend_full: act_dtype %d", act_dtype);
    if (std::isnan(scale)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "attend_full: scale is NaN");
    if (batch == 0) return ATTNCACHE_OK;
    if (!Q || !K || !V || !O) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "attend_full: NULL Q/K/V/O");
    if (!is_device_ptr(Q) || !is_device_ptr(K) || !is_device_ptr(V) || !is_device_ptr(O) || (skip && !is_device_ptr(skip)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "attend_full: Q/K/V/O/skip must be device memory");
    if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O) || ((int64_t)dd * dtype_size(act_dtype)) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "attend_full: base or row pitch (head_dim*elem) not 16-byte aligned");
    if (!attend_tc_supported(act_dtype, S, dd) && S > kSimtMaxLen)
        return fail(ATTNCACHE_ERR_SHAPE, "attend_full: seq_len %d takes the CUDA-core kernel (dtype %d, head_dim %d), "
                    "which holds at most %d keys per row", S, act_dtype, dd, kSimtMaxLen);
    DeviceGuard g(ctx->device);
    cudaStream_t st = (cudaStream_t)stream;
    void *list = nullptr;
    attncache_status s = scratch(ctx, st, kScAttendList, rowlist_bytes(batch), &list);
    if (s) return s;
    AttendArgs a;
    a.L = L;
    a.H = H;
    a.S = S;
    a.d = dd;
    a.dt = act_dtype;
    a.scale = scale > 0.f ? scale : 1.0f / sqrtf((float)dd);
    a.Hkv = n_kv_heads;
    a.Q = Q;
    a.K = K;
    a.V = V;
    a.O = O;
    a.list = rowlist_view(list, batch);
    a.max_rows = batch;
    if (attend_tc_fused_select(a, batch) && fused_select_ok(ctx)) {
        // the attention kernel selects the rows in its prologue (one launch fewer; the same order-preserving list)
        a.sel.mask = skip;
        a.sel.n = batch;
        AC_CUDA(launch_attend_tc(a, sm_override("AC_ATTEND_SMS", ctx->compute_sms), st));
        return ATTNCACHE_OK;
    }
    AC_CUDA(launch_select_attend(skip, batch, a.list, st));
    if (attend_tc_supported(act_dtype, S, dd)) {
        AC_CUDA(launch_attend_tc(a, sm_override("AC_ATTEND_SMS", ctx->compute_sms), st));
    } else {
        AC_CUDA(launch_attend_ffma(a, ctx->compute_sms, st));
    }
    return ATTNCACHE_OK;
}

// ---- feature projector (f2) ---------------------------------------------------------------------

attncache_status attncache_project_features(attncache_ctx *ctx, const void *h, int64_t n, int32_t in_dim,
                                            int32_t act_dtype, const void *W1, const float *b1, int32_t hidden_dim,
                                            const void *W2, const float *b2, int32_t feat_dim, int32_t feat_dtype,
                                            void *features, void *stream) {
    AC_NVTX("attncache_project_features");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: ctx is NULL");
    if (n < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: n < 0");
    if (in_dim <= 0 || hidden_dim <= 0 || feat_dim <= 0)
        return fail(ATTNCACHE_ERR_SHAPE, "project_features: in_dim=%d hidden_dim=%d feat_dim=%d", in_dim, hidden_dim, feat_dim);
    if (!dtype_valid(act_dtype) || !dtype_valid(feat_dtype))
        return fail(ATTNCACHE_ERR_DTYPE, "project_features: act_dtype %d feat_dtype %d", act_dtype, feat_dtype);
    if (!W1 || !b1 || !W2 || !b2) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: NULL weights");
    if (!is_device_ptr(W1) || !is_device_ptr(b1) || !is_device_ptr(W2) || !is_device_ptr(b2))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: weights must be device memory");
    if (n == 0) return ATTNCACHE_OK;
    if (!h || !features) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: NULL h/features");
    if (!is_device_ptr(h) || !is_device_ptr(features))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "project_features: h/features must be device memory");
    const int es = dtype_size(act_dtype);
    if (!aligned16(h) || !aligned16(W1) || !aligned16(W2) || !aligned16(b1) || !aligned16(b2) || !aligned16(features) ||
        ((int64_t)in_dim * es) % 16 || ((int64_t)hidden_dim * es) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "project_features: bases or row pitches (in_dim, hidden_dim) not 16-byte aligned");
    DeviceGuard g(ctx->device);
    // scratch: z [n][Hd] (act dtype) then y [n][D] fp32, 256-byte aligned
    const size_t zb = ((size_t)n * hidden_dim * es + 255) & ~(size_t)255;
    const size_t yb = (size_t)n * feat_dim * 4;
    void *buf = nullptr;
    attncache_status s = scratch(ctx, (cudaStream_t)stream, kScProject, zb + yb, &buf);
    if (s) return s;
    ProjectArgs a;
    a.M = n;
    a.E = in_dim;
    a.Hd = hidden_dim;
    a.D = feat_dim;
    a.dt = act_dtype;
    a.feat_dt = feat_dtype;
    a.h = h;
    a.W1 = W1;
    a.W2 = W2;
    a.b1 = b1;
    a.b2 = b2;
    a.z = buf;
    a.y = (float *)((uint8_t *)buf + zb);
    a.f = features;
    AC_CUDA(launch_project(a, ctx->aux_sms, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

// ---- projection GEMM (f4) ------------------------------------------------------------------------

attncache_status attncache_linear(attncache_ctx *ctx, const void *X, int64_t M, int32_t K, const void *W, int32_t N,
                                  int32_t dtype, const float *bias, int32_t seq_len, int32_t head_dim, void *Y,
                                  void *stream) {
    AC_NVTX("attncache_linear");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "linear: ctx is NULL");
    if (M < 0 || K <= 0 || N <= 0 || seq_len <= 0 || head_dim <= 0)
        return fail(ATTNCACHE_ERR_SHAPE, "linear: M=%lld K=%d N=%d S=%d d=%d", (long long)M, K, N, seq_len, head_dim);
    if (M % seq_len || N % head_dim)
        return fail(ATTNCACHE_ERR_SHAPE, "linear: M=%lld must be whole sequences of %d rows and N=%d whole heads of %d",
                    (long long)M, seq_len, N, head_dim);
    if (!dtype_valid(dtype)) return fail(ATTNCACHE_ERR_DTYPE, "linear: dtype %d", dtype);
    if (M == 0) return ATTNCACHE_OK;
    if (!X || !W || !Y) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "linear: NULL X/W/Y");
    if (!is_device_ptr(X) || !is_device_ptr(W) || !is_device_ptr(Y) || (bias && !is_device_ptr(bias)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "linear: X/W/Y/bias must be device memory");
    const int es = dtype_size(dtype);
    if (!aligned16(X) || !aligned16(W) || !aligned16(Y) || (bias && !aligned16(bias)) || ((int64_t)K * es) % 16 ||
        ((int64_t)head_dim * es) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "linear: bases or rows (K, head_dim elements) not 16-byte aligned");
    DeviceGuard g(ctx->device);
    AC_CUDA(launch_linear_heads(dtype, X, M, K, W, N, bias, seq_len, head_dim, Y, ctx->compute_sms, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

// ---- RoPE (f4) ----------------------------------------------------------------------------------

attncache_status attncache_rope(void *X, int64_t n_units, int32_t S, int32_t d, int32_t dt, float base, void *stream) {
    AC_NVTX("attncache_rope");
    if (n_units < 0 || S <= 0 || d <= 0) return fail(ATTNCACHE_ERR_SHAPE, "rope: n_units=%lld S=%d d=%d", (long long)n_units, S, d);
    if (d % 2) return fail(ATTNCACHE_ERR_SHAPE, "rope: head_dim %d is odd", d);
    if (!dtype_valid(dt)) return fail(ATTNCACHE_ERR_DTYPE, "rope: dtype %d", dt);
    if (!(base > 1.f)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "rope: base must be > 1");
    if (n_units == 0) return ATTNCACHE_OK;
    if (!X || !is_device_ptr(X)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "rope: X must be device memory");
    AC_CUDA(launch_rope(X, n_units, S, d, dt, base, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

// ---- capture (DB building) ------------------------------------------------------------------

attncache_status attncache_capture_maps(attncache_ctx *ctx, int64_t batch, int32_t L, int32_t H, int32_t S, int32_t dd,
                                        int32_t act_dtype, const void *Q, const void *K, float scale,
                                        const uint8_t *skip, int32_t map_dtype, int32_t map_layout, void *maps_out,
                                        void *stream) {
    return attncache_capture_maps_gqa(ctx, batch, L, H, H, S, dd, act_dtype, Q, K, scale, skip, map_dtype, map_layout,
                                      maps_out, stream);
}

attncache_status attncache_capture_maps_gqa(attncache_ctx *ctx, int64_t batch, int32_t L, int32_t H, int32_t n_kv_heads,
                                            int32_t S, int32_t dd, int32_t act_dtype, const void *Q, const void *K,
                                            float scale, const uint8_t *skip, int32_t map_dtype, int32_t map_layout,
                                            void *maps_out, void *stream) {
    AC_NVTX("attncache_capture_maps");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: ctx is NULL");
    if (H > 0 && (n_kv_heads <= 0 || H % n_kv_heads))
        return fail(ATTNCACHE_ERR_SHAPE, "capture_maps: n_kv_heads %d does not divide n_heads %d", n_kv_heads, H);
    if (batch < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: batch < 0");
    if (L <= 0 || H <= 0 || S <= 0 || dd <= 0) return fail(ATTNCACHE_ERR_SHAPE, "capture_maps: L=%d H=%d S=%d d=%d", L, H, S, dd);
    if (S % 8 || S > 8192) return fail(ATTNCACHE_ERR_SHAPE, "capture_maps: seq_len %d (needs S %% 8 == 0, <= 8192)", S);
    if (!dtype_valid(act_dtype)) return fail(ATTNCACHE_ERR_DTYPE, "capture_maps: act_dtype %d", act_dtype);
    if (map_dtype != ATTNCACHE_F16 && map_dtype != ATTNCACHE_BF16)
        return fail(ATTNCACHE_ERR_DTYPE, "capture_maps: map_dtype must be F16 or BF16");
    if (map_layout != ATTNCACHE_MAPS_DENSE && map_layout != ATTNCACHE_MAPS_PACKED)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: map_layout %d", map_layout);
    if (std::isnan(scale)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: scale is NaN");
    if (batch == 0) return ATTNCACHE_OK;
    if (!Q || !K || !maps_out) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: NULL Q/K/maps_out");
    if (!is_device_ptr(Q) || !is_device_ptr(K) || !is_device_ptr(maps_out) || (skip && !is_device_ptr(skip)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "capture_maps: Q/K/maps_out/skip must be device memory");
    if (!aligned16(Q) || !aligned16(K) || !aligned16(maps_out) || ((int64_t)dd * dtype_size(act_dtype)) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "capture_maps: base or row pitch not 16-byte aligned");
    if (!capture_tc_supported(act_dtype, S, dd) && S > kSimtMaxLen)
        return fail(ATTNCACHE_ERR_SHAPE, "capture_maps: seq_len %d takes the CUDA-core kernel (dtype %d, head_dim %d), "
                    "which holds at most %d keys per row", S, act_dtype, dd, kSimtMaxLen);
    DeviceGuard g(ctx->device);
    cudaStream_t st = (cudaStream_t)stream;
    void *list = nullptr;
    attncache_status s = scratch(ctx, st, kScAttendList, rowlist_bytes(batch), &list);
    if (s) return s;
    CaptureArgs a;
    a.L = L;
    a.H = H;
    a.S = S;
    a.d = dd;
    a.dt = act_dtype;
    a.map_dt = map_dtype;
    a.map_layout = map_layout;
    a.map_stride = map_elems(S, map_layout);
    a.scale = scale > 0.f ? scale : 1.0f / sqrtf((float)dd);
    a.Hkv = n_kv_heads;
    a.Q = Q;
    a.K = K;
    a.maps = maps_out;
    a.list = rowlist_view(list, batch);
    a.max_rows = batch;
    AC_CUDA(launch_select_attend(skip, batch, a.list, st));
    if (capture_tc_supported(act_dtype, S, dd)) {
        AC_CUDA(launch_capture_tc(a, ctx->compute_sms, st));
    } else {
        AC_CUDA(launch_capture_simt(a, ctx->compute_sms, st));
    }
    return ATTNCACHE_OK;
}

// ---- routing --------------------------------------------------------------------------------

attncache_status attncache_route_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const int64_t *shard_begins,
                                      int32_t world, int32_t *owner, int32_t *counts, int64_t *order, void *stream) {
    if (n < 0 || world <= 0 || world > 1024) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "route_plan: n=%lld world=%d", (long long)n, world);
    if (!shard_begins || !counts || (n > 0 && (!idx || !hit || !owner || !order)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "route_plan: NULL argument");
    AC_CUDA(launch_route_plan(idx, hit, n, shard_begins, world, owner, counts, order, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

attncache_status attncache_affinity_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const int64_t *sb,
                                         int32_t world, double hit_cost, double miss_cost, int32_t *assign,
                                         double *load) {
    if (n < 0 || world <= 0 || world > 1024)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan: n=%lld world=%d", (long long)n, world);
    if (!sb || (n > 0 && (!idx || !hit || !assign))) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan: NULL argument");
    if (!(hit_cost >= 0.0) || !(miss_cost >= 0.0))  // also rejects NaN
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan: costs must be non-negative numbers");
    for (int r = 0; r < world; ++r)
        if (sb[r + 1] < sb[r]) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan: shard_begins decreasing at %d", r);
    double acc[1024];
    for (int r = 0; r < world; ++r) acc[r] = 0.0;
    // hits: the owner of the entry (its maps are local there)
    for (int64_t b = 0; b < n; ++b) {
        if (!hit[b]) continue;
        const int64_t e = idx[b];
        if (e < sb[0] || e >= sb[world])
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan: hit row %lld has idx %lld outside [%lld, %lld)",
                        (long long)b, (long long)e, (long long)sb[0], (long long)sb[world]);
        int lo = 0, hi = world - 1;  // the last r with sb[r] <= e (binary search; empty shards skipped)
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (sb[mid] <= e) lo = mid; else hi = mid - 1;
        }
        assign[b] = lo;
        acc[lo] += hit_cost;
    }
    // misses: ascending b, each on the least-loaded rank (lowest rank on ties)
    for (int64_t b = 0; b < n; ++b) {
        if (hit[b]) continue;
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (acc[r] < acc[best]) best = r;
        assign[b] = best;
        acc[best] += miss_cost;
    }
    if (load)
        for (int r = 0; r < world; ++r) load[r] = acc[r];
    return ATTNCACHE_OK;
}

attncache_status attncache_affinity_plan_device(attncache_ctx *ctx, const int64_t *idx, const uint8_t *hit, int64_t n,
                                                const int64_t *sb, int32_t world, double hit_cost, double miss_cost,
                                                int32_t rank, const int64_t *hb, int32_t *assign, double *load,
                                                int64_t *loc, int64_t *idx_loc, uint8_t *hit_loc, int64_t *send_order,
                                                int32_t *counts, void *stream) {
    AC_NVTX("attncache_affinity_plan_device");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: ctx is NULL");
    if (n < 0 || world <= 0 || world > ac::kPlanMaxWorld || rank < 0 || rank >= world)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: n=%lld world=%d rank=%d (world <= %d)",
                    (long long)n, world, rank, ac::kPlanMaxWorld);
    if (!sb || !hb || !load || !counts || (n > 0 && (!idx || !hit || !assign || !loc || !idx_loc || !hit_loc || !send_order)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: NULL argument");
    if (!(hit_cost >= 0.0) || !(miss_cost >= 0.0))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: costs must be non-negative numbers");
    if (hb[0] != 0 || hb[world] != n)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: home_begins must span [0, n_rows]");
    for (int r = 0; r < world; ++r)
        if (sb[r + 1] < sb[r] || hb[r + 1] < hb[r])
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "affinity_plan_device: begins decreasing at %d", r);
    DeviceGuard g(ctx->device);
    void *buf = nullptr;
    attncache_status s = scratch(ctx, (cudaStream_t)stream, kScPlan, (size_t)std::max<int64_t>(n, 1) * sizeof(int64_t), &buf);
    if (s) return s;
    ac::PlanArgs a;
    a.world = world;
    a.rank = rank;
    a.hit_cost = hit_cost;
    a.miss_cost = miss_cost;
    for (int r = 0; r <= world; ++r) {
        a.shard_begins[r] = sb[r];
        a.home_begins[r] = hb[r];
    }
    AC_CUDA(ac::launch_affinity_plan(idx, hit, n, a, assign, load, (int64_t *)buf, loc, idx_loc, hit_loc,
                                     send_order, counts, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

static attncache_status copy_rows(const void *src, const int64_t *rows, int64_t n, int64_t row_bytes, void *dst,
                                  bool gather, void *stream) {
    if (n < 0 || row_bytes <= 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "copy_rows: n=%lld row_bytes=%lld", (long long)n, (long long)row_bytes);
    if (n == 0) return ATTNCACHE_OK;
    if (!src || !rows || !dst) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "copy_rows: NULL argument");
    const bool ok16 = row_bytes % 16 == 0 && aligned16(src) && aligned16(dst);
    const bool ok8 = row_bytes % 8 == 0 && ((uintptr_t)src & 7) == 0 && ((uintptr_t)dst & 7) == 0;
    if (!ok16 && !ok8) return fail(ATTNCACHE_ERR_ALIGNMENT, "copy_rows: rows and bases must be 8-byte multiples/aligned");
    AC_CUDA(launch_copy_rows(src, rows, n, row_bytes, dst, gather, ok16, 148, (cudaStream_t)stream));  // no ctx: B200
    return ATTNCACHE_OK;
}

attncache_status attncache_gather_rows(const void *src, const int64_t *rows, int64_t n, int64_t row_bytes, void *dst,
                                       void *stream) {
    return copy_rows(src, rows, n, row_bytes, dst, true, stream);
}

attncache_status attncache_scatter_rows(const void *src, const int64_t *rows, int64_t n, int64_t row_bytes, void *dst,
                                        void *stream) {
    return copy_rows(src, rows, n, row_bytes, dst, false, stream);
}

// ---- fetch (debug: literal AttnMapsDB.get) ---------------------------------------------------

attncache_status attncache_fetch_maps(attncache_db *db, int64_t idx, int32_t layer_begin, int32_t layer_end, void *out,
                                      void *stream) {
    if (!db || !out) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "fetch_maps: NULL argument");
    const attncache_db_desc &d = db->d;
    if (d.n_layers <= 0) return fail(ATTNCACHE_ERR_STATE, "fetch_maps: this database holds no maps");
    if (idx < d.shard_begin || idx >= d.shard_begin + d.shard_count)
        return fail(ATTNCACHE_ERR_NOT_FOUND, "fetch_maps: index %lld not in this shard", (long long)idx);
    if (layer_begin < 0 || layer_end > d.n_layers || layer_begin >= layer_end)
        return fail(ATTNCACHE_ERR_SHAPE, "fetch_maps: layers [%d, %d)", layer_begin, layer_end);
    const int64_t maps_per_layer = d.n_heads;
    const int64_t stride = map_elems(d.seq_len, d.map_layout);
    const uint16_t *src = (const uint16_t *)d.maps +
                          ((idx - d.shard_begin) * d.n_layers + layer_begin) * maps_per_layer * stride;
    const int64_t n_maps = maps_per_layer * (layer_end - layer_begin);
    DeviceGuard g(db->ctx->device);
    if (d.map_layout == ATTNCACHE_MAPS_DENSE) {
        AC_CUDA(cudaMemcpyAsync(out, src, (size_t)n_maps * stride * 2, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    } else {
        AC_CUDA(launch_pack_maps(out, n_maps, d.seq_len, const_cast<uint16_t *>(src), /*unpack=*/true,
                                 (cudaStream_t)stream));
    }
    return ATTNCACHE_OK;
}

// ---- DB building: packed layout --------------------------------------------------------------

int64_t attncache_packed_map_elems(int32_t seq_len) {
    return (seq_len > 0 && seq_len % 8 == 0) ? packed_row_off(seq_len) : 0;
}

attncache_status attncache_pack_maps(const void *dense, int64_t n_maps, int32_t S, void *packed, void *stream) {
    if (n_maps < 0 || S <= 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "pack_maps: n_maps=%lld S=%d", (long long)n_maps, S);
    if (S % 8) return fail(ATTNCACHE_ERR_SHAPE, "pack_maps: seq_len %d is not a multiple of 8", S);
    if (n_maps == 0) return ATTNCACHE_OK;
    if (!dense || !packed) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "pack_maps: NULL argument");
    if (!aligned16(dense) || !aligned16(packed)) return fail(ATTNCACHE_ERR_ALIGNMENT, "pack_maps: 16-byte alignment");
    AC_CUDA(launch_pack_maps(dense, n_maps, S, packed, /*unpack=*/false, (cudaStream_t)stream));
    return ATTNCACHE_OK;
}

}  // extern "C"
