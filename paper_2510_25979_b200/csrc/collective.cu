// collective.cu — the multi-GPU half of the C ABI: a library-owned NCCL communicator per ctx and the
// collective calls of include/attncache.h (north_star: "the (score, index) pairs are reduced with an NCCL
// allgather over NVLink.  Hit queries are then routed to the owning GPU, whose A.V output returns to the
// query's home GPU by NCCL send/recv").
//
// NCCL is reached through dlopen (the library keeps no link-time dependency on libnccl or libcuda, so it
// loads on a GPU-less host): ATTNCACHE_NCCL_LIB when set, else the copy already in the process (e.g. the one
// torch loaded), else libnccl.so.2 from the loader path.  Every collective is
// enqueued on the caller's stream; the only host round trips are the documented ones (count exchanges).
#include <dlfcn.h>
#include <stdio.h>
#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <numeric>
#include <thread>

#include "abi_internal.cuh"

namespace ac {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    ncclResult_t (*GetVersion)(int *);
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;  // optional: CommDestroy stands in when absent
    bool ok = false;
    char why[256] = "";
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
    void *h = nullptr;
    const char *env = getenv("ATTNCACHE_NCCL_LIB");  // an explicit choice wins (e.g. the tests' fake_nccl)
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch (or another user) loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
        snprintf(g_nccl.why, sizeof g_nccl.why, "dlopen(libnccl.so.2) failed: %s", dlerror());
        return;
    }
#define AC_SYM(field, name)                                                                  \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));                  \
    if (!g_nccl.field) {                                                                     \
        snprintf(g_nccl.why, sizeof g_nccl.why, "libnccl.so.2 has no symbol %s", name);       \
        return;                                                                              \
    }
    AC_SYM(GetUniqueId, "ncclGetUniqueId")
    AC_SYM(CommInitRank, "ncclCommInitRank")
    AC_SYM(CommDestroy, "ncclCommDestroy")
    AC_SYM(AllGather, "ncclAllGather")
    AC_SYM(AllReduce, "ncclAllReduce")
    AC_SYM(Send, "ncclSend")
    AC_SYM(Recv, "ncclRecv")
    AC_SYM(GroupStart, "ncclGroupStart")
    AC_SYM(GroupEnd, "ncclGroupEnd")
    AC_SYM(GetErrorString, "ncclGetErrorString")
    AC_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
    AC_SYM(GetVersion, "ncclGetVersion")
#undef AC_SYM
    g_nccl.CommAbort = reinterpret_cast<decltype(g_nccl.CommAbort)>(dlsym(h, "ncclCommAbort"));
    g_nccl.ok = true;
}

const NcclApi *nccl() {
    std::call_once(g_nccl_once, load_nccl);
    return g_nccl.ok ? &g_nccl : nullptr;
}

attncache_status nccl_status(ncclResult_t r, const char *what) {
    return fail(ATTNCACHE_ERR_NCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "NCCL error");
}

#define AC_NCCL(call)                                                   \
    do {                                                                \
        ncclResult_t r_ = (call);                                       \
        if (r_ != ncclSuccess) return ::ac::nccl_status(r_, #call);     \
    } while (0)

inline ncclComm_t comm_of(const attncache_ctx *ctx) { return (ncclComm_t)ctx->comm; }

// Records the completion of the NCCL work just enqueued on `st` (attncache_ctx_sync polls it; see comm_wait).
attncache_status comm_mark(attncache_ctx *ctx, cudaStream_t st) {
    if (!ctx->comm_ev) AC_CUDA(cudaEventCreateWithFlags(&ctx->comm_ev, cudaEventDisableTiming));
    AC_CUDA(cudaEventRecord(ctx->comm_ev, st));
    ctx->comm_ev_pending = true;
    return ATTNCACHE_OK;
}

}  // namespace

// Host wait for the collective work on `st` (or, st == nullptr, for the last marked one) that polls the
// communicator's asynchronous error while it waits: a peer that died leaves NCCL's kernels waiting forever, and
// NCCL reports it only through ncclCommGetAsyncError.  On such an error comm_check aborts the
// communicator, which also releases the waiting kernels, and the wait returns ATTNCACHE_ERR_NCCL.
attncache_status comm_wait(attncache_ctx *ctx, cudaStream_t st, bool marked_only) {
    if (!ctx->comm) {
        if (!marked_only) AC_CUDA(cudaStreamSynchronize(st));
        return ATTNCACHE_OK;
    }
    if (marked_only) {
        if (!ctx->comm_ev_pending) return ATTNCACHE_OK;
    } else {
        attncache_status s = comm_mark(ctx, st);
        if (s) return s;
    }
    for (;;) {
        const cudaError_t q = cudaEventQuery(ctx->comm_ev);
        if (q == cudaSuccess) break;
        if (q != cudaErrorNotReady) AC_CUDA(q);
        attncache_status s = comm_check(ctx);
        if (s) return s;
        std::this_thread::yield();
    }
    ctx->comm_ev_pending = false;
    return ATTNCACHE_OK;
}

namespace {

// Rows of `row_bytes` bytes from every rank to every rank: rank r sends send_n[p] rows starting at row
// send_off[p] of `send` to peer p, and receives recv_n[p] rows from p at row recv_off[p] of `recv` (one NCCL
// group of send/recv pairs; moved as bytes, so any dtype).
attncache_status exchange_rows(attncache_ctx *ctx, const void *send, const int64_t *send_n, const int64_t *send_off,
                               void *recv, const int64_t *recv_n, const int64_t *recv_off, size_t row_bytes,
                               cudaStream_t st) {
    const NcclApi *N = nccl();
    AC_NCCL(N->GroupStart());
    for (int p = 0; p < ctx->world; ++p) {
        if (send_n[p])
            AC_NCCL(N->Send((const uint8_t *)send + send_off[p] * row_bytes, (size_t)send_n[p] * row_bytes, ncclUint8, p,
                            comm_of(ctx), st));
        if (recv_n[p])
            AC_NCCL(N->Recv((uint8_t *)recv + recv_off[p] * row_bytes, (size_t)recv_n[p] * row_bytes, ncclUint8, p,
                            comm_of(ctx), st));
    }
    AC_NCCL(N->GroupEnd());
    return comm_mark(ctx, st);
}

// The home batch size of every rank: the declared layout, or one all-gather of the int64 counts and a host
// sync (documented in include/attncache.h).
attncache_status home_counts(attncache_ctx *ctx, int64_t n_home, cudaStream_t st, std::vector<int64_t> &out) {
    if (!ctx->layout.empty()) {
        if (ctx->layout[ctx->rank] != n_home)
            return fail(ATTNCACHE_ERR_STATE, "batch layout declares %lld home rows for rank %d, the call passes %lld",
                        (long long)ctx->layout[ctx->rank], ctx->rank, (long long)n_home);
        out = ctx->layout;
        return ATTNCACHE_OK;
    }
    const NcclApi *N = nccl();
    ctx->h_pinned[0] = n_home;
    AC_CUDA(cudaMemcpyAsync(ctx->d_small, ctx->h_pinned, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    AC_NCCL(N->AllGather(ctx->d_small, ctx->d_small + 8, 1, ncclInt64, comm_of(ctx), st));
    if (attncache_status s = comm_mark(ctx, st)) return s;
    AC_CUDA(cudaMemcpyAsync(ctx->h_pinned + 8, ctx->d_small + 8, sizeof(int64_t) * ctx->world, cudaMemcpyDeviceToHost,
                            st));
    if (attncache_status s = comm_wait(ctx, st, false)) return s;
    out.assign(ctx->h_pinned + 8, ctx->h_pinned + 8 + ctx->world);
    return ATTNCACHE_OK;
}

}  // namespace

attncache_status comm_init(attncache_ctx *ctx, int rank, int world, const uint8_t uid[128]) {
    const NcclApi *N = nccl();
    if (!N) return fail(ATTNCACHE_ERR_NCCL, "ctx_create: %s", g_nccl.why);
    ncclUniqueId id;
    memcpy(id.internal, uid, sizeof id.internal);
    ncclComm_t c = nullptr;
    AC_NCCL(N->CommInitRank(&c, world, id, rank));
    ctx->comm = c;
    ctx->rank = rank;
    ctx->world = world;
    return ATTNCACHE_OK;
}

void comm_destroy(attncache_ctx *ctx) {
    if (ctx->comm && nccl()) nccl()->CommDestroy(comm_of(ctx));
    ctx->comm = nullptr;
}

// Polls the communicator's asynchronous error (SURVEY.md §5 failure detection).  On an error the communicator is
// aborted (ncclCommAbort: no barrier with peers that may be gone) and the ctx is marked so that every later
// collective call fails with ATTNCACHE_ERR_NCCL instead of waiting on a dead communicator.
attncache_status comm_check(attncache_ctx *ctx) {
    if (ctx->comm_failed) return comm_failed_status();
    if (!ctx->comm) return ATTNCACHE_OK;
    ncclResult_t r = ncclSuccess;
    AC_NCCL(nccl()->CommGetAsyncError(comm_of(ctx), &r));
    if (r != ncclSuccess && r != ncclInProgress) {
        const NcclApi *N = nccl();
        (N->CommAbort ? N->CommAbort : N->CommDestroy)(comm_of(ctx));
        ctx->comm = nullptr;
        ctx->comm_failed = true;
        return nccl_status(r, "asynchronous NCCL error (the communicator was aborted)");
    }
    return ATTNCACHE_OK;
}

attncache_status comm_failed_status() {
    return fail(ATTNCACHE_ERR_NCCL, "the ctx's NCCL communicator was aborted after an asynchronous error; destroy "
                "the ctx and create a new one");
}

// Collective db_load check: every rank's descriptor agrees on the global fields and the shards tile
// [0, n_global) contiguously in rank order ("partitioned by contiguous entry ranges").
attncache_status db_load_collective(attncache_db *db) {
    attncache_ctx *ctx = db->ctx;
    if (ctx->comm_failed) return comm_failed_status();
    const int w = ctx->world;
    const attncache_db_desc &d = db->d;
    db->shard_begins.assign(w + 1, 0);
    if (ctx->comm) {
        constexpr int kF = 12;
        if ((w + 1) * kF + 8 > kPinnedInts) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: world too large");
        int64_t mine[kF] = {d.n_global, d.shard_begin, d.shard_count, d.feat_dim, d.feat_dtype, d.n_layers,
                            d.n_heads, d.seq_len, d.map_dtype, d.map_layout, d.maps_noncausal, d.maps ? 1 : 0};
        memcpy(ctx->h_pinned, mine, sizeof mine);
        cudaStream_t st = 0;
        AC_CUDA(cudaMemcpyAsync(ctx->d_small, ctx->h_pinned, sizeof mine, cudaMemcpyHostToDevice, st));
        AC_NCCL(nccl()->AllGather(ctx->d_small, ctx->d_small + kF, kF, ncclInt64, comm_of(ctx), st));
        if (attncache_status s = comm_mark(ctx, st)) return s;
        AC_CUDA(cudaMemcpyAsync(ctx->h_pinned + kF, ctx->d_small + kF, sizeof(int64_t) * kF * w, cudaMemcpyDeviceToHost, st));
        if (attncache_status s = comm_wait(ctx, st, false)) return s;
        int64_t next = 0;
        for (int r = 0; r < w; ++r) {
            const int64_t *f = ctx->h_pinned + kF * (r + 1);
            for (int k : {0, 3, 4, 5, 6, 7, 8, 9, 10})
                if (f[k] != mine[k])
                    return fail(ATTNCACHE_ERR_SHAPE, "db_load: rank %d disagrees with rank %d on descriptor field %d",
                                r, ctx->rank, k);
            if (f[1] != next)
                return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: rank %d's shard begins at %lld, expected %lld "
                            "(shards must tile [0, n_global) in rank order)", r, (long long)f[1], (long long)next);
            db->shard_begins[r] = f[1];
            next = f[1] + f[2];
        }
        if (next != d.n_global)
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "db_load: shards cover [0, %lld) of n_global %lld", (long long)next,
                        (long long)d.n_global);
        db->shard_begins[w] = next;
    } else {
        db->shard_begins = {0, d.n_global};
        if (d.shard_begin != 0 || d.shard_count != d.n_global) db->shard_begins = {d.shard_begin, d.shard_begin + d.shard_count};
    }
    AC_CUDA(cudaMalloc(&db->d_shard_begins, sizeof(int64_t) * db->shard_begins.size()));
    AC_CUDA(cudaMemcpy(db->d_shard_begins, db->shard_begins.data(), sizeof(int64_t) * db->shard_begins.size(),
                       cudaMemcpyHostToDevice));
    return ATTNCACHE_OK;
}

// C1 + K1 + C2 + K2 (Alg. 1 l.255-257 over a sharded DB).  Decodes rows [out_begin, out_begin + out_n) of
// the global batch into idx/score/hit.
attncache_status search_collective(attncache_db *db, const void *q, int64_t n_home, float tau, bool all,
                                   int64_t *idx, float *score, uint8_t *hit, cudaStream_t st) {
    attncache_ctx *ctx = db->ctx;
    const NcclApi *N = nccl();
    std::vector<int64_t> cnt;
    attncache_status s = home_counts(ctx, n_home, st, cnt);
    if (s) return s;
    const int w = ctx->world;
    std::vector<int64_t> off(w + 1, 0);
    for (int r = 0; r < w; ++r) off[r + 1] = off[r] + cnt[r];
    const int64_t total = off[w];
    if (total == 0) return ATTNCACHE_OK;
    const size_t row = (size_t)db->d.feat_dim * dtype_size(db->d.feat_dtype);
    void *q_all = nullptr, *keys = nullptr;
    if ((s = scratch(ctx, st, kScQueries, row * (size_t)total, &q_all))) return s;
    if ((s = scratch(ctx, st, kScSearchKeys, sizeof(uint64_t) * (size_t)total, &keys))) return s;
    // C1: the query batch on every rank (all-gather when the home blocks are equal, else send/recv pairs)
    bool equal = true;
    for (int r = 1; r < w; ++r) equal = equal && cnt[r] == cnt[0];
    if (equal) {
        AC_NCCL(N->AllGather(q, q_all, row * (size_t)n_home, ncclUint8, comm_of(ctx), st));
        if (attncache_status s = comm_mark(ctx, st)) return s;
    } else {
        std::vector<int64_t> sn(w, n_home), so(w, 0);
        if ((s = exchange_rows(ctx, q, sn.data(), so.data(), q_all, cnt.data(), off.data(), row, st))) return s;
    }
    // K1: this shard's top-1 key of every query
    if ((s = search_keys_impl(db, q_all, total, (uint64_t *)keys, st))) return s;
    // C2: max over shards of the packed keys = the global top-1 with the lowest-index tie-break (reading R3)
    AC_NCCL(N->AllReduce(keys, keys, (size_t)total, ncclUint64, ncclMax, comm_of(ctx), st));
    if (attncache_status s = comm_mark(ctx, st)) return s;
    // K2: decode + tau gate (the home block, or the whole batch)
    const int64_t b0 = all ? 0 : off[ctx->rank], n = all ? total : n_home;
    if (n) AC_CUDA(launch_keys_decode((const uint64_t *)keys + b0, 1, n, tau, idx, score, hit, st));
    return ATTNCACHE_OK;
}

// a5-a7: route the home hits to the owner of their entry, A.V there, O back home (Alg. 2 l.373-375 with the
// maps read in place on the owner; north_star's routing).  Misses' O rows are untouched.
attncache_status apply_routed(attncache_db *db, const int64_t *idx, const uint8_t *hit, int64_t n_home,
                              int32_t layer_begin, int32_t layer_end, int32_t head_dim, int32_t n_kv_heads,
                              int32_t act_dtype, const void *V, void *O, cudaStream_t st) {
    attncache_ctx *ctx = db->ctx;
    const NcclApi *N = nccl();
    const int w = ctx->world;
    const attncache_db_desc &d = db->d;
    const int64_t n_lay = layer_end - layer_begin;
    const int es = dtype_size(act_dtype);
    const size_t row_v = (size_t)n_lay * n_kv_heads * d.seq_len * head_dim * es;
    const size_t row_o = (size_t)n_lay * d.n_heads * d.seq_len * head_dim * es;
    // K3: owners, per-owner counts and the home hit rows grouped by owner
    void *route = nullptr;
    const size_t nh = (size_t)std::max<int64_t>(n_home, 1);
    attncache_status s = scratch(ctx, st, kScRoute, nh * (4 + 8 + 8) + 256, &route);
    if (s) return s;
    int32_t *owner = (int32_t *)route;
    int64_t *order = (int64_t *)((uint8_t *)route + ((nh * 4 + 15) & ~(size_t)15));
    int64_t *idx_send = order + nh;
    // int32 [world] send counts | [world] receive counts, in a region of the small staging buffers that the
    // count exchange of home_counts (elements [0, 8 + world)) never touches
    int32_t *counts = (int32_t *)(ctx->d_small + kPinnedInts / 2);
    if (n_home) {
        AC_CUDA(launch_route_plan(idx, hit, n_home, db->d_shard_begins, w, owner, counts, order, st));
    } else {
        AC_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * w, st));
    }
    // C3: per-peer counts (one int32 to and from every rank), then one host round trip sizes the transfers
    int32_t *recv_counts = counts + w;
    AC_NCCL(N->GroupStart());
    for (int p = 0; p < w; ++p) {
        AC_NCCL(N->Send(counts + p, 1, ncclInt32, p, comm_of(ctx), st));
        AC_NCCL(N->Recv(recv_counts + p, 1, ncclInt32, p, comm_of(ctx), st));
    }
    AC_NCCL(N->GroupEnd());
    if (attncache_status s = comm_mark(ctx, st)) return s;
    int32_t *hc = (int32_t *)(ctx->h_pinned + kPinnedInts / 2);
    AC_CUDA(cudaMemcpyAsync(hc, counts, sizeof(int32_t) * 2 * w, cudaMemcpyDeviceToHost, st));
    if (attncache_status s = comm_wait(ctx, st, false)) return s;
    std::vector<int64_t> sn(w), rn(w), so(w + 1, 0), ro(w + 1, 0);
    for (int p = 0; p < w; ++p) {
        sn[p] = hc[p];
        rn[p] = hc[w + p];
        so[p + 1] = so[p] + sn[p];
        ro[p + 1] = ro[p] + rn[p];
    }
    const int64_t n_send = so[w], n_recv = ro[w];
    void *v_send = nullptr, *v_recv = nullptr, *o_recv = nullptr, *o_back = nullptr;
    if ((s = scratch(ctx, st, kScSend, row_v * (size_t)n_send + 8 * (size_t)n_send, &v_send))) return s;
    if ((s = scratch(ctx, st, kScRecv, row_v * (size_t)n_recv + 8 * (size_t)n_recv + 16, &v_recv))) return s;
    if ((s = scratch(ctx, st, kScOut, row_o * (size_t)n_recv, &o_recv))) return s;
    if ((s = scratch(ctx, st, kScBack, row_o * (size_t)n_send, &o_back))) return s;
    int64_t *idx_recv = (int64_t *)((uint8_t *)v_recv + ((row_v * (size_t)n_recv + 15) & ~(size_t)15));
    // C4: V rows and their entry indices to the owners
    if (n_send) {
        const bool ok16 = row_v % 16 == 0 && aligned16(V) && aligned16(v_send);
        AC_CUDA(launch_copy_rows(V, order, n_send, (int64_t)row_v, v_send, true, ok16, ctx->aux_sms, st));
        AC_CUDA(launch_copy_rows(idx, order, n_send, 8, idx_send, true, false, ctx->aux_sms, st));
    }
    if ((s = exchange_rows(ctx, v_send, sn.data(), so.data(), v_recv, rn.data(), ro.data(), row_v, st))) return s;
    if ((s = exchange_rows(ctx, idx_send, sn.data(), so.data(), idx_recv, rn.data(), ro.data(), 8, st))) return s;
    // K4: A.V on this shard for the received rows
    if (n_recv) {
        s = apply_local_impl(db, idx_recv, nullptr, n_recv, layer_begin, layer_end, head_dim, n_kv_heads, act_dtype, v_recv,
                             o_recv, st);
        if (s) return s;
    }
    // C5: O rows back to their home rank; K3: scatter into O
    if ((s = exchange_rows(ctx, o_recv, rn.data(), ro.data(), o_back, sn.data(), so.data(), row_o, st))) return s;
    if (n_send) {
        const bool ok16 = row_o % 16 == 0 && aligned16(O) && aligned16(o_back);
        AC_CUDA(launch_copy_rows(o_back, order, n_send, (int64_t)row_o, O, false, ok16, ctx->aux_sms, st));
    }
    return ATTNCACHE_OK;
}

}  // namespace ac

using namespace ac;

extern "C" {

attncache_status attncache_get_unique_id(uint8_t *out) {
    if (!out) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "get_unique_id: out is NULL");
    const NcclApi *N = nccl();
    if (!N) return fail(ATTNCACHE_ERR_NCCL, "get_unique_id: %s", g_nccl.why);
    ncclUniqueId id;
    AC_NCCL(N->GetUniqueId(&id));
    memcpy(out, id.internal, sizeof id.internal);
    return ATTNCACHE_OK;
}

attncache_status attncache_set_batch_layout(attncache_ctx *ctx, const int64_t *home_counts, int32_t world) {
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "set_batch_layout: ctx is NULL");
    if (!home_counts) {
        ctx->layout.clear();
        return ATTNCACHE_OK;
    }
    if (world != ctx->world)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "set_batch_layout: %d counts for a world of %d", world, ctx->world);
    for (int r = 0; r < world; ++r)
        if (home_counts[r] < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "set_batch_layout: negative count");
    ctx->layout.assign(home_counts, home_counts + world);
    return ATTNCACHE_OK;
}

attncache_status attncache_relocate_rows(attncache_ctx *ctx, const void *src, int64_t n_home, int64_t row_bytes,
                                         const int64_t *send_order, const int32_t *counts, void *dst, void *stream) {
    AC_NVTX("attncache_relocate_rows");
    if (!ctx) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: ctx is NULL");
    if (ctx->comm_failed) return comm_failed_status();
    if (n_home < 0 || row_bytes <= 0 || row_bytes % 8)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: n_home=%lld row_bytes=%lld (a multiple of 8)",
                    (long long)n_home, (long long)row_bytes);
    if (!counts) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: counts is NULL");
    const int w = ctx->world;
    std::vector<int64_t> sn(w), rn(w), so(w + 1, 0), ro(w + 1, 0);
    for (int p = 0; p < w; ++p) {
        if (counts[p] < 0 || counts[w + p] < 0) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: negative count");
        sn[p] = counts[p];
        rn[p] = counts[w + p];
        so[p + 1] = so[p] + sn[p];
        ro[p + 1] = ro[p] + rn[p];
    }
    if (so[w] != n_home) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: send counts sum to %lld, n_home %lld",
                                     (long long)so[w], (long long)n_home);
    if ((n_home && (!src || !send_order)) || (ro[w] && !dst))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: NULL buffer");
    if ((n_home && (!is_device_ptr(src) || !is_device_ptr(send_order))) || (ro[w] && !is_device_ptr(dst)))
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: buffers must be device memory");
    DeviceGuard g(ctx->device);
    cudaStream_t st = (cudaStream_t)stream;
    // rows that stay on this rank are gathered straight into their place in dst (one copy, no NCCL); the rows
    // for the other ranks are gathered into a send buffer and exchanged in one NCCL group
    const int me = (w == 1 || !ctx->comm) ? 0 : ctx->rank;
    const bool ok8 = row_bytes % 8 == 0;
    if (sn[me] && rn[me] != sn[me])
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "relocate_rows: %lld rows to self but %lld from self",
                    (long long)sn[me], (long long)rn[me]);
    if (sn[me]) {
        uint8_t *d = (uint8_t *)dst + (size_t)row_bytes * ro[me];
        const bool ok16 = row_bytes % 16 == 0 && aligned16(src) && aligned16(d);
        AC_CUDA(launch_copy_rows(src, send_order + so[me], sn[me], row_bytes, d, true, ok16 && ok8, ctx->aux_sms, st));
    }
    if (w == 1 || !ctx->comm) return ATTNCACHE_OK;
    const int64_t n_out = n_home - sn[me];
    void *send = nullptr;
    attncache_status s = scratch(ctx, st, kScSend, (size_t)row_bytes * (size_t)std::max<int64_t>(n_out, 1), &send);
    if (s) return s;
    // send buffer: the rows of ranks below me at [0, so[me]), above me at [so[me], n_out)
    const bool ok16 = row_bytes % 16 == 0 && aligned16(src) && aligned16(send);
    if (so[me]) AC_CUDA(launch_copy_rows(src, send_order, so[me], row_bytes, send, true, ok16, ctx->aux_sms, st));
    if (so[w] > so[me + 1])
        AC_CUDA(launch_copy_rows(src, send_order + so[me + 1], so[w] - so[me + 1], row_bytes,
                                 (uint8_t *)send + (size_t)row_bytes * so[me], true,
                                 ok16 && ((size_t)row_bytes * so[me]) % 16 == 0, ctx->aux_sms, st));
    std::vector<int64_t> sn2 = sn, so2(w, 0), rn2 = rn;
    for (int p = 0; p < w; ++p) so2[p] = p < me ? so[p] : so[p] - sn[me];
    sn2[me] = 0;
    rn2[me] = 0;
    return exchange_rows(ctx, send, sn2.data(), so2.data(), dst, rn2.data(), ro.data(), (size_t)row_bytes, st);
}

}  // extern "C"
