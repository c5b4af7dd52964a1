// host_prefill.cu — the single-rank step end to end from host buffers (include/attncache.h
// attncache_prefill_host): Alg. 1 search, then Alg. 2 per layer for every row (hit: O = A.V; miss: causal
// softmax attention), with every host<->device copy inside the call.
#include <string.h>

#include <algorithm>
#include <cmath>

#include <vector>

#include "abi_internal.cuh"

using namespace ac;

namespace {

// Contiguous runs of rows [b, e) of `want` (a per-row flag) inside [b0, b1): one copy per run.
template <typename F>
void for_runs(const uint8_t *want, int64_t b0, int64_t b1, F f) {
    int64_t b = b0;
    while (b < b1) {
        while (b < b1 && !want[b]) ++b;
        int64_t e = b;
        while (e < b1 && want[e]) ++e;
        if (e > b) f(b, e);
        b = e;
    }
}

}  // namespace

extern "C" attncache_status attncache_prefill_host(attncache_db *db, const void *q, int64_t n, float tau,
                                                   const void *Q, const void *K, const void *V, int32_t head_dim,
                                                   int32_t act_dtype, void *O, int64_t *idx, float *score,
                                                   uint8_t *hit, int32_t chunk, int32_t depth) {
    AC_NVTX("attncache_prefill_host");
    if (!db) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "prefill_host: db is NULL");
    attncache_ctx *ctx = db->ctx;
    const attncache_db_desc &d = db->d;
    if (ctx->comm && ctx->world > 1)
        return fail(ATTNCACHE_ERR_STATE, "prefill_host: single-rank call (the ctx has a world of %d)", ctx->world);
    if (d.shard_count != d.n_global) return fail(ATTNCACHE_ERR_STATE, "prefill_host: the db must hold every entry");
    if (d.n_global == 0) return fail(ATTNCACHE_ERR_EMPTY, "prefill_host: the database has no entries");
    if (d.n_layers <= 0) return fail(ATTNCACHE_ERR_STATE, "prefill_host: this database holds no maps");
    if (n < 0 || chunk <= 0 || depth < 2 || depth > 8)
        return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "prefill_host: n=%lld chunk=%d depth=%d (depth in [2, 8])",
                    (long long)n, chunk, depth);
    if (std::isnan(tau)) return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "prefill_host: tau is NaN");
    if (!dtype_valid(act_dtype) || !(act_dtype == ATTNCACHE_F32 || act_dtype == d.map_dtype))
        return fail(ATTNCACHE_ERR_DTYPE, "prefill_host: act_dtype %d", act_dtype);
    if (head_dim <= 0 || ((int64_t)head_dim * dtype_size(act_dtype)) % 16)
        return fail(ATTNCACHE_ERR_ALIGNMENT, "prefill_host: head_dim %d rows not 16-byte multiples", head_dim);
    if (n == 0) return ATTNCACHE_OK;
    const void *hp[] = {q, Q, K, V, O, idx, score, hit};
    for (const void *p : hp)
        if (!p || !is_pinned_host_ptr(p))
            return fail(ATTNCACHE_ERR_INVALID_ARGUMENT, "prefill_host: every buffer must be page-locked host memory "
                        "(cudaHostAlloc / cudaHostRegister)");
    DeviceGuard g(ctx->device);
    for (int i = 0; i < 3; ++i)
        if (!ctx->io_stream[i]) AC_CUDA(cudaStreamCreateWithFlags(&ctx->io_stream[i], cudaStreamNonBlocking));
    cudaStream_t cin = ctx->io_stream[0], comp = ctx->io_stream[1], cout = ctx->io_stream[2];
    const int es = dtype_size(act_dtype);
    const size_t qrow = (size_t)d.feat_dim * dtype_size(d.feat_dtype);
    const size_t row = (size_t)d.n_layers * d.n_heads * d.seq_len * head_dim * es;  // one query's Q/K/V/O
    const int64_t c = std::min<int64_t>(chunk, n);
    // device staging: queries, idx/score/hit, then a ring of `depth` slots of V, Q, K, O chunks
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t off_q = 0, off_idx = up(qrow * n), off_score = off_idx + up(8 * n), off_hit = off_score + up(4 * n);
    const size_t off_ring = off_hit + up(n), slot = up(row * c);
    const size_t total = off_ring + 4 * slot * (size_t)depth;
    void *base = nullptr;
    attncache_status s = scratch(ctx, comp, kScHost, total, &base);
    if (s) return s;
    uint8_t *b8 = (uint8_t *)base;
    int64_t *d_idx = (int64_t *)(b8 + off_idx);
    float *d_score = (float *)(b8 + off_score);
    uint8_t *d_hit = b8 + off_hit;
    auto ring = [&](int kind, int r) { return (void *)(b8 + off_ring + ((size_t)kind * depth + r) * slot); };
    // Alg. 1: H2D queries, search, D2H of the decisions (the host must know the misses: Alg. 2 computes q, k
    // only on a miss, l.376-378, so only their Q and K cross PCIe)
    AC_CUDA(cudaMemcpyAsync(b8 + off_q, q, qrow * n, cudaMemcpyHostToDevice, comp));
    void *keys = nullptr;
    if ((s = scratch(ctx, comp, kScSearchKeys, sizeof(uint64_t) * (size_t)n, &keys))) return s;
    if ((s = search_keys_impl(db, b8 + off_q, n, (uint64_t *)keys, comp))) return s;
    AC_CUDA(launch_keys_decode((const uint64_t *)keys, 1, n, tau, d_idx, d_score, d_hit, comp));
    AC_CUDA(cudaMemcpyAsync(idx, d_idx, 8 * n, cudaMemcpyDeviceToHost, comp));
    AC_CUDA(cudaMemcpyAsync(score, d_score, 4 * n, cudaMemcpyDeviceToHost, comp));
    AC_CUDA(cudaMemcpyAsync(hit, d_hit, n, cudaMemcpyDeviceToHost, comp));
    AC_CUDA(cudaStreamSynchronize(comp));
    std::vector<uint8_t> miss(n);
    for (int64_t b = 0; b < n; ++b) miss[b] = hit[b] ? 0 : 1;
    // Alg. 2 in chunks: copy-in | compute | copy-out on three streams, a ring of `depth` slots
    std::vector<cudaEvent_t> ev(3 * depth);
    for (auto &e : ev) AC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::vector<bool> used(depth, false);
    const int64_t n_chunks = (n + c - 1) / c;
    attncache_status st_out = ATTNCACHE_OK;
    for (int64_t k = 0; k < n_chunks && !st_out; ++k) {
        const int r = (int)(k % depth);
        const int64_t b0 = k * c, b1 = std::min(n, b0 + c), m = b1 - b0;
        cudaEvent_t ev_in = ev[3 * r], ev_comp = ev[3 * r + 1], ev_out = ev[3 * r + 2];
        void *Vd = ring(0, r), *Qd = ring(1, r), *Kd = ring(2, r), *Od = ring(3, r);
        if (used[r] && cudaStreamWaitEvent(cin, ev_comp, 0) != cudaSuccess) { st_out = cuda_status(cudaGetLastError(), "prefill_host"); break; }
        cudaError_t e = cudaMemcpyAsync(Vd, (const uint8_t *)V + row * b0, row * m, cudaMemcpyHostToDevice, cin);
        for_runs(miss.data(), b0, b1, [&](int64_t x, int64_t y) {
            if (e == cudaSuccess)
                e = cudaMemcpyAsync((uint8_t *)Qd + row * (x - b0), (const uint8_t *)Q + row * x, row * (y - x),
                                    cudaMemcpyHostToDevice, cin);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync((uint8_t *)Kd + row * (x - b0), (const uint8_t *)K + row * x, row * (y - x),
                                    cudaMemcpyHostToDevice, cin);
        });
        if (e == cudaSuccess) e = cudaEventRecord(ev_in, cin);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(comp, ev_in, 0);
        if (e == cudaSuccess && used[r]) e = cudaStreamWaitEvent(comp, ev_out, 0);  // O slot drained
        if (e != cudaSuccess) { st_out = cuda_status(e, "prefill_host: copy-in"); break; }
        st_out = apply_local_impl(db, d_idx + b0, d_hit + b0, m, 0, d.n_layers, head_dim, d.n_heads, act_dtype, Vd, Od,
                                  comp);
        if (!st_out)
            st_out = attncache_attend_full(ctx, m, d.n_layers, d.n_heads, d.seq_len, head_dim, act_dtype, Qd, Kd, Vd,
                                           0.f, d_hit + b0, Od, comp);
        if (st_out) break;
        e = cudaEventRecord(ev_comp, comp);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cout, ev_comp, 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync((uint8_t *)O + row * b0, Od, row * m, cudaMemcpyDeviceToHost, cout);
        if (e == cudaSuccess) e = cudaEventRecord(ev_out, cout);
        if (e != cudaSuccess) { st_out = cuda_status(e, "prefill_host: copy-out"); break; }
        used[r] = true;
    }
    cudaError_t e1 = cudaStreamSynchronize(cin), e2 = cudaStreamSynchronize(comp), e3 = cudaStreamSynchronize(cout);
    for (auto &e : ev) cudaEventDestroy(e);
    if (st_out) return st_out;
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
        return cuda_status(e1 != cudaSuccess ? e1 : e2 != cudaSuccess ? e2 : e3, "prefill_host: stream");
    return ATTNCACHE_OK;
}
