// kernels.cuh — host-side launchers of the device kernels (internal to libattncache).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace ac {

// Compacted selection list living in ctx scratch:
//   int32 count | pad to 16 B | int32 rows[cap] | int64 ents[cap] (apply only)
struct RowList {
    int32_t *count;
    int32_t *rows;
    int64_t *ents;
    int64_t cap;
};
RowList rowlist_view(void *base, int64_t cap);
size_t rowlist_bytes(int64_t cap);

// Order-preserving block compaction by every thread of one CTA (blockDim.x a multiple of 32, <= 1024): the select
// kernels (one CTA of 1024 threads; n up to a few 10^5 rows) and the fused prologues of the A.V / attention kernels
// (out in shared memory).
template <typename Pred>
__device__ void compact_rows(int64_t n, Pred pred, RowList out) {
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) base = 0;
    __syncthreads();
    for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
        int64_t b = b0 + tid;
        int64_t ent = -1;
        bool sel = (b < n) && pred(b, ent);
        unsigned m = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) warp_tot[warp] = __popc(m);
        __syncthreads();
        if (tid == 0) {
            int run = base;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                int t = warp_tot[w];
                warp_tot[w] = run;
                run += t;
            }
            base = run;
        }
        __syncthreads();
        if (sel) {
            int pos = warp_tot[warp] + __popc(m & ((1u << lane) - 1u));
            out.rows[pos] = (int32_t)b;
            out.ents[pos] = ent;
        }
        __syncthreads();
    }
    if (tid == 0) *out.count = base;
}


// Row selection done inside a persistent kernel's prologue instead of a select launch (n <= the kernel's shared-memory
// list capacity): apply: rows with (hit ? hit[b] : idx[b] >= 0) and entry idx[b] - shard_begin in the shard (else
// *err |= 1, dropped); attend: rows with skip == NULL || skip[b] == 0.  n == 0: the kernel reads its global list.
struct SelectArgs {
    const int64_t *idx = nullptr;
    const uint8_t *mask = nullptr;  // hit (apply) or skip (attend)
    int64_t n = 0;
    int64_t shard_begin = 0, shard_count = 0;
    int *err = nullptr;
};
__device__ __forceinline__ bool select_apply_pred(const SelectArgs &s, int64_t b, int64_t &ent) {
    const bool want = s.mask ? (s.mask[b] != 0) : (s.idx[b] >= 0);
    if (!want) return false;
    const int64_t e = s.idx[b] - s.shard_begin;
    if (e < 0 || e >= s.shard_count) {
        if (blockIdx.x == 0) atomicOr(s.err, 1);
        return false;
    }
    ent = e;
    return true;
}
__device__ __forceinline__ bool select_attend_pred(const SelectArgs &s, int64_t b, int64_t &ent) {
    ent = b;
    return s.mask == nullptr || s.mask[b] == 0;
}

// Rows with (hit ? hit[b] : idx[b] >= 0); entry = idx[b] - shard_begin must lie in
// [0, shard_count) else *err |= 1 and the row is dropped.
cudaError_t launch_select_apply(const int64_t *idx, const uint8_t *hit, int64_t n, int64_t shard_begin,
                                int64_t shard_count, RowList out, int *err, cudaStream_t st);
// Rows with skip == NULL || skip[b] == 0.
cudaError_t launch_select_attend(const uint8_t *skip, int64_t n, RowList out, cudaStream_t st);

// ---- search ----
cudaError_t launch_search_ffma(int32_t dt, const void *q, const void *x, int64_t B, int64_t n, int32_t D,
                               int64_t gbase, uint64_t *keys, cudaStream_t st);
bool search_tc_supported(int32_t dt, int32_t D);
// K2 fused into the search kernel (single GPU): the last CTA to finish gates the keys into idx/score/hit and
// re-zeroes them and the arrival counter `done` (both zero before the launch).
struct SearchDecode {
    int64_t *idx;
    float *score;
    uint8_t *hit;
    float tau;
    unsigned int *done;
};
cudaError_t launch_search_tc(const void *q, const void *x, int64_t B, int64_t n, int32_t D, int64_t gbase,
                             uint64_t *keys, int sm_count, cudaStream_t st, const SearchDecode *dec = nullptr);
cudaError_t launch_keys_decode(const uint64_t *keys, int32_t n_shards, int64_t n, float tau, int64_t *idx, float *score, uint8_t *hit,
                               cudaStream_t st);

// ---- apply (O = A . V) ----
struct ApplyArgs {
    const void *maps;  // shard maps [n_loc][L][H][S][S]
    int32_t L, H, S, d;
    int32_t layer_begin, n_lay;  // layer slice of V/O
    int32_t map_dt, act_dt;
    int32_t map_layout;  // ATTNCACHE_MAPS_DENSE / _PACKED
    int64_t map_stride;  // elements per S x S map
    int32_t causal;      // 1: lower-triangular maps (decoder); 0: full maps (encoder, f3)
    int32_t Hkv;         // V heads (grouped-query attention: map head h reads V head h / (H / Hkv)); H for MHA
    const void *V;
    void *O;
    RowList list;
    int64_t max_rows;  // host upper bound on list count (n_rows)
    SelectArgs sel;    // sel.n > 0: the kernel selects the rows itself (apply_tc_fused_select)
};
cudaError_t launch_apply_ffma(const ApplyArgs &a, int sm_count, cudaStream_t st);
bool apply_tc_supported(int32_t map_dt, int32_t act_dt, int32_t S, int32_t d);
// true when launch_apply_tc can select the rows in its prologue (then no launch_select_apply is needed)
bool apply_tc_fused_select(const ApplyArgs &a, int64_t n_rows);
cudaError_t launch_apply_tc(const ApplyArgs &a, int sm_count, cudaStream_t st);

// ---- attend (causal softmax attention) ----
struct AttendArgs {
    int32_t L, H, S, d, dt;
    int32_t Hkv;  // K/V heads (grouped-query attention: query head h reads K/V head h / (H / Hkv)); H for MHA
    float scale;
    const void *Q, *K, *V;
    void *O;
    RowList list;
    int64_t max_rows;
    SelectArgs sel;  // sel.n > 0: the kernel selects the rows itself (attend_tc_fused_select)
};
cudaError_t launch_attend_ffma(const AttendArgs &a, int sm_count, cudaStream_t st);
// The CUDA-core attention / capture / search fallbacks keep one fp32 row of S (or D) values per warp in shared
// memory (8 warps): 32 * S bytes <= 227 KB.
constexpr int32_t kSimtMaxLen = 7264;
bool attend_tc_supported(int32_t dt, int32_t S, int32_t d);
bool attend_tc_fused_select(const AttendArgs &a, int64_t n_rows);
int64_t attend_split_sel_cap();  // rows the d = 128 split kernel selects in its prologue
cudaError_t launch_attend_tc(const AttendArgs &a, int sm_count, cudaStream_t st);
cudaError_t launch_attend_split(const AttendArgs &a, int sm_count, cudaStream_t st);  // d = 128, double-buffered S
// The four 3-D tensor maps of an attention launch: Q, K, V boxes [128 rows][64 cols], O box [32][64].
cudaError_t make_attend_tmaps(const AttendArgs &a, int d, CUtensorMap *tq, CUtensorMap *tk, CUtensorMap *tv,
                              CUtensorMap *to);

// ---- capture (DB building: the causal maps of a prefill) ----
struct CaptureArgs {
    int32_t L, H, S, d, dt;  // dt: Q/K dtype
    int32_t Hkv;             // K heads (grouped-query attention); H for MHA
    int32_t map_dt, map_layout;
    int64_t map_stride;      // elements per S x S map in map_layout
    float scale;
    const void *Q, *K;
    void *maps;              // [rows][L][H][map]
    RowList list;
    int64_t max_rows;
};
cudaError_t launch_capture_simt(const CaptureArgs &a, int sm_count, cudaStream_t st);
bool capture_tc_supported(int32_t dt, int32_t S, int32_t d);
cudaError_t launch_capture_tc(const CaptureArgs &a, int sm_count, cudaStream_t st);

// ---- feature projector (f2): z = relu(W1 h + b1), y = W2 z + b2, f = y / ||y|| ----
struct ProjectArgs {
    int64_t M;            // rows (sentences)
    int32_t E, Hd, D;     // input, hidden, feature dims
    int32_t dt, feat_dt;  // dtype of h/W1/W2/z; dtype of f
    const void *h, *W1, *W2;
    const float *b1, *b2;
    void *z;              // scratch [M][Hd] in dt
    float *y;             // scratch [M][D] fp32
    void *f;              // [M][D] in feat_dt
};
bool linear_tc_supported(int32_t dt, int32_t K, int32_t Nout);
// Y = X W^T stored head-major [M / S][N / d][S][d] (+ bias when non-NULL), rounded once to dt (f4 projections).
cudaError_t launch_linear_heads(int32_t dt, const void *X, int64_t M, int32_t K, const void *W, int32_t N,
                                const float *bias, int32_t S, int32_t d, void *Y, int sm_count, cudaStream_t st);

// ---- owner-affinity placement on the device (kernels_plan.cu) ----
constexpr int kPlanMaxWorld = 32;
struct PlanArgs {
    int32_t world, rank;
    double hit_cost, miss_cost;
    int64_t shard_begins[kPlanMaxWorld + 1];
    int64_t home_begins[kPlanMaxWorld + 1];
};
cudaError_t launch_affinity_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const PlanArgs &a, int32_t *assign,
                                 double *load, int64_t *scratch, int64_t *loc, int64_t *idx_loc, uint8_t *hit_loc,
                                 int64_t *send_order, int32_t *counts, cudaStream_t st);
cudaError_t launch_project(const ProjectArgs &a, int sm_count, cudaStream_t st);

// ---- RoPE (f4 block-level comparison) ----
cudaError_t launch_rope(void *X, int64_t n_units, int32_t S, int32_t d, int32_t dt, float base, cudaStream_t st);

// ---- TMA descriptors (tma_host.cu) ----
cudaError_t make_tmap_2d_16(CUtensorMap *out, const void *base, bool bf16, uint64_t inner, uint64_t outer,
                            uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

// [outer][mid][inner] 16-bit tensor (e.g. [units][S][d]) with box [1][box_mid][box_inner]: rows past `mid`
// read as zeros and are clipped on store, so a unit's last partial 128-row block needs no masking in the
// kernels, and the unit index is its own coordinate (no 2^31 limit on units * S rows).
cudaError_t make_tmap_3d_16(CUtensorMap *out, const void *base, bool bf16, uint64_t inner, uint64_t mid, uint64_t outer,
                            uint64_t row_bytes, uint64_t plane_bytes, uint32_t box_inner, uint32_t box_mid,
                            int swizzle_bytes);

// ---- packed map layout ----
cudaError_t launch_pack_maps(const void *dense, int64_t n_maps, int32_t S, void *packed, bool unpack, cudaStream_t st);

// ---- routing ----
cudaError_t launch_route_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const int64_t *shard_begins,
                              int32_t world, int32_t *owner, int32_t *counts, int64_t *order, cudaStream_t st);
// ok16: row_bytes % 16 == 0 and both bases 16-byte aligned (int4 accesses); else 8-byte accesses.
cudaError_t launch_copy_rows(const void *src, const int64_t *rows, int64_t n_rows, int64_t row_bytes, void *dst,
                             bool gather, bool ok16, int sms, cudaStream_t st);  // sms: CTA budget (~16 per SM)

}  // namespace ac
