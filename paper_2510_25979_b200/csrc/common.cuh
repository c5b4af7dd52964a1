// common.cuh — shared internals of libattncache (not part of the ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/attncache.h"

namespace ac {

constexpr int kNumSMs = 148;  // B200; the runtime value is queried at ctx creation

// ---- status plumbing ------------------------------------------------------
void set_error(const char *fmt, ...);
attncache_status fail(attncache_status s, const char *fmt, ...);
attncache_status cuda_status(cudaError_t e, const char *what);
void count_launches(int n);  // every kernel launch of the library goes through this
uint64_t launch_count();

#define AC_CUDA(call)                                              \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return ::ac::cuda_status(e_, #call); \
    } while (0)

#define AC_LAUNCH_CHECK(what)                                      \
    do {                                                           \
        cudaError_t e_ = cudaGetLastError();                       \
        if (e_ != cudaSuccess) return ::ac::cuda_status(e_, what); \
    } while (0)

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// PACKED map layout (include/attncache.h): row i starts at element 8*(4q(q+1) + r(q+1)), q = i/8,
// r = i%8, and holds 8*(q+1) elements; a map holds packed_row_off(S) elements (S % 8 == 0).
__host__ __device__ __forceinline__ int64_t packed_row_off(int64_t i) {
    const int64_t q = i >> 3, r = i & 7;
    return 8 * (4 * q * (q + 1) + r * (q + 1));
}
__host__ __device__ __forceinline__ int64_t map_elems(int32_t S, int32_t layout) {
    return layout == ATTNCACHE_MAPS_PACKED ? packed_row_off(S) : (int64_t)S * S;
}
// Element offset of map row i in either layout.
__host__ __device__ __forceinline__ int64_t map_row_off(int64_t i, int32_t S, int32_t layout) {
    return layout == ATTNCACHE_MAPS_PACKED ? packed_row_off(i) : i * S;
}

inline int dtype_size(int32_t dt) { return dt == ATTNCACHE_F32 ? 4 : 2; }
inline bool dtype_valid(int32_t dt) { return dt == ATTNCACHE_F32 || dt == ATTNCACHE_F16 || dt == ATTNCACHE_BF16; }

// ---- device element access -----------------------------------------------
template <int DT> struct Elem;
template <> struct Elem<ATTNCACHE_F32> {
    using T = float;
    static __device__ __forceinline__ float ld(const float *p, int64_t i) { return p[i]; }
    static __device__ __forceinline__ void st(float *p, int64_t i, float v) { p[i] = v; }
};
template <> struct Elem<ATTNCACHE_F16> {
    using T = __half;
    static __device__ __forceinline__ float ld(const __half *p, int64_t i) { return __half2float(p[i]); }
    static __device__ __forceinline__ void st(__half *p, int64_t i, float v) { p[i] = __float2half_rn(v); }
};
template <> struct Elem<ATTNCACHE_BF16> {
    using T = __nv_bfloat16;
    static __device__ __forceinline__ float ld(const __nv_bfloat16 *p, int64_t i) { return __bfloat162float(p[i]); }
    static __device__ __forceinline__ void st(__nv_bfloat16 *p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }
};

// ---- packed top-1 key (reading R3) -----------------------------------------
// key = ord(s) << 32 | (0xFFFFFFFF - i); max key = max score, then min index.
__device__ __forceinline__ uint32_t score_ord(float s) {
    s = s + 0.0f;  // canonicalise -0.0 to +0.0
    uint32_t b = __float_as_uint(s);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord_score(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
__device__ __forceinline__ uint64_t pack_key(float s, uint32_t gidx) {
    return ((uint64_t)score_ord(s) << 32) | (uint64_t)(0xFFFFFFFFu - gidx);
}

// ---- scratch owned by a ctx -------------------------------------------------
struct Scratch {
    void *ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace ac

struct attncache_ctx {
    int device = 0;
    int sm_count = 148;
    int *d_error = nullptr;  // deferred device-side error flags (bit 0: NOT_FOUND)
    ac::Scratch apply_list;  // compacted (row, entry) list for apply
    ac::Scratch attend_list; // compacted row list for attend
    ac::Scratch search_keys; // per-query keys for single-rank search
    ac::Scratch project_buf; // feature projector intermediates (z, y)
    ac::Scratch plan_buf;    // device affinity plan: the miss list
};

struct attncache_db {
    attncache_ctx *ctx = nullptr;
    attncache_db_desc d{};
};

namespace ac {
attncache_status ensure_scratch(Scratch &s, size_t bytes);
}
