// common.cuh — shared internals of libattncache (not part of the ABI).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/attncache.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: a no-op unless a tool (ncu --nvtx, nsys) is attached

namespace ac {
// One NVTX range per C-ABI compute call (SURVEY.md §5 tracing): the calls show up by name in a tool's timeline.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace ac
#define AC_NVTX(name) ::ac::NvtxRange ac_nvtx_range_(name)

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
// K2: the tau gate on a (cross-shard maximum) key; key 0 = no entry anywhere (empty shards)
__device__ __forceinline__ void decode_key(uint64_t k, float tau, int64_t *idx, float *score, uint8_t *hit) {
    if (k == 0) {
        *idx = -1;
        *score = -INFINITY;
        *hit = 0;
    } else {
        const float s = ord_score((uint32_t)(k >> 32));
        *idx = (int64_t)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFu));
        *score = s;
        *hit = s >= tau ? 1 : 0;  // inclusive gate
    }
}

// ---- scratch owned by a ctx -------------------------------------------------
struct Scratch {
    void *ptr = nullptr;
    size_t bytes = 0;
};

// Scratch kinds.  Scratch is PER STREAM (work on two streams never shares a buffer) and stream-ordered
// (cudaMallocAsync / cudaFreeAsync on the call's stream: growing a buffer never stalls the device, and the
// old buffer is released only after the work queued before it on that stream).  A call issued while its
// stream is being captured into a CUDA graph gets buffers of its own that live as long as the ctx, so a
// graph's scratch is never freed or reused by later eager calls.
enum ScratchKind : int {
    kScApplyList = 0,  // compacted (row, entry) list for apply
    kScAttendList,     // compacted row list for attend / capture
    kScSearchKeys,     // per-query packed keys
    kScSearchFused,    // single-GPU search with the decode fused in: arrival counter + keys, kept zero between calls
    kScProject,        // feature projector intermediates (z, y)
    kScPlan,           // device affinity plan: the miss list
    kScQueries,        // collective search: the gathered query batch
    kScRoute,          // collective apply: owners, counts, order, idx rows
    kScSend,           // collective apply / relocate: rows sent
    kScRecv,           // collective apply / relocate: rows received
    kScOut,            // collective apply: O of the received rows
    kScBack,           // collective apply: O rows returned home
    kScHost,           // host prefill: device staging
    kNumScratch
};
struct StreamScratch {
    Scratch s[kNumScratch];
};

}  // namespace ac

#include <mutex>
#include <unordered_map>
#include <vector>

struct attncache_ctx {
    int device = 0;
    int sm_count = 148;
    int compute_sms = 148, aux_sms = 148;  // CTA caps (attncache_ctx_set_sm_budget); default sm_count
    int *d_error = nullptr;  // deferred device-side error flags (bit 0: NOT_FOUND)
    // collectives (one NCCL communicator per ctx; world == 1 and comm == nullptr for a local ctx)
    int rank = 0, world = 1;
    void *comm = nullptr;            // ncclComm_t
    bool comm_failed = false;        // the comm was aborted after an asynchronous NCCL error (comm_check)
    cudaEvent_t comm_ev = nullptr;   // completion of the last collective work enqueued (comm_wait polls it)
    bool comm_ev_pending = false;
    int64_t *h_pinned = nullptr;     // pinned host staging for counts (kPinnedInts int64)
    int64_t *d_small = nullptr;      // device staging for small exchanges (kPinnedInts int64)
    std::vector<int64_t> layout;     // the per-rank home batch sizes set by attncache_set_batch_layout (or empty)
    bool force_route = false;        // ATTNCACHE_FORCE_ROUTE=1: run the routed apply even at world 1 (tests)
    cudaStream_t io_stream[3] = {};  // host prefill: copy-in, compute, copy-out (created on first use)
    // scratch
    std::mutex mu;
    std::unordered_map<cudaStream_t, ac::StreamScratch> scratch;
    std::vector<void *> graph_owned;  // buffers of calls captured into CUDA graphs (freed at destroy)
};

struct attncache_db {
    attncache_ctx *ctx = nullptr;
    int device = 0;
    attncache_db_desc d{};
    std::vector<int64_t> shard_begins;  // [world + 1] global entry ranges of every rank (collective load)
    int64_t *d_shard_begins = nullptr;  // device copy
};

namespace ac {
constexpr int kPinnedInts = 4 * 1024 + 16;  // small int64 staging (host pinned and device): world <= 1024
// Device scratch of at least `bytes` for (stream, kind); see ScratchKind.
bool fused_select_ok(const attncache_ctx *ctx);  // row selection inside the layer kernels (local ctx only)
// fresh (optional): set when the returned buffer is newly allocated (its contents are undefined)
attncache_status scratch(attncache_ctx *ctx, cudaStream_t st, int kind, size_t bytes, void **out, bool *fresh = nullptr);

// A device pointer check: rejects host (unregistered or pinned) memory when the runtime can tell.
inline bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}
// Page-locked (pinned or registered) host memory: the only host memory the async copies accept.
inline bool is_pinned_host_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ---- collectives (collective.cu) ----
attncache_status comm_init(attncache_ctx *ctx, int rank, int world, const uint8_t uid[128]);
void comm_destroy(attncache_ctx *ctx);
}  // namespace ac
