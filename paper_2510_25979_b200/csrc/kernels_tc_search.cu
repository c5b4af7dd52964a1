// kernels_tc_search.cu — Alg. 1 l.255 "VecDB.search" as a tcgen05 GEMM with a fused top-1.
//
// s[b][i] = sum_k q[b][k] x[i][k] (bf16 inputs, fp32 accumulation in TMEM) over this shard,
// reduced on the fly to one packed (score, index) key per query (reading R3): the score matrix is
// never written to memory.  Work item = (128-query tile, 64/128/256-entry tile), ordered
// entry-tile-major so concurrently running CTAs share the same DB rows through L2 (the DB streams
// from HBM once).  Roles (192 threads): warp 0 TMA loader, warp 1 MMA issuer (M=128 queries,
// N=entry tile, K=16), warps 2-5 epilogue: each thread owns one query (= TMEM lane), scans its scores in ascending
// entry order keeping the first maximum, and merges with atomicMax on the packed key.
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 192;
constexpr int kTileQ = 128;
constexpr int kChunk = 64;                       // K elements per stage (one 128-byte swizzle row)
constexpr int kQBytes = kTileQ * kChunk * 2;

// Entry-tile width kTileE in {64, 128, 256}: wide tiles cut the L2 re-reads of the query tile for
// large batches (tensor-bound); narrow tiles give small searches enough CTAs.
template <int kTileE>
struct Cfg {
    static constexpr int kXBytes = kTileE * kChunk * 2;
    static constexpr int kStageBytes = kQBytes + kXBytes;
    static constexpr int kStages = kTileE == 256 ? 4 : kTileE == 128 ? 6 : 8;
    static constexpr uint32_t kTmemCols = 2 * kTileE;  // double-buffered fp32 accumulator
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

template <int kTileE>
__global__ void __launch_bounds__(kThreads, 1)
    search_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX, int64_t B,
                     int64_t n, int D, int64_t gbase, unsigned long long *keys, uint32_t idesc, uint32_t q_rows,
                     const SearchDecode dec) {
    using C = Cfg<kTileE>;
    constexpr int kStages = C::kStages, kStageBytes = C::kStageBytes;
    constexpr uint32_t kTmemCols = C::kTmemCols;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    uint64_t *tfull = empty + kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmX);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t n_qt = (B + kTileQ - 1) / kTileQ;
    const int64_t n_et = (n + kTileE - 1) / kTileE;
    const int64_t items = n_qt * n_et;
    const int n_kc = D / kChunk;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t cnt = 0;
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
                AC_STRESS_DELAY(423u);
                const int32_t qt = (int32_t)(t % n_qt), et = (int32_t)(t / n_qt);
                for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                    const uint32_t s = cnt % kStages, ph = (cnt / kStages) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    // small batches load only q_rows query rows; the MMA's other rows read stale shared
                    // memory, which only reaches TMEM lanes the epilogue never reads (b >= B)
                    mbar_arrive_expect_tx(&full[s], (q_rows + kTileE) * (kChunk * 2));
                    const uint32_t base = smem_u32(smem + s * kStageBytes);
                    tma_load_2d(base, &tmQ, &full[s], kc * kChunk, qt * kTileQ);
                    tma_load_2d(base + kQBytes, &tmX, &full[s], kc * kChunk, et * kTileE);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t cnt = 0, item = 0;
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x, ++item) {
                AC_STRESS_DELAY(781u);
                const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                mbar_wait(&tempty[acc], aph ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * kTileE;
                for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                    const uint32_t s = cnt % kStages, ph = (cnt / kStages) & 1u;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t qa = smem_u32(smem + s * kStageBytes), xa = qa + kQBytes;
#pragma unroll
                    for (int k = 0; k < kChunk / 16; ++k)
                        umma_f16(d_tmem, smem_desc(qa + k * 32, 16, 1024, kSwizzle128B),
                                 smem_desc(xa + k * 32, 16, 1024, kSwizzle128B), idesc, (kc | k) != 0);
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        const int q = warp & 3;
        const int r = q * 32 + lane;
        uint32_t item = 0;
        for (int64_t t = blockIdx.x; t < items; t += gridDim.x, ++item) {
            AC_STRESS_DELAY(490u);
            const int64_t qt = t % n_qt, et = t / n_qt;
            const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int64_t e0 = et * kTileE;
            const int valid = (int)min64(kTileE, n - e0);
            float best = -INFINITY;
            int bi = -1;
#pragma unroll
            for (int c = 0; c < kTileE / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + acc * kTileE + c * 32, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const float sc = __uint_as_float(v[e]);
                    if (c * 32 + e < valid && sc > best) {  // ascending scan, strict '>': first maximum
                        best = sc;
                        bi = c * 32 + e;
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            const int64_t b = qt * kTileQ + r;
            if (b < B && bi >= 0) atomicMax(&keys[b], (unsigned long long)pack_key(best, (uint32_t)(gbase + e0 + bi)));
        }
    }
    __threadfence();  // this thread's atomicMax results are visible device-wide before the CTA arrives
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
    if (dec.done) {
        // K2 fused (single GPU): the last CTA to arrive sees every CTA's keys, gates them and re-zeroes them (and
        // the counter) for the next launch, which then needs neither a memset nor a decode launch
        __shared__ unsigned int s_last;
        if (threadIdx.x == 0) s_last = atomicAdd(dec.done, 1u) == gridDim.x - 1 ? 1u : 0u;
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
                const unsigned long long k = atomicExch(&keys[b], 0ull);
                decode_key(k, dec.tau, &dec.idx[b], &dec.score[b], &dec.hit[b]);
            }
            if (threadIdx.x == 0) *dec.done = 0u;
        }
    }
}

}  // namespace

bool search_tc_supported(int32_t dt, int32_t D) { return dt == ATTNCACHE_BF16 && D >= kChunk && D % kChunk == 0; }

template <int kTileE>
static cudaError_t launch_t(const void *q, const void *x, int64_t B, int64_t n, int32_t D, int64_t gbase,
                           uint64_t *keys, int sm_count, cudaStream_t st, const SearchDecode *dec) {
    using C = Cfg<kTileE>;
    CUtensorMap tq, tx;
    const uint32_t q_rows = B >= kTileQ ? kTileQ : (uint32_t)((B + 7) / 8 * 8);
    cudaError_t e = make_tmap_2d_16(&tq, q, true, D, B, (uint64_t)D * 2, kChunk, q_rows, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tx, x, true, D, n, (uint64_t)D * 2, kChunk, kTileE, 128);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(search_tc_kernel<kTileE>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const int64_t items = ((B + kTileQ - 1) / kTileQ) * ((n + kTileE - 1) / kTileE);
    const int grid = (int)min64(items, sm_count);
    const uint32_t idesc = idesc_f16(kTileQ, kTileE, 1u, 0u, 0u);
    const SearchDecode d = dec ? *dec : SearchDecode{nullptr, nullptr, nullptr, 0.f, nullptr};
    search_tc_kernel<kTileE><<<grid, kThreads, C::kSmem, st>>>(tq, tx, B, n, D, gbase, (unsigned long long *)keys, idesc,
                                                             q_rows, d);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_search_tc(const void *q, const void *x, int64_t B, int64_t n, int32_t D, int64_t gbase,
                             uint64_t *keys, int sm_count, cudaStream_t st, const SearchDecode *dec) {
    if (B == 0 || n == 0) return cudaSuccess;
    // the widest entry tile that still gives every SM at least two work items
    const int64_t n_qt = (B + kTileQ - 1) / kTileQ;
    if (n_qt * ((n + 255) / 256) >= 2 * sm_count) return launch_t<256>(q, x, B, n, D, gbase, keys, sm_count, st, dec);
    if (n_qt * ((n + 127) / 128) >= 2 * sm_count) return launch_t<128>(q, x, B, n, D, gbase, keys, sm_count, st, dec);
    return launch_t<64>(q, x, B, n, D, gbase, keys, sm_count, st, dec);
}

}  // namespace ac
