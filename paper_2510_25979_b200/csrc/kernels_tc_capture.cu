// kernels_tc_capture.cu — DB building, capture (Fig. 4 step 1):
// the post-softmax causal attention maps of a prefill, P = softmax(Q K^T * scale, keys j > i masked),
// rounded to the map dtype and written straight into a DB entry (DENSE or PACKED layout).
//
// Work item = (unit, 128-query block qb).  Two passes over the key blocks j = 0..qb:
//   pass 0: S = Q K_j^T on tcgen05 (M=128, N=128, K=d, fp32 in TMEM); each epilogue thread keeps
//           its row's running max m and sum l of exp2(s*scale*log2e - m)           (row statistics)
//   pass 1: S again; P = exp2(s*scale*log2e - m - log2 l), masked, rounded, stored.
// Recomputing S (2x the Q K^T flops) keeps the kernel one launch with no score round trip through
// HBM; the kernel is bound by writing the maps.
// Roles (192 threads): warp 0 TMA loader, warp 1 MMA issuer + TMEM owner (2 S buffers), warps 2-5
// epilogue (TMEM lane quarter = warp % 4, one query row per thread).
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 192;
constexpr int kBlk = 128;

template <int kD>
struct Cfg {
    static constexpr int kTile = kBlk * kD * 2;
    static constexpr int kQSlots = 2;
    static constexpr int kKSlots = kD == 64 ? 6 : 4;
    static constexpr int kSmem = (kQSlots + kKSlots) * kTile + 1024 + 512;
    static constexpr uint32_t kTmemCols = 256;  // two 128-column S buffers
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int kD>
__global__ void __launch_bounds__(kThreads, 1)
    capture_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const CaptureArgs a, const uint32_t idesc) {
    using C = Cfg<kD>;
    constexpr int NQ = C::kQSlots, NK = C::kKSlots;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = smem, *sK = smem + NQ * C::kTile;
    uint64_t *bars = (uint64_t *)(sK + NK * C::kTile);
    uint64_t *q_full = bars, *q_empty = q_full + NQ;
    uint64_t *k_full = q_empty + NQ, *k_empty = k_full + NK;
    uint64_t *s_full = k_empty + NK, *s_free = s_full + 2;
    uint32_t *tmem_slot = (uint32_t *)(s_free + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NQ; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < NK; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t S = (uint32_t)a.S;
    const uint32_t n_qb = S / kBlk;
    const uint32_t per_row = (uint32_t)(a.L * a.H);
    const uint32_t units = (uint32_t)(*a.list.count) * per_row;
    const uint32_t items = units * n_qb;
    // item t -> (selected row, (layer, head), qb): units in L2-sized groups (K of a group fits in ~48 MB;
    // both passes re-read it), heaviest query blocks first inside a group
    const uint32_t l2_group = max(1u, (48u << 20) / (S * (uint32_t)a.d * 2u));
    auto decode = [&](uint32_t t, int64_t &row, uint32_t &lh, int &qb) {
        const uint32_t gi = t / (l2_group * n_qb), w = t - gi * (l2_group * n_qb);
        const uint32_t gbase = gi * l2_group, gsize = min(l2_group, units - gbase);
        qb = (int)(n_qb - 1 - w / gsize);
        const uint32_t u = gbase + w % gsize;
        row = a.list.rows[u / per_row];
        lh = u % per_row;
    };

    if (warp < 2) {
        if (lane == 0) {
            uint32_t it = 0, blk = 0;
            for (uint32_t t = blockIdx.x; t < items; t += gridDim.x, ++it) {
                int64_t row;
                uint32_t lh;
                int qb;
                decode(t, row, lh, qb);
                const int64_t row0 = (row * per_row + lh) * (int64_t)S;  // first Q/K row of the unit
                const uint32_t qs = it % NQ, qph = (it / NQ) & 1u;
                if (warp == 0) {
                    mbar_wait(&q_empty[qs], qph ^ 1u);
                    mbar_arrive_expect_tx(&q_full[qs], C::kTile);
                    for (int h = 0; h < kD / 64; ++h)
                        tma_load_2d(smem_u32(sQ + qs * C::kTile + h * (kBlk * 128)), &tmQ, &q_full[qs], h * 64,
                                    (int32_t)(row0 + qb * kBlk));
                } else {
                    mbar_wait(&q_full[qs], qph);
                }
                for (int pass = 0; pass < 2; ++pass) {
                    for (int j = 0; j <= qb; ++j, ++blk) {
                        const uint32_t ks = blk % NK, kph = (blk / NK) & 1u;
                        if (warp == 0) {
                            mbar_wait(&k_empty[ks], kph ^ 1u);
                            mbar_arrive_expect_tx(&k_full[ks], C::kTile);
                            for (int h = 0; h < kD / 64; ++h)
                                tma_load_2d(smem_u32(sK + ks * C::kTile + h * (kBlk * 128)), &tmK, &k_full[ks],
                                            h * 64, (int32_t)(row0 + j * kBlk));
                        } else {
                            const uint32_t buf = blk & 1u, bph = (blk >> 1) & 1u;
                            mbar_wait(&k_full[ks], kph);
                            mbar_wait(&s_free[buf], bph ^ 1u);
                            tc_fence_after();
                            const uint32_t q_base = smem_u32(sQ + qs * C::kTile), k_base = smem_u32(sK + ks * C::kTile);
#pragma unroll
                            for (int k = 0; k < kD / 16; ++k) {
                                const uint32_t off = (k >> 2) * (kBlk * 128) + (k & 3) * 32;
                                umma_f16(tmem + buf * kBlk, smem_desc(q_base + off, 16, 1024, kSwizzle128B),
                                         smem_desc(k_base + off, 16, 1024, kSwizzle128B), idesc, k != 0);
                            }
                            umma_commit(&s_full[buf]);
                            umma_commit(&k_empty[ks]);
                            if (pass == 1 && j == qb) umma_commit(&q_empty[qs]);
                        }
                    }
                }
            }
        }
    } else {
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;
        uint16_t *maps = (uint16_t *)a.maps;
        const bool bf16 = a.map_dt == ATTNCACHE_BF16;
        const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
        uint32_t blk = 0;
        for (uint32_t t = blockIdx.x; t < items; t += gridDim.x) {
            int64_t row;
            uint32_t lh;
            int qb;
            decode(t, row, lh, qb);
            const int R = qb * kBlk + r;  // this thread's query row in the unit
            uint16_t *mrow = maps + ((row * per_row + lh) * a.map_stride) + map_row_off(R, S, a.map_layout);
            // packed rows hold 8*(R/8 + 1) elements; dense rows S (zeros above the diagonal)
            const int stored = packed ? 8 * (R / 8 + 1) : (int)S;
            float m = -INFINITY, l = 0.f, off = 0.f;
            for (int pass = 0; pass < 2; ++pass) {
                for (int j = 0; j <= qb; ++j, ++blk) {
                    const uint32_t buf = blk & 1u, bph = (blk >> 1) & 1u;
                    const bool diag = j == qb;
                    const int lim = diag ? r : kBlk - 1;
                    const int n_chunks = diag ? q + 1 : kBlk / 32;
                    mbar_wait(&s_full[buf], bph);
                    tc_fence_after();
                    const uint32_t s_addr = tmem + lane_addr + buf * kBlk;
                    if (pass == 0) {
                        for (int c = 0; c < n_chunks; ++c) {
                            uint32_t v[32];
                            tmem_ld_32x32b_x32(s_addr + c * 32, v);
                            tmem_ld_wait();
                            float mx = -INFINITY;
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (c * 32 + e <= lim) mx = fmaxf(mx, __uint_as_float(v[e]) * sl2);
                            const float m_new = fmaxf(m, mx);
                            float sum = 0.f;
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if (c * 32 + e <= lim) sum += ex2(fmaf(__uint_as_float(v[e]), sl2, -m_new));
                            l = l * ex2(m - m_new) + sum;
                            m = m_new;
                        }
                        tc_fence_before();
                        mbar_arrive(&s_free[buf]);
                        if (diag) off = m + lg2(l);  // P = exp2(s*sl2 - off)
                    } else {
                        // this block's columns [128j, 128j + 128) that the row stores (the TMEM loads
                        // are warp-uniform; only the stores depend on the lane's row length)
                        const int c0 = j * kBlk;
                        const int ncols = min(kBlk, stored - c0);
#pragma unroll
                        for (int c = 0; c < kBlk / 32; ++c) {
                            uint32_t v[32];
                            if (c < n_chunks) {
                                tmem_ld_32x32b_x32(s_addr + c * 32, v);
                                tmem_ld_wait();
                            }
                            uint32_t w[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                const int k0 = c * 32 + 2 * e;
                                const float p0 = (c < n_chunks && k0 <= lim) ? ex2(fmaf(__uint_as_float(v[2 * e]), sl2, -off)) : 0.f;
                                const float p1 =
                                    (c < n_chunks && k0 + 1 <= lim) ? ex2(fmaf(__uint_as_float(v[2 * e + 1]), sl2, -off)) : 0.f;
                                if (bf16) {
                                    __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                                    w[e] = *reinterpret_cast<uint32_t *>(&h2);
                                } else {
                                    __half2 h2 = __floats2half2_rn(p0, p1);
                                    w[e] = *reinterpret_cast<uint32_t *>(&h2);
                                }
                            }
                            uint4 *dst = (uint4 *)(mrow + c0 + c * 32);
#pragma unroll
                            for (int pc = 0; pc < 4; ++pc)
                                if (c * 32 + pc * 8 < ncols) dst[pc] = make_uint4(w[4 * pc], w[4 * pc + 1], w[4 * pc + 2], w[4 * pc + 3]);
                        }
                        tc_fence_before();
                        mbar_arrive(&s_free[buf]);
                    }
                }
            }
            // dense maps: the columns right of this block's diagonal are exact zeros (reading R11)
            if (!packed) {
                for (int c0 = (qb + 1) * kBlk; c0 < (int)S; c0 += 8)
                    *(uint4 *)(mrow + c0) = make_uint4(0, 0, 0, 0);
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

template <int kD>
cudaError_t launch(const CaptureArgs &a, int sm_count, cudaStream_t st) {
    using C = Cfg<kD>;
    const bool bf16 = a.dt == ATTNCACHE_BF16;
    const uint64_t rows = (uint64_t)a.max_rows * a.L * a.H * a.S;
    CUtensorMap tq, tk;
    cudaError_t e = make_tmap_2d_16(&tq, a.Q, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tk, a.K, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(capture_tc_kernel<kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t idesc = idesc_f16(kBlk, kBlk, bf16 ? 1u : 0u, 0u, 0u);
    capture_tc_kernel<kD><<<sm_count, kThreads, C::kSmem, st>>>(tq, tk, a, idesc);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

bool capture_tc_supported(int32_t dt, int32_t S, int32_t d) {
    return (dt == ATTNCACHE_BF16 || dt == ATTNCACHE_F16) && S >= kBlk && S % kBlk == 0 && (d == 64 || d == 128);
}

cudaError_t launch_capture_tc(const CaptureArgs &a, int sm_count, cudaStream_t st) {
    const uint64_t rows = (uint64_t)a.max_rows * a.L * a.H * a.S;
    if (rows >= (1ull << 31) || (uint64_t)a.max_rows * a.L * a.H * (a.S / kBlk) >= (1ull << 31))
        return cudaErrorInvalidValue;
    return a.d == 64 ? launch<64>(a, sm_count, st) : launch<128>(a, sm_count, st);
}

}  // namespace ac
