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
// Roles (384 threads): two independent groups (two item streams per CTA), each with a TMA loader thread
// (warp 2g), an MMA thread (warp 2g+1; two 128-column S buffers per group) and a 4-warp epilogue group
// (warps 4-7 / 8-11; TMEM lane quarter = warp % 4, one query row per thread, the S row held in
// registers: one TMEM load per block).  A single epilogue group left the kernel at 0.29 of its HBM
// roofline (bench stages.capture_misses, configs[1]).
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 384;  // 3 warpgroups: producers (warps 0-3), epilogue group 0 (4-7), group 1 (8-11)
constexpr int kBlk = 128;

template <int kD>
struct Cfg {
    static constexpr int kTile = kBlk * kD * 2;
    static constexpr int kKSlots = 2;  // per group
    static constexpr int kSmem = (2 + 2 * kKSlots) * kTile + 1024 + 512;
    static constexpr uint32_t kTmemCols = 512;  // per group two 128-column S buffers
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
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

template <int kD>
__global__ void __launch_bounds__(kThreads, 1)
    capture_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const CaptureArgs a, const uint32_t idesc) {
    using C = Cfg<kD>;
    constexpr int NK = C::kKSlots;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = smem, *sK = smem + 2 * C::kTile;  // Q: [group]; K: [group][NK]
    uint64_t *bars = (uint64_t *)(sK + 2 * NK * C::kTile);
    uint64_t *q_full = bars, *q_empty = q_full + 2;        // [group]
    uint64_t *k_full = q_empty + 2, *k_empty = k_full + 2 * NK;  // [group][NK]
    uint64_t *s_full = k_empty + 2 * NK, *s_free = s_full + 4;   // [group][2 S buffers]
    uint32_t *tmem_slot = (uint32_t *)(s_free + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < 2 * NK; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int i = 0; i < 4; ++i) {
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
    const uint32_t stride = 2 * gridDim.x;  // two item streams per CTA (one per group)
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

    if (warp < 4) {
        // Producers: per group g, warp 2g loads Q (per item) and K_j (per block and pass), warp 2g+1
        // issues S_j = Q K_j^T into one of the group's two S buffers.  The two groups are independent
        // pipelines sharing the tensor pipe (as in kernels_tc_attend.cu).
        setmaxnreg_dec<56>();
        const int g = warp >> 1;
        if (lane == 0) {
            uint32_t it = 0, blk = 0;
            for (uint32_t t = blockIdx.x + g * gridDim.x; t < items; t += stride, ++it) {
                int64_t row;
                uint32_t lh;
                int qb;
                decode(t, row, lh, qb);
                const int64_t row0 = (row * per_row + lh) * (int64_t)S;  // first Q row of the unit
                // first K row: the unit's K head under grouped-query attention (Hkv = H for MHA)
                const int64_t krow0 = ((row * a.L + lh / (uint32_t)a.H) * a.Hkv + (lh % (uint32_t)a.H) / (uint32_t)(a.H / a.Hkv)) * (int64_t)S;
                const uint32_t qph = it & 1u;
                if ((warp & 1) == 0) {
                    mbar_wait(&q_empty[g], qph ^ 1u);
                    mbar_arrive_expect_tx(&q_full[g], C::kTile);
                    for (int h = 0; h < kD / 64; ++h)
                        tma_load_2d(smem_u32(sQ + g * C::kTile + h * (kBlk * 128)), &tmQ, &q_full[g], h * 64,
                                    (int32_t)(row0 + qb * kBlk));
                } else {
                    mbar_wait(&q_full[g], qph);
                }
                for (int pass = 0; pass < 2; ++pass) {
                    for (int j = 0; j <= qb; ++j, ++blk) {
                        const uint32_t ks = g * NK + blk % NK, kph = (blk / NK) & 1u;
                        if ((warp & 1) == 0) {
                            mbar_wait(&k_empty[ks], kph ^ 1u);
                            mbar_arrive_expect_tx(&k_full[ks], C::kTile);
                            for (int h = 0; h < kD / 64; ++h)
                                tma_load_2d(smem_u32(sK + ks * C::kTile + h * (kBlk * 128)), &tmK, &k_full[ks],
                                            h * 64, (int32_t)(krow0 + j * kBlk));
                        } else {
                            const uint32_t buf = blk & 1u, bph = (blk >> 1) & 1u;
                            mbar_wait(&k_full[ks], kph);
                            mbar_wait(&s_free[g * 2 + buf], bph ^ 1u);
                            tc_fence_after();
                            const uint32_t q_base = smem_u32(sQ + g * C::kTile), k_base = smem_u32(sK + ks * C::kTile);
#pragma unroll
                            for (int k = 0; k < kD / 16; ++k) {
                                const uint32_t off = (k >> 2) * (kBlk * 128) + (k & 3) * 32;
                                umma_f16(tmem + g * 256 + buf * kBlk, smem_desc(q_base + off, 16, 1024, kSwizzle128B),
                                         smem_desc(k_base + off, 16, 1024, kSwizzle128B), idesc, k != 0);
                            }
                            umma_commit(&s_full[g * 2 + buf]);
                            umma_commit(&k_empty[ks]);
                            if (pass == 1 && j == qb) umma_commit(&q_empty[g]);
                        }
                    }
                }
            }
        }
    } else {
        // ------------------------------ epilogue group g (one query row per thread) -----------------
        setmaxnreg_inc<224>();
        const int g = (warp - 4) >> 2;
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;
        uint16_t *maps = (uint16_t *)a.maps;
        const bool bf16 = a.map_dt == ATTNCACHE_BF16;
        const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
        uint32_t blk = 0;
        for (uint32_t t = blockIdx.x + g * gridDim.x; t < items; t += stride) {
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
                    mbar_wait(&s_full[g * 2 + buf], bph);
                    tc_fence_after();
                    const uint32_t s_addr = tmem + lane_addr + g * 256 + buf * kBlk;
                    // the whole S row of the block in registers (one TMEM round trip); masked keys -inf
                    uint32_t sv[kBlk];
                    tmem_ld_32x32b_x64(s_addr, sv);
                    tmem_ld_32x32b_x64(s_addr + 64, sv + 64);
                    tmem_ld_wait();
                    tc_fence_before();
                    mbar_arrive(&s_free[g * 2 + buf]);  // S is in registers: the buffer may be refilled
                    if (diag) {
#pragma unroll
                        for (int e = 0; e < kBlk; ++e)
                            if (e > lim) sv[e] = 0xff800000u;
                    }
                    if (pass == 0) {
                        float m8[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) m8[i] = fmaxf(__uint_as_float(sv[i]), __uint_as_float(sv[8 + i]));
#pragma unroll
                        for (int e = 16; e < kBlk; e += 16)
#pragma unroll
                            for (int i = 0; i < 8; ++i)
                                m8[i] = fmaxf(m8[i], fmaxf(__uint_as_float(sv[e + i]), __uint_as_float(sv[e + 8 + i])));
                        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * sl2;
                        const float m_new = fmaxf(m, mx);
                        // row sum on MUFU.EX2 (an FMA-pipe polynomial for 2-8 of every 8 pairs was measured
                        // slower: scripts/capture_poly.sh at configs 1/2)
                        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int e = 0; e < kBlk; ++e) s4[e & 3] += ex2(fmaf(__uint_as_float(sv[e]), sl2, -m_new));
                        l = l * ex2(m - m_new) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
                        m = m_new;
                        if (diag) off = m + lg2(l);  // P = exp2(s*sl2 - off)
                    } else {
                        // this block's columns [128j, 128j + 128) that the row stores
                        const int c0 = j * kBlk;
                        const int ncols = min(kBlk, stored - c0);
#pragma unroll
                        for (int c = 0; c < kBlk / 32; ++c) {
                            uint32_t w[16];
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                const float p0 = ex2(fmaf(__uint_as_float(sv[c * 32 + 2 * e]), sl2, -off));
                                const float p1 = ex2(fmaf(__uint_as_float(sv[c * 32 + 2 * e + 1]), sl2, -off));
                                if (bf16) {
                                    __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                                    w[e] = *reinterpret_cast<uint32_t *>(&h2);
                                } else {
                                    __half2 h2 = __floats2half2_rn(p0, p1);
                                    w[e] = *reinterpret_cast<uint32_t *>(&h2);
                                }
                            }
                            uint4 *dst = (uint4 *)(mrow + c0 + c * 32);
#if defined(CAP_EXP) && CAP_EXP == 1  // experiment: no map stores
                            if (w[0] == 0x12345678u && w[15] == 0x9abcdef0u) dst[0] = make_uint4(w[1], w[2], w[3], w[4]);
#else
#pragma unroll
                            for (int pc = 0; pc < 4; ++pc)
                                if (c * 32 + pc * 8 < ncols) dst[pc] = make_uint4(w[4 * pc], w[4 * pc + 1], w[4 * pc + 2], w[4 * pc + 3]);
#endif
                        }
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
    if (e == cudaSuccess)
        e = make_tmap_2d_16(&tk, a.K, bf16, kD, (uint64_t)a.max_rows * a.L * a.Hkv * a.S, (uint64_t)kD * 2, 64, kBlk, 128);
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
