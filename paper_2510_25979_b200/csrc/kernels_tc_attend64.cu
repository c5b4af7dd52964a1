// kernels_tc_attend64.cu — causal softmax attention on tcgen05, d = 64 variant (the miss branch of Alg. 2,
// PAPER.md:376-381; Eq. 5): O = softmax(Q K^T * scale, keys j > i masked) . V.
//
// Work item = (unit, 128-query block qb); it visits key blocks j = 0..qb (causal block skipping).
// Per key block (global block counter blk, double-buffered in TMEM):
//   S   = Q K_j^T            tcgen05 SS, M=128 queries, N=128 keys, K=d; fp32 in TMEM cols [128b, 128b+128)
//   P   = exp2(S*scale*log2e - m)  one query row per thread; bf16 P written back over the first 64
//                            columns of the same S buffer (two keys per 32-bit column)
//   PV  = P V_j              tcgen05 TS (A = P from TMEM), M=128, N=d, K=128 keys; fp32 in TMEM
//   O   = (O + PV_prev) * exp2(m_prev - m)  in fp32 registers; O / l at the item's end.
// The softmax of block blk overlaps the tensor core's PV of block blk-1 (software pipeline that
// runs across item boundaries).  Q, K and V stream through separate TMA rings so Q and K slots are
// released as soon as their S MMA retires.
// Roles (192 threads): warp 0 TMA loader, warp 1 MMA issuer + TMEM owner, warps 2-5 softmax/epilogue.
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {


constexpr int kThreads = 192;
constexpr int kBlk = 128;  // queries per item = keys per block

// kTwoCTA: two co-resident CTAs per SM (d = 64), each with one S/P buffer, 2-slot rings and 256 TMEM
// columns, so one CTA's softmax latency hides behind the other's; else one CTA per SM with
// double-buffered S/P.
template <int kD, bool kTwoCTA>
struct Cfg {
    static constexpr int kTile = kBlk * kD * 2;                          // one [128][d] 16-bit tile
    static constexpr int kRing = kTwoCTA ? 2 : (kD == 64 ? 4 : 2);      // slots per Q / K / V ring
    static constexpr int kSBufs = kTwoCTA ? 1 : 2;                       // S/P buffers (128 cols each)
    static constexpr uint32_t kPVBase = 128 * kSBufs;                    // PV: 2 x d columns
    static constexpr uint32_t kTmemCols = kTwoCTA ? 256 : 512;
    static constexpr int kMinBlocks = kTwoCTA ? 2 : 1;
    static constexpr int kSmem = 3 * kRing * kTile + 1024 + 512;
    static_assert(kPVBase + 2 * kD <= kTmemCols, "TMEM budget");
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct Ring {
    uint32_t slot, phase;
};
template <int N>
__device__ __forceinline__ Ring ring(uint32_t i) {
    return {i % N, (i / N) & 1u};
}

template <int kD, bool kTwoCTA>
__global__ void __launch_bounds__(kThreads, Cfg<kD, kTwoCTA>::kMinBlocks)
    attend64_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttendArgs a, const uint32_t idesc_s,
                     const uint32_t idesc_pv) {
    using C = Cfg<kD, kTwoCTA>;
    constexpr int R = C::kRing;
    constexpr int NS = C::kSBufs;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = smem, *sK = smem + R * C::kTile, *sV = smem + 2 * R * C::kTile;
    uint64_t *bars = (uint64_t *)(smem + 3 * R * C::kTile);
    uint64_t *q_full = bars, *q_empty = q_full + R;
    uint64_t *k_full = q_empty + R, *k_empty = k_full + R;
    uint64_t *v_full = k_empty + R, *v_empty = v_full + R;
    uint64_t *s_full = v_empty + R;    // [2] S computed
    uint64_t *p_full = s_full + 2;     // [2] P written (128 threads)
    uint64_t *s_free = p_full + 2;     // [2] the PV that read P retired: S/P buffer reusable
    uint64_t *pv_full = s_free + 2;    // [2]
    uint64_t *pv_empty = pv_full + 2;  // [2] (128 threads)
    uint32_t *tmem_slot = (uint32_t *)(pv_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&s_free[i], 1);
            mbar_init(&pv_full[i], 1);
            mbar_init(&pv_empty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
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
    // item t -> (unit, qb): units in L2-sized groups (their K and V fit in ~48 MB, so a unit's query
    // blocks re-read K/V from L2), heaviest query blocks first inside a group so the persistent CTAs
    // finish together (kernels_tc_attend.cu, Stream).
    const uint32_t l2_group = max(1u, (48u << 20) / (2u * S * kD * 2u));
    auto decode = [&](uint32_t t, int64_t &unit_row0, int &qb) {
        const uint32_t gi = t / (l2_group * n_qb), w = t - gi * (l2_group * n_qb);
        const uint32_t gbase = gi * l2_group, gsize = min(l2_group, units - gbase);
        qb = (int)(n_qb - 1 - w / gsize);
        const uint32_t u = gbase + w % gsize;
        unit_row0 = ((int64_t)a.list.rows[u / per_row] * per_row + u % per_row) * S;
    };

    if (warp == 0) {
        // ------------------------------ TMA loader -------------------------------------------
        if (lane == 0) {
            uint32_t it = 0, blk = 0;
            for (uint32_t t = blockIdx.x; t < items; t += gridDim.x, ++it) {
                int64_t row0;
                int qb;
                decode(t, row0, qb);
                const Ring rq = ring<R>(it);
                mbar_wait(&q_empty[rq.slot], rq.phase ^ 1u);
                mbar_arrive_expect_tx(&q_full[rq.slot], C::kTile);
                for (int h = 0; h < kD / 64; ++h)
                    tma_load_2d(smem_u32(sQ + rq.slot * C::kTile + h * (kBlk * 128)), &tmQ, &q_full[rq.slot], h * 64,
                                (int32_t)(row0 + qb * kBlk));
                for (int j = 0; j <= qb; ++j, ++blk) {
                    const Ring rk = ring<R>(blk);
                    mbar_wait(&k_empty[rk.slot], rk.phase ^ 1u);
                    mbar_arrive_expect_tx(&k_full[rk.slot], C::kTile);
                    for (int h = 0; h < kD / 64; ++h)
                        tma_load_2d(smem_u32(sK + rk.slot * C::kTile + h * (kBlk * 128)), &tmK, &k_full[rk.slot],
                                    h * 64, (int32_t)(row0 + j * kBlk));
                    mbar_wait(&v_empty[rk.slot], rk.phase ^ 1u);
                    mbar_arrive_expect_tx(&v_full[rk.slot], C::kTile);
                    for (int h = 0; h < kD / 64; ++h)
                        tma_load_2d(smem_u32(sV + rk.slot * C::kTile + h * (kBlk * 128)), &tmV, &v_full[rk.slot],
                                    h * 64, (int32_t)(row0 + j * kBlk));
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer -------------------------------------------
        if (lane == 0) {
            auto issue_pv = [&](uint32_t c) {
                const Ring rv = ring<R>(c);
                const Ring rs = ring<NS>(c);                        // S/P buffer
                const uint32_t buf = c & 1u, bph = (c >> 1) & 1u;   // PV buffer
                mbar_wait(&p_full[rs.slot], rs.phase);
                mbar_wait(&v_full[rv.slot], rv.phase);
                mbar_wait(&pv_empty[buf], bph ^ 1u);
                tc_fence_after();
                const uint32_t v_base = smem_u32(sV + rv.slot * C::kTile);
                const uint32_t d_tmem = tmem + C::kPVBase + buf * kD;
#pragma unroll
                for (int k = 0; k < kBlk / 16; ++k) {
                    // A = P in TMEM (8 columns = 16 keys per step); B = V, MN-major SW128, 16 rows per step
                    const uint64_t bd = smem_desc(v_base + k * 2048, kBlk * 128, 1024, kSwizzle128B);
                    umma_f16_ts(d_tmem, tmem + rs.slot * kBlk + k * 8, bd, idesc_pv, k != 0);
                }
                umma_commit(&pv_full[buf]);
                umma_commit(&v_empty[rv.slot]);
                umma_commit(&s_free[rs.slot]);
            };
            uint32_t it = 0, blk = 0;
            for (uint32_t t = blockIdx.x; t < items; t += gridDim.x, ++it) {
                int64_t row0;
                int qb;
                decode(t, row0, qb);
                const Ring rq = ring<R>(it);
                mbar_wait(&q_full[rq.slot], rq.phase);
                const uint32_t q_base = smem_u32(sQ + rq.slot * C::kTile);
                for (int j = 0; j <= qb; ++j, ++blk) {
                    const Ring rk = ring<R>(blk);
                    const Ring rs = ring<NS>(blk);
                    const uint32_t buf = rs.slot;
                    // With one S/P buffer, S(blk) reuses the buffer PV(blk-1) reads: issue PV first.
                    if (NS == 1 && blk > 0) issue_pv(blk - 1);
                    mbar_wait(&k_full[rk.slot], rk.phase);
                    mbar_wait(&s_free[buf], rs.phase ^ 1u);
                    tc_fence_after();
                    const uint32_t k_base = smem_u32(sK + rk.slot * C::kTile);
#pragma unroll
                    for (int k = 0; k < kD / 16; ++k) {
                        const uint32_t off = (k >> 2) * (kBlk * 128) + (k & 3) * 32;
                        umma_f16(tmem + buf * kBlk, smem_desc(q_base + off, 16, 1024, kSwizzle128B),
                                 smem_desc(k_base + off, 16, 1024, kSwizzle128B), idesc_s, k != 0);
                    }
                    umma_commit(&s_full[buf]);
                    umma_commit(&k_empty[rk.slot]);
                    if (j == qb) umma_commit(&q_empty[rq.slot]);
                    if (NS > 1 && blk > 0) issue_pv(blk - 1);
                }
            }
            if (blk > 0) issue_pv(blk - 1);
        }
    } else {
        // ------------------------------ softmax + epilogue -----------------------------------
        const int q = warp & 3;
        const int r = q * 32 + lane;  // query row inside the block == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;  // scale * log2(e)
        uint16_t *O = (uint16_t *)a.O;
        const bool bf16 = a.dt == ATTNCACHE_BF16;
        float o[kD];
#pragma unroll
        for (int c = 0; c < kD; ++c) o[c] = 0.f;
        float m = -INFINITY, l = 0.f;  // running statistics of the current item
        int64_t prev_row0 = 0;         // item whose last PV is pending
        int prev_qb = 0;
        float prev_l = 1.f;
        float alpha = 1.f;
        bool pend = false, pend_last = false;
        uint32_t blk = 0;

        // Folds PV of block blk-1 into o (rescaled by `alpha` unless it closed its item; then the
        // item's epilogue normalises, rounds and stores O and o restarts from zero).
        auto fold_pending = [&]() {
            const uint32_t pb = (blk - 1) & 1u, pph = ((blk - 1) >> 1) & 1u;
            mbar_wait(&pv_full[pb], pph);
            tc_fence_after();
            const float al = pend_last ? 1.f : alpha;
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem + lane_addr + C::kPVBase + pb * kD + c * 32, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) o[c * 32 + e] = (o[c * 32 + e] + __uint_as_float(v[e])) * al;
            }
            tc_fence_before();
            mbar_arrive(&pv_empty[pb]);
            if (pend_last) {
                const float inv = 1.f / prev_l;
                uint16_t *dst = O + (prev_row0 + prev_qb * kBlk + r) * (int64_t)kD;
#pragma unroll
                for (int c16 = 0; c16 < kD / 16; ++c16) {  // 32-byte stores: whole sectors, no partial writes
                    uint32_t w[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float lo = o[c16 * 16 + 2 * e] * inv, hi = o[c16 * 16 + 2 * e + 1] * inv;
                        if (bf16) {
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
                            w[e] = *reinterpret_cast<uint32_t *>(&h2);
                        } else {
                            __half2 h2 = __floats2half2_rn(lo, hi);
                            w[e] = *reinterpret_cast<uint32_t *>(&h2);
                        }
                    }
                    st_global_v8(dst + c16 * 16, w);
                }
#pragma unroll
                for (int c = 0; c < kD; ++c) o[c] = 0.f;
            }
        };

        for (uint32_t t = blockIdx.x; t < items; t += gridDim.x) {
            int64_t row0;
            int qb;
            decode(t, row0, qb);
            m = -INFINITY;
            l = 0.f;
            for (int j = 0; j <= qb; ++j, ++blk) {
                const Ring rsb = ring<NS>(blk);
                const uint32_t buf = rsb.slot, bph = rsb.phase;
                const bool diag = j == qb;
                const int lim = diag ? r : kBlk - 1;            // keys k <= lim are visible (causal mask)
                const int n_chunks = diag ? q + 1 : kBlk / 32;  // warp-uniform: 32-key chunks with visible keys
                mbar_wait(&s_full[buf], bph);
                tc_fence_after();
                const uint32_t s_addr = tmem + lane_addr + buf * kBlk;
                float mx = -INFINITY;
                for (int c = 0; c < n_chunks; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(s_addr + c * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (c * 32 + e <= lim) mx = fmaxf(mx, __uint_as_float(v[e]));
                }
                const float m_new = fmaxf(m, mx * sl2);
                float rs = 0.f;
#pragma unroll
                for (int c = 0; c < kBlk / 32; ++c) {
                    uint32_t w[16];
                    if (c < n_chunks) {
                        uint32_t v[32];
                        tmem_ld_32x32b_x32(s_addr + c * 32, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const int k0 = c * 32 + 2 * e;
                            const float p0 = k0 <= lim ? ex2(fmaf(__uint_as_float(v[2 * e]), sl2, -m_new)) : 0.f;
                            const float p1 = k0 + 1 <= lim ? ex2(fmaf(__uint_as_float(v[2 * e + 1]), sl2, -m_new)) : 0.f;
                            if (bf16) {
                                __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                                rs += __low2float(h2) + __high2float(h2);
                                w[e] = *reinterpret_cast<uint32_t *>(&h2);
                            } else {
                                __half2 h2 = __floats2half2_rn(p0, p1);
                                rs += __low2float(h2) + __high2float(h2);
                                w[e] = *reinterpret_cast<uint32_t *>(&h2);
                            }
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) w[e] = 0u;
                    }
                    // keys [32c, 32c+32) -> P columns [16c, 16c+16) (already read as S chunk c/2 <= c)
                    tmem_st_32x32b_x16(s_addr + c * 16, w);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[buf]);
                alpha = ex2(m - m_new);  // 0 on an item's first block (m = -inf)
                l = l * alpha + rs;
                m = m_new;
                if (pend) fold_pending();
                pend = true;
                pend_last = diag;
                if (diag) {
                    prev_row0 = row0;
                    prev_qb = qb;
                    prev_l = l;
                }
            }
        }
        if (pend) fold_pending();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

template <int kD, bool kTwoCTA>
cudaError_t launch64(const AttendArgs &a, int sm_count, cudaStream_t st) {
    using C = Cfg<kD, kTwoCTA>;
    const bool bf16 = a.dt == ATTNCACHE_BF16;
    const uint64_t rows = (uint64_t)a.max_rows * a.L * a.H * a.S;
    CUtensorMap tq, tk, tv;
    cudaError_t e = make_tmap_2d_16(&tq, a.Q, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tk, a.K, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tv, a.V, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attend64_kernel<kD, kTwoCTA>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t fmt = bf16 ? 1u : 0u;
    const uint32_t idesc_s = idesc_f16(kBlk, kBlk, fmt, 0u, 0u);  // Q K-major x K K-major
    const uint32_t idesc_pv = idesc_f16(kBlk, kD, fmt, 0u, 1u);   // P (TMEM) x V MN-major
    attend64_kernel<kD, kTwoCTA><<<sm_count * C::kMinBlocks, kThreads, C::kSmem, st>>>(tq, tk, tv, a, idesc_s, idesc_pv);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

// d = 64: two co-resident CTAs per SM, O accumulated in registers (kernels_tc_attend.cu holds the
// two-warp-group TMEM-accumulator kernel used for d = 128).
cudaError_t launch_attend_tc64(const AttendArgs &a, int sm_count, cudaStream_t st) {
    return launch64<64, true>(a, sm_count, st);
}

}  // namespace ac
