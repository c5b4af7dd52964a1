// kernels_tc_attend.cu — causal softmax attention on tcgen05 (the miss branch of Alg. 2,
// PAPER.md:376-381; Eq. 5): O = softmax(Q K^T * scale, keys j > i masked) . V.
//
// Work item = (unit, 128-query block qb); it visits key blocks j = 0..qb (causal block skipping).
// Per key block:  S_j = Q K_j^T   (tcgen05, M=128 queries, N=128 keys, K=d, fp32 in TMEM)
//                 P_j = exp2(S_j*scale*log2e - m_j)  (online softmax, one query row per thread)
//                 PV_j = P_j V_j   (tcgen05, M=128, N=d, K=128 keys; P staged bf16 in smem)
//                 O   = (O + PV_{j-1}) * exp2(m_{j-1} - m_j)   (fp32 registers), O /= l at the end.
// Roles (192 threads): warp 0 TMA loader (Q, K_j, V_j per stage), warp 1 MMA issuer + TMEM owner,
// warps 2-5 softmax + epilogue (TMEM lane quarter = warp % 4).
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 192;
constexpr int kBlk = 128;  // queries per item = keys per block

template <int kD>
struct Cfg {
    static constexpr int kTile = kBlk * kD * 2;      // one [128][d] bf16 tile
    static constexpr int kStageBytes = 3 * kTile;    // Q, K_j, V_j
    static constexpr int kStages = kD == 64 ? 3 : 2;
    static constexpr int kPBufs = kD == 64 ? 2 : 1;
    static constexpr int kPBytes = kBlk * kBlk * 2;  // P tile, two 64-key chunks
    static constexpr int kSmem = kStages * kStageBytes + kPBufs * kPBytes + 1024 + 512;
    static constexpr uint32_t kTmemCols = 512;       // S: 2 x 128 cols, PV: 2 x d cols
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int kD>
__global__ void __launch_bounds__(kThreads, 1)
    attend_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const AttendArgs a, const uint32_t idesc_s,
                     const uint32_t idesc_pv) {
    using C = Cfg<kD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *pbuf = smem + C::kStages * C::kStageBytes;
    uint64_t *bars = (uint64_t *)(pbuf + C::kPBufs * C::kPBytes);
    uint64_t *kv_full = bars;                    // [kStages]
    uint64_t *kv_empty = kv_full + C::kStages;   // [kStages]
    uint64_t *s_full = kv_empty + C::kStages;    // [2]
    uint64_t *s_empty = s_full + 2;              // [2]
    uint64_t *p_full = s_empty + 2;              // [kPBufs]
    uint64_t *p_empty = p_full + C::kPBufs;      // [kPBufs]
    uint64_t *pv_full = p_empty + C::kPBufs;     // [2]
    uint64_t *pv_empty = pv_full + 2;            // [2]
    uint32_t *tmem_slot = (uint32_t *)(pv_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_empty[i], 128);
            mbar_init(&pv_full[i], 1);
            mbar_init(&pv_empty[i], 128);
        }
        for (int i = 0; i < C::kPBufs; ++i) {
            mbar_init(&p_full[i], 128);
            mbar_init(&p_empty[i], 1);
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

    const int S = a.S;
    const int n_qb = S / kBlk;
    const int64_t per_row = (int64_t)a.L * a.H;
    const int64_t units = (int64_t)(*a.list.count) * per_row;
    const int64_t items = units * n_qb;
    // item t -> (unit, qb): heaviest query blocks first so the persistent CTAs finish together
    auto decode = [&](int64_t t, int64_t &unit_row0, int &qb) {
        qb = n_qb - 1 - (int)(t / units);
        const int64_t u = t % units;
        const int64_t slot = u / per_row, lh = u % per_row;
        unit_row0 = ((int64_t)a.list.rows[slot] * per_row + lh) * S;  // first [S][d] row of the unit
    };

    if (warp == 0) {
        // ------------------------------ TMA loader -------------------------------------------
        if (lane == 0) {
            uint32_t cnt = 0;
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
                int64_t row0;
                int qb;
                decode(t, row0, qb);
                for (int j = 0; j <= qb; ++j, ++cnt) {
                    const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                    mbar_wait(&kv_empty[s], ph ^ 1u);
                    mbar_arrive_expect_tx(&kv_full[s], C::kStageBytes);
                    const uint32_t base = smem_u32(smem + s * C::kStageBytes);
#pragma unroll
                    for (int h = 0; h < kD / 64; ++h) {
                        tma_load_2d(base + h * (kBlk * 128), &tmQ, &kv_full[s], h * 64, (int32_t)(row0 + qb * kBlk));
                        tma_load_2d(base + C::kTile + h * (kBlk * 128), &tmK, &kv_full[s], h * 64,
                                    (int32_t)(row0 + j * kBlk));
                        tma_load_2d(base + 2 * C::kTile + h * (kBlk * 128), &tmV, &kv_full[s], h * 64,
                                    (int32_t)(row0 + j * kBlk));
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------ MMA issuer -------------------------------------------
        if (lane == 0) {
            uint32_t cnt = 0;   // key blocks over all items (stage ring, S/PV double buffers)
            auto issue_pv = [&](uint32_t c) {
                const uint32_t s = c % C::kStages;
                const uint32_t pb = c % C::kPBufs, pph = (c / C::kPBufs) & 1u;
                const uint32_t buf = c & 1u, bph = (c >> 1) & 1u;
                mbar_wait(&p_full[pb], pph);
                mbar_wait(&pv_empty[buf], bph ^ 1u);
                tc_fence_after();
                const uint32_t p_base = smem_u32(pbuf + pb * C::kPBytes);
                const uint32_t v_base = smem_u32(smem + s * C::kStageBytes + 2 * C::kTile);
                const uint32_t d_tmem = tmem + 256 + buf * kD;
#pragma unroll
                for (int k = 0; k < kBlk / 16; ++k) {
                    // P: K-major SW128, two 64-key chunks of 16 KB; V: MN-major SW128, 16 rows per step.
                    const uint64_t ad = smem_desc(p_base + (k >> 2) * (kBlk * 128) + (k & 3) * 32, 16, 1024, kSwizzle128B);
                    const uint64_t bd = smem_desc(v_base + k * 2048, kBlk * 128, 1024, kSwizzle128B);
                    umma_f16(d_tmem, ad, bd, idesc_pv, k != 0);
                }
                umma_commit(&pv_full[buf]);
                umma_commit(&p_empty[pb]);
                umma_commit(&kv_empty[s]);
            };
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
                int64_t row0;
                int qb;
                decode(t, row0, qb);
                for (int j = 0; j <= qb; ++j, ++cnt) {
                    const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                    const uint32_t buf = cnt & 1u, bph = (cnt >> 1) & 1u;
                    mbar_wait(&kv_full[s], ph);
                    mbar_wait(&s_empty[buf], bph ^ 1u);
                    tc_fence_after();
                    const uint32_t q_base = smem_u32(smem + s * C::kStageBytes);
                    const uint32_t k_base = q_base + C::kTile;
                    const uint32_t d_tmem = tmem + buf * kBlk;
#pragma unroll
                    for (int k = 0; k < kD / 16; ++k) {
                        const uint32_t off = (k >> 2) * (kBlk * 128) + (k & 3) * 32;
                        const uint64_t ad = smem_desc(q_base + off, 16, 1024, kSwizzle128B);
                        const uint64_t bd = smem_desc(k_base + off, 16, 1024, kSwizzle128B);
                        umma_f16(d_tmem, ad, bd, idesc_s, k != 0);
                    }
                    umma_commit(&s_full[buf]);
                    // PV of the previous key block (possibly of the previous item) overlaps the
                    // softmax of this one: the pipeline runs across item boundaries.
                    if (cnt > 0) issue_pv(cnt - 1);
                }
            }
            if (cnt > 0) issue_pv(cnt - 1);
        }
    } else {
        // ------------------------------ softmax + epilogue -----------------------------------
        // Software-pipelined over key blocks across items: P of block cnt is produced before PV of
        // block cnt-1 is folded in, so the tensor core computes PV(cnt-1) while this warp group
        // runs the exponentials of block cnt; an item's epilogue runs once its last PV is folded.
        const int q = warp & 3;
        const int r = q * 32 + lane;  // query row inside the block == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;  // scale * log2(e)
        uint16_t *O = (uint16_t *)a.O;
        const bool bf16 = a.dt == ATTNCACHE_BF16;
        float o[kD];
#pragma unroll
        for (int c = 0; c < kD; ++c) o[c] = 0.f;
        float m = -INFINITY, l = 0.f;        // running stats of the item being processed
        float alpha_pend = 1.f;              // rescale to apply when folding the pending PV
        int64_t prev_row0 = -1;              // pending item (its last PV not yet folded)
        int prev_qb = 0;
        float prev_l = 0.f;
        bool pend = false;                   // a PV (block cnt-1) is outstanding
        bool pend_last = false;              // ... and it is the last block of its item
        uint32_t cnt = 0;

        auto fold_pending = [&]() {
            const uint32_t pbuf_idx = (cnt - 1) & 1u, pvph = ((cnt - 1) >> 1) & 1u;
            mbar_wait(&pv_full[pbuf_idx], pvph);
            tc_fence_after();
            const float al = pend_last ? 1.f : alpha_pend;
#pragma unroll
            for (int c = 0; c < kD / 32; ++c) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem + lane_addr + 256 + pbuf_idx * kD + c * 32, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) o[c * 32 + e] = (o[c * 32 + e] + __uint_as_float(v[e])) * al;
            }
            tc_fence_before();
            mbar_arrive(&pv_empty[pbuf_idx]);
            if (pend_last) {  // epilogue of the finished item: normalise, round, store
                const float inv = 1.f / prev_l;
                uint4 *dst = (uint4 *)(O + (prev_row0 + prev_qb * kBlk + r) * (int64_t)kD);
#pragma unroll
                for (int c8 = 0; c8 < kD / 8; ++c8) {
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float lo = o[c8 * 8 + 2 * e] * inv, hi = o[c8 * 8 + 2 * e + 1] * inv;
                        if (bf16) {
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
                            w[e] = *reinterpret_cast<uint32_t *>(&h2);
                        } else {
                            __half2 h2 = __floats2half2_rn(lo, hi);
                            w[e] = *reinterpret_cast<uint32_t *>(&h2);
                        }
                    }
                    dst[c8] = make_uint4(w[0], w[1], w[2], w[3]);
                }
#pragma unroll
                for (int c = 0; c < kD; ++c) o[c] = 0.f;
            }
        };

        for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
            int64_t row0;
            int qb;
            decode(t, row0, qb);
            for (int j = 0; j <= qb; ++j, ++cnt) {
                const uint32_t buf = cnt & 1u, bph = (cnt >> 1) & 1u;
                const uint32_t pb = cnt % C::kPBufs, pph = (cnt / C::kPBufs) & 1u;
                const bool diag = j == qb;
                const int lim = diag ? r : kBlk - 1;           // keys k <= lim are visible (causal mask)
                const int n_chunks = diag ? q + 1 : kBlk / 32; // warp-uniform: 32-key chunks with visible keys
                if (j == 0) {
                    m = -INFINITY;
                    l = 0.f;
                }
                mbar_wait(&s_full[buf], bph);
                tc_fence_after();
                const uint32_t s_addr = tmem + lane_addr + buf * kBlk;
                // pass 1: row max of the visible scores
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
                // pass 2: p = exp2(s*scale*log2e - m_new), rounded, written to P (K-major SW128)
                mbar_wait(&p_empty[pb], pph ^ 1u);
                uint8_t *prow = pbuf + pb * C::kPBytes;
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
                    // columns [32c, 32c+32): chunk (32c)/64, 16-byte pieces 4*(c&1) .. +3
                    uint8_t *chunk = prow + (c >> 1) * (kBlk * 128);
#pragma unroll
                    for (int pc = 0; pc < 4; ++pc)
                        *reinterpret_cast<uint4 *>(chunk + sw128_offset(r, (c & 1) * 4 + pc)) =
                            make_uint4(w[4 * pc], w[4 * pc + 1], w[4 * pc + 2], w[4 * pc + 3]);
                }
                tc_fence_before();
                mbar_arrive(&s_empty[buf]);
                fence_proxy_async_smem();
                mbar_arrive(&p_full[pb]);
                const float alpha = ex2(m - m_new);  // 0 on the first block of an item (m = -inf)
                l = l * alpha + rs;
                m = m_new;
                // Fold the previous block's PV (the tensor core computed it while we made P): within
                // an item it is relative to the previous max and is rescaled by this block's alpha;
                // if it closed the previous item, that item's epilogue runs now.
                alpha_pend = alpha;
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

template <int kD>
cudaError_t launch(const AttendArgs &a, int sm_count, cudaStream_t st) {
    using C = Cfg<kD>;
    const bool bf16 = a.dt == ATTNCACHE_BF16;
    const uint64_t rows = (uint64_t)a.max_rows * a.L * a.H * a.S;
    CUtensorMap tq, tk, tv;
    cudaError_t e = make_tmap_2d_16(&tq, a.Q, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tk, a.K, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tv, a.V, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attend_tc_kernel<kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t fmt = bf16 ? 1u : 0u;
    const uint32_t idesc_s = idesc_f16(kBlk, kBlk, fmt, 0u, 0u);   // Q K-major x K K-major
    const uint32_t idesc_pv = idesc_f16(kBlk, kD, fmt, 0u, 1u);    // P K-major x V MN-major
    attend_tc_kernel<kD><<<sm_count, kThreads, C::kSmem, st>>>(tq, tk, tv, a, idesc_s, idesc_pv);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

bool attend_tc_supported(int32_t dt, int32_t S, int32_t d) {
    return (dt == ATTNCACHE_BF16 || dt == ATTNCACHE_F16) && S >= kBlk && S % kBlk == 0 && (d == 64 || d == 128);
}

cudaError_t launch_attend_tc(const AttendArgs &a, int sm_count, cudaStream_t st) {
    if ((uint64_t)a.max_rows * a.L * a.H * a.S >= (1ull << 31)) return cudaErrorInvalidValue;
    return a.d == 64 ? launch<64>(a, sm_count, st) : launch<128>(a, sm_count, st);
}

}  // namespace ac
