// kernels_tc_attend.cu — causal softmax attention on tcgen05 (the miss branch of Alg. 2,
// PAPER.md:376-381; Eq. 5): O = softmax(Q K^T * scale, keys j > i masked) . V.
//
// Work item = (unit, 128-query block qb); it visits key blocks j = 0..qb (causal block skipping).
// Two softmax warp groups (WG0 = warps 4-7, WG1 = warps 8-11) own two independent item streams of
// the CTA (items blockIdx.x + (2k + g) * gridDim.x), each with its own loader and MMA thread, and
// share the tensor core: while WG g turns S into P, the pipe runs the other group's S or PV.  Per WG,
// in TMEM:
//   S/P  (128 columns)  S = Q K_j^T (SS MMA, M=128 queries, N=128 keys, K=d, fp32); the softmax
//                       writes bf16 P back over the first 64 columns (two keys per column).
//   O    (d columns)    O += P V_j (TS MMA: A = P from TMEM, B = V MN-major from smem).
// Online softmax with lazy rescaling: P is taken relative to a reference max m_ref that only
// moves (rescaling O in TMEM and l) when the running max exceeds it by more than 8 (log2 units),
// so P <= 2^8 and the correction is rare.  At the item's end O / l is rounded, staged per warp in a
// 128B-swizzled shared tile and written with TMA stores.
// Roles (384 threads): per group g, warp 2g loads its Q (per item), K_j and V_j by TMA and warp 2g+1
// issues its MMAs (warp 1 also owns TMEM); the producer warpgroup drops to 56 registers, warps 4-11 the two
// softmax/epilogue groups with 224 registers each (TMEM lane quarter = warp % 4), which keep the
// whole S row in registers: one TMEM load per key block, packed f32x2 FMA/add.
#include "kernels.cuh"
#include "sm100.cuh"

#include <type_traits>

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 384;  // 3 warpgroups: producers (warps 0-3), softmax group 0 (4-7), group 1 (8-11)
constexpr int kBlk = 128;                 // queries per item = keys per block
constexpr float kRescaleThreshold = 8.f;  // log2 units: P <= 2^8 between rescales

#ifndef ATT_DEPTH
#define ATT_DEPTH 1
#endif
template <int kD>
struct Cfg {
    static constexpr int kTile = kBlk * kD * 2;       // one [128][d] 16-bit tile
    static constexpr int kDepth = kD == 64 ? ATT_DEPTH : 1;  // Q / K / V slots per group
    static constexpr int kQSlots = kDepth;            // per stream
    static constexpr int kK = 2 * kDepth;             // K: kDepth slots per group
    static constexpr int kV = 2 * kDepth;             // V: kDepth slots per group
    static constexpr int kOutWarp = 32 * 64 * 2;     // per softmax warp: O staging [32 rows][64 cols] (128B swizzle)
    // rows the prologue can select into shared memory (12 B each; 0: the separate select kernel always runs)
    static constexpr int kSelCap = kD == 64 ? 1024 : 0;
    static constexpr int kSmem = (2 * kQSlots + kK + kV) * kTile + 8 * kOutWarp + 1024 + 512 +
                                 (kSelCap ? 16 + 12 * kSelCap : 0);
    static constexpr uint32_t kTmemCols = 512;        // S/P: 2 x 128 at 0; O: 2 x d at 256
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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

#if defined(ATT_TRACE)  // timeline experiment (scripts/attend_trace.py): clock64 stamps of CTA 0
__device__ unsigned long long g_att_trace[2][256][6];     // softmax warps 4 / 8, lane 0, first 256 blocks
__device__ unsigned long long g_att_trace_mma[512][8];    // MMA warp, first 512 events
#define ATT_TRACE_REC(slot)                                                                       \
    do {                                                                                          \
        if (blockIdx.x == 0 && lane == 0 && (warp == 4 || warp == 8) && b < 256)                   \
            g_att_trace[warp == 8][b][slot] = clock64();                                           \
    } while (0)
#define ATT_TRACE_MMA(ev, slot)                                                                   \
    do {                                                                                          \
        if (blockIdx.x == 0 && warp == 1 && (ev) < 512) g_att_trace_mma[(ev)][slot] = clock64();   \
    } while (0)
#else
#define ATT_TRACE_REC(slot) \
    do {                    \
    } while (0)
#define ATT_TRACE_MMA(ev, slot) \
    do {                        \
    } while (0)
#endif

// Key pairs (of every 8) whose exp2 runs as a polynomial on the FMA pipe on off-diagonal blocks.  0: the
// sweep (scripts/attend_poly.sh; configs[3]: 0 -> 1.52 ms, 2 -> 1.54, 3 -> 1.56, 4 -> 1.63) shows the
// softmax is bound by its instruction stream and latency, not by MUFU throughput, on this kernel.
#ifndef ATT_POLY_PAIRS
#define ATT_POLY_PAIRS 0
#endif
constexpr int kPolyPairs = ATT_POLY_PAIRS;

struct Ring {
    uint32_t slot, phase;
};
template <int N>
__device__ __forceinline__ Ring ring(uint32_t i) {
    return {i % N, (i / N) & 1u};
}

// One CTA-local item stream: items t = first, first + stride, ...; item -> (unit, query block qb).  Units are taken in L2-sized groups of `group` units (K/V of a group fit in about
// 48 MB of L2) and inside a group the heaviest query blocks come first: every query block of a unit
// re-reads the unit's K/V blocks, and ordering all units' qb = n_qb-1 blocks first (the previous
// order) made those re-reads come from HBM (3.3x the algorithmic bytes at configs[3]).  The last
// group is the batch's tail, still heaviest first, so the persistent CTAs finish together.
// j walks the item's key blocks.  (The FastDiv decode of item_sched.cuh, which the d = 128 kernel and the
// capture use, measured 3 % slower here at configs[1]: 0.270 -> 0.280 ms, with fewer instructions.)
struct Stream {
    uint32_t t, stride, items, units, per_row, n_qb, S, group, H, Hkv, L;
    const int32_t *rows;
    bool active = false;
    int32_t unit = 0;     // the Q / O unit (outer coordinate of the 3-D tensor maps)
    int32_t kv_unit = 0;  // the K / V unit (its K/V head under grouped-query attention)
    int qb = 0, j = 0;
    __device__ void init(uint32_t first, uint32_t stride_, uint32_t items_, uint32_t units_, uint32_t per_row_,
                         uint32_t n_qb_, uint32_t S_, uint32_t group_, const int32_t *rows_, uint32_t H_, uint32_t Hkv_) {
        t = first, stride = stride_, items = items_, units = units_, per_row = per_row_, n_qb = n_qb_, S = S_;
        group = group_, H = H_, Hkv = Hkv_, L = per_row_ / H_;
        rows = rows_;
        start_item();
    }
    __device__ void start_item() {
        active = t < items;
        if (!active) return;
        const uint32_t gi = t / (group * n_qb), w = t - gi * (group * n_qb);
        const uint32_t gbase = gi * group, gsize = min(group, units - gbase);
        const uint32_t u = gbase + w % gsize;
        qb = (int)(n_qb - 1 - w / gsize);
        const int64_t row = rows[u / per_row];
        const uint32_t lh = u % per_row;
        unit = (int32_t)(row * per_row + lh);
        kv_unit = (int32_t)((row * L + lh / H) * Hkv + (lh % H) / (H / Hkv));
        j = 0;
    }
    // Moves past the current key block; returns true when that block ended the item.
    __device__ bool advance() {
        if (++j > qb) {
            t += stride;
            start_item();
            return true;
        }
        return false;
    }
};

// k3D: 3-D [units][S][d] tensor maps (any S: the last, partial block is zero-filled / clipped by TMA);
// else 2-D [units * S][d] maps (S % 128 == 0 and fewer than 2^31 rows), 3 % faster at configs[1]
// (0.275 vs 0.284 ms for the 51 misses; scripts/attend_ab.sh).
template <int kD, bool kBF16, bool k3D>
__global__ void __launch_bounds__(kThreads, 1)
    attend_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     const AttendArgs a, const uint32_t idesc_s, const uint32_t idesc_pv) {
    using C = Cfg<kD>;
    constexpr int NQ = C::kQSlots, NK = C::kK, NV = C::kV, DP = C::kDepth;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = smem;                    // [2 streams][NQ][tile]
    uint8_t *sK = sQ + 2 * NQ * C::kTile;  // [NK][tile]
    uint8_t *sV = sK + NK * C::kTile;      // [NV][tile]
    uint8_t *sOut = sV + NV * C::kTile;    // [8 softmax warps][kOutWarp]
    uint64_t *bars = (uint64_t *)(sOut + 8 * C::kOutWarp);
    uint64_t *q_full = bars, *q_empty = q_full + 2 * NQ;
    uint64_t *k_full = q_empty + 2 * NQ, *k_empty = k_full + NK;
    uint64_t *v_full = k_empty + NK, *v_empty = v_full + NV;
    uint64_t *s_full = v_empty + NV;   // [2] S of WG g computed
    uint64_t *p_full = s_full + 2;     // [2] P of WG g written (128 arrivals)
    uint64_t *pv_done = p_full + 2;    // [2] PV of WG g retired (S/P buffer reusable, O complete)
    uint32_t *tmem_slot = (uint32_t *)(pv_done + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2 * NQ; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < NK; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < NV; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int g = 0; g < 2; ++g) {
            mbar_init(&s_full[g], 1);
            mbar_init(&p_full[g], 128);
            mbar_init(&pv_done[g], 1);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    RowList list = a.list;
    if constexpr (C::kSelCap > 0) {
        if (a.sel.n > 0) {  // row selection in the prologue (no select launch): every CTA builds the same list
            uint8_t *sel_base = (uint8_t *)bars + 512;  // after the 512 barrier bytes
            list.count = (int32_t *)sel_base;
            list.rows = (int32_t *)(sel_base + 16);
            list.ents = (int64_t *)(sel_base + 16 + 4 * C::kSelCap);
            list.cap = C::kSelCap;
            compact_rows(a.sel.n, [&](int64_t b, int64_t &ent) { return select_attend_pred(a.sel, b, ent); }, list);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t S = (uint32_t)a.S;
    // a last, partial block when S % 128 != 0: Q / K / V rows past S read as zeros (3-D tensor maps) and only
    // padded query rows (never stored: the O store clips at S) see padded keys through the causal mask
    const uint32_t n_qb = (S + kBlk - 1) / kBlk;
    const uint32_t per_row = (uint32_t)(a.L * a.H);
    const uint32_t units = (uint32_t)(*list.count) * per_row;
    const uint32_t items = units * n_qb;
    const uint32_t stride = 2 * gridDim.x;
    const uint32_t l2_group = max(1u, (48u << 20) / (2u * S * kD * 2u));  // units whose K and V fit in ~48 MB

    if (warp < 4) {
        // Producer warpgroup: two independent per-group pipelines.  Group g (= item stream g) has its own
        // loader thread (warp 2g: Q per item, K_j and V_j per key block, one smem slot each) and its own
        // MMA-issuing thread (warp 2g+1: S_j, then PV_j once the group's softmax has written P_j).  Both
        // MMA threads feed the one tensor pipe, so while one thread waits for its softmax or pays the
        // per-event bookkeeping the other keeps the pipe busy (a single issuing thread left it idle for
        // ~45% of each key block, measured with scripts/attend_trace.py).  The registers go to the
        // softmax groups (setmaxnreg; the register file is split per SM sub-partition, each holding one
        // warp of every warpgroup: 56 + 2 x 224).
        setmaxnreg_dec<56>();
        const int g = warp >> 1;
        if (lane == 0) {
            Stream st;
            st.init(blockIdx.x + g * gridDim.x, stride, items, units, per_row, n_qb, S, l2_group, list.rows, a.H, a.Hkv);
            uint32_t b = 0, it = 0;  // key blocks and items of this stream
            if ((warp & 1) == 0) {
                // ------------------------------ TMA loader of group g ----------------------------
                while (st.active) {
                    AC_STRESS_DELAY(137u);
                    const int32_t r_j = st.j * kBlk;
                    if (st.j == 0) {
                        const uint32_t qs = g * DP + it % DP, q_s = smem_u32(sQ + qs * C::kTile);
                        mbar_wait(&q_empty[qs], ((it / DP) & 1u) ^ 1u);
                        mbar_arrive_expect_tx(&q_full[qs], C::kTile);
                        for (int h = 0; h < kD / 64; ++h) {
                            if constexpr (k3D)
                                tma_load_3d(q_s + h * (kBlk * 128), &tmQ, &q_full[qs], h * 64, st.qb * kBlk, st.unit);
                            else
                                tma_load_2d(q_s + h * (kBlk * 128), &tmQ, &q_full[qs], h * 64, st.unit * S + st.qb * kBlk);
                        }
                    }
                    const uint32_t ks = g * DP + b % DP, k_s = smem_u32(sK + ks * C::kTile);
                    const uint32_t v_s = smem_u32(sV + ks * C::kTile);
                    mbar_wait(&k_empty[ks], ((b / DP) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&k_full[ks], C::kTile);
                    for (int h = 0; h < kD / 64; ++h) {
                        if constexpr (k3D)
                            tma_load_3d(k_s + h * (kBlk * 128), &tmK, &k_full[ks], h * 64, r_j, st.kv_unit);
                        else
                            tma_load_2d(k_s + h * (kBlk * 128), &tmK, &k_full[ks], h * 64, st.kv_unit * S + r_j);
                    }
                    mbar_wait(&v_empty[ks], ((b / DP) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&v_full[ks], C::kTile);
                    for (int h = 0; h < kD / 64; ++h) {
                        if constexpr (k3D)
                            tma_load_3d(v_s + h * (kBlk * 128), &tmV, &v_full[ks], h * 64, r_j, st.kv_unit);
                        else
                            tma_load_2d(v_s + h * (kBlk * 128), &tmV, &v_full[ks], h * 64, st.kv_unit * S + r_j);
                    }
                    ++b;
                    if (st.advance()) ++it;
                }
            } else {
                // ------------------------------ MMA issuer of group g ----------------------------
                // S_j overwrites the S/P columns PV_{j-1} reads: tcgen05.mma ops of one thread execute in
                // issue order (the tcgen05 pipeline), so S_j is issued right behind PV_{j-1}.
                const uint32_t s_t = tmem + g * kBlk, o_t = tmem + 256 + g * kD;
                while (st.active) {
                    AC_STRESS_DELAY(17u);
                    const int j = st.j;
                    const uint32_t qs = g * DP + it % DP, ks = g * DP + b % DP;
                    const uint32_t q_b = smem_u32(sQ + qs * C::kTile), k_b = smem_u32(sK + ks * C::kTile);
                    const uint32_t v_b = smem_u32(sV + ks * C::kTile);
                    ATT_TRACE_MMA(b * 2 + g, 0);
                    if (j == 0) mbar_wait(&q_full[qs], (it / DP) & 1u);
                    mbar_wait(&k_full[ks], (b / DP) & 1u);
                    ATT_TRACE_MMA(b * 2 + g, 1);
                    tc_fence_after();
                    if constexpr (kD == 128) {  // 8 K-steps of 16 over two 64-column swizzle halves
                        umma_f16_ss_k8<kBlk * 128 / 16>(s_t, smem_desc(q_b, 16, 1024, kSwizzle128B),
                                                       smem_desc(k_b, 16, 1024, kSwizzle128B), idesc_s, 0u);
                    } else {  // d = 64: 4 K-steps inside one swizzle atom column
#pragma unroll
                        for (int k = 0; k < kD / 16; ++k)
                            umma_f16(s_t, smem_desc(q_b + k * 32, 16, 1024, kSwizzle128B),
                                     smem_desc(k_b + k * 32, 16, 1024, kSwizzle128B), idesc_s, k != 0);
                    }
                    umma_commit(&s_full[g]);
                    umma_commit(&k_empty[ks]);
                    if (j == st.qb) umma_commit(&q_empty[qs]);
                    ATT_TRACE_MMA(b * 2 + g, 2);
                    mbar_wait(&p_full[g], b & 1u);
                    ATT_TRACE_MMA(b * 2 + g, 4);
                    mbar_wait(&v_full[ks], (b / DP) & 1u);
                    ATT_TRACE_MMA(b * 2 + g, 5);
                    tc_fence_after();
                    // A = P (8 TMEM columns = 16 keys per step), B = V MN-major: 8 steps in one statement
                    umma_f16_ts_k8(o_t, s_t, smem_desc(v_b, kBlk * 128, 1024, kSwizzle128B), idesc_pv, j == 0 ? 0u : 1u);
                    umma_commit(&v_empty[ks]);
                    umma_commit(&pv_done[g]);
                    ATT_TRACE_MMA(b * 2 + g, 6);
                    ++b;
                    if (st.advance()) ++it;
                }
            }
        }
    } else {
        // ------------------------------ softmax + epilogue (one WG per stream) -------------------
        setmaxnreg_inc<224>();  // the whole S row (128 fp32) stays in registers
        const int g = (warp - 4) >> 2;
        const int q = warp & 3;       // TMEM lane quarter
        const int r = q * 32 + lane;  // query row inside the block == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const uint32_t s_addr = tmem + lane_addr + g * kBlk;
        const uint32_t o_addr = tmem + lane_addr + 256 + g * kD;
        uint8_t *stage_o = sOut + (warp - 4) * C::kOutWarp;
        const uint32_t stage_o_u32 = smem_u32(stage_o);
        const float sl2 = a.scale * 1.4426950408889634f;  // scale * log2(e)
        Stream s;
        s.init(blockIdx.x + g * gridDim.x, stride, items, units, per_row, n_qb, S, l2_group, list.rows, a.H, a.Hkv);
        uint32_t b = 0;  // key blocks of this stream
        float m_ref = 0.f, l = 0.f;
        while (s.active) {
            AC_STRESS_DELAY(818u);
            const int j = s.j;
            const bool diag = j == s.qb;
            const int lim = diag ? r : kBlk - 1;            // keys k <= lim are visible (causal mask)
            ATT_TRACE_REC(0);
            mbar_wait(&s_full[g], b & 1u);
            ATT_TRACE_REC(1);
            tc_fence_after();
            // The whole S row (128 keys) is loaded from TMEM once (two back-to-back loads, one wait) and
            // kept in registers for the max and the exponentials.  Diagonal blocks set keys k > r to -inf,
            // which the exponential turns into an exact 0.
            {
            uint32_t sv[kBlk];
            tmem_ld_32x32b_x64(s_addr, sv);
            tmem_ld_32x32b_x64(s_addr + 64, sv + 64);
            tmem_ld_wait();
            ATT_TRACE_REC(2);
            if (diag) {
#pragma unroll
                for (int e = 0; e < kBlk; ++e)
                    if (e > lim) sv[e] = 0xff800000u;  // -inf
            }
            float m8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) m8[i] = fmaxf(__uint_as_float(sv[i]), __uint_as_float(sv[8 + i]));
#pragma unroll
            for (int e = 16; e < kBlk; e += 16)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    m8[i] = fmaxf(m8[i], fmaxf(__uint_as_float(sv[e + i]), __uint_as_float(sv[e + 8 + i])));
            const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                   fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
            ATT_TRACE_REC(3);
            const float m_blk = mx * sl2;
            if (j == 0) {
                m_ref = m_blk;
                l = 0.f;
            } else if (m_blk > m_ref + kRescaleThreshold) {
                // lazy rescale of O (every PV so far; complete once the previous PV retired) and l
                const float alpha = ex2(m_ref - m_blk);
                mbar_wait(&pv_done[g], (b - 1) & 1u);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < kD / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(o_addr + c * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t w[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) w[e] = __float_as_uint(__uint_as_float(v[h * 16 + e]) * alpha);
                        tmem_st_32x32b_x16(o_addr + c * 32 + h * 16, w);
                    }
                }
                l *= alpha;
                m_ref = m_blk;
            }
            // p = exp2(s * scale * log2e - m_ref) for key pairs (packed f32x2 FMA / add), rounded to the MMA
            // dtype two keys per 32-bit word, written in place (sv[e] <- keys 2e, 2e+1) and then over the
            // consumed S columns; l sums the unrounded p (an unbiased estimate of the rounded sum, within
            // 2^-9 relative; keeps the row sum off the critical path).
            {
                const uint64_t scale2 = pack2(sl2, sl2), neg_m2 = pack2(-m_ref, -m_ref);
                uint64_t rs2[4] = {0ull, 0ull, 0ull, 0ull};
                // Off-diagonal blocks may compute kPolyPairs of every 8 key pairs with a polynomial exp2 on
                // the FMA pipe (exp2_poly2), the rest on MUFU.EX2; diagonal blocks (masked keys at -inf)
                // use MUFU only.
                auto exp_pass = [&](auto poly) {
#pragma unroll
                    for (int c = 0; c < kBlk / 32; ++c) {
                        // diagonal blocks: warp q's rows are < 32(q+1), so its key chunks c > q are all masked:
                        // P = 0 there without spending MUFU work (a warp-uniform branch)
                        if (!decltype(poly)::value && c > q) {
#pragma unroll
                            for (int i = 0; i < 16; ++i) sv[c * 16 + i] = 0u;
                            continue;
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int e = c * 16 + i;
                            const uint64_t x2 = ffma2(((uint64_t)sv[2 * e + 1] << 32) | sv[2 * e], scale2, neg_m2);
                            float p0, p1;
                            if (decltype(poly)::value && (e & 7) < kPolyPairs) {
                                exp2_poly2(x2, p0, p1);
                            } else {
                                p0 = ex2(__uint_as_float((uint32_t)x2));
                                p1 = ex2(__uint_as_float((uint32_t)(x2 >> 32)));
                            }
                            rs2[e & 3] = fadd2(rs2[e & 3], pack2(p0, p1));
                            if constexpr (kBF16) {
                                __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                                sv[e] = *reinterpret_cast<uint32_t *>(&h2);
                            } else {
                                __half2 h2 = __floats2half2_rn(p0, p1);
                                sv[e] = *reinterpret_cast<uint32_t *>(&h2);
                            }
                        }
                    }
                };
                if (diag)
                    exp_pass(std::false_type{});
                else
                    exp_pass(std::true_type{});
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t w[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) w[e] = sv[c * 16 + e];
                    tmem_st_32x32b_x16(s_addr + c * 16, w);  // keys [32c, 32c+32) -> P columns [16c, 16c+16)
                }
                const uint64_t t2 = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
                l += __uint_as_float((uint32_t)t2) + __uint_as_float((uint32_t)(t2 >> 32));
            }
            }
            tmem_st_wait();
            ATT_TRACE_REC(4);
            tc_fence_before();
            mbar_arrive(&p_full[g]);
            ATT_TRACE_REC(5);
            if (diag) {
                // epilogue: the item's last PV retired -> O / l -> act dtype -> 32-byte stores
                mbar_wait(&pv_done[g], b & 1u);
                tc_fence_after();
                const float inv = 1.f / l;
                // TMEM -> registers -> act dtype -> this warp's 128B-swizzled staging tile -> TMA store of the
                // warp's 32 rows, 64 columns at a time (full-line writes; per-thread row stores stalled the
                // group on the LSU and delayed its next P)
                const int32_t orow = s.qb * kBlk + q * 32;  // rows >= S are clipped by the tensor map
#pragma unroll
                for (int half = 0; half < kD / 64; ++half) {
                    uint32_t v[64];
                    tmem_ld_32x32b_x32(o_addr + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    tmem_ld_32x32b_x32(o_addr + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    tmem_ld_wait();
                    if (lane == 0) bulk_wait_read<0>();  // the previous TMA store has read the staging tile
                    __syncwarp();
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        uint32_t w[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float lo = __uint_as_float(v[c8 * 8 + 2 * e]) * inv;
                            const float hi = __uint_as_float(v[c8 * 8 + 2 * e + 1]) * inv;
                            if constexpr (kBF16) {
                                __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
                                w[e] = *reinterpret_cast<uint32_t *>(&h2);
                            } else {
                                __half2 h2 = __floats2half2_rn(lo, hi);
                                w[e] = *reinterpret_cast<uint32_t *>(&h2);
                            }
                        }
                        *reinterpret_cast<uint4 *>(stage_o + sw128_offset(lane, c8)) = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (k3D)
                            tma_store_3d(&tmO, stage_o_u32, half * 64, orow, s.unit);
                        else
                            tma_store_2d(&tmO, stage_o_u32, half * 64, s.unit * S + orow);
                        bulk_commit();
                    }
                }
                tc_fence_before();
            }
            ++b;
            s.advance();
        }
        if (lane == 0) bulk_wait<0>();  // O stores complete before the CTA (and its smem) retires
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

template <int kD, bool kBF16, bool k3D>
cudaError_t launch_t(const AttendArgs &a, int sm_count, cudaStream_t st) {
    using C = Cfg<kD>;
    const bool bf16 = a.dt == ATTNCACHE_BF16;
    CUtensorMap tq, tk, tv, to;
    cudaError_t e;
    if constexpr (!k3D) {
    const uint64_t rows = (uint64_t)a.max_rows * a.L * a.H * a.S, kvrows = (uint64_t)a.max_rows * a.L * a.Hkv * a.S;
    e = make_tmap_2d_16(&tq, a.Q, bf16, kD, rows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&to, a.O, bf16, kD, rows, (uint64_t)kD * 2, 64, 32, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tk, a.K, bf16, kD, kvrows, (uint64_t)kD * 2, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tv, a.V, bf16, kD, kvrows, (uint64_t)kD * 2, 64, kBlk, 128);
    } else {
        e = make_attend_tmaps(a, kD, &tq, &tk, &tv, &to);
    }
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attend_tc_kernel<kD, kBF16, k3D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t fmt = bf16 ? 1u : 0u;
    const uint32_t idesc_s = idesc_f16(kBlk, kBlk, fmt, 0u, 0u);  // Q K-major x K K-major
    const uint32_t idesc_pv = idesc_f16(kBlk, kD, fmt, 0u, 1u);   // P (TMEM) x V MN-major
    attend_tc_kernel<kD, kBF16, k3D><<<sm_count, kThreads, C::kSmem, st>>>(tq, tk, tv, to, a, idesc_s, idesc_pv);
    count_launches(1);
    return cudaGetLastError();
}

template <int kD, bool kBF16>
cudaError_t launch(const AttendArgs &a, int sm_count, cudaStream_t st) {
    const bool flat = a.S % kBlk == 0 && (uint64_t)a.max_rows * a.L * a.H * a.S < (1ull << 31);
    return flat ? launch_t<kD, kBF16, false>(a, sm_count, st) : launch_t<kD, kBF16, true>(a, sm_count, st);
}

}  // namespace

cudaError_t make_attend_tmaps(const AttendArgs &a, int d, CUtensorMap *tq, CUtensorMap *tk, CUtensorMap *tv,
                              CUtensorMap *to) {
    const bool bf16 = a.dt == ATTNCACHE_BF16;
    const uint64_t units = (uint64_t)a.max_rows * a.L * a.H, kvunits = (uint64_t)a.max_rows * a.L * a.Hkv;
    const uint64_t row = (uint64_t)d * 2, plane = (uint64_t)a.S * d * 2;
    cudaError_t e = make_tmap_3d_16(tq, a.Q, bf16, d, a.S, units, row, plane, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_3d_16(to, a.O, bf16, d, a.S, units, row, plane, 64, 32, 128);
    if (e == cudaSuccess) e = make_tmap_3d_16(tk, a.K, bf16, d, a.S, kvunits, row, plane, 64, kBlk, 128);
    if (e == cudaSuccess) e = make_tmap_3d_16(tv, a.V, bf16, d, a.S, kvunits, row, plane, 64, kBlk, 128);
    return e;
}

bool attend_tc_supported(int32_t dt, int32_t S, int32_t d) {
    return (dt == ATTNCACHE_BF16 || dt == ATTNCACHE_F16) && S >= 1 && (d == 64 || d == 128);
}

bool attend_tc_fused_select(const AttendArgs &a, int64_t n_rows) {
    // the two-group kernel (d = 64) and the split kernel (d = 128) select up to their kSelCap rows in the prologue
    if (!attend_tc_supported(a.dt, a.S, a.d) || n_rows <= 0) return false;
#if defined(ATT_TWO_GROUP128)
    if (a.d == 128) return false;
#endif
    return n_rows <= (a.d == 64 ? Cfg<64>::kSelCap : attend_split_sel_cap());
}

cudaError_t launch_attend_tc(const AttendArgs &a, int sm_count, cudaStream_t st) {
    // unit indices are int32 TMA coordinates; items = units * ceil(S / 128) is a uint32 loop bound
    const uint64_t units = (uint64_t)a.max_rows * a.L * a.H;
    if (units >= (1ull << 31) || units * ((a.S + kBlk - 1) / kBlk) >= (1ull << 31)) return cudaErrorInvalidValue;
    // d = 64 uses the same two-group kernel (the earlier two-CTA-per-SM d = 64 kernel with O in registers
    // reached 78 % of the HBM roofline at configs[1]; this one 94 %)
    if (a.d == 64) return a.dt == ATTNCACHE_BF16 ? launch<64, true>(a, sm_count, st) : launch<64, false>(a, sm_count, st);
    // d = 128: the double-buffered-S, column-split kernel (kernels_tc_attend2.cu; configs[2] 0.63 -> 0.60 ms,
    // configs[3] 1.51 -> 1.49 ms against this file's two-group kernel, kept for d = 64 and under
    // ATT_TWO_GROUP128 for comparison)
#if defined(ATT_TWO_GROUP128)
    return a.dt == ATTNCACHE_BF16 ? launch<128, true>(a, sm_count, st) : launch<128, false>(a, sm_count, st);
#else
    return launch_attend_split(a, sm_count, st);
#endif
}

}  // namespace ac
#if defined(ATT_TRACE)
extern "C" int attncache_debug_att_trace(void *out) {
    return (int)cudaMemcpyFromSymbol(out, ac::g_att_trace, sizeof(ac::g_att_trace));
}
extern "C" int attncache_debug_att_trace_mma(void *out) {
    return (int)cudaMemcpyFromSymbol(out, ac::g_att_trace_mma, sizeof(ac::g_att_trace_mma));
}
#endif
