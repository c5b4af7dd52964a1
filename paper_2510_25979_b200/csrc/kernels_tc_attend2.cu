// kernels_tc_attend2.cu — causal softmax attention, d = 128, with a double-buffered S and a column-split
// softmax (the miss branch of Alg. 2; Eq. 5):
//   O = softmax(Q K^T * scale, keys j > i masked) . V.
//
// Work item = (unit, 128-query block qb) visiting key blocks j = 0..qb; one item stream per CTA; blocks are
// numbered b across items.  TMEM (384 of 512 columns): two S/P buffers of 128 columns (S_b in buffer b % 2)
// and O (128 columns).  P_b is written over the first 64 columns of its S buffer (two bf16 keys per column).
// The MMA thread issues S_0, S_1, then for every b: PV_b (once the softmax wrote P_b) followed by S_{b+2}
// into the buffer PV_b just read -- tcgen05.mma ops of one thread execute in issue order, so S_{b+2} is
// queued behind PV_b -- and the softmax of block b+1 overlaps PV_b and S_{b+2} on the tensor pipe.
// (kernels_tc_attend.cu keeps one S buffer per group, so a group's next S always waited for its PV.)
// The softmax runs on 8 warps: warp w handles rows 32(w%4)..+31 (its TMEM lane quarter) and key half
// w/4 - 1 (64 keys).  The two warps of a row quarter exchange their partial row maxima through spare TMEM
// columns behind a 64-thread named barrier, so both use the same reference max; each owns half of P and
// half of O (lazy rescale).  Online softmax with lazy rescaling (the reference max moves only when the
// block max exceeds it by > 8 in log2 units).  At an item's last block each writes its row sum to TMEM.
// Roles (512 threads = 4 warpgroups): warp 0 TMA loader (Q per item into a 2-slot ring, K_b / V_b into
// 2-slot rings), warp 1 MMA issuer (the whole warp runs the issue loop, one elected lane issues, so the
// descriptor arithmetic stays in uniform registers) + TMEM owner, warps 2-3 idle; warps 4-7 and 8-11 the
// softmax halves; warps 12-15 the epilogue (O / l -> act dtype -> TMA store), off the softmax's path: the
// MMA restarts O for the next item once the epilogue has read it (o_free).  setmaxnreg moves registers
// from the producers and the epilogue to the softmax warps.  (Epilogue in the softmax warps, deferred past
// the next block's softmax: configs[3] 1.385 ms / configs[2] 0.555 ms; here 1.363 / 0.566.  Double-
// buffering O by item parity, with the exchanges moved to shared memory to make TMEM room: 1.378 / 0.561.)
#include "kernels.cuh"
#include "item_sched.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 512;
constexpr int kBlk = 128;
constexpr int kD = 128;
constexpr float kRescaleThreshold = 8.f;
constexpr int kTile = kBlk * kD * 2;    // one [128][128] 16-bit tile (two 64-column swizzle halves)
constexpr int kOutWarp = 32 * 64 * 2;   // per softmax warp: O staging [32 rows][64 cols]
// Rings: Q 2 slots (one item ahead), K kNK slots, V kNV slots (shared memory holds 6 tiles next to the O staging;
// K 3 / V 1 measured 45 % slower than 2 / 2: a one-slot V ring serializes PV with the next V load; moving the
// V loads to a thread of their own, so K_{b+1} is not held behind V_b, measured 1 % / 9 % slower at configs[3] / [2]).
#ifndef SPLIT_NK
#define SPLIT_NK 2
#endif
#ifndef SPLIT_NV
#define SPLIT_NV (4 - SPLIT_NK)
#endif
#ifndef SPLIT_NQ
#define SPLIT_NQ 2
#endif
#ifndef SPLIT_STAGE
#define SPLIT_STAGE 2  // O staging tiles per epilogue warp (2: the two 64-column halves in flight)
#endif
constexpr int kNK = SPLIT_NK, kNV = SPLIT_NV, kNQ = SPLIT_NQ, kStage = SPLIT_STAGE;
static_assert(kNK >= 1 && kNV >= 1 && kNQ >= 1 && kNK <= 4 && kNV <= 4 && kNQ <= 2, "ring sizes");
constexpr int kSelCap = 128;  // rows the prologue can select into shared memory (12 B each; the rings leave ~1.7 KB)
constexpr int kSmem = (kNQ + kNK + kNV) * kTile + 4 * kStage * kOutWarp + 1024 + 256 + 16 + 12 * kSelCap;
static_assert(kSmem + 160 <= 232448, "shared memory (dynamic + compact_rows static words, 132 B)");
// TMEM columns (of 512): S/P buffers [0, 256), O [256, 384), the pair exchange of partial row maxima
// (parity-double-buffered, kXmax + 2 * parity + half) and the row sums for the epilogue (item-parity
// double-buffered, kXsum + 2 * parity + half) at [384, 392): the warps address their own lanes only.
constexpr uint32_t kOCol = 256, kXmax = 384, kXsum = 388;
// Registers per thread after setmaxnreg (4 warpgroups share 64 K): producers, softmax, epilogue.
constexpr uint32_t kRegProducer = 56, kRegSoftmax = 176, kRegEpilogue = 96;
static_assert(128 * (kRegProducer + 2 * kRegSoftmax + kRegEpilogue) <= 65536, "register file");
constexpr uint32_t kTmemCols = 512;
// Key pairs (of every 8) whose exp2 runs as a polynomial on the FMA pipe on off-diagonal blocks: 0, the
// sweep was slower at every ratio (configs[3]: 0 -> 1.49 ms, 1 -> 1.54, 2 -> 1.58, 4 -> 1.69).
#ifndef SPLIT_POLY
#define SPLIT_POLY 0
#endif
constexpr int kSplitPoly = SPLIT_POLY;

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
// Named barrier over the 64 threads of one row quarter's two softmax warps.
__device__ __forceinline__ void pair_sync(int q) { asm volatile("bar.sync %0, 64;" ::"r"(q + 1) : "memory"); }

// Item order and walker: item_sched.cuh (L2-sized unit groups, heaviest query blocks first).
using Walker = ItemWalker;

#if defined(ATT_TRACE)  // timeline experiment (scripts/attend_trace.py --split): clock64 stamps of CTA 0
__device__ unsigned long long g_split_trace_sm[256][6];   // softmax warp 4, lane 0, first 256 blocks
__device__ unsigned long long g_split_trace_mma[256][6];  // MMA thread, first 256 blocks
__device__ unsigned long long g_split_trace_arr[256][8][5];  // every softmax warp (lane 0), first 256 blocks:
                                                               // start, S ok, exchanged, P stored, arrived
#define SPLIT_TR_ARR(slot)                                                                              \
    do {                                                                                                \
        if (blockIdx.x == 0 && lane == 0 && b < 256) g_split_trace_arr[b][warp - 4][slot] = clock64();  \
    } while (0)
#define SPLIT_TR_SM(slot)                                                                          \
    do {                                                                                           \
        if (blockIdx.x == 0 && warp == 4 && lane == 0 && b < 256) g_split_trace_sm[b][slot] = clock64(); \
    } while (0)
#define SPLIT_TR_MMA(bb, slot)                                                                     \
    do {                                                                                           \
        if (blockIdx.x == 0 && (bb) < 256) g_split_trace_mma[(bb)][slot] = clock64();              \
    } while (0)
#else
#define SPLIT_TR_SM(slot) \
    do {                  \
    } while (0)
#define SPLIT_TR_MMA(bb, slot) \
    do {                       \
    } while (0)
#define SPLIT_TR_ARR(slot) \
    do {                   \
    } while (0)
#endif

template <bool kBF16>
__global__ void __launch_bounds__(kThreads, 1)
    attend_split_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                        const AttendArgs a, const __grid_constant__ ItemSched sc, const uint32_t idesc_s,
                        const uint32_t idesc_pv) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sQ = smem;               // [2][tile]
    uint8_t *sK = sQ + kNQ * kTile;   // [kNK][tile]
    uint8_t *sV = sK + kNK * kTile;   // [kNV][tile]
    uint8_t *sOut = sV + kNV * kTile; // [4 epilogue warps][kStage][kOutWarp]
    uint64_t *bars = (uint64_t *)(sOut + 4 * kStage * kOutWarp);
    uint64_t *q_full = bars, *q_empty = q_full + 2;
    uint64_t *k_full = q_empty + 2, *k_empty = k_full + kNK;
    uint64_t *v_full = k_empty + kNK, *v_empty = v_full + kNV;
    uint64_t *s_full = v_empty + kNV;  // [2] S_b computed in buffer b % 2
    uint64_t *p_full = s_full + 2;     // [2] P_b written (256 softmax arrivals)
    uint64_t *pv_done = p_full + 2;    // PV_b retired (one phase per block; the lazy rescale waits on it)
    uint64_t *o_full = pv_done + 1;    // an item's last PV retired: O complete (one phase per item)
    uint64_t *o_free = o_full + 1;     // the epilogue has read O (128 arrivals, one phase per item)
    uint64_t *sum_free = o_free + 1;   // [2] the epilogue has read the row sums of an item of parity p
    uint32_t *tmem_slot = (uint32_t *)(sum_free + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 4; ++s) {
            if (s < 2) {
                mbar_init(&q_full[s], 1);
                mbar_init(&q_empty[s], 1);
                mbar_init(&s_full[s], 1);
                mbar_init(&p_full[s], 256);
                mbar_init(&sum_free[s], 128);
            }
            if (s < kNK) {
                mbar_init(&k_full[s], 1);
                mbar_init(&k_empty[s], 1);
            }
            if (s < kNV) {
                mbar_init(&v_full[s], 1);
                mbar_init(&v_empty[s], 1);
            }
        }
        mbar_init(pv_done, 1);
        mbar_init(o_full, 1);
        mbar_init(o_free, 128);
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    RowList list = a.list;
    if (a.sel.n > 0) {  // row selection in the prologue (no select launch): every CTA builds the same list
        uint8_t *sel_base = (uint8_t *)bars + 256;
        list.count = (int32_t *)sel_base;
        list.rows = (int32_t *)(sel_base + 16);
        list.ents = (int64_t *)(sel_base + 16 + 4 * kSelCap);
        list.cap = kSelCap;
        compact_rows(a.sel.n, [&](int64_t b, int64_t &ent) { return select_attend_pred(a.sel, b, ent); }, list);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const uint32_t units = (uint32_t)(*list.count) * sc.per_row;
    const uint32_t items = units * sc.n_qb;

    if (warp < 4) {
        setmaxnreg_dec<kRegProducer>();
        if (warp == 0 && lane == 0) {
            // ------------------------------ TMA loader -------------------------------------------
            Walker w;
            w.init(sc, blockIdx.x, gridDim.x, items, units, list.rows);
            uint32_t b = 0, it = 0;
#if defined(ATT2_POL)  // experiment (scripts/attend_policy_ab.sh): Q read once -> evict_first; 2: K/V evict_last
            const uint64_t pol_q = policy_evict_first();
#if ATT2_POL == 2
            const uint64_t pol_kv = policy_evict_last();
#else
            uint64_t pol_kv;
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_kv));
#endif
#define ATT2_LOAD_Q(dst, map, bar, c0, c1, c2) tma_load_3d_hint(dst, map, bar, c0, c1, c2, pol_q)
#define ATT2_LOAD_KV(dst, map, bar, c0, c1, c2) tma_load_3d_hint(dst, map, bar, c0, c1, c2, pol_kv)
#else
#define ATT2_LOAD_Q(dst, map, bar, c0, c1, c2) tma_load_3d(dst, map, bar, c0, c1, c2)
#define ATT2_LOAD_KV(dst, map, bar, c0, c1, c2) tma_load_3d(dst, map, bar, c0, c1, c2)
#endif
            while (w.active) {
                AC_STRESS_DELAY(716u);
                if (w.j == 0) {
                    const uint32_t qs = it % kNQ;
                    mbar_wait(&q_empty[qs], ((it / kNQ) & 1u) ^ 1u);
                    mbar_arrive_expect_tx(&q_full[qs], kTile);
                    for (int h = 0; h < 2; ++h)
                        ATT2_LOAD_Q(smem_u32(sQ + qs * kTile + h * (kBlk * 128)), &tmQ, &q_full[qs], h * 64,
                                    w.qb * kBlk, w.unit);
                }
                const int32_t r_j = w.j * kBlk;
                const uint32_t kk = b % kNK, kkph = ((b / kNK) & 1u) ^ 1u;
                const uint32_t vv = b % kNV, vvph = ((b / kNV) & 1u) ^ 1u;
                mbar_wait(&k_empty[kk], kkph);
                mbar_arrive_expect_tx(&k_full[kk], kTile);
                for (int h = 0; h < 2; ++h)
                    ATT2_LOAD_KV(smem_u32(sK + kk * kTile + h * (kBlk * 128)), &tmK, &k_full[kk], h * 64, r_j, w.kv_unit);
                mbar_wait(&v_empty[vv], vvph);
                mbar_arrive_expect_tx(&v_full[vv], kTile);
                for (int h = 0; h < 2; ++h)
                    ATT2_LOAD_KV(smem_u32(sV + vv * kTile + h * (kBlk * 128)), &tmV, &v_full[vv], h * 64, r_j, w.kv_unit);
                ++b;
                if (w.advance(sc)) ++it;
            }
        } else if (warp == 1) {
            // ------------------------------ MMA issuer (whole warp; one elected lane issues) --------
            // wS runs two blocks ahead of wP: S_0, S_1, then PV_b followed by S_{b+2}.  The first PV of an
            // item restarts O, so it waits until the epilogue has read the previous item's O (o_free).
            Walker wS, wP;
            wS.init(sc, blockIdx.x, gridDim.x, items, units, list.rows);
            wP.init(sc, blockIdx.x, gridDim.x, items, units, list.rows);
            uint32_t bS = 0, itS = 0, bP = 0, itP = 0;
            auto issue_s = [&]() {
                const uint32_t buf = bS & 1u, qs = itS % kNQ;
                if (wS.j == 0) mbar_wait(&q_full[qs], (itS / kNQ) & 1u);
                mbar_wait(&k_full[bS % kNK], (bS / kNK) & 1u);
                SPLIT_TR_MMA(bS, 5);  // K (and Q) of S_{bS} ready
                tc_fence_after();
                umma_f16_ss_k8_w<kBlk * 128 / 16>(tmem + buf * kBlk,
                                               smem_desc(smem_u32(sQ + qs * kTile), 16, 1024, kSwizzle128B),
                                               smem_desc(smem_u32(sK + (bS % kNK) * kTile), 16, 1024, kSwizzle128B),
                                               idesc_s, 0u);
                umma_commit_w(&s_full[buf]);
                umma_commit_w(&k_empty[bS % kNK]);
                if (wS.j == wS.qb) umma_commit_w(&q_empty[qs]);
                ++bS;
                if (wS.advance(sc)) ++itS;
            };
            if (wS.active) issue_s();
            if (wS.active) issue_s();
            while (wP.active) {
                AC_STRESS_DELAY(146u);
                const uint32_t buf = bP & 1u, ph = (bP >> 1) & 1u;
                SPLIT_TR_MMA(bP, 0);
                mbar_wait(&p_full[buf], ph);
                SPLIT_TR_MMA(bP, 1);
                mbar_wait(&v_full[bP % kNV], (bP / kNV) & 1u);
                // the epilogue of item itP - 1 has read O (it cannot be further along: item itP's epilogue
                // waits for this item's PVs)
                if (wP.j == 0 && itP > 0) mbar_wait(o_free, (itP - 1) & 1u);
                SPLIT_TR_MMA(bP, 2);
                tc_fence_after();
                umma_f16_ts_k8_w(tmem + kOCol, tmem + buf * kBlk,
                               smem_desc(smem_u32(sV + (bP % kNV) * kTile), kBlk * 128, 1024, kSwizzle128B), idesc_pv,
                               wP.j == 0 ? 0u : 1u);
                umma_commit_w(&v_empty[bP % kNV]);
                umma_commit_w(pv_done);
                if (wP.j == wP.qb) umma_commit_w(o_full);
                SPLIT_TR_MMA(bP, 3);
                ++bP;
                if (wP.advance(sc)) ++itP;
                if (wS.active) issue_s();  // into the buffer PV_b reads: queued behind it
                SPLIT_TR_MMA(bP - 1, 4);
            }
        }
    } else if (warp < 12) {
        // ------------------------------ softmax (8 warps) ------------------------------------------
        setmaxnreg_inc<kRegSoftmax>();
        const int half = (warp - 4) >> 2;   // key half (64 keys) and O half (64 columns, rescale) of this warp
        const int q = warp & 3;             // TMEM lane quarter
        const int r = q * 32 + lane;        // query row inside the block == TMEM lane
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        const uint32_t o_addr = tmem + lane_addr + kOCol + half * 64;
        const float sl2 = a.scale * 1.4426950408889634f;
        Walker w;
        w.init(sc, blockIdx.x, gridDim.x, items, units, list.rows);
        uint32_t b = 0, it = 0;
        float m_ref = 0.f, l = 0.f;
        while (w.active) {
            AC_STRESS_DELAY(178u);
            const int j = w.j;
            const bool diag = j == w.qb;
            const uint32_t buf = b & 1u;
            const uint32_t s_addr = tmem + lane_addr + buf * kBlk;
            SPLIT_TR_SM(0);
            SPLIT_TR_ARR(0);
            mbar_wait(&s_full[buf], (b >> 1) & 1u);
            SPLIT_TR_SM(1);
            SPLIT_TR_ARR(1);
            tc_fence_after();
            uint32_t sv[64];  // this warp's 64 keys of its row
            tmem_ld_32x32b_x64(s_addr + half * 64, sv);
            tmem_ld_wait();
            if (diag) {  // keys 64*half + e > r are masked
#pragma unroll
                for (int e = 0; e < 64; ++e)
                    if (half * 64 + e > r) sv[e] = 0xff800000u;  // -inf
            }
            float m8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) m8[i] = fmaxf(__uint_as_float(sv[i]), __uint_as_float(sv[8 + i]));
#pragma unroll
            for (int e = 16; e < 64; e += 16)
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    m8[i] = fmaxf(m8[i], fmaxf(__uint_as_float(sv[e + i]), __uint_as_float(sv[e + 8 + i])));
            float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
            // the row's max over both key halves, exchanged through TMEM (after the barrier both warps have
            // read their S columns, so the P writes below cannot clobber S the partner still needs)
            const uint32_t xcol = tmem + lane_addr + kXmax + 2 * (b & 1u);
            tmem_st_32x32b_x1(xcol + half, __float_as_uint(mx));
            tmem_st_wait();
            tc_fence_before();
            pair_sync(q);
            tc_fence_after();
            mx = fmaxf(mx, __uint_as_float(tmem_ld_32x32b_x1(xcol + (half ^ 1))));
            tmem_ld_wait();
            SPLIT_TR_SM(2);
            SPLIT_TR_ARR(2);
            const float m_blk = mx * sl2;
            if (j == 0) {
                m_ref = m_blk;
                l = 0.f;
            } else if (m_blk > m_ref + kRescaleThreshold) {
                // lazy rescale of this warp's O half (complete once PV_{b-1} retired: s_full(b) implied
                // PV_{b-2}, so the parity wait is unambiguous) and l
                const float alpha = ex2(m_ref - m_blk);
                mbar_wait(pv_done, (b - 1) & 1u);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(o_addr + c * 32, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        uint32_t wv[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) wv[e] = __float_as_uint(__uint_as_float(v[h2 * 16 + e]) * alpha);
                        tmem_st_32x32b_x16(o_addr + c * 32 + h2 * 16, wv);
                    }
                }
                l *= alpha;
                m_ref = m_blk;
            }
            // p = exp2(s * scale * log2e - m_ref), rounded to the MMA dtype, keys 64*half.. -> P columns
            // 32*half..; l sums the unrounded p (an unbiased estimate of the rounded sum)
            {
                const uint64_t scale2 = pack2(sl2, sl2), neg_m2 = pack2(-m_ref, -m_ref);
                uint64_t rs2[4] = {0ull, 0ull, 0ull, 0ull};
                // off-diagonal blocks may compute kSplitPoly of every 8 key pairs with the FMA-pipe
                // polynomial (exp2_poly2; masked -inf keys only occur on diagonal blocks, which stay on MUFU)
                const bool poly_ok = !diag;
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const uint64_t x2 = ffma2(((uint64_t)sv[2 * e + 1] << 32) | sv[2 * e], scale2, neg_m2);
                    float p0, p1;
                    if ((e & 7) < kSplitPoly && poly_ok) {
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
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t wv[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) wv[e] = sv[c * 16 + e];
                    tmem_st_32x32b_x16(s_addr + half * 32 + c * 16, wv);
                }
                const uint64_t t2 = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
                l += __uint_as_float((uint32_t)t2) + __uint_as_float((uint32_t)(t2 >> 32));
            }
            if (diag) {
                // the item's row sum (this warp's keys) for the epilogue, in the sum slot of the item's
                // parity, once the epilogue has read that slot for item it - 2 (parity wait unambiguous:
                // item it's epilogue needs this block's PV)
                if (it >= 2) mbar_wait(&sum_free[it & 1u], ((it >> 1) & 1u) ^ 1u);
                tmem_st_32x32b_x1(tmem + lane_addr + kXsum + 2 * (it & 1u) + half, __float_as_uint(l));
            }
            tmem_st_wait();
            SPLIT_TR_SM(3);
            SPLIT_TR_ARR(3);
            tc_fence_before();
            mbar_arrive(&p_full[buf]);
            SPLIT_TR_SM(4);
            SPLIT_TR_ARR(4);
            ++b;
            if (w.advance(sc)) ++it;
        }
    } else {
        // ------------------------------ epilogue (4 warps, one per TMEM lane quarter) -------------
        // per item: O complete (o_full) -> row sums of both key halves -> O / (l_0 + l_1) in two 64-column
        // halves -> act dtype -> 128B-swizzled staging tile -> TMA store of 32 rows x 64 columns
        setmaxnreg_dec<kRegEpilogue>();
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
        uint8_t *stage = sOut + q * kStage * kOutWarp;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < items; t += gridDim.x, ++it) {
            AC_STRESS_DELAY(99u);
            const ItemSched::Item item = sc.decode(t, units, list.rows);
            const int32_t orow = item.qb * kBlk + q * 32;  // rows >= S are clipped by the tensor map
            mbar_wait(o_full, it & 1u);
            tc_fence_after();
            uint32_t ls[2];
            tmem_ld_32x32b_x2(tmem + lane_addr + kXsum + 2 * (it & 1u), ls);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&sum_free[it & 1u]);
            const float inv = 1.f / (__uint_as_float(ls[0]) + __uint_as_float(ls[1]));
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                uint32_t v[64];
                tmem_ld_32x32b_x32(tmem + lane_addr + kOCol + h * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                tmem_ld_32x32b_x32(tmem + lane_addr + kOCol + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                tmem_ld_wait();
                if (h == 1) {  // all of O is in registers or staged: the next item's first PV may restart it
                    tc_fence_before();
                    mbar_arrive(o_free);
                }
                uint8_t *st = stage + (h % kStage) * kOutWarp;
                if (lane == 0) bulk_wait_read<kStage - 1>();  // the store that last read this staging tile
                __syncwarp();
#pragma unroll
                for (int c8 = 0; c8 < 8; ++c8) {
                    uint32_t wv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float lo = __uint_as_float(v[c8 * 8 + 2 * e]) * inv;
                        const float hi = __uint_as_float(v[c8 * 8 + 2 * e + 1]) * inv;
                        if constexpr (kBF16) {
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(lo, hi);
                            wv[e] = *reinterpret_cast<uint32_t *>(&h2);
                        } else {
                            __half2 h2 = __floats2half2_rn(lo, hi);
                            wv[e] = *reinterpret_cast<uint32_t *>(&h2);
                        }
                    }
                    *reinterpret_cast<uint4 *>(st + sw128_offset(lane, c8)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_3d(&tmO, smem_u32(st), h * 64, orow, item.unit);
                    bulk_commit();
                }
            }
        }
        if (lane == 0) bulk_wait<0>();  // O stores complete before the CTA (and its smem) retires
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

template <bool kBF16>
cudaError_t launch_t(const AttendArgs &a, int sm_count, cudaStream_t st) {
    const bool bf16 = kBF16;
    CUtensorMap tq, tk, tv, to;
    cudaError_t e = make_attend_tmaps(a, kD, &tq, &tk, &tv, &to);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(attend_split_kernel<kBF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t fmt = bf16 ? 1u : 0u;
    const uint32_t idesc_s = idesc_f16(kBlk, kBlk, fmt, 0u, 0u);  // Q K-major x K K-major
    const uint32_t idesc_pv = idesc_f16(kBlk, kD, fmt, 0u, 1u);   // P (TMEM) x V MN-major
    // units whose K and V fill ~48 MB of L2 form a group
    // wave order (item_sched.cuh): the sm_count item streams work on few units at a time, so a unit's K/V
    // blocks, re-read by each of its query blocks, stay in L2 (configs[2] 13 rows 0.566 -> 0.532 ms, all
    // 128 rows 5.53-5.68 -> 5.18-5.41, configs[3] 1.364 -> 1.349 against L2-sized unit groups in
    // heaviest-first order)
#ifndef ATT_WAVE_STREAMS_X4
#define ATT_WAVE_STREAMS_X4 4  // wave size in quarters of the stream count (2 / 8 / 16 measured: configs[2]
                                // 0.703 / 0.533 / 0.544 ms against 0.529, configs[3] within 1 %)
#endif
    const ItemSched sc = ItemSched::make_wave((uint32_t)a.S, (uint32_t)a.L, (uint32_t)a.H, (uint32_t)a.Hkv, kBlk,
                                              (uint32_t)sm_count * ATT_WAVE_STREAMS_X4 / 4);
    attend_split_kernel<kBF16><<<sm_count, kThreads, kSmem, st>>>(tq, tk, tv, to, a, sc, idesc_s, idesc_pv);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

int64_t attend_split_sel_cap() { return kSelCap; }

cudaError_t launch_attend_split(const AttendArgs &a, int sm_count, cudaStream_t st) {
    return a.dt == ATTNCACHE_BF16 ? launch_t<true>(a, sm_count, st) : launch_t<false>(a, sm_count, st);
}

}  // namespace ac
#if defined(ATT_TRACE)
extern "C" int attncache_debug_split_trace(void *sm, void *mma) {
    cudaError_t e = cudaMemcpyFromSymbol(sm, ac::g_split_trace_sm, sizeof(ac::g_split_trace_sm));
    if (e == cudaSuccess) e = cudaMemcpyFromSymbol(mma, ac::g_split_trace_mma, sizeof(ac::g_split_trace_mma));
    return (int)e;
}
extern "C" int attncache_debug_split_trace_arr(void *arr) {
    return (int)cudaMemcpyFromSymbol(arr, ac::g_split_trace_arr, sizeof(ac::g_split_trace_arr));
}
#endif
