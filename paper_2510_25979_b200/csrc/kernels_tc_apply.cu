// kernels_tc_apply.cu — O = A . V on 5th-gen tensor cores (Alg. 2 l.373-375).
//
// One persistent CTA per SM walks the (hit, layer, head) units of the compacted hit list.  A unit
// is split into 128-row blocks; row block rb needs map columns [0, 128(rb+1)) only (the maps are
// causal: exact zeros above the diagonal, reading R11), processed as 64-column chunks.  A
// non-causal (encoder, f3) DB visits every column.
//
// Roles (320 threads):
//   warps 0-3  map loader: cp.async 16-byte pieces of the lower triangle straight from the DB
//              (no "attention cache" copy, reading R18); pieces entirely above the diagonal are
//              zero-filled in shared memory without touching HBM (normal L2 policy).  Writes the 128B-swizzled
//              K-major layout tcgen05 reads.
//   warp 4     V loader: TMA 3-D loads ([units][S][d]) of V rows [64kc, 64kc+64) (128B swizzle, MN-major B).
//
// Any S % 8 == 0 (the paper's contexts are 94-1019 tokens, Table 3): a unit has ceil(S / 128) row blocks and
// ceil(S / 64) column chunks; map pieces of rows >= S or columns >= S are zero-filled in shared memory, V rows
// past S read as zeros (3-D tensor map bounds) and O rows past S are clipped by the TMA store.
//   warp 5     MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=d, K=16, fp32 in TMEM;
//              owns TMEM allocation (2 accumulators: the epilogue of one row block overlaps the
//              MMAs of the next).
//   warps 6-9  epilogue: tcgen05.ld -> fp32 -> act dtype (RN) -> 16-byte global stores of O.
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 320;
constexpr int kRows = 128;     // MMA M
constexpr int kChunk = 64;     // map columns (= V rows) per pipeline stage
constexpr int kABytes = kRows * kChunk * 2;

template <int kD>
struct Cfg {
    static constexpr int kVBytes = kChunk * kD * 2;
    static constexpr int kStageBytes = kABytes + kVBytes;
    static constexpr int kStages = kD == 64 ? 8 : 6;
    static constexpr int kLag = kStages - 2;  // cp.async groups a loader thread keeps in flight
    static constexpr uint32_t kTmemCols = 2 * kD;
    static constexpr int kOutWarpBytes = 32 * kD * 2;  // epilogue staging: one warp's 32 rows of O
    // rows the prologue can select into shared memory (12 B each; 0: the separate select kernel always runs)
    static constexpr int kSelCap = kD == 64 ? 1024 : 0;
    static constexpr int kSmem = kStages * kStageBytes + 4 * kOutWarpBytes + 1024 /*align*/ + 256 /*barriers*/ +
                                 (kSelCap ? 16 + 12 * kSelCap : 0);
};

// Walks this CTA's units u = blockIdx.x, +gridDim.x, ... of the compacted hit list.  The hit-list
// entry (batch row and/or DB entry) of the next unit is loaded one unit ahead so its latency hides
// behind the current unit instead of stalling the pipeline once per unit.
template <bool kRow, bool kEnt>
struct UnitIter {
    uint32_t u, stride, units, per_row;
    const int32_t *rows;
    const int64_t *ents;
    int32_t next_row = 0;
    int64_t next_ent = 0;
    __device__ UnitIter(uint32_t first, uint32_t stride_, uint32_t units_, uint32_t per_row_, const RowList &l)
        : u(first), stride(stride_), units(units_), per_row(per_row_), rows(l.rows), ents(l.ents) {
        fetch();
    }
    __device__ __forceinline__ void fetch() {
        if (u < units) {
            if (kRow) next_row = rows[u / per_row];
            if (kEnt) next_ent = ents[u / per_row];
        }
    }
    // lh = (layer - layer_begin) * H + head of the unit
    __device__ __forceinline__ bool next(uint32_t &lh, int64_t &row, int64_t &ent) {
        if (u >= units) return false;
        lh = u % per_row;
        row = next_row;
        ent = next_ent;
        u += stride;
        fetch();
        return true;
    }
};

template <int kD>
__global__ void __launch_bounds__(kThreads, 1)
    apply_tc_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const ApplyArgs a,
                    const uint32_t idesc) {
    using C = Cfg<kD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sOut = smem + C::kStages * C::kStageBytes;  // [4 warps][kD/64 halves][32 rows][128 B]
    uint64_t *full = (uint64_t *)(sOut + 4 * C::kOutWarpBytes);
    uint64_t *empty = full + C::kStages;
    uint64_t *tfull = empty + C::kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);
    // the prologue's row list (sel.n > 0): count | rows[kSelCap] | ents[kSelCap], after the 256 barrier bytes
    uint8_t *sel_base = (uint8_t *)full + 256;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 128 + 1);  // 128 map-loader threads + the V loader's expect_tx arrival
            mbar_init(&empty[s], 1);       // tcgen05.commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
    }
    if (warp == 5) tmem_alloc<C::kTmemCols>(tmem_slot);
    RowList list = a.list;
    if constexpr (C::kSelCap > 0) {
        if (a.sel.n > 0) {  // row selection in the prologue (no select launch): every CTA builds the same list
            list.count = (int32_t *)sel_base;
            list.rows = (int32_t *)(sel_base + 16);
            list.ents = (int64_t *)(sel_base + 16 + 4 * C::kSelCap);
            list.cap = C::kSelCap;
            compact_rows(a.sel.n, [&](int64_t b, int64_t &ent) { return select_apply_pred(a.sel, b, ent); }, list);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int S = a.S;
    const int n_rb = (S + kRows - 1) / kRows;
    const int n_cc = (S + kChunk - 1) / kChunk;  // column chunks holding at least one stored column
    const uint32_t per_row = (uint32_t)(a.n_lay * a.H);
    const uint32_t units = (uint32_t)(*list.count) * per_row;

    if (warp < 4) {
        // ------------------------------ map loader ------------------------------------------
        // Thread tid owns 16-byte piece c = tid % 8 of tile rows r0 + 16j (j = 0..7), r0 = tid / 8.
        // Rows r0 + 16j share r0 % 8, so their 128B-swizzle XOR is the same and the shared-memory
        // offsets are soff + 2048 j; only the row pointers change per row block.
        const int tid = threadIdx.x;
        const int c = tid & 7, r0 = tid >> 3;
        const uint32_t soff = (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + ((c ^ (r0 & 7)) << 4));
        // Maps are read once, but a 32-byte sector of a PACKED map can straddle two 16-byte pieces read
        // in different pipeline stages (rows start at 16-byte multiples): the normal L2 policy keeps it
        // for the second piece (evict_first measured the same within noise: scripts/apply_experiment.sh).
#if defined(APPLY_EXP) && APPLY_EXP == 1  // experiment: evict_first for the maps (the previous policy)
        const uint64_t policy = policy_evict_first();
#else
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
#endif
        const __nv_bfloat16 *maps = (const __nv_bfloat16 *)a.maps;  // 16-bit payload (bf16 or f16)
        const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
        uint32_t cnt = 0, pending = 0;
        UnitIter<false, true> iter(blockIdx.x, gridDim.x, units, per_row, list);
        uint32_t lh;
        int64_t row, ent;
        while (iter.next(lh, row, ent)) {
            AC_STRESS_DELAY(809u);
            const int l = (int)(lh / a.H), h = (int)(lh % a.H);
            const __nv_bfloat16 *A = maps + ((ent * a.L + a.layer_begin + l) * a.H + h) * a.map_stride + c * 8;
            for (int rb = 0; rb < n_rb; ++rb) {
                const __nv_bfloat16 *rowp[8];
                int lim[8];  // the last stored column of the row (-1: a padded row past S); one compare per piece
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int R = rb * kRows + r0 + 16 * j;
                    lim[j] = R < S ? (a.causal ? R : S - 1) : -1;
                    const int Rc = R < S ? R : S - 1;  // rows >= S are zero-filled below
                    rowp[j] = A + (packed ? packed_row_off(Rc) : (int64_t)Rc * S);
                }
                const int n_kc = a.causal ? min(2 * (rb + 1), n_cc) : n_cc;
                for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                    const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    const uint32_t dst = smem_u32(smem + s * C::kStageBytes) + soff;
                    const int col = kc * kChunk + c * 8;  // first column of this thread's piece
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        // the piece holds at least one stored entry (on/below the diagonal, inside the S x S
                        // map; S % 8 == 0 so a piece is entirely in or out), else zero-fill
                        // (two equivalent forms: the per-row limit hoisted out of the chunk loop measured
                        // 0.773 vs 0.944 ms at configs[1] (d = 64), the form evaluated here 3.70 vs 3.84 ms at
                        // configs[2] (d = 128); scripts/apply_variants.sh)
                        bool need;
                        if constexpr (kD == 128) {
                            const int R = rb * kRows + r0 + 16 * j;
                            need = R < S && col < S && (!a.causal || col <= R);
                        } else {
                            need = col <= lim[j];
                        }
                        cp_async_16_hint(dst + 2048 * j, rowp[j] + (need ? kc * kChunk : 0), need ? 16u : 0u, policy);
                    }
                    cp_async_commit();
                    if (++pending > (uint32_t)C::kLag) {
                        cp_async_wait<C::kLag>();
                        fence_proxy_async_smem();
                        mbar_arrive(&full[(cnt - C::kLag) % C::kStages]);
                        --pending;
                    }
                }
            }
        }
        cp_async_wait<0>();
        fence_proxy_async_smem();
        for (uint32_t i = cnt - pending; i < cnt; ++i) mbar_arrive(&full[i % C::kStages]);
    } else if (warp == 4) {
        // ------------------------------ V loader (TMA) ---------------------------------------
        if (lane == 0) {
            uint32_t cnt = 0;
            UnitIter<true, false> iter(blockIdx.x, gridDim.x, units, per_row, list);
            // V is re-read by every row block of the unit (S > 128): keep it in L2 (evict_last) while
            // the maps stream through with evict_first.
#if defined(APPLY_EXP) && APPLY_EXP == 2  // experiment: V with the normal policy
            uint64_t v_policy;
            asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(v_policy));
#elif defined(APPLY_EXP) && APPLY_EXP == 3  // experiment: evict_first when one row block reads V once (S <= 128)
            const uint64_t v_policy = S <= kRows ? policy_evict_first() : policy_evict_last();
#else
            const uint64_t v_policy = policy_evict_last();
#endif
            uint32_t lh;
            int64_t row, ent;
            while (iter.next(lh, row, ent)) {
                AC_STRESS_DELAY(574u);
                // V head of map head h under grouped-query attention: h / (H / Hkv) (Hkv = H for MHA)
                const uint32_t l = lh / (uint32_t)a.H, h = lh % (uint32_t)a.H;
                const int32_t vunit = (int32_t)((row * a.n_lay + l) * a.Hkv + h / (uint32_t)(a.H / a.Hkv));
                for (int rb = 0; rb < n_rb; ++rb) {
                    const int n_kc = a.causal ? min(2 * (rb + 1), n_cc) : n_cc;
                    for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                        const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                        mbar_wait(&empty[s], ph ^ 1u);
                        mbar_arrive_expect_tx(&full[s], C::kVBytes);
                        const uint32_t dst = smem_u32(smem + s * C::kStageBytes + kABytes);
#pragma unroll
                        for (int half = 0; half < kD / 64; ++half)
                            tma_load_3d_hint(dst + half * (kChunk * 128), &tmV, &full[s], half * 64, kc * kChunk, vunit,
                                             v_policy);
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------ MMA issuer -------------------------------------------
        if (lane == 0) {
            uint32_t cnt = 0, item = 0;
            for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
                AC_STRESS_DELAY(426u);
                for (int rb = 0; rb < n_rb; ++rb, ++item) {
                    const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                    mbar_wait(&tempty[acc], aph ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem + acc * kD;
                    const int n_kc = a.causal ? min(2 * (rb + 1), n_cc) : n_cc;
                    for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                        const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        const uint32_t a_base = smem_u32(smem + s * C::kStageBytes);
                        const uint32_t v_base = a_base + kABytes;
#pragma unroll
                        for (int k = 0; k < kChunk / 16; ++k) {
                            // A: K-major SW128, +32 B per K=16 step inside the 128-byte row.
                            const uint64_t ad = smem_desc(a_base + k * 32, 16, 1024, kSwizzle128B);
                            // B (V): MN-major SW128, 16 K-rows = 2048 B per step; LBO = next 64 columns.
                            const uint64_t bd = smem_desc(v_base + k * 2048, kChunk * 128, 1024, kSwizzle128B);
                            umma_f16(d_tmem, ad, bd, idesc, (kc | k) != 0);
                        }
                        umma_commit(&empty[s]);
                    }
                    umma_commit(&tfull[acc]);
                }
            }
        }
    } else {
        // ------------------------------ epilogue ---------------------------------------------
        // TMEM -> registers -> act dtype -> this warp's 128B-swizzled staging tile -> TMA store of
        // the warp's 32 rows (full-line writes instead of per-thread 16-byte stores).
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        uint32_t item = 0;
        const bool bf16 = a.act_dt == ATTNCACHE_BF16;
        uint8_t *stage_o = sOut + (warp - 6) * C::kOutWarpBytes;
        const uint32_t stage_o_u32 = smem_u32(stage_o);
        UnitIter<true, false> iter(blockIdx.x, gridDim.x, units, per_row, list);
        uint32_t lh;
        int64_t row, ent;
        while (iter.next(lh, row, ent)) {
            AC_STRESS_DELAY(66u);
            const int32_t ounit = (int32_t)(row * per_row + lh);  // the O unit (3-D tensor map coordinate)
            for (int rb = 0; rb < n_rb; ++rb, ++item) {
                const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                mbar_wait(&tfull[acc], aph);
                tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * kD;
                if (lane == 0) bulk_wait_read<0>();  // the previous TMA store has read the staging tile
                __syncwarp();
#pragma unroll
                for (int half = 0; half < kD / 64; ++half) {  // 64 columns at a time (register budget)
                    uint32_t v[64];
                    tmem_ld_32x32b_x32(taddr + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                    tmem_ld_32x32b_x32(taddr + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                    tmem_ld_wait();
                    if (half == kD / 64 - 1) {
                        tc_fence_before();
                        mbar_arrive(&tempty[acc]);  // accumulator drained: the next row block may start
                    }
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        uint32_t w[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float lo = __uint_as_float(v[c8 * 8 + 2 * e]), hi = __uint_as_float(v[c8 * 8 + 2 * e + 1]);
                            if (bf16) {
                                __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
                                w[e] = *reinterpret_cast<uint32_t *>(&p);
                            } else {
                                __half2 p = __floats2half2_rn(lo, hi);
                                w[e] = *reinterpret_cast<uint32_t *>(&p);
                            }
                        }
                        *reinterpret_cast<uint4 *>(stage_o + half * 4096 + sw128_offset(lane, c8)) =
                            make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    const int32_t orow = rb * kRows + q * 32;  // rows >= S are clipped by the tensor map
#pragma unroll
                    for (int half = 0; half < kD / 64; ++half)
                        tma_store_3d(&tmO, stage_o_u32 + half * 4096, half * 64, orow, ounit);
                    bulk_commit();
                }
            }
        }
        if (lane == 0) bulk_wait<0>();
    }
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

// ---- paired row blocks (S > 128) -----------------------------------------------------------------------
// The kernel above re-reads a unit's V chunk for every row block that needs it: at S = 1024 (8 row blocks)
// 72 V chunks (1.15 MB from L2) per unit against 16 stored, next to 1.05 MB of map, and the L2 -> SM traffic
// caps the kernel (0.85 of the HBM peak at configs[3]).  Here adjacent row blocks (2g, 2g + 1) of a unit are
// processed together: a stage holds the A tiles of both row blocks for one 64-column chunk and ONE V chunk,
// the MMA thread accumulates both row blocks (4 TMEM accumulators: two per pair, double-buffered so the
// epilogue of a pair overlaps the MMAs of the next), and each V chunk is read once per pair (40 chunks per
// unit at S = 1024, 6 at S = 256 where it was 8).
template <int kD>
struct PairCfg {
    static constexpr int kVBytes = kChunk * kD * 2;
    static constexpr int kStageBytes = 2 * kABytes + kVBytes;
    static constexpr int kStages = kD == 64 ? 5 : 4;
    static constexpr int kLag = kStages - 2;
    static constexpr uint32_t kTmemCols = 4 * kD;                // [pair parity][row block of the pair]
    static constexpr int kOutWarpBytes = 32 * kD * 2;
    static constexpr int kSelCap = kD == 64 ? 512 : 128;  // prologue row list (12 B per row; the ring leaves ~1.7 KB)
    static constexpr int kSmem = kStages * kStageBytes + 4 * kOutWarpBytes + 1024 + 256 + 16 + 12 * kSelCap;
};

template <int kD>
__global__ void __launch_bounds__(kThreads, 1)
    apply_pair_kernel(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const ApplyArgs a,
                      const uint32_t idesc) {
    using C = PairCfg<kD>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sOut = smem + C::kStages * C::kStageBytes;  // [4 warps][kD/64 halves][32 rows][128 B]
    uint64_t *full = (uint64_t *)(sOut + 4 * C::kOutWarpBytes);
    uint64_t *empty = full + C::kStages;
    uint64_t *tfull = empty + C::kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 128 + 1);  // 128 map-loader threads + the V loader's expect_tx arrival
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        fence_barrier_init();
    }
    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&tmV);
        tma_prefetch_desc(&tmO);
    }
    if (warp == 5) tmem_alloc<C::kTmemCols>(tmem_slot);
    RowList list = a.list;
    if (a.sel.n > 0) {  // row selection in the prologue (no select launch): every CTA builds the same list
        uint8_t *sel_base = (uint8_t *)full + 256;
        list.count = (int32_t *)sel_base;
        list.rows = (int32_t *)(sel_base + 16);
        list.ents = (int64_t *)(sel_base + 16 + 4 * C::kSelCap);
        list.cap = C::kSelCap;
        compact_rows(a.sel.n, [&](int64_t b, int64_t &ent) { return select_apply_pred(a.sel, b, ent); }, list);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int S = a.S;
    const int n_rb = (S + kRows - 1) / kRows;
    const int n_pairs = (n_rb + 1) / 2;
    const int n_cc = (S + kChunk - 1) / kChunk;
    const uint32_t per_row = (uint32_t)(a.n_lay * a.H);
    const uint32_t units = (uint32_t)(*list.count) * per_row;
    // chunks row block rb needs; a pair's chunk loop runs to its second (larger) row block's count
    auto rb_chunks = [&](int rb) { return a.causal ? min(2 * (rb + 1), n_cc) : n_cc; };

    if (warp < 4) {
        // ------------------------------ map loader (both row blocks of a pair) -------------------------
        const int tid = threadIdx.x;
        const int c = tid & 7, r0 = tid >> 3;
        const uint32_t soff = (uint32_t)((r0 >> 3) * 1024 + (r0 & 7) * 128 + ((c ^ (r0 & 7)) << 4));
        uint64_t policy;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
        const __nv_bfloat16 *maps = (const __nv_bfloat16 *)a.maps;
        const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
        uint32_t cnt = 0, pending = 0;
        UnitIter<false, true> iter(blockIdx.x, gridDim.x, units, per_row, list);
        uint32_t lh;
        int64_t row, ent;
        while (iter.next(lh, row, ent)) {
            AC_STRESS_DELAY(809u);
            const int l = (int)(lh / a.H), h = (int)(lh % a.H);
            const __nv_bfloat16 *A = maps + ((ent * a.L + a.layer_begin + l) * a.H + h) * a.map_stride + c * 8;
            for (int pr = 0; pr < n_pairs; ++pr) {
                const int rb0 = 2 * pr, rb1 = 2 * pr + 1;
                const bool has1 = rb1 < n_rb;
                const int nk0 = rb_chunks(rb0), nk = has1 ? rb_chunks(rb1) : nk0;
                const __nv_bfloat16 *rowp[2][8];
                int lim[2][8];
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int R = (rb0 + t) * kRows + r0 + 16 * j;
                        lim[t][j] = R < S ? (a.causal ? R : S - 1) : -1;
                        const int Rc = R < S ? R : S - 1;
                        rowp[t][j] = A + (packed ? packed_row_off(Rc) : (int64_t)Rc * S);
                    }
                for (int kc = 0; kc < nk; ++kc, ++cnt) {
                    const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    const uint32_t dst = smem_u32(smem + s * C::kStageBytes) + soff;
                    const int col = kc * kChunk + c * 8;
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (t == 0 ? kc >= nk0 : !has1) continue;  // this row block's MMA is skipped
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const bool need = col <= lim[t][j];
                            cp_async_16_hint(dst + t * kABytes + 2048 * j, rowp[t][j] + (need ? kc * kChunk : 0),
                                             need ? 16u : 0u, policy);
                        }
                    }
                    cp_async_commit();
                    if (++pending > (uint32_t)C::kLag) {
                        cp_async_wait<C::kLag>();
                        fence_proxy_async_smem();
                        mbar_arrive(&full[(cnt - C::kLag) % C::kStages]);
                        --pending;
                    }
                }
            }
        }
        cp_async_wait<0>();
        fence_proxy_async_smem();
        for (uint32_t i = cnt - pending; i < cnt; ++i) mbar_arrive(&full[i % C::kStages]);
    } else if (warp == 4) {
        // ------------------------------ V loader (TMA): one V chunk per pair and chunk --------------
        if (lane == 0) {
            uint32_t cnt = 0;
            UnitIter<true, false> iter(blockIdx.x, gridDim.x, units, per_row, list);
            const uint64_t v_policy = policy_evict_last();
            // every pair re-reads the V chunks of the pairs before it, so the unit's last pair is the last reader of
            // every chunk: its loads demote the lines (evict_first), or finished units' V would pile up as
            // evict_last in L2 and push out the V of the units in flight (configs[3]: DRAM reads 5.75 -> 5.58 GB,
            // 1.062 -> 1.043 ms; scripts/apply_vlast_ab.sh)
            const uint64_t v_last_policy = policy_evict_first();
            uint32_t lh;
            int64_t row, ent;
            while (iter.next(lh, row, ent)) {
                AC_STRESS_DELAY(574u);
                const uint32_t l = lh / (uint32_t)a.H, h = lh % (uint32_t)a.H;
                const int32_t vunit = (int32_t)((row * a.n_lay + l) * a.Hkv + h / (uint32_t)(a.H / a.Hkv));
                for (int pr = 0; pr < n_pairs; ++pr) {
                    const uint64_t pol = pr == n_pairs - 1 ? v_last_policy : v_policy;
                    const int nk = 2 * pr + 1 < n_rb ? rb_chunks(2 * pr + 1) : rb_chunks(2 * pr);
                    for (int kc = 0; kc < nk; ++kc, ++cnt) {
                        const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                        mbar_wait(&empty[s], ph ^ 1u);
                        mbar_arrive_expect_tx(&full[s], C::kVBytes);
                        const uint32_t dst = smem_u32(smem + s * C::kStageBytes + 2 * kABytes);
#pragma unroll
                        for (int half = 0; half < kD / 64; ++half)
                            tma_load_3d_hint(dst + half * (kChunk * 128), &tmV, &full[s], half * 64, kc * kChunk, vunit,
                                             pol);
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------ MMA issuer -------------------------------------------------
        if (lane == 0) {
            uint32_t cnt = 0, item = 0;
            for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
                AC_STRESS_DELAY(426u);
                for (int pr = 0; pr < n_pairs; ++pr, ++item) {
                    const bool has1 = 2 * pr + 1 < n_rb;
                    const int nk0 = rb_chunks(2 * pr), nk = has1 ? rb_chunks(2 * pr + 1) : nk0;
                    const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                    mbar_wait(&tempty[acc], aph ^ 1u);
                    tc_fence_after();
                    for (int kc = 0; kc < nk; ++kc, ++cnt) {
                        const uint32_t s = cnt % C::kStages, ph = (cnt / C::kStages) & 1u;
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        const uint32_t a_base = smem_u32(smem + s * C::kStageBytes);
                        const uint32_t v_base = a_base + 2 * kABytes;
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            if (t == 0 ? kc >= nk0 : !has1) continue;
                            const uint32_t d_tmem = tmem + (acc * 2 + t) * kD;
#pragma unroll
                            for (int k = 0; k < kChunk / 16; ++k)
                                umma_f16(d_tmem, smem_desc(a_base + t * kABytes + k * 32, 16, 1024, kSwizzle128B),
                                         smem_desc(v_base + k * 2048, kChunk * 128, 1024, kSwizzle128B), idesc,
                                         (kc | k) != 0);
                        }
                        umma_commit(&empty[s]);
                    }
                    umma_commit(&tfull[acc]);
                }
            }
        }
    } else {
        // ------------------------------ epilogue: both row blocks of a pair --------------------------
        const int q = warp & 3;
        uint32_t item = 0;
        const bool bf16 = a.act_dt == ATTNCACHE_BF16;
        uint8_t *stage_o = sOut + (warp - 6) * C::kOutWarpBytes;
        const uint32_t stage_o_u32 = smem_u32(stage_o);
        UnitIter<true, false> iter(blockIdx.x, gridDim.x, units, per_row, list);
        uint32_t lh;
        int64_t row, ent;
        while (iter.next(lh, row, ent)) {
            AC_STRESS_DELAY(66u);
            const int32_t ounit = (int32_t)(row * per_row + lh);
            for (int pr = 0; pr < n_pairs; ++pr, ++item) {
                const int n_t = 2 * pr + 1 < n_rb ? 2 : 1;
                const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                mbar_wait(&tfull[acc], aph);
                tc_fence_after();
                for (int t = 0; t < n_t; ++t) {
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (acc * 2 + t) * kD;
                    if (lane == 0) bulk_wait_read<0>();  // the previous TMA store has read the staging tile
                    __syncwarp();
#pragma unroll
                    for (int half = 0; half < kD / 64; ++half) {
                        uint32_t v[64];
                        tmem_ld_32x32b_x32(taddr + half * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
                        tmem_ld_32x32b_x32(taddr + half * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
                        tmem_ld_wait();
                        if (t == n_t - 1 && half == kD / 64 - 1) {
                            tc_fence_before();
                            mbar_arrive(&tempty[acc]);  // both accumulators drained: the next pair may start
                        }
#pragma unroll
                        for (int c8 = 0; c8 < 8; ++c8) {
                            uint32_t w[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float lo = __uint_as_float(v[c8 * 8 + 2 * e]), hi = __uint_as_float(v[c8 * 8 + 2 * e + 1]);
                                if (bf16) {
                                    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
                                    w[e] = *reinterpret_cast<uint32_t *>(&p);
                                } else {
                                    __half2 p = __floats2half2_rn(lo, hi);
                                    w[e] = *reinterpret_cast<uint32_t *>(&p);
                                }
                            }
                            *reinterpret_cast<uint4 *>(stage_o + half * 4096 + sw128_offset(lane, c8)) =
                                make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int32_t orow = (2 * pr + t) * kRows + q * 32;  // rows >= S are clipped
#pragma unroll
                        for (int half = 0; half < kD / 64; ++half)
                            tma_store_3d(&tmO, stage_o_u32 + half * 4096, half * 64, orow, ounit);
                        bulk_commit();
                    }
                }
            }
        }
        if (lane == 0) bulk_wait<0>();
    }
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

template <int kD>
cudaError_t launch(const ApplyArgs &a, int sm_count, cudaStream_t st) {
    using C = Cfg<kD>;
    const bool bf16 = a.act_dt == ATTNCACHE_BF16;
    const uint64_t units = (uint64_t)a.max_rows * a.n_lay * a.H, vunits = (uint64_t)a.max_rows * a.n_lay * a.Hkv;
    const uint64_t plane = (uint64_t)a.S * kD * 2;
    CUtensorMap tmV, tmO;
    cudaError_t e = make_tmap_3d_16(&tmV, a.V, bf16, kD, a.S, vunits, (uint64_t)kD * 2, plane, 64, kChunk, 128);
    if (e == cudaSuccess) e = make_tmap_3d_16(&tmO, a.O, bf16, kD, a.S, units, (uint64_t)kD * 2, plane, 64, 32, 128);
    if (e != cudaSuccess) return e;
    const uint32_t idesc = idesc_f16(kRows, kD, bf16 ? 1u : 0u, /*a_mn=*/0u, /*b_mn=*/1u);
#if !defined(APPLY_NO_PAIR)
    if (a.S > kRows) {  // two or more row blocks per unit: pairs share their V chunks
        e = cudaFuncSetAttribute(apply_pair_kernel<kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairCfg<kD>::kSmem);
        if (e != cudaSuccess) return e;
        apply_pair_kernel<kD><<<sm_count, kThreads, PairCfg<kD>::kSmem, st>>>(tmV, tmO, a, idesc);
        count_launches(1);
        return cudaGetLastError();
    }
#endif
    e = cudaFuncSetAttribute(apply_tc_kernel<kD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    apply_tc_kernel<kD><<<sm_count, kThreads, C::kSmem, st>>>(tmV, tmO, a, idesc);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

bool apply_tc_supported(int32_t map_dt, int32_t act_dt, int32_t S, int32_t d) {
    return map_dt == act_dt && (map_dt == ATTNCACHE_BF16 || map_dt == ATTNCACHE_F16) && S >= 8 && S % 8 == 0 &&
           (d == 64 || d == 128);
}

bool apply_tc_fused_select(const ApplyArgs &a, int64_t n_rows) {
    // the single-row-block kernel (S <= 128) at d = 64 and the paired kernel (S > 128) select up to their kSelCap
    // rows in the prologue
#if defined(APPLY_NO_PAIR)
    const bool single = true;
#else
    const bool single = a.S <= kRows;
#endif
    if (!apply_tc_supported(a.map_dt, a.act_dt, a.S, a.d) || n_rows <= 0) return false;
    if (single) return a.d == 64 && n_rows <= Cfg<64>::kSelCap;
    return n_rows <= (a.d == 64 ? PairCfg<64>::kSelCap : PairCfg<128>::kSelCap);
}

cudaError_t launch_apply_tc(const ApplyArgs &a, int sm_count, cudaStream_t st) {
    // unit indices are int32 TMA coordinates and units * per_row is a uint32 loop bound
    if ((uint64_t)a.max_rows * a.n_lay * a.H >= (1ull << 31)) return cudaErrorInvalidValue;
    return a.d == 64 ? launch<64>(a, sm_count, st) : launch<128>(a, sm_count, st);
}

}  // namespace ac
