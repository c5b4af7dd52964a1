// kernels_tc_capture.cu — DB building, capture (Fig. 4 step 1):
// the post-softmax causal attention maps of a prefill, P = softmax(Q K^T * scale, keys j > i masked),
// rounded to the map dtype and written straight into a DB entry (DENSE or PACKED layout).
//
// Work item = (unit, 128-query block qb).  Two passes over the key blocks j = 0..qb:
//   pass 0: S = Q K_j^T on tcgen05 (M=128, N=128, K=d, fp32 in TMEM); each epilogue thread keeps
//           its row's running max m and sum l of exp2(s*scale*log2e - m)           (row statistics)
//   pass 1: S again; P = exp2(s*scale*log2e - m - log2 l), masked, rounded, stored.
// Recomputing S (2x the Q K^T flops) keeps the kernel one launch with no score round trip through
// HBM.  The maps are written with 32-byte stores straight from the registers (store_seg): the store path's
// request rate, not HBM, is what the map writes cost (configs[3]: 1.21 ms with the stores compiled out).
// Roles (384 threads): two independent groups (two item streams per CTA), each with a TMA loader thread
// (warp 2g), an MMA thread (warp 2g+1; two 128-column S buffers per group) and a 4-warp epilogue group
// (warps 4-7 / 8-11; TMEM lane quarter = warp % 4, one query row per thread, the S row held in
// registers: one TMEM load per block).  A single epilogue group left the kernel at 0.29 of its HBM
// roofline (bench stages.capture_misses, configs[1]).
#include "kernels.cuh"
#include "item_sched.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

// Experiment switches (scripts/capture_ab.sh): pass-1 key-block order (descending when 1) and the L2
// policy of the K loads (0 evict_first, 1 evict_normal, 2 evict_last).  Measured (packed bf16 maps,
// configs 1 / 2 / 3): descending 0.272 / 0.582 / 2.40 ms vs ascending 0.250 / 0.551 / 2.44 (plain
// stores); K evict_last vs normal neutral at S <= 256, 2.27 -> 2.18 ms at S = 1024 with streamed stores.
#ifndef CAP_DESC
#define CAP_DESC 0
#endif
#ifndef CAP_KPOL
#define CAP_KPOL 2
#endif
constexpr bool kCapDesc = CAP_DESC;

#if defined(CAP_TRACE)  // timeline experiment (scripts/capture_trace.py): clock64 stamps of CTA 0, lane 0 of
                        // warps 4-11, first 512 block-passes of each: top, S ok, S loaded, body done
__device__ unsigned long long g_cap_trace[8][512][4];
#define CAP_TR(slot)                                                                                  \
    do {                                                                                              \
        if (blockIdx.x == 0 && lane == 0 && blk < 512) g_cap_trace[warp - 4][blk][slot] = clock64();  \
    } while (0)
#else
#define CAP_TR(slot) \
    do {             \
    } while (0)
#endif
constexpr int kCapKPol = CAP_KPOL;

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

template <int kD, bool kStreamOut>
__global__ void __launch_bounds__(kThreads, 1)
    capture_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const CaptureArgs a, const __grid_constant__ ItemSched sc, const uint32_t idesc) {
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
    const uint32_t per_row = sc.per_row;
    const uint32_t units = (uint32_t)(*a.list.count) * per_row;
    const uint32_t items = units * sc.n_qb;
    const uint32_t stride = 2 * gridDim.x;  // two item streams per CTA (one per group)
    // item t -> (selected row, (layer, head), qb): item_sched.cuh (units in L2-sized groups -- K of a group
    // fits in ~48 MB; both passes re-read it -- heaviest query blocks first inside a group)

    if (warp < 4) {
        // Producers: per group g, warp 2g loads Q (per item) and K_j (per block and pass), warp 2g+1
        // issues S_j = Q K_j^T into one of the group's two S buffers.  The two groups are independent
        // pipelines sharing the tensor pipe (as in kernels_tc_attend.cu).
        setmaxnreg_dec<56>();
        const int g = warp >> 1;
        if (lane == 0) {
            // Q is read once, K twice (both passes) within an item: Q evict_first, K per CAP_KPOL
            const uint64_t pol_q = policy_evict_first();
            const uint64_t pol_k = kCapKPol == 2 ? policy_evict_last() : kCapKPol == 1 ? policy_evict_normal() : policy_evict_first();
            uint32_t it = 0, blk = 0;
            for (uint32_t t = blockIdx.x + g * gridDim.x; t < items; t += stride, ++it) {
                AC_STRESS_DELAY(390u);
                const ItemSched::Item item = sc.decode(t, units, a.list.rows);
                const int qb = item.qb;
                const uint32_t qph = it & 1u;
                if ((warp & 1) == 0) {
                    mbar_wait(&q_empty[g], qph ^ 1u);
                    mbar_arrive_expect_tx(&q_full[g], C::kTile);
                    for (int h = 0; h < kD / 64; ++h)
                        tma_load_3d_hint(smem_u32(sQ + g * C::kTile + h * (kBlk * 128)), &tmQ, &q_full[g], h * 64,
                                         qb * kBlk, item.unit, pol_q);
                } else {
                    mbar_wait(&q_full[g], qph);
                }
                // pass 0 visits key blocks 0..qb (row max and sum), pass 1 blocks qb-1..0 (the diagonal
                // block's P is written in pass 0 from registers; descending, so the 32-byte sectors a row
                // shares between neighbouring blocks are completed back to back while still in L2 -- the
                // ascending order measured 10 % slower at configs[3]'s S = 1024)
                for (int i = 0; i <= 2 * qb; ++i, ++blk) {
                    const int j = i <= qb ? i : kCapDesc ? 2 * qb - i : i - qb - 1;
                    const uint32_t ks = g * NK + blk % NK, kph = (blk / NK) & 1u;
                    if ((warp & 1) == 0) {
                        mbar_wait(&k_empty[ks], kph ^ 1u);
                        mbar_arrive_expect_tx(&k_full[ks], C::kTile);
                        for (int h = 0; h < kD / 64; ++h)
                            tma_load_3d_hint(smem_u32(sK + ks * C::kTile + h * (kBlk * 128)), &tmK, &k_full[ks], h * 64,
                                             j * kBlk, item.kv_unit, pol_k);
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
                        if (i == 2 * qb) umma_commit(&q_empty[g]);
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
        const uint64_t pol_out = policy_evict_first();  // maps: written once (used when kStreamOut)
        uint16_t *maps = (uint16_t *)a.maps;
        const bool bf16 = a.map_dt == ATTNCACHE_BF16;
        const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
        uint32_t blk = 0;
        auto pack = [&](float p0, float p1) -> uint32_t {
            if (bf16) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
                return *reinterpret_cast<uint32_t *>(&h2);
            }
            __half2 h2 = __floats2half2_rn(p0, p1);
            return *reinterpret_cast<uint32_t *>(&h2);
        };
        // Stores the first n (a multiple of 8) of the 128 packed P values w[0..63] (two per word) of one row's block
        // segment `seg` (16-byte aligned) with 32-byte stores: each store request then carries a whole sector (the
        // 16-byte form made the L1 -> L2 request rate the bound of the store-heavy blocks).  A segment that is not
        // 32-byte aligned starts with one 16-byte store.  All indices into w are compile-time.
        auto st16 = [&](uint16_t *p, const uint32_t *w4) {
            const uint4 v = make_uint4(w4[0], w4[1], w4[2], w4[3]);
            if constexpr (kStreamOut) st_global_16_hint(p, v, pol_out);
            else *reinterpret_cast<uint4 *>(p) = v;
        };
        auto st32 = [&](uint16_t *p, const uint32_t *w8) {
            if constexpr (kStreamOut) st_global_v8_hint(p, w8, pol_out);
            else st_global_v8(p, *reinterpret_cast<const uint32_t(*)[8]>(w8));
        };
        auto store_seg = [&](uint16_t *seg, const uint32_t (&w)[kBlk], int n) {
#if defined(CAP_EXP) && CAP_EXP == 1  // experiment: no map stores (the values stay live through this test)
            if (w[0] == 0x12345678u && w[kBlk / 2 - 1] == 0x9abcdef0u) st16(seg, &w[0]);
            return;
#endif
            if ((reinterpret_cast<uintptr_t>(seg) & 31u) == 0) {
#pragma unroll
                for (int k = 0; k < kBlk / 16; ++k) {
                    if (16 * k + 16 <= n) st32(seg + 16 * k, &w[8 * k]);
                    else if (16 * k + 8 <= n) st16(seg + 16 * k, &w[8 * k]);
                }
            } else {
                if (n >= 8) st16(seg, &w[0]);
#pragma unroll
                for (int k = 0; k < kBlk / 16 - 1; ++k) {
                    const int e0 = 8 + 16 * k;
                    if (e0 + 16 <= n) st32(seg + e0, &w[4 + 8 * k]);
                    else if (e0 + 8 <= n) st16(seg + e0, &w[4 + 8 * k]);
                }
                if (n >= kBlk) st16(seg + kBlk - 8, &w[kBlk / 2 - 4]);
            }
        };
        for (uint32_t t = blockIdx.x + g * gridDim.x; t < items; t += stride) {
            AC_STRESS_DELAY(312u);
            const ItemSched::Item item = sc.decode(t, units, a.list.rows);
            const int qb = item.qb;
            const int R = qb * kBlk + r;  // this thread's query row in the unit
            const bool valid = R < (int)S;  // rows of a last, partial block past S are computed, never stored
            uint16_t *mrow = maps + ((item.row * per_row + item.lh) * a.map_stride) +
                             map_row_off(valid ? R : 0, S, a.map_layout);
            // packed rows hold 8*(R/8 + 1) elements; dense rows S (zeros above the diagonal)
            const int stored = !valid ? 0 : packed ? 8 * (R / 8 + 1) : (int)S;
            float m = -INFINITY, l = 0.f, off = 0.f;
            // pass 0: key blocks 0..qb (row max and sum; the diagonal block, visited last, keeps its
            // exponentials in registers and writes its P at once); pass 1: blocks qb-1..0 write P
            for (int i = 0; i <= 2 * qb; ++i, ++blk) {
                const bool pass0 = i <= qb;
                const int j = pass0 ? i : kCapDesc ? 2 * qb - i : i - qb - 1;
                const uint32_t buf = blk & 1u, bph = (blk >> 1) & 1u;
                const bool diag = j == qb;
                const int lim = diag ? r : kBlk - 1;
                CAP_TR(0);
                mbar_wait(&s_full[g * 2 + buf], bph);
                CAP_TR(1);
                tc_fence_after();
                const uint32_t s_addr = tmem + lane_addr + g * 256 + buf * kBlk;
                // the whole S row of the block in registers (one TMEM round trip); masked keys -inf
                uint32_t sv[kBlk];
                tmem_ld_32x32b_x64(s_addr, sv);
                tmem_ld_32x32b_x64(s_addr + 64, sv + 64);
                tmem_ld_wait();
                CAP_TR(2);
                tc_fence_before();
                mbar_arrive(&s_free[g * 2 + buf]);  // S is in registers: the buffer may be refilled
                if (diag) {
#pragma unroll
                    for (int e = 0; e < kBlk; ++e)
                        if (e > lim) sv[e] = 0xff800000u;
                }
                if (pass0) {
                    float m8[8];
#pragma unroll
                    for (int i8 = 0; i8 < 8; ++i8) m8[i8] = fmaxf(__uint_as_float(sv[i8]), __uint_as_float(sv[8 + i8]));
#pragma unroll
                    for (int e = 16; e < kBlk; e += 16)
#pragma unroll
                        for (int i8 = 0; i8 < 8; ++i8)
                            m8[i8] = fmaxf(m8[i8], fmaxf(__uint_as_float(sv[e + i8]), __uint_as_float(sv[e + 8 + i8])));
                    const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))) * sl2;
                    const float m_new = fmaxf(m, mx);
                    // row sum on MUFU.EX2 (an FMA-pipe polynomial for 2-8 of every 8 pairs was measured
                    // slower: scripts/capture_poly.sh at configs 1/2)
                    float s4[4] = {0.f, 0.f, 0.f, 0.f};
                    if (!diag) {
#pragma unroll
                        for (int e = 0; e < kBlk; ++e) s4[e & 3] += ex2(fmaf(__uint_as_float(sv[e]), sl2, -m_new));
                        l = l * ex2(m - m_new) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
                        m = m_new;
                    } else {
                        // p = exp2(s * sl2 - m_new) once, row sum, then P = p / l for this block
#pragma unroll
                        for (int e = 0; e < kBlk; ++e) {
                            const float pe = ex2(fmaf(__uint_as_float(sv[e]), sl2, -m_new));
                            sv[e] = __float_as_uint(pe);
                            s4[e & 3] += pe;
                        }
                        l = l * ex2(m - m_new) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
                        m = m_new;
                        off = m + lg2(l);  // pass 1: P = exp2(s * sl2 - off)
                        const float inv = 1.f / l;
#pragma unroll
                        for (int e = 0; e < kBlk / 2; ++e)
                            sv[e] = pack(__uint_as_float(sv[2 * e]) * inv, __uint_as_float(sv[2 * e + 1]) * inv);
                        store_seg(mrow + qb * kBlk, sv, min(kBlk, stored - qb * kBlk));  // stored = 0: no stores
                    }
                } else {
                    // pass-1 blocks are whole (j < qb: all 128 columns lie inside row R's stored length)
#pragma unroll
                    for (int e = 0; e < kBlk / 2; ++e)
                        sv[e] = pack(ex2(fmaf(__uint_as_float(sv[2 * e]), sl2, -off)),
                                     ex2(fmaf(__uint_as_float(sv[2 * e + 1]), sl2, -off)));
                    if (valid) store_seg(mrow + j * kBlk, sv, kBlk);
                }
                CAP_TR(3);
            }
            // dense maps: the columns right of this block's diagonal are exact zeros (reading R11)
            if (!packed && valid) {
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
    const uint64_t plane = (uint64_t)a.S * kD * 2;
    CUtensorMap tq, tk;
    cudaError_t e = make_tmap_3d_16(&tq, a.Q, bf16, kD, a.S, (uint64_t)a.max_rows * a.L * a.H, (uint64_t)kD * 2, plane,
                                    64, kBlk, 128);
    if (e == cudaSuccess)
        e = make_tmap_3d_16(&tk, a.K, bf16, kD, a.S, (uint64_t)a.max_rows * a.L * a.Hkv, (uint64_t)kD * 2, plane, 64,
                            kBlk, 128);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(capture_tc_kernel<kD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(capture_tc_kernel<kD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    const uint32_t idesc = idesc_f16(kBlk, kBlk, bf16 ? 1u : 0u, 0u, 0u);
    // units whose K fills ~48 MB of L2 form a group (both passes re-read it)
    // wave order (item_sched.cuh): the 2 x sm_count item streams work on few units at a time, so the K
    // blocks both passes re-read stay in L2 (configs 2 / 3: 0.556 -> 0.547, 2.194 -> 2.156 ms against
    // L2-sized unit groups in heaviest-first order)
#if defined(CAP_GROUPS)  // experiment: L2-sized unit groups, heaviest first
    const ItemSched sc = ItemSched::make((uint32_t)a.S, (uint32_t)a.L, (uint32_t)a.H, (uint32_t)a.Hkv, kBlk,
                                         (uint32_t)a.S * kD * 2u);
#else
    const ItemSched sc = ItemSched::make_wave((uint32_t)a.S, (uint32_t)a.L, (uint32_t)a.H, (uint32_t)a.Hkv, kBlk,
                                              2u * (uint32_t)sm_count);
#endif
    // map stores with an L2 evict_first policy from S = CAP_STREAM_MIN_S on.  With 16-byte stores the hint paid
    // at S = 1024 (configs[3]: 2.44 -> 2.19 ms: the streamed maps no longer pushed a unit's K out of L2); with the
    // 32-byte stores the plain store is as fast or faster at every config (configs 1 / 2 / 3: 0.277 / 0.523 /
    // 1.922 ms plain against 0.292 / 0.539 / 1.941 hinted), so the hint is off by default.
#ifndef CAP_STREAM_MIN_S
#define CAP_STREAM_MIN_S (1 << 30)
#endif
    if (a.S >= CAP_STREAM_MIN_S)
        capture_tc_kernel<kD, true><<<sm_count, kThreads, C::kSmem, st>>>(tq, tk, a, sc, idesc);
    else
        capture_tc_kernel<kD, false><<<sm_count, kThreads, C::kSmem, st>>>(tq, tk, a, sc, idesc);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

bool capture_tc_supported(int32_t dt, int32_t S, int32_t d) {
    return (dt == ATTNCACHE_BF16 || dt == ATTNCACHE_F16) && S >= 8 && S % 8 == 0 && (d == 64 || d == 128);
}

cudaError_t launch_capture_tc(const CaptureArgs &a, int sm_count, cudaStream_t st) {
    // unit indices are int32 TMA coordinates; items = units * ceil(S / 128) is a uint32 loop bound
    const uint64_t units = (uint64_t)a.max_rows * a.L * a.H;
    if (units >= (1ull << 31) || units * ((a.S + kBlk - 1) / kBlk) >= (1ull << 31)) return cudaErrorInvalidValue;
    return a.d == 64 ? launch<64>(a, sm_count, st) : launch<128>(a, sm_count, st);
}

}  // namespace ac
#if defined(CAP_TRACE)
extern "C" int attncache_debug_cap_trace(void *out) {
    return (int)cudaMemcpyFromSymbol(out, ac::g_cap_trace, sizeof(ac::g_cap_trace));
}
#endif
