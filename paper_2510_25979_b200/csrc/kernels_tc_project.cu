// kernels_tc_project.cu — the feature projector of Alg. 1 l.254:
//
//   z = relu(W1 h + b1)   (layer 1: tcgen05 GEMM, bias + ReLU fused in the epilogue, z rounded to bf16/fp16)
//   y = W2 z + b2         (layer 2: the same GEMM, bias fused, y kept in fp32)
//   f = y / ||y||_2       (row normalisation, rounded once to the DB's feature dtype; readings R30-R32)
//
// The GEMM reuses the search kernel's structure (kernels_tc_search.cu): persistent CTAs over (128-row,
// 64/128/256-column) output tiles, ordered row-tile-fastest so concurrently running CTAs share weight
// tiles through L2; warp 0 TMA-loads 64-element K chunks of the activations and the weights (128B
// swizzle, K-major), warp 1 issues tcgen05.mma (M=128, N=tile, K=16) into a double-buffered TMEM
// accumulator, warps 2-5 drain TMEM (one output row per thread), add the bias, apply the activation and
// store.  fp32 inputs (or shapes the tensor-core path does not take) run a shared-memory tiled FFMA GEMM.
#include "kernels.cuh"
#include "sm100.cuh"

namespace ac {
using namespace sm100;

namespace {

constexpr int kThreads = 192;
constexpr int kTileM = 128;
constexpr int kChunk = 64;  // K elements per stage (one 128-byte swizzle row)
constexpr int kABytes = kTileM * kChunk * 2;

template <int kTileN>
struct Cfg {
    static constexpr int kWBytes = kTileN * kChunk * 2;
    static constexpr int kStageBytes = kABytes + kWBytes;
    static constexpr int kStages = kTileN == 256 ? 4 : kTileN == 128 ? 6 : 8;
    static constexpr uint32_t kTmemCols = 2 * kTileN;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

// Output modes of the GEMM epilogue.
//   kOutF32  : Y [M][Nout] fp32, + bias (projector layer 2)
//   kOutRelu : Y [M][Nout] in the input 16-bit type, relu(. + bias) (projector layer 1)
//   kOutHeads: head-major Y [M / S][Nout / d][S][d] in the input type (+ bias when non-NULL): row m = (b, s),
//              column n = (h, c) -> Y[b][h][s][c], the layout the attention and A.V kernels read (the Eq. 5
//              block's Q/K/V projections, f4), so no permute pass follows the GEMM
enum { kOutF32 = 0, kOutRelu = 1, kOutHeads = 2 };
struct OutShape {
    int32_t S, d;  // kOutHeads: sequence length and head dim (d % 32 == 0)
};

// Y[m][n] = epilogue(sum_k A[m][k] W[n][k]) per kMode.
template <int kTileN, int kMode, bool kBf16>
__global__ void __launch_bounds__(kThreads, 1)
    linear_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW, int64_t M,
                     int Nout, int K, const float *__restrict__ bias, void *Y, uint32_t idesc, uint32_t a_rows,
                     OutShape osh) {
    constexpr bool kF32Out = kMode == kOutF32;
    using C = Cfg<kTileN>;
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
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int64_t n_mt = (M + kTileM - 1) / kTileM;
    const int64_t n_nt = (Nout + kTileN - 1) / kTileN;
    const int64_t items = n_mt * n_nt;
    const int n_kc = K / kChunk;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t cnt = 0;
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x) {
                AC_STRESS_DELAY(719u);
                const int32_t mt = (int32_t)(t % n_mt), nt = (int32_t)(t / n_mt);
                for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                    const uint32_t s = cnt % kStages, ph = (cnt / kStages) & 1u;
                    mbar_wait(&empty[s], ph ^ 1u);
                    // small batches load only a_rows rows; the MMA's other rows read stale shared memory,
                    // which only reaches TMEM lanes the epilogue never stores (m >= M)
                    mbar_arrive_expect_tx(&full[s], (a_rows + kTileN) * (kChunk * 2));
                    const uint32_t base = smem_u32(smem + s * kStageBytes);
                    tma_load_2d(base, &tmA, &full[s], kc * kChunk, mt * kTileM);
                    tma_load_2d(base + kABytes, &tmW, &full[s], kc * kChunk, nt * kTileN);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            uint32_t cnt = 0, item = 0;
            for (int64_t t = blockIdx.x; t < items; t += gridDim.x, ++item) {
                AC_STRESS_DELAY(446u);
                const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
                mbar_wait(&tempty[acc], aph ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem + acc * kTileN;
                for (int kc = 0; kc < n_kc; ++kc, ++cnt) {
                    const uint32_t s = cnt % kStages, ph = (cnt / kStages) & 1u;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t aa = smem_u32(smem + s * kStageBytes), wa = aa + kABytes;
#pragma unroll
                    for (int k = 0; k < kChunk / 16; ++k)
                        umma_f16(d_tmem, smem_desc(aa + k * 32, 16, 1024, kSwizzle128B),
                                 smem_desc(wa + k * 32, 16, 1024, kSwizzle128B), idesc, (kc | k) != 0);
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
            AC_STRESS_DELAY(165u);
            const int64_t mt = t % n_mt, nt = t / n_mt;
            const uint32_t acc = item & 1u, aph = (item >> 1) & 1u;
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            const int64_t m = mt * kTileM + r;
#pragma unroll 1
            for (int c = 0; c < kTileN / 32; ++c) {
                const int col0 = (int)nt * kTileN + c * 32;
                if (col0 >= Nout) break;  // Nout % 64 == 0: a 32-column chunk is all in or all out
                uint32_t v[32];
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + acc * kTileN + c * 32, v);
                tmem_ld_wait();
                if (m < M) {
                    float o[32];
                    if (bias) {
                        const float4 *b4 = reinterpret_cast<const float4 *>(bias + col0);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const float4 bb = __ldg(b4 + i);
                            o[4 * i + 0] = __uint_as_float(v[4 * i + 0]) + bb.x;
                            o[4 * i + 1] = __uint_as_float(v[4 * i + 1]) + bb.y;
                            o[4 * i + 2] = __uint_as_float(v[4 * i + 2]) + bb.z;
                            o[4 * i + 3] = __uint_as_float(v[4 * i + 3]) + bb.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(v[i]);
                    }
                    if constexpr (kF32Out) {
                        float4 *dst = reinterpret_cast<float4 *>((float *)Y + m * (int64_t)Nout + col0);
#pragma unroll
                        for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
                    } else {
                        uint32_t w[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float x0 = kMode == kOutRelu ? fmaxf(o[2 * i], 0.f) : o[2 * i];
                            const float x1 = kMode == kOutRelu ? fmaxf(o[2 * i + 1], 0.f) : o[2 * i + 1];
                            if constexpr (kBf16) {
                                __nv_bfloat162 p = __floats2bfloat162_rn(x0, x1);
                                w[i] = *reinterpret_cast<uint32_t *>(&p);
                            } else {
                                __half2 p = __floats2half2_rn(x0, x1);
                                w[i] = *reinterpret_cast<uint32_t *>(&p);
                            }
                        }
                        int64_t off = m * (int64_t)Nout + col0;
                        if constexpr (kMode == kOutHeads) {  // [b][h][s][c]: 64 contiguous bytes of one head row
                            const int64_t b = m / osh.S, sq = m - b * osh.S;
                            const int h = col0 / osh.d, c0 = col0 - h * osh.d;
                            off = ((b * (Nout / osh.d) + h) * osh.S + sq) * osh.d + c0;
                        }
                        uint4 *dst = reinterpret_cast<uint4 *>((uint16_t *)Y + off);
#pragma unroll
                        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

// ---- FFMA fallback: shared-memory tiled GEMM, 32 x 32 outputs per 256-thread block ---------------------
constexpr int kST = 32, kSK = 16;

template <int DT, int kMode>
__global__ void __launch_bounds__(256) linear_simt_kernel(const void *A_, const void *W_, int64_t M, int Nout, int K,
                                                         const float *__restrict__ bias, void *Y, OutShape osh) {
    using E = Elem<DT>;
    using T = typename E::T;
    const T *A = (const T *)A_, *W = (const T *)W_;
    __shared__ float sa[kST][kSK + 1], sw[kST][kSK + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2 x 2 outputs each
    const int64_t m0 = (int64_t)blockIdx.y * kST;
    const int n0 = blockIdx.x * kST;
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    for (int k0 = 0; k0 < K; k0 += kSK) {
        for (int i = threadIdx.x; i < kST * kSK; i += 256) {
            const int rr = i / kSK, kk = i % kSK;
            const int64_t m = m0 + rr;
            const int n = n0 + rr, k = k0 + kk;
            sa[rr][kk] = (m < M && k < K) ? E::ld(A, m * K + k) : 0.f;
            sw[rr][kk] = (n < Nout && k < K) ? E::ld(W, (int64_t)n * K + k) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kSK; ++kk)
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[i][j] = fmaf(sa[ty + 16 * i][kk], sw[tx + 16 * j][kk], acc[i][j]);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int64_t m = m0 + ty + 16 * i;
            const int n = n0 + tx + 16 * j;
            if (m >= M || n >= Nout) continue;
            const float v = acc[i][j] + (bias ? bias[n] : 0.f);
            if constexpr (kMode == kOutF32) {
                ((float *)Y)[m * Nout + n] = v;
            } else if constexpr (kMode == kOutRelu) {
                E::st((T *)Y, m * Nout + n, fmaxf(v, 0.f));
            } else {
                const int64_t b = m / osh.S, sq = m - b * osh.S;
                const int h = n / osh.d, c = n - h * osh.d;
                E::st((T *)Y, ((b * (Nout / osh.d) + h) * osh.S + sq) * osh.d + c, v);
            }
        }
}

// f = y / ||y||_2 per row (one warp per row, fixed summation order: deterministic); y = 0 gives f = 0.
template <int DT>
__global__ void normalize_rows_kernel(const float *__restrict__ Yf, int64_t M, int D, void *F_) {
    using E = Elem<DT>;
    using T = typename E::T;
    T *F = (T *)F_;
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= M) return;
    const float *y = Yf + row * D;
    float ss = 0.f;
    for (int c = lane; c < D; c += 32) ss = fmaf(y[c], y[c], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = ss > 0.f ? 1.0f / sqrtf(ss) : 0.f;
    for (int c = lane; c < D; c += 32) E::st(F, row * D + c, y[c] * inv);
}

template <int kTileN, int kMode>
cudaError_t launch_linear_tc_t(const void *A, const void *W, int64_t M, int Nout, int K, const float *bias, void *Y,
                               bool bf16, int sm_count, cudaStream_t st, OutShape osh) {
    using C = Cfg<kTileN>;
    CUtensorMap ta, tw;
    const uint32_t a_rows = M >= kTileM ? kTileM : (uint32_t)((M + 7) / 8 * 8);
    cudaError_t e = make_tmap_2d_16(&ta, A, bf16, K, M, (uint64_t)K * 2, kChunk, a_rows, 128);
    if (e == cudaSuccess) e = make_tmap_2d_16(&tw, W, bf16, K, Nout, (uint64_t)K * 2, kChunk, kTileN, 128);
    if (e != cudaSuccess) return e;
    const int64_t items = ((M + kTileM - 1) / kTileM) * ((Nout + kTileN - 1) / kTileN);
    const int grid = (int)min64(items, sm_count);
    const uint32_t idesc = idesc_f16(kTileM, kTileN, bf16 ? 1u : 0u, 0u, 0u);
    if (bf16) {
        auto k = linear_tc_kernel<kTileN, kMode, true>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        k<<<grid, kThreads, C::kSmem, st>>>(ta, tw, M, Nout, K, bias, Y, idesc, a_rows, osh);
    } else {
        auto k = linear_tc_kernel<kTileN, kMode, false>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        k<<<grid, kThreads, C::kSmem, st>>>(ta, tw, M, Nout, K, bias, Y, idesc, a_rows, osh);
    }
    count_launches(1);
    return cudaGetLastError();
}

template <int kMode>
cudaError_t launch_linear_tc(const void *A, const void *W, int64_t M, int Nout, int K, const float *bias, void *Y,
                             bool bf16, int sm_count, cudaStream_t st, OutShape osh = {1, 32}) {
    // the widest column tile that still gives every SM at least one work item
    const int64_t n_mt = (M + kTileM - 1) / kTileM;
    if (n_mt * ((Nout + 255) / 256) >= sm_count)
        return launch_linear_tc_t<256, kMode>(A, W, M, Nout, K, bias, Y, bf16, sm_count, st, osh);
    if (n_mt * ((Nout + 127) / 128) >= sm_count)
        return launch_linear_tc_t<128, kMode>(A, W, M, Nout, K, bias, Y, bf16, sm_count, st, osh);
    return launch_linear_tc_t<64, kMode>(A, W, M, Nout, K, bias, Y, bf16, sm_count, st, osh);
}

template <int kMode>
cudaError_t launch_linear_simt(int32_t dt, const void *A, const void *W, int64_t M, int Nout, int K, const float *bias,
                               void *Y, cudaStream_t st, OutShape osh = {1, 32}) {
    dim3 grid((Nout + kST - 1) / kST, (unsigned)((M + kST - 1) / kST));
    switch (dt) {
    case ATTNCACHE_F32: linear_simt_kernel<ATTNCACHE_F32, kMode><<<grid, 256, 0, st>>>(A, W, M, Nout, K, bias, Y, osh); break;
    case ATTNCACHE_F16: linear_simt_kernel<ATTNCACHE_F16, kMode><<<grid, 256, 0, st>>>(A, W, M, Nout, K, bias, Y, osh); break;
    default: linear_simt_kernel<ATTNCACHE_BF16, kMode><<<grid, 256, 0, st>>>(A, W, M, Nout, K, bias, Y, osh); break;
    }
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace

bool linear_tc_supported(int32_t dt, int32_t K, int32_t Nout) {
    return (dt == ATTNCACHE_BF16 || dt == ATTNCACHE_F16) && K >= kChunk && K % kChunk == 0 && Nout >= 64 &&
           Nout % 64 == 0;
}

cudaError_t launch_project(const ProjectArgs &a, int sm_count, cudaStream_t st) {
    if (a.M == 0) return cudaSuccess;
    cudaError_t e;
    // layer 1: z = relu(W1 h + b1) in the activation dtype
    if (linear_tc_supported(a.dt, a.E, a.Hd))
        e = launch_linear_tc<kOutRelu>(a.h, a.W1, a.M, a.Hd, a.E, a.b1, a.z, a.dt == ATTNCACHE_BF16, sm_count, st);
    else
        e = launch_linear_simt<kOutRelu>(a.dt, a.h, a.W1, a.M, a.Hd, a.E, a.b1, a.z, st);
    if (e != cudaSuccess) return e;
    // layer 2: y = W2 z + b2 in fp32
    if (linear_tc_supported(a.dt, a.Hd, a.D))
        e = launch_linear_tc<kOutF32>(a.z, a.W2, a.M, a.D, a.Hd, a.b2, a.y, a.dt == ATTNCACHE_BF16, sm_count, st);
    else
        e = launch_linear_simt<kOutF32>(a.dt, a.z, a.W2, a.M, a.D, a.Hd, a.b2, a.y, st);
    if (e != cudaSuccess) return e;
    // f = y / ||y|| in the feature dtype
    const int rows_per_block = 8;
    const unsigned grid = (unsigned)((a.M + rows_per_block - 1) / rows_per_block);
    switch (a.feat_dt) {
    case ATTNCACHE_F32: normalize_rows_kernel<ATTNCACHE_F32><<<grid, 32 * rows_per_block, 0, st>>>(a.y, a.M, a.D, a.f); break;
    case ATTNCACHE_F16: normalize_rows_kernel<ATTNCACHE_F16><<<grid, 32 * rows_per_block, 0, st>>>(a.y, a.M, a.D, a.f); break;
    default: normalize_rows_kernel<ATTNCACHE_BF16><<<grid, 32 * rows_per_block, 0, st>>>(a.y, a.M, a.D, a.f); break;
    }
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_linear_heads(int32_t dt, const void *X, int64_t M, int32_t K, const void *W, int32_t N,
                                const float *bias, int32_t S, int32_t d, void *Y, int sm_count, cudaStream_t st) {
    if (M == 0) return cudaSuccess;
    const OutShape osh{S, d};
    if (linear_tc_supported(dt, K, N) && d % 32 == 0)
        return launch_linear_tc<kOutHeads>(X, W, M, N, K, bias, Y, dt == ATTNCACHE_BF16, sm_count, st, osh);
    return launch_linear_simt<kOutHeads>(dt, X, W, M, N, K, bias, Y, st, osh);
}

}  // namespace ac
