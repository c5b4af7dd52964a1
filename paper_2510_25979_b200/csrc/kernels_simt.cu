// kernels_simt.cu — CUDA-core (FFMA) kernels: the fp32 / mixed-dtype paths of search, A.V and
// causal attention, plus selection (compaction), key decoding and routing helpers.
//
// These are the generic-dtype paths (BASELINE.json configs[0] keeps fp32 features and fp32 V,
// which the bf16/fp16 tensor-core kernels do not cover).  Tensor-core kernels live in
// kernels_tc_*.cu.
#include "kernels.cuh"

namespace ac {

// ============================================================================================
// selection lists
// ============================================================================================
size_t rowlist_bytes(int64_t cap) { return 16 + (size_t)cap * 4 + 8 + (size_t)cap * 8; }

RowList rowlist_view(void *base, int64_t cap) {
    RowList r;
    char *p = (char *)base;
    r.count = (int32_t *)p;
    r.rows = (int32_t *)(p + 16);
    size_t off = 16 + (size_t)cap * 4;
    off = (off + 7) & ~(size_t)7;
    r.ents = (int64_t *)(p + off);
    r.cap = cap;
    return r;
}

__global__ void select_apply_kernel(const int64_t *idx, const uint8_t *hit, int64_t n, int64_t shard_begin,
                                    int64_t shard_count, RowList out, int *err) {
    compact_rows(n,
                 [&](int64_t b, int64_t &ent) {
                     bool want = hit ? (hit[b] != 0) : (idx[b] >= 0);
                     if (!want) return false;
                     int64_t e = idx[b] - shard_begin;
                     if (e < 0 || e >= shard_count) {
                         atomicOr(err, 1);
                         return false;
                     }
                     ent = e;
                     return true;
                 },
                 out);
}

__global__ void select_attend_kernel(const uint8_t *skip, int64_t n, RowList out) {
    compact_rows(n, [&](int64_t b, int64_t &ent) { ent = b; return skip == nullptr || skip[b] == 0; }, out);
}

cudaError_t launch_select_apply(const int64_t *idx, const uint8_t *hit, int64_t n, int64_t shard_begin,
                                int64_t shard_count, RowList out, int *err, cudaStream_t st) {
    select_apply_kernel<<<1, 1024, 0, st>>>(idx, hit, n, shard_begin, shard_count, out, err);
    return count_launches(1), cudaGetLastError();
}

cudaError_t launch_select_attend(const uint8_t *skip, int64_t n, RowList out, cudaStream_t st) {
    select_attend_kernel<<<1, 1024, 0, st>>>(skip, n, out);
    return count_launches(1), cudaGetLastError();
}

// ============================================================================================
// search: s[b][i] = q_b . x_i (fp32 accumulation), running top-1 per query, packed-key max
// (Alg. 1 l.255; reading R3)
// ============================================================================================
constexpr int kSearchQPB = 8;       // queries per CTA
constexpr int kSearchThreads = 256;

template <int DT>
__global__ void __launch_bounds__(kSearchThreads) search_simt_kernel(const typename Elem<DT>::T *__restrict__ q,
                                                                     const typename Elem<DT>::T *__restrict__ x,
                                                                     int64_t B, int64_t n, int D, int64_t gbase,
                                                                     int64_t per_block, uint64_t *keys) {
    extern __shared__ float sq[];  // [kSearchQPB][D]
    __shared__ unsigned long long skey[kSearchQPB];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.y * kSearchQPB;
    const int nq = (int)min64(kSearchQPB, B - b0);
    for (int i = tid; i < kSearchQPB * D; i += blockDim.x) {
        int qq = i / D;
        sq[i] = qq < nq ? Elem<DT>::ld(q, (b0 + qq) * D + (i % D)) : 0.f;
    }
    if (tid < kSearchQPB) skey[tid] = 0ull;
    __syncthreads();
    const int64_t e0 = (int64_t)blockIdx.x * per_block, e1 = min64(n, e0 + per_block);
    float best[kSearchQPB];
    uint32_t barg[kSearchQPB];
#pragma unroll
    for (int qq = 0; qq < kSearchQPB; ++qq) best[qq] = -INFINITY, barg[qq] = 0xFFFFFFFFu;
    for (int64_t e = e0 + warp; e < e1; e += nwarps) {
        float acc[kSearchQPB];
#pragma unroll
        for (int qq = 0; qq < kSearchQPB; ++qq) acc[qq] = 0.f;
        for (int k = lane; k < D; k += 32) {
            float xv = Elem<DT>::ld(x, e * D + k);
#pragma unroll
            for (int qq = 0; qq < kSearchQPB; ++qq) acc[qq] = fmaf(sq[qq * D + k], xv, acc[qq]);
        }
#pragma unroll
        for (int qq = 0; qq < kSearchQPB; ++qq) {
#pragma unroll
            for (int o = 16; o; o >>= 1) acc[qq] += __shfl_xor_sync(0xffffffffu, acc[qq], o);
            if (acc[qq] > best[qq]) best[qq] = acc[qq], barg[qq] = (uint32_t)(gbase + e);
        }
    }
    if (lane == 0) {
        for (int qq = 0; qq < nq; ++qq)
            if (barg[qq] != 0xFFFFFFFFu) atomicMax(&skey[qq], (unsigned long long)pack_key(best[qq], barg[qq]));
    }
    __syncthreads();
    if (tid < nq && skey[tid]) atomicMax((unsigned long long *)&keys[b0 + tid], skey[tid]);
}

cudaError_t launch_search_ffma(int32_t dt, const void *q, const void *x, int64_t B, int64_t n, int32_t D,
                               int64_t gbase, uint64_t *keys, cudaStream_t st) {
    if (B == 0 || n == 0) return cudaSuccess;
    const int64_t per_block = 256;
    dim3 grid((unsigned)((n + per_block - 1) / per_block), (unsigned)((B + kSearchQPB - 1) / kSearchQPB));
    size_t smem = sizeof(float) * kSearchQPB * D;
    switch (dt) {
    case ATTNCACHE_F32:
        if (cudaError_t e = cudaFuncSetAttribute(search_simt_kernel<ATTNCACHE_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem)) return e;
        search_simt_kernel<ATTNCACHE_F32><<<grid, kSearchThreads, smem, st>>>(
            (const float *)q, (const float *)x, B, n, D, gbase, per_block, keys);
        break;
    case ATTNCACHE_BF16:
        if (cudaError_t e = cudaFuncSetAttribute(search_simt_kernel<ATTNCACHE_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem)) return e;
        search_simt_kernel<ATTNCACHE_BF16><<<grid, kSearchThreads, smem, st>>>(
            (const __nv_bfloat16 *)q, (const __nv_bfloat16 *)x, B, n, D, gbase, per_block, keys);
        break;
    default:
        return cudaErrorInvalidValue;
    }
    return count_launches(1), cudaGetLastError();
}

__global__ void keys_decode_kernel(const uint64_t *keys, int n_shards, int64_t n, float tau, int64_t *idx,
                                   float *score, uint8_t *hit) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = 0;
        for (int r = 0; r < n_shards; ++r) {  // cross-shard top-1: max of packed keys (reading R3)
            uint64_t kr = keys[(int64_t)r * n + b];
            k = kr > k ? kr : k;
        }
        decode_key(k, tau, &idx[b], &score[b], &hit[b]);
    }
}

cudaError_t launch_keys_decode(const uint64_t *keys, int32_t n_shards, int64_t n, float tau, int64_t *idx, float *score,
                               uint8_t *hit, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int blocks = (int)min64((n + 255) / 256, 1024);
    keys_decode_kernel<<<blocks, 256, 0, st>>>(keys, n_shards, n, tau, idx, score, hit);
    return count_launches(1), cudaGetLastError();
}

// ============================================================================================
// apply (CUDA cores): one warp per output row i of a unit; lanes over columns.
//   O[i][c] = sum_{j <= i} A[i][j] V[j][c]   (causal maps: entries j > i are exact zeros; R11)
//   O[i][c] = sum_j A[i][j] V[j][c]          (non-causal encoder maps, f3)
// ============================================================================================
template <int MDT, int VDT>
__global__ void __launch_bounds__(256) apply_simt_kernel(ApplyArgs a) {
    using MT = typename Elem<MDT>::T;
    using VT = typename Elem<VDT>::T;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t count = *a.list.count;
    const int64_t units_per_row = (int64_t)a.n_lay * a.H;
    const int64_t total = count * units_per_row * a.S;
    const MT *maps = (const MT *)a.maps;
    const VT *V = (const VT *)a.V;
    VT *O = (VT *)a.O;
    for (int64_t w = gw; w < total; w += nw) {
        const int i = (int)(w % a.S);
        const int64_t u = w / a.S;              // unit within the selected rows
        const int64_t slot = u / units_per_row;
        const int64_t lh = u % units_per_row;   // (layer - layer_begin) * H + h
        const int l = (int)(lh / a.H), h = (int)(lh % a.H);
        const int64_t row = a.list.rows[slot], ent = a.list.ents[slot];
        const MT *A = maps + ((ent * a.L + a.layer_begin + l) * a.H + h) * a.map_stride + map_row_off(i, a.S, a.map_layout);
        const int64_t vbase = ((row * a.n_lay + l) * a.Hkv + h / (a.H / a.Hkv)) * (int64_t)a.S * a.d;
        const int64_t obase = ((row * a.n_lay + l) * a.H + h) * (int64_t)a.S * a.d;
        for (int c0 = 0; c0 < a.d; c0 += 32) {
            const int c = c0 + lane;
            float acc = 0.f;
            if (c < a.d)
                for (int j = 0, jn = a.causal ? i : a.S - 1; j <= jn; ++j)
                    acc = fmaf(Elem<MDT>::ld(A, j), Elem<VDT>::ld(V, vbase + (int64_t)j * a.d + c), acc);
            if (c < a.d) Elem<VDT>::st(O, obase + (int64_t)i * a.d + c, acc);
        }
    }
}

cudaError_t launch_apply_ffma(const ApplyArgs &a, int sm_count, cudaStream_t st) {
    int blocks = sm_count * 8;
#define AC_APPLY(MDT, VDT)                                                      \
    if (a.map_dt == MDT && a.act_dt == VDT) {                                  \
        apply_simt_kernel<MDT, VDT><<<blocks, 256, 0, st>>>(a);                \
        return count_launches(1), cudaGetLastError();                                             \
    }
    AC_APPLY(ATTNCACHE_F16, ATTNCACHE_F32)
    AC_APPLY(ATTNCACHE_BF16, ATTNCACHE_F32)
    AC_APPLY(ATTNCACHE_F16, ATTNCACHE_F16)
    AC_APPLY(ATTNCACHE_BF16, ATTNCACHE_BF16)
#undef AC_APPLY
    return cudaErrorInvalidValue;
}

// ============================================================================================
// attend (CUDA cores): one warp per query row i of a unit.
//   z_j = scale * Q_i . K_j (j <= i); p_j = exp(z_j - max); O_i = sum_j p_j V_j / sum_j p_j
// ============================================================================================
template <int DT>
__global__ void __launch_bounds__(256) attend_simt_kernel(AttendArgs a) {
    using T = typename Elem<DT>::T;
    extern __shared__ float sp[];  // [warps][S]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *p = sp + (int64_t)warp * a.S;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t count = *a.list.count;
    const int64_t units_per_row = (int64_t)a.L * a.H;
    const int64_t total = count * units_per_row * a.S;
    const T *Q = (const T *)a.Q, *K = (const T *)a.K, *V = (const T *)a.V;
    T *O = (T *)a.O;
    for (int64_t w = gw; w < total; w += nw) {
        const int i = (int)(w % a.S);
        const int64_t u = w / a.S;
        const int64_t slot = u / units_per_row, lh = u % units_per_row;
        const int64_t row = a.list.rows[slot];
        const int64_t base = (row * units_per_row + lh) * (int64_t)a.S * a.d;  // Q and O
        const int64_t kvbase =
            ((row * a.L + lh / a.H) * a.Hkv + (lh % a.H) / (a.H / a.Hkv)) * (int64_t)a.S * a.d;  // K and V
        float m = -INFINITY;
        for (int j = lane; j <= i; j += 32) {
            float z = 0.f;
            for (int c = 0; c < a.d; ++c)
                z = fmaf(Elem<DT>::ld(Q, base + (int64_t)i * a.d + c), Elem<DT>::ld(K, kvbase + (int64_t)j * a.d + c), z);
            z *= a.scale;
            p[j] = z;
            m = fmaxf(m, z);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float sum = 0.f;
        for (int j = lane; j <= i; j += 32) {
            float e = expf(p[j] - m);
            p[j] = e;
            sum += e;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        const float inv = 1.f / sum;
        for (int c = lane; c < a.d; c += 32) {
            float acc = 0.f;
            for (int j = 0; j <= i; ++j) acc = fmaf(p[j], Elem<DT>::ld(V, kvbase + (int64_t)j * a.d + c), acc);
            Elem<DT>::st(O, base + (int64_t)i * a.d + c, acc * inv);
        }
        __syncwarp();
    }
}

cudaError_t launch_attend_ffma(const AttendArgs &a, int sm_count, cudaStream_t st) {
    int blocks = sm_count * 4;
    size_t smem = sizeof(float) * 8 * a.S;
#define AC_ATTEND(DT)                                                                                   \
    if (a.dt == DT) {                                                                                  \
        cudaError_t e_ = cudaFuncSetAttribute(attend_simt_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e_ != cudaSuccess) return e_;                                                              \
        attend_simt_kernel<DT><<<blocks, 256, smem, st>>>(a);                                         \
        return count_launches(1), cudaGetLastError();                                                                     \
    }
    AC_ATTEND(ATTNCACHE_F32)
    AC_ATTEND(ATTNCACHE_F16)
    AC_ATTEND(ATTNCACHE_BF16)
#undef AC_ATTEND
    return cudaErrorInvalidValue;
}

// ============================================================================================
// capture (CUDA cores): one warp per query row i of a unit; P_ij = exp(z_ij - m) / sum, j <= i,
// rounded to the map dtype; entries j > i that the layout stores are written as +0.0.
// ============================================================================================
template <int DT, int MDT>
__global__ void __launch_bounds__(256) capture_simt_kernel(CaptureArgs a) {
    using T = typename Elem<DT>::T;
    using MT = typename Elem<MDT>::T;
    extern __shared__ float sp[];  // [warps][S]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *p = sp + (int64_t)warp * a.S;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t count = *a.list.count;
    const int64_t units_per_row = (int64_t)a.L * a.H;
    const int64_t total = count * units_per_row * a.S;
    const T *Q = (const T *)a.Q, *K = (const T *)a.K;
    MT *maps = (MT *)a.maps;
    const bool packed = a.map_layout == ATTNCACHE_MAPS_PACKED;
    for (int64_t w = gw; w < total; w += nw) {
        const int i = (int)(w % a.S);
        const int64_t u = w / a.S;
        const int64_t slot = u / units_per_row, lh = u % units_per_row;
        const int64_t row = a.list.rows[slot];
        const int64_t base = (row * units_per_row + lh) * (int64_t)a.S * a.d;  // Q
        const int64_t kbase = ((row * a.L + lh / a.H) * a.Hkv + (lh % a.H) / (a.H / a.Hkv)) * (int64_t)a.S * a.d;
        MT *mrow = maps + (row * units_per_row + lh) * a.map_stride + map_row_off(i, a.S, a.map_layout);
        const int stored = packed ? 8 * (i / 8 + 1) : a.S;
        float m = -INFINITY;
        for (int j = lane; j <= i; j += 32) {
            float z = 0.f;
            for (int c = 0; c < a.d; ++c)
                z = fmaf(Elem<DT>::ld(Q, base + (int64_t)i * a.d + c), Elem<DT>::ld(K, kbase + (int64_t)j * a.d + c), z);
            z *= a.scale;
            p[j] = z;
            m = fmaxf(m, z);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float sum = 0.f;
        for (int j = lane; j <= i; j += 32) {
            float e = expf(p[j] - m);
            p[j] = e;
            sum += e;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        const float inv = 1.f / sum;
        for (int j = lane; j < stored; j += 32) Elem<MDT>::st(mrow, j, j <= i ? p[j] * inv : 0.f);
        __syncwarp();
    }
}

cudaError_t launch_capture_simt(const CaptureArgs &a, int sm_count, cudaStream_t st) {
    int blocks = sm_count * 4;
    size_t smem = sizeof(float) * 8 * a.S;
#define AC_CAPTURE(DT, MDT)                                                                                  \
    if (a.dt == DT && a.map_dt == MDT) {                                                                    \
        cudaError_t e_ = cudaFuncSetAttribute(capture_simt_kernel<DT, MDT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e_ != cudaSuccess) return e_;                                                                   \
        capture_simt_kernel<DT, MDT><<<blocks, 256, smem, st>>>(a);                                         \
        return count_launches(1), cudaGetLastError();                                                       \
    }
    AC_CAPTURE(ATTNCACHE_F32, ATTNCACHE_F16)
    AC_CAPTURE(ATTNCACHE_F32, ATTNCACHE_BF16)
    AC_CAPTURE(ATTNCACHE_F16, ATTNCACHE_F16)
    AC_CAPTURE(ATTNCACHE_BF16, ATTNCACHE_BF16)
    AC_CAPTURE(ATTNCACHE_F16, ATTNCACHE_BF16)
    AC_CAPTURE(ATTNCACHE_BF16, ATTNCACHE_F16)
#undef AC_CAPTURE
    return cudaErrorInvalidValue;
}

// ============================================================================================
// RoPE (rotate-half): one thread per (unit, position, pair i < d/2); fp32 angle and rotation
// ============================================================================================
template <int DT>
__global__ void rope_kernel(typename Elem<DT>::T *X, int64_t n_units, int S, int d, float log2_base) {
    const int half = d / 2;
    const int64_t total = n_units * S * half;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t % half);
        const int64_t rs = t / half;  // (unit, position) row
        const int p = (int)(rs % S);
        const float theta = exp2f(-2.f * i / d * log2_base);
        float sn, cs;
        sincosf((float)p * theta, &sn, &cs);
        const int64_t row = rs * d;
        const float x1 = Elem<DT>::ld(X, row + i), x2 = Elem<DT>::ld(X, row + i + half);
        Elem<DT>::st(X, row + i, x1 * cs - x2 * sn);
        Elem<DT>::st(X, row + i + half, x2 * cs + x1 * sn);
    }
}

// 16-bit RoPE with 16-byte accesses: one thread rotates 8 consecutive pairs (i0..i0+7, i0+d/2..i0+d/2+7) of a
// row; angle p*theta reduced to [-pi, pi] in fp32, then the MUFU sine/cosine (|error| ~1e-6, far below bf16)
template <int DT>
__global__ void rope16_kernel(typename Elem<DT>::T *X, int64_t n_rows, int S, int d, float log2_base) {
    using T = typename Elem<DT>::T;
    const int half = d / 2, groups = half / 8;
    const int64_t total = n_rows * groups;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int i0 = (int)(t % groups) * 8;
        const int64_t rs = t / groups;  // (unit, position) row
        const float p = (float)(rs % S);
        T *x = X + rs * d;
        uint4 ua = *reinterpret_cast<const uint4 *>(x + i0), ub = *reinterpret_cast<const uint4 *>(x + half + i0);
        T *a = reinterpret_cast<T *>(&ua), *b = reinterpret_cast<T *>(&ub);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float ang = p * exp2f(-2.f * (float)(i0 + k) / (float)d * log2_base);
            ang = fmaf(-6.28318530717958647692f, rintf(ang * 0.15915494309189533577f), ang);
            float sn, cs;
            __sincosf(ang, &sn, &cs);
            const float x1 = Elem<DT>::ld(a, k), x2 = Elem<DT>::ld(b, k);
            Elem<DT>::st(a, k, x1 * cs - x2 * sn);
            Elem<DT>::st(b, k, x2 * cs + x1 * sn);
        }
        *reinterpret_cast<uint4 *>(x + i0) = ua;
        *reinterpret_cast<uint4 *>(x + half + i0) = ub;
    }
}

cudaError_t launch_rope(void *X, int64_t n_units, int32_t S, int32_t d, int32_t dt, float base, cudaStream_t st) {
    const int64_t total = n_units * S * (d / 2);
    if (total == 0) return cudaSuccess;
    const float lb = log2f(base);
    if (dt != ATTNCACHE_F32 && d % 16 == 0 && ((uintptr_t)X & 15) == 0) {
        const int64_t work = n_units * S * (d / 16);
        const int blocks = (int)min64((work + 255) / 256, 148 * 16);
        if (dt == ATTNCACHE_F16)
            rope16_kernel<ATTNCACHE_F16><<<blocks, 256, 0, st>>>((__half *)X, n_units * S, S, d, lb);
        else
            rope16_kernel<ATTNCACHE_BF16><<<blocks, 256, 0, st>>>((__nv_bfloat16 *)X, n_units * S, S, d, lb);
        return count_launches(1), cudaGetLastError();
    }
    const int blocks = (int)min64((total + 255) / 256, 148 * 32);
    switch (dt) {
    case ATTNCACHE_F32: rope_kernel<ATTNCACHE_F32><<<blocks, 256, 0, st>>>((float *)X, n_units, S, d, lb); break;
    case ATTNCACHE_F16: rope_kernel<ATTNCACHE_F16><<<blocks, 256, 0, st>>>((__half *)X, n_units, S, d, lb); break;
    default: rope_kernel<ATTNCACHE_BF16><<<blocks, 256, 0, st>>>((__nv_bfloat16 *)X, n_units, S, d, lb); break;
    }
    return count_launches(1), cudaGetLastError();
}

// ============================================================================================
// packed map layout: one warp per map row, lanes over 16-byte pieces
// ============================================================================================
__global__ void pack_maps_kernel(const uint4 *dense, int64_t n_maps, int S, uint4 *packed, bool unpack) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t rows = n_maps * S;
    const int64_t dense_pieces = (int64_t)S * S / 8, packed_pieces = packed_row_off(S) / 8;
    const int per_row = S / 8;
    for (int64_t w = gw; w < rows; w += nw) {
        const int64_t m = w / S;
        const int i = (int)(w % S);
        const uint4 *drow = dense + m * dense_pieces + (int64_t)i * per_row;
        const uint4 *prow = packed + m * packed_pieces + packed_row_off(i) / 8;
        const int stored = i / 8 + 1;  // pieces kept for row i
        for (int c = lane; c < per_row; c += 32) {
            if (!unpack) {
                if (c < stored) ((uint4 *)prow)[c] = drow[c];
            } else {
                ((uint4 *)drow)[c] = c < stored ? prow[c] : make_uint4(0, 0, 0, 0);
            }
        }
    }
}

cudaError_t launch_pack_maps(const void *dense, int64_t n_maps, int32_t S, void *packed, bool unpack, cudaStream_t st) {
    if (n_maps == 0) return cudaSuccess;
    const int64_t warps = n_maps * S;
    const int blocks = (int)min64((warps * 32 + 255) / 256, 148 * 64);
    pack_maps_kernel<<<blocks, 256, 0, st>>>((const uint4 *)dense, n_maps, S, (uint4 *)packed, unpack);
    return count_launches(1), cudaGetLastError();
}

// ============================================================================================
// routing helpers
// ============================================================================================
__global__ void route_plan_kernel(const int64_t *idx, const uint8_t *hit, int64_t n, const int64_t *sb, int world,
                                  int32_t *owner, int32_t *counts, int64_t *order) {
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t b = tid; b < n; b += blockDim.x) {
        int o = -1;
        if (hit ? hit[b] != 0 : idx[b] >= 0) {
            int64_t e = idx[b];
            for (int r = 0; r < world; ++r)
                if (e >= sb[r] && e < sb[r + 1]) o = r;
        }
        owner[b] = o;
    }
    if (tid == 0) base = 0;
    __syncthreads();
    for (int r = 0; r < world; ++r) {
        int start = base;
        for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
            int64_t b = b0 + tid;
            bool sel = b < n && owner[b] == r;
            unsigned m = __ballot_sync(0xffffffffu, sel);
            if (lane == 0) warp_tot[warp] = __popc(m);
            __syncthreads();
            if (tid == 0) {
                int run = base;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                    int t = warp_tot[w];
                    warp_tot[w] = run;
                    run += t;
                }
                base = run;
            }
            __syncthreads();
            if (sel) order[warp_tot[warp] + __popc(m & ((1u << lane) - 1u))] = b;
            __syncthreads();
        }
        if (tid == 0) counts[r] = base - start;
        __syncthreads();
    }
}

cudaError_t launch_route_plan(const int64_t *idx, const uint8_t *hit, int64_t n, const int64_t *shard_begins,
                              int32_t world, int32_t *owner, int32_t *counts, int64_t *order, cudaStream_t st) {
    route_plan_kernel<<<1, 1024, 0, st>>>(idx, hit, n, shard_begins, world, owner, counts, order);
    return count_launches(1), cudaGetLastError();
}

template <typename W>
__global__ void copy_rows_kernel(const W *src, const int64_t *rows, int64_t n_rows, int64_t row_words, W *dst,
                                 bool gather) {
    // rows over blockIdx.y (grid-stride), words of a row over blockIdx.x: no per-element 64-bit division
    for (int64_t k = blockIdx.y; k < n_rows; k += gridDim.y) {
        const int64_t r = rows[k];
        const W *s = src + (gather ? r : k) * row_words;
        W *d = dst + (gather ? k : r) * row_words;
        for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < row_words; w += (int64_t)gridDim.x * blockDim.x)
            d[w] = s[w];
    }
}

cudaError_t launch_copy_rows(const void *src, const int64_t *rows, int64_t n_rows, int64_t row_bytes, void *dst,
                             bool gather, bool ok16, int sms, cudaStream_t st) {
    if (n_rows == 0) return cudaSuccess;
    const int64_t words = ok16 ? row_bytes / 16 : row_bytes / 8;
    // about 16 resident CTAs per SM of the budget in total: split between the rows and the words of a row
    const int64_t gy = min64(n_rows, 65535);
    const int64_t gx = max64(1, min64((words + 255) / 256, ((int64_t)sms * 16 + gy - 1) / gy));
    const dim3 grid((unsigned)gx, (unsigned)gy);
    if (ok16)  // 16-byte rows AND 16-byte aligned bases (an 8-byte aligned base takes the int2 path)
        copy_rows_kernel<int4><<<grid, 256, 0, st>>>((const int4 *)src, rows, n_rows, words, (int4 *)dst, gather);
    else
        copy_rows_kernel<int2><<<grid, 256, 0, st>>>((const int2 *)src, rows, n_rows, words, (int2 *)dst, gather);
    return count_launches(1), cudaGetLastError();
}

}  // namespace ac
