// Microbenchmark (sm_100a): does concurrent TMA (bulk copy) traffic into shared memory slow the attention's
// MMAs, and how much L2 -> SM bandwidth do 148 SMs get?  One CTA per SM; thread 0 issues `iters` groups of
// the d = 128 attention block's MMAs (S = Q K^T: 8 x M128 N128 K16, SS or with Q in TMEM (TS); PV: 8 x TS
// M128 N128 K16, B MN-major), thread 32 streams 32 KB bulk copies from an L2-resident buffer into a ring of
// shared-memory slots the MMAs do not read.  Prints cycles per group for both and the copy rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_25979_b200/csrc -o /tmp/mvt \
//        scripts/microbench/mma_vs_tma.cu && /tmp/mvt
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ac::sm100;

constexpr int kChunk = 32 * 1024;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// s_mode: 0 no S, 1 S SS, 2 S TS (Q in TMEM); pv: 0/1; loads_per_group: 32 KB copies per MMA group (x2 = 64 KB)
template <int s_mode, int pv, int kRing, int tm = 0>
__global__ void bench(int iters, int n_loads, const uint8_t *src, size_t src_chunks, unsigned long long *out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, full[kRing];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < kRing; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t q = smem_u32(smem), k = q + kChunk, v = k + kChunk, ring = v + kChunk;
    if (warp == 0 && lane == 0) {
        const uint32_t id_s = idesc_f16(128, 128, 1, 0, 0), id_pv = idesc_f16(128, 128, 1, 0, 1);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t sbuf = tmem + (it & 1) * 128;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
                if (s_mode == 1)
                    umma_f16(sbuf, smem_desc(q + off, 16, 1024, kSwizzle128B), smem_desc(k + off, 16, 1024, kSwizzle128B),
                             id_s, kk != 0);
                else if (s_mode == 2)
                    umma_f16_ts(sbuf, tmem + 384 + kk * 8, smem_desc(k + off, 16, 1024, kSwizzle128B), id_s, kk != 0);
            }
            if (pv) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tmem + 256, sbuf + kk * 8, smem_desc(v + kk * 2048, 128 * 128, 1024, kSwizzle128B), id_pv,
                                kk != 0);
            }
            umma_commit(&bar);
        }
        if (iters) mbar_wait(&bar, (iters - 1) & 1);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    } else if (warp == 1 && lane == 0) {
        long long t0 = clock64();
        for (int i = 0; i < n_loads; ++i) {
            const int s = i % kRing;
            if (i >= kRing) mbar_wait(&full[s], ((i / kRing) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], kChunk);
            const size_t c = ((size_t)blockIdx.x * 7 + i) % src_chunks;
            bulk_g2s(ring + s * kChunk, src + c * kChunk, kChunk, &full[s]);
        }
        for (int i = n_loads > kRing ? n_loads - kRing : 0; i < n_loads; ++i)
            mbar_wait(&full[i % kRing], (i / kRing) & 1);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[1] = t1 - t0;
    }
    else if (tm && warp >= 4) {
        // TMEM traffic of a softmax: per round a 64-column load (tm & 1) and a 32-column store (tm & 2) of
        // columns 448.. of this warp's lane quarter, `rounds` times (the MMAs do not touch them)
        const uint32_t addr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 448;
        uint32_t acc = 0;
        const int rounds = (tm & 4) ? iters : iters * 8;
        for (int r = 0; r < rounds; ++r) {
            if (tm & 4) __nanosleep(400);  // ~ one softmax block's TMEM traffic per MMA group
            uint32_t v[64];
            if (tm & 1) {
                tmem_ld_32x32b_x64(addr, v);
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 64; ++e) acc += v[e];
            }
            if (tm & 2) {
                uint32_t w[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) w[e] = acc + e;
                tmem_st_32x32b_x16(addr, w);
                tmem_st_32x32b_x16(addr + 16, w);
                tmem_st_wait();
            }
        }
        if (acc == 0x12345678u) out[2] = acc;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int s_mode, int pv, int kRing = 2, int tm = 0>
void run(const char *name, int iters, int n_loads, const uint8_t *src, size_t chunks, unsigned long long *d) {
    const int smem = (3 + kRing) * kChunk + 1024;
    cudaFuncSetAttribute(bench<s_mode, pv, kRing, tm>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(d, 0, 16);
    bench<s_mode, pv, kRing, tm><<<148, tm ? 384 : 128, smem>>>(iters, n_loads, src, chunks, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<s_mode, pv, kRing, tm><<<148, tm ? 384 : 128, smem>>>(iters, n_loads, src, chunks, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const int n_mma = (s_mode ? 8 : 0) + (pv ? 8 : 0);
    const double per_group = iters ? (double)h[0] / iters : 0;
    const double load_bpc = n_loads ? (double)n_loads * kChunk / h[1] : 0;
    const double clk = (double)(h[0] > h[1] ? h[0] : h[1]) / (ms * 1e-3) / 1e9;
    printf("ring %d %-40s mma %7.1f cyc/group (%5.1f/MMA, floor 64)  copy %6.1f B/cyc/SM (%6.2f TB/s)  %.3f ms ~%.2f GHz [%s]\n",
           kRing, name, per_group, n_mma ? per_group / n_mma : 0.0, load_bpc, (double)n_loads * kChunk * 148 / (ms * 1e-3) / 1e12,
           ms, clk, cudaGetErrorString(e));
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 16);
    const size_t chunks = 1024;  // 32 MB source: L2-resident
    uint8_t *src;
    cudaMalloc(&src, chunks * kChunk);
    cudaMemset(src, 0, chunks * kChunk);
    const int it = 4000;
    run<1, 0>("S SS only", it, 0, src, chunks, d);
    run<2, 0>("S TS (Q in TMEM) only", it, 0, src, chunks, d);
    run<1, 1>("S SS + PV", it, 0, src, chunks, d);
    run<2, 1>("S TS + PV", it, 0, src, chunks, d);
    run<0, 0>("copies only (8000 x 32 KB)", 0, 2 * it, src, chunks, d);
    run<1, 0>("S SS + 32 KB copies/group", it, it, src, chunks, d);
    run<1, 1>("S SS + PV + 64 KB copies/group", it, 2 * it, src, chunks, d);
    run<2, 1>("S TS + PV + 64 KB copies/group", it, 2 * it, src, chunks, d);
    run<1, 1>("S SS + PV + 32 KB copies/group", it, it, src, chunks, d);
    run<2, 1>("S TS + PV + 32 KB copies/group", it, it, src, chunks, d);
    run<1, 1>("S SS + PV + 96 KB copies/group", it, 3 * it, src, chunks, d);
    run<1, 1, 2, 1>("S SS + PV + 8 warps TMEM ld x64", it, 0, src, chunks, d);
    run<1, 1, 2, 3>("S SS + PV + 8 warps TMEM ld x64 + st 2x16", it, 0, src, chunks, d);
    run<1, 1, 2, 2>("S SS + PV + 8 warps TMEM st 2x16", it, 0, src, chunks, d);
    run<1, 1, 2, 3>("S SS + PV + TMEM ld/st + 64 KB copies", it, 2 * it, src, chunks, d);
    run<1, 1, 2, 7>("S SS + PV + paced TMEM ld/st", it, 0, src, chunks, d);
    run<1, 1, 2, 7>("S SS + PV + paced TMEM ld/st + 64 KB copies", it, 2 * it, src, chunks, d);
    run<0, 0, 4>("copies only (8000 x 32 KB)", 0, 2 * it, src, chunks, d);
    run<1, 1, 4>("S SS + PV + 64 KB copies/group", it, 2 * it, src, chunks, d);
    run<2, 1, 4>("S TS + PV + 64 KB copies/group", it, 2 * it, src, chunks, d);
    run<1, 1, 4>("S SS + PV + 32 KB copies/group", it, it, src, chunks, d);
    return 0;
}
