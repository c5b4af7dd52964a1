// Microbenchmark (sm_100a): does a warp that issues tcgen05.mma into a busy tensor pipe slow the other warps
// of its SM sub-partition (SMSP = warp % 4)?  One CTA per SM, 12 warps: warp `mma_warp` issues `iters` groups of
// 16 M128 N128 K16 MMAs (whole warp in the loop, one elected lane issuing, as the attention kernels do, or
// lane 0 only), warps 4-11 each run the same MUFU-bound exp2 loop; prints each exp warp's cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_25979_b200/csrc -o /tmp/msm \
//        scripts/microbench/mma_smsp.cu && /tmp/msm
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ac::sm100;

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// mode 0: no MMAs; 1: whole warp, elected lane issues (umma_*_w); 2: lane 0 only issues; 3: whole warp but
// each group waits for the previous group's commit before issuing (the queue never backs up); 4: as 3 with a
// suspend-time hint on the wait (mbar_wait_hint)
template <int mode>
__global__ void bench(int iters, int exp_iters, int mma_warp, unsigned long long *out, float *sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t q = smem_u32(smem), k = q + 32768;
    if (mode != 0 && warp == mma_warp && (mode != 2 || lane == 0)) {
        const uint32_t id_s = idesc_f16(128, 128, 1, 0, 0);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (mode == 3 && it > 0) mbar_wait(&bar, (it - 1) & 1);
            if (mode == 4 && it > 0) mbar_wait_hint(&bar, (it - 1) & 1);
            for (int h = 0; h < 2; ++h) {
                if (mode == 2)
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
                        umma_f16(tmem + h * 128, smem_desc(q + off, 16, 1024, kSwizzle128B),
                                 smem_desc(k + off, 16, 1024, kSwizzle128B), id_s, kk != 0);
                    }
                else
                    umma_f16_ss_k8_w<128 * 128 / 16>(tmem + h * 128, smem_desc(q, 16, 1024, kSwizzle128B),
                                                     smem_desc(k, 16, 1024, kSwizzle128B), id_s, 0u);
            }
            if (mode == 2) umma_commit(&bar);
            else umma_commit_w(&bar);
        }
        mbar_wait(&bar, (iters - 1) & 1);
        if (blockIdx.x == 0 && lane == 0) out[12] = clock64() - t0;
    } else if (warp >= 4) {
        float x = 0.001f * lane, acc = 0.f;
        long long t0 = clock64();
        for (int i = 0; i < exp_iters; ++i) {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
                const float p0 = ex2(x + e * 0.01f), p1 = ex2(x - e * 0.01f);
                acc += p0 + p1;
            }
            x += 1e-7f;
        }
        if (blockIdx.x == 0 && lane == 0) out[warp] = clock64() - t0;
        if (acc == 12345.f) sink[threadIdx.x] = acc;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int mode>
void run(const char *name, int mma_warp, int iters, int exp_iters, unsigned long long *d, float *sink) {
    const int smem = 65 * 1024;
    cudaFuncSetAttribute(bench<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(d, 0, 16 * 8);
    bench<mode><<<148, 384, smem>>>(iters, exp_iters, mma_warp, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[16];
    cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
    printf("%-46s mma warp %d: MMA %8.1f cyc/16 MMAs | exp warps 4..11 (SMSP w%%4):", name, mma_warp,
           iters ? (double)h[12] / iters : 0.0);
    for (int w = 4; w < 12; ++w) printf(" %7.0f", (double)h[w] / exp_iters);
    printf("  cyc/64 exps [%s]\n", cudaGetErrorString(e));
}

int main() {
    unsigned long long *d;
    float *sink;
    cudaMalloc(&d, 16 * 8);
    cudaMalloc(&sink, 4096);
    const int exp_iters = 4000, iters = 1000;  // MMA work ~4000 x 1024 cycles, exps ~4000 x ~1024 (2 warps / SMSP)
    run<0>("no MMA", 1, iters, exp_iters, d, sink);
    run<1>("whole warp, elected issue (blocking)", 1, iters * 4, exp_iters, d, sink);
    run<2>("lane 0 only issues (blocking)", 1, iters * 4, exp_iters, d, sink);
    run<3>("whole warp, waits for previous group", 1, iters * 4, exp_iters, d, sink);
    run<4>("whole warp, hinted wait for previous group", 1, iters * 4, exp_iters, d, sink);
    run<1>("whole warp, elected issue, on warp 2", 2, iters * 4, exp_iters, d, sink);
    return 0;
}
