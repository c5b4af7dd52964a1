// Microbenchmark (sm_100a): tcgen05.mma issue-to-retire throughput per SM for the shapes the attention and
// A.V kernels use.  One CTA per SM, one thread issues `iters` groups of 8 MMAs (K = 8 x 16 = 128) and
// commits each group to an mbarrier; the thread waits for the last commit.  Prints cycles per MMA
// instruction and the implied fraction of the M*N/256-cycle floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_25979_b200/csrc -o /tmp/mma scripts/microbench/mma_rate.cu && /tmp/mma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ac::sm100;

// mode: 0 SS N=128, 1 SS N=256, 2 SS N=64, 3 TS (A in TMEM) N=128 B MN-major, 4 alternate SS N=128 / TS N=128,
//       5 TS N=128 B K-major, 6 SS N=128 B MN-major, 7 TS N=256 B MN-major, 8 TS N=256 B K-major,
//       9 SS N=128 A MN-major B K-major, 10 SS N=256 A MN-major B K-major, 11 SS N=128 both MN-major
template <int mode>
__global__ void mma_rate(int iters, unsigned long long *cycles) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc<512>(&slot);
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = a + 32 * 1024;
        const uint32_t id128 = idesc_f16(128, 128, 1, 0, 0), id256 = idesc_f16(128, 256, 1, 0, 0);
        const uint32_t id64 = idesc_f16(128, 64, 1, 0, 0), idts = idesc_f16(128, 128, 1, 0, 1);
        const uint32_t idtsk = idesc_f16(128, 128, 1, 0, 0), idssmn = idesc_f16(128, 128, 1, 0, 1);
        const uint32_t idts256 = idesc_f16(128, 256, 1, 0, 1), idts256k = idesc_f16(128, 256, 1, 0, 0);
        const uint32_t idamn = idesc_f16(128, 128, 1, 1, 0), idamn256 = idesc_f16(128, 256, 1, 1, 0);
        const uint32_t idbothmn = idesc_f16(128, 128, 1, 1, 1);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int m = mode == 4 ? (it & 1) * 3 : mode;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t off = (k >> 2) * (128 * 128) + (k & 3) * 32;
                if (m == 0 || m == 12 || m == 13)
                    umma_f16(tmem + (it & 1) * 128, smem_desc(a + off, 16, 1024, kSwizzle128B),
                             smem_desc(b + off, 16, 1024, kSwizzle128B), id128, k != 0);
                else if (m == 1)
                    umma_f16(tmem + (it & 1) * 256, smem_desc(a + off, 16, 1024, kSwizzle128B),
                             smem_desc(b + off, 16, 1024, kSwizzle128B), id256, k != 0);
                else if (m == 2)
                    umma_f16(tmem + (it & 1) * 64, smem_desc(a + off, 16, 1024, kSwizzle128B),
                             smem_desc(b + off, 16, 1024, kSwizzle128B), id64, k != 0);
                else if (m == 3)
                    umma_f16_ts(tmem + 256 + (it & 1) * 128, tmem + k * 8,
                                smem_desc(b + k * 2048, 128 * 128, 1024, kSwizzle128B), idts, k != 0);
                else if (m == 5)
                    umma_f16_ts(tmem + 256 + (it & 1) * 128, tmem + k * 8,
                                smem_desc(b + off, 16, 1024, kSwizzle128B), idtsk, k != 0);
                else if (m == 6)
                    umma_f16(tmem + (it & 1) * 128, smem_desc(a + off, 16, 1024, kSwizzle128B),
                             smem_desc(b + k * 2048, 128 * 128, 1024, kSwizzle128B), idssmn, k != 0);
                else if (m == 7)
                    umma_f16_ts(tmem + 256, tmem + k * 8, smem_desc(b + k * 2048, 128 * 128, 1024, kSwizzle128B),
                                idts256, k != 0);
                else if (m == 8)
                    umma_f16_ts(tmem + 256, tmem + k * 8, smem_desc(b + off, 16, 1024, kSwizzle128B), idts256k, k != 0);
                else if (m == 9)
                    umma_f16(tmem + (it & 1) * 128, smem_desc(a + k * 2048, 128 * 128, 1024, kSwizzle128B),
                             smem_desc(b + off, 16, 1024, kSwizzle128B), idamn, k != 0);
                else if (m == 10)
                    umma_f16(tmem + (it & 1) * 256, smem_desc(a + k * 2048, 128 * 128, 1024, kSwizzle128B),
                             smem_desc(b + off, 16, 1024, kSwizzle128B), idamn256, k != 0);
                else
                    umma_f16(tmem + (it & 1) * 128, smem_desc(a + k * 2048, 128 * 128, 1024, kSwizzle128B),
                             smem_desc(b + k * 2048, 128 * 128, 1024, kSwizzle128B), idbothmn, k != 0);
            }
            if (mode == 13) {
                umma_commit(&bar2);
                umma_commit(&bar2);
            }
            if (mode == 12) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma_f16_ts(tmem + 256, tmem + k * 8, smem_desc(b + k * 2048, 128 * 128, 1024, kSwizzle128B), idts,
                                k != 0);
            }
            umma_commit(&bar);
        }
        mbar_wait(&bar, (iters - 1) & 1);
        long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

template <int mode>
void run(const char *name, int n, unsigned long long *d) {
    unsigned long long h;
    const int smem = 97 * 1024;
    cudaFuncSetAttribute(mma_rate<mode>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    mma_rate<mode><<<148, 128, smem>>>(iters, d);
    mma_rate<mode><<<148, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / (iters * (mode == 12 ? 16.0 : 8.0));
    const double floor = 128.0 * n / 256.0;
    printf("%-40s %7.1f cycles/MMA (floor %5.1f) -> %5.1f%% of floor   [%s]\n", name, per, floor, 100.0 * floor / per,
           cudaGetErrorString(e));
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 8);
    run<0>("SS M128 N128", 128, d);
    run<1>("SS M128 N256", 256, d);
    run<2>("SS M128 N64", 64, d);
    run<3>("TS M128 N128 (A in TMEM, B MN-major)", 128, d);
    run<4>("alternating SS N128 / TS N128", 128, d);
    run<5>("TS M128 N128 B K-major", 128, d);
    run<6>("SS M128 N128 B MN-major", 128, d);
    run<7>("TS M128 N256 B MN-major", 256, d);
    run<8>("TS M128 N256 B K-major", 256, d);
    run<9>("SS N128 A MN-major B K-major", 128, d);
    run<10>("SS N256 A MN-major B K-major", 256, d);
    run<11>("SS N128 A MN-major B MN-major", 128, d);
    run<12>("SS N128 x8 then TS N128 x8 (per 16)", 128, d);
    run<13>("SS N128, 3 commits per 8 MMAs", 128, d);
    return 0;
}
