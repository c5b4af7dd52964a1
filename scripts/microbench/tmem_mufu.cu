// Microbenchmark (sm_100a): TMEM load throughput and MUFU.EX2 throughput per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tmem_mufu.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__global__ void tmem_bw(int iters, int wait_each, unsigned long long *cycles, uint32_t *sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t r[32];
        ld32(base + (i & 3) * 32, r);
        if (wait_each) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        else if ((i & 3) == 3) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= r[e];
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__global__ void mufu_bw(int iters, unsigned long long *cycles, float *sink) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = -0.001f * (threadIdx.x + k);
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    unsigned long long *cyc;
    uint32_t *sink;
    float *fs;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sink, 1 << 20);
    cudaMalloc(&fs, 1 << 20);
    const int iters = 4096;
    for (int warps : {4, 8}) {
        for (int we : {1, 0}) {
            tmem_bw<<<1, warps * 32>>>(iters, we, cyc, sink);
            cudaDeviceSynchronize();
            unsigned long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            double bytes = (double)iters * warps * 32 * 32 * 4;
            printf("TMEM ld x32: %d warps, wait_each=%d: %.1f cycles per warp-load, %.1f B/cycle per SM  (%s)\n", warps, we,
                   (double)c / iters, bytes / c, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (int warps : {4, 8, 16}) {
        mufu_bw<<<1, warps * 32>>>(iters, cyc, fs);
        cudaDeviceSynchronize();
        unsigned long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double ops = (double)iters * 8 * warps * 32;
        printf("MUFU.EX2: %d warps: %.2f lane-ops/cycle per SM\n", warps, ops / c);
    }
    return 0;
}
