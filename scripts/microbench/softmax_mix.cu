// Microbenchmark (sm_100a): the d = 128 attention softmax's exponential loop in isolation -- per key pair
// FFMA2 (scale, -max), two MUFU.EX2, FADD2 (row sum), F2FP (bf16 pack) -- with 2 warps per SM sub-partition
// (8 warps per CTA, one CTA per SM) as in attend_split_kernel, optionally computing `poly` of every 8 pairs
// with the FMA-pipe polynomial exp2_poly2.  Prints cycles per 64-pair block per SMSP (MUFU floor: 1024).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2510_25979_b200/csrc -o /tmp/smx scripts/microbench/softmax_mix.cu && /tmp/smx
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

#include "sm100.cuh"

using namespace ac::sm100;

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int kPoly>
__global__ void __launch_bounds__(256, 1) mix(int iters, uint32_t *out, unsigned long long *cyc) {
    uint32_t sv[64];
#pragma unroll
    for (int e = 0; e < 64; ++e) sv[e] = __float_as_uint(-0.01f * (float)((threadIdx.x + e) & 63));
    const uint64_t scale2 = pack2(1.1f, 1.1f), neg_m2 = pack2(-0.5f, -0.5f);
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint64_t rs2[4] = {0ull, 0ull, 0ull, 0ull};
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const uint64_t x2 = ffma2(((uint64_t)sv[2 * e + 1] << 32) | sv[2 * e], scale2, neg_m2);
            float p0, p1;
            if ((e & 7) < kPoly) {
                exp2_poly2(x2, p0, p1);
            } else {
                p0 = ex2f(__uint_as_float((uint32_t)x2));
                p1 = ex2f(__uint_as_float((uint32_t)(x2 >> 32)));
            }
            rs2[e & 3] = fadd2(rs2[e & 3], pack2(p0, p1));
            __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
            pk[e] = *reinterpret_cast<uint32_t *>(&h2);
        }
        const uint64_t t2 = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += pk[e];
        acc += (uint32_t)t2;
        sv[it & 63] ^= acc & 1u;  // keep the loop from being hoisted
    }
    __syncthreads();
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int kPoly>
void run(uint32_t *o, unsigned long long *c) {
    const int iters = 2000;
    mix<kPoly><<<148, 256>>>(iters, o, c);
    mix<kPoly><<<148, 256>>>(iters, o, c);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("poly %d/8: %.0f cycles per block (2 warps x 32 pairs per SMSP; MUFU floor %d)\n", kPoly, (double)h / iters,
           1024 * (8 - kPoly) / 8);
}

int main() {
    uint32_t *o;
    unsigned long long *c;
    cudaMalloc(&o, 148 * 256 * 4);
    cudaMalloc(&c, 8);
    run<0>(o, c);
    run<1>(o, c);
    run<2>(o, c);
    run<3>(o, c);
    return 0;
}
