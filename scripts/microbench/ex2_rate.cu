// Microbenchmark (sm_100a): MUFU ex2 throughput per SM for f32, f16x2 and bf16x2 operands (148 CTAs x 1024
// threads, 8 independent chains per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ex2 scripts/microbench/ex2_rate.cu && /tmp/ex2
#include <cstdio>
#include <cstdint>
template <int mode>
__global__ void k(int iters, uint32_t *out, unsigned long long *cyc) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) x[i] = 0xbc00bc00u ^ (threadIdx.x + i);  // f16x2 around -1
    float f[8];
    for (int i = 0; i < 8; ++i) f[i] = -1.f - 0.001f * (threadIdx.x + i);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (mode == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            else if (mode == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
            else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[i]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < 8; ++i) acc ^= x[i] ^ __float_as_uint(f[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int mode>
void run(const char *n, uint32_t *o, unsigned long long *c) {
    const int iters = 4096;
    k<mode><<<148, 1024>>>(iters, o, c);
    k<mode><<<148, 1024>>>(iters, o, c);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    // instructions per SM: 32 warps * iters * 8
    double instr = 32.0 * iters * 8;
    printf("%-10s %.2f cycles per warp-instruction per SM -> %.1f lanes/clk/SM, %.1f results/clk/SM\n", n, h / instr,
           32.0 * instr / h, (mode ? 64.0 : 32.0) * instr / h);
}
int main() {
    uint32_t *o; unsigned long long *c;
    cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
    run<0>("f32", o, c); run<1>("f16x2", o, c); run<2>("bf16x2", o, c);
    // accuracy of f16x2 ex2 incl. subnormal outputs
    return 0;
}
