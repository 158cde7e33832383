// FP64 dependent-chain latencies on one warp (asm volatile so nothing is folded or moved across the clocks).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* clk, double a, double b) {
    double x = a;
    long long t0, t1;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(a), "d"(b));
    t1 = clock64(); if (threadIdx.x == 0) clk[0] = (t1 - t0) / 64;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(a));
    t1 = clock64(); if (threadIdx.x == 0) clk[1] = (t1 - t0) / 64;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(b));
    t1 = clock64(); if (threadIdx.x == 0) clk[2] = (t1 - t0) / 64;
    // rsqrt chain via the CUDA math function, kept dependent through an asm add
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) { x = rsqrt(x); asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(b)); }
    t1 = clock64(); if (threadIdx.x == 0) clk[3] = (t1 - t0) / 32;
    // shuffle of a double, dependent
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) { x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31); asm volatile("" : "+d"(x)); }
    t1 = clock64(); if (threadIdx.x == 0) clk[4] = (t1 - t0) / 64;
    // 8 independent fma chains: issue interval
    double y[8]; for (int j = 0; j < 8; ++j) y[j] = a + j;
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(y[j]) : "d"(a), "d"(b));
    t1 = clock64(); if (threadIdx.x == 0) clk[5] = (t1 - t0) / 256;
    for (int j = 0; j < 8; ++j) x += y[j];
    out[threadIdx.x] = x;
}
int main() {
    double* out; long long* clk; cudaMalloc(&out, 8192); cudaMalloc(&clk, 256);
    for (int threads : {32, 128, 256}) {
        k<<<1, threads>>>(out, clk, 1.0000001, 0.5); cudaDeviceSynchronize();
        long long h[8]; cudaMemcpy(h, clk, 64, cudaMemcpyDeviceToHost);
        printf("threads=%d  dfma_lat=%lld dmul_lat=%lld dadd_lat=%lld rsqrt+add=%lld shfl64_lat=%lld dfma_issue(8 chains)=%lld cycles\n",
               threads, h[0], h[1], h[2], h[3], h[4], h[5]);
    }
    return 0;
}
