// double-precision sincos on sm_100a: latency of one call in a dependent chain, and the cost per call of
// four independent calls issued back to back (do they interleave?).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* clk, double a) {
    double x = a + threadIdx.x * 1e-3, s, c;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) { sincos(x, &s, &c); x = s * 0.3 + c * 0.1; }
    long long t1 = clock64();
    if (threadIdx.x == 0) clk[0] = (t1 - t0) / 64;
    double y[4] = {x, x + 0.1, x + 0.2, x + 0.3};
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) {
        double sn[4], cs[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) sincos(y[j], &sn[j], &cs[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) y[j] = sn[j] * 0.3 + cs[j] * 0.1;
    }
    t1 = clock64();
    if (threadIdx.x == 0) clk[1] = (t1 - t0) / 256;
    out[threadIdx.x] = x + y[0] + y[1] + y[2] + y[3];
}
int main() {
    double* out; long long* clk; cudaMalloc(&out, 8192); cudaMalloc(&clk, 256);
    for (int threads : {32, 256}) {
        k<<<1, threads>>>(out, clk, 0.05); cudaDeviceSynchronize();
        long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
        printf("threads=%d  sincos(double) dependent: %lld cycles per call;  four independent calls: %lld cycles per call\n", threads, h[0], h[1]);
    }
    return 0;
}
