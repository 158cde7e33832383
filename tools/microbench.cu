// Latency microbenchmarks for the FP64 building blocks of the front kernel (one warp / one CTA).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* clk, double seed) {
    __shared__ double sm[1024];
    int tid = threadIdx.x;
    sm[tid] = seed + tid; __syncthreads();
    double x = seed + 1.5, y = seed + 0.25, acc = 0;
    long long t0, t1;
    // 1. dependent DFMA chain
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) x = fma(x, 1.0000001, y);
    t1 = clock64(); if (tid == 0) clk[0] = (t1 - t0) / 64; acc += x;
    // 2. dependent rsqrt chain
    x = seed + 2.0; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) x = rsqrt(x) + 1.0;
    t1 = clock64(); if (tid == 0) clk[1] = (t1 - t0) / 32; acc += x;
    // 3. dependent sqrt chain
    x = seed + 2.0; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) x = sqrt(x) + 1.0;
    t1 = clock64(); if (tid == 0) clk[2] = (t1 - t0) / 32; acc += x;
    // 4. dependent division chain
    x = seed + 2.0; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) x = 3.0 / x + 1.0;
    t1 = clock64(); if (tid == 0) clk[3] = (t1 - t0) / 32; acc += x;
    // 5. dependent DMMA chain
    double c0 = 0, c1 = 0; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) dmma(c0, c1, x, y);
    t1 = clock64(); if (tid == 0) clk[4] = (t1 - t0) / 32; acc += c0 + c1;
    // 6. 4 independent DMMA chains (throughput per warp)
    double d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) { dmma(c0, c1, x, y); dmma(d0, d1, x, y); dmma(e0, e1, x, y); dmma(f0, f1, x, y); }
    t1 = clock64(); if (tid == 0) clk[5] = (t1 - t0) / 128; acc += c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1;
    // 7. __syncthreads round
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) __syncthreads();
    t1 = clock64(); if (tid == 0) clk[6] = (t1 - t0) / 32;
    // 8. smem store -> sync -> load round trip
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) { sm[tid] = x; __syncthreads(); x = sm[(tid + 1) % blockDim.x] + 1.0; __syncthreads(); }
    t1 = clock64(); if (tid == 0) clk[7] = (t1 - t0) / 32; acc += x;
    // 9. dependent LDS chain (pointer chase)
    int idx = tid; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 32; ++i) idx = (int)sm[idx & 1023] & 1023;
    t1 = clock64(); if (tid == 0) clk[8] = (t1 - t0) / 32; acc += idx;
    // 10. DFMA throughput: 8 independent chains per thread
    double a[8]; for (int i = 0; i < 8; ++i) a[i] = seed + i; t0 = clock64();
#pragma unroll
    for (int i = 0; i < 64; ++i) { for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 1.0000001, y); }
    t1 = clock64(); if (tid == 0) clk[9] = (t1 - t0); for (int j = 0; j < 8; ++j) acc += a[j];
    out[tid] = acc;
}
__global__ void gl(const double* __restrict__ src, const int* __restrict__ chase, long long* clk, double* out, int n) {
    // global pointer chase (L2 hit latency) after a warm-up pass
    int idx = threadIdx.x; double acc = 0;
    for (int i = 0; i < 64; ++i) idx = chase[idx];
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) idx = chase[idx];
    long long t1 = clock64(); if (threadIdx.x == 0) clk[10] = (t1 - t0) / 64;
    out[threadIdx.x] = acc + idx + src[idx % n];
}
int main() {
    double* out; long long* clk; cudaMalloc(&out, 8192); cudaMalloc(&clk, 256); cudaMemset(clk, 0, 256);
    for (int threads : {32, 256}) {
        k<<<1, threads>>>(out, clk, 1.0); cudaDeviceSynchronize();
        long long h[16]; cudaMemcpy(h, clk, 128, cudaMemcpyDeviceToHost);
        printf("threads=%d  dfma_lat=%lld rsqrt_chain=%lld sqrt_chain=%lld div_chain=%lld dmma_lat=%lld dmma_4chains_per_mma=%lld sync=%lld sts_sync_lds_sync=%lld lds_chain=%lld dfma_512_total=%lld\n",
               threads, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
    }
    int n = 1 << 20; int* chase; double* src; cudaMalloc(&chase, n * 4); cudaMalloc(&src, n * 8); cudaMemset(src, 0, n * 8);
    int* hc = new int[n]; for (int i = 0; i < n; ++i) hc[i] = (int)(((long long)i * 7919 + 12345) % n); cudaMemcpy(chase, hc, n * 4, cudaMemcpyHostToDevice);
    gl<<<1, 32>>>(src, chase, clk, out, n); cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, clk, 128, cudaMemcpyDeviceToHost);
    printf("global dependent load (L2) latency = %lld cycles\n", h[10]);
    // empty-kernel launch latency in a graph: 100 dependent tiny kernels
    cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 100; ++i) gl<<<1, 32, 0, s>>>(src, chase, clk, out, n);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaStreamSynchronize(s);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of 100 dependent small kernels (each 128 dependent L2 loads): %.2f us per kernel\n", ms * 10);
    return 0;
}
