// L2 / DRAM dependent-load latency and effective SM clock on the box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fill(int* chase, int n, int stride) { int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) chase[i] = (i + stride) % n; }
__global__ void chase_k(const int* __restrict__ chase, long long* out, int hops, int use_ldg) {
    int idx = threadIdx.x * 97;
    unsigned long long g0, g1; long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    t0 = clock64();
    for (int i = 0; i < hops; ++i) idx = use_ldg ? __ldg(chase + idx) : chase[idx];
    t1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / hops; out[1] = (long long)(g1 - g0); out[2] = t1 - t0; out[3] = idx; }
}
__global__ void mlp_k(const double* __restrict__ src, long long* out, int n, int stride) {
    // 16 independent loads per lane, one warp: time until all arrive
    double v[16]; long long t0 = clock64();
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = __ldg(src + ((size_t)(threadIdx.x + 32 * q) * stride) % n);
    double s = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s += v[q];
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[4] = t1 - t0; out[5] = (long long)s; }
}
int main() {
    long long* out; cudaMalloc(&out, 256); long long h[8];
    for (int mb : {1, 16, 64, 512}) {
        int n = mb * 1024 * 1024 / 4; int* chase; cudaMalloc(&chase, (size_t)n * 4);
        fill<<<(n + 255) / 256, 256>>>(chase, n, 4099 * 33);   // jumps > 128 B lines, written by a kernel (stays in L2 if it fits)
        cudaDeviceSynchronize();
        for (int ldg : {0, 1}) {
            chase_k<<<1, 32>>>(chase, out, 2000, ldg); cudaDeviceSynchronize();
            cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
            printf("buffer %4d MB ldg=%d: %lld cycles/hop, clock %.0f MHz\n", mb, ldg, h[0], h[2] * 1000.0 / h[1]);
        }
        cudaFree(chase);
    }
    int n = 8 * 1024 * 1024; double* src; cudaMalloc(&src, (size_t)n * 8); cudaMemset(src, 0, (size_t)n * 8);
    mlp_k<<<1, 32>>>(src, out, n, 1); cudaDeviceSynchronize();   // warm
    for (int stride : {1, 17, 4099}) { mlp_k<<<1, 32>>>(src, out, n, stride); cudaDeviceSynchronize(); cudaMemcpy(h, out, 64, cudaMemcpyDeviceToHost);
        printf("16 independent warp loads, stride %d: %lld cycles until all arrive\n", stride, h[4]); }
    return 0;
}
