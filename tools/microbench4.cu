// FP64 tensor-pipe shapes on sm_100a: cycles per mma.sync for m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 with
// NCH independent accumulator chains per warp, W warps per CTA, one or two CTAs on the SM; and the plain DFMA rate.
#include <cstdio>
#include <cuda_runtime.h>
template <int SHAPE> struct Acc { static constexpr int N = SHAPE == 0 ? 2 : 4; };
template <int SHAPE> __device__ __forceinline__ void mma(double* c, const double* a, const double* b) {
    if constexpr (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]));
    else if constexpr (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    else if constexpr (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
template <int SHAPE, int NCH>
__global__ void k(double* out, long long* clk, double av, double bv) {
    double c[NCH][4], a[8], b[4];
    for (int j = 0; j < NCH; ++j) for (int q = 0; q < 4; ++q) c[j][q] = 0.0;
    for (int q = 0; q < 8; ++q) a[q] = av + q * 1e-3 + threadIdx.x * 1e-5;
    for (int q = 0; q < 4; ++q) b[q] = bv + q * 1e-3;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i)
#pragma unroll
        for (int j = 0; j < NCH; ++j) mma<SHAPE>(c[j], a, b);
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
    double s = 0; for (int j = 0; j < NCH; ++j) for (int q = 0; q < 4; ++q) s += c[j][q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NCH>
__global__ void kf(double* out, long long* clk, double av, double bv) {
    double y[NCH]; for (int j = 0; j < NCH; ++j) y[j] = av + j + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i)
#pragma unroll
        for (int j = 0; j < NCH; ++j) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(y[j]) : "d"(av), "d"(bv));
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
    double s = 0; for (int j = 0; j < NCH; ++j) s += y[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SHAPE, int NCH> void run(const char* name, double flops, double* out, long long* clk) {
    for (int threads : {32, 128, 256, 512}) {
        k<SHAPE, NCH><<<1, threads>>>(out, clk, 1.0000001, 0.5); cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
        const double per = (double)h / (64.0 * NCH);                 // cycles per MMA of one warp
        const double sm = per / (threads / 32);                      // cycles per MMA, SM-wide
        printf("%-9s chains=%d warps=%2d: %7.1f cycles per MMA per warp, %6.2f cycles per MMA on the SM -> %6.1f flop/clk/SM\n",
               name, NCH, threads / 32, per, sm, flops / sm);
    }
}
int main() {
    double* out; long long* clk; cudaMalloc(&out, 1 << 20); cudaMalloc(&clk, 256);
    run<0, 1>("m8n8k4", 512, out, clk);   run<0, 4>("m8n8k4", 512, out, clk);
    run<1, 1>("m16n8k4", 1024, out, clk); run<1, 4>("m16n8k4", 1024, out, clk);
    run<2, 1>("m16n8k8", 2048, out, clk); run<2, 4>("m16n8k8", 2048, out, clk);
    run<3, 1>("m16n8k16", 4096, out, clk); run<3, 4>("m16n8k16", 4096, out, clk);
    for (int threads : {32, 128, 256, 512}) {
        kf<8><<<1, threads>>>(out, clk, 1.0000001, 0.5); cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
        const double per = (double)h / (64.0 * 8), sm = per / (threads / 32);
        printf("dfma      chains=8 warps=%2d: %7.1f cycles per warp FMA, %6.2f on the SM -> %6.1f flop/clk/SM\n", threads / 32, per, sm, 64.0 / sm);
    }
    return 0;
}
