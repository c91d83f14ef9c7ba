// Probe: B200 fp64 throughput, vector DFMA vs DMMA (mma.sync m8n8k4 f64), all SMs.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__global__ void dfma_kernel(double *out, double s) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, 1e-7);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r += a[i];
    if (r == 12345.0) out[threadIdx.x] = r;
}
__global__ void dmma_kernel(double *out, double s) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = s;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += acc[i][0] + acc[i][1];
    if (r == 12345.0) out[threadIdx.x] = r;
}
int main() {
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out;
    cudaMalloc(&out, 4096 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        for (int rep = 0; rep < 2; ++rep) {
            const int grid = sms * (threads == 1024 ? 1 : 2048 / threads);
            cudaEventRecord(e0);
            dfma_kernel<<<grid, threads>>>(out, 0.999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fmas = (double)grid * threads * ITERS * 16;
            if (rep) printf("DFMA  threads %4d grid %d: %.2f ms, %.1f TFLOP/s (FMA=2), %.1f FMA/clk/SM at %d MHz\n", threads, grid, ms,
                            2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
            cudaEventRecord(e0);
            dmma_kernel<<<grid, threads>>>(out, 0.999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double mfmas = (double)grid * (threads / 32) * ITERS * 8 * 256;
            if (rep) printf("DMMA  threads %4d grid %d: %.2f ms, %.1f TFLOP/s (FMA=2), %.1f FMA/clk/SM\n", threads, grid, ms,
                            2 * mfmas / ms / 1e9, mfmas / (ms * 1e-3) / sms / (clk * 1e3));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
