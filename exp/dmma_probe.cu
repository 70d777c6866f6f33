// DMMA (mma.sync m8n8k4 f64) throughput probe on B200 vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dmma(int iters, double seed, double* out) {
    double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
    double c[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) { c[k][0] = k; c[k][1] = -k; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}
__global__ void k_dfma(int iters, double seed, double* out) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = seed + 1e-3 * (threadIdx.x + k);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999999999, 1e-9);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[threadIdx.x] = s;
}
int main() {
    double* d; cudaMalloc(&d, 1024 * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 2048, blocks = sms * 2, threads = warps * 32 / 2;
        float best = 1e9, bestf = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); k_dmma<<<blocks, threads>>>(iters, 1.0, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = ms < best ? ms : best;
            cudaEventRecord(e0); k_dfma<<<blocks, threads>>>(iters, 1.0, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1); if (r) bestf = ms < bestf ? ms : bestf;
        }
        const double nw = double(blocks) * threads / 32;
        const double fl_mma = nw * iters * 8 * 512.0;        // 8x8x4 x 2 flops per mma per warp
        const double fl_fma = double(blocks) * threads * iters * 8 * 2.0;
        printf("warps/SM %2d: DMMA %.1f TFLOP/s   DFMA %.1f TFLOP/s\n", warps, fl_mma / best / 1e9, fl_fma / bestf / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
