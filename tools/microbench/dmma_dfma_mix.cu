// Can the FP64 tensor (DMMA) and FP64 CUDA-core (DFMA) pipes run concurrently on B200?
// Warps 0..nd-1 of each CTA run DMMA chains, the rest DFMA chains; report combined TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix(double* out, int iters, int nd_warps) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if (warp < nd_warps) {
        double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
        double c[8][2];
#pragma unroll
        for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
    } else {
        double x[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) x[t] = threadIdx.x * 1e-3 + t;
        // 8 DMMA (512 flop each per warp) per iteration ~ match flops: DFMA per warp instr = 64 flop
        for (int i = 0; i < iters * 4; ++i) {
#pragma unroll
            for (int t = 0; t < 16; ++t) x[t] = fma(x[t], 1.0000001, 1e-9);
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) s += x[t];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
    const int threads = 512, blocks = sms * 2, iters = 2048;  // 32 warps / SM
    for (int nd : {16, 12, 8, 4, 0}) {
        mix<<<blocks, threads>>>(out, 16, nd);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        mix<<<blocks, threads>>>(out, iters, nd);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double dmma = 512.0 * 8 * iters * double(blocks) * nd;
        const double dfma = 64.0 * 16 * iters * 4 * double(blocks) * (16 - nd);
        printf("DMMA warps %2d / DFMA warps %2d per CTA: %.2f ms, DMMA %.1f + DFMA %.1f = %.1f TFLOP/s\n", nd, 16 - nd, ms,
               dmma / ms / 1e9, dfma / ms / 1e9, (dmma + dfma) / ms / 1e9);
    }
    return 0;
}
