// DMMA m8n8k4 throughput vs warps per SM and independent accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dmma_ilp(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[CH][2];
#pragma unroll
    for (int t = 0; t < CH; ++t) c[t][0] = c[t][1] = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < CH; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int warps_per_sm, int sms, double* out) {
    const int threads = 128, blocks = sms * warps_per_sm / 4, iters = 2048;
    dmma_ilp<CH><<<blocks, threads>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_ilp<CH><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 512.0 * CH * iters * double(blocks) * (threads / 32);
    printf("warps/SM %3d chains/warp %2d: %.2f TFLOP/s\n", warps_per_sm, CH, flops / ms / 1e9);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * 148 * 64 * 32 * 4);
    for (int w : {4, 8, 16, 24, 32, 64}) { run<4>(w, sms, out); run<16>(w, sms, out); }
    return 0;
}
