// Ceiling of the GEMM inner loop: DMMA m8n8k4 fed by the same shared-memory fragment loads as
// dgemm_pipe_kernel (CTA 128 x 64 / 8 warps of 32 x 32, padded pitches 20 / 68), no global loads and
// no barriers, 2 CTAs per SM. Variants: warp tile 32 x 32 (8 LDS per 16 DMMA) and 32 x 64
// (12 LDS per 32 DMMA), plus a "barrier per 16-deep k-slice" variant of the 32 x 32 loop.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int PSA = 20, PSB = 68;

template <int WN, bool SYNC>  // warp tile 32 x WN
__global__ void __launch_bounds__(256, 2) loop(double* out, int iters) {
    __shared__ double as[128 * PSA];
    __shared__ double bs[16 * PSB];
    for (int i = threadIdx.x; i < 128 * PSA; i += 256) as[i] = 1e-3 * (i % 97);
    for (int i = threadIdx.x; i < 16 * PSB; i += 256) bs[i] = 1e-3 * (i % 89);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWN = 64 / WN;  // warps along n
    const int wm = (warp / NWN) * 32 % 128, wn = (warp % NWN) * WN;
    const int gq = lane >> 2, tq = lane & 3;
    double acc[4][WN / 8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 16; ks += 4) {
            double af[4], bf[WN / 8];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(wm + 8 * i + gq) * PSA + ks + tq];
#pragma unroll
            for (int j = 0; j < WN / 8; ++j) bf[j] = bs[(ks + tq) * PSB + wn + 8 * j + gq];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < WN / 8; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (SYNC) __syncthreads();
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < WN / 8; ++j) s += acc[i][j][0] + acc[i][j][1];
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

// the same loop with the pipelined kernel's operand stream: per 16-deep slice every thread issues
// 4 + 2 cp.async of 16 bytes (A 128 x 16, B 16 x 64 doubles) from an L2-resident buffer into a
// 3-stage ring, then wait_group 1 + barrier, exactly as dgemm_pipe_kernel's main loop
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 16;" ::"r"(d), "l"(src) : "memory");
}
__global__ void __launch_bounds__(256, 2) loop_cp(double* out, const double* __restrict__ src, int iters) {
    extern __shared__ __align__(16) double sm[];
    double* As = sm;                    // 3 x 128 x 20
    double* Bs = sm + 3 * 128 * PSA;    // 3 x 16 x 68
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    auto issue = [&](int it) {
        const int st = it % 3;
        const double* A = src + (size_t(blockIdx.x) * 64 + (it & 63)) * 4096;  // 32 KB window per slice
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = tid + q * 256, row = c >> 3, kc = (c & 7) * 2;
            cp16(As + st * 128 * PSA + row * PSA + kc, A + row * 16 + kc);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int c = tid + q * 256, row = c >> 5, cc = (c & 31) * 2;
            cp16(Bs + st * 16 * PSB + row * PSB + cc, A + 2048 + row * 64 + cc);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    issue(1);
    double acc[4][4][2] = {};
    for (int it = 0; it < iters; ++it) {
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        issue(it + 2);
        const double* as = As + (it % 3) * 128 * PSA;
        const double* bs = Bs + (it % 3) * 16 * PSB;
#pragma unroll
        for (int ks = 0; ks < 16; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(wm + 8 * i + gq) * PSA + ks + tq];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[(ks + tq) * PSB + wn + 8 * j + gq];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    double s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j][0] + acc[i][j][1];
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int WN, bool SYNC>
void run(const char* name, int sms, double* out) {
    const int blocks = 2 * sms, iters = 4096;
    loop<WN, SYNC><<<blocks, 256>>>(out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    loop<WN, SYNC><<<blocks, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per_iter = 4.0 * 4 * (WN / 8) * 512.0 * 8;  // flops per CTA iteration (8 warps)
    printf("%-44s %.2f TFLOP/s\n", name, per_iter * iters * blocks / ms / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * 2 * sms * 256);
    run<32, false>("warp 32x32, LDS + DMMA, no barrier", sms, out);
    run<32, true>("warp 32x32, LDS + DMMA, barrier per k-slice", sms, out);
    run<64, false>("warp 32x64 (4 warps/CTA tile rows x2), no barrier", sms, out);
    {
        const int blocks = 2 * sms, iters = 4096;
        const size_t smem = (3 * 128 * PSA + 3 * 16 * PSB) * sizeof(double);
        double* src;
        cudaMalloc(&src, sizeof(double) * (size_t(blocks) * 64 + 64) * 4096);  // 512 MB: HBM-resident windows
        cudaMemset(src, 0, sizeof(double) * (size_t(blocks) * 64 + 64) * 4096);
        cudaFuncSetAttribute(loop_cp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        loop_cp<<<blocks, 256, smem>>>(out, src, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        loop_cp<<<blocks, 256, smem>>>(out, src, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %.2f TFLOP/s\n", "warp 32x32 + cp.async 3-stage ring (HBM src)", 4.0 * 4 * 4 * 512.0 * 8 * iters * blocks / ms / 1e9);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
