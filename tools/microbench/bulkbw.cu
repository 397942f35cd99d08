// cp.async.bulk (1-D TMA) global -> shared bandwidth per SM: one thread issues COPY-byte copies into
// a STAGES-deep ring, consumed (released) immediately; source = a buffer of SRC bytes read cyclically
// (HBM-resident when large, L2-resident when small). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__global__ void k(const uint8_t* src, size_t srcbytes, int copy, int stages, int iters, int* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16];
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        size_t off = (size_t(blockIdx.x) * 7919 * copy) % srcbytes;
        for (int i = 0; i < iters + stages; ++i) {
            const int st = i % stages;
            if (i >= stages) {  // wait for the copy issued into this stage
                const uint32_t ph = ((i / stages) - 1) & 1;
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(&full[st])), "r"(ph));
            }
            if (i < iters) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])), "r"(copy));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + size_t(st) * copy)), "l"(src + off), "r"(copy), "r"(su32(&full[st])) : "memory");
                off += copy;
                if (off + copy > srcbytes) off = 0;
            }
        }
        if (sm[5] == 123) sink[0] = 1;
    }
}
int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* big;
    int* sink;
    const size_t BIG = size_t(4) << 30;
    cudaMalloc(&big, BIG);
    cudaMemset(big, 1, BIG);
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct C { size_t src; int copy, stages; };
    C cs[] = {{BIG, 16384, 4}, {BIG, 16384, 8}, {BIG, 16384, 12}, {BIG, 8192, 16}, {BIG, 32768, 6}, {64 << 20, 16384, 4}, {64 << 20, 16384, 8}, {64 << 20, 16384, 12}};
    for (C c : cs) {
        const int iters = 2000;
        k<<<nsm, 32, size_t(c.copy) * c.stages>>>(big, c.src, c.copy, c.stages, 50, sink);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<nsm, 32, size_t(c.copy) * c.stages>>>(big, c.src, c.copy, c.stages, iters, sink);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(nsm) * iters * c.copy;
        printf("src %5zu MB copy %5d stages %2d: %.2f TB/s total, %.1f B/clk/SM  %s\n", c.src >> 20, c.copy, c.stages, bytes / (ms * 1e-3) / 1e12, bytes / nsm / (ms * 1e-3 * 1.965e9), cudaGetErrorString(cudaGetLastError()));
    }
}
