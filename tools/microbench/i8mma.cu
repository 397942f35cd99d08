// tcgen05.mma kind::i8 bring-up and throughput probe (B200, sm_100a).
//   correctness: C[128 x N] (int32) = A[128 x 128] * B[N x 128]^T, both int8, K-major, 128-byte
//   swizzled smem images (the layout the Ozaki GEMM uses), one CTA, compared with a host product.
//   throughput: one CTA per SM issues R back-to-back MMAs (operands resident in smem) into TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8mma i8mma.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// smem matrix descriptor, K-major, SWIZZLE_128B: start>>4, LBO (ignored) = 1, SBO = 1024 B between 8-row atoms,
// version 1 (sm_100), layout type 2 (128B swizzle)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t(1) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// instruction descriptor: kind::i8, D = s32, A = B = signed int8 (or unsigned), K-major both, N, M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int N, int asig, int bsig) {
    return (2u << 4) | (uint32_t(asig) << 7) | (uint32_t(bsig) << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                 ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}

// swizzled K-major image: row r (of R), 16-byte chunk c -> (r/8)*1024 + (r%8)*128 + ((c ^ (r%8)) * 16)
__host__ __device__ inline size_t swz(int r, int kbyte) {
    const int c = kbyte >> 4, o = kbyte & 15;
    return size_t(r >> 3) * 1024 + size_t(r & 7) * 128 + size_t(((c ^ (r & 7)) << 4) | o);
}

template <int N>
__global__ void __launch_bounds__(128, 1) k_check(const int8_t* A, const int8_t* B, int32_t* C, int unsig) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;            // 16 KB
    uint8_t* sB = sm + 16384;    // N * 128 B
    for (int i = threadIdx.x; i < 16384 / 16; i += 128) reinterpret_cast<int4*>(sA)[i] = reinterpret_cast<const int4*>(A)[i];
    for (int i = threadIdx.x; i < N * 128 / 16; i += 128) reinterpret_cast<int4*>(sB)[i] = reinterpret_cast<const int4*>(B)[i];
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(N, unsig ? 0 : 1, unsig ? 0 : 1);
        for (int k = 0; k < 4; ++k)
            mma_i8(tm, sdesc(su32(sA) + 32 * k), sdesc(su32(sB) + 32 * k), id, k > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = w * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + (uint32_t(w * 32) << 16) + uint32_t(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = int32_t(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// throughput: R rounds of 4 MMAs (K = 128) into NACC accumulators of N columns, operands resident
template <int N>
__global__ void __launch_bounds__(128, 1) k_rate(int R, int nacc, int32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(N, 1, 1);
        for (int r = 0; r < R; ++r)
            for (int k = 0; k < 4; ++k)
                mma_i8(tm + uint32_t((r % nacc) * N), sdesc(su32(sA) + 32 * k), sdesc(su32(sB) + 32 * k), id, 1);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = int32_t(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// hoisted descriptors, 8 MMAs per iteration cycling 2 accumulators; TC TMEM columns per CTA (2 CTAs/SM with 256)
template <int N, int TC>
__global__ void __launch_bounds__(128) k_rate2(int R, int32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "n"(TC));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(N, 1, 1);
        const uint64_t a0 = sdesc(su32(sA)), b0 = sdesc(su32(sB));
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                mma_i8(tm + uint32_t((k >> 2) * N), a0 + 2 * (k & 3), b0 + 2 * (k & 3), id, 1);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = int32_t(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(TC));
}

template <int N, int TC>
void rate2(int cps) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int smem = 16384 + N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_rate2<N, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 2048;
    k_rate2<N, TC><<<nsm * cps, 128, smem>>>(32, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate2<N, TC><<<nsm * cps, 128, smem>>>(R, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = double(nsm) * cps * R * 8 * 128.0 * N * 32.0;
    printf("rate2 N=%3d ctas/SM=%d: %.3f ms, %.1f TOPS, %.0f clk/MMA per SM\n", N, cps, ms, 2 * macs / (ms * 1e-3) / 1e12,
           ms * 1e-3 * 1.965e9 / (R * 8.0 * cps));
    cudaFree(sink);
}

// TMEM read throughput: W warps each issue R tcgen05.ld 32x32b.xX (+ wait) over the 512 allocated columns
template <int X>
__global__ void k_ldtm(int R, int32_t* sink) {
    __shared__ uint32_t tbase;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase + (uint32_t(((threadIdx.x >> 5) & 3) * 32) << 16);
    uint32_t acc = 0;
    for (int r = 0; r < R; ++r) {
        const uint32_t col = uint32_t((r * X + (threadIdx.x >> 7) * 64) & 511);
        if (X == 16) {
            uint32_t v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(tm + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int j = 0; j < 16; ++j) acc += v[j];
        } else {
            uint32_t v[32];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                         "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                           "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                           "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                         : "r"(tm + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int j = 0; j < 32; ++j) acc += v[j];
        }
    }
    if (acc == 0x12345678u) sink[0] = int32_t(acc);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int X>
void ldtm(int warps) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int R = 4096;
    k_ldtm<X><<<nsm, 32 * warps>>>(16, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_ldtm<X><<<nsm, 32 * warps>>>(R, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(R) * warps * 32 * X * 4;  // per SM
    printf("ldtm x%d warps=%2d: %.1f B/clk per SM\n", X, warps, bytes / (ms * 1e-3 * 1.965e9));
    cudaFree(sink);
}

// I2F.F64 vs magic-number int32 -> fp64 conversion throughput (per SM, 8 warps)
__global__ void k_cvt(int R, int mode, double* sink) {
    int x = threadIdx.x * 7919;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int r = 0; r < R; ++r) {
        x = x * 1664525 + 1013904223;
        const int y = x ^ 0x5bd1e995, z = x + 12345, w = x >> 3;
        if (mode == 0) {
            a0 += double(x); a1 += double(y); a2 += double(z); a3 += double(w);
        } else {
            a0 += __hiloint2double(0x43380000 + (x >> 31), x) - 6755399441055744.0;
            a1 += __hiloint2double(0x43380000 + (y >> 31), y) - 6755399441055744.0;
            a2 += __hiloint2double(0x43380000 + (z >> 31), z) - 6755399441055744.0;
            a3 += __hiloint2double(0x43380000 + (w >> 31), w) - 6755399441055744.0;
        }
    }
    if (a0 + a1 + a2 + a3 == 1.2345) sink[0] = a0;
}
void cvt(int mode) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double* sink;
    CK(cudaMalloc(&sink, 8));
    const int R = 1 << 16;
    k_cvt<<<nsm, 256>>>(64, mode, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_cvt<<<nsm, 256>>>(R, mode, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cvt %s: %.1f conversions+adds /clk per SM\n", mode ? "magic" : "I2F.F64", 4.0 * R * 256 / (ms * 1e-3 * 1.965e9));
    cudaFree(sink);
}

// Ozaki pattern: 6 A slices x 6 B slices resident, digit-major pairs d + d' <= 6 into 7 accumulators
template <int N, int ORDER>
__global__ void __launch_bounds__(128, 1) k_rate3(int R, int32_t* sink, int sg) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, bar2[4];
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 6 * 16384;
    for (int i = threadIdx.x; i < (6 * 16384 + 6 * N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a0 = su32(sA), b0 = su32(sB);
        for (int r = 0; r < R; ++r) {
            if (ORDER == 2) {  // level-major with a commit after every level (the GEMM's accfull pattern)
                for (int L = 0; L < 7; ++L) {
                    for (int d = (L > 5 ? L - 5 : 0); d <= L && d < 6; ++d)
                        for (int k = 0; k < 4; ++k)
                            mma_i8(tm + uint32_t((L % 4) * N), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + (L - d) * N * 128) + 2 * k,
                                   idesc_i8(N, 1, 1), 1);
                    commit(&bar2[L % 4]);
                }
            } else if (ORDER == 3) {  // level-major, no commits
                for (int L = 0; L < 7; ++L)
                    for (int d = (L > 5 ? L - 5 : 0); d <= L && d < 6; ++d)
                        for (int k = 0; k < 4; ++k)
                            mma_i8(tm + uint32_t((L % 4) * N), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + (L - d) * N * 128) + 2 * k,
                                   idesc_i8(N, 1, 1), 1);
            } else if (ORDER == 0) {  // digit-major, k inner
                for (int d = 0; d < 6; ++d)
                    for (int dp = 0; dp <= (6 - d < 5 ? 6 - d : 5); ++dp)
                        for (int k = 0; k < 4; ++k)
                            mma_i8(tm + uint32_t(((d + dp) % (512 / N)) * N), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + dp * N * 128) + 2 * k,
                                   sg == 0 ? idesc_i8(N, 1, 1) : sg == 1 ? idesc_i8(N, 0, 0) : idesc_i8(N, d == 0, dp == 0), 1);
            } else {  // k outer: consecutive MMAs go to different accumulators
                for (int d = 0; d < 6; ++d)
                    for (int k = 0; k < 4; ++k)
                        for (int dp = 0; dp <= (6 - d < 5 ? 6 - d : 5); ++dp)
                            mma_i8(tm + uint32_t(((d + dp) % (512 / N)) * N), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + dp * N * 128) + 2 * k, idesc_i8(N, 1, 1), 1);
            }
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = int32_t(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
template <int N>
__global__ void __launch_bounds__(128, 1) k_rate4(int R, int32_t* sink, const uint8_t* big, size_t bigsz, int ncopy) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, cb[4];
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 6 * 16384;
    uint8_t* sC = sB + 6 * N * 128;  // 4 x 16 KB copy ring
    for (int i = threadIdx.x; i < (6 * 16384 + 6 * N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a0 = su32(sA), b0 = su32(sB);
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < 6; ++d)
                for (int dp = 0; dp <= (6 - d < 5 ? 6 - d : 5); ++dp)
                    for (int k = 0; k < 4; ++k)
                        mma_i8(tm + uint32_t(((d + dp) % (512 / N)) * N), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + dp * N * 128) + 2 * k, idesc_i8(N, 1, 1), 1);
        commit(&bar);
    } else if (threadIdx.x == 32 && ncopy) {  // concurrent TMA stream
        size_t off = (size_t(blockIdx.x) * 7919 * 16384) % bigsz;
        for (int i = 0; i < ncopy + 2; ++i) {
            const int st = i & 1;
            if (i >= 2) mbar_wait(&cb[st], ((i >> 1) - 1) & 1);
            if (i < ncopy) {
                mbar_expect(&cb[st], 16384);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sC + st * 16384)), "l"(big + off), "r"(16384), "r"(su32(&cb[st])) : "memory");
                off += 16384;
                if (off + 16384 > bigsz) off = 0;
            }
        }
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = int32_t(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int N>
void rate4(int ncopy) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    uint8_t* big;
    const size_t BIG = size_t(2) << 30;
    CK(cudaMalloc(&big, BIG));
    CK(cudaMemset(big, 1, BIG));
    const int smem = 6 * 16384 + 6 * N * 128 + 2 * 16384 + 1024;
    CK(cudaFuncSetAttribute(k_rate4<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 200;
    k_rate4<N><<<nsm, 128, smem>>>(4, sink, big, BIG, 0);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate4<N><<<nsm, 128, smem>>>(R, sink, big, BIG, ncopy);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double nmma = double(R) * 26 * 4;
    printf("rate4 N=%3d copies=%d (%.0f GB/s per SM): %.0f clk/MMA\n", N, ncopy, ncopy * 16384.0 / (ms * 1e-3) / 1e9,
           ms * 1e-3 * 1.965e9 / nmma);
    cudaFree(sink);
    cudaFree(big);
}

// latency from issuing NM MMAs (M=128, N=128, K=32 each) + commit to the mbarrier completing, as seen by the issuing
// thread (wait) - per level of the Ozaki GEMM
__global__ void __launch_bounds__(128, 1) k_lat(int nm, int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < (2 * 16384) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int r = 0; r < reps; ++r) {
            unsigned long long t0, t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (int i = 0; i < nm; ++i)
                mma_i8(tm + uint32_t((r & 3) * 128), sdesc(su32(sm)) + 2 * (i & 3), sdesc(su32(sm) + 16384) + 2 * (i & 3), idesc_i8(128, 1, 1), i > 0);
            commit(&bar);
            mbar_wait(&bar, r & 1);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            tot += t1 - t0;
        }
        if (blockIdx.x == 0) out[0] = tot / reps;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
void lat(int nm, int grid) {
    unsigned long long* d;
    CK(cudaMalloc(&d, 8));
    CK(cudaFuncSetAttribute(k_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024));
    k_lat<<<grid, 128, 33 * 1024>>>(nm, 50, d);
    CK(cudaDeviceSynchronize());
    unsigned long long h;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("lat: %3d MMAs + commit + wait: %llu ns (grid %d)\n", nm, h, grid);
    cudaFree(d);
}

// MMA rate (N = 128, digit-major pattern, 3 accumulators at columns 0..383) while warps 4.. stream
// tcgen05.ld over columns 384..511 (the epilogue's TMEM reads)
__global__ void __launch_bounds__(384, 1) k_rate5(int R, int nld, int32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ volatile int done;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 6 * 16384;
    for (int i = threadIdx.x; i < (12 * 16384) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); done = 0; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        const uint32_t a0 = su32(sA), b0 = su32(sB);
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < 6; ++d)
                for (int dp = 0; dp <= (6 - d < 5 ? 6 - d : 5); ++dp)
                    for (int k = 0; k < 4; ++k)
                        mma_i8(tm + uint32_t(((d + dp) % 3) * 128), sdesc(a0 + d * 16384) + 2 * k, sdesc(b0 + dp * 16384) + 2 * k, idesc_i8(128, 1, 1), 1);
        commit(&bar);
        mbar_wait(&bar, 0);
        done = 1;
    } else if (warp >= 4 && nld == 2) {  // FP64 load: the epilogue's DADD + DFMA stream
        double a0 = threadIdx.x, a1 = 1.0, a2 = 2.0, a3 = 3.0, x = 1.0 + 1e-9 * threadIdx.x;
        while (!done) {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                a0 = fma(a0, x, 1e-7); a1 = fma(a1, x, 2e-7); a2 = a2 + x; a3 = fma(a3, x, a2);
            }
        }
        if (a0 + a1 + a2 + a3 == 1.2345) sink[0] = 1;
    } else if (warp >= 4 && nld) {
        const uint32_t tq = tm + (uint32_t((warp & 3) * 32) << 16) + 384;
        uint32_t acc = 0;
        while (!done) {
            uint32_t v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(tq + uint32_t((acc & 7) * 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int j = 0; j < 16; ++j) acc += v[j];
        }
        if (acc == 0x12345678u) sink[0] = int32_t(acc);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
void rate5(int nld) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int smem = 12 * 16384 + 1024;
    CK(cudaFuncSetAttribute(k_rate5, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 200;
    k_rate5<<<nsm, 384, smem>>>(4, nld, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate5<<<nsm, 384, smem>>>(R, nld, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double nmma = double(R) * 26 * 4;
    printf("rate5 N=128 with TMEM loads %d: %.0f clk/MMA\n", nld, ms * 1e-3 * 1.965e9 / nmma);
    cudaFree(sink);
}

template <int N, int ORDER>
void rate3(int sg = 0) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int smem = 6 * 16384 + 6 * N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_rate3<N, ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 200;
    k_rate3<N, ORDER><<<nsm, 128, smem>>>(4, sink, sg);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate3<N, ORDER><<<nsm, 128, smem>>>(R, sink, sg);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double nmma = double(R) * 26 * 4;
    printf("rate3 N=%3d order=%d sign=%d: %.0f clk/MMA, %.1f TOPS\n", N, ORDER, sg, ms * 1e-3 * 1.965e9 / nmma,
           2.0 * nsm * nmma * 128 * N * 32 / (ms * 1e-3) / 1e12);
    cudaFree(sink);
}

__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(tmem_d), "r"(tmem_a), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void cp128x256(uint32_t taddr, uint64_t sd) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sd));
}
// A copied smem -> TMEM (4 x tcgen05.cp 128x256b from the swizzled K-major image), TS products
template <int N>
__global__ void __launch_bounds__(128, 1) k_check_ts(const int8_t* A, const int8_t* B, int32_t* C) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    for (int i = threadIdx.x; i < 16384 / 16; i += 128) reinterpret_cast<int4*>(sA)[i] = reinterpret_cast<const int4*>(A)[i];
    for (int i = threadIdx.x; i < N * 128 / 16; i += 128) reinterpret_cast<int4*>(sB)[i] = reinterpret_cast<const int4*>(B)[i];
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t ta = tm + 256;
        for (int k = 0; k < 4; ++k) cp128x256(ta + 8 * k, sdesc(su32(sA) + 32 * k));
        const uint32_t id = idesc_i8(N, 1, 1);
        for (int k = 0; k < 4; ++k) mma_i8_ts(tm, ta + 8 * k, sdesc(su32(sB) + 32 * k), id, k > 0);
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = w * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + (uint32_t(w * 32) << 16) + uint32_t(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = int32_t(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
// TS rate: A_d copied into a 2 x 32-column TMEM buffer per digit step, B from smem, 7 accumulators of N
template <int N>
__global__ void __launch_bounds__(128, 1) k_rate_ts(int R, int32_t* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 6 * 16384;
    for (int i = threadIdx.x; i < (6 * 16384 + 6 * N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a0 = su32(sA), b0 = su32(sB);
        const uint32_t id = idesc_i8(N, 1, 1);
        int s = 0;
        for (int r = 0; r < R; ++r)
            for (int d = 0; d < 6; ++d, ++s) {
                const uint32_t ta = tm + 448 + uint32_t((s & 1) * 32);
                for (int k = 0; k < 4; ++k) cp128x256(ta + 8 * k, sdesc(a0 + d * 16384 + 32 * k));
                for (int dp = 0; dp <= (6 - d < 5 ? 6 - d : 5); ++dp)
                    for (int k = 0; k < 4; ++k)
                        mma_i8_ts(tm + uint32_t((d + dp) * N), ta + 8 * k, sdesc(b0 + dp * N * 128) + 2 * k, id, 1);
            }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tm + (uint32_t((threadIdx.x >> 5) * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x12345678u) sink[0] = int32_t(v);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
template <int N>
void rate_ts() {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int smem = 6 * 16384 + 6 * N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_rate_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 200;
    k_rate_ts<N><<<nsm, 128, smem>>>(4, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate_ts<N><<<nsm, 128, smem>>>(R, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double nmma = double(R) * 26 * 4;
    printf("rate_ts N=%3d: %.0f clk/MMA, %.1f TOPS\n", N, ms * 1e-3 * 1.965e9 / nmma, 2.0 * nsm * nmma * 128 * N * 32 / (ms * 1e-3) / 1e12);
    cudaFree(sink);
}

// B stored MN-major: [k][n] rows of N bytes (N = 128 = one 128-byte swizzle width), 8-k-row atoms of 1 KB;
// K-step advance = 32 k-rows = 4 KB; b_major = 1 in the instruction descriptor
__global__ void __launch_bounds__(128, 1) k_check_mn(const int8_t* A, const int8_t* B, int32_t* C, uint32_t lbo) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t* sA = sm;
    uint8_t* sB = sm + 16384;
    for (int i = threadIdx.x; i < 16384 / 16; i += 128) reinterpret_cast<int4*>(sA)[i] = reinterpret_cast<const int4*>(A)[i];
    for (int i = threadIdx.x; i < 16384 / 16; i += 128) reinterpret_cast<int4*>(sB)[i] = reinterpret_cast<const int4*>(B)[i];
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(128, 1, 1) | (1u << 16);  // b_major = MN
        for (int k = 0; k < 4; ++k) {
            uint64_t bd = sdesc(su32(sB) + 4096 * k);
            bd = (bd & ~(uint64_t(0x3FFF) << 16)) | (uint64_t(lbo >> 4) << 16);
            mma_i8(tm, sdesc(su32(sA) + 32 * k), bd, id, k > 0);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = w * 32 + lane;
    for (int c0 = 0; c0 < 128; c0 += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + (uint32_t(w * 32) << 16) + uint32_t(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[row * 128 + c0 + j] = int32_t(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
bool check_mn() {
    std::vector<int8_t> a(128 * 128), b(128 * 128), sa(128 * 128), sb(128 * 128);
    srand(99);
    for (auto& x : a) x = int8_t((rand() % 255) - 127);
    for (auto& x : b) x = int8_t((rand() % 255) - 127);  // b[n * 128 + k] (logical B^T rows n)
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 128; ++k) sa[swz(r, k)] = a[r * 128 + k];
    for (int k = 0; k < 128; ++k)
        for (int n = 0; n < 128; ++n) sb[swz(k, n)] = b[n * 128 + k];  // MN-major: row = k, byte = n
    int8_t *dA, *dB;
    int32_t* dC;
    CK(cudaMalloc(&dA, a.size()));
    CK(cudaMalloc(&dB, b.size()));
    CK(cudaMalloc(&dC, 128 * 128 * 4));
    CK(cudaMemcpy(dA, sa.data(), a.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, sb.data(), b.size(), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_check_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024));
    bool any = false;
    for (uint32_t lbo : {16u, 1024u, 8192u}) {
        k_check_mn<<<1, 128, 33 * 1024>>>(dA, dB, dC, lbo);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<int32_t> c(128 * 128);
        CK(cudaMemcpy(c.data(), dC, c.size() * 4, cudaMemcpyDeviceToHost));
        long bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                long s = 0;
                for (int k = 0; k < 128; ++k) s += long(a[i * 128 + k]) * long(b[j * 128 + k]);
                bad += int32_t(s) != c[i * 128 + j];
            }
        printf("check MN-major B (lbo %u): %s (%ld bad)\n", lbo, bad ? "FAIL" : "ok", bad);
        any |= bad == 0;
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
    return any;
}

template <int N>
bool check(int unsig) {
    std::vector<int8_t> a(128 * 128), b(N * 128), sa(128 * 128), sb(N * 128);
    srand(1 + N + unsig);
    for (auto& x : a) x = int8_t(unsig ? (rand() & 255) : (rand() % 255) - 127);
    for (auto& x : b) x = int8_t(unsig ? (rand() & 255) : (rand() % 255) - 127);
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 128; ++k) sa[swz(r, k)] = a[r * 128 + k];
    for (int r = 0; r < N; ++r)
        for (int k = 0; k < 128; ++k) sb[swz(r, k)] = b[r * 128 + k];
    int8_t *dA, *dB;
    int32_t* dC;
    CK(cudaMalloc(&dA, a.size()));
    CK(cudaMalloc(&dB, b.size()));
    CK(cudaMalloc(&dC, 128 * N * 4));
    CK(cudaMemcpy(dA, sa.data(), a.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, sb.data(), b.size(), cudaMemcpyHostToDevice));
    const int smem = 16384 + N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_check<N><<<1, 128, smem>>>(dA, dB, dC, unsig);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> c(128 * N);
    CK(cudaMemcpy(c.data(), dC, c.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < 128; ++i)
        for (int j = 0; j < N; ++j) {
            long s = 0;
            for (int k = 0; k < 128; ++k)
                s += unsig ? long(uint8_t(a[i * 128 + k])) * long(uint8_t(b[j * 128 + k])) : long(a[i * 128 + k]) * long(b[j * 128 + k]);
            if (int32_t(s) != c[i * N + j]) {
                if (bad < 5) printf("  mismatch (%d,%d): got %d want %ld\n", i, j, c[i * N + j], s);
                ++bad;
            }
        }
    printf("check N=%d %s: %s (%ld bad)\n", N, unsig ? "u8" : "s8", bad ? "FAIL" : "ok", bad);
    if (!unsig) {
        CK(cudaFuncSetAttribute(k_check_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        k_check_ts<N><<<1, 128, smem>>>(dA, dB, dC);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<int32_t> c2(128 * N);
        CK(cudaMemcpy(c2.data(), dC, c2.size() * 4, cudaMemcpyDeviceToHost));
        long bad2 = 0;
        for (size_t i = 0; i < c2.size(); ++i) bad2 += c2[i] != c[i];
        printf("check TS (A via tcgen05.cp) N=%d: %s (%ld differ from SS)\n", N, bad2 || bad ? "FAIL" : "ok", bad2);
        bad += bad2;
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dC);
    return bad == 0;
}

template <int N>
void rate(int nacc) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    int32_t* sink;
    CK(cudaMalloc(&sink, 4));
    const int smem = 16384 + N * 128 + 1024;
    CK(cudaFuncSetAttribute(k_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int R = 4096;
    k_rate<N><<<nsm, 128, smem>>>(64, nacc, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_rate<N><<<nsm, 128, smem>>>(R, nacc, sink);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = double(nsm) * R * 128.0 * N * 128.0;
    printf("rate N=%3d nacc=%d: %.3f ms, %.1f TOPS (int8, 2 ops/MAC), %.0f clk/MMA(K=32) @1.965GHz\n", N, nacc, ms,
           2 * macs / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 / (R * 4.0));
    cudaFree(sink);
}

int main() {
    check_mn();
    bool ok = check<64>(0) & check<128>(0) & check<256>(0) & check<64>(1) & check<16>(0);
    rate<64>(6);
    rate<128>(4);
    rate<256>(2);
    rate<32>(6);
    rate2<64, 512>(1);
    rate2<64, 256>(2);
    rate2<128, 512>(1);
    rate2<128, 256>(2);
    rate2<256, 512>(1);
    rate2<32, 128>(2);
    rate_ts<64>();
    rate3<64, 0>();
    rate3<64, 1>();
    rate3<128, 0>();
    lat(1, 1); lat(4, 1); lat(20, 1); lat(100, 1); lat(4, 148); lat(20, 148);
    rate5(0); rate5(1); rate5(2);
    rate4<128>(0);
    rate4<128>(200);
    rate4<128>(1000);
    rate4<128>(3000);
    rate3<128, 2>();
    rate3<128, 3>();
    rate3<128, 0>(1);
    rate3<128, 0>(2);
    rate3<128, 1>();
    ldtm<16>(4);
    ldtm<16>(8);
    ldtm<32>(4);
    ldtm<32>(8);
    ldtm<32>(16);
    cvt(0);
    cvt(1);
    return ok ? 0 : 1;
}
