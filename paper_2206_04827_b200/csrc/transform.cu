// CCF value <-> coefficient transforms (reference: proj/src/transform.cpp:81-203).
//
// Chebyshev directions: dense FP64 contractions on the tensor cores (DMMA
// m8n8k4, mma.sync .f64) through one batched GEMM kernel; the r-direction uses
// the parity-compressed (m/2 x m/2) synthesis / analysis matrices of each
// Fourier slot (only coefficients with (j + w + cls) even exist), evaluated on
// the r > 0 half of the doubled grid (the r < 0 half is its parity image).
// Theta direction: radix-2 FFT in shared memory fused with the pointwise
// cylindrical cross product v x omega of the nonlinear term
// (proj/src/ptns.cpp:121-139): 6 half-spectra in, 3 half-spectra out per
// (r, z) point, two real signals packed per complex FFT.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ccf {

// ---------------------------------------------------------------------------------------------
// Batched DGEMM: C[b] = alpha * A[b] * B[b] + beta * C[b]   (row-major, DMMA m8n8k4)
// CTA tile 64 x 64, BK = 16, 4 warps of 32 x 32.
namespace {
constexpr int BM = 64, BN = 64, BK = 16, SA = BK + 4, SB = BN + 4;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
}  // namespace

__global__ void __launch_bounds__(128) dgemm_batched_kernel(GemmBatch g) {
    __shared__ double As[2][BM * SA];
    __shared__ double Bs[2][BK * SB];
    const int b = blockIdx.z;
    int t0 = b, t1 = b + 1;  // terms of this batch: C[b] = alpha * sum_t A[t] B[t] + beta C[b]
    if (g.tstart) {
        t0 = g.tstart[b];
        t1 = g.tstart[b + 1];
    }
    double* __restrict__ C;
    if (g.coff) {
        const long o = g.coff[b];
        C = g.cbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
    } else {
        C = g.C[b];
    }
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nkt = (g.K + BK - 1) / BK;  // k tiles per term
    double ra[8], rb[8];
    auto gload = [&](int it) {
        const int term = t0 + it / nkt, k0 = (it % nkt) * BK;
        const double* __restrict__ A;
        if (g.aoff) {
            const long o = g.aoff[term];
            A = g.bbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            A = g.A[term];
        }
        const double* __restrict__ B;
        if (g.boff) {
            const long o = g.boff[term];
            B = g.bbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            B = g.B[term];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid + q * 128;  // 0..1023
            const int ar = e >> 4, ak = e & 15;
            const int gr = m0 + ar, gk = k0 + ak;
            ra[q] = (gr < g.M && gk < g.K) ? __ldg(A + long(gr) * g.lda + gk) : 0.0;
            const int bk = e >> 6, bc = e & 63;
            const int hk = k0 + bk, hc = n0 + bc;
            rb[q] = (hk < g.K && hc < g.N) ? __ldg(B + long(hk) * g.ldb + hc) : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = tid + q * 128;
            As[buf][(e >> 4) * SA + (e & 15)] = ra[q];
            Bs[buf][(e >> 6) * SB + (e & 63)] = rb[q];
        }
    };
    const int nk = (t1 - t0) * nkt;
    if (nk > 0) {
        gload(0);
        sstore(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) gload(kt + 1);
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[buf][(wm + 8 * i + gq) * SA + ks + tq];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][(ks + tq) * SB + wn + 8 * j + gq];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (kt + 1 < nk) sstore(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int r = m0 + wm + 8 * i + gq, c = n0 + wn + 8 * j + 2 * tq + q;
                if (r < g.M && c < g.N) {
                    double* dst = C + long(r) * g.ldc + c;
                    double v = g.alpha * acc[i][j][q];
                    if (g.dl) v *= __ldg(g.dl[b] + long(r) * g.ldd + c);  // 1 / (lambda_r + mu_c), M x N table
                    *dst = g.beta == 0.0 ? v : fma(g.beta, *dst, v);
                }
            }
}

// ---------------------------------------------------------------------------------------------
// Batched DGEMM, pipelined variant: CTA tile 128 x 64 (8 warps of 32 x 32), BK = 16, 3-stage
// cp.async (LDGSTS, 16-byte, zero-filled at the M / N / K edges) straight into shared memory.
// Requires 16-byte aligned A / B bases and even lda / ldb (checked on the host: GemmPlan::upload).
namespace {
constexpr int PN = 64, PK = 16, PSTAGES = 3, PSA = PK + 4, PSB = PN + 4;
constexpr int P_B_STAGE = PK * PSB;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace

size_t dgemm_pipe_smem(int bm) { return size_t(PSTAGES) * (size_t(bm) * PSA + P_B_STAGE) * sizeof(double); }

template <int PM>
__global__ void __launch_bounds__(2 * PM, PM == 128 ? 2 : 4) dgemm_pipe_kernel(GemmBatch g) {
    constexpr int NT = 2 * PM;  // threads: (PM / 32) x 2 warps of 32 x 32
    constexpr int P_A_STAGE = PM * PSA;
    extern __shared__ __align__(16) double psm[];
    double* As = psm;
    double* Bs = psm + PSTAGES * P_A_STAGE;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    // items (batch, m-tile, n-tile) [w0, w1) per CTA (g.ipc consecutive items for single-term batches,
    // so the cp.async stream runs on across item boundaries and the per-tile fill is paid once)
    const int tn = (g.N + PN - 1) / PN, tmn = ((g.M + PM - 1) / PM) * tn;
    const int nitems = g.nbatch * tmn;
    const int w0 = blockIdx.x * g.ipc, w1 = min(nitems, w0 + g.ipc);
    const int nkt = (g.K + PK - 1) / PK;
    struct Item {
        int b, m0, n0, t0, nk;
    };
    auto decode = [&](int w) {
        Item it;
        it.b = w / tmn;
        const int rem = w - it.b * tmn;
        it.m0 = (rem / tn) * PM;
        it.n0 = (rem - (rem / tn) * tn) * PN;
        it.t0 = g.tstart ? g.tstart[it.b] : it.b;
        it.nk = (g.tstart ? g.tstart[it.b + 1] - it.t0 : 1) * nkt;
        return it;
    };
    // load cursor: item lw, k-tile lk within the item (term lt, k-tile lkt within the term)
    int lw = w0, lk = 0, lt = 0, lkt = 0, lstage = 0;
    Item LI = decode(w0);
    const double* LA = nullptr;
    const double* LB = nullptr;
    auto set_term = [&]() {
        if (g.aoff) {
            const long o = g.aoff[lt];
            LA = g.bbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            LA = g.A[lt];
        }
        if (g.boff) {
            const long o = g.boff[lt];
            LB = g.bbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            LB = g.B[lt];
        }
    };
    auto next_item = [&]() {  // advance the load cursor to the next item with work
        while (lw < w1 && lk >= LI.nk) {
            if (++lw < w1) LI = decode(lw);
            lk = 0;
            lkt = 0;
            lt = LI.t0;
            if (lw < w1 && LI.nk > 0) set_term();
        }
    };
    lt = LI.t0;
    if (LI.nk > 0) set_term();
    next_item();
    auto issue = [&]() {
        if (lw < w1) {
            const int k0 = lkt * PK, m0 = LI.m0, n0 = LI.n0;
            double* as = As + lstage * P_A_STAGE;
            double* bs = Bs + lstage * P_B_STAGE;
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // A: PM rows x 8 chunks of 2 doubles
                const int c = tid + q * NT;
                const int row = c >> 3, kc = (c & 7) * 2;
                const int gr = m0 + row, gk = k0 + kc;
                const int nv = (gr < g.M) ? max(0, min(2, g.K - gk)) : 0;
                const double* src = nv ? LA + long(gr) * g.lda + gk : LA;
                cp_async16(as + row * PSA + kc, src, nv * 8);
            }
#pragma unroll
            for (int q = 0; q < 512 / NT; ++q) {  // B: 16 rows x 32 chunks
                const int c = tid + q * NT;
                const int row = c >> 5, cc = (c & 31) * 2;
                const int gk = k0 + row, gc = n0 + cc;
                const int nv = (gk < g.K) ? max(0, min(2, g.N - gc)) : 0;
                const double* src = nv ? LB + long(gk) * g.ldb + gc : LB;
                cp_async16(bs + row * PSB + cc, src, nv * 8);
            }
            lstage = lstage + 1 == PSTAGES ? 0 : lstage + 1;
            ++lk;
            if (++lkt == nkt && lk < LI.nk) {
                lkt = 0;
                ++lt;
                set_term();
            }
            next_item();
        }
        cp_async_commit();
    };
#pragma unroll
    for (int s = 0; s < PSTAGES - 1; ++s) issue();
    int cstage = 0;
    for (int cw = w0; cw < w1; ++cw) {
        const Item I = decode(cw);
        const int b = I.b, m0 = I.m0, n0 = I.n0, nk = I.nk;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<PSTAGES - 2>();
            __syncthreads();
            issue();
            const double* as = As + cstage * P_A_STAGE;
            const double* bs = Bs + cstage * P_B_STAGE;
            cstage = cstage + 1 == PSTAGES ? 0 : cstage + 1;
#pragma unroll
            for (int ks = 0; ks < PK; ks += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) af[i] = as[(wm + 8 * i + gq) * PSA + ks + tq];
#pragma unroll
                for (int j = 0; j < 4; ++j) bf[j] = bs[(ks + tq) * PSB + wn + 8 * j + gq];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
        double* __restrict__ C;
        if (g.coff) {
            const long o = g.coff[b];
            C = g.cbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            C = g.C[b];
        }
        const double* __restrict__ dl = g.dl ? g.dl[b] : nullptr;
        // paired columns (2 tq, 2 tq + 1) go out as one 16-byte store when aligned and in range
        const bool vec = ((reinterpret_cast<uintptr_t>(C) | (uintptr_t(g.ldc) * 8)) & 15) == 0 && !dl && g.beta == 0.0;
    #pragma unroll
        for (int i = 0; i < 4; ++i)
    #pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = m0 + wm + 8 * i + gq, c = n0 + wn + 8 * j + 2 * tq;
                if (r >= g.M) continue;
                double* dst = C + long(r) * g.ldc + c;
                if (vec && c + 1 < g.N) {
                    *reinterpret_cast<double2*>(dst) = make_double2(g.alpha * acc[i][j][0], g.alpha * acc[i][j][1]);
                    continue;
                }
    #pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (c + q < g.N) {
                        double v = g.alpha * acc[i][j][q];
                        if (dl) v *= __ldg(dl + long(r) * g.ldd + c + q);
                        dst[q] = g.beta == 0.0 ? v : fma(g.beta, dst[q], v);
                    }
                }
            }
    }
    cp_async_wait<0>();
}

template __global__ void dgemm_pipe_kernel<128>(GemmBatch g);
template __global__ void dgemm_pipe_kernel<64>(GemmBatch g);

// ---------------------------------------------------------------------------------------------
// Batched DGEMM, TMA variant. Same CTA tile (128 x 64, 8 consumer warps of 32 x 32, BK = 16) as
// dgemm_pipe_kernel, operands moved by the tensor-memory accelerator: per k-slice one elected
// producer thread issues one 16 x 128 box of A and four 16 x 16 boxes of B
// (cp.async.bulk.tensor.2d, 128-byte swizzle, completion counted in bytes on the stage's "full"
// mbarrier). The consumer warps only wait on mbarriers, load fragments (swizzle-aware, conflict
// free) and issue DMMAs, then release the stage on its "empty" mbarrier. CTAs are persistent
// (grid-stride over items), so the producer fills the next item's stages during the epilogue.
// Tensor maps (one per operand allocation, __grid_constant__ parameter) and per-term box
// coordinates are built by GemmPlan::upload; rows / columns past an allocation read as zero, and
// the one K edge on the path (K = 127, eigen back transforms) meets zero pad columns of A.
namespace {
constexpr int TS_STAGES = 4;
constexpr int TS_A_BYTES = 128 * 128;  // 128 rows x 16 doubles
constexpr int TS_B_BYTES = 4 * 2048;   // 4 boxes x (16 rows x 16 doubles)
constexpr int TS_STAGE_BYTES = TS_A_BYTES + TS_B_BYTES;

__device__ __forceinline__ unsigned s_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void tb_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void tb_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tb_arrive_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tb_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TW_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(unsigned dst, const CUtensorMap* map, int c0, int c1, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
}  // namespace

size_t dgemm_tma_smem() { return size_t(TS_STAGES) * TS_STAGE_BYTES + 1024 + 2 * TS_STAGES * sizeof(uint64_t); }

__global__ void __launch_bounds__(288, 2)
    dgemm_tma_kernel(GemmBatch g, const __grid_constant__ TmaMaps maps, const int4* __restrict__ ta,
                     const int2* __restrict__ tb) {
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    // 128-byte swizzle repeats every 1024 bytes: align the stage ring to 1024
    const unsigned raw = s_u32(tsm_raw);
    const unsigned base = (raw + 1023u) & ~1023u;
    unsigned char* tsm = tsm_raw + (base - raw);
    const unsigned bars = base + TS_STAGES * TS_STAGE_BYTES;  // full[s] at bars + 8 s, empty[s] at bars + 8 (S + s)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < TS_STAGES; ++s) {
            tb_init(bars + 8 * s, 1);                // producer arrival + transaction bytes
            tb_init(bars + 8 * (TS_STAGES + s), 8);  // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tn = (g.N + PN - 1) / PN, tmn = ((g.M + 127) / 128) * tn;
    const int nitems = g.nbatch * tmn;
    const int nkt = (g.K + PK - 1) / PK;
    struct Item {
        int b, m0, n0, t0, nk;
    };
    auto decode = [&](int w) {
        Item it;
        it.b = w / tmn;
        const int rem = w - it.b * tmn;
        it.m0 = (rem / tn) * 128;
        it.n0 = (rem - (rem / tn) * tn) * PN;
        it.t0 = g.tstart ? g.tstart[it.b] : it.b;
        it.nk = (g.tstart ? g.tstart[it.b + 1] - it.t0 : 1) * nkt;
        return it;
    };
    if (warp == 8) {
        // ---------------- producer (one thread)
        if (lane == 0) {
            int stage = 0;
            unsigned phase = 0;
            for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
                const Item I = decode(w);
                int t = I.t0, kt = 0;
                int4 a = __ldg(ta + t);
                int2 b = __ldg(tb + t);
                for (int kk = 0; kk < I.nk; ++kk) {
                    const int k0 = kt * PK;
                    tb_wait(bars + 8 * (TS_STAGES + stage), phase ^ 1u);
                    const unsigned full = bars + 8 * stage;
                    tb_arrive_tx(full, TS_STAGE_BYTES);
                    const unsigned sa = base + stage * TS_STAGE_BYTES, sb = sa + TS_A_BYTES;
                    tma_2d(sa, &maps.m[a.x], a.y + k0, a.z + I.m0, full);
#pragma unroll
                    for (int q = 0; q < 4; ++q) tma_2d(sb + 2048 * q, &maps.m[a.w], b.x + I.n0 + 16 * q, b.y + k0, full);
                    if (++stage == TS_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                    if (++kt == nkt && kk + 1 < I.nk) {
                        kt = 0;
                        ++t;
                        a = __ldg(ta + t);
                        b = __ldg(tb + t);
                    }
                }
            }
        }
        return;
    }
    // ---------------- consumers
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int gq = lane >> 2, tq = lane & 3;
    // swizzled byte offsets of this lane's fragments within a stage, k-step s = 0..3 (k = 4 s + tq):
    //   A(row, k) = row * 128 + (((k >> 1) ^ (row & 7)) << 4) + (k & 1) * 8,  row = wm + 8 i + gq
    //             = abase + i * 1024 + ((2 s ^ (gq & 6)) << 4)
    //   B(k, n)   = (n >> 4) * 2048 + k * 128 + ((((n & 15) >> 1) ^ (k & 7)) << 4) + (n & 1) * 8,  n = wn + 8 j + gq
    //             = bbase + (j >> 1) * 2048 + s * 512 + (((j ^ s) & 1) << 6)
    const int g6 = gq & 6;
    const int abase = (wm + gq) * 128 + ((((tq >> 1) ^ gq) & 1) << 4) + (tq & 1) * 8;
    const int bbase = (wn >> 4) * 2048 + tq * 128 + ((((gq >> 1) ^ tq) & 3) << 4) + (gq & 1) * 8;
    int stage = 0;
    unsigned phase = 0;
    Item I = decode(blockIdx.x < nitems ? blockIdx.x : 0);
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        // next item's term range in flight during this item's main loop
        const Item In = decode(w + int(gridDim.x) < nitems ? w + int(gridDim.x) : w);
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kt = 0; kt < I.nk; ++kt) {
            tb_wait(bars + 8 * stage, phase);
            const unsigned char* sa = tsm + stage * TS_STAGE_BYTES;
            const unsigned char* sb = sa + TS_A_BYTES;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                double af[4], bf[4];
                const int ao = abase + (((2 * s) ^ g6) << 4);
#pragma unroll
                for (int i = 0; i < 4; ++i) af[i] = *reinterpret_cast<const double*>(sa + ao + i * 1024);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    bf[j] = *reinterpret_cast<const double*>(sb + bbase + (j >> 1) * 2048 + s * 512 + (((j ^ s) & 1) << 6));
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
            __syncwarp();
            if (lane == 0) tb_arrive(bars + 8 * (TS_STAGES + stage));
            if (++stage == TS_STAGES) {
                stage = 0;
                phase ^= 1u;
            }
        }
        double* __restrict__ C;
        if (g.coff) {
            const long o = g.coff[I.b];
            C = g.cbase[o >> kBaseShift] + (o & ((1L << kBaseShift) - 1));
        } else {
            C = g.C[I.b];
        }
        const double* __restrict__ dl = g.dl ? g.dl[I.b] : nullptr;
        const bool vec = ((reinterpret_cast<uintptr_t>(C) | (uintptr_t(g.ldc) * 8)) & 15) == 0 && !dl && g.beta == 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int r = I.m0 + wm + 8 * i + gq, c = I.n0 + wn + 8 * j + 2 * tq;
                if (r >= g.M) continue;
                double* dst = C + long(r) * g.ldc + c;
                if (vec && c + 1 < g.N) {
                    *reinterpret_cast<double2*>(dst) = make_double2(g.alpha * acc[i][j][0], g.alpha * acc[i][j][1]);
                    continue;
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (c + q < g.N) {
                        double v = g.alpha * acc[i][j][q];
                        if (dl) v *= __ldg(dl + long(r) * g.ldd + c + q);
                        dst[q] = g.beta == 0.0 ? v : fma(g.beta, dst[q], v);
                    }
                }
            }
        I = In;
    }
}

// ---------------------------------------------------------------------------------------------
// Theta direction.
//
// Reference conventions (transform.cpp:144-163, 175-191): values f(theta_l) =
// sum_w c_w e^{i w theta_l}, theta_l = (2l - p) pi / p, i.e. with X[w mod p] =
// (-1)^w c_w the values are the unnormalised inverse DFT of X; analysis c_w =
// (-1)^w X[w mod p] / p with X the forward DFT of the samples. Synthesis keeps
// the real part (transform.cpp:201), so c_0 and the Nyquist coefficient
// contribute their real parts only.
namespace {

// In-place radix-2 DIT FFT on `cnt` complex arrays of length P (power of two),
// data already in bit-reversed order; sign = +1 inverse, -1 forward.
__device__ void fft_pow2_block(double2* __restrict__ d, int cnt, int P, int logP, const double2* __restrict__ tw,
                               int sign) {
    for (int s = 1; s <= logP; ++s) {
        const int half = 1 << (s - 1);
        const int tstep = P >> s;  // twiddle index step
        const int nbf = cnt * (P >> 1);
        for (int i = threadIdx.x; i < nbf; i += blockDim.x) {
            const int arr = i / (P >> 1), bfl = i % (P >> 1);
            const int grp = bfl / half, pos = bfl % half;
            const int i0 = grp * 2 * half + pos, i1 = i0 + half;
            double2 w = tw[pos * tstep];  // exp(-2 pi i pos tstep / P)
            if (sign > 0) w.y = -w.y;
            double2* base = d + arr * P;
            const double2 a = base[i0], bb = base[i1];
            const double2 t = make_double2(w.x * bb.x - w.y * bb.y, w.x * bb.y + w.y * bb.x);
            base[i0] = make_double2(a.x + t.x, a.y + t.y);
            base[i1] = make_double2(a.x - t.x, a.y - t.y);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int bitrev(int x, int logP) { return logP < 0 ? x : int(__brev(unsigned(x)) >> (32 - logP)); }

// Dense DFT of `cnt` complex arrays of length P (any P) from src to dst, natural order both sides:
// dst[k] = sum_j src[j] exp(sign 2 pi i j k / P); twf[q] = exp(-2 pi i q / P). The fallback for p that is not a
// power of two (the reference's FFTW plans take any even p, transform.cpp:19-60): O(P^2) per pencil.
__device__ void dft_dense_block(const double2* __restrict__ src, double2* __restrict__ dst, int cnt, int P,
                                const double2* __restrict__ twf, int sign) {
    for (int i = threadIdx.x; i < cnt * P; i += blockDim.x) {
        const int arr = i / P, k = i % P;
        const double2* x = src + arr * P;
        double re = 0.0, im = 0.0;
        int q = 0;  // j k mod P
        for (int j = 0; j < P; ++j) {
            double2 w = twf[q];
            if (sign > 0) w.y = -w.y;
            re = fma(x[j].x, w.x, fma(-x[j].y, w.y, re));
            im = fma(x[j].x, w.y, fma(x[j].y, w.x, im));
            q += k;
            if (q >= P) q -= P;
        }
        dst[i] = make_double2(re, im);
    }
    __syncthreads();
}

}  // namespace

// Fused theta synthesis -> cross product -> theta analysis (stage X of the NS step).
// in[0..5] = (v_r, v_theta, v_z, w_r, w_theta, w_z), out[0..2] = (a_r, a_theta, a_z),
// all in the (r,z)-value / theta-half-spectrum layout [slot][plane][jr][E | O] (z-parity split
// values: position i < nh holds E_i, i + nh holds O_i, f(+-z_{nh+i}) = E_i +- O_i).
// Generic path: one CTA per (jr, tile of TJ/2 positions = TJ points); shared-memory radix-2 FFTs for a
// power-of-two p, dense DFTs (second buffer behind the first) for any other even p (logp < 0).
__global__ void theta_cross_kernel(ThetaCross t) {
    extern __shared__ double2 sd[];
    const Geo& g = t.g;
    const int P = g.p, logP = t.logp, S = g.nslots;
    const int TJ = t.tj;                 // points per CTA (even): point 2i -> +z, 2i+1 -> -z
    const int jr = t.row0 + blockIdx.y;  // r > 0 grid row
    const int q0 = blockIdx.x * (TJ / 2);  // first position of the tile
    const int ntj = min(TJ / 2, g.nh - q0);
    double2* Z = sd;                       // 3 * TJ arrays of P (packed pairs)
    const double2* tw = t.tw;              // P/2 twiddles exp(-2 pi i q / P)
    // ---- gather Hermitian spectra of pairs (0,1) (2,3) (4,5) into bit-reversed slots
    const int tot = 3 * TJ * P;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        const int jl = e % TJ;              // point fastest -> coalesced gathers
        const int tt = (e / TJ) % P;        // frequency index t in [0, P)
        const int pr = e / (TJ * P);        // pair
        const int pos = jl >> 1;
        const double sgz = (jl & 1) ? -1.0 : 1.0;  // f(-z) = E - O
        double2 z = make_double2(0.0, 0.0);
        if (pos < ntj) {
            // X[t] = (-1)^w c_w with w = t (t < P/2), Nyquist at t = P/2, conj mirror above
            int w;
            bool conjg = false;
            if (tt < P / 2) w = tt;
            else if (tt == P / 2) w = -P / 2;
            else {
                w = P - tt;
                conjg = true;
            }
            const int s = (w == -P / 2) ? P / 2 : w;
            const double sg = ((w & 1) ? -1.0 : 1.0);
            const long off = long(s) * g.slot_stride + long(jr) * g.n + q0 + pos + theta_slot_delta(t, s);
            const long ps = g.plane_stride, oo = g.nh;
            double2 xa, xb;
            {
                const double* fa = t.in[2 * pr];
                const double* fb = t.in[2 * pr + 1];
                xa = make_double2(sg * fma(sgz, fa[off + oo], fa[off]), sg * fma(sgz, fa[off + oo + ps], fa[off + ps]));
                xb = make_double2(sg * fma(sgz, fb[off + oo], fb[off]), sg * fma(sgz, fb[off + oo + ps], fb[off + ps]));
            }
            if (w == 0 || w == -P / 2) {  // Re only (transform.cpp:201)
                xa.y = 0.0;
                xb.y = 0.0;
            }
            if (conjg) {
                xa.y = -xa.y;
                xb.y = -xb.y;
            }
            z = make_double2(xa.x - xb.y, xa.y + xb.x);  // Xa + i Xb
        }
        Z[(pr * TJ + jl) * P + bitrev(tt, logP)] = z;
    }
    __syncthreads();
    double2* Z2 = sd + 3 * TJ * P;  // (dense-DFT path only)
    if (logP >= 0) {
        fft_pow2_block(Z, 3 * TJ, P, logP, tw, +1);
    } else {
        dft_dense_block(Z, Z2, 3 * TJ, P, t.twfull, +1);
        for (int e = threadIdx.x; e < 3 * TJ * P; e += blockDim.x) Z[e] = Z2[e];
        __syncthreads();
    }
    // ---- pointwise cross product a = v x w (ptns.cpp:127-132); repack (a_r + i a_t), (a_z + 0 i)
    for (int e = threadIdx.x; e < TJ * P; e += blockDim.x) {
        const int jl = e / P, l = e % P;
        const double2 p0 = Z[(0 * TJ + jl) * P + l], p1 = Z[(1 * TJ + jl) * P + l], p2 = Z[(2 * TJ + jl) * P + l];
        const double vr = p0.x, vt = p0.y, vz = p1.x, wr = p1.y, wt = p2.x, wz = p2.y;
        const double ar = vt * wz - vz * wt;
        const double at = vz * wr - vr * wz;
        const double az = vr * wt - vt * wr;
        // store in bit-reversed order for the forward transform
        const int lr = bitrev(l, logP);
        Z[(0 * TJ + jl) * P + l] = make_double2(ar, at);
        Z[(1 * TJ + jl) * P + l] = make_double2(az, 0.0);
        (void)lr;
    }
    __syncthreads();
    // bit-reverse permutation in place for the two packed outputs
    for (int e = threadIdx.x; e < 2 * TJ * P; e += blockDim.x) {
        const int a = e / P, l = e % P, lr = bitrev(l, logP);
        if (l < lr) {
            double2* base = Z + a * P;
            const double2 x = base[l];
            base[l] = base[lr];
            base[lr] = x;
        }
    }
    __syncthreads();
    if (logP >= 0) {
        fft_pow2_block(Z, 2 * TJ, P, logP, tw, -1);
    } else {  // (bitrev is the identity: the permutation above moved nothing)
        dft_dense_block(Z, Z2, 2 * TJ, P, t.twfull, -1);
        for (int e = threadIdx.x; e < 2 * TJ * P; e += blockDim.x) Z[e] = Z2[e];
        __syncthreads();
    }
    // ---- unpack X_a = (Z[t] + conj Z[P-t]) / 2, X_b = (Z[t] - conj Z[P-t]) / (2i); c_w = (-1)^w X[w mod P] / P
    const double invp = 1.0 / double(P);
    const int TP = TJ / 2;
    for (int e = threadIdx.x; e < 3 * S * 2 * TP; e += blockDim.x) {
        const int pos = e % TP;
        const int pl = (e / TP) % 2;
        const int s = (e / (2 * TP)) % S;
        const int f = e / (2 * TP * S);  // output field 0..2
        if (pos >= ntj) continue;
        const int w = (s == P / 2) ? -P / 2 : s;
        const int tt = (w % P + P) % P;
        const int pair = f < 2 ? 0 : 1;
        double xv[2];
        for (int h = 0; h < 2; ++h) {
            const double2* base = Z + (pair * TJ + 2 * pos + h) * P;
            const double2 zt = base[tt], zm = base[(P - tt) % P];
            double2 X;
            if (f == 0 || f == 2) X = make_double2(0.5 * (zt.x + zm.x), 0.5 * (zt.y - zm.y));
            else X = make_double2(0.5 * (zt.y + zm.y), -0.5 * (zt.x - zm.x));
            xv[h] = pl ? X.y : X.x;
        }
        const double sg = ((w & 1) ? -1.0 : 1.0) * invp * 0.5;
        const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride + long(jr) * g.n + q0 + pos +
                         theta_slot_delta(t, s);
        t.out[f][off] = sg * (xv[0] + xv[1]);         // E' = (f(+z) + f(-z)) / 2
        t.out[f][off + g.nh] = sg * (xv[0] - xv[1]);  // O' = (f(+z) - f(-z)) / 2
    }
    if (t.world > 1) __threadfence_system();  // peer stores performed before the rank barrier
}

// ---------------------------------------------------------------------------------------------
// p = 256 fast path: the same fused stage with register FFTs (256 = 16 x 16, two radix-16
// passes, one shared-memory transpose each) instead of eight shared-memory radix-2 stages.
// CTA = 8 points (4 z positions x {+z, -z}) of one r row, 8 half-warp groups of 16 threads;
// each group runs one 256-point FFT at a time (16 values per thread). The cross product is
// fused into the first pass of the forward transforms.
namespace {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// radix-4 butterfly with W4 = e^{S i pi / 2}
template <int S>
__device__ __forceinline__ void r4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = csub(a1, a3);
    const double2 u = S > 0 ? make_double2(-t3.y, t3.x) : make_double2(t3.y, -t3.x);  // S i t3
    a0 = cadd(t0, t2);
    a1 = cadd(t1, u);
    a2 = csub(t0, t2);
    a3 = csub(t1, u);
}

// x * W16^e, W16 = e^{S 2 pi i / 16}, e in {1, 2, 3, 4, 6, 9} (compile-time after unrolling)
template <int S>
__device__ __forceinline__ double2 tw16(double2 x, int e) {
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, c2 = 0.70710678118654752440;
    switch (e) {
        case 1: return cmul(x, make_double2(c1, S * s1));
        case 2: return cmul(x, make_double2(c2, S * c2));
        case 3: return cmul(x, make_double2(s1, S * c1));
        case 4: return S > 0 ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
        case 6: return cmul(x, make_double2(-c2, S * c2));
        case 9: return cmul(x, make_double2(-c1, -S * s1));
        default: return x;
    }
}

// in-place 16-point DFT X[k] = sum_n x[n] e^{S 2 pi i n k / 16}; X[k1 + 4 k2] lands in v[4 k1 + k2]
template <int S>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) r4<S>(v[n2], v[4 + n2], v[8 + n2], v[12 + n2]);
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) v[n2 + 4 * k1] = tw16<S>(v[n2 + 4 * k1], n2 * k1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) r4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
}
__device__ __forceinline__ int d16(int k) { return 4 * (k & 3) + (k >> 2); }  // slot of X[k] after dft16

constexpr int kT256Pts = 4;    // points per CTA (2 z positions x {+z, -z}); 16 threads per point
constexpr int kT256Pos = kT256Pts / 2;
constexpr int kT256Arr = 272;  // complex slots per array (16 x 17 transposed layout)

// pass 1 of a 256-point DFT on Z (natural order): DFT over n1 of x[16 n1 + lane], twiddle,
// store transposed T[k1 * 17 + lane]. twf[16 k1 + lane] = e^{-2 pi i lane k1 / 256} (lane-fastest:
// conflict-free shared loads).
template <int S>
__device__ __forceinline__ void f256_pass1(double2 (&v)[16], double2* Z, int lane, const double2* twf) {
    dft16<S>(v);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) {
        double2 w = twf[16 * k1 + lane];
        if (S > 0) w.y = -w.y;
        Z[k1 * 17 + lane] = k1 == 0 ? v[d16(k1)] : cmul(v[d16(k1)], w);
    }
}
// pass 2: DFT over n2 of T[lane * 17 + n2] -> X[lane + 16 k2], stored in natural order.
template <int S>
__device__ __forceinline__ void f256_pass2(double2* Z, int lane, unsigned gmask) {
    double2 v[16];
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) v[n2] = Z[lane * 17 + n2];
    __syncwarp(gmask);
    dft16<S>(v);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) Z[lane + 16 * k2] = v[d16(k2)];
}

}  // namespace

__global__ void __launch_bounds__(16 * kT256Pts, 4) theta_cross256_kernel(ThetaCross t) {
    extern __shared__ double2 sd[];
    double2* twf = sd + kT256Pts * 3 * kT256Arr;
    const Geo& g = t.g;
    const int S = g.nslots;  // 129
    const int jr = blockIdx.y;
    const int i0 = blockIdx.x * kT256Pos;
    const int npos = min(kT256Pos, g.nh - i0);
    const int tid = threadIdx.x;
    for (int x = tid; x < 256; x += blockDim.x) {
        const int e = (x >> 4) * (x & 15);  // k1 * lane < 256
        twf[x] = e < 128 ? t.tw[e] : make_double2(-t.tw[e - 128].x, -t.tw[e - 128].y);
    }
    // ---- gather the Hermitian spectra of the pairs (v_r, v_t), (v_z, w_r), (w_t, w_z) at 8 points
    const long ps = g.plane_stride, oo = g.nh;
#pragma unroll 2
    for (int e = tid; e < S * 3; e += blockDim.x) {
        const int s = e % S, pr = e / S;
        const double sg = (s & 1) ? -1.0 : 1.0;  // (-1)^w (w = s, or -128 for the Nyquist slot s = 128)
        const bool reonly = (s == 0 || s == 128);
        const long off = long(s) * g.slot_stride + long(jr) * g.n + i0;
        const double* __restrict__ fa = t.in[2 * pr] + off;
        const double* __restrict__ fb = t.in[2 * pr + 1] + off;
#pragma unroll
        for (int ip = 0; ip < kT256Pos; ++ip) {
            double ar = 0.0, ai = 0.0, aro = 0.0, aio = 0.0, br = 0.0, bi = 0.0, bro = 0.0, bio = 0.0;
            if (ip < npos) {
                ar = __ldg(fa + ip);
                ai = __ldg(fa + ps + ip);
                aro = __ldg(fa + oo + ip);
                aio = __ldg(fa + oo + ps + ip);
                br = __ldg(fb + ip);
                bi = __ldg(fb + ps + ip);
                bro = __ldg(fb + oo + ip);
                bio = __ldg(fb + oo + ps + ip);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double sz = h ? -1.0 : 1.0;
                const double xar = sg * fma(sz, aro, ar), xai = reonly ? 0.0 : sg * fma(sz, aio, ai);
                const double xbr = sg * fma(sz, bro, br), xbi = reonly ? 0.0 : sg * fma(sz, bio, bi);
                double2* Z = sd + ((2 * ip + h) * 3 + pr) * kT256Arr;
                Z[s] = make_double2(xar - xbi, xai + xbr);
                if (s > 0 && s < 128) Z[256 - s] = make_double2(xar + xbi, xbr - xai);
            }
        }
    }
    __syncthreads();
    const int grp = tid >> 4, lane = tid & 15;
    const unsigned gmask = 0xFFFFu << (16 * (grp & 1));
    // ---- inverse transforms (synthesis in theta): 24 arrays, 8 groups
    for (int a = grp; a < kT256Pts * 3; a += kT256Pts) {
        double2* Z = sd + a * kT256Arr;
        double2 v[16];
#pragma unroll
        for (int n1 = 0; n1 < 16; ++n1) v[n1] = Z[16 * n1 + lane];
        __syncwarp(gmask);
        f256_pass1<+1>(v, Z, lane, twf);
        __syncwarp(gmask);
        f256_pass2<+1>(Z, lane, gmask);
        __syncwarp(gmask);
    }
    __syncthreads();
    // ---- cross product a = v x w (ptns.cpp:127-132) fused into pass 1 of the forward transforms
    {
        const int pt = grp;
        double2* Z0 = sd + (pt * 3 + 0) * kT256Arr;
        double2* Z1 = sd + (pt * 3 + 1) * kT256Arr;
        const double2* Z2 = sd + (pt * 3 + 2) * kT256Arr;
        double2 v[16], u[16];
#pragma unroll
        for (int n1 = 0; n1 < 16; ++n1) {
            const int l = 16 * n1 + lane;
            const double2 p0 = Z0[l], p1 = Z1[l], p2 = Z2[l];
            const double vr = p0.x, vt = p0.y, vz = p1.x, wr = p1.y, wt = p2.x, wz = p2.y;
            v[n1] = make_double2(vt * wz - vz * wt, vz * wr - vr * wz);  // a_r + i a_t
            u[n1] = make_double2(vr * wt - vt * wr, 0.0);               // a_z
        }
        __syncwarp(gmask);
        f256_pass1<-1>(v, Z0, lane, twf);
        f256_pass1<-1>(u, Z1, lane, twf);
        __syncwarp(gmask);
        f256_pass2<-1>(Z0, lane, gmask);
        f256_pass2<-1>(Z1, lane, gmask);
    }
    __syncthreads();
    // ---- unpack c_w = (-1)^w X[w mod 256] / 256 per point; store E' = (f+ + f-)/2, O' = (f+ - f-)/2
    for (int e = tid; e < S * 3; e += blockDim.x) {
        const int s = e % S, f = e / S;
        const int tt = s, tm = (256 - s) & 255;
        const double sg = ((s & 1) ? -1.0 : 1.0) * (0.5 / 256.0);
        const int arr = f < 2 ? 0 : 1;
        const long off = long(s) * g.slot_stride + long(jr) * g.n + i0;
        double* o = t.out[f] + off;
#pragma unroll
        for (int ip = 0; ip < kT256Pos; ++ip) {
            if (ip >= npos) break;
            double xr[2], xi[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double2* base = sd + ((2 * ip + h) * 3 + arr) * kT256Arr;
                const double2 zt = base[tt], zm = base[tm];
                if (f == 1) {
                    xr[h] = 0.5 * (zt.y + zm.y);
                    xi[h] = -0.5 * (zt.x - zm.x);
                } else {
                    xr[h] = 0.5 * (zt.x + zm.x);
                    xi[h] = 0.5 * (zt.y - zm.y);
                }
            }
            o[ip] = sg * (xr[0] + xr[1]);
            o[oo + ip] = sg * (xr[0] - xr[1]);
            o[ps + ip] = sg * (xi[0] + xi[1]);
            o[ps + oo + ip] = sg * (xi[0] - xi[1]);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// p = 256, warp-per-point variant: 32 lanes per 256-point FFT as 16 lane pairs; in every radix-16
// pass each lane loads the 16 inputs of its column and produces the 8 outputs of one parity
// (half-DFT16 = radix-2 split + DFT8). The three (v, w) pairs are synthesized one after the other
// through a single shared array per point (their time samples stay in registers: lane (k1, h)
// holds l = k1 + 16 k2 for k2 = h (mod 2)), so the cross product and the first forward pass run in
// registers (the k2-parity halves combine through one shuffle). 8.5 KB of shared memory per point
// instead of 12.75 KB and twice the threads: 16 warps per SM instead of 8.
namespace {

template <int S>
__device__ __forceinline__ double2 w8mul(double2 x, int n) {  // x * W8^n, W8 = e^{S 2 pi i / 8}, n in 0..3
    constexpr double c = 0.70710678118654752440;
    switch (n) {
        case 1: return cmul(x, make_double2(c, S * c));
        case 2: return S > 0 ? make_double2(-x.y, x.x) : make_double2(x.y, -x.x);
        case 3: return cmul(x, make_double2(-c, S * c));
        default: return x;
    }
}

// in-place DFT8, natural-order output
template <int S>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
    double2 a[4], b[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
        a[n] = cadd(v[n], v[n + 4]);
        b[n] = w8mul<S>(csub(v[n], v[n + 4]), n);
    }
    r4<S>(a[0], a[1], a[2], a[3]);
    r4<S>(b[0], b[1], b[2], b[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = a[k];
        v[2 * k + 1] = b[k];
    }
}

// outputs X[2k + h], k = 0..7, of the DFT16 of x[0..15] (W16 = e^{S 2 pi i / 16})
template <int S>
__device__ __forceinline__ void half_dft16(const double2 (&x)[16], int h, double2 (&out)[8]) {
#pragma unroll
    for (int n = 0; n < 8; ++n) {
        const double2 sum = cadd(x[n], x[n + 8]);
        const double2 dif = csub(x[n], x[n + 8]);
        out[n] = h ? tw16<S>(dif, n) : sum;
    }
    // tw16 covers the exponents of the radix-4 x radix-4 DFT16; here the radix-2 twiddles W16^n,
    // n = 0..7, are applied explicitly below for n = 5 and 7 (tw16 handles 1, 2, 3, 4, 6)
    if (h) {
        constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
        out[5] = cmul(csub(x[5], x[13]), make_double2(-s1, S * c1));
        out[7] = cmul(csub(x[7], x[15]), make_double2(-c1, S * s1));
    }
    dft8<S>(out);
}

constexpr int kTWArr = 272;
// point stride: the two arrays plus one double2, so the points 4 apart that neighbouring threads of the
// spectrum assembly / unpack tasks touch (z-position pairs q = 0, 1) sit in different 16-byte bank groups
constexpr int kTWPt = 2 * kTWArr + 1;

}  // namespace

// NQ z-position pairs per CTA (4 NQ points, one warp each); load / store tasks are (slot, pair)
// so that the two threads of one slot cover a full 32-byte sector when NQ = 2
template <int NQ>
__global__ void __launch_bounds__(128 * NQ, 4 / NQ) theta_cross256w_kernel(ThetaCross t) {
    constexpr int kPts = 4 * NQ;
    extern __shared__ double2 sd[];
    double2* twf = sd + kPts * kTWPt;  // twf[16 k1 + n2] = e^{-2 pi i n2 k1 / 256} (forward stage)
    const Geo& g = t.g;
    const int S = g.nslots;  // 129
    const int jr = t.row0 + blockIdx.y;
    const int i0 = blockIdx.x * (2 * NQ);
    const int npos = min(2 * NQ, g.nh - i0);
    // 16-byte global accesses when every stride is even (per pair: both positions present)
    const bool even = ((g.slot_stride | g.plane_stride | long(g.n) | long(g.nh)) & 1) == 0;
    const int tid = threadIdx.x;
    const int pt = tid >> 5, lane = tid & 31, col = lane & 15, h = lane >> 4;
    for (int x = tid; x < 256; x += blockDim.x) {
        const int e = (x >> 4) * (x & 15);
        twf[x] = e < 128 ? t.tw[e] : make_double2(-t.tw[e - 128].x, -t.tw[e - 128].y);
    }
    double2* Z = sd + pt * kTWPt;  // this point's two arrays
    double2 tv[3][8];                   // time samples of the three pairs at l = col + 16 (2j + h)
    const long ps = g.plane_stride, oo = g.nh;
    const long ooi = t.vquad ? long(g.nh) * g.mh : long(g.nh);  // odd-z half of the inputs
    // raw spectra of one (v, w) pair for task a = (slot a / NQ, position pair a % NQ), prefetched into
    // registers one pair ahead so the global-load latency overlaps the previous pair's FFTs (tasks
    // beyond the thread count, i.e. the Nyquist slot, are loaded in place)
    const int NT = NQ * S;
    double raw[2][8];
    auto fetch_slot = [&](int pr, int a, double (&r)[2][8]) {
#pragma unroll
        for (int ip = 0; ip < 2; ++ip)
#pragma unroll
            for (int u = 0; u < 8; ++u) r[ip][u] = 0.0;
        const int s = a / NQ, q = a - s * NQ;
        const int nq = min(2, npos - 2 * q);
        if (nq <= 0) return;
        const bool vec = even && nq == 2;
        const int z = i0 + 2 * q;
        const long off = long(s) * g.slot_stride +
                         (t.vquad ? long(z >> 2) * 4 * g.mh + long(jr) * 4 + (z & 3) : long(jr) * g.n + z) +
                         theta_slot_delta(t, s);
        const double* __restrict__ fa = t.in[2 * pr] + off;
        const double* __restrict__ fb = t.in[2 * pr + 1] + off;
        if (vec) {  // both z positions: 16-byte loads
            const double* src[8] = {fa, fa + ps, fa + ooi, fa + ooi + ps, fb, fb + ps, fb + ooi, fb + ooi + ps};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(src[u]));
                r[0][u] = v.x;
                r[1][u] = v.y;
            }
            return;
        }
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) {
            if (ip >= nq) continue;
            r[ip][0] = __ldg(fa + ip);
            r[ip][1] = __ldg(fa + ps + ip);
            r[ip][2] = __ldg(fa + ooi + ip);
            r[ip][3] = __ldg(fa + ooi + ps + ip);
            r[ip][4] = __ldg(fb + ip);
            r[ip][5] = __ldg(fb + ps + ip);
            r[ip][6] = __ldg(fb + ooi + ip);
            r[ip][7] = __ldg(fb + ooi + ps + ip);
        }
    };
    auto put_slot = [&](int a, const double (&r)[2][8], int arr) {
        const int s = a / NQ, q = a - s * NQ;
        const double sg = (s & 1) ? -1.0 : 1.0;
        const bool reonly = (s == 0 || s == 128);
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) {
            const double ar = r[ip][0], ai = r[ip][1], aro = r[ip][2], aio = r[ip][3];
            const double br = r[ip][4], bi = r[ip][5], bro = r[ip][6], bio = r[ip][7];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const double sz = hh ? -1.0 : 1.0;
                const double xar = sg * fma(sz, aro, ar), xai = reonly ? 0.0 : sg * fma(sz, aio, ai);
                const double xbr = sg * fma(sz, bro, br), xbi = reonly ? 0.0 : sg * fma(sz, bio, bi);
                double2* Zp = sd + (2 * (2 * q + ip) + hh) * kTWPt + arr * kTWArr;
                Zp[s] = make_double2(xar - xbi, xai + xbr);
                if (s > 0 && s < 128) Zp[256 - s] = make_double2(xar + xbi, xbr - xai);
            }
        }
    };
    // Hermitian spectrum of pair pr for the CTA's points into array arr, then prefetch pair pr + 1
    auto put_pair = [&](int pr, int arr) {
        if (tid < NT) put_slot(tid, raw, arr);
        for (int a = tid + blockDim.x; a < NT; a += blockDim.x) {  // Nyquist slot tasks
            double r2[2][8];
            fetch_slot(pr, a, r2);
            put_slot(a, r2, arr);
        }
        if (pr < 2 && tid < NT) fetch_slot(pr + 1, tid, raw);
    };
    // inverse FFT of this warp's point from array ZA into the lane's 8 time samples
    auto inverse = [&](double2* ZA, double2 (&out)[8]) {
        double2 x[16], o[8];
        // pass 1: lane (n2 = col, h): DFT16 over n1 of x[16 n1 + n2] -> k1 = 2k + h
#pragma unroll
        for (int n1 = 0; n1 < 16; ++n1) x[n1] = ZA[16 * n1 + col];
        __syncwarp();
        half_dft16<+1>(x, h, o);
        {  // conj twiddles e^{+2 pi i col (2k + h) / 256} by recurrence: base e^{2 pi i col h / 256}, step e^{4 pi i col / 256}
            const double2 b = __ldg(t.tw + col), st0 = __ldg(t.tw + 2 * col);
            double2 w = h ? make_double2(b.x, -b.y) : make_double2(1.0, 0.0);
            const double2 st = make_double2(st0.x, -st0.y);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int k1 = 2 * k + h;
                ZA[k1 * 17 + col] = (k || h) ? cmul(o[k], w) : o[0];
                if (k < 7) w = (k || h) ? cmul(w, st) : st;
            }
        }
        __syncwarp();
        // pass 2: lane (k1 = col, h): DFT16 over n2 -> samples l = k1 + 16 (2j + h)
#pragma unroll
        for (int n2 = 0; n2 < 16; ++n2) x[n2] = ZA[col * 17 + n2];
        half_dft16<+1>(x, h, out);
    };
    // the three pairs alternate between the point's two arrays, so one CTA barrier per pair
    // separates the cross-point spectrum writes from the warp-local FFTs
    if (tid < NT) fetch_slot(0, tid, raw);
    put_pair(0, 0);
    __syncthreads();  // pair 0 in array 0 (and the twiddle table) visible
    put_pair(1, 1);
    inverse(Z, tv[0]);
    __syncthreads();  // pair 1 in array 1; every point's array 0 consumed
    put_pair(2, 0);
    inverse(Z + kTWArr, tv[1]);
    __syncthreads();  // pair 2 in array 0
    inverse(Z, tv[2]);
    // ---- cross product a = v x w (ptns.cpp:127-132) at this lane's 8 samples
    double2 ya[8], yz[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const double vr = tv[0][j].x, vt = tv[0][j].y, vz = tv[1][j].x, wr = tv[1][j].y, wt = tv[2][j].x,
                     wz = tv[2][j].y;
        ya[j] = make_double2(vt * wz - vz * wt, vz * wr - vr * wz);  // a_r + i a_t
        yz[j] = make_double2(vr * wt - vt * wr, 0.0);               // a_z
    }
    // ---- forward pass 1 (DFT16 over k2 for k1 = col): this lane holds k2 = 2j + h; radix-2 combine
    //      with the partner lane (h ^ 1), then twiddle and transpose into arrays 0 (a_r + i a_t), 1 (a_z)
    __syncwarp();  // this warp's reads of its point's arrays done (no other warp touches them now)
    dft8<-1>(ya);
    dft8<-1>(yz);
    {
        constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, c2 = 0.70710678118654752440;
        const double2 w16[8] = {make_double2(1.0, 0.0), make_double2(c1, -s1), make_double2(c2, -c2),
                                make_double2(s1, -c1), make_double2(0.0, -1.0), make_double2(-s1, -c1),
                                make_double2(-c2, -c2), make_double2(-c1, -s1)};
        auto combine = [&](double2 (&y)[8], double2* T) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                // E = even-k2 DFT8 (lane h = 0), O = odd-k2 DFT8 (lane h = 1)
                const double ox = __shfl_xor_sync(0xffffffffu, y[k].x, 16);
                const double oy = __shfl_xor_sync(0xffffffffu, y[k].y, 16);
                const double2 E = h ? make_double2(ox, oy) : y[k];
                const double2 O = h ? y[k] : make_double2(ox, oy);
                const double2 wo = cmul(O, w16[k]);
                const double2 Y = h ? csub(E, wo) : cadd(E, wo);  // Y[k + 8 h]
                const int kp = k + 8 * h;
                T[kp * 17 + col] = cmul(Y, twf[16 * kp + col]);
            }
        };
        combine(ya, Z);
        combine(yz, Z + kTWArr);
    }
    __syncwarp();
    // ---- forward pass 2: lane (k' = col, h): DFT16 over k1 -> Y[k' + 16 (2k + h)], natural order
#pragma unroll
    for (int arr = 0; arr < 2; ++arr) {
        double2* T = Z + arr * kTWArr;
        double2 x[16], o[8];
#pragma unroll
        for (int k1 = 0; k1 < 16; ++k1) x[k1] = T[col * 17 + k1];
        __syncwarp();
        half_dft16<-1>(x, h, o);
#pragma unroll
        for (int k = 0; k < 8; ++k) T[col + 16 * (2 * k + h)] = o[k];
        __syncwarp();
    }
    __syncthreads();
    // ---- unpack c_w = (-1)^w X[w mod 256] / 256 per point; store E' = (f+ + f-)/2, O' = (f+ - f-)/2;
    //      tasks (slot, output f, position pair q)
    for (int e = tid; e < S * 3 * NQ; e += blockDim.x) {
        const int q = e % NQ, sf = e / NQ;
        const int s = sf % S, f = sf / S;
        const int nq = min(2, npos - 2 * q);
        if (nq <= 0) continue;
        const int tt = s, tm = (256 - s) & 255;
        const double sg = ((s & 1) ? -1.0 : 1.0) * (0.5 / 256.0);
        const int arr = f < 2 ? 0 : 1;
        const long off = long(s) * g.slot_stride + long(jr) * g.n + i0 + 2 * q + theta_slot_delta(t, s);
        double* o = t.out[f] + off;
        double ov[4][2];
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) {
            if (ip >= nq) break;
            double xr[2], xi[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const double2* base = sd + (2 * (2 * q + ip) + hh) * kTWPt + arr * kTWArr;
                const double2 zt = base[tt], zm = base[tm];
                if (f == 1) {
                    xr[hh] = 0.5 * (zt.y + zm.y);
                    xi[hh] = -0.5 * (zt.x - zm.x);
                } else {
                    xr[hh] = 0.5 * (zt.x + zm.x);
                    xi[hh] = 0.5 * (zt.y - zm.y);
                }
            }
            ov[0][ip] = sg * (xr[0] + xr[1]);
            ov[1][ip] = sg * (xr[0] - xr[1]);
            ov[2][ip] = sg * (xi[0] + xi[1]);
            ov[3][ip] = sg * (xi[0] - xi[1]);
        }
        double* dst[4] = {o, o + oo, o + ps, o + ps + oo};
        if (even && nq == 2) {
#pragma unroll
            for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(dst[u]) = make_double2(ov[u][0], ov[u][1]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) dst[u][0] = ov[u][0];
        }
    }
    if (t.world > 1) __threadfence_system();  // peer stores performed before the rank barrier
}

template __global__ void theta_cross256w_kernel<1>(ThetaCross);
template __global__ void theta_cross256w_kernel<2>(ThetaCross);

// ---------------------------------------------------------------------------------------------
// p = 512 path: the generic kernel's structure (TJ points per CTA, three packed pairs in shared
// memory) with three radix-8 passes (512 = 8^3, register DFT8 per butterfly) instead of nine
// radix-2 stages. Input is stored in base-8 digit-reversed order and the passes are in-place DIT;
// arrays are padded (index i + i / 8 + i / 64) so that the passes and the digit-reversed spectrum
// writes are bank-conflict free for 16-byte accesses. Global loads / stores are (pair or output,
// slot) tasks covering the CTA's two z positions with 16-byte accesses, as in the p = 256 kernel.
namespace {

constexpr int kP512 = 512, kA512 = 584;  // padded array length
// padding: one element per 8 and per 64, so unit-stride, stride-8 and stride-64 (digit-reversed
// neighbours) 16-byte accesses of 8 lanes hit 8 distinct 4-bank groups
__device__ __forceinline__ int zp512(int i) { return i + (i >> 3) + (i >> 6); }
__device__ __forceinline__ int digrev8(int t) { return ((t & 7) << 6) | (t & 56) | (t >> 6); }

template <int S>
__device__ __forceinline__ void fft512_r8(double2* __restrict__ d, int cnt, const double2* __restrict__ tw) {
#pragma unroll 1
    for (int ls = 0; ls < 9; ls += 3) {  // span L = 8^(ls/3) of the merged sub-transforms
        const int L = 1 << ls;
        const int nbf = cnt * 64;
        for (int i = threadIdx.x; i < nbf; i += blockDim.x) {
            const int arr = i >> 6, j = i & 63;
            const int pos = j & (L - 1), grp = j >> ls;
            double2* base = d + arr * kA512;
            const int i0 = grp * 8 * L + pos;
            double2 v[8];
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = base[zp512(i0 + r * L)];
            if (L > 1) {
                // W_{8L}^{pos r} = w1^r, w1 = e^{S 2 pi i pos 64 / (L 512)} (one table load, then a
                // register recurrence: the per-r table loads were the kernel's top stall)
                double2 w1 = tw[pos << (6 - ls)];
                if (S > 0) w1.y = -w1.y;
                double2 w = w1;
#pragma unroll
                for (int r = 1; r < 8; ++r) {
                    v[r] = cmul(v[r], w);
                    if (r < 7) w = cmul(w, w1);
                }
            }
            dft8<S>(v);
#pragma unroll
            for (int k = 0; k < 8; ++k) base[zp512(i0 + k * L)] = v[k];
        }
        __syncthreads();
    }
}

}  // namespace

__global__ void __launch_bounds__(kTheta512Threads, 2) theta_cross512_kernel(ThetaCross t) {
    extern __shared__ double2 sd[];
    const Geo& g = t.g;
    constexpr int P = kP512;
    const int S = g.nslots;
    constexpr int TJ = kTheta512Points;  // points per CTA (even): point 2i -> +z, 2i+1 -> -z
    const int jr = t.row0 + blockIdx.y;  // r > 0 grid row
    const int q0 = blockIdx.x * (TJ / 2);
    const int ntj = min(TJ / 2, g.nh - q0);
    double2* Z = sd;  // 3 * TJ padded arrays (packed pairs)
    const double2* tw = t.tw;  // P/2 twiddles exp(-2 pi i q / P)
    const long ps = g.plane_stride, oo = g.nh;
    // ---- Hermitian spectra of pairs (0,1) (2,3) (4,5) into digit-reversed slots; task (pair, slot)
    //      loads both z positions of the tile and writes the 2 x 2 points' values at t = s and P - s
    const bool vec = ((g.slot_stride | g.plane_stride | long(g.n) | long(g.nh)) & 1) == 0 && ntj == 2;
    for (int a = threadIdx.x; a < 3 * (P / 2 + 1); a += blockDim.x) {
        const int pr = a / (P / 2 + 1), s = a - pr * (P / 2 + 1);
        const double sg = (s & 1) ? -1.0 : 1.0;
        const bool reonly = (s == 0 || s == P / 2);  // Re only (transform.cpp:201)
        const long off = long(s) * g.slot_stride + long(jr) * g.n + q0 + theta_slot_delta(t, s);
        const double* __restrict__ fa = t.in[2 * pr] + off;
        const double* __restrict__ fb = t.in[2 * pr + 1] + off;
        double r[2][8];
        if (vec) {
            const double* src[8] = {fa, fa + ps, fa + oo, fa + oo + ps, fb, fb + ps, fb + oo, fb + oo + ps};
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(src[u]));
                r[0][u] = v.x;
                r[1][u] = v.y;
            }
        } else {
#pragma unroll
            for (int ip = 0; ip < 2; ++ip) {
                const bool in = ip < ntj;
                r[ip][0] = in ? __ldg(fa + ip) : 0.0;
                r[ip][1] = in ? __ldg(fa + ps + ip) : 0.0;
                r[ip][2] = in ? __ldg(fa + oo + ip) : 0.0;
                r[ip][3] = in ? __ldg(fa + oo + ps + ip) : 0.0;
                r[ip][4] = in ? __ldg(fb + ip) : 0.0;
                r[ip][5] = in ? __ldg(fb + ps + ip) : 0.0;
                r[ip][6] = in ? __ldg(fb + oo + ip) : 0.0;
                r[ip][7] = in ? __ldg(fb + oo + ps + ip) : 0.0;
            }
        }
        const int ts = zp512(digrev8(s)), tm = zp512(digrev8((P - s) & (P - 1)));
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) {
            const double ar = r[ip][0], ai = r[ip][1], aro = r[ip][2], aio = r[ip][3];
            const double br = r[ip][4], bi = r[ip][5], bro = r[ip][6], bio = r[ip][7];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // point 2 ip + hh: f(+-z) = E +- O
                const double sz = hh ? -1.0 : 1.0;
                const double xar = sg * fma(sz, aro, ar), xai = reonly ? 0.0 : sg * fma(sz, aio, ai);
                const double xbr = sg * fma(sz, bro, br), xbi = reonly ? 0.0 : sg * fma(sz, bio, bi);
                double2* Zp = Z + (pr * TJ + 2 * ip + hh) * kA512;
                Zp[ts] = make_double2(xar - xbi, xai + xbr);                       // Xa + i Xb at t = s
                if (s > 0 && s < P / 2) Zp[tm] = make_double2(xar + xbi, xbr - xai);  // conj mirror at P - s
            }
        }
    }
    __syncthreads();
    fft512_r8<+1>(Z, 3 * TJ, tw);
    // ---- pointwise cross product a = v x w (ptns.cpp:127-132); (a_r + i a_t) and (a_z + 0 i) are
    //      written digit-reversed into arrays [0, TJ) and [TJ, 2 TJ) for the forward transform. The
    //      permutation crosses threads, so every sample is read (kPer per thread) before any write.
    constexpr int kPer = TJ * P / kTheta512Threads;  // samples per thread
    static_assert(kPer * kTheta512Threads == TJ * P && TJ == 4, "theta512: task mapping assumes TJ = 4");
    double2 A[kPer], B[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kTheta512Threads;
        if (e < TJ * P) {
            const int jl = e >> 9, l = e & (P - 1);
            const double2 p0 = Z[(0 * TJ + jl) * kA512 + zp512(l)], p1 = Z[(1 * TJ + jl) * kA512 + zp512(l)],
                          p2 = Z[(2 * TJ + jl) * kA512 + zp512(l)];
            const double vr = p0.x, vt = p0.y, vz = p1.x, wr = p1.y, wt = p2.x, wz = p2.y;
            A[u] = make_double2(vt * wz - vz * wt, vz * wr - vr * wz);
            B[u] = make_double2(vr * wt - vt * wr, 0.0);
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
        const int e = threadIdx.x + u * kTheta512Threads;
        if (e < TJ * P) {
            const int jl = e >> 9, l = zp512(digrev8(e & (P - 1)));
            Z[(0 * TJ + jl) * kA512 + l] = A[u];
            Z[(1 * TJ + jl) * kA512 + l] = B[u];
        }
    }
    __syncthreads();
    fft512_r8<-1>(Z, 2 * TJ, tw);
    // ---- unpack X_a = (Z[t] + conj Z[P-t]) / 2, X_b = (Z[t] - conj Z[P-t]) / (2i); c_w = (-1)^w X[w mod P] / P;
    //      task (output f, slot s) stores E' = (f+ + f-)/2, O' = (f+ - f-)/2 of both positions and planes
    for (int e = threadIdx.x; e < 3 * S; e += blockDim.x) {
        const int f = e / S, s = e - f * S;
        const int arr0 = f < 2 ? 0 : TJ;
        const double sg = ((s & 1) ? -1.0 : 1.0) * (0.5 / double(P));
        const int tt = zp512(s), tm = zp512((P - s) & (P - 1));  // s = P/2: Nyquist, w = -P/2 = P/2 (mod P)
        double ov[4][2];
#pragma unroll
        for (int ip = 0; ip < 2; ++ip) {
            double xr[2], xi[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const double2* base = Z + (arr0 + 2 * ip + hh) * kA512;
                const double2 zt = base[tt], zm = base[tm];
                if (f == 1) {
                    xr[hh] = 0.5 * (zt.y + zm.y);
                    xi[hh] = -0.5 * (zt.x - zm.x);
                } else {
                    xr[hh] = 0.5 * (zt.x + zm.x);
                    xi[hh] = 0.5 * (zt.y - zm.y);
                }
            }
            ov[0][ip] = sg * (xr[0] + xr[1]);
            ov[1][ip] = sg * (xr[0] - xr[1]);
            ov[2][ip] = sg * (xi[0] + xi[1]);
            ov[3][ip] = sg * (xi[0] - xi[1]);
        }
        double* o = t.out[f] + long(s) * g.slot_stride + long(jr) * g.n + q0 + theta_slot_delta(t, s);
        double* dst[4] = {o, o + oo, o + ps, o + ps + oo};
        if (vec) {
#pragma unroll
            for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(dst[u]) = make_double2(ov[u][0], ov[u][1]);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                dst[u][0] = ov[u][0];
                if (ntj > 1) dst[u][1] = ov[u][1];
            }
        }
    }
    if (t.world > 1) __threadfence_system();  // peer stores performed before the rank barrier
}

size_t theta_cross512_smem() { return size_t(3) * kTheta512Points * kA512 * sizeof(double2); }

size_t theta_cross256w_smem(int nq) { return (size_t(4 * nq) * kTWPt + 256) * sizeof(double2); }

size_t theta_cross256_smem() { return (size_t(kT256Pts) * 3 * kT256Arr + 256) * sizeof(double2); }
int theta_cross256_positions() { return kT256Pos; }
int theta_cross256_threads() { return 16 * kT256Pts; }

// Full-spectrum complex theta DFT for the API transforms (any even p):
// data [l][k][j] complex interleaved; dir = +1 synthesis (c -> values), -1 analysis.
__global__ void theta_dft_full_kernel(const double* __restrict__ in, double* __restrict__ out, int m, int n, int p,
                                      int dir, const double2* __restrict__ twp) {
    extern __shared__ double2 sx[];
    const long mn = long(m) * n;
    const long q = blockIdx.x;  // one (k, j) pencil per CTA
    if (q >= mn) return;
    for (int l = threadIdx.x; l < p; l += blockDim.x) {
        const int w = l - p / 2;
        const int t = ((w % p) + p) % p;
        const double sg = (w & 1) ? -1.0 : 1.0;
        const double re = in[2 * (long(l) * mn + q)], im = in[2 * (long(l) * mn + q) + 1];
        if (dir > 0) sx[t] = make_double2(sg * re, sg * im);  // X[w mod p] = (-1)^w c_w
        else sx[l] = make_double2(re, im);
    }
    __syncthreads();
    // naive O(p^2) DFT with a p-periodic twiddle table (twp[x] = exp(-2 pi i x / p))
    for (int o = threadIdx.x; o < p; o += blockDim.x) {
        double sr = 0.0, si = 0.0;
        for (int x = 0; x < p; ++x) {
            double2 w = twp[(long(o) * x) % p];
            if (dir > 0) w.y = -w.y;
            const double2 v = sx[x];
            sr += v.x * w.x - v.y * w.y;
            si += v.x * w.y + v.y * w.x;
        }
        if (dir > 0) {
            out[2 * (long(o) * mn + q)] = sr;  // Re kept by the caller after the r,z sweeps
            out[2 * (long(o) * mn + q) + 1] = si;
        } else {
            // analysis: slice l with w = l - p/2 takes X[w mod p] * (-1)^w / p
            // (scatter: output index o is t; map back to l)
            const int t = o;
            const int w = t < p / 2 ? t : t - p;  // w in [-p/2, p/2)
            const int l = w + p / 2;
            const double sg = ((w & 1) ? -1.0 : 1.0) / double(p);
            out[2 * (long(l) * mn + q)] = sg * sr;
            out[2 * (long(l) * mn + q) + 1] = sg * si;
        }
    }
}

}  // namespace ccf
