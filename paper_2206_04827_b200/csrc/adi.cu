// Batched ADI Sylvester solver for the per-Fourier-mode Poisson / Helmholtz
// problems of the CCF method (reference: proj/src/adi.cpp:150-202 driven by
// proj/src/solvers.cpp:77-98, proj/src/solvers.cpp:142-169 and
// proj/src/timestep.cpp:61-108).
//
// One CTA owns one real sub-problem (Fourier slot, k-parity, Re/Im plane): the
// reference's complex (m-2)x(n-2) modal system splits exactly into four real
// ((m-2)/2)x((n-2)/2) systems because every operator has even band offsets and
// real entries. The iterate stays resident in shared memory for all J
// iterations. Per-shift banded factors and the constant E' are streamed into
// shared memory with TMA bulk copies (cp.async.bulk + mbarrier) overlapped with
// the opposite sweep.
//
// Iteration (algebraically identical to the reference's two half steps
//   (vC - A) X' B = C X (vB + D) - E ;  C X'' (uB + D) = (uC - A) X' B + E,
// eliminating E from the second half step), with the state G_j = X_j (v_j B + D):
//   W_j     = (v_j C - A)^-1 [ (u_j C - A) G_j - (u_j - v_j) E ]      column sweep
//   X_{j+1} = W_j (u_j B + D)^-1 ;  G_{j+1} = X_{j+1} (v_{j+1} B + D)   row sweep
// so each iteration costs one banded multiply + one banded solve per side and no
// inverse of B or C at all. (A variant carrying Y = G B^-1 with E B^-1 precomputed
// loses ~50x in attainable residual through cond(B) ~ n^2; this form reaches
// ~4e-16 on the w = 0, 256^2 Poisson block where the reference plateaus near 5e-13.)
// The relative Frobenius residual ||A X B + C X D - E|| / ||E|| is evaluated on
// chip after every round of J iterations (adi.cpp:188-192); the round logic
// (<= 4 rounds, accept <= tol, fail > 10 tol) lives in adi_round_check.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace ccf {

namespace {

constexpr int kChunk = 8;  // E' rows per bulk chunk

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

__device__ __forceinline__ void swap2(double& a, double& b) {
    const double t = a;
    a = b;
    b = t;
}
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// Column multiply (no solve): out_a = sum_{d=-2..3} c[a][d] y[a+d] + alpha * e[a]
// in place over rows 0..M-1 of column `col` (stride pitch). Optional second
// multiplier writes q (global). Used once per round (prologue / residual).
__device__ __forceinline__ void col_mul(double* __restrict__ col, int pitch, int M, const double* __restrict__ cf,
                                        int cstride, int coff, const double* __restrict__ e, long estride, double alpha,
                                        int coff2, double* __restrict__ q, long qstride) {
    double ym2 = 0.0, ym1 = 0.0, y0 = col[0], y1 = col[pitch], y2 = col[2 * pitch], y3 = col[3 * pitch];
    for (int a = 0; a < M; ++a) {
        const double* c = cf + a * cstride + coff;
        double acc = fma(c[0], ym2, c[1] * ym1) + fma(c[2], y0, c[3] * y1) + fma(c[4], y2, c[5] * y3);
        if (e) acc = fma(alpha, e[a * estride], acc);
        if (q) {
            const double* c2 = cf + a * cstride + coff2;
            q[a * qstride] = fma(c2[0], ym2, c2[1] * ym1) + fma(c2[2], y0, c2[3] * y1) + fma(c2[4], y2, c2[5] * y3);
        }
        const double ynext = col[(a + 4) * pitch];
        col[a * pitch] = acc;
        ym2 = ym1;
        ym1 = y0;
        y0 = y1;
        y1 = y2;
        y2 = y3;
        y3 = ynext;
    }
}

// Row multiply + banded solve (right operators, transposed form, kl = 1):
//   y = LU^-1 ( MUL z ), in place over b in [0,N).
// mul: 4 coefficients at offsets -1..2 (stride ms); lu fields (stride ls):
//   [L | piv | inv | 0 | Uf0 Uf1 Uf2 | 0]  (Uf2 = 0 without pivoting).
template <bool PIV, bool SQ>
__device__ __forceinline__ double row_solve(double* __restrict__ row, int N, const double* __restrict__ mul, int ms,
                                            const double* __restrict__ lu, int ls, double* __restrict__ keep = nullptr) {
    double s0 = row[0], s1 = row[1], s2 = row[2], s3 = row[3];
    double2 m01 = ld2(mul), m23 = ld2(mul + 2);
    double x0 = fma(m01.y, s0, m23.x * s1) + m23.y * s2;
    double sq = x0 * x0;
    if (keep) keep[0] = x0;
    for (int k = 0; k < N; ++k) {
        double x1 = 0.0;
        if (k + 1 < N) {
            m01 = ld2(mul + (k + 1) * ms);
            m23 = ld2(mul + (k + 1) * ms + 2);
            x1 = fma(m01.x, s0, m01.y * s1) + fma(m23.x, s2, m23.y * s3);
            if (SQ) sq = fma(x1, x1, sq);
            if (keep) keep[k + 1] = x1;
        }
        const double2 lp = ld2(lu + k * ls);
        if (PIV && lp.y == 1.0) swap2(x0, x1);
        x1 = fma(-lp.x, x0, x1);
        const double snext = row[k + 4];
        row[k] = x0;
        x0 = x1;
        s0 = s1;
        s1 = s2;
        s2 = s3;
        s3 = snext;
    }
    double xa = 0.0, xb = 0.0, xc = 0.0;
    for (int k = N - 1; k >= 0; --k) {
        const double* c = lu + k * ls;
        const double2 iv = ld2(c + 2);
        const double2 u01 = ld2(c + 4);
        double acc = fma(-u01.y, xb, row[k] * iv.x);
        if (PIV) acc = fma(-c[6], xc, acc);
        acc = fma(-u01.x, xa, acc);
        row[k] = acc;
        xc = xb;
        xb = xa;
        xa = acc;
    }
    return SQ ? sq : 0.0;
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < int(blockDim.x >> 5); ++i) s += red[i];
    return s;
}

// Column sweep of one iteration (all threads participate; lanes b >= N shadow column
// N-1 and never store):
//   z = (vC - A)^-1 [ (uC - A) y + alpha e' ]        kl = 2 (ku = 3 without pivoting)
// left coefficients cf (shared, stride 16, Mpad+2 rows, zero-padded):
//   [mul -2..3 | L0 L1 | inv | piv | Uf0..4 | 0]
// e' streams through a 3-deep ring of kChunk-row shared buffers (TMA bulk copies);
// block barriers only between chunks, the 8 steps of a chunk are fully unrolled.
template <bool PIV>
__device__ __forceinline__ void col_phase(double* __restrict__ Y, int pitch, int Mpad, int N,
                                          const double* __restrict__ cf, double alpha, const double* __restrict__ eg,
                                          double* __restrict__ ebuf, uint64_t* ebar, int iter) {
    const int tid = threadIdx.x;
    // lanes >= N shadow column N-1 (valid reads, predicated-off stores)
    const bool act = tid < N;
    const int b = act ? tid : N - 1;
    double* __restrict__ col = Y + b;
    const int nch = Mpad / kChunk;
    const unsigned cbytes = unsigned(kChunk) * N * sizeof(double);
    const long cstride = long(kChunk) * N;
    // parity of the q-th use of barrier q%3 in column phase `iter`
    auto ewait = [&](int q) {
        const int bb = q % 3;
        const int uses = (nch - bb + 2) / 3;
        mbar_wait(&ebar[bb], unsigned(iter * uses + q / 3) & 1u);
    };
    if (tid == 0)
        for (int q = 0; q < 3 && q < nch; ++q) bulk_load(ebuf + q * cstride, eg + q * cstride, cbytes, &ebar[q]);
    ewait(0);
    const double* ecur = ebuf + b;  // chunk c of e' (column b)
    auto rrow = [&](const double* c, double e, double y0, double y1, double y2, double y3, double y4, double y5) {
        const double2 c01 = ld2(c), c23 = ld2(c + 2), c45 = ld2(c + 4);
        const double t0 = fma(c23.x, y2, fma(c01.y, y1, c01.x * y0));
        const double t1 = fma(c45.y, y5, fma(c45.x, y4, fma(c23.y, y3, alpha * e)));
        return t0 + t1;
    };
    double R0 = 0.0, R1 = 0.0, R2 = col[0], R3 = col[pitch], R4 = col[2 * pitch], R5 = col[3 * pitch];
    double x0 = rrow(cf, ecur[0], R0, R1, R2, R3, R4, R5);
    R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = col[4 * pitch];
    double x1 = rrow(cf + kLeftW, ecur[N], R0, R1, R2, R3, R4, R5);
    R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = col[5 * pitch];  // ring = y[0..5]
    for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) ewait(c + 1);
        const double* enext = ebuf + ((c + 1) % 3) * cstride + b;
        const double* cfc = cf + c * kChunk * kLeftW;
        double* colc = col + c * kChunk * pitch;
#pragma unroll
        for (int q = 0; q < kChunk; ++q) {
            const double e2 = (q + 2 < kChunk) ? ecur[(q + 2) * N] : enext[(q + 2 - kChunk) * N];
            double x2 = rrow(cfc + (q + 2) * kLeftW, e2, R0, R1, R2, R3, R4, R5);
            const double* cc = cfc + q * kLeftW;
            const double2 l01 = ld2(cc + 6);
            if (PIV) {
                const double pv = cc[9];
                if (pv == 1.0) swap2(x0, x1);
                else if (pv == 2.0) swap2(x0, x2);
            }
            x1 = fma(-l01.x, x0, x1);
            x2 = fma(-l01.y, x0, x2);
            const double ynext = colc[(q + 6) * pitch];
            if (act) colc[q * pitch] = x0;
            x0 = x1;
            x1 = x2;
            R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = ynext;
        }
        ecur = enext;
        __syncthreads();  // chunk c of e' fully consumed
        if (tid == 0 && c + 3 < nch)
            bulk_load(ebuf + ((c + 3) % 3) * cstride, eg + long(c + 3) * cstride, cbytes, &ebar[(c + 3) % 3]);
    }
    double xa = 0.0, xb = 0.0, xc = 0.0, xd = 0.0, xe = 0.0;
    for (int c = nch - 1; c >= 0; --c) {
#pragma unroll
        for (int q = kChunk - 1; q >= 0; --q) {
            const int k = c * kChunk + q;
            const double* cc = cf + k * kLeftW;
            const double2 iv = ld2(cc + 8);
            const double2 u01 = ld2(cc + 10);
            const double2 u23 = ld2(cc + 12);
            double acc = fma(-u23.x, xc, col[k * pitch] * iv.x);
            acc = fma(-u01.y, xb, acc);
            if (PIV) acc = fma(-u23.y, xd, fma(-cc[14], xe, acc));
            acc = fma(-u01.x, xa, acc);
            if (act) col[k * pitch] = acc;
            xe = xd;
            xd = xc;
            xc = xb;
            xb = xa;
            xa = acc;
        }
    }
}

// Row sweep of one iteration, thread per row a (< M), columns padded to Npad:
//   x = w (uB + D)^-1   (forward L, backward U; kl = 1, ku = 2 without pivoting)
//   g = x (v'B + D)     (fused into the backward sweep; identity on the last shift -> X)
// right coefficients (shared, stride 12, Npad+2 rows): [mul -1..2 | L | piv | inv | 0 | Uf0..2 | 0]
template <bool PIV>
__device__ __forceinline__ void row_phase(double* __restrict__ row, int Npad, const double* __restrict__ cr) {
    const int nch = Npad / kChunk;
    double x0 = row[0];
    for (int c = 0; c < nch; ++c) {
#pragma unroll
        for (int q = 0; q < kChunk; ++q) {
            const int k = c * kChunk + q;
            double x1 = row[k + 1];
            const double2 lp = ld2(cr + k * kRightW + 4);
            if (PIV && lp.y == 1.0) swap2(x0, x1);
            x1 = fma(-lp.x, x0, x1);
            row[k] = x0;
            x0 = x1;
        }
    }
    double xa = 0.0, xb = 0.0, xc = 0.0;  // x[k+1], x[k+2], x[k+3]
    for (int c = nch - 1; c >= 0; --c) {
#pragma unroll
        for (int q = kChunk - 1; q >= 0; --q) {
            const int k = c * kChunk + q;
            const double* cc = cr + k * kRightW;
            const double2 iv = ld2(cc + 6);
            const double2 u01 = ld2(cc + 8);
            double acc = fma(-u01.y, xb, row[k] * iv.x);
            if (PIV) acc = fma(-cc[10], xc, acc);
            acc = fma(-u01.x, xa, acc);
            // g_{k+1} = m(-1) x[k] + m(0) x[k+1] + m(1) x[k+2] + m(2) x[k+3]
            const double2 m01 = ld2(cc + kRightW), m23 = ld2(cc + kRightW + 2);
            row[k + 1] = fma(m01.x, acc, m01.y * xa) + fma(m23.x, xb, m23.y * xc);
            xc = xb;
            xb = xa;
            xa = acc;
        }
    }
    const double2 m01 = ld2(cr), m23 = ld2(cr + 2);
    row[0] = fma(m01.y, xa, m23.x * xb) + m23.y * xc;
}

// Row multiply in place: z_b <- sum_{d=-1..2} mul[b][d] z[b+d] over b in [0,N); returns sum z_b^2 if SQ.
template <bool SQ>
__device__ __forceinline__ double row_mul(double* __restrict__ row, int N, const double* __restrict__ mul, int ms) {
    double zm1 = 0.0, z0 = row[0], z1 = row[1], z2 = row[2];
    double sq = 0.0;
    for (int b = 0; b < N; ++b) {
        const double2 m01 = ld2(mul + b * ms), m23 = ld2(mul + b * ms + 2);
        const double e = fma(m01.x, zm1, m01.y * z0) + fma(m23.x, z1, m23.y * z2);
        if (SQ) sq = fma(e, e, sq);
        const double znext = row[b + 3];
        row[b] = e;
        zm1 = z0;
        z0 = z1;
        z1 = z2;
        z2 = znext;
    }
    return sq;
}

// ---------------------------------------------------------------------------------------------
// Two-way partitioned sweeps (SPIKE) for unpivoted slots: 2 x lanes threads, thread
// (half, lt). Each banded solve along a line of the tile is split at row / column h;
// both halves run their local recurrences concurrently and the coupling is restored
// with the precomputed spike vectors (modal.cpp, add_left_spikes / add_right_spikes):
//   forward : the lower half starts from zero coupling, x_k = x'_k + F . (boundary x of
//             the upper half), applied on the fly in its backward sweep
//   backward: the upper half starts from zero boundary, z_k = z'_k + G . (z_h, z_h+1, ..)
//             applied in a short parallel fix-up pass.
// This doubles the independent recurrences per SM (the single-CTA tile admits only one
// thread per line otherwise) at ~1.25 sweeps of sequential work per thread instead of 2.

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Column sweep, split at row hc (multiple of kChunk). xch: 2 x lanes doubles.
__device__ __forceinline__ void col_phase_spike(double* __restrict__ Y, int pitch, int Mpad, int N,
                                                const double* __restrict__ cf, double alpha,
                                                const double* __restrict__ eg, double* __restrict__ ebuf,
                                                uint64_t* ebar, int iter, int hc, int lanes, double* xch) {
    const int tid = threadIdx.x;
    const int half = tid >= lanes ? 1 : 0;
    const int lt = tid - half * lanes;
    const bool act = lt < N;
    const int b = act ? lt : N - 1;
    double* __restrict__ col = Y + b;
    const int r0 = half ? hc : 0;
    const int c0 = r0 / kChunk, nchR = (half ? Mpad - hc : hc) / kChunk;
    const unsigned cbytes = unsigned(kChunk) * N * sizeof(double);
    const long cstride = long(kChunk) * N;
    double* ring = ebuf + half * 3 * cstride;
    uint64_t* bars = ebar + half * 3;
    const double* egR = eg + long(c0) * cstride;
    auto ewait = [&](int q) {
        const int bb = q % 3;
        const int uses = (nchR - bb + 2) / 3;
        mbar_wait(&bars[bb], unsigned(iter * uses + q / 3) & 1u);
    };
    if (lt == 0)
        for (int q = 0; q < 3 && q < nchR; ++q) bulk_load(ring + q * cstride, egR + q * cstride, cbytes, &bars[q]);
    // window y[r0-2 .. r0+5] and the upper half's halo y[hc .. hc+2], read before anyone stores
    double R0 = half ? col[(r0 - 2) * pitch] : 0.0, R1 = half ? col[(r0 - 1) * pitch] : 0.0;
    double R2 = col[r0 * pitch], R3 = col[(r0 + 1) * pitch], R4 = col[(r0 + 2) * pitch], R5 = col[(r0 + 3) * pitch];
    const double R6 = col[(r0 + 4) * pitch], R7 = col[(r0 + 5) * pitch];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (!half) {
        s0 = col[hc * pitch];
        s1 = col[(hc + 1) * pitch];
        s2 = col[(hc + 2) * pitch];
    }
    __syncthreads();
    auto rrow = [&](const double* c, double e, double y0, double y1, double y2, double y3, double y4, double y5) {
        const double2 c01 = ld2(c), c23 = ld2(c + 2), c45 = ld2(c + 4);
        const double t0 = fma(c23.x, y2, fma(c01.y, y1, c01.x * y0));
        const double t1 = fma(c45.y, y5, fma(c45.x, y4, fma(c23.y, y3, alpha * e)));
        return t0 + t1;
    };
    ewait(0);
    const double* ecur = ring + b;
    double x0 = rrow(cf + r0 * kLeftW, ecur[0], R0, R1, R2, R3, R4, R5);
    R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = R6;
    double x1 = rrow(cf + (r0 + 1) * kLeftW, ecur[N], R0, R1, R2, R3, R4, R5);
    R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = R7;
    auto chunk = [&]<bool HALO>(int gc, const double* enext) {
        const double* cfc = cf + gc * kChunk * kLeftW;
        double* colc = col + gc * kChunk * pitch;
#pragma unroll
        for (int q = 0; q < kChunk; ++q) {
            const double e2 = (q + 2 < kChunk) ? ecur[(q + 2) * N] : enext[(q + 2 - kChunk) * N];
            double x2 = rrow(cfc + (q + 2) * kLeftW, e2, R0, R1, R2, R3, R4, R5);
            const double2 l01 = ld2(cfc + q * kLeftW + 6);
            x1 = fma(-l01.x, x0, x1);
            x2 = fma(-l01.y, x0, x2);
            double ynext;
            if (HALO && q >= 2) ynext = (q == 2) ? s0 : (q == 3) ? s1 : (q == 4) ? s2 : 0.0;
            else ynext = colc[(q + 6) * pitch];
            if (act) colc[q * pitch] = x0;
            x0 = x1;
            x1 = x2;
            R0 = R1; R1 = R2; R2 = R3; R3 = R4; R4 = R5; R5 = ynext;
        }
    };
    for (int c = 0; c < nchR; ++c) {
        const bool more = c + 1 < nchR;
        if (more) ewait(c + 1);
        const double* enext = more ? ring + ((c + 1) % 3) * cstride + b : ecur;
        if (!half && !more) chunk.template operator()<true>(c0 + c, enext);
        else chunk.template operator()<false>(c0 + c, enext);
        ecur = enext;
        named_sync(1 + half, lanes);  // chunk c of this half's e' ring fully consumed
        if (lt == 0 && c + 3 < nchR)
            bulk_load(ring + ((c + 3) % 3) * cstride, egR + long(c + 3) * cstride, cbytes, &bars[(c + 3) % 3]);
    }
    if (!half) {  // boundary of the upper half for the lower half's correction
        xch[lt] = col[(hc - 1) * pitch];
        xch[lanes + lt] = col[(hc - 2) * pitch];
    }
    __syncthreads();
    if (half) {
        const double X1 = xch[lt], X2 = xch[lanes + lt];
        double xa = 0.0, xb = 0.0, xc = 0.0;
        for (int c = Mpad / kChunk - 1; c >= c0; --c) {
#pragma unroll
            for (int q = kChunk - 1; q >= 0; --q) {
                const int k = c * kChunk + q;
                const double* cc = cf + k * kLeftW;
                const double2 iv = ld2(cc + 8);
                const double2 u01 = ld2(cc + 10);
                const double2 u23 = ld2(cc + 12);  // (Uf2, F1)
                const double2 f2 = ld2(cc + 14);   // (F2, -)
                const double x = fma(u23.y, X1, fma(f2.x, X2, col[k * pitch]));
                double acc = fma(-u23.x, xc, x * iv.x);
                acc = fma(-u01.y, xb, acc);
                acc = fma(-u01.x, xa, acc);
                if (act) col[k * pitch] = acc;
                xc = xb;
                xb = xa;
                xa = acc;
            }
        }
    } else {
        double xa = 0.0, xb = 0.0, xc = 0.0;
        for (int c = hc / kChunk - 1; c >= 0; --c) {
#pragma unroll
            for (int q = kChunk - 1; q >= 0; --q) {
                const int k = c * kChunk + q;
                const double* cc = cf + k * kLeftW;
                const double2 iv = ld2(cc + 8);
                const double2 u01 = ld2(cc + 10);
                const double u2 = cc[12];
                double acc = fma(-u2, xc, col[k * pitch] * iv.x);
                acc = fma(-u01.y, xb, acc);
                acc = fma(-u01.x, xa, acc);
                if (act) col[k * pitch] = acc;
                xc = xb;
                xb = xa;
                xa = acc;
            }
        }
    }
    __syncthreads();
    if (act) {  // fix-up of the upper half: rows [half * hc/2, (half+1) * hc/2)
        const double Z0 = col[hc * pitch], Z1 = col[(hc + 1) * pitch], Z2 = col[(hc + 2) * pitch];
        const int hh = hc / 2;
        for (int k = half * hh; k < (half + 1) * hh; ++k) {
            const double* cc = cf + k * kLeftW;
            const double g1 = cc[13];
            const double2 g23 = ld2(cc + 14);
            col[k * pitch] = fma(g1, Z0, fma(g23.x, Z1, fma(g23.y, Z2, col[k * pitch])));
        }
    }
}

// Row sweep (+ fused G multiply), split at column hr (multiple of kChunk). rch: 4 x lanes doubles.
__device__ __forceinline__ void row_phase_spike(double* __restrict__ Y, int pitch, int M, int Npad,
                                                const double* __restrict__ cr, int hr, int lanes, double* rch) {
    const int tid = threadIdx.x;
    const int half = tid >= lanes ? 1 : 0;
    const int lt = tid - half * lanes;
    const bool act = lt < M;
    double* __restrict__ row = Y + (act ? lt : 0) * pitch;
    if (act) {
        const int ca = half ? hr / kChunk : 0, cb = half ? Npad / kChunk : hr / kChunk;
        double x0 = row[ca * kChunk];
        for (int c = ca; c < cb; ++c) {
#pragma unroll
            for (int q = 0; q < kChunk; ++q) {
                const int k = c * kChunk + q;
                double x1 = row[k + 1];
                x1 = fma(-cr[k * kRightW + 4], x0, x1);
                row[k] = x0;
                x0 = x1;
            }
        }
        if (!half) rch[lt] = row[hr - 1];
    }
    __syncthreads();
    double gh = 0.0;  // upper half: g'_hr (row[hr] is still read by the lower half)
    if (act) {
        if (half) {
            const double X = rch[lt];
            double xa = 0.0, xb = 0.0, xc = 0.0;  // z[k+1], z[k+2], z[k+3]
            for (int c = Npad / kChunk - 1; c >= hr / kChunk; --c) {
#pragma unroll
                for (int q = kChunk - 1; q >= 0; --q) {
                    const int k = c * kChunk + q;
                    const double* cc = cr + k * kRightW;
                    const double2 iv = ld2(cc + 6);
                    const double2 u01 = ld2(cc + 8);
                    const double x = fma(cc[5], X, row[k]);
                    double acc = fma(-u01.y, xb, x * iv.x);
                    acc = fma(-u01.x, xa, acc);
                    const double2 m01 = ld2(cc + kRightW), m23 = ld2(cc + kRightW + 2);
                    row[k + 1] = fma(m01.x, acc, m01.y * xa) + fma(m23.x, xb, m23.y * xc);
                    xc = xb;
                    xb = xa;
                    xa = acc;
                }
            }
            rch[lanes + lt] = xa;
            rch[2 * lanes + lt] = xb;
            rch[3 * lanes + lt] = xc;
        } else {
            double xa = 0.0, xb = 0.0, xc = 0.0;
            for (int c = hr / kChunk - 1; c >= 0; --c) {
#pragma unroll
                for (int q = kChunk - 1; q >= 0; --q) {
                    const int k = c * kChunk + q;
                    const double* cc = cr + k * kRightW;
                    const double inv = cc[6];
                    const double2 u01 = ld2(cc + 8);
                    double acc = fma(-u01.y, xb, row[k] * inv);
                    acc = fma(-u01.x, xa, acc);
                    const double2 m01 = ld2(cc + kRightW), m23 = ld2(cc + kRightW + 2);
                    const double gn = fma(m01.x, acc, m01.y * xa) + fma(m23.x, xb, m23.y * xc);
                    if (k + 1 < hr) row[k + 1] = gn;
                    else gh = gn;
                    xc = xb;
                    xb = xa;
                    xa = acc;
                }
            }
            const double2 m01 = ld2(cr), m23 = ld2(cr + 2);
            row[0] = fma(m01.y, xa, m23.x * xb) + m23.y * xc;
        }
    }
    __syncthreads();
    if (act) {  // g = g' + H1 z_hr + H2 z_hr+1 (+ H3 z_hr+2 at hr): half 0 -> [0, hh) + {hr}, half 1 -> [hh, hr)
        const double Zh = rch[lanes + lt], Zh1 = rch[2 * lanes + lt];
        const int hh = hr / 2;
        for (int k = half * hh; k < (half + 1) * hh; ++k) {
            const double2 h12 = ld2(cr + k * kRightW + 10);
            row[k] = fma(h12.x, Zh, fma(h12.y, Zh1, row[k]));
        }
        if (!half) {
            const double* cc = cr + hr * kRightW;
            const double2 h12 = ld2(cc + 10);
            row[hr] = fma(h12.x, Zh, fma(h12.y, Zh1, fma(cc[7], rch[3 * lanes + lt], gh)));
        }
    }
}

// In-place banded column multiply (prologue R2 f, residual A X / C X), rows split at h:
//   out_a = sum_{d=-2..3} c[a][d] y[a+d] (+ second multiplier into q), a in [0, M).
__device__ __forceinline__ void col_mul_split(double* __restrict__ Y, int pitch, int M, int ncols,
                                              const double* __restrict__ cf, int cstride, int coff, int coff2,
                                              double* __restrict__ q, long qstride, int h, int lanes) {
    const int tid = threadIdx.x;
    const int half = tid >= lanes ? 1 : 0;
    const int lt = tid - half * lanes;
    const bool act = lt < ncols;
    double* col = Y + (act ? lt : 0);
    double h0 = 0.0, h1 = 0.0, h2 = 0.0;
    if (act) {
        if (!half) {
            h0 = col[h * pitch];
            h1 = col[(h + 1) * pitch];
            h2 = col[(h + 2) * pitch];
        } else {
            h0 = col[(h - 2) * pitch];
            h1 = col[(h - 1) * pitch];
        }
    }
    __syncthreads();
    if (!act) return;
    auto ld = [&](int j) {
        if (!half && j >= h) return j == h ? h0 : (j == h + 1 ? h1 : (j == h + 2 ? h2 : 0.0));
        return col[j * pitch];
    };
    const int a0 = half ? h : 0, a1 = half ? M : h;
    double ym2 = half ? h0 : 0.0, ym1 = half ? h1 : 0.0;
    double y0 = ld(a0), y1 = ld(a0 + 1), y2 = ld(a0 + 2), y3 = ld(a0 + 3);
    for (int a = a0; a < a1; ++a) {
        const double* c = cf + a * cstride + coff;
        const double acc = fma(c[0], ym2, c[1] * ym1) + fma(c[2], y0, c[3] * y1) + fma(c[4], y2, c[5] * y3);
        if (q) {
            const double* c2 = cf + a * cstride + coff2;
            q[a * qstride + lt] =
                fma(c2[0], ym2, c2[1] * ym1) + fma(c2[2], y0, c2[3] * y1) + fma(c2[4], y2, c2[5] * y3);
        }
        const double ynext = ld(a + 4);
        col[a * pitch] = acc;
        ym2 = ym1;
        ym1 = y0;
        y0 = y1;
        y1 = y2;
        y2 = y3;
        y3 = ynext;
    }
}

// In-place banded row multiply z_b <- sum_{d=-1..2} mul[b][d] z[b+d], b in [0, N), columns
// split at h; rows a in [0, M). Returns the thread's sum of squares of the outputs if SQ.
template <bool SQ>
__device__ __forceinline__ double row_mul_split(double* __restrict__ Y, int pitch, int M, int N,
                                                const double* __restrict__ mul, int ms, int h, int lanes) {
    const int tid = threadIdx.x;
    const int half = tid >= lanes ? 1 : 0;
    const int lt = tid - half * lanes;
    const bool act = lt < M;
    double* row = Y + (act ? lt : 0) * pitch;
    double h0 = 0.0, h1 = 0.0;
    if (act) {
        if (!half) {
            h0 = row[h];
            h1 = row[h + 1];
        } else {
            h0 = row[h - 1];
        }
    }
    __syncthreads();
    if (!act) return 0.0;
    auto ld = [&](int j) {
        if (!half && j >= h) return j == h ? h0 : (j == h + 1 ? h1 : 0.0);
        return row[j];
    };
    const int b0 = half ? h : 0, b1 = half ? N : h;
    double zm1 = half ? h0 : 0.0, z0 = ld(b0), z1 = ld(b0 + 1), z2 = ld(b0 + 2);
    double sq = 0.0;
    for (int b = b0; b < b1; ++b) {
        const double2 m01 = ld2(mul + b * ms), m23 = ld2(mul + b * ms + 2);
        const double e = fma(m01.x, zm1, m01.y * z0) + fma(m23.x, z1, m23.y * z2);
        if (SQ) sq = fma(e, e, sq);
        const double znext = ld(b + 3);
        row[b] = e;
        zm1 = z0;
        z0 = z1;
        z1 = z2;
        z2 = znext;
    }
    return sq;
}

// ---------------------------------------------------------------------------------------------
// Once-per-round passes, thread per column b (coalesced global access, coefficients of the right
// operators in registers), rows split between the line sets when 2 x lanes threads run. Both are
// read-only on the tile (sliding windows along the rows), so no halo exchange is needed.

// E = (R2 f C02^T) restricted to M x N -> escr (rows >= M zero); returns the thread's sum of E^2.
// f: rows [0, mh) x columns [0, nh) of the tile; sleft fields 0..5 = R2 (d = -2..3), sright 0..3 = C02.
__device__ __forceinline__ double prologue_E(const double* __restrict__ Y, int pitch, int M, int N, int Mpad,
                                            const double* __restrict__ sleft, const double* __restrict__ sright,
                                            double* __restrict__ escr, int r0, int r1, int b) {
    const double2 c01 = ld2(sright + b * kStatW), c23 = ld2(sright + b * kStatW + 2);
    const double* col = Y + b;
    const bool left = b > 0;
    auto H = [&](int i) -> double {  // (f C02^T)[i][b]
        if (i < 0) return 0.0;
        const double* r = col + i * pitch;
        return fma(c01.x, left ? r[-1] : 0.0, c01.y * r[0]) + fma(c23.x, r[1], c23.y * r[2]);
    };
    double h0 = H(r0 - 2), h1 = H(r0 - 1), h2 = H(r0), h3 = H(r0 + 1), h4 = H(r0 + 2);
    double esq = 0.0;
    for (int a = r0; a < r1; ++a) {
        const double h5 = H(a + 3);
        const double* c = sleft + a * kStatW;
        const double2 r01 = ld2(c), r23 = ld2(c + 2), r45 = ld2(c + 4);
        const double e = (fma(r01.x, h0, r01.y * h1) + fma(r23.x, h2, r23.y * h3)) + fma(r45.x, h4, r45.y * h5);
        escr[a * N + b] = e;
        esq = fma(e, e, esq);
        h0 = h1;
        h1 = h2;
        h2 = h3;
        h3 = h4;
        h4 = h5;
    }
    return esq;
}

// Residual of the Sylvester equation R = A X B + C X D - E (adi.cpp:106-112) as A (X B) + C (X D) - E;
// returns the thread's sum of R^2 over rows [r0, r1) of column b.
__device__ __forceinline__ double residual_col(const double* __restrict__ Y, int pitch, int N,
                                              const double* __restrict__ sleft, const double* __restrict__ sright,
                                              const double* __restrict__ escr, int r0, int r1, int b) {
    const double* cb = sright + b * kStatW;
    const double2 b01 = ld2(cb + 12), b23 = ld2(cb + 14), d01 = ld2(cb + 16), d23 = ld2(cb + 18);
    const double* col = Y + b;
    const bool left = b > 0;
    double xb[6], xd[6];
    auto XBD = [&](int i, double& ob, double& od) {
        if (i < 0) {
            ob = od = 0.0;
            return;
        }
        const double* r = col + i * pitch;
        const double xm = left ? r[-1] : 0.0, x0 = r[0], x1 = r[1], x2 = r[2];
        ob = fma(b01.x, xm, b01.y * x0) + fma(b23.x, x1, b23.y * x2);
        od = fma(d01.x, xm, d01.y * x0) + fma(d23.x, x1, d23.y * x2);
    };
#pragma unroll
    for (int d = 0; d < 5; ++d) XBD(r0 - 2 + d, xb[d], xd[d]);
    double rsq = 0.0;
    for (int a = r0; a < r1; ++a) {
        XBD(a + 3, xb[5], xd[5]);
        const double* c = sleft + a * kStatW;
        const double2 a01 = ld2(c + 6), a23 = ld2(c + 8), a45 = ld2(c + 10);
        const double2 e01 = ld2(c + 12), e23 = ld2(c + 14), e45 = ld2(c + 16);
        const double ra = (fma(a01.x, xb[0], a01.y * xb[1]) + fma(a23.x, xb[2], a23.y * xb[3])) +
                          fma(a45.x, xb[4], a45.y * xb[5]);
        const double rc = (fma(e01.x, xd[0], e01.y * xd[1]) + fma(e23.x, xd[2], e23.y * xd[3])) +
                          fma(e45.x, xd[4], e45.y * xd[5]);
        const double r = (ra + rc) - escr[a * N + b];
        rsq = fma(r, r, rsq);
#pragma unroll
        for (int d = 0; d < 5; ++d) {
            xb[d] = xb[d + 1];
            xd[d] = xd[d + 1];
        }
    }
    return rsq;
}

}  // namespace

// Shared-memory tile: rows [0, Mpad+6) x pitch (pitch >= nh+3, odd), followed by the
// left / right coefficient stages, the e' chunk rings (one per half when split) and the
// spike exchange slots (4 x lanes).
// SPLIT: unpivoted slot with 2 x lanes threads (partitioned sweeps); otherwise the
// sequential sweeps (any thread count, lanes >= N shadow).
// TM, TN > 0: sizes fixed at compile time (M = TM, N = TN, pitch = (Npad + 4) | 1, as
// Ctx computes them) so every tile / coefficient offset folds into an immediate.
template <bool PIV, bool SPLIT, int TM, int TN>
__device__ __forceinline__ void adi_body(const AdiParams& P, const AdiTask& task, const AdiSlot& so, double* sm,
                                         uint64_t* bars, double* red) {
    const int t = task.tensor, s = task.slot, k0 = task.k0, plane = task.plane;
    const Geo& g = P.g;
    constexpr bool FIX = TM > 0 && TN > 0;
    const int M = FIX ? TM : P.M, N = FIX ? TN : P.N;
    const int Mpad = FIX ? ((TM + 7) / 8) * 8 : P.Mpad, Npad = FIX ? ((TN + 7) / 8) * 8 : P.Npad;
    const int pitch = FIX ? ((((TN + 7) / 8) * 8 + 4) | 1) : P.pitch;
    const int mh = M + 1, nh = N + 1;
    const int lrows = Mpad + 2, rrows = Npad + 2;
    const int tid = threadIdx.x, nt = FIX ? (SPLIT ? 2 : 1) * ((((TM > TN ? TM : TN) + 31) / 32) * 32) : blockDim.x;
    const int lanes = FIX ? ((((TM > TN ? TM : TN) + 31) / 32) * 32) : P.lanes;
    const int hc = FIX ? (SPLIT ? spike_split(Mpad) : 0) : P.hc, hr = FIX ? (SPLIT ? spike_split(Npad) : 0) : P.hr;
    const bool split_mul = FIX ? SPLIT : P.hc > 0;  // 2 x lanes threads: split the once-per-round multiplies too
    const int rows = Mpad + 6;
    double* Y = sm;
    const long ysize = ((long(rows) * pitch + 1) / 2) * 2;
    double* bufL = sm + ysize;
    double* bufR = bufL + long(lrows) * kLeftW;
    double* bufE = bufR + long(rrows) * kRightW;
    double* xch = bufE + (split_mul ? 6L : 3L) * kChunk * N;
    const long toff = long(s) * g.slot_stride + long(plane) * g.plane_stride;
    const double* sleft = P.coef + so.sleft;
    const double* sright = P.coef + (k0 ? so.sright1 : so.sright0);

    // ---- prologue: f (RHS assembly, fused BDF/IMEX combination) -> F = R2 f C02^T -> E
    for (int i = tid; i < rows * pitch; i += nt) Y[i] = 0.0;
    __syncthreads();
    {
        const int ns = P.nsrc[t];
        const double* const* src = P.src[t];
        const double* wv = P.wsrc[t];
        constexpr int U = 4;  // independent rows in flight per thread
        for (int i0 = tid; i0 < mh * nh; i0 += U * nt) {
            double acc[U];
            long off[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nt;
                const int a = i / nh, b = i - a * nh;
                off[u] = toff + long(a) * g.n + long(k0) * nh + b;
                acc[u] = 0.0;
            }
            for (int q = 0; q < ns; ++q) {
                const double* sq = src[q];
                const double wq = wv[q];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (i0 + u * nt < mh * nh) acc[u] = fma(wq, __ldg(sq + off[u]), acc[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nt;
                if (i < mh * nh) {
                    const int a = i / nh, b = i - a * nh;
                    Y[a * pitch + b] = acc[u];
                }
            }
        }
    }
    __syncthreads();
    double esq = 0.0;
    double* escr = P.escr + long(blockIdx.x) * P.estride;  // E (top-left block of R2 f C02^T), rows padded to Mpad
    double* xscr = P.xscr + long(blockIdx.x) * P.estride;  // X of the previous round (restart)
    {
        const int lh = split_mul ? (tid >= lanes ? 1 : 0) : 0;
        const int b = split_mul ? tid - lh * lanes : tid;
        const int r0 = split_mul ? (lh ? hc : 0) : 0, r1 = split_mul ? (lh ? M : hc) : M;
        if (b < N) esq = prologue_E(Y, pitch, M, N, Mpad, sleft, sright, escr, r0, r1, b);
        for (int i = M * N + tid; i < Mpad * N; i += nt) escr[i] = 0.0;
    }
    fence_proxy_async();  // E generic stores -> async-proxy (bulk copy) reads
    __syncthreads();
    for (int i = tid; i < rows * pitch; i += nt) Y[i] = 0.0;
    const double* left = P.coef + so.left;
    const double* right = P.coef + (k0 ? so.right1 : so.right0);
    const unsigned lbytes = unsigned(lrows) * kLeftW * sizeof(double);
    const unsigned rbytes = unsigned(rrows) * kRightW * sizeof(double);
    if (tid == 0) {
        bulk_load(bufL, left, lbytes, &bars[0]);
        bulk_load(bufR, right, rbytes, &bars[1]);
    }
    __syncthreads();

    if (P.round > 0) {
        // restart from the previous round's X (adi.cpp:163-187 continue the same iteration)
        for (int i = tid; i < M * N; i += nt) Y[(i / N) * pitch + (i % N)] = xscr[i];
        __syncthreads();
        if (split_mul) row_mul_split<false>(Y, pitch, M, N, sright + 20, kStatW, hr, lanes);  // G = X (v_0 B + D)
        else
            for (int a = tid; a < M; a += nt) row_mul<false>(Y + a * pitch, N, sright + 20, kStatW);
        __syncthreads();
    }

    // ---- J iterations, tile resident in shared memory
    const double* dsv = P.coef + so.ds;
    for (int j = 0; j < so.J; ++j) {
        const double alpha = -__ldg(dsv + j);
        mbar_wait(&bars[0], unsigned(j) & 1u);
        if (SPLIT) col_phase_spike(Y, pitch, Mpad, N, bufL, alpha, escr, bufE, bars + 2, j, hc, lanes, xch);
        else col_phase<PIV>(Y, pitch, Mpad, N, bufL, alpha, escr, bufE, bars + 2, j);
        __syncthreads();
        if (tid == 0 && j + 1 < so.J) bulk_load(bufL, left + long(j + 1) * lrows * kLeftW, lbytes, &bars[0]);
        mbar_wait(&bars[1], unsigned(j) & 1u);
        if (SPLIT) row_phase_spike(Y, pitch, M, Npad, bufR, hr, lanes, xch);
        else
            for (int a = tid; a < M; a += nt) row_phase<PIV>(Y + a * pitch, Npad, bufR);
        __syncthreads();
        if (tid == 0 && j + 1 < so.J) bulk_load(bufR, right + long(j + 1) * rrows * kRightW, rbytes, &bars[1]);
    }

    // ---- epilogue: u = S_r X S_z^T (Dirichlet recombination, solvers.cpp:97), parity-compressed store
    double* u = P.out[t];
    for (int i = tid; i < mh * nh; i += nt) {
        const int a = i / nh, b = i - a * nh;
        const double x00 = Y[a * pitch + b];
        const double x10 = a > 0 ? Y[(a - 1) * pitch + b] : 0.0;
        const double x01 = b > 0 ? Y[a * pitch + b - 1] : 0.0;
        const double x11 = (a > 0 && b > 0) ? Y[(a - 1) * pitch + b - 1] : 0.0;
        u[toff + long(a) * g.n + long(k0) * nh + b] = (x00 - x10) - (x01 - x11);
    }
    for (int i = tid; i < M * N; i += nt) xscr[i] = Y[(i / N) * pitch + (i % N)];
    __syncthreads();
    // ---- residual R = A X B + C X D - E (adi.cpp:106-112), read-only on the tile
    double rsq = 0.0;
    {
        const int lh = split_mul ? (tid >= lanes ? 1 : 0) : 0;
        const int b = split_mul ? tid - lh * lanes : tid;
        const int r0 = split_mul ? (lh ? hc : 0) : 0, r1 = split_mul ? (lh ? M : hc) : M;
        if (b < N) rsq = residual_col(Y, pitch, N, sleft, sright, escr, r0, r1, b);
    }
    const double rs = block_sum(rsq, red);
    const double es = block_sum(esq, red);
    if (tid == 0) {
        atomicAdd(P.res2 + t * g.nslots + s, rs);
        atomicAdd(P.e2 + t * g.nslots + s, es);
    }
}

template <int TM, int TN>
__global__ void __launch_bounds__((TM > 0 && TM <= 128 && TN <= 128) ? 256 : 512, 1) adi_kernel(const AdiParams P) {
    extern __shared__ __align__(16) double sm[];
    __shared__ uint64_t bars[8];
    __shared__ double red[16];
    const AdiTask task = P.tasks[blockIdx.x];
    if (!P.active[task.tensor * P.g.nslots + task.slot]) return;
    const AdiSlot so = P.slots[task.slot];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (so.pivot) adi_body<true, false, TM, TN>(P, task, so, sm, bars, red);
    else if (P.hc > 0) adi_body<false, true, TM, TN>(P, task, so, sm, bars, red);
    else adi_body<false, false, TM, TN>(P, task, so, sm, bars, red);
}

namespace {
// compile-time size classes: the n = m = 256 / 128 / 64 benchmark grids; anything else runs generic
using AdiFn = void (*)(const AdiParams);
struct AdiInst {
    int M, N;
    AdiFn fn;
};
const AdiInst kAdiInst[] = {{127, 127, adi_kernel<127, 127>}, {63, 63, adi_kernel<63, 63>},
                            {31, 31, adi_kernel<31, 31>}, {0, 0, adi_kernel<0, 0>}};
AdiFn adi_pick(int M, int N) {
    for (const AdiInst& k : kAdiInst)
        if ((k.M == M && k.N == N) || k.M == 0) return k.fn;
    return adi_kernel<0, 0>;
}
}  // namespace

size_t adi_static_smem() {
    size_t mx = 0;
    for (const AdiInst& k : kAdiInst) {
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, k.fn) == cudaSuccess) mx = mx > fa.sharedSizeBytes ? mx : fa.sharedSizeBytes;
    }
    return mx;
}

cudaError_t adi_set_smem(int bytes) {
    for (const AdiInst& k : kAdiInst) {
        const cudaError_t e = cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

void adi_launch(const AdiParams& P, int threads, size_t smem, cudaStream_t stream) {
    adi_pick(P.M, P.N)<<<P.ntasks, threads, smem, stream>>>(P);
}

__global__ void adi_init_kernel(int* active, double* res2, double* e2, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        active[i] = 1;
        res2[i] = 0.0;
        e2[i] = 0.0;
    }
}

// Round bookkeeping per (tensor, slot): accept <= tol, restart up to 4 rounds,
// fail > 10 tol after the last round (adi.cpp:163-200).
__global__ void adi_round_check(RoundCheck c) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.ntensor * c.nslots) return;
    if (!c.active[i]) return;
    const double e = c.e2[i];
    const double rel = e > 0.0 ? sqrt(c.res2[i] / e) : sqrt(c.res2[i]);
    c.history[i * 4 + c.round] = rel;
    c.rounds[i] = c.round + 1;
    atomicAdd(c.iters, (unsigned long long)(4 * c.J[i % c.nslots]));
    c.res2[i] = 0.0;
    c.e2[i] = 0.0;
    if (!(rel > c.tol)) {
        c.active[i] = 0;
        return;
    }
    if (c.round == 3) {
        c.active[i] = 0;
        if (!(rel <= 10.0 * c.tol)) {
            if (atomicCAS(c.err, 0, 4) == 0) {
                c.err[1] = i / c.nslots;
                c.err[2] = i % c.nslots;
            }
        }
    }
}

}  // namespace ccf
