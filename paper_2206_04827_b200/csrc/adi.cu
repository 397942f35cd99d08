// Batched ADI Sylvester solver for the per-Fourier-mode Poisson / Helmholtz
// problems of the CCF method (reference: proj/src/adi.cpp:150-202 driven by
// proj/src/solvers.cpp:77-98, proj/src/solvers.cpp:142-169 and
// proj/src/timestep.cpp:61-108).
//
// One CTA owns one real sub-problem (Fourier slot, k-parity, Re/Im plane): the
// reference's complex (m-2)x(n-2) modal system splits exactly into four real
// ((m-2)/2)x((n-2)/2) systems because every operator has even band offsets and
// real entries. The iterate stays resident in shared memory for all J
// iterations; only E' (L2-resident scratch) and the per-shift banded factors are
// read from global memory.
//
// Iteration (algebraically identical to the reference's two half steps, with
// Y_j = X_j (v_j B + D) B^-1 and E' = E B^-1):
//   Z_j     = (v_j C - A)^-1 [ (u_j C - A) Y_j - (u_j - v_j) E' ]      column sweep
//   Y_{j+1} = Z_j (v_{j+1} B + D) (u_j B + D)^-1                       row sweep
//   X_J     = Z_{J-1} B (u_{J-1} B + D)^-1
// so each iteration costs one banded multiply + one pivoted banded solve per side.
// The relative Frobenius residual ||A X B + C X D - E|| / ||E|| is evaluated on
// chip after every round of J iterations (adi.cpp:188-192); the round logic
// (<= 4 rounds, accept <= tol, fail > 10 tol) lives in adi_round_check.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ccf {

namespace {

__device__ __forceinline__ void swap2(double& a, double& b) {
    const double t = a;
    a = b;
    b = t;
}

// Column multiply (no solve): out_a = sum_{d=-2..3} c[a][d] y[a+d] + alpha * e[a]
// in place over rows 0..M-1 of column `col` (stride pitch). Rows >= M read as the
// zero padding of the tile. Optional second multiplier c2 writes to q (global).
__device__ __forceinline__ void col_mul(double* __restrict__ col, int pitch, int M, const double* __restrict__ cf,
                                        int cstride, int coff, const double* __restrict__ e, long estride, double alpha,
                                        int coff2, double* __restrict__ q, long qstride) {
    double ym2 = 0.0, ym1 = 0.0, y0 = col[0], y1 = col[pitch], y2 = col[2 * pitch], y3 = col[3 * pitch];
    for (int a = 0; a < M; ++a) {
        const double* c = cf + a * cstride + coff;
        double acc = c[0] * ym2;
        acc = fma(c[1], ym1, acc);
        acc = fma(c[2], y0, acc);
        acc = fma(c[3], y1, acc);
        acc = fma(c[4], y2, acc);
        acc = fma(c[5], y3, acc);
        if (e) acc = fma(alpha, e[a * estride], acc);
        if (q) {
            const double* c2 = cf + a * cstride + coff2;
            double a2 = c2[0] * ym2;
            a2 = fma(c2[1], ym1, a2);
            a2 = fma(c2[2], y0, a2);
            a2 = fma(c2[3], y1, a2);
            a2 = fma(c2[4], y2, a2);
            a2 = fma(c2[5], y3, a2);
            q[a * qstride] = a2;
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

// Column multiply + pivoted banded solve (left operators, kl = 2, ku = 3 in
// compressed coordinates):  z = LU^-1 ( MUL y + alpha e ), in place.
// cf row layout (stride 16): [mul -2..3 | L0 L1 | piv | Uf0..Uf4 | inv | pad].
__device__ __forceinline__ void col_solve(double* __restrict__ col, int pitch, int M, const double* __restrict__ cf,
                                          const double* __restrict__ e, long estride, double alpha) {
    auto rrow = [&](int a, double ym2, double ym1, double y0, double y1, double y2, double y3) {
        const double* c = cf + a * kLeftW;
        double acc = c[0] * ym2;
        acc = fma(c[1], ym1, acc);
        acc = fma(c[2], y0, acc);
        acc = fma(c[3], y1, acc);
        acc = fma(c[4], y2, acc);
        acc = fma(c[5], y3, acc);
        return fma(alpha, e[a * estride], acc);
    };
    const double v0 = col[0], v1 = col[pitch], v2 = col[2 * pitch], v3 = col[3 * pitch], v4 = col[4 * pitch];
    double x0 = rrow(0, 0.0, 0.0, v0, v1, v2, v3);
    double x1 = rrow(1, 0.0, v0, v1, v2, v3, v4);
    double r0 = v0, r1 = v1, r2 = v2, r3 = v3, r4 = v4, r5 = col[5 * pitch];
    for (int k = 0; k < M; ++k) {
        double x2 = (k + 2 < M) ? rrow(k + 2, r0, r1, r2, r3, r4, r5) : 0.0;
        const double* c = cf + k * kLeftW;
        const int pv = int(c[8]);
        if (pv == 1) swap2(x0, x1);
        else if (pv == 2) swap2(x0, x2);
        x1 = fma(-c[6], x0, x1);
        x2 = fma(-c[7], x0, x2);
        const double ynext = col[(k + 6) * pitch];
        col[k * pitch] = x0;
        x0 = x1;
        x1 = x2;
        r0 = r1;
        r1 = r2;
        r2 = r3;
        r3 = r4;
        r4 = r5;
        r5 = ynext;
    }
    double xa = 0.0, xb = 0.0, xc = 0.0, xd = 0.0, xe = 0.0;
    for (int k = M - 1; k >= 0; --k) {
        const double* c = cf + k * kLeftW;
        double acc = col[k * pitch] * c[14];
        acc = fma(-c[13], xe, acc);
        acc = fma(-c[12], xd, acc);
        acc = fma(-c[11], xc, acc);
        acc = fma(-c[10], xb, acc);
        acc = fma(-c[9], xa, acc);
        col[k * pitch] = acc;
        xe = xd;
        xd = xc;
        xc = xb;
        xb = xa;
        xa = acc;
    }
}

// Row multiply + pivoted banded solve (right operators, transposed form,
// kl = 1, ku = 2): y = LU^-1 ( MUL z ), in place over b in [0,N).
// mul: 4 coefficients at offsets -1..2 (stride ms); lu: [L | piv | Uf0..2 | inv] (stride ls).
__device__ __forceinline__ void row_solve(double* __restrict__ row, int N, const double* __restrict__ mul, int ms,
                                          const double* __restrict__ lu, int ls, double* esq) {
    auto rrow = [&](int b, double zm1, double z0, double z1, double z2) {
        const double* c = mul + b * ms;
        double acc = c[0] * zm1;
        acc = fma(c[1], z0, acc);
        acc = fma(c[2], z1, acc);
        return fma(c[3], z2, acc);
    };
    double s0 = row[0], s1 = row[1], s2 = row[2], s3 = row[3];
    double x0 = rrow(0, 0.0, s0, s1, s2);
    double sq = x0 * x0;
    for (int k = 0; k < N; ++k) {
        double x1 = 0.0;
        if (k + 1 < N) {
            x1 = rrow(k + 1, s0, s1, s2, s3);
            sq = fma(x1, x1, sq);
        }
        const double* c = lu + k * ls;
        if (int(c[1]) == 1) swap2(x0, x1);
        x1 = fma(-c[0], x0, x1);
        const double snext = row[k + 4];
        row[k] = x0;
        x0 = x1;
        s0 = s1;
        s1 = s2;
        s2 = s3;
        s3 = snext;
    }
    if (esq) *esq += sq;
    double xa = 0.0, xb = 0.0, xc = 0.0;
    for (int k = N - 1; k >= 0; --k) {
        const double* c = lu + k * ls;
        double acc = row[k] * c[5];
        acc = fma(-c[4], xc, acc);
        acc = fma(-c[3], xb, acc);
        acc = fma(-c[2], xa, acc);
        row[k] = acc;
        xc = xb;
        xb = xa;
        xa = acc;
    }
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

}  // namespace

// Shared-memory tile: rows [0, mh+6) x pitch (pitch >= nh+3, odd).
__global__ void __launch_bounds__(128) adi_kernel(const AdiParams P) {
    extern __shared__ double sm[];
    double* Y = sm;
    __shared__ double red[8];
    const AdiTask task = P.tasks[blockIdx.x];
    const int t = task.tensor, s = task.slot, k0 = task.k0, plane = task.plane;
    const Geo& g = P.g;
    if (!P.active[t * g.nslots + s]) return;
    const AdiSlot so = P.slots[s];
    const int M = P.M, N = P.N, mh = g.mh, nh = g.nh, pitch = P.pitch;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int rows = mh + 6;
    const long toff = long(s) * g.slot_stride + long(plane) * g.plane_stride;
    double* ep = P.eprime + long(blockIdx.x) * M * N;
    const double* sleft = P.coef + so.sleft;
    const double* sright = P.coef + (k0 ? so.sright1 : so.sright0);

    // ---- prologue: f (RHS assembly, fused BDF/IMEX combination) -> F = R2 f C02^T -> E' = E B^-1
    for (int i = tid; i < rows * pitch; i += nt) Y[i] = 0.0;
    __syncthreads();
    for (int b = 0; b < nh; ++b) {
        const long off = toff + long(2 * b + k0) * mh;
        for (int a = tid; a < mh; a += nt) {
            double acc = 0.0;
            for (int i = 0; i < P.nsrc[t]; ++i) acc = fma(P.wsrc[t][i], P.src[t][i][off + a], acc);
            Y[a * pitch + b] = acc;
        }
    }
    __syncthreads();
    for (int b = tid; b < nh; b += nt) col_mul(Y + b, pitch, M, sleft, kStatW, 0, nullptr, 0, 0.0, 0, nullptr, 0);
    __syncthreads();
    // row M (= mh-1) of F is outside the truncated system
    for (int b = tid; b < pitch; b += nt) Y[M * pitch + b] = 0.0;
    __syncthreads();
    double esq = 0.0;
    for (int a = tid; a < M; a += nt) {
        // columns >= N of row a: N holds F data outside the system; zero after use below
        row_solve(Y + a * pitch, N, sright + 0, kStatW, sright + 4, kStatW, &esq);
    }
    __syncthreads();
    for (int i = tid; i < M * N; i += nt) {
        const int a = i / N, b = i % N;
        ep[i] = Y[a * pitch + b];
    }
    __syncthreads();
    for (int i = tid; i < rows * pitch; i += nt) Y[i] = 0.0;
    __syncthreads();

    if (P.round > 0) {
        // restart from the previous round's X, recovered from u = S X S^T by prefix sums
        const double* u = P.out[t];
        for (int b = 0; b < N; ++b) {
            const long off = toff + long(2 * b + k0) * mh;
            for (int a = tid; a < M; a += nt) Y[a * pitch + b] = u[off + a];
        }
        __syncthreads();
        for (int b = tid; b < N; b += nt) {
            double acc = 0.0;
            for (int a = 0; a < M; ++a) {
                acc += Y[a * pitch + b];
                Y[a * pitch + b] = acc;
            }
        }
        __syncthreads();
        for (int a = tid; a < M; a += nt) {
            double acc = 0.0;
            for (int b = 0; b < N; ++b) {
                acc += Y[a * pitch + b];
                Y[a * pitch + b] = acc;
            }
            row_solve(Y + a * pitch, N, sright + 18, kStatW, sright + 4, kStatW, nullptr);
        }
        __syncthreads();
    }

    // ---- J iterations, tile resident in shared memory
    const double* left = P.coef + so.left;
    const double* right = P.coef + (k0 ? so.right1 : so.right0);
    const double* dsv = P.coef + so.ds;
    for (int j = 0; j < so.J; ++j) {
        const double* cl = left + long(j) * M * kLeftW;
        const double* cr = right + long(j) * N * kRightW;
        const double alpha = -dsv[j];
        for (int b = tid; b < N; b += nt) col_solve(Y + b, pitch, M, cl, ep + b, N, alpha);
        __syncthreads();
        for (int a = tid; a < M; a += nt) row_solve(Y + a * pitch, N, cr, kRightW, cr + 4, kRightW, nullptr);
        __syncthreads();
    }

    // ---- epilogue: u = S_r X S_z^T (Dirichlet recombination, solvers.cpp:97), parity-compressed store
    double* u = P.out[t];
    for (int b = 0; b < nh; ++b) {
        const long off = toff + long(2 * b + k0) * mh;
        for (int a = tid; a < mh; a += nt) {
            const double x00 = Y[a * pitch + b];
            const double x10 = a > 0 ? Y[(a - 1) * pitch + b] : 0.0;
            const double x01 = b > 0 ? Y[a * pitch + b - 1] : 0.0;
            const double x11 = (a > 0 && b > 0) ? Y[(a - 1) * pitch + b - 1] : 0.0;
            u[off + a] = (x00 - x10) - (x01 - x11);
        }
    }
    __syncthreads();
    // ---- residual: P = A X - E' (shared), Q = C X (scratch), R^T = B^T P^T + D^T Q^T
    for (int b = tid; b < N; b += nt) col_mul(Y + b, pitch, M, sleft, kStatW, 6, ep + b, N, -1.0, 12, ep + b, N);
    __syncthreads();
    double rsq = 0.0;
    for (int a = tid; a < M; a += nt) {
        const double* prow = Y + a * pitch;
        const double* qrow = ep + long(a) * N;
        double pm1 = 0.0, p0 = prow[0], p1 = prow[1], p2 = prow[2];
        double qm1 = 0.0, q0 = qrow[0], q1 = N > 1 ? qrow[1] : 0.0, q2 = N > 2 ? qrow[2] : 0.0;
        for (int b = 0; b < N; ++b) {
            const double* c = sright + b * kStatW;
            double r = c[10] * pm1;
            r = fma(c[11], p0, r);
            r = fma(c[12], p1, r);
            r = fma(c[13], p2, r);
            r = fma(c[14], qm1, r);
            r = fma(c[15], q0, r);
            r = fma(c[16], q1, r);
            r = fma(c[17], q2, r);
            rsq = fma(r, r, rsq);
            pm1 = p0;
            p0 = p1;
            p1 = p2;
            p2 = prow[b + 3];
            qm1 = q0;
            q0 = q1;
            q1 = q2;
            q2 = (b + 3 < N) ? qrow[b + 3] : 0.0;
        }
    }
    const double rs = block_sum(rsq, red);
    const double es = block_sum(esq, red);
    if (tid == 0) {
        atomicAdd(P.res2 + t * g.nslots + s, rs);
        atomicAdd(P.e2 + t * g.nslots + s, es);
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
