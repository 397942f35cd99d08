// Fused fast-diagonalization modal solve (see diag.hpp): one CTA per real sub-problem
// (tensor, slot, k-parity, plane) runs the four products
//     T1 = PL f,   Z = (T1 PR) .* RT,   T3 = QL Z,   u = T3 QR
// with the 128 x 128 intermediate resident in shared memory, so only f is read and u written
// (the unfused chain moves T1, Z and T3 through HBM and takes four launches).
//
// 8 warps (4 along M x 2 along N), each a 32 x 64 accumulator tile of mma.sync m8n8k4.f64;
// streamed operands go through a 2-stage cp.async ring of 16-row / 16-column k-slices.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

namespace ccf {

namespace {

constexpr int FT = 128;       // tile edge (M, N, K of every product <= 128)
constexpr int FSP = FT + 4;   // intermediate pitch (doubles)
constexpr int FK = 16;        // k-slice
constexpr int FSA = FK + 4;   // pitch of a streamed A slice (FT rows x FK)
constexpr int FSB = FT + 4;   // pitch of a streamed B slice (FK rows x FT)
constexpr int FSTAGE = FT * FSA > FK * FSB ? FT * FSA : FK * FSB;  // doubles per stage (either operand)
constexpr int FSTAGES = 3;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src, int bytes) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// stream a k-slice of a global row-major operand into a stage buffer
//   A slice: rows [0, FT) x cols [k0, k0 + FK) of A (rows < R, cols < Kd valid), pitch FSA
//   B slice: rows [k0, k0 + FK) x cols [0, FT) of B (rows < Kd, cols < C valid), pitch FSB
__device__ __forceinline__ void load_a_slice(double* st, const double* __restrict__ A, long lda, int R, int Kd,
                                             int k0) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 128 rows x 8 chunks
        const int c = tid + q * 256;
        const int row = c >> 3, kc = (c & 7) * 2;
        const int gk = k0 + kc;
        const int nv = row < R ? max(0, min(2, Kd - gk)) : 0;
        cp16(st + row * FSA + kc, nv ? A + long(row) * lda + gk : A, nv * 8);
    }
}
__device__ __forceinline__ void load_b_slice(double* st, const double* __restrict__ B, long ldb, int Kd, int Cc,
                                             int k0) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 16 rows x 64 chunks
        const int c = tid + q * 256;
        const int row = c >> 6, cc = (c & 63) * 2;
        const int gk = k0 + row;
        const int nv = gk < Kd ? max(0, min(2, Cc - cc)) : 0;
        cp16(st + row * FSB + cc, nv ? B + long(gk) * ldb + cc : B, nv * 8);
    }
}

struct Acc {
    double v[4][8][2];
};
using True = std::integral_constant<bool, true>;
using False = std::integral_constant<bool, false>;

__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a.v[i][j][0] = a.v[i][j][1] = 0.0;
}

// one 4-deep k step: A fragment rows wm + 8 i + gq at column ka + tq, B fragment rows kb + tq at
// columns wn + 8 j + gq
__device__ __forceinline__ void kstep(Acc& acc, const double* a, int pa, int ka, const double* b, int pb, int kb,
                                      int wm, int wn, int gq, int tq) {
    double af[4], bf[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = a[(wm + 8 * i + gq) * pa + ka + tq];
#pragma unroll
    for (int j = 0; j < 8; ++j) bf[j] = b[(kb + tq) * pb + wn + 8 * j + gq];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma(acc.v[i][j][0], acc.v[i][j][1], af[i], bf[j]);
}

}  // namespace

// Per task: A/B/C pointer arrays of the four products (see Pipeline::modal_solve for the layout).
__global__ void __launch_bounds__(256, 1) fdsolve_kernel(FdSolve p) {
    extern __shared__ __align__(16) double fsm[];
    double* S = fsm;                  // FT x FSP intermediate
    double* ST = fsm + FT * FSP;      // FSTAGES x FSTAGE stream ring
    const int task = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 64;
    const int gq = lane >> 2, tq = lane & 3;
    const int M = p.M, N = p.N, mh = p.mh, nh = p.nh;
    const FdTask tk = p.tasks[task];
    const double* f = p.fbase[tk.t] + tk.off;
    double* u = p.obase[tk.t] + tk.off;
    Acc acc;

    // The four products stream one operand each (phase 1: PL as A against f in S; 2: PR as B
    // against T1; 3: QL as A against Z; 4: QR as B against T3). One continuous cp.async ring runs
    // FSTAGES - 1 k-slices ahead across the phase boundaries, so the next phase's operand arrives
    // while the current phase's epilogue rewrites S.
    const int nk[4] = {(mh + FK - 1) / FK, (nh + FK - 1) / FK, (M + FK - 1) / FK, (N + FK - 1) / FK};
    const int total = nk[0] + nk[1] + nk[2] + nk[3];
    int lph = 0, lkt = 0, lissued = 0;
    auto issue = [&]() {
        if (lissued < total) {
            double* st = ST + (lissued % FSTAGES) * FSTAGE;
            const int k0 = lkt * FK;
            switch (lph) {
                case 0: load_a_slice(st, tk.PL, mh, M, mh, k0); break;
                case 1: load_b_slice(st, tk.PR, p.ldpr, nh, N, k0); break;
                case 2: load_a_slice(st, tk.QL, p.ldql, mh, M, k0); break;
                default: load_b_slice(st, tk.QR, nh, N, nh, k0); break;
            }
            ++lissued;
            if (++lkt == nk[lph]) {
                lkt = 0;
                ++lph;
            }
        }
        cp_commit();
    };

    // ---- stage f (mh x nh) into S, start the operand stream
    for (int i = tid; i < FT * FSP; i += blockDim.x) S[i] = 0.0;
    __syncthreads();
    for (int c = tid; c < mh * (nh / 2); c += blockDim.x) {  // f: 16-byte chunks
        const int row = c / (nh / 2), cc = (c - row * (nh / 2)) * 2;
        cp16(S + row * FSP + cc, f + long(row) * p.ldf + cc, 16);
    }
    cp_commit();
#pragma unroll
    for (int s = 0; s < FSTAGES - 1; ++s) issue();
    int consumed = 0;
#pragma unroll 1
    for (int ph = 0; ph < 4; ++ph) {
        acc_zero(acc);
        for (int kt = 0; kt < nk[ph]; ++kt, ++consumed) {
            cp_wait<FSTAGES - 2>();
            __syncthreads();
            issue();
            const double* st = ST + (consumed % FSTAGES) * FSTAGE;
            const bool a_streamed = (ph == 0 || ph == 2);
#pragma unroll
            for (int ks = 0; ks < FK; ks += 4) {
                if (a_streamed) kstep(acc, st, FSA, ks, S, FSP, kt * FK + ks, wm, wn, gq, tq);
                else kstep(acc, S, FSP, kt * FK + ks, st, FSB, ks, wm, wn, gq, tq);
            }
        }
        __syncthreads();  // every warp is done reading S for this phase
        if (ph == 3) break;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int r = wm + 8 * i + gq, c = wn + 8 * j + 2 * tq;
                double v0 = acc.v[i][j][0], v1 = acc.v[i][j][1];
                if (ph == 0) {  // T1 (M x nh), RHS weight
                    v0 = r < M ? p.alpha * v0 : 0.0;
                    v1 = r < M ? p.alpha * v1 : 0.0;
                } else if (ph == 1) {  // T1 PR (M x N); the .* RT pass follows
                    v0 = (r < M && c < N) ? v0 : 0.0;
                    v1 = (r < M && c + 1 < N) ? v1 : 0.0;
                } else {  // T3 (mh x N)
                    v0 = (r < mh && c < N) ? v0 : 0.0;
                    v1 = (r < mh && c + 1 < N) ? v1 : 0.0;
                }
                *reinterpret_cast<double2*>(S + r * FSP + c) = make_double2(v0, v1);
            }
        if (ph == 1) {  // Z = (T1 PR) .* RT with coalesced 16-byte loads of the table (ld ldrt)
            __syncthreads();
            const int ch = p.ldrt / 2;  // 16-byte chunks per table row
            for (int e = tid; e < M * ch; e += blockDim.x) {
                const int r = e / ch, c = (e - r * ch) * 2;
                const double2 rt = __ldg(reinterpret_cast<const double2*>(tk.RT + long(r) * p.ldrt + c));
                double2* z = reinterpret_cast<double2*>(S + r * FSP + c);
                const double2 zv = *z;
                *z = make_double2(zv.x * rt.x, zv.y * rt.y);
            }
        }
        // the next phase's first slices were issued before this epilogue; its first iteration
        // synchronizes before reading S
    }
    cp_wait<0>();
    // ---- u = T3 QR -> output tensor (mh x nh)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int r = wm + 8 * i + gq, c = wn + 8 * j + 2 * tq;
            if (r < mh && c < nh) {
                if (c + 1 < nh) *reinterpret_cast<double2*>(u + long(r) * p.ldf + c) = make_double2(acc.v[i][j][0], acc.v[i][j][1]);
                else u[long(r) * p.ldf + c] = acc.v[i][j][0];
            }
        }
}

size_t fdsolve_smem() { return size_t(FT * FSP + FSTAGES * FSTAGE) * sizeof(double); }

}  // namespace ccf
