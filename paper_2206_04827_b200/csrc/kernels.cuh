// Kernel declarations shared between the .cu translation units and the host driver.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "ccf_device.cuh"

namespace ccf {

// adi.cu
// ADI sweeps (adi.cu): size-specialised instantiations behind one launcher
size_t adi_static_smem();
cudaError_t adi_set_smem(int bytes);
void adi_launch(const AdiParams& P, int threads, size_t smem, cudaStream_t stream);
struct RoundCheck {
    int ntensor, nslots, round;
    double tol;
    double* res2;
    double* e2;
    int* active;
    double* history;
    int* rounds;
    int* err;
    const int* J;          // per slot
    unsigned long long* iters;  // executed sub-problem iterations (4 sub-problems per (tensor, slot))
};
__global__ void adi_round_check(RoundCheck c);
__global__ void adi_init_kernel(int* active, double* res2, double* e2, int n);

// layout.cu
__global__ void ref_to_h_kernel(const double* __restrict__ ref, double* __restrict__ out, Geo g, int full, int cls);
__global__ void h_to_ref_kernel(const double* __restrict__ in, double* __restrict__ ref, Geo g, int full, int cls,
                                int accumulate);
__global__ void real_to_complex_kernel(const double* __restrict__ in, double* __restrict__ out, long n);
__global__ void complex_re_kernel(const double* __restrict__ in, double* __restrict__ out, long n);
__global__ void finite_check_kernel(const double* __restrict__ x, long n, int* flag);
struct Combo {
    const double* src[kMaxSrc];
    double w[kMaxSrc];
    int nsrc;
    double* out;
    long n;
};
__global__ void combo_kernel(Combo c);

// solve.cu: fused fast-diagonalization modal solve (one CTA per real sub-problem, sizes <= 128)
struct FdTask {
    int t;     // tensor (base index)
    long off;  // offset of the sub-problem block in the input / output tensor
    const double *PL, *PR, *RT, *QL, *QR;
};
struct FdSolve {
    const FdTask* tasks;
    const double* fbase[2];
    double* obase[2];
    int M, N, mh, nh;
    long ldf, ldpr, ldql, ldrt;
    double alpha;
};
__global__ void fdsolve_kernel(FdSolve p);
size_t fdsolve_smem();

// pipeline.cu: eigen-coordinate RHS out_t = factor * (sum_q w_q src_t,q) .* RT[(s, k0)]
struct EigRhs {
    const double* src[2][kMaxSrc];
    double w[kMaxSrc];
    int nsrc, ntensor;
    double* out[2];
    const double* const* rt;
    double factor;
    int M, N, Np, nslots, slo;  // slots [slo, slo + nslots)
    double* outp;              // optional: -out[0] .* rtp (the next step's Poisson RHS in eigen coordinates)
    const double* const* rtp;  // RT table of the Poisson set
    int* flag;                 // optional: set to 1 on a non-finite output (NaN guard, ptns.cpp:260-262)
    // optional (INT8 product path, ozaki.hpp): also write out[0], out[1], outp as row-scaled digit panels, the
    // back transform's A operands: panel ((s - slo) * 2 + pl) * 2 + k0 of tensor t at pan[t] (16 KB slices,
    // 96 KB panels), row scales at psc[t] + panel * 128 (eigen row i = panel row)
    uint8_t* pan[3];
    double* psc[3];
};

// transform.cu
struct GemmBatch {
    const double* const* A;
    const double* const* B;
    double* const* C;
    int M, N, K;
    long lda, ldb, ldc;
    double alpha, beta;
    const int* tstart;  // optional: batch b sums the terms [tstart[b], tstart[b+1]) (A, B indexed by term)
    const double* const* dl;  // optional epilogue C[i][j] = acc * dl[b][i * N + j] (fast diagonalization:
    const double* const* dr;  //   reciprocals of lambda_i + mu_j; dr unused)
    // optional base-relative B (per term) / C (per batch): pointer = base[off >> 40] + (off & (2^40 - 1)),
    // so a captured plan can be relaunched on other tensors (ring buffers) with new bases
    const long* boff;
    const long* coff;
    const double* bbase[3];
    double* cbase[2];
    int nbatch;  // number of batches
    long ldd;    // leading dimension of the dl tables
    int ipc;     // items (batch x m-tile x n-tile) per CTA, pipelined kernel
    const long* aoff;  // optional base-relative A per term (same bases as B; not together with boff)
};
constexpr long kBaseShift = 40;
__global__ void dgemm_batched_kernel(GemmBatch g);
template <int PM>
__global__ void dgemm_pipe_kernel(GemmBatch g);  // PM x 64 tiles (PM = 128 | 64), cp.async pipeline (aligned operands)
size_t dgemm_pipe_smem(int bm);
// TMA variant: tensor maps of the operand allocations (A boxes 16 x 128, B boxes 16 x 16, f64,
// 128-byte swizzle), per-term box origins ta[t] = {A map, A col, A row, B map}, tb[t] = {B col, B row}
constexpr int kTmaMaps = 8;
struct TmaMaps {
    CUtensorMap m[kTmaMaps];
};
__global__ void dgemm_tma_kernel(GemmBatch g, const __grid_constant__ TmaMaps maps, const int4* ta, const int2* tb);
size_t dgemm_tma_smem();
struct ThetaCross {
    Geo g;
    int logp, tj;
    const double* in[6];
    double* out[3];
    const double2* tw;
    const double2* twfull;  // p twiddles exp(-2 pi i q / p): the dense-DFT path of theta_cross_kernel (p not 2^k)
    // mode sharding (csrc/shard.cu): this launch covers rows row0 + blockIdx.y; slot s is read from
    // and written to the exchange buffer of its owning rank q (sb[q] <= s < sb[q+1]), rdelta[q]
    // doubles away from the local one (peer memory over NVLink); world == 1: local, delta 0
    int row0, world;
    int sb[9];
    long rdelta[8];
    // input value layout: 0 = [jr][z] rows (leading dimension n); 1 = column-quad major [z / 4][jr][z % 4], written
    // by the INT8 X1 product (coalesced epilogue stores; theta_cross256w_kernel only)
    int vquad;
};
// doubles from the local exchange tensors to those of the owner of slot s
__device__ __forceinline__ long theta_slot_delta(const ThetaCross& t, int s) {
    if (t.world <= 1) return 0;
    int q = 0;
#pragma unroll 1
    while (q + 1 < t.world && s >= t.sb[q + 1]) ++q;
    return t.rdelta[q];
}
__global__ void theta_cross_kernel(ThetaCross t);
__global__ void theta_cross256_kernel(ThetaCross t);  // p = 256 register-FFT path
size_t theta_cross256_smem();
int theta_cross256_positions();
int theta_cross256_threads();
template <int NQ>
__global__ void theta_cross256w_kernel(ThetaCross t);  // warp-per-point variant, NQ z-position pairs per CTA
size_t theta_cross256w_smem(int nq);
// p = 512: radix-8 passes; the sample / task mapping is written for exactly these two constants
constexpr int kTheta512Points = 4;     // points (TJ) per CTA
constexpr int kTheta512Threads = 256;  // threads per CTA
__global__ void theta_cross512_kernel(ThetaCross t);
size_t theta_cross512_smem();
__global__ void theta_dft_full_kernel(const double* __restrict__ in, double* __restrict__ out, int m, int n, int p,
                                      int dir, const double2* __restrict__ twp);

// pencil.cu
struct DzBatch {
    Geo g;
    int count;
    const double* in[6];
    double* out[6];
};
__global__ void dz_kernel(DzBatch d);
struct PtSynth {
    Geo g;
    int count;
    const double* lam[2];
    const double* gam[2];
    const double* dzg[2];
    double* vr[2];
    double* vt[2];
    double* vz[2];
    double* scratch;  // count * nslots * n * 2 * mh
    const double* q;  // odd interpolation coefficients of 1/r (mh)
};
__global__ void pt_synth_kernel(PtSynth a);
struct CurlDecomp {
    Geo g;
    int decompose_only;  // 1: (ar, at, az) are already (v_r, v_t, v_z); dzat unused
    const double *ar, *at, *az, *dzar, *dzat;
    double *out_r, *out_t, *out_z;  // optional curl components
    double *lam, *gam;              // optional PT scalars of the curl
    double* scratch;                // nslots * n * 6 * mh
    const double* q;
    const double* hpc;  // per slot: M x 8 LU(recombine(L_w)) [L, piv, inv, Uf0..2, 0, 0]
    const double* hpr;  // per parity: M x 8 compressed R R C02 rows (offsets -1..3)
};
__global__ void curl_decomp_kernel(CurlDecomp a);
struct HpArgs {
    Geo g;
    const double* in;
    double* out;
    double* scratch;
    const double* hpc;
    const double* hpr;
};
__global__ void hp_kernel(HpArgs a);
struct CalcArgs {
    Geo g;
    int op, cls;
    const double* in;
    double* out;
    double* scratch;
    const double* q;
};
__global__ void calc_kernel(CalcArgs a);

}  // namespace ccf
