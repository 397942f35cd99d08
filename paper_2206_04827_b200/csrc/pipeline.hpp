// NS time-step pipeline on the device (reference: proj/src/ptns.cpp:217-267).
//
// Per step (half-spectrum, parity-compressed tensors):
//   P  lambda_psi = Poisson3D(-lambda_w)                           ADI (Poisson set)
//   V  dz gamma, pt_synthesize(v), pt_synthesize(w)               dz_kernel, pt_synth_kernel
//   X  r,z synthesis (DMMA GEMMs) -> theta FFT x cross x FFT -> r,z analysis
//   C  dz a, curl_vector + pt_decompose (horizontal Poisson)      curl_decomp_kernel
//   H  BDF history + kappa * IMEX(N history) -> Helmholtz ADI for (lambda, gamma)
// State (omega history, N history) stays on the device; ring indices rotate.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <vector>

#include <map>
#include <memory>
#include <set>
#include <string>

#include "composite.hpp"
#include "context.hpp"

namespace ccf {

// Chebyshev synthesis / analysis matrices (device, row-major) and theta twiddles.
struct TransformPlan {
    DBuf SrT[2], ArT[2];  // [j0]: mh x mh  (A operands of the r-GEMMs, r > 0 half grid)
    DBuf Sz, Az;          // [2][nh x nh] z synthesis / analysis between parity-split coefficients and [E | O] values
    DBuf Szf, Azf;        // n x n z synthesis [kz][k] / analysis [k][kz] in natural order (API transforms)
    DBuf Rfull_S, Rfull_A;  // m x m dense r synthesis / analysis (API transforms on arbitrary fields)
    DBuf q;               // mh: odd Chebyshev coefficients of the interpolant of 1/r_j
    DBuf tw;              // p/2 complex twiddles exp(-2 pi i q / p)
    DBuf twfull;          // p complex twiddles (naive DFT path)
    DBuf hpc, hpr;        // horizontal-Poisson LU per half slot; R R C02 per parity
    DBuf DzS, ADz;        // [2][nh x nh] z synthesis of dz f / dz of the z analysis (derivative_z folded in)
    RadialTables rt;      // host copies for the composite radial operators (composite.hpp)
    int logp = -1;        // log2 p, or -1 if p is not a power of two
    explicit TransformPlan(Ctx& c);
};

// Reusable batched-GEMM launcher with device pointer arrays.
struct GemmPlan {
    std::vector<const double*> A, B;  // per term (= per batch unless tstart is set)
    std::vector<double*> C;           // per batch
    std::vector<int> tstart;          // optional: batch b sums terms [tstart[b], tstart[b+1])
    std::vector<const double*> DL, DR;  // optional per-batch epilogue divisors (dl_i + dr_j)
    std::vector<long> Boff, Coff;       // optional base-relative B / C (see GemmBatch)
    std::vector<long> Aoff;             // optional base-relative A (A then holds one placeholder per term)
    long* dAoff = nullptr;
    long ldd = 0;                       // leading dimension of the epilogue table (0: N)
    const double** dA = nullptr;
    const double** dB = nullptr;
    double** dC = nullptr;
    int* dT = nullptr;
    const double** dDL = nullptr;
    const double** dDR = nullptr;
    long* dBoff = nullptr;
    long* dCoff = nullptr;
    bool pipe = false;  // operands qualify for dgemm_pipe_kernel (set by upload)
    // TMA variant (dgemm_tma_kernel): set by upload when the operands map onto <= 8 tensor maps
    // (<= 5 with a base-relative B: slots 5 / 6 / 7 hold the launch bases, encoded at launch and cached)
    bool tma = false;
    std::vector<CUtensorMap> tmaps;
    void* dTA = nullptr;  // int4 per term
    void* dTB = nullptr;  // int2 per term
    mutable std::vector<std::pair<const double*, CUtensorMap>> bmap_cache;
    int M = 0, N = 0, K = 0;
    // columns of every A row past K that the caller guarantees to be zero (padding): the TMA kernel reads
    // whole 16-column k-boxes, so it is only used when K is a multiple of 16 or this padding covers the box
    int kzero = 0;
    long lda = 0, ldb = 0, ldc = 0;
    double alpha = 1.0, beta = 0.0;
    void upload();
    void launch(cudaStream_t s, const double* b0 = nullptr, const double* b1 = nullptr, double* c0 = nullptr,
                double* c1 = nullptr, const double* b2 = nullptr) const;
    double flops() const { return 2.0 * M * N * K * double(A.size()); }  // every term is one M x N x K product
    ~GemmPlan();
};

struct OzPipe;
struct EigRhs;

class Pipeline {
public:
    explicit Pipeline(Ctx& c);
    ~Pipeline();
    Ctx& c;
    TransformPlan tp;
    long T;  // doubles per half-spectrum tensor
    // ---- stage building blocks (all on c.stream, capture-safe)
    void dz(const std::vector<const double*>& in, const std::vector<double*>& out);
    void pt_synthesize(int count, const double* const* lam, const double* const* gam, double* const* vr,
                       double* const* vt, double* const* vz);
    // coefficient (class per tensor) -> (r,z)-values / theta-coefficients, and back
    void rz_synth(int count, const double* const* in, const int* cls, double* const* out);
    void rz_analyze(int count, const double* const* in, const int* cls, double* const* out);
    void theta_cross(const double* const* v6, double* const* a3);
    // the warp-per-point p = 256 theta kernel will run (the only one reading column-quad-major values)
    bool theta_quad_ok() const;
    bool val_quad_ = false;  // the theta inputs in the next theta_cross are column-quad major (OzPipe::rsynth)
    void curl_decompose(const double* ar, const double* at, const double* az, double* out_r, double* out_t,
                        double* out_z, double* lam, double* gam);
    // eig != nullptr: output N~ = PL_P N PR in the eigen layout of that (Poisson) set's modal basis
    // zpre: scratch(0..5) already hold the z-synthesized inputs (lambda_v = gamma_w aliased to scratch(4));
    // eigY: those are eigen-coordinate Y tensors (eigen_ysynth), synthesized with the QL-folded blocks
    // dealias: the reference's 2/3 rule on the analyzed cross product (ptns.cpp:100-110, 140-144): the j / k masks
    // are folded into the analysis matrices, the |w| mask zeroes the output slots
    void nonlinear(const double* lam_v, const double* gam_v, const double* lam_w, const double* gam_w, double* lam_n,
                   double* gam_n, DevSet* eig = nullptr, bool zpre = false, bool eigY = false, bool dealias = false);
    void eigen_ysynth(int ntensor, const double* const* z, double* const* outS, double* const* outD);
    // eigen-coordinate NS state (see pipeline.cu)
    long eig_off(int s, int pl, int k0) const;
    void ensure_eigen(DevSet& pset);
    const double* const* eig_rt(DevSet& set);
    void eigen_rhs(DevSet& set, int ntensor, const double* const* s0, const double* const* s1, const double* w, int nsrc,
                   double factor, double* out0, double* out1, double* outp = nullptr,
                   DevSet* pset = nullptr, int* flag = nullptr, bool panels = false);
    void eigen_back(DevSet& set, int ntensor, const double* z0, const double* z1, double* out0, double* out1);
    void to_eigen(DevSet& pset, const double* u, double* z);
    void poisson(const double* f, double w, double* u);  // u = Poisson3D(w * f), half mode
    // Modal Sylvester solves of a solver set for 1 or 2 tensors with fused RHS combinations
    // (out_t = Solve(sum_i w_t[i] src_t[i])): fast diagonalization on the tensor cores, or the
    // ADI kernel (ctx flag bit 2 / sets without diagonalization data).
    bool modal_solve_from_z(DevSet& set, double w, double* out);
    bool last_z_valid_ = false;  // the last modal_solve left its eigen-coordinates Z in dZ_
    const void* z_owner_ = nullptr;  // NSState whose lambda_omega Z is what dZ_ holds (any other solve clears it)
    void modal_solve(DevSet& set, bool full, int ntensor, const double* const* src0, const double* w0, int n0,
                     const double* const* src1, const double* w1, int n1, double* out0, double* out1,
                     const char* rhs_mark = nullptr);
    void decompose(const double* vr, const double* vt, const double* vz, double* lam, double* gam);
    void hpoisson(const double* rhs, double* u);
    void calculus(int op, int cls, const double* in, double* out);  // ops of include/ccf.h ccf_calculus
    void scale(double* x, double a);
    void analyze_full(const double* values, double* coeffs);     // reference layouts, host or device
    void synthesize_full(const double* coeffs, double* values);
    double* scratch(int i);  // internal scratch tensors
    const void* zw_owner_ = nullptr;  // NSState whose omega z tensors occupy scratch 3..5
    double* big_scratch(size_t doubles);

    const double* full_rT();
    const double* full_sT();
    double* big2(size_t doubles);

public:  // internal state (used by the NS stepper and the C-ABI layer)
    std::vector<DBuf> scr_;
    DBuf big_, big2_, rAT_, rST_;
    bool theta_attr_ = false, theta_generic_ = false, theta_w_ = true;  // CCF_THETA_GENERIC=1 forces the radix-2 path
    int theta_nq_ = 2;                                                  // z-position pairs per CTA (warp kernel)
    std::map<std::string, std::unique_ptr<GemmPlan>> gemms_;
    GemmPlan& gemm(const std::string& key, bool& fresh);
    // composite radial operators of the nonlinear term (built on first use)
    bool comp_ready_ = false, comp_off_ = false;  // CCF_NONLINEAR_PENCIL=1: sequential pencil path
    CompositeSet synth_, anal_;
    DBuf dsynth_, danal_, dsynth_eig_;
    bool composite_off() const { return comp_off_; }
    void ensure_composite();
    void nonlinear_pencil(const double* lam_v, const double* gam_v, const double* lam_w, const double* gam_w,
                          double* lam_n, double* gam_n);
    DBuf fcomb_[2], dT1_, dZ_, dT3_;  // fast-diagonalization scratch
    std::map<std::string, std::pair<FdTask*, int>> fdtasks_;  // fused-solve task lists (device)
    std::map<const void*, const double**> zrt_;               // per set: RT table per Poisson task
    DevSet* eig_set_ = nullptr;                               // modal basis the folded blocks below belong to
    DBuf eig_AzP_, eig_ADzP_, eig_anal_, eig_QS_, eig_QD_;
    // 2/3-dealiased analysis side (built on first use): z analysis (+ dz) with k >= 2n/3 masked, composite
    // curl / decompose blocks with j >= 2m/3 masked, and their eigen-coordinate forms
    bool dealias_ready_ = false;
    DBuf AzD_, ADzD_, danalD_, eig_AzPD_, eig_ADzPD_, eig_analD_;
    CompositeSet analD_;
    DevSet* eigD_set_ = nullptr;
    void ensure_dealias(DevSet* eig);
    std::map<const void*, const double* const*> eig_rt_;      // per set: RT table per (slot, k0)
    bool fd_fused_ = false, fd_attr_ = false;                    // CCF_FDSOLVE_FUSED=1: fused solve kernel
    std::unique_ptr<OzPipe> oz_;                                 // INT8 tensor-core (Ozaki) product stages
    OzPipe& oz();
};

// The NS step's dense product stages on the INT8 tensor cores (ozpipe.cu, ozaki.hpp).
struct OzPipe {
    explicit OzPipe(Pipeline& p);
    ~OzPipe();
    Pipeline& P;
    bool on = false;
    int mask = 7;
    // each returns false when the stage is not available (size, first build during a graph capture):
    // the caller then runs its FP64 DMMA plan
    bool ysynth(int ntensor, const double* const* z, double* const* outS, double* const* outD);
    // the NS step's RHS pass writes the back transform's A panels itself (EigRhs::pan): fill the targets of
    // ysynth's split plan for (z0, z1, z2) if it exists; ysynth then skips that split
    bool rhs_panels(const double* z0, const double* z1, const double* z2, EigRhs& a);
    bool rsynth(double* const (&Z)[2][3], double* const* val);
    bool analyze(double* const* av, double* const* Y, double* lam_n, double* gam_n);

private:
    struct Stage;
    struct Panels {
        DBuf pan, pe;
    };
    std::map<const double*, Panels> panels_;  // INT8 panels standing for pipeline tensors
    std::set<const double*> panel_only_;      // tensors whose current value exists as panels only
    Panels& panels(const double* buf);
    std::map<std::string, std::unique_ptr<Stage>> stages_;
    Stage* stage(const std::string& key, bool& fresh);
    bool ensure_const();
    const DevSet* const_set_ = nullptr;
    DBuf cpan_, csc_, cpe_, ysp_, ysc_, rsp_, rsc_, rpe_, zap_, zasc_, rap_, rasc_, rape_;
    int syn0_ = 0, ana0_ = 0;
    std::string rhs_split_;  // the ysynth split key whose panels the last RHS pass wrote
};

struct NSState {
    Pipeline* pl = nullptr;
    double reynolds = 100, h = 1e-2;
    int order = 4, steps = 0;
    int ocount = 1;  // valid omega history entries (1 after construction; NSStepper::seed installs up to 4)
    // the next step's nonlinear term runs on the coefficient-space omega of the head slot (initial data or a
    // seeded history need not lie in the range of the modal basis); such a step is never graph-captured
    bool coeff_first = true;
    bool disable_nonlinear = false;
    bool dealias = false;        // NSConfig::dealias_two_thirds
    bool gamma_psi = false;      // NSConfig::compute_gamma_psi (evaluated on read, ccf_ns_gamma_psi)
    double time = 0;
    // omega history ring and nonlinear-term history ring, 5 slots each (the Helmholtz output
    // never aliases a live input; both heads advance in lockstep -> 5 graph phases)
    DBuf lam[5], gam[5], nl[5], ng[5];
    int head = 0;               // ring slot of the newest omega; history i at (head + i) % 5
    int nhead = 0, ncount = 0;  // N ring: entry i at (nhead + i) % 5
    int* dflag = nullptr;       // device non-finite flag (NaN guard, ptns.cpp:260-262)
    cudaGraphExec_t graphs[25] = {};  // steady-state step per (head, nhead) ring phase
    // ring phases this stepper has run eagerly once: a phase is captured only afterwards, so every pointer-keyed
    // product plan of the phase exists before the capture (orders < 4 and seeded histories reach the steady
    // state before all five phases have been visited)
    bool phase_warm[25] = {};
    bool graph_z[25] = {};  // the captured step starts from dZ_ (coefficient-space state, zvalid at capture)
    long launches_per_step = 0;
    bool use_graphs = true;
    bool zvalid = false;  // the last Helmholtz solve left Z(lambda_omega) in the shared modal basis
    bool eigen = false;   // eigen-coordinate state (Z / N~ rings in the shared modal basis)
    DBuf zl[5], zg[5];    // omega history in eigen coordinates (same ring slots as lam / gam)
    int coeff_head = 0;   // ring slot whose lam / gam hold the coefficient-space omega (-1: none)
    DBuf zpsi;            // Poisson RHS -Z_lambda .* RT_P of ring slot zp_head (left by the Helmholtz pass)
    int zp_head = -1;
    int zv_head = -1;     // ring slot whose velocity z tensors (scratch 1, 2) are current (while zw_owner_)
    // HeatStepper (timestep.cpp:110-144): one scalar field in lam (gam unused), optional forcing per step
    bool scalar = false;
    bool forced = false;  // the next step adds kappa * forcing (zf: eigen coordinates, fh: coefficients)
    DBuf fh, zf;
    DBuf ztmp, ctmp;  // velocity() / gamma_psi() scratch
    void velocity_coeff(double* lam_v, double* gam_v);  // NSStepper::velocity (ptns.cpp:205-215), coefficients
    void gamma_psi_coeff(double* out);                   // state().gamma_psi (ptns.cpp:248-253), coefficients
    ~NSState();
    void zsynth_omega(int r);
    void velocity(int r);
    void omega_coeff();
    void seed(int n_omega, const double* const* lam_h, const double* const* gam_h, int n_nl,
              const double* const* nl_l, const double* const* nl_g, double t, int steps_taken);
    void step_once();
    void enqueue(int b, int eo, int cur, int out, int nnew);
};

}  // namespace ccf
