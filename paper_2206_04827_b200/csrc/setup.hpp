// Host-side setup numerics for the B200 CCF solver (not on the per-step path).
//
// Everything here runs once per (size, wavenumber^2, scale): ultraspherical
// operator bands, Dirichlet recombination, the spectral enclosure of the
// recombined pencils, Zolotarev shift plans, and the parity-compressed banded
// LU factors the ADI kernel streams per shift. Semantics follow the reference:
//   operators      proj/src/ultraop.cpp:9-138
//   enclosure      proj/src/adi.cpp:22-49, proj/src/solvers.cpp:15-42
//   shift plan     proj/src/adi.cpp:68-104, proj/src/special.cpp
//   banded LU      proj/src/banded.cpp:150-187 (partial pivoting inside the band)
// Layout decision (B200-first): every operator has even band offsets only, so a
// Fourier mode's system splits by j-parity and k-parity. Matrices are stored
// "parity-compressed": entry (2a+j0, 2b+j0) -> (a, b).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ccf {

// Exceptions mirror proj/include/cylspec/errors.hpp:10-40; the C-ABI maps them
// one-to-one to ccf_status codes.
struct Error : std::runtime_error {
    int status;
    int slice = -1, shift_index = -1;
    std::vector<double> history;
    Error(int st, const std::string& w) : std::runtime_error(w), status(st) {}
};
enum Status { OK = 0, DOMAIN_ERROR = 1, CONFIG_ERROR = 2, SINGULAR = 3, NON_CONVERGENCE = 4, NOT_INCOMPRESSIBLE = 5,
              NUMERICAL = 6, CUDA_ERR = 7, FIELDFILE_ERR = 8, INTERNAL = 9 };

// Dense row-major square/rect matrix helper (setup only).
struct Dense {
    int r = 0, c = 0;
    std::vector<double> a;
    Dense() = default;
    Dense(int r_, int c_) : r(r_), c(c_), a(size_t(r_) * c_, 0.0) {}
    double& operator()(int i, int j) { return a[size_t(i) * c + j]; }
    double operator()(int i, int j) const { return a[size_t(i) * c + j]; }
};
Dense matmul(const Dense& x, const Dense& y);
Dense transpose(const Dense& x);

// Full (uncompressed) ultraspherical operators, ultraop.cpp:9-51.
struct Ultra {
    int n = 0;
    Dense c01, c12, c02, r, r2, d1, d2, rrc02, l0;  // l0 = R C12 D1 + R R D2 (w = 0 radial Laplacian)
    explicit Ultra(int n);
};
Dense radial_laplacian(const Ultra& u, int w);  // L_w = l0 - w^2 C02, ultraop.cpp:73-81
Dense recombine(const Dense& M);                 // (M S)[:r-2, :c-2], ultraop.cpp:135-138

// Compressed band of a matrix restricted to parity p: rows a in [0,rows), band offsets [lo,hi].
struct CBand {
    int rows = 0, lo = 0, hi = 0;
    std::vector<double> v;  // rows x (hi-lo+1), v[a*(w)+(d-lo)] = M(2a+p, 2(a+d)+p)
    double at(int a, int d) const { return (d < lo || d > hi) ? 0.0 : v[size_t(a) * (hi - lo + 1) + (d - lo)]; }
};
CBand compress(const Dense& M, int parity, int rows, int cols, int lo, int hi);

// Banded LU with partial pivoting on a compressed square band matrix (kl, ku),
// identical algorithm to proj/src/banded.cpp:150-187 applied to one parity block.
struct CLU {
    int n = 0, kl = 0, ku = 0;
    std::vector<double> L;    // n x kl: multiplier for row k+1+t at step k
    std::vector<int> piv;     // pivot offset (0..kl)
    std::vector<double> U;    // n x (kl+ku): U(k, k+1+t)
    std::vector<double> inv;  // 1/U(k,k)
};
CLU banded_lu(const CBand& A, int kl, int ku);  // throws Error(SINGULAR)

// Generalised spectrum extremes of the compressed pencil blocks (all parity
// blocks together), with the reference's padding and checks (adi.cpp:22-49).
// Eigenvalues of C^-1 A via Hessenberg reduction + Francis double-shift QR.
std::vector<double> eigenvalues_real_checked(const Dense& A, const Dense& C, double* radius, double* worst_imag);
struct Range { double lo, hi; };
Range padded_range(const std::vector<Dense>& As, const std::vector<Dense>& Cs, bool q2_endpoint_pad);

// Zolotarev shift plan, adi.cpp:68-104.
struct Plan {
    double a = 0, b = 0, c = 0, d = 0, gamma = 0, alpha = 0, modulus = 0, tol = 0;
    int J = 0;
    std::vector<double> u, v;
};
Plan shift_plan(Range ca, Range db, double tol);
double elliptic_K_kp(double kprime);
double jacobi_dn_kp(double u, double kprime);

}  // namespace ccf
