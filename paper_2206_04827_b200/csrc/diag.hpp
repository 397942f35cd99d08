// Fast-diagonalization data for the per-mode Sylvester systems (host setup).
//
// Every modal system of the reference's Poisson / Helmholtz solves (proj/src/solvers.cpp:77-98,
// 142-169; timestep.cpp:61-108) is, per parity block,
//     A X B^ + C X D^ = E,   E = R2 f C02^T (top-left block),   u = S X S^T
// with banded A, C (radial, per |w|) and B^, D^ (vertical, per k-parity). The reference solves it
// by ADI with Zolotarev shifts to a relative residual of tol. The generalized eigenproblems
// A v = lambda C v and D^ w = mu B^ w are real, simple and well conditioned (cond(V) ~ 30 at 256),
// so the exact solution is
//     X = V [ ((C V)^-1 E (B^-1 U)) ./ (lambda_i + mu_j) ] (B^ W)^-1,   W = B^-1 U,
// i.e. four small dense products per mode on the FP64 tensor cores. Folding the RHS operators
// and the Dirichlet recombination into the transforms keeps all four matrices well conditioned:
//     PL = (C V)^-1 R2m   (M x mh)      QL = S_r V            (mh x M)
//     PR = C02m W         (nh x N)      QR = (B^ W)^-1 S_z^T  (N x nh)
//     u  = QL [ (PL f PR) ./ (lambda_i + mu_j) ] QR.
// Eigenpairs are refined by inverse iteration in long double from Hessenberg-QR estimates;
// the solution then has a residual ~1e-15 relative (three orders below the ADI tolerance).
#pragma once

#include <vector>

#include "setup.hpp"

namespace ccf {

struct DiagLeft {
    std::vector<double> PL, QL, lam;  // M x mh, mh x M, M
    std::vector<long double> lam_ld;  // eigenvalues before rounding (for 1 / (lambda + mu))
    std::vector<long double> PL_ld;   // PL before rounding (for the scaled Helmholtz variant)
};
struct DiagRight {
    std::vector<double> PR, QR, mu;  // nh x N, N x nh, N
    std::vector<long double> mu_ld;
};

// Left side from the compressed bands of one parity block: A, C (M x M, offsets -2..3) and
// R2 (rows M, cols mh, offsets -1..3).
DiagLeft diag_left(const CBand& A, const CBand& C, const CBand& R2, int M, int mh);
// Right side from the stored (transposed) vertical bands: Bt, Dt (N x N, offsets -1..2,
// B^ = Bt^T, D^ = Dt^T) and C02 (rows N, cols nh, offsets 0..2).
DiagRight diag_right(const CBand& Bt, const CBand& Dt, const CBand& C02, int N, int nh);

// Mass-only pair (Helmholtz scale 0, solvers.cpp:57-62, 84-91): X = A^-1 E B^^-1 with A = Ab (R2 recombined, one
// parity block) and B^ = Bt^T (C02 recombined), in the same four-product form u = QL [(PL f PR) .* 1] QR:
// PL = A^-1 R2m (M x mh), QL = S_r (mh x M), lambda = 1; PR = C02m B^^-1 (nh x N), QR = S_z^T (N x nh), mu = 0
// (R2b / C02b as in diag_left / diag_right; identity bands give the raw, truncated right-hand side).
DiagLeft mass_left(const CBand& Ab, const CBand& R2b, int M, int mh);
DiagRight mass_right(const CBand& Bt, const CBand& C02b, int N, int nh);

}  // namespace ccf
