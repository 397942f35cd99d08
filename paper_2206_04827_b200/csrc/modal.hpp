// Host builder for the packed per-slot operator blocks consumed by adi_kernel
// (layout documented in ccf_device.cuh::AdiSlot).
//   ModalSolver ctor   proj/src/solvers.cpp:46-75
//   AdiWorkspace ctor  proj/src/adi.cpp:114-148
#pragma once

#include <map>
#include <vector>

#include "ccf_device.cuh"
#include "diag.hpp"
#include "setup.hpp"

namespace ccf {

struct SizeOps {  // per-size operator cache (setup only)
    int m = 0, n = 0;
    Ultra ur, uz;
    Dense R2rec, C02recZ, D2recZ;  // recombined full operators
    Range vertical;                // padded enclosure of spec(-D2', C02')
    bool vertical_ok = false;
    // fast-diagonalization cache: the radial eigenpairs of the Poisson pencil (L_w, R2) per |w| (every
    // Helmholtz pencil R2 - s L_w, -s R2 has the same eigenvectors, lambda = nu - 1/s), and the
    // vertical data per k-parity; sharing them makes all solver sets use one modal basis
    std::map<int, DiagLeft> diag_poisson;
    bool diag_right_ok = false;
    DiagRight diag_right_data[2];
    SizeOps(int m_, int n_);
};

// Radial pencil range for (m, w^2): enclosure of spec(R2'^-1 L_w'), solvers.cpp:15-28.
Range radial_range(const SizeOps& so, int w, bool q2_pad);
Range vertical_range(SizeOps& so, bool q2_pad);

struct SlotPlan {
    int w = 0;
    Plan plan;
    bool has_plan = false;
};

// A "solver set": one (poisson | helmholtz scale) family over a list of slots.
struct SolverSet {
    bool poisson = true;
    double scale = 1.0, tol = 1e-12;
    std::vector<SlotPlan> plans;   // per slot
    std::vector<AdiSlot> slots;    // per slot descriptors
    std::vector<double> coef;      // packed blocks (host copy)
    int maxJ = 0;
    long iters_per_round = 0;      // sum over slots of J (one round)
    // fast-diagonalization data (diag.hpp), when built: per slot [PL | QL | lam], per k-parity
    // [PR | QR | mu], all in `dg` (offsets in doubles, 16-byte aligned)
    bool has_diag = false;
    std::vector<double> dg;
    std::vector<long> dg_left;  // per slot
    long dg_right[2] = {0, 0};
};

// Build the packed set. slot_w: wavenumber per slot. radial: cached radial
// ranges per |w| (computed on demand). Throws ccf::Error on reference failures
// (overlapping intervals -> DOMAIN_ERROR, singular operators -> SINGULAR).
// plan_margin: executed shifts planned for tol / plan_margin (1 = the reference's shift count).
// with_diag: also build the fast-diagonalization data (diag.hpp). with_adi = false: only the diagonalization
// data (no enclosures, shift plans or ADI blocks: any size, fast setup; the ADI kernel cannot run on the set).
// keep_static = false (with with_adi = false): not even the static operator bands of diag_check_residual.
SolverSet build_solver_set(SizeOps& so, const std::vector<int>& slot_w, bool poisson, double scale, double tol,
                           std::map<int, Range>& radial_cache, bool q2_pad, double plan_margin = 1.0,
                           bool with_diag = false, bool with_adi = true, bool keep_static = true);

// Host check of the packed fast-diagonalization data of one (slot, k-parity) sub-problem: for a
// seeded random RHS f (mh x nh), u = QL [(PL f PR) .* RT] QR in double (the device arithmetic),
// X = S_r^-1 u S_z^-T, and the relative Sylvester residual ||A X B^ + C X D^ - R2 f C02^T|| /
// ||R2 f C02^T|| in long double from the static operator blocks the ADI kernel uses.
double diag_check_residual(const SolverSet& set, int slot, int k0, int M, int N, unsigned long long seed);

}  // namespace ccf
