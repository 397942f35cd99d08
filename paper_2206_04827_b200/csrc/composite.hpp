// Composite radial operators of the NS nonlinear term (host builder).
//
// Every radial step of pt_synthesize (proj/src/ptns.cpp:42-57) and of curl_vector +
// pt_decompose (ptns.cpp:25-33, 59-77) is linear along the compressed radial index jj of
// one Fourier slot: derivative_r, divide_r (quirk Q1: Re part only on 0 < w < p/2),
// w-multiplications from derivative_theta, and the horizontal Poisson solve. Per slot the
// whole radial program is therefore one small dense matrix per (input field, plane) ->
// (output field, plane) pair. We obtain those matrices exactly as the device pencil kernels
// define them, by running host mirrors of the pencil programs (same recurrences, long double)
// on basis vectors, and fold the r synthesis (values at r_jr > 0) resp. r analysis into them.
// The NS nonlinear term then runs as batched DMMA GEMMs (sum over terms per output block)
// instead of sequential O(m) recurrences per pencil.
#pragma once

#include <vector>

namespace ccf {

struct CompositeTerm {
    int out;   // output field * 2 + plane
    int in;    // input tensor * 2 + plane
    long off;  // offset of the mh x mh block (row-major) in CompositeSet::blocks
};

struct CompositeSet {
    int mh = 0, nslots = 0;
    std::vector<double> blocks;
    std::vector<std::vector<CompositeTerm>> terms;  // per slot
};

struct RadialTables {  // host copies of the device tables (TransformPlan)
    int m = 0, mh = 0, M = 0, p = 0, nslots = 0;
    std::vector<double> q;        // mh: interpolant of 1/r (divide_r, even -> odd)
    std::vector<double> hpc;      // nslots x M x 8: horizontal-Poisson LU rows per slot
    std::vector<double> hpr;      // 2 x M x 8: R R C02 rows per parity
    std::vector<double> SrT[2];   // [j0] mh x mh: [jr][i] synthesis at r_{mh+jr}
    std::vector<double> ArT[2];   // [j0] mh x mh: [i][jr] analysis
};

// Synthesis side: inputs (0 lambda, 1 gamma, 2 dz gamma) of one PT pair (coefficients in r,
// anything in z), outputs the r-values (0 V_r, 1 V_theta, 2 V_z) at r_{mh+jr}:
//   out[F][plane] = sum_terms block (mh_jr x mh_jj) * in[X][plane'].
CompositeSet build_synth_composite(const RadialTables& t);

// Analysis side: inputs the r-values of (0 a_r, 1 a_theta, 2 a_z, 3 dz a_r, 4 dz a_theta),
// outputs the PT coefficients (0 gamma, 1 lambda) of curl(a) (pt_decompose without the
// divergence check, as in nonlinear_term): block (mh_jj x mh_jr).
CompositeSet build_anal_composite(const RadialTables& t);

}  // namespace ccf
