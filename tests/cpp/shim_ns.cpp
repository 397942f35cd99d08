// Drop-in check of include/cylspec_b200.hpp: the reference-API program shape (cylspec_main.cpp
// run_poisson / run_ns) compiled against the B200 shim. Prints results for the GPU test to verify.
#include <cmath>
#include <cstdio>
#include <random>

#include "cylspec_b200.hpp"

using namespace cylspec;

int main(int argc, char** argv) {
    const int m = argc > 1 ? std::atoi(argv[1]) : 16;
    GridSpec spec(m, m, m);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd(0.0, 1.0);
    CoeffTensor f(spec);
    for (int l = spec.p / 2; l < spec.p; ++l)
        for (int k = 0; k < spec.n; ++k)
            for (int j = 0; j < spec.m; ++j) {
                const int w = spec.wavenumber(l);
                if ((j + w) % 2) continue;
                const double d = std::pow(0.7, j + k + w);
                const Complex v(nd(rng) * d, w == 0 ? 0.0 : nd(rng) * d);
                f.at(j, k, l) = v;
                if (w > 0) f.at(j, k, spec.p - l) = std::conj(v);
            }
    CoeffTensor u = solve_poisson_3d(f, BoundaryCondition::homogeneous());
    GridField g = synthesize(u);
    CoeffTensor back = analyze(g);
    double err = 0, mx = 0;
    for (size_t i = 0; i < u.data.size(); ++i) {
        err = std::max(err, std::abs(back.data[i] - u.data[i]));
        mx = std::max(mx, std::abs(u.data[i]));
    }
    NSConfig nc;
    nc.spec = spec;
    nc.reynolds = 100.0;
    nc.h = 1e-3;
    NSRunResult run = ns_run(nc, curl_pt(PTScalars(f, u)), 3);
    // ns_run with the substeps bootstrap (ptns.cpp:272-311) equals its restatement from the public pieces
    // (fine BDF2 run, replayed nonlinear terms, NSStepper::seed), and seed() refuses an empty history
    NSConfig ns3 = nc;
    ns3.order = 3;
    ns3.bootstrap = NSBootstrap::substeps;
    // (small amplitude: the reference's explicit nonlinear term lets O(1) data blow up within the 64 fine steps)
    PTScalars w0 = curl_pt(PTScalars(f, u));
    w0.lambda *= Complex(1e-3);
    w0.gamma *= Complex(1e-3);
    NSRunResult sub = ns_run(ns3, w0, 4, 2);
    double seed_err = 1.0;
    bool seed_threw = false;
    {
        NSConfig fine_c = ns3;
        fine_c.order = 2;
        fine_c.h = ns3.h / 32;
        fine_c.bootstrap = NSBootstrap::ramp;
        std::deque<PTScalars> hist{w0}, replay;
        {
            NSStepper fine(fine_c, w0);
            for (int big = 1; big <= 2; ++big) {
                fine.steps(32);
                hist.push_front(fine.omega());
            }
        }
        for (int i = 2; i >= 1; --i) replay.push_front(nonlinear_term(velocity_from_vorticity(hist[size_t(i)]), hist[size_t(i)]));
        NSStepper st(ns3, hist.front());
        st.seed(hist, replay, 2 * ns3.h, 2);
        st.steps(2);
        const PTScalars& o = st.omega();
        double d = 0, mxo = 0;
        for (size_t i = 0; i < o.lambda.data.size(); ++i) {
            d = std::max({d, std::abs(o.lambda.data[i] - sub.final_omega.lambda.data[i]),
                          std::abs(o.gamma.data[i] - sub.final_omega.gamma.data[i])});
            mxo = std::max({mxo, std::abs(o.lambda.data[i]), std::abs(o.gamma.data[i])});
        }
        seed_err = d / mxo;
        try {
            st.seed({}, {}, 0.0, 0);
        } catch (const DomainError&) {
            seed_threw = true;
        }
    }
    const bool seed_ok = seed_err < 1e-13 && seed_threw && sub.snapshots.size() == 1 && sub.snapshot_times.size() == 1 &&
                         std::abs(sub.snapshot_times[0] - 4 * ns3.h) < 1e-15 && std::abs(sub.final_time - 4 * ns3.h) < 1e-15;
    // per-mode API, the reference's own cases (test_solvers.cpp:13-17, 46-105) through the shim types
    double modal_err = 0.0;
    bool modal_ok = true;
    {
        auto dense_apply = [](const std::vector<double>& A, int na, const MatrixXcd& x, const std::vector<double>& B, int nb) {
            MatrixXcd t(na, nb), y(na, nb);  // y = A x B (row-major dense A: na x na, B: nb x nb)
            for (int i = 0; i < na; ++i)
                for (int k = 0; k < nb; ++k)
                    for (int j = 0; j < na; ++j) t(i, k) += A[size_t(i) * na + j] * x(j, k);
            for (int i = 0; i < na; ++i)
                for (int k = 0; k < nb; ++k)
                    for (int j = 0; j < nb; ++j) y(i, k) += t(i, j) * B[size_t(j) * nb + k];
            return y;
        };
        const int mm = 12, nn = 12;
        const double q[3] = {0.5, 0.0, -0.5};
        auto manufactured = [&](double s, double wall, MatrixXcd& u) {
            u = MatrixXcd::Zero(mm, nn);
            MatrixXcd lap = MatrixXcd::Zero(mm, nn);
            for (int j = 0; j < 3; ++j)
                for (int k = 0; k < 3; ++k) u(j, k) += q[j] * q[k];
            u(0, 0) += wall;
            for (int k = 0; k < 3; ++k) lap(0, k) += -4.0 * q[k];
            for (int j = 0; j < 3; ++j) lap(j, 0) += -2.0 * q[j];
            return u - Complex(s) * lap;
        };
        // modal_rhs: F = R2 g C02^T; the Poisson quadruple carries C = R2 and B = C02^T
        const ModalOperator pop = assemble_modal_poisson(mm, nn, 0);
        auto modal_rhs = [&](const MatrixXcd& g) { return dense_apply(pop.C, mm, g, pop.B, nn); };
        MatrixXcd u;
        {
            const MatrixXcd g = manufactured(0.05, 0.0, u);
            const ModalOperator op = assemble_modal_helmholtz(mm, nn, 0, 0.05);
            modal_err = std::max(modal_err, (solve_modal_helmholtz(op, modal_rhs(g), BoundaryCondition::homogeneous(), 1e-13) - u).max_abs());
            modal_ok = modal_ok && solve_modal_helmholtz(op, MatrixXcd::Zero(mm, nn), BoundaryCondition::homogeneous()).max_abs() == 0.0;
        }
        {
            const MatrixXcd g = manufactured(0.02, 1.0, u);
            CoeffTensor lift(GridSpec(mm, nn, 4));
            lift.at(0, 0, 2) = 1.0;
            const ModalOperator op = assemble_modal_helmholtz(mm, nn, 0, 0.02);
            modal_err = std::max(modal_err, (solve_modal_helmholtz(op, modal_rhs(g), BoundaryCondition::lifted(lift), 1e-13) - u).max_abs());
        }
        {
            ModalSolverCache cache(mm, nn, 1e-12);
            const ModalSolver& ms = cache.get(-3, 1.0, true);
            modal_ok = modal_ok && &ms == &cache.get(3, 1.0, true) && ms.plan() && ms.plan()->J > 0 &&
                       int(ms.plan()->u.size()) == ms.plan()->J && ModalSolver(mm, nn, 0, 0.0, false).plan() == nullptr;
            MatrixXcd frand(mm, nn);
            for (int k = 0; k < nn; ++k)
                for (int j = 0; j < mm; ++j) frand(j, k) = Complex(nd(rng), nd(rng)) * std::pow(0.8, j + k);
            ms.solve(frand);
            modal_ok = modal_ok && ms.last_residual() < 1e-12;
            try {
                ms.solve(MatrixXcd::Zero(mm, nn + 2));
                modal_ok = false;
            } catch (const DomainError&) {
            }
        }
        // lifted 3-D Poisson: u = lift + homogeneous part; the wall values are the lift's (u - lift vanishes there)
        {
            CoeffTensor lift(spec);
            lift.at(0, 0, spec.zero_mode()) = 1.0;
            lift.at(2, 1, spec.zero_mode()) = 0.25;
            const CoeffTensor ul = solve_poisson_3d(f, BoundaryCondition::lifted(lift));
            double wall = 0.0;  // r = 1: sum_j (u - lift)(j, k, l) = 0 for every k, l
            for (int l = 0; l < spec.p; ++l)
                for (int k = 0; k < spec.n; ++k) {
                    Complex acc(0);
                    for (int j = 0; j < spec.m; ++j)
                        if ((j + spec.wavenumber(l)) % 2 == 0) acc += ul.at(j, k, l) - lift.at(j, k, l);
                    wall = std::max(wall, std::abs(acc));
                }
            modal_ok = modal_ok && wall < 1e-11 * std::max(1.0, ul.max_abs());
        }
        // pt_decompose(check_divergence): a non-solenoidal field is refused (ptns.cpp:60-67)
        {
            VectorFieldCoeffs bad(spec);
            bad.comp_z = f;
            bool refused = false;
            try {
                pt_decompose(bad, true);
            } catch (const NotIncompressibleError& e) {
                refused = e.divergence > 0.0;
            }
            modal_ok = modal_ok && refused;
        }
        // coeffs.hpp helpers: a solver output is Hermitian and parity-clean; the flipped class is its complement
        {
            const CoeffTensor& wl = run.final_omega.lambda;
            const CoeffTensor flip = parity_project(wl, Parity::azimuthal_flip);
            modal_ok = modal_ok && hermitian_symmetry_error(wl) < 1e-13 * wl.max_abs() && wl.all_finite() &&
                       (parity_project(wl) - wl).max_abs() == 0.0 && flip.max_abs() == 0.0 &&
                       (Complex(2.0) * wl - wl - wl).max_abs() == 0.0;
        }
        modal_ok = modal_ok && modal_err < 1e-10;
    }
    bool threw = false;
    try {
        GridSpec bad(m, m, 7);
    } catch (const DomainError&) {
        threw = true;
    }
    // heat_run on the manufactured problem of test_timestep.cpp:151-187 (exact forcing at t + h)
    auto pt = [](int i, int c) { return std::cos(double(c - 1 - i) * M_PI / double(c - 1)); };
    auto field = [&](auto fn) {
        GridField gf(spec);
        for (int l = 0; l < spec.p; ++l)
            for (int k = 0; k < spec.n; ++k)
                for (int j = 0; j < spec.m; ++j)
                    gf.values[(size_t(l) * spec.n + k) * spec.m + j] = fn(pt(j, spec.m), pt(k, spec.n));
        return gf;
    };
    auto exact = [&](double t) { return field([t](double r, double z) { return std::exp(-t) * (1 - r * r) * (1 - z * z); }); };
    HeatConfig hc;
    hc.spec = spec;
    hc.alpha = 1.0;
    hc.h = 0.01;
    HeatRunResult hr = heat_run(hc, exact(0.0), [&](double t) {
        return field([t](double r, double z) {
            return -std::exp(-t) * (1 - r * r) * (1 - z * z) + std::exp(-t) * (4 * (1 - z * z) + 2 * (1 - r * r));
        });
    }, 100);
    const GridField ref = exact(hr.final_time);
    double herr = 0, hmx = 0;
    for (size_t i = 0; i < ref.values.size(); ++i) {
        herr = std::max(herr, std::abs(hr.snapshots.back().values[i] - ref.values[i]));
        hmx = std::max(hmx, std::abs(ref.values[i]));
    }
    // spec mismatches are DomainErrors with the reference messages (ptns.cpp:185-187, timestep.cpp:69-70,113-114)
    int spec_errors = 0;
    const GridSpec other(m, m, m + 2);
    auto expect = [&](auto fn, const char* msg) {
        try {
            fn();
        } catch (const DomainError& e) {
            spec_errors += std::string(e.what()).find(msg) != std::string::npos;
        }
    };
    expect([&] { NSStepper s(nc, PTScalars(CoeffTensor(other), CoeffTensor(other))); }, "NSStepper: initial vorticity spec mismatch");
    expect([&] { HeatStepper h(hc, GridField(other)); }, "HeatStepper: initial data spec mismatch");
    expect([&] { HeatStepper h(hc, CoeffTensor(other)); }, "HeatStepper: initial data spec mismatch");
    expect([&] {
        HeatStepper h(hc, exact(0.0));
        const CoeffTensor bad(other);
        h.step(&bad);
    }, "HelmholtzTensorStepper: forcing spec mismatch");
    expect([&] {
        HelmholtzTensorStepper hs(spec, 1.0, 0.01, 1e-12);
        std::deque<CoeffTensor> hist{CoeffTensor(spec)};
        const CoeffTensor bad(other);
        hs.step(hist, BDFScheme::of_order(1), &bad);
    }, "HelmholtzTensorStepper: forcing spec mismatch");
    expect([&] { nonlinear_term(PTScalars(f, u), PTScalars(CoeffTensor(other), CoeffTensor(other))); }, "spec mismatch");
    const bool spec_ok = spec_errors == 6 && hr.worst_residual > 0.0 && hr.worst_residual < 1e-12;
    // FieldFile round trip of the final NS vorticity (io.cpp:42-109)
    write_field("/tmp/shim_lambda.ccf", run.final_omega.lambda);
    const CoeffTensor rd = std::get<CoeffTensor>(read_field("/tmp/shim_lambda.ccf"));
    const bool io_ok = rd.data == run.final_omega.lambda.data && crc32_ieee(reinterpret_cast<const uint8_t*>("123456789"), 9) == 0xCBF43926u;
    std::printf("shim ok: roundtrip %.3e final_time %.6f domain_error %d heat_err %.3e io %d spec_errors %d/6 "
                "worst_residual %.3e seed %d (%.2e) modal %d (%.2e)\n", err / mx, run.final_time, int(threw), herr / hmx, int(io_ok), spec_errors,
                hr.worst_residual, int(seed_ok), seed_err, int(modal_ok), modal_err);
    return (err / mx < 1e-12 && threw && herr / hmx < 1e-4 && io_ok && spec_ok && seed_ok && modal_ok) ? 0 : 1;
}
