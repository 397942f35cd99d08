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
    bool threw = false;
    try {
        GridSpec bad(m, m, 7);
    } catch (const DomainError&) {
        threw = true;
    }
    std::printf("shim ok: roundtrip %.3e final_time %.6f domain_error %d\n", err / mx, run.final_time, int(threw));
    return (err / mx < 1e-12 && threw) ? 0 : 1;
}
