// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// extern "C" surface of the oracle for the Python test harness (ctypes).
// Tensors use the reference layout: index (l*n + k)*m + j, complex interleaved
// (re, im) for coefficients, plain f64 for grid values (proj/include/cylspec/coeffs.hpp:16-45).
#include <cstring>
#include <chrono>
#include <cmath>
#include <random>

#include "oracle.hpp"

using namespace oracle;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    if (dynamic_cast<const NonConvergenceError*>(&e)) return 4;
    if (dynamic_cast<const SingularOperatorError*>(&e)) return 3;
    if (dynamic_cast<const NotIncompressibleError*>(&e)) return 5;
    if (dynamic_cast<const NumericalError*>(&e)) return 6;
    if (dynamic_cast<const ConfigError*>(&e)) return 2;
    if (dynamic_cast<const DomainError*>(&e)) return 1;
    return 9;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

Coeff load(int m, int n, int p, const double* x) {
    Coeff c(Spec(m, n, p));
    std::memcpy(c.d.data(), x, c.d.size() * sizeof(cd));
    return c;
}
void store(const Coeff& c, double* x) { std::memcpy(x, c.d.data(), c.d.size() * sizeof(cd)); }
Field loadf(int m, int n, int p, const double* x) {
    Field f(Spec(m, n, p));
    std::memcpy(f.v.data(), x, f.v.size() * sizeof(double));
    return f;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_threads(n); }
void orc_set_eig_provider(EigProvider p) { set_eig_provider(p); }

int orc_points(int kind, int count, double* out) {
    return guard([&] {
        auto v = kind == 0 ? chebyshev_points(count) : fourier_points(count);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

int orc_analyze(int m, int n, int p, const double* vals, double* coef) {
    return guard([&] { store(analyze(loadf(m, n, p, vals)), coef); });
}

int orc_synthesize(int m, int n, int p, const double* coef, double* vals) {
    return guard([&] {
        Field f = synthesize(load(m, n, p, coef));
        std::memcpy(vals, f.v.data(), f.v.size() * 8);
    });
}

int orc_evaluate_at(int m, int n, int p, const double* coef, double r, double z, double th, double* out2) {
    return guard([&] {
        cd v = evaluate_at(load(m, n, p, coef), r, z, th);
        out2[0] = v.real();
        out2[1] = v.imag();
    });
}

// op: 0 d/dr, 1 d/dz, 2 d/dtheta, 3 multiply_r, 4 divide_r, 5 horizontal_laplacian, 6 laplacian
int orc_calculus(int op, int m, int n, int p, const double* in, double* out) {
    return guard([&] {
        Coeff f = load(m, n, p, in);
        Coeff o;
        switch (op) {
            case 0: o = derivative_r(f); break;
            case 1: o = derivative_z(f); break;
            case 2: o = derivative_theta(f); break;
            case 3: o = multiply_r(f); break;
            case 4: o = divide_r(f); break;
            case 5: o = horizontal_laplacian(f); break;
            case 6: o = laplacian(f); break;
            default: throw DomainError("orc_calculus: bad op");
        }
        store(o, out);
    });
}

int orc_parity_project(int m, int n, int p, int parity, double* inout) {
    return guard([&] {
        Coeff c = load(m, n, p, inout);
        parity_project_in_place(c, parity ? Parity::azimuthal_flip : Parity::scalar);
        store(c, inout);
    });
}

double orc_hermitian_error(int m, int n, int p, const double* coef) {
    return hermitian_symmetry_error(load(m, n, p, coef));
}

int orc_poisson3d(int m, int n, int p, double tol, const double* f, const double* lift, double* u) {
    return guard([&] {
        BoundaryCondition bc;
        if (lift) {
            bc.lifted = true;
            bc.lift = load(m, n, p, lift);
        }
        store(solve_poisson_3d(load(m, n, p, f), bc, tol), u);
    });
}

int orc_hpoisson(int m, int n, int p, const double* rhs, double* u) {
    return guard([&] { store(solve_horizontal_poisson(load(m, n, p, rhs)), u); });
}

int orc_pt_synthesize(int m, int n, int p, const double* lam, const double* gam, double* vr, double* vt, double* vz) {
    return guard([&] {
        Vec3 v = pt_synthesize({load(m, n, p, lam), load(m, n, p, gam)});
        store(v.r, vr);
        store(v.t, vt);
        store(v.z, vz);
    });
}

int orc_pt_decompose(int m, int n, int p, const double* vr, const double* vt, const double* vz, int check, double* lam,
                     double* gam) {
    return guard([&] {
        PT s = pt_decompose({load(m, n, p, vr), load(m, n, p, vt), load(m, n, p, vz)}, check != 0);
        store(s.lambda, lam);
        store(s.gamma, gam);
    });
}

int orc_curl_vector(int m, int n, int p, const double* r, const double* t, const double* z, double* orr, double* ot,
                    double* oz) {
    return guard([&] {
        Vec3 o = curl_vector({load(m, n, p, r), load(m, n, p, t), load(m, n, p, z)});
        store(o.r, orr);
        store(o.t, ot);
        store(o.z, oz);
    });
}

int orc_divergence(int m, int n, int p, const double* r, const double* t, const double* z, double* out) {
    return guard([&] { store(divergence({load(m, n, p, r), load(m, n, p, t), load(m, n, p, z)}), out); });
}

int orc_curl_pt(int m, int n, int p, const double* lam, const double* gam, double* ol, double* og) {
    return guard([&] {
        PT o = curl_pt({load(m, n, p, lam), load(m, n, p, gam)});
        store(o.lambda, ol);
        store(o.gamma, og);
    });
}

int orc_velocity_from_vorticity(int m, int n, int p, double tol, const double* wl, const double* wg, double* vl,
                                double* vg) {
    return guard([&] {
        ModalSolverCache cache(m, n, tol);
        PT v = velocity_from_vorticity({load(m, n, p, wl), load(m, n, p, wg)}, cache);
        store(v.lambda, vl);
        store(v.gamma, vg);
    });
}

int orc_nonlinear(int m, int n, int p, const double* vl, const double* vg, const double* wl, const double* wg,
                  int dealias, double* ol, double* og) {
    return guard([&] {
        PT o = nonlinear_term({load(m, n, p, vl), load(m, n, p, vg)}, {load(m, n, p, wl), load(m, n, p, wg)}, dealias != 0);
        store(o.lambda, ol);
        store(o.gamma, og);
    });
}

// ---- per-mode solver API (solvers.hpp:35-82): f, x are m x n complex, column-major
namespace {
MatC load_mat(int m, int n, const double* x) {
    MatC a(m, n);
    std::memcpy(a.a.data(), x, a.a.size() * sizeof(cd));
    return a;
}
}  // namespace
// ModalSolver(m, n, w, scale, poisson, tol).solve(f_full) (solvers.cpp:46-98); scale 0: the mass pair
int orc_modal_solve(int m, int n, int w, double scale, int poisson, double tol, const double* f, double* x, double* resid) {
    return guard([&] {
        ModalSolver s(m, n, w, scale, poisson != 0, tol);
        const MatC out = s.solve(load_mat(m, n, f));
        std::memcpy(x, out.a.data(), out.a.size() * sizeof(cd));
        if (resid) *resid = s.last_residual();
    });
}
// ModalOperator::apply (ultraop.cpp:83-87) of assemble_modal_poisson / assemble_modal_helmholtz
int orc_modal_apply(int m, int n, int w, double scale, int poisson, const double* x, double* y) {
    return guard([&] {
        const ModalOperator op = poisson ? assemble_modal_poisson(m, n, w) : assemble_modal_helmholtz(m, n, w, scale);
        const MatC out = op.apply(load_mat(m, n, x));
        std::memcpy(y, out.a.data(), out.a.size() * sizeof(cd));
    });
}
// solve_modal_helmholtz (solvers.cpp:125-140) with optional lifted boundary data (a p-mode tensor)
int orc_modal_helmholtz(int m, int n, int w, double scale, double tol, const double* f, int lift_p, const double* lift,
                        double* x) {
    return guard([&] {
        BoundaryCondition bc;
        if (lift) {
            bc.lifted = true;
            bc.lift = load(m, n, lift_p, lift);
        }
        const MatC out = solve_modal_helmholtz(assemble_modal_helmholtz(m, n, w, scale), load_mat(m, n, f), bc, tol);
        std::memcpy(x, out.a.data(), out.a.size() * sizeof(cd));
    });
}

// history: `order` (>= scheme order) tensors, newest first; lift: optional lifted boundary data (timestep.cpp:52-59)
int orc_helmholtz_step_lifted(int m, int n, int p, double diffusivity, double h, double tol, int order, int nhist,
                              const double* const* hist, const double* forcing, const double* lift, double* out) {
    return guard([&] {
        BoundaryCondition bc;
        if (lift) {
            bc.lifted = true;
            bc.lift = load(m, n, p, lift);
        }
        HelmholtzTensorStepper st(Spec(m, n, p), diffusivity, h, tol, bc);
        std::deque<Coeff> hd;
        for (int i = 0; i < nhist; ++i) hd.push_back(load(m, n, p, hist[i]));
        Coeff f;
        if (forcing) f = load(m, n, p, forcing);
        store(st.step(hd, BDFScheme::of_order(order), forcing ? &f : nullptr), out);
    });
}

// history: `order` (>= scheme order) tensors, newest first.
int orc_helmholtz_step(int m, int n, int p, double diffusivity, double h, double tol, int order, int nhist,
                       const double* const* hist, const double* forcing, double* out) {
    return guard([&] {
        HelmholtzTensorStepper st(Spec(m, n, p), diffusivity, h, tol);
        std::deque<Coeff> hd;
        for (int i = 0; i < nhist; ++i) hd.push_back(load(m, n, p, hist[i]));
        Coeff f;
        if (forcing) f = load(m, n, p, forcing);
        store(st.step(hd, BDFScheme::of_order(order), forcing ? &f : nullptr), out);
    });
}

// ---- NS stepper handle
void* orc_ns_create(int m, int n, int p, double re, double h, int order, double tol, int disable_nonlinear,
                    const double* lam0, const double* gam0) {
    try {
        NSConfig cfg;
        cfg.spec = Spec(m, n, p);
        cfg.reynolds = re;
        cfg.h = h;
        cfg.order = order;
        cfg.tol = tol;
        cfg.disable_nonlinear = (disable_nonlinear & 1) != 0;  // flags: bit 0 disable_nonlinear, bit 1 dealias
        cfg.dealias = (disable_nonlinear & 2) != 0;
        return new NSStepper(cfg, {load(m, n, p, lam0), load(m, n, p, gam0)});
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int orc_ns_step(void* h, int nsteps) {
    return guard([&] {
        for (int i = 0; i < nsteps; ++i) static_cast<NSStepper*>(h)->step();
    });
}
int orc_ns_get(void* h, double* lam, double* gam, double* time, int* steps) {
    return guard([&] {
        auto* s = static_cast<NSStepper*>(h);
        store(s->omega().lambda, lam);
        store(s->omega().gamma, gam);
        if (time) *time = s->time();
        if (steps) *steps = s->steps_taken();
    });
}
void orc_ns_destroy(void* h) { delete static_cast<NSStepper*>(h); }
// NSStepper::seed (ptns.cpp:195-203): nom omega pairs and nnl nonlinear pairs, newest first
int orc_ns_seed(void* h, int m, int n, int p, int nom, const double* const* lam_h, const double* const* gam_h, int nnl,
                const double* const* nl_l, const double* const* nl_g, double time, int steps) {
    return guard([&] {
        std::deque<PT> oh, nh;
        for (int i = 0; i < nom; ++i) oh.push_back({load(m, n, p, lam_h[i]), load(m, n, p, gam_h[i])});
        for (int i = 0; i < nnl; ++i) nh.push_back({load(m, n, p, nl_l[i]), load(m, n, p, nl_g[i])});
        static_cast<NSStepper*>(h)->seed(std::move(oh), std::move(nh), time, steps);
    });
}
// ns_run (ptns.cpp:269-324); flags: bit 0 disable_nonlinear, bit 1 dealias, bit 2 NSBootstrap::substeps
int orc_ns_run(int m, int n, int p, double re, double h, int order, double tol, int flags, const double* lam0,
               const double* gam0, int steps, double* lam, double* gam, double* time) {
    return guard([&] {
        NSConfig cfg;
        cfg.spec = Spec(m, n, p);
        cfg.reynolds = re;
        cfg.h = h;
        cfg.order = order;
        cfg.tol = tol;
        cfg.disable_nonlinear = (flags & 1) != 0;
        cfg.dealias = (flags & 2) != 0;
        const PT out = ns_run(cfg, {load(m, n, p, lam0), load(m, n, p, gam0)}, steps, (flags & 4) != 0, time);
        store(out.lambda, lam);
        store(out.gamma, gam);
    });
}

// ---- heat stepper handle (HeatStepper, proj/src/timestep.cpp:110-144)
void* orc_heat_create(int m, int n, int p, double alpha, double h, int order, double tol, const double* initial_coef) {
    try {
        HeatConfig cfg;
        cfg.spec = Spec(m, n, p);
        cfg.alpha = alpha;
        cfg.h = h;
        cfg.order = order;
        cfg.tol = tol;
        return new HeatStepper(cfg, load(m, n, p, initial_coef));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int orc_heat_step(void* h, const double* forcing_coef) {
    return guard([&] {
        auto* s = static_cast<HeatStepper*>(h);
        if (forcing_coef) {
            const Spec sp = s->current().s;
            Coeff f = load(sp.m, sp.n, sp.p, forcing_coef);
            s->step(&f);
        } else {
            s->step(nullptr);
        }
    });
}
int orc_heat_get(void* h, double* coef, double* time, int* order) {
    return guard([&] {
        auto* s = static_cast<HeatStepper*>(h);
        store(s->current(), coef);
        if (time) *time = s->time();
        if (order) *order = s->current_order();
    });
}
void orc_heat_destroy(void* h) { delete static_cast<HeatStepper*>(h); }

// ---- shift plans (proj/src/adi.cpp:68-104) and modal solver plans (solvers.cpp:46-75)
// info[0..7] = a, b, c, d, gamma, alpha, modulus, J ; u, v sized >= J (cap)
int orc_compute_shifts(double a, double b, double c, double d, double tol, double* info, double* u, double* v, int cap) {
    return guard([&] {
        ShiftPlan p = compute_shifts({a, b}, {c, d}, tol);
        double vals[8] = {p.a, p.b, p.c, p.d, p.gamma_cr, p.alpha_z, p.modulus, double(p.J)};
        std::memcpy(info, vals, sizeof vals);
        for (int j = 0; j < p.J && j < cap; ++j) {
            u[j] = p.u[size_t(j)];
            v[j] = p.v[size_t(j)];
        }
    });
}

int orc_modal_plan(int m, int n, int w, double scale, int poisson, double tol, double* info, double* u, double* v, int cap) {
    return guard([&] {
        ModalSolver s(m, n, w, scale, poisson != 0, tol);
        const ShiftPlan* p = s.plan();
        if (!p) throw DomainError("orc_modal_plan: mass solver has no plan");
        double vals[8] = {p->a, p->b, p->c, p->d, p->gamma_cr, p->alpha_z, p->modulus, double(p->J)};
        std::memcpy(info, vals, sizeof vals);
        for (int j = 0; j < p->J && j < cap; ++j) {
            u[j] = p->u[size_t(j)];
            v[j] = p->v[size_t(j)];
        }
    });
}

int orc_pencil_range(int kind, int size, int w, double* lohi) {
    return guard([&] {
        auto r = kind == 0 ? radial_pencil_range(size, w) : vertical_pencil_range(size);
        lohi[0] = r.first;
        lohi[1] = r.second;
    });
}

// Reference test_adi.cpp:22-45 helmholtz_problem + plan_for, solved by ADI and the dense oracle.
int orc_adi_vs_dense(int m, int n, int w, double scale, unsigned seed, double tol, double* rel, double* resid, int* iters) {
    return guard([&] {
        ModalOperator op = assemble_modal_helmholtz(m, n, w, scale);
        SylvesterProblem p;
        p.A = recombine(op.A);
        p.C = recombine(op.C);
        p.B = recombine(op.B.transposed()).transposed();
        p.D = recombine(op.D.transposed()).transposed();
        std::mt19937_64 rng(seed);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        p.E = MatC(m - 2, n - 2);
        for (int j = 0; j < m - 2; ++j)
            for (int k = 0; k < n - 2; ++k) {
                const double re = dist(rng);
                const double im = dist(rng);
                p.E(j, k) = cd(re, im);
            }
        auto ca = spectral_bounds(p.A, p.C);
        Banded negD = p.D.transposed();
        negD *= -1.0;
        auto db = spectral_bounds(negD, p.B.transposed());
        ShiftPlan plan = compute_shifts(ca, db, tol);
        AdiResult r = adi_solve_detailed(p, plan);
        MatC ref = dense_sylvester_oracle(p);
        double num = 0, den = 0;
        for (size_t i = 0; i < ref.a.size(); ++i) {
            num += std::norm(r.X.a[i] - ref.a[i]);
            den += std::norm(ref.a[i]);
        }
        *rel = std::sqrt(num / den);
        *resid = r.history.back();
        *iters = r.iterations;
    });
}

// which: 0 C01, 1 C12, 2 C02, 3 R, 4 R2, 5 D1, 6 D2, 7 S (n x n-2)
int orc_operator_dense(int n, int which, double* out) {
    return guard([&] {
        Banded b;
        const UltraOps& o = UltraOps::get(n);
        switch (which) {
            case 0: b = o.c01; break;
            case 1: b = o.c12; break;
            case 2: b = o.c02; break;
            case 3: b = o.r; break;
            case 4: b = o.r2; break;
            case 5: b = o.d1; break;
            case 6: b = o.d2; break;
            case 7: b = dirichlet_recombination(n); break;
            default: throw DomainError("orc_operator_dense: bad which");
        }
        auto d = b.dense();
        std::memcpy(out, d.data(), d.size() * 8);
    });
}

// Recombined radial pencil (L_w', R2') or vertical pencil (-D2', C02') as dense (size-2)^2 matrices.
int orc_pencil_dense(int kind, int size, int w, double* A, double* C) {
    return guard([&] {
        const UltraOps& o = UltraOps::get(size);
        Banded a, c;
        if (kind == 0) {
            a = recombine(radial_modal_laplacian(size, w));
            c = recombine(o.r2);
        } else {
            a = recombine(o.d2);
            a *= -1.0;
            c = recombine(o.c02);
        }
        auto da = a.dense(), dc = c.dense();
        std::memcpy(A, da.data(), da.size() * 8);
        std::memcpy(C, dc.data(), dc.size() * 8);
    });
}

double orc_elliptic_K(double k) {
    try {
        return elliptic_K(k);
    } catch (...) {
        return -1.0;
    }
}
int orc_jacobi(double u, double k, double* out3) {
    return guard([&] {
        Jacobi j = jacobi_elliptic(u, k);
        out3[0] = j.sn;
        out3[1] = j.cn;
        out3[2] = j.dn;
    });
}
int orc_mobius_from_points(const double* s, const double* t, double* coef4) {
    return guard([&] {
        Mobius mm = mobius_from_points({s[0], s[1], s[2], s[3]}, {t[0], t[1], t[2], t[3]});
        for (int i = 0; i < 4; ++i) coef4[i] = mm.c[size_t(i)];
    });
}

void orc_adi_stats(long* solves, long* iterations, int* max_rounds, double* worst) {
    AdiStats s = adi_stats();
    *solves = s.solves;
    *iterations = s.iterations;
    *max_rounds = s.max_rounds;
    *worst = s.worst_residual;
}
void orc_adi_stats_reset() { adi_stats_reset(); }

uint32_t orc_crc32(const uint8_t* data, size_t len) { return crc32_ieee(data, len); }

// ---- bounded CPU-baseline sample of one NS step (bench.py cpu_baseline / --impl reference).
// Times, at full size: the modal solves (RHS assembly R2 f C02^T + ModalSolver::solve) of
// `ns` sampled Fourier slices for the Poisson (velocity) and Helmholtz (BDF4, nu = 1/Re)
// solvers, one analyze and one synthesize. Solver setup (QZ bounds, factorizations) is not
// timed (it is cached across steps in the reference, ModalSolverCache).
// out: [t_poisson_sample, t_helmholtz_sample (one tensor), t_analyze, t_synthesize, J_poisson_mean, J_helm_mean]
int orc_ns_step_sample(int m, int n, int p, double re, double h, int ns, int threads, unsigned seed, double* out) {
    return guard([&] {
        set_threads(threads);
        const Spec s(m, n, p);
        const double scale = (12.0 / 25.0) * h / re;
        ModalSolverCache cache(m, n, 1e-12);
        std::vector<int> slices;
        for (int i = 0; i < ns; ++i) slices.push_back(int((long(i) * p) / ns));
        std::mt19937_64 rng(seed);
        std::normal_distribution<double> nd(0.0, 1.0);
        std::vector<MatC> rhs;
        for (int l : slices) {
            MatC f(m, n);
            const int w = s.wavenumber(l);
            for (int k = 0; k < n; ++k)
                for (int j = 0; j < m; ++j)
                    if (((j + w) % 2 + 2) % 2 == 0) f(j, k) = cd(nd(rng), nd(rng)) * std::pow(0.9, j + k + std::abs(w));
            rhs.push_back(f);
        }
        double jp = 0, jh = 0;
        for (int l : slices) {  // setup (untimed)
            jp += cache.get(s.wavenumber(l), 1.0, true).plan()->J;
            jh += cache.get(s.wavenumber(l), scale, false).plan()->J;
        }
        const UltraOps& ro = UltraOps::get(m);
        const Banded c02t = UltraOps::get(n).c02.transposed();
        auto run = [&](bool poisson) {
            const auto t0 = std::chrono::steady_clock::now();
            parallel_for(long(slices.size()), [&](long i) {
                const ModalSolver& sv = cache.get(s.wavenumber(slices[size_t(i)]), poisson ? 1.0 : scale, poisson);
                MatC ff = c02t.apply_right(ro.r2.apply_left(rhs[size_t(i)]));
                MatC x = sv.solve(ff);
                (void)x;
            });
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        };
        out[0] = run(true);
        out[1] = run(false);
        Field f(s);
        for (double& v : f.v) v = nd(rng);
        auto t0 = std::chrono::steady_clock::now();
        Coeff c = analyze(f);
        out[2] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        t0 = std::chrono::steady_clock::now();
        Field g = synthesize(c);
        out[3] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        out[4] = jp / double(slices.size());
        out[5] = jh / double(slices.size());
        set_threads(1);
    });
}

}  // extern "C"
