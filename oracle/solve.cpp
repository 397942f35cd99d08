// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// ADI (proj/src/adi.cpp), modal solvers (proj/src/solvers.cpp),
// BDF/IMEX time stepping (proj/src/timestep.cpp), PT / Navier–Stokes (proj/src/ptns.cpp).
#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- stats
static std::mutex g_stats_mu;
static AdiStats g_stats;
void adi_stats_reset() {
    std::lock_guard<std::mutex> g(g_stats_mu);
    g_stats = AdiStats{};
}
AdiStats adi_stats() {
    std::lock_guard<std::mutex> g(g_stats_mu);
    return g_stats;
}

// ---------------------------------------------------------------- adi (proj/src/adi.cpp)
static EigProvider g_eig = nullptr;
void set_eig_provider(EigProvider p) { g_eig = p; }

void SylvesterProblem::check() const {  // adi.cpp:11-19
    const int m = A.rows(), n = B.rows();
    if (A.cols() != m || C.rows() != m || C.cols() != m) throw DomainError("SylvesterProblem: A/C must be square and equal-sized");
    if (B.cols() != n || D.rows() != n || D.cols() != n) throw DomainError("SylvesterProblem: B/D must be square and equal-sized");
    if (E.r != m || E.c != n) throw DomainError("SylvesterProblem: E must be m x n");
}

std::pair<double, double> spectral_bounds(const Banded& A, const Banded& C) {  // adi.cpp:22-49
    if (A.rows() != A.cols() || C.rows() != C.cols() || A.rows() != C.rows())
        throw DomainError("spectral_bounds: square equal-sized matrices required");
    if (!g_eig) throw std::runtime_error("oracle: no generalized eigenvalue provider registered");
    const int n = A.rows();
    std::vector<double> a = A.dense(), c = C.dense(), ar(static_cast<size_t>(n)), ai(static_cast<size_t>(n)), be(static_cast<size_t>(n));
    if (g_eig(n, a.data(), c.data(), ar.data(), ai.data(), be.data()) != 0)
        throw NumericalError("spectral_bounds: eigenvalue provider failed");
    double beta_max = 0.0;
    for (double b : be) beta_max = std::max(beta_max, std::abs(b));
    double lo = std::numeric_limits<double>::infinity(), hi = -lo, radius = 0.0, worst_imag = 0.0;
    for (int i = 0; i < n; ++i) {
        if (std::abs(be[size_t(i)]) <= 1e-13 * beta_max)
            throw SingularOperatorError("spectral_bounds: infinite eigenvalue (singular C)");
        const cd lam = cd(ar[size_t(i)], ai[size_t(i)]) / be[size_t(i)];
        radius = std::max(radius, std::abs(lam));
        worst_imag = std::max(worst_imag, std::abs(lam.imag()));
        lo = std::min(lo, lam.real());
        hi = std::max(hi, lam.real());
    }
    if (worst_imag > 1e-6 * radius) throw NumericalError("spectral_bounds: spectrum of C^-1 A is not real");
    const double pad = 1e-8 * std::max(1.0, hi - lo) + 1e-12 * radius;  // adi.cpp:47
    return {lo - pad, hi + pad};
}

std::pair<double, double> spectral_bounds_gershgorin(const Banded& A, const Banded& C) {  // adi.cpp:51-66
    const int n = A.rows();
    BandedLU luC(C);
    std::vector<double> m = A.dense();
    luC.solve_in_place_real(m, n);
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (int i = 0; i < n; ++i) {
        double rad = 0;
        for (int j = 0; j < n; ++j)
            if (j != i) rad += std::abs(m[size_t(j) * n + i]);
        lo = std::min(lo, m[size_t(i) * n + i] - rad);
        hi = std::max(hi, m[size_t(i) * n + i] + rad);
    }
    return {lo, hi};
}

ShiftPlan compute_shifts(std::pair<double, double> ca, std::pair<double, double> db, double tol) {  // adi.cpp:68-104
    ShiftPlan p;
    p.a = ca.first;
    p.b = ca.second;
    p.c = db.first;
    p.d = db.second;
    p.tol = tol;
    if (!(p.b < p.c || p.d < p.a)) throw DomainError("compute_shifts: spectral intervals overlap");
    if (!(tol > 0.0) || tol >= 1.0) throw DomainError("compute_shifts: tol must be in (0,1)");
    p.gamma_cr = std::abs(p.c - p.a) * std::abs(p.d - p.b) / (std::abs(p.c - p.b) * std::abs(p.d - p.a));
    const double g = p.gamma_cr;
    p.alpha_z = -1.0 + 2.0 * g + 2.0 * std::sqrt(g * g - g);
    const double alpha = p.alpha_z;
    const double kp = 1.0 / alpha;
    p.modulus = std::sqrt(std::max(0.0, (1.0 - kp) * (1.0 + kp)));
    p.J = std::max(1, int(std::ceil(std::log(16.0 * g) * std::log(4.0 / tol) / (std::numbers::pi * std::numbers::pi))));
    const double K = elliptic_K_from_kprime(kp);
    const Mobius T = mobius_from_points({-alpha, -1.0, 1.0, alpha}, {p.a, p.b, p.c, p.d});
    p.u.resize(size_t(p.J));
    p.v.resize(size_t(p.J));
    for (int j = 0; j < p.J; ++j) {
        const double arg = (2.0 * j + 1.0) / (2.0 * p.J) * K;
        const double dn = jacobi_elliptic_from_kprime(arg, kp).dn;
        p.u[size_t(j)] = T(-alpha * dn);
        p.v[size_t(j)] = T(alpha * dn);
    }
    return p;
}

static MatC add(MatC a, const MatC& b, double s = 1.0) {
    for (size_t i = 0; i < a.a.size(); ++i) a.a[i] += s * b.a[i];
    return a;
}
static MatC transpose(const MatC& x) {
    MatC t(x.c, x.r);
    for (int j = 0; j < x.c; ++j)
        for (int i = 0; i < x.r; ++i) t(j, i) = x(i, j);
    return t;
}

double sylvester_residual(const SylvesterProblem& p, const MatC& x) {  // adi.cpp:106-112
    MatC r = p.B.apply_right(p.A.apply_left(x));
    r = add(r, p.D.apply_right(p.C.apply_left(x)));
    r = add(r, p.E, -1.0);
    const double en = p.E.norm();
    return en > 0.0 ? r.norm() / en : r.norm();
}

AdiWorkspace::AdiWorkspace(const SylvesterProblem& shape, const ShiftPlan& plan)  // adi.cpp:114-148
    : plan_(plan), A_(shape.A), B_(shape.B), C_(shape.C), D_(shape.D) {
    if (int(plan.u.size()) != plan.J || int(plan.v.size()) != plan.J) throw DomainError("AdiWorkspace: malformed shift plan");
    luBt_.factorize(B_.transposed());
    try {
        luC_.factorize(C_);
    } catch (const SingularOperatorError&) {
        throw SingularOperatorError("AdiWorkspace: C is singular; ADI needs invertible C");
    }
    for (int j = 0; j < plan.J; ++j) {
        Banded sh = C_;
        sh *= plan.v[size_t(j)];
        sh -= A_;
        try {
            lu_shiftA_.emplace_back(sh);
        } catch (const SingularOperatorError&) {
            throw SingularOperatorError("ADI: singular (v_j C - A)", j);
        }
        Banded ubd = B_;
        ubd *= plan.u[size_t(j)];
        ubd += D_;
        try {
            lu_shiftBt_.emplace_back(ubd.transposed());
        } catch (const SingularOperatorError&) {
            throw SingularOperatorError("ADI: singular (u_j B + D)", j);
        }
    }
}

AdiResult AdiWorkspace::solve(const MatC& e) const {  // adi.cpp:150-202
    const int m = A_.rows(), n = B_.rows();
    if (e.r != m || e.c != n) throw DomainError("AdiWorkspace::solve: bad E");
    SylvesterProblem prob{A_, B_, C_, D_, e};
    AdiResult res;
    res.X = MatC(m, n);
    const double enorm = e.norm();
    if (enorm == 0.0) {
        res.history.push_back(0.0);
        return res;
    }
    const int J = plan_.J;
    for (int round = 0; round < 4; ++round) {
        for (int j = 0; j < J; ++j) {
            // (v_j C - A) X' B = C X (v_j B + D) - E           adi.cpp:166-175
            MatC cx = C_.apply_left(res.X);
            MatC rhs = add(D_.apply_right(cx), B_.apply_right(cx), plan_.v[size_t(j)]);
            rhs = add(rhs, e, -1.0);
            lu_shiftA_[size_t(j)].solve_in_place(rhs);
            MatC xt = transpose(rhs);
            luBt_.solve_in_place(xt);
            MatC xh = transpose(xt);
            // C X'' (u_j B + D) = (u_j C - A) X' B + E          adi.cpp:177-186
            MatC cxh = C_.apply_left(xh);
            MatC axh = A_.apply_left(xh);
            MatC t(m, n);
            for (size_t i = 0; i < t.a.size(); ++i) t.a[i] = plan_.u[size_t(j)] * cxh.a[i] - axh.a[i];
            MatC rhs2 = add(B_.apply_right(t), e);
            luC_.solve_in_place(rhs2);
            MatC x2t = transpose(rhs2);
            lu_shiftBt_[size_t(j)].solve_in_place(x2t);
            res.X = transpose(x2t);
        }
        res.iterations += J;
        const double rel = sylvester_residual(prob, res.X);
        res.history.push_back(rel);
        if (rel <= plan_.tol) return res;
    }
    const double fin = res.history.back();
    if (fin > 10.0 * plan_.tol) {
        res.converged = false;
        throw NonConvergenceError("ADI did not converge: relative residual " + std::to_string(fin) + " after " +
                                      std::to_string(res.iterations) + " iterations",
                                  res.history);
    }
    return res;
}

AdiResult adi_solve_detailed(const SylvesterProblem& p, const ShiftPlan& plan) {
    p.check();
    AdiWorkspace ws(p, plan);
    return ws.solve(p.E);
}

MatC dense_sylvester_oracle(const SylvesterProblem& p) {  // adi.cpp:214-255
    p.check();
    const int m = p.A.rows(), n = p.B.rows();
    if (long(m) * n > 4096) throw DomainError("dense_sylvester_oracle: m*n exceeds the 4096 guard");
    const auto a = p.A.dense(), b = p.B.dense(), c = p.C.dense(), d = p.D.dense();
    const long mn = long(m) * n;
    std::vector<double> K(static_cast<size_t>(mn * mn), 0.0);  // column-major
    auto Kat = [&](long i, long j) -> double& { return K[size_t(j * mn + i)]; };
    for (int jb = 0; jb < n; ++jb)
        for (int ib = 0; ib < n; ++ib) {
            const double wb = b[size_t(jb) * n + ib], wd = d[size_t(jb) * n + ib];
            if (wb == 0.0 && wd == 0.0) continue;
            for (int cc = 0; cc < m; ++cc)
                for (int rr = 0; rr < m; ++rr)
                    Kat(long(jb) * m + rr, long(ib) * m + cc) += wb * a[size_t(cc) * m + rr] + wd * c[size_t(cc) * m + rr];
        }
    // partial-pivot LU (stands in for Eigen::PartialPivLU)
    std::vector<long> perm(static_cast<size_t>(mn));
    for (long i = 0; i < mn; ++i) perm[size_t(i)] = i;
    for (long k = 0; k < mn; ++k) {
        long pr = k;
        double pm = std::abs(Kat(k, k));
        for (long i = k + 1; i < mn; ++i)
            if (std::abs(Kat(i, k)) > pm) {
                pm = std::abs(Kat(i, k));
                pr = i;
            }
        if (pr != k) {
            for (long j = 0; j < mn; ++j) std::swap(Kat(k, j), Kat(pr, j));
            std::swap(perm[size_t(k)], perm[size_t(pr)]);
        }
        const double piv = Kat(k, k);
        if (piv == 0.0) continue;
        for (long i = k + 1; i < mn; ++i) Kat(i, k) /= piv;
        for (long j = k + 1; j < mn; ++j) {
            const double f = Kat(k, j);
            if (f == 0.0) continue;
            for (long i = k + 1; i < mn; ++i) Kat(i, j) -= Kat(i, k) * f;
        }
    }
    double dmin = std::numeric_limits<double>::infinity(), dmax = 0;
    for (long i = 0; i < mn; ++i) {
        dmin = std::min(dmin, std::abs(Kat(i, i)));
        dmax = std::max(dmax, std::abs(Kat(i, i)));
    }
    if (dmin == 0.0 || dmin < 1e-14 * dmax) throw SingularOperatorError("dense_sylvester_oracle: singular system");
    MatC x(m, n);
    for (int part = 0; part < 2; ++part) {
        std::vector<double> v(static_cast<size_t>(mn));
        for (long i = 0; i < mn; ++i) {
            const cd e = p.E.a[size_t(perm[size_t(i)])];
            v[size_t(i)] = part == 0 ? e.real() : e.imag();
        }
        for (long i = 0; i < mn; ++i)
            for (long j = 0; j < i; ++j) v[size_t(i)] -= Kat(i, j) * v[size_t(j)];
        for (long i = mn - 1; i >= 0; --i) {
            for (long j = i + 1; j < mn; ++j) v[size_t(i)] -= Kat(i, j) * v[size_t(j)];
            v[size_t(i)] /= Kat(i, i);
        }
        for (long i = 0; i < mn; ++i) {
            if (part == 0) x.a[size_t(i)].real(v[size_t(i)]);
            else x.a[size_t(i)].imag(v[size_t(i)]);
        }
    }
    return x;
}

// ---------------------------------------------------------------- solvers (proj/src/solvers.cpp)
std::pair<double, double> radial_pencil_range(int m, int w) {  // solvers.cpp:15-28
    static std::mutex mu;
    static std::map<std::pair<int, int>, std::pair<double, double>> cache;
    const int w2 = w * w;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find({m, w2});
        if (it != cache.end()) return it->second;
    }
    const UltraOps& o = UltraOps::get(m);
    const Banded lw = recombine(radial_modal_laplacian(m, w));
    const Banded r2 = recombine(o.r2);
    auto range = spectral_bounds(lw, r2);
    std::lock_guard<std::mutex> g(mu);
    cache[{m, w2}] = range;
    return range;
}

std::pair<double, double> vertical_pencil_range(int n) {  // solvers.cpp:30-42
    static std::mutex mu;
    static std::map<int, std::pair<double, double>> cache;
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(n);
        if (it != cache.end()) return it->second;
    }
    const UltraOps& o = UltraOps::get(n);
    Banded negd2 = recombine(o.d2);
    negd2 *= -1.0;
    auto range = spectral_bounds(negd2, recombine(o.c02));
    std::lock_guard<std::mutex> g(mu);
    cache[n] = range;
    return range;
}

ModalSolver::ModalSolver(int m, int n, int w, double scale, bool poisson, double tol) {  // solvers.cpp:46-75
    op_ = poisson ? assemble_modal_poisson(m, n, w) : assemble_modal_helmholtz(m, n, w, scale);
    shape_.A = recombine(op_.A);
    shape_.B = recombine(op_.B.transposed()).transposed();
    shape_.C = recombine(op_.C);
    shape_.D = recombine(op_.D.transposed()).transposed();
    shape_.E = MatC(m - 2, n - 2);
    recomb_r_ = dirichlet_recombination(m);
    recomb_z_ = dirichlet_recombination(n);
    if (!poisson && scale == 0.0) {
        mass_lu_r_ = std::make_unique<BandedLU>(shape_.A);
        mass_lu_zt_ = std::make_unique<BandedLU>(shape_.B.transposed());
        return;
    }
    const auto [lo, hi] = radial_pencil_range(m, w);
    std::pair<double, double> ca = poisson ? std::make_pair(lo, hi) : std::make_pair(-1.0 / scale + lo, -1.0 / scale + hi);
    const auto cdr = vertical_pencil_range(n);
    plan_ = compute_shifts(ca, cdr, tol);
    adi_ = std::make_unique<AdiWorkspace>(shape_, *plan_);
}

MatC ModalSolver::solve(const MatC& f_full) const {  // solvers.cpp:77-98
    const int m = op_.m, n = op_.n;
    if (f_full.r != m || f_full.c != n) throw DomainError("ModalSolver::solve: right-hand side has wrong shape");
    MatC f(m - 2, n - 2);
    for (int k = 0; k < n - 2; ++k)
        for (int j = 0; j < m - 2; ++j) f(j, k) = f_full(j, k);
    MatC y;
    if (mass_lu_r_) {
        y = f;
        mass_lu_r_->solve_in_place(y);
        MatC yt = transpose(y);
        mass_lu_zt_->solve_in_place(yt);
        y = transpose(yt);
        SylvesterProblem chk = shape_;
        chk.E = f;
        last_residual_ = sylvester_residual(chk, y);
        last_iterations_ = 0;
    } else {
        AdiResult r = adi_->solve(f);
        y = std::move(r.X);
        last_residual_ = r.history.back();
        last_iterations_ = r.iterations;
        std::lock_guard<std::mutex> g(g_stats_mu);
        g_stats.solves++;
        g_stats.iterations += r.iterations;
        g_stats.max_rounds = std::max<int>(g_stats.max_rounds, int(r.history.size()));
        g_stats.worst_residual = std::max(g_stats.worst_residual, r.history.back());
    }
    return recomb_z_.transposed().apply_right(recomb_r_.apply_left(y));
}

const ModalSolver& ModalSolverCache::get(int w, double scale, bool poisson) const {  // solvers.cpp:100-109
    std::lock_guard<std::mutex> g(mu_);
    auto key = std::make_tuple(w * w, scale, poisson);
    auto& s = cache_[key];
    if (!s) s = std::make_unique<ModalSolver>(m_, n_, std::abs(w), scale, poisson, tol_);
    return *s;
}

static MatC slice_mat(const Coeff& t, int l) {
    MatC x(t.s.m, t.s.n);
    std::copy(t.slice(l), t.slice(l) + size_t(t.s.m) * t.s.n, x.a.begin());
    return x;
}

MatC solve_modal_helmholtz(const ModalOperator& op, const MatC& f, const BoundaryCondition& bc, double tol) {  // solvers.cpp:125-140
    ModalSolver solver(op.m, op.n, op.wavenumber, op.scale, false, tol);
    MatC rhs = f, lift;
    if (bc.lifted) {
        if (!bc.lift) throw DomainError("BoundaryCondition: lifted kind without lift data");
        lift = slice_mat(*bc.lift, op.wavenumber + bc.lift->s.p / 2);
        rhs = add(rhs, op.apply(lift), -1.0);
    }
    MatC x = solver.solve(rhs);
    if (!lift.a.empty()) x = add(x, lift);
    return x;
}

Coeff solve_poisson_3d(const Coeff& f, const BoundaryCondition& bc, const ModalSolverCache& cache) {  // solvers.cpp:142-169
    const Spec& s = f.s;
    if (!f.all_finite()) throw NumericalError("solve_poisson_3d: non-finite right-hand side");
    if (cache.m() != s.m || cache.n() != s.n) throw DomainError("solve_poisson_3d: cache size mismatch");
    const UltraOps& ro = UltraOps::get(s.m);
    const UltraOps& zo = UltraOps::get(s.n);
    const Banded c02t = zo.c02.transposed();
    Coeff rhs = parity_project(f);
    Coeff out(s);
    for (int l = 0; l < s.p; ++l) cache.get(s.wavenumber(l), 1.0, true);  // build solvers before the parallel loop
    parallel_for(s.p, [&](long li) {
        const int l = int(li);
        const ModalSolver& solver = cache.get(s.wavenumber(l), 1.0, true);
        MatC fl = slice_mat(rhs, l), lift;
        if (bc.lifted) lift = slice_mat(*bc.lift, l);
        MatC ff = c02t.apply_right(ro.r2.apply_left(fl));
        if (!lift.a.empty()) ff = add(ff, solver.raw().apply(lift), -1.0);
        MatC x = solver.solve(ff);
        if (!lift.a.empty()) x = add(x, lift);
        std::copy(x.a.begin(), x.a.end(), out.slice(l));
    });
    parity_project_in_place(out);
    return out;
}

Coeff solve_poisson_3d(const Coeff& f, const BoundaryCondition& bc, double tol) {  // solvers.cpp:171-175
    ModalSolverCache cache(f.s.m, f.s.n, tol);
    return solve_poisson_3d(f, bc, cache);
}

Coeff solve_horizontal_poisson(const Coeff& rhs_in) {  // solvers.cpp:177-203
    const Spec& s = rhs_in.s;
    if (!rhs_in.all_finite()) throw NumericalError("solve_horizontal_poisson: non-finite right-hand side");
    const UltraOps& o = UltraOps::get(s.m);
    const Banded r2c02 = o.r * o.r * o.c02;
    const Banded recomb = dirichlet_recombination(s.m);
    Coeff rhs = parity_project(rhs_in);
    Coeff out(s);
    parallel_for(s.p, [&](long li) {
        const int l = int(li);
        const Banded lred = recombine(radial_modal_laplacian(s.m, s.wavenumber(l)));
        BandedLU lu;
        try {
            lu.factorize(lred);  // refactored every call, as in the reference (solvers.cpp:189-195)
        } catch (const SingularOperatorError&) {
            throw SingularOperatorError("solve_horizontal_poisson: singular column system");
        }
        MatC cols = r2c02.apply_left(slice_mat(rhs, l));
        MatC red(s.m - 2, s.n);
        for (int k = 0; k < s.n; ++k)
            for (int j = 0; j < s.m - 2; ++j) red(j, k) = cols(j, k);
        lu.solve_in_place(red);
        MatC x = recomb.apply_left(red);
        std::copy(x.a.begin(), x.a.end(), out.slice(l));
    });
    parity_project_in_place(out);
    return out;
}

// ---------------------------------------------------------------- timestep (proj/src/timestep.cpp)
BDFScheme BDFScheme::of_order(int b) {  // timestep.cpp:5-29
    BDFScheme s;
    s.order = b;
    switch (b) {
        case 1: s.kappa_over_h = 1.0; s.w = {1.0}; break;
        case 2: s.kappa_over_h = 2.0 / 3.0; s.w = {4.0 / 3.0, -1.0 / 3.0}; break;
        case 3: s.kappa_over_h = 6.0 / 11.0; s.w = {18.0 / 11.0, -9.0 / 11.0, 2.0 / 11.0}; break;
        case 4: s.kappa_over_h = 12.0 / 25.0; s.w = {48.0 / 25.0, -36.0 / 25.0, 16.0 / 25.0, -3.0 / 25.0}; break;
        default: throw DomainError("BDFScheme: order must be in {1,2,3,4}");
    }
    return s;
}

std::vector<double> imex_coefficients(int order) {  // timestep.cpp:31-39
    switch (order) {
        case 1: return {1.0};
        case 2: return {2.0, -1.0};
        case 3: return {3.0, -3.0, 1.0};
        case 4: return {4.0, -6.0, 4.0, -1.0};
        default: throw DomainError("imex_coefficients: order must be in {1,2,3,4}");
    }
}

Coeff bdf_rhs(const std::deque<Coeff>& hist, const BDFScheme& s) {  // timestep.cpp:41-51
    if (int(hist.size()) < s.order) throw DomainError("bdf_rhs: insufficient history for the requested order");
    Coeff out(hist.front().s);
    for (int i = 0; i < s.order; ++i) {
        const double w = s.w[size_t(i)];
        const Coeff& h = hist[size_t(i)];
        for (size_t t = 0; t < out.d.size(); ++t) out.d[t] += w * h.d[t];
    }
    return out;
}

HelmholtzTensorStepper::HelmholtzTensorStepper(const Spec& spec, double diff, double h, double tol, BoundaryCondition bc)
    : spec_(spec), diff_(diff), h_(h), bc_(std::move(bc)), cache_(spec.m, spec.n, tol) {
    spec.validate();
}

Coeff HelmholtzTensorStepper::step(const std::deque<Coeff>& hist, const BDFScheme& s, const Coeff* forcing) const {  // timestep.cpp:61-108
    const double kappa = s.kappa(h_);
    const double scale = kappa * diff_;
    Coeff rhs = bdf_rhs(hist, s);
    if (forcing) {
        if (!(forcing->s == spec_)) throw DomainError("HelmholtzTensorStepper: forcing spec mismatch");
        for (size_t t = 0; t < rhs.d.size(); ++t) rhs.d[t] += kappa * forcing->d[t];
    }
    parity_project_in_place(rhs);
    const UltraOps& ro = UltraOps::get(spec_.m);
    const UltraOps& zo = UltraOps::get(spec_.n);
    const Banded c02t = zo.c02.transposed();
    Coeff out(spec_);
    for (int l = 0; l < spec_.p; ++l) cache_.get(spec_.wavenumber(l), scale, false);
    std::vector<double> resid(static_cast<size_t>(spec_.p), 0.0);
    parallel_for(spec_.p, [&](long li) {
        const int l = int(li);
        const ModalSolver& solver = cache_.get(spec_.wavenumber(l), scale, false);
        MatC fl = slice_mat(rhs, l), lift;
        if (bc_.lifted && bc_.lift && l < bc_.lift->s.p) lift = slice_mat(*bc_.lift, l);
        MatC ff = c02t.apply_right(ro.r2.apply_left(fl));
        if (!lift.a.empty()) ff = add(ff, solver.raw().apply(lift), -1.0);
        MatC x;
        try {
            x = solver.solve(ff);
        } catch (const NonConvergenceError& e) {
            throw NonConvergenceError("modal solve failed for Fourier slice " + std::to_string(l) + ": " + e.what(), e.history);
        }
        if (!lift.a.empty()) x = add(x, lift);
        std::copy(x.a.begin(), x.a.end(), out.slice(l));
        resid[size_t(l)] = solver.last_residual();
    });
    for (double r : resid) worst_ = std::max(worst_, r);
    parity_project_in_place(out);
    if (!out.all_finite()) throw NumericalError("HelmholtzTensorStepper: non-finite state");
    return out;
}

HeatStepper::HeatStepper(const HeatConfig& cfg, Coeff initial)  // timestep.cpp:112-118
    : cfg_(cfg), stepper_(cfg.spec, cfg.alpha, cfg.h, cfg.tol) {
    if (!(initial.s == cfg.spec)) throw DomainError("HeatStepper: initial data spec mismatch");
    parity_project_in_place(initial);
    hist_.push_front(std::move(initial));
}

void HeatStepper::step(const Coeff* forcing) {  // timestep.cpp:126-133
    const BDFScheme s = BDFScheme::of_order(current_order());
    Coeff next = stepper_.step(hist_, s, forcing);
    hist_.push_front(std::move(next));
    while (int(hist_.size()) > cfg_.order) hist_.pop_back();
    time_ += cfg_.h;
    ++steps_;
}

void HeatStepper::step_with_callback(const ForcingCallback& f) {  // timestep.cpp:135-144
    if (!f) {
        step(nullptr);
        return;
    }
    const double t = cfg_.exact_forcing ? time_ + cfg_.h : time_;
    Coeff g = analyze(f(t));
    step(&g);
}

// ---------------------------------------------------------------- ptns (proj/src/ptns.cpp)
Vec3 curl_vector(const Vec3& v) {  // ptns.cpp:25-33
    Vec3 o;
    o.r = divide_r(derivative_theta(v.z)) - derivative_z(v.t);
    o.t = derivative_z(v.r) - derivative_r(v.z);
    Coeff zp = derivative_r(v.t);
    zp += divide_r(v.t - derivative_theta(v.r));
    o.z = zp;
    return o;
}

Coeff divergence(const Vec3& v) {  // ptns.cpp:35-40
    Coeff o = derivative_r(v.r);
    o += divide_r(v.r + derivative_theta(v.t));
    o += derivative_z(v.z);
    return o;
}

Vec3 pt_synthesize(const PT& s) {  // ptns.cpp:42-57
    if (s.lambda.s.m % 2 != 0) throw DomainError("pt_synthesize: even m required (no r = 0 grid node)");
    Vec3 v;
    const Coeff dzg = derivative_z(s.gamma);
    v.r = divide_r(derivative_theta(s.lambda)) + derivative_r(dzg);
    v.t = divide_r(derivative_theta(dzg)) - derivative_r(s.lambda);
    Coeff hl = horizontal_laplacian(s.gamma);
    hl *= cd(-1.0);
    v.z = hl;
    parity_project_in_place(v.r, Parity::azimuthal_flip);
    parity_project_in_place(v.t, Parity::azimuthal_flip);
    parity_project_in_place(v.z, Parity::scalar);
    return v;
}

PT pt_decompose(const Vec3& v, bool check, double div_tol) {  // ptns.cpp:59-77
    if (check) {
        const double div = divergence(v).max_abs();
        const double sc = std::max({1.0, v.r.max_abs(), v.t.max_abs(), v.z.max_abs()});
        if (div > div_tol * sc) throw NotIncompressibleError("pt_decompose: field has divergence " + std::to_string(div), div);
    }
    Coeff vz = v.z;
    vz *= cd(-1.0);
    Coeff gamma = solve_horizontal_poisson(vz);
    Coeff cz = derivative_r(v.t);
    cz += divide_r(v.t - derivative_theta(v.r));
    cz *= cd(-1.0);
    Coeff lambda = solve_horizontal_poisson(cz);
    return {std::move(lambda), std::move(gamma)};
}

PT curl_pt(const PT& s) {  // ptns.cpp:79-83
    Coeff lam = laplacian(s.gamma);
    lam *= cd(-1.0);
    return {std::move(lam), s.lambda};
}

PT velocity_from_vorticity(const PT& omega, const ModalSolverCache& cache) {  // ptns.cpp:85-91
    Coeff rhs = omega.lambda;
    rhs *= cd(-1.0);
    Coeff lpsi = solve_poisson_3d(rhs, BoundaryCondition{}, cache);
    return {omega.gamma, std::move(lpsi)};
}

static void dealias_tensor(Coeff& t) {  // ptns.cpp:100-110
    const Spec& s = t.s;
    const int jmax = 2 * s.m / 3, kmax = 2 * s.n / 3, wmax = 2 * (s.p / 2) / 3;
    for (int l = 0; l < s.p; ++l) {
        const int w = std::abs(s.wavenumber(l));
        for (int k = 0; k < s.n; ++k)
            for (int j = 0; j < s.m; ++j)
                if (j >= jmax || k >= kmax || w >= wmax) t.at(j, k, l) = cd(0);
    }
}

PT nonlinear_term(const PT& v, const PT& omega, bool dealias) {  // ptns.cpp:114-149
    const Spec& s = v.lambda.s;
    if (s.m % 2 != 0) throw DomainError("nonlinear_term: even m required");
    const Vec3 vc = pt_synthesize(v);
    const Vec3 wc = pt_synthesize(omega);
    const Field vr = synthesize(vc.r), vt = synthesize(vc.t), vz = synthesize(vc.z);
    const Field wr = synthesize(wc.r), wt = synthesize(wc.t), wz = synthesize(wc.z);
    Field ar(s), at(s), az(s);
    for (size_t i = 0; i < ar.v.size(); ++i) {
        ar.v[i] = vt.v[i] * wz.v[i] - vz.v[i] * wt.v[i];
        at.v[i] = vz.v[i] * wr.v[i] - vr.v[i] * wz.v[i];
        az.v[i] = vr.v[i] * wt.v[i] - vt.v[i] * wr.v[i];
    }
    Vec3 a;
    a.r = analyze(ar);
    a.t = analyze(at);
    a.z = analyze(az);
    parity_project_in_place(a.r, Parity::azimuthal_flip);
    parity_project_in_place(a.t, Parity::azimuthal_flip);
    parity_project_in_place(a.z, Parity::scalar);
    if (dealias) {
        dealias_tensor(a.r);
        dealias_tensor(a.t);
        dealias_tensor(a.z);
    }
    const Vec3 ca = curl_vector(a);
    return pt_decompose(ca, false);
}

NSStepper::NSStepper(const NSConfig& cfg, PT omega0)  // ptns.cpp:177-193
    : cfg_(cfg), stepper_(cfg.spec, 1.0 / cfg.reynolds, cfg.h, cfg.tol), poisson_cache_(cfg.spec.m, cfg.spec.n, cfg.tol) {
    if (!(omega0.lambda.s == cfg.spec) || !(omega0.gamma.s == cfg.spec)) throw DomainError("NSStepper: initial vorticity spec mismatch");
    if (cfg.spec.m % 2 != 0) throw DomainError("NSStepper: even m required for the nonlinear pipeline");
    parity_project_in_place(omega0.lambda);
    parity_project_in_place(omega0.gamma);
    omega_.push_front(std::move(omega0));
}

void NSStepper::seed(std::deque<PT> omega_hist, std::deque<PT> nonlinear_hist, double time, int steps_taken) {
    if (omega_hist.empty()) throw DomainError("NSStepper::seed: empty history");
    omega_ = std::move(omega_hist);
    nonlinear_ = std::move(nonlinear_hist);
    time_ = time;
    steps_ = steps_taken;
}

PT NSStepper::velocity() const { return velocity_from_vorticity(omega_.front(), poisson_cache_); }

void NSStepper::step() {  // ptns.cpp:217-267
    const int b = std::min(cfg_.order, steps_ + 1);
    const BDFScheme scheme = BDFScheme::of_order(b);
    std::deque<Coeff> lam_h, gam_h;
    for (const PT& s : omega_) {
        lam_h.push_back(s.lambda);
        gam_h.push_back(s.gamma);
    }
    const Coeff *lf = nullptr, *gf = nullptr;
    Coeff lext, gext;
    if (!cfg_.disable_nonlinear) {
        const PT v = velocity();
        nonlinear_.push_front(nonlinear_term(v, omega_.front(), cfg_.dealias));
        while (int(nonlinear_.size()) > cfg_.order) nonlinear_.pop_back();
        const int eo = std::min(b, int(nonlinear_.size()));
        const std::vector<double> w = imex_coefficients(eo);
        lext = Coeff(cfg_.spec);
        gext = Coeff(cfg_.spec);
        for (int i = 0; i < eo; ++i) {
            const PT& a = nonlinear_[size_t(i)];
            for (size_t t = 0; t < lext.d.size(); ++t) {
                lext.d[t] += w[size_t(i)] * a.lambda.d[t];
                gext.d[t] += w[size_t(i)] * a.gamma.d[t];
            }
        }
        lf = &lext;
        gf = &gext;
    }
    PT next;
    next.lambda = stepper_.step(lam_h, scheme, lf);
    next.gamma = stepper_.step(gam_h, scheme, gf);
    if (!next.lambda.all_finite() || !next.gamma.all_finite())
        throw NumericalError("NSStepper: non-finite state at step " + std::to_string(steps_ + 1));
    omega_.push_front(std::move(next));
    while (int(omega_.size()) > cfg_.order) omega_.pop_back();
    time_ += cfg_.h;
    ++steps_;
}

// Restatement of ns_run (ptns.cpp:269-324). Ramp start: step the full-order stepper from omega0. Substeps start
// (:272-311): sample a BDF-min(2, b) run with 32 sub-steps per h at t = h .. (b-1) h, rebuild the nonlinear terms
// of the older samples, seed the full-order stepper with both histories at steps_taken = b - 1, and finish the run.
PT ns_run(const NSConfig& cfg, const PT& omega0, int steps, bool substeps, double* final_time) {
    const int b = cfg.order;
    const bool bootstrap = substeps && b > 1 && steps > 0;
    std::deque<PT> samples{omega0};  // newest first
    if (bootstrap) {
        constexpr int kSub = 32;
        NSConfig fine_cfg = cfg;
        fine_cfg.order = std::min(2, b);
        fine_cfg.h = cfg.h / kSub;
        NSStepper fine(fine_cfg, omega0);
        for (int level = 1; level < b; ++level) {
            for (int q = 0; q < kSub; ++q) fine.step();
            samples.push_front(fine.omega());
        }
    }
    NSStepper full(cfg, samples.front());
    int done = 0;
    if (bootstrap) {
        std::deque<PT> nl;  // N of samples[1..], newest first
        if (!cfg.disable_nonlinear) {
            ModalSolverCache cache(cfg.spec.m, cfg.spec.n, cfg.tol);
            for (size_t i = 1; i < samples.size(); ++i)
                nl.push_back(nonlinear_term(velocity_from_vorticity(samples[i], cache), samples[i], cfg.dealias));
        }
        done = b - 1;
        full.seed(samples, nl, done * cfg.h, done);
    }
    for (int s = done; s < steps; ++s) full.step();
    if (final_time) *final_time = full.time();
    return full.omega();
}

}  // namespace oracle
