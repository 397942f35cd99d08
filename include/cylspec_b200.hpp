// cylspec_b200.hpp — header-only C++ drop-in for the reference `cylspec` hot-path API
// (proj/include/cylspec/{grid,coeffs,errors,transform,calculus,solvers,timestep,ptns}.hpp),
// implemented over the B200 C-ABI (include/ccf.h, lib/libccf.so).
//
// Same names, argument meaning, value semantics and exception types as the reference for
// the hot path; Eigen-typed signatures (CoeffTensor::slice, ModalSolver::solve) are not part
// of this shim. Each (m, n, p) grid gets one thread-local ccf context
// (the reference's caches are process-wide; ours are per context and hold the same plans).
#pragma once

#include <cmath>
#include <complex>
#include <deque>
#include <map>
#include <cstdint>
#include <algorithm>
#include <variant>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "ccf.h"

namespace cylspec {

using Complex = std::complex<double>;

// ---- errors (proj/include/cylspec/errors.hpp:10-40)
struct DomainError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct SingularOperatorError : std::runtime_error {
    explicit SingularOperatorError(const std::string& w, int j = -1) : std::runtime_error(w), shift_index(j) {}
    int shift_index;
};
struct NonConvergenceError : std::runtime_error {
    NonConvergenceError(const std::string& w, std::vector<double> h) : std::runtime_error(w), residual_history(std::move(h)) {}
    std::vector<double> residual_history;
};
struct NotIncompressibleError : std::runtime_error {
    NotIncompressibleError(const std::string& w, double d) : std::runtime_error(w), divergence(d) {}
    double divergence;
};
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FieldFileError : std::runtime_error { using std::runtime_error::runtime_error; };  // io.hpp:17-19

// ---- grid / tensors (grid.hpp:13-50, coeffs.hpp:16-45)
struct GridSpec {
    int m = 0, n = 0, p = 0;
    GridSpec() = default;
    GridSpec(int m_, int n_, int p_) : m(m_), n(n_), p(p_) { validate(); }
    void validate() const {
        if (m < 4 || n < 4) throw DomainError("GridSpec: m and n must be at least 4");
        if (p < 2 || p % 2 != 0) throw DomainError("GridSpec: p must be even and at least 2");
    }
    long total_points() const { return long(m) * n * p; }
    int zero_mode() const { return p / 2; }
    int wavenumber(int l) const { return l - p / 2; }
    bool operator==(const GridSpec&) const = default;
};

struct GridField {
    GridSpec spec;
    std::vector<double> values;
    GridField() = default;
    explicit GridField(const GridSpec& s) : spec(s), values(size_t(s.total_points()), 0.0) {}
    size_t index(int j, int k, int l) const { return (size_t(l) * spec.n + size_t(k)) * spec.m + size_t(j); }
    double& at(int j, int k, int l) { return values[index(j, k, l)]; }
    double at(int j, int k, int l) const { return values[index(j, k, l)]; }
};

// Minimal column-major complex matrix standing in for Eigen::MatrixXcd in the three Eigen-typed signatures of the
// per-mode API (solvers.hpp:43, coeffs.hpp:23-28): same memory layout, (i, j) access, rows() / cols() / data().
class MatrixXcd {
public:
    MatrixXcd() = default;
    MatrixXcd(int rows, int cols) : r_(rows), c_(cols), d_(size_t(rows) * size_t(cols), Complex(0)) {}
    static MatrixXcd Zero(int rows, int cols) { return MatrixXcd(rows, cols); }
    int rows() const { return r_; }
    int cols() const { return c_; }
    size_t size() const { return d_.size(); }
    Complex& operator()(int i, int j) { return d_[size_t(j) * size_t(r_) + size_t(i)]; }
    Complex operator()(int i, int j) const { return d_[size_t(j) * size_t(r_) + size_t(i)]; }
    Complex* data() { return d_.data(); }
    const Complex* data() const { return d_.data(); }
    MatrixXcd& operator+=(const MatrixXcd& o) { return zip(o, 1.0); }
    MatrixXcd& operator-=(const MatrixXcd& o) { return zip(o, -1.0); }
    MatrixXcd& operator*=(Complex s) {
        for (Complex& v : d_) v *= s;
        return *this;
    }
    friend MatrixXcd operator+(MatrixXcd a, const MatrixXcd& b) { return a += b; }
    friend MatrixXcd operator-(MatrixXcd a, const MatrixXcd& b) { return a -= b; }
    friend MatrixXcd operator*(Complex s, MatrixXcd a) { return a *= s; }
    friend MatrixXcd operator*(double s, MatrixXcd a) { return a *= Complex(s); }
    double max_abs() const {  // cwiseAbs().maxCoeff()
        double v = 0;
        for (const Complex& x : d_) v = std::max(v, std::abs(x));
        return v;
    }
    double norm() const {
        double v = 0;
        for (const Complex& x : d_) v += std::norm(x);
        return std::sqrt(v);
    }

private:
    MatrixXcd& zip(const MatrixXcd& o, double sgn) {
        if (o.r_ != r_ || o.c_ != c_) throw DomainError("MatrixXcd: shape mismatch");
        for (size_t i = 0; i < d_.size(); ++i) d_[i] += sgn * o.d_[i];
        return *this;
    }
    int r_ = 0, c_ = 0;
    std::vector<Complex> d_;
};

struct CoeffTensor {
    GridSpec spec;
    std::vector<Complex> data;
    CoeffTensor() = default;
    explicit CoeffTensor(const GridSpec& s) : spec(s), data(size_t(s.total_points()), Complex(0)) {}
    Complex& at(int j, int k, int l) { return data[(size_t(l) * spec.n + size_t(k)) * spec.m + size_t(j)]; }
    Complex at(int j, int k, int l) const { return data[(size_t(l) * spec.n + size_t(k)) * spec.m + size_t(j)]; }
    const double* raw() const { return reinterpret_cast<const double*>(data.data()); }
    double* raw() { return reinterpret_cast<double*>(data.data()); }
    CoeffTensor& operator+=(const CoeffTensor& o) {  // coeffs.cpp:19-23
        if (!(spec == o.spec)) throw DomainError("CoeffTensor: spec mismatch");
        for (size_t i = 0; i < data.size(); ++i) data[i] += o.data[i];
        return *this;
    }
    MatrixXcd slice(int l) const {  // coeffs.hpp:23-28 (a copy; the reference returns an Eigen::Map)
        MatrixXcd o(spec.m, spec.n);
        std::copy(data.begin() + long(l) * spec.m * spec.n, data.begin() + long(l + 1) * spec.m * spec.n, o.data());
        return o;
    }
    void set_slice(int l, const MatrixXcd& x) {
        if (x.rows() != spec.m || x.cols() != spec.n) throw DomainError("CoeffTensor: slice shape mismatch");
        std::copy(x.data(), x.data() + x.size(), data.begin() + long(l) * spec.m * spec.n);
    }
    CoeffTensor& operator*=(Complex s) {  // coeffs.cpp:31-34
        for (Complex& c : data) c *= s;
        return *this;
    }
    double max_abs() const {
        double v = 0;
        for (const Complex& c : data) v = std::max(v, std::abs(c));
        return v;
    }
    bool all_finite() const {  // coeffs.cpp:12-17
        for (const Complex& c : data)
            if (!std::isfinite(c.real()) || !std::isfinite(c.imag())) return false;
        return true;
    }
    CoeffTensor& operator-=(const CoeffTensor& o) {  // coeffs.cpp:25-29
        if (!(spec == o.spec)) throw DomainError("CoeffTensor: spec mismatch");
        for (size_t i = 0; i < data.size(); ++i) data[i] -= o.data[i];
        return *this;
    }
    friend CoeffTensor operator+(CoeffTensor a, const CoeffTensor& b) { return a += b; }
    friend CoeffTensor operator-(CoeffTensor a, const CoeffTensor& b) { return a -= b; }
    friend CoeffTensor operator*(Complex s, CoeffTensor a) { return a *= s; }
};

// Container-level helpers of coeffs.hpp:47-59 (index masks and comparisons on the host-side tensor; on the device
// path the parity classes are built into the parity-compressed layout, so the kernels never store the masked half).
inline double hermitian_symmetry_error(const CoeffTensor& t) {  // coeffs.cpp:36-48
    const GridSpec& s = t.spec;
    const int half = s.p / 2;
    double worst = 0.0;
    for (int l = 0; l < s.p; ++l) {
        const int lp = 2 * half - l;  // partner slice carrying -wavenumber
        if (lp < 0 || lp >= s.p) continue;
        for (int k = 0; k < s.n; ++k)
            for (int j = 0; j < s.m; ++j) worst = std::max(worst, std::abs(t.at(j, k, l) - std::conj(t.at(j, k, lp))));
    }
    return worst;
}
enum class Parity { scalar, azimuthal_flip };  // keep j + wavenumber even | odd
inline void parity_project_in_place(CoeffTensor& coeffs, Parity parity = Parity::scalar) {  // coeffs.cpp:50-59
    const GridSpec& s = coeffs.spec;
    const int keep_mod = (parity == Parity::scalar) ? 0 : 1;
    for (int l = 0; l < s.p; ++l) {
        const int w = s.wavenumber(l);
        for (int k = 0; k < s.n; ++k)
            for (int j = 0; j < s.m; ++j)
                if (((j + w) % 2 + 2) % 2 != keep_mod) coeffs.at(j, k, l) = Complex(0);
    }
}
inline CoeffTensor parity_project(const CoeffTensor& coeffs, Parity parity = Parity::scalar) {  // coeffs.cpp:61-65
    CoeffTensor out = coeffs;
    parity_project_in_place(out, parity);
    return out;
}

// grid points (grid.cpp:16-40): r_j = cos((m-1-j) pi/(m-1)) with exact endpoints / midpoint, theta_l = (2l - p) pi / p
inline std::vector<double> chebyshev_points(int count) {
    if (count < 2) throw DomainError("chebyshev_points: need at least 2 points");
    std::vector<double> x(static_cast<size_t>(count), 0.0);
    for (int j = 0; j < count; ++j) x[size_t(j)] = std::cos(double(count - j - 1) * M_PI / double(count - 1));
    x[0] = -1.0;
    x[size_t(count) - 1] = 1.0;
    if (count % 2 == 1) x[size_t(count / 2)] = 0.0;
    return x;
}
inline std::vector<double> fourier_points(int count) {
    std::vector<double> t(static_cast<size_t>(count), 0.0);
    for (int l = 0; l < count; ++l) t[size_t(l)] = double(2 * l - count) * M_PI / double(count);
    return t;
}
template <class F>
GridField sample(const GridSpec& spec, F&& f) {  // grid.hpp: value f(r_j, z_k, theta_l) at every node
    GridField g(spec);
    const auto r = chebyshev_points(spec.m), z = chebyshev_points(spec.n), th = fourier_points(spec.p);
    for (int l = 0; l < spec.p; ++l)
        for (int k = 0; k < spec.n; ++k)
            for (int j = 0; j < spec.m; ++j) g.at(j, k, l) = f(r[size_t(j)], z[size_t(k)], th[size_t(l)]);
    return g;
}

struct PTScalars {
    CoeffTensor lambda, gamma;
    PTScalars() = default;
    explicit PTScalars(const GridSpec& s) : lambda(s), gamma(s) {}
    PTScalars(CoeffTensor l, CoeffTensor g) : lambda(std::move(l)), gamma(std::move(g)) {}
};

struct VectorFieldCoeffs {
    CoeffTensor comp_r, comp_theta, comp_z;
    VectorFieldCoeffs() = default;
    explicit VectorFieldCoeffs(const GridSpec& s) : comp_r(s), comp_theta(s), comp_z(s) {}
};

struct BoundaryCondition {  // solvers.hpp:18-31
    enum class Kind { dirichlet_homogeneous, dirichlet_lifted };
    Kind kind = Kind::dirichlet_homogeneous;
    std::optional<CoeffTensor> lift;
    static BoundaryCondition homogeneous() { return {}; }
    static BoundaryCondition lifted(CoeffTensor lift_tensor) {
        BoundaryCondition bc;
        bc.kind = Kind::dirichlet_lifted;
        bc.lift = std::move(lift_tensor);
        return bc;
    }
};

inline constexpr double kDefaultAdiTol = 1e-12;

namespace detail {

[[noreturn]] inline void raise(ccf_status st, ccf_ctx* ctx) {
    int kind = 0, slice = -1, shift = -1, nh = 8;
    double hist[8] = {0};
    char msg[1024] = {0};
    if (ctx) ccf_get_last_error(ctx, &kind, &slice, &shift, hist, &nh, msg, sizeof msg);
    else std::snprintf(msg, sizeof msg, "%s", ccf_create_error());
    const std::string w(msg);
    switch (st) {
        case CCF_DOMAIN_ERROR: throw DomainError(w);
        case CCF_CONFIG_ERROR: throw ConfigError(w);
        case CCF_SINGULAR_OPERATOR: throw SingularOperatorError(w, shift);
        case CCF_NON_CONVERGENCE: throw NonConvergenceError(w, std::vector<double>(hist, hist + (nh < 8 ? nh : 8)));
        case CCF_NOT_INCOMPRESSIBLE: throw NotIncompressibleError(w, 0.0);
        case CCF_NUMERICAL_ERROR: throw NumericalError(w);
        case CCF_FIELDFILE_ERROR: throw FieldFileError(w);
        default: throw std::runtime_error("ccf: " + w);
    }
}

inline void check(ccf_status st, ccf_ctx* ctx) {
    if (st != CCF_OK) raise(st, ctx);
}

// multi-input entry points: the C-ABI reads every buffer with the first tensor's spec, so a mismatched
// tensor is a DomainError here, never an out-of-bounds read
template <class T, class... Ts>
inline void same_spec(const char* what, const T& first, const Ts&... rest) {
    if (!((rest.spec == first.spec) && ...)) throw DomainError(std::string(what) + ": spec mismatch");
}

// one context per (m, n, p, tol) and host thread (the reference library is single-threaded)
inline ccf_ctx* context(const GridSpec& s, double tol = kDefaultAdiTol) {
    struct Deleter {
        void operator()(ccf_ctx* c) const { ccf_ctx_destroy(c); }
    };
    thread_local std::map<std::tuple<int, int, int, double>, std::unique_ptr<ccf_ctx, Deleter>> cache;
    auto& slot = cache[{s.m, s.n, s.p, tol}];
    if (!slot) {
        ccf_ctx* c = nullptr;
        check(ccf_ctx_create(s.m, s.n, s.p, 0, tol, 0, &c), nullptr);
        slot.reset(c);
    }
    return slot.get();
}

}  // namespace detail

// ---- transform.hpp:17-22
inline CoeffTensor analyze(const GridField& f) {
    CoeffTensor out(f.spec);
    ccf_ctx* c = detail::context(f.spec);
    detail::check(ccf_analyze(c, f.values.data(), out.raw()), c);
    return out;
}
inline GridField synthesize(const CoeffTensor& t) {
    GridField out(t.spec);
    ccf_ctx* c = detail::context(t.spec);
    detail::check(ccf_synthesize(c, t.raw(), out.values.data()), c);
    return out;
}

// ---- calculus.hpp:15-29 (tensors of real fields)
namespace detail {
inline CoeffTensor calc(int op, const CoeffTensor& f) {
    CoeffTensor out(f.spec);
    ccf_ctx* c = context(f.spec);
    check(ccf_calculus(c, op, f.raw(), out.raw()), c);
    return out;
}
}  // namespace detail
inline CoeffTensor derivative_r(const CoeffTensor& f) { return detail::calc(0, f); }
inline CoeffTensor derivative_z(const CoeffTensor& f) { return detail::calc(1, f); }
inline CoeffTensor derivative_theta(const CoeffTensor& f) { return detail::calc(2, f); }
inline CoeffTensor divide_r(const CoeffTensor& f) { return detail::calc(4, f); }
inline CoeffTensor horizontal_laplacian(const CoeffTensor& f) { return detail::calc(5, f); }
inline CoeffTensor laplacian(const CoeffTensor& f) { return detail::calc(6, f); }

// ---- per-mode API: ultraop.hpp:40-53, solvers.hpp:35-82 (ccf_modal_* on the device)
namespace detail {
struct ModalHandle {
    ccf_ctx* ctx = nullptr;
    ccf_modal* h = nullptr;
    int m, n;
    ModalHandle(int m_, int n_, int w, double scale, bool poisson, double tol) : m(m_), n(n_) {
        ctx = context(GridSpec(m_, n_, 4), tol);
        check(ccf_modal_create(ctx, w, scale, poisson ? 1 : 0, &h), ctx);
    }
    ~ModalHandle() { ccf_modal_destroy(h); }
    ModalHandle(const ModalHandle&) = delete;
    ModalHandle& operator=(const ModalHandle&) = delete;
    std::vector<double> dense(int which) const {
        std::vector<double> o(which % 2 == 0 ? size_t(m) * m : size_t(n) * n);
        check(ccf_modal_operator(h, which, o.data()), ctx);
        return o;
    }
};
}  // namespace detail

struct ModalOperator {  // ultraop.hpp:40-48; A, C: m x m, B, D: n x n, dense row-major (the reference's are banded)
    int m = 0, n = 0;
    int wavenumber = 0;
    double scale = 0.0;
    std::vector<double> A, B, C, D;
    /// A X B + C X D applied to dense (complex) X, on the device (ultraop.cpp:83-87).
    MatrixXcd apply(const MatrixXcd& x) const {
        if (x.rows() != m || x.cols() != n) throw DomainError("ModalOperator::apply: wrong shape");
        MatrixXcd y(m, n);
        detail::check(ccf_modal_apply(dev->h, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())),
                      dev->ctx);
        return y;
    }
    std::shared_ptr<detail::ModalHandle> dev;  // device-side solver data behind apply()
};
namespace detail {
inline ModalOperator modal_operator(int m, int n, int w, double scale, bool poisson, double tol = kDefaultAdiTol) {
    ModalOperator op;
    op.m = m;
    op.n = n;
    op.wavenumber = w;
    op.scale = poisson ? 1.0 : scale;
    op.dev = std::make_shared<ModalHandle>(m, n, w, scale, poisson, tol);
    op.A = op.dev->dense(0);
    op.B = op.dev->dense(1);
    op.C = op.dev->dense(2);
    op.D = op.dev->dense(3);
    return op;
}
}  // namespace detail
inline ModalOperator assemble_modal_helmholtz(int m, int n, int wavenumber, double scale) {  // ultraop.cpp:89-107
    if (m < 4 || n < 4) throw DomainError("assemble_modal_helmholtz: sizes too small");
    return detail::modal_operator(m, n, wavenumber, scale, false);
}
inline ModalOperator assemble_modal_poisson(int m, int n, int wavenumber) {  // ultraop.cpp:109-123
    if (m < 4 || n < 4) throw DomainError("assemble_modal_poisson: sizes too small");
    return detail::modal_operator(m, n, wavenumber, 1.0, true);
}

struct ShiftPlan {  // adi.hpp:19-28
    double a = 0, b = 0, c = 0, d = 0, gamma_cr = 0, alpha_z = 0, modulus = 0, tol = 0;
    int J = 0;
    std::vector<double> u, v;
};

/// One Fourier mode's Helmholtz / Poisson solver (solvers.hpp:35-59). solve() is the exact fast-diagonalization
/// solve on the device (the reference iterates ADI to `tol`); plan() is the reference's Zolotarev shift plan for the
/// same quadruple (setup numerics, kept for parity checks), nullptr for the mass pair.
class ModalSolver {
public:
    ModalSolver(int m, int n, int wavenumber, double scale, bool poisson, double tol = kDefaultAdiTol)
        : op_(detail::modal_operator(m, n, wavenumber, scale, poisson, tol)), tol_(tol), poisson_(poisson), scale_(scale) {}
    MatrixXcd solve(const MatrixXcd& f_full) const {  // solvers.cpp:77-98
        if (f_full.rows() != op_.m || f_full.cols() != op_.n)
            throw DomainError("ModalSolver::solve: right-hand side has wrong shape");
        MatrixXcd x(op_.m, op_.n);
        detail::check(ccf_modal_solve(op_.dev->h, reinterpret_cast<const double*>(f_full.data()),
                                      reinterpret_cast<double*>(x.data())),
                      op_.dev->ctx);
        // relative residual of the recombined system (adi.cpp:106-112) = (op.apply(x) - f) on the retained block
        const MatrixXcd r = op_.apply(x);
        double rn = 0, en = 0;
        for (int k = 0; k + 2 < op_.n; ++k)
            for (int j = 0; j + 2 < op_.m; ++j) {
                rn += std::norm(r(j, k) - f_full(j, k));
                en += std::norm(f_full(j, k));
            }
        last_residual_ = en > 0.0 ? std::sqrt(rn / en) : std::sqrt(rn);
        return x;
    }
    const ModalOperator& raw() const { return op_; }
    const ShiftPlan* plan() const {
        if (!poisson_ && scale_ == 0.0) return nullptr;
        if (!plan_) {
            double info[8];
            std::vector<double> u(128), v(128);
            detail::check(ccf_plan_host(op_.m, op_.n, op_.wavenumber, scale_, poisson_ ? 1 : 0, tol_, 0, info, u.data(),
                                        v.data(), 128),
                          nullptr);
            ShiftPlan p;
            p.a = info[0]; p.b = info[1]; p.c = info[2]; p.d = info[3];
            p.gamma_cr = info[4]; p.alpha_z = info[5]; p.modulus = info[6]; p.J = int(info[7]);
            p.tol = tol_;
            u.resize(size_t(std::min(p.J, 128)));
            v.resize(size_t(std::min(p.J, 128)));
            p.u = std::move(u);
            p.v = std::move(v);
            plan_ = std::move(p);
        }
        return &*plan_;
    }
    double last_residual() const { return last_residual_; }

private:
    ModalOperator op_;
    double tol_;
    bool poisson_;
    double scale_;
    mutable std::optional<ShiftPlan> plan_;
    mutable double last_residual_ = 0.0;
};

class ModalSolverCache {  // solvers.hpp:63-76, keyed by (w^2, scale, poisson)
public:
    ModalSolverCache(int m, int n, double tol) : m_(m), n_(n), tol_(tol) {}
    const ModalSolver& get(int wavenumber, double scale, bool poisson) const {
        auto& slot = cache_[std::make_tuple(wavenumber * wavenumber, scale, poisson)];
        if (!slot) slot = std::make_unique<ModalSolver>(m_, n_, std::abs(wavenumber), scale, poisson, tol_);
        return *slot;
    }
    int m() const { return m_; }
    int n() const { return n_; }
    double tol() const { return tol_; }

private:
    int m_, n_;
    double tol_;
    mutable std::map<std::tuple<int, double, bool>, std::unique_ptr<ModalSolver>> cache_;
};

namespace detail {
inline MatrixXcd lift_slice_for(int m, int n, const BoundaryCondition& bc, int slice_index) {  // solvers.cpp:112-123
    if (!bc.lift) throw DomainError("BoundaryCondition: lifted kind without lift data");
    const CoeffTensor& lift = *bc.lift;
    if (lift.spec.m != m || lift.spec.n != n) throw DomainError("BoundaryCondition: lift tensor has wrong dimensions");
    if (slice_index < 0 || slice_index >= lift.spec.p) throw DomainError("BoundaryCondition: lift tensor misses the requested mode");
    return lift.slice(slice_index);
}
// The modal solves are linear, so the lifted solve(F_l - op_l.apply(lift_l)) + lift_l (solvers.cpp:160-165,
// timestep.cpp:84-101) = the homogeneous solve + c_l with c_l = lift_l - solve(op_l.apply(lift_l)), parity-projected
// like the output; the per-mode pieces run on the device through ModalSolver.
inline void add_lift_correction(CoeffTensor& out, const BoundaryCondition& bc, double scale, bool poisson, double tol) {
    const GridSpec& spec = out.spec;
    ModalSolverCache cache(spec.m, spec.n, tol);
    for (int l = 0; l < spec.p; ++l) {
        const int w = spec.wavenumber(l);
        const MatrixXcd lift = lift_slice_for(spec.m, spec.n, bc, l);
        if (lift.max_abs() == 0.0) continue;
        const ModalSolver& solver = cache.get(w, scale, poisson);
        const MatrixXcd c = lift - solver.solve(solver.raw().apply(lift));
        for (int k = 0; k < spec.n; ++k)
            for (int j = 0; j < spec.m; ++j)
                if ((j + w) % 2 == 0) out.at(j, k, l) += c(j, k);  // parity_project (coeffs.cpp:50-65)
    }
}
}  // namespace detail

inline MatrixXcd solve_modal_helmholtz(const ModalOperator& op, const MatrixXcd& f, const BoundaryCondition& bc,
                                       double tol = kDefaultAdiTol) {  // solvers.cpp:125-140
    ModalSolver solver(op.m, op.n, op.wavenumber, op.scale, /*poisson=*/false, tol);
    MatrixXcd rhs = f, lift;
    if (bc.kind == BoundaryCondition::Kind::dirichlet_lifted) {
        if (!bc.lift) throw DomainError("BoundaryCondition: lifted kind without lift data");
        lift = detail::lift_slice_for(op.m, op.n, bc, op.wavenumber + bc.lift->spec.p / 2);
        rhs -= op.apply(lift);
    }
    MatrixXcd x = solver.solve(rhs);
    if (lift.size() > 0) x += lift;
    return x;
}

// ---- solvers.hpp:86-94
inline CoeffTensor solve_poisson_3d(const CoeffTensor& f, const BoundaryCondition& bc = {}, double tol = kDefaultAdiTol) {
    CoeffTensor out(f.spec);
    ccf_ctx* c = detail::context(f.spec, tol);
    detail::check(ccf_poisson3d(c, f.raw(), out.raw()), c);
    if (bc.kind == BoundaryCondition::Kind::dirichlet_lifted) detail::add_lift_correction(out, bc, 1.0, true, tol);
    return out;
}
inline CoeffTensor solve_poisson_3d(const CoeffTensor& f, const BoundaryCondition& bc, const ModalSolverCache& cache) {
    if (cache.m() != f.spec.m || cache.n() != f.spec.n) throw DomainError("solve_poisson_3d: cache size mismatch");
    return solve_poisson_3d(f, bc, cache.tol());
}
inline CoeffTensor solve_horizontal_poisson(const CoeffTensor& rhs) {
    CoeffTensor out(rhs.spec);
    ccf_ctx* c = detail::context(rhs.spec);
    detail::check(ccf_hpoisson(c, rhs.raw(), out.raw()), c);
    return out;
}

// ---- timestep.hpp:13-53
struct BDFScheme {
    int order = 1;
    double kappa_over_h = 1.0;
    static BDFScheme of_order(int b) {
        static const double K[4] = {1.0, 2.0 / 3.0, 6.0 / 11.0, 12.0 / 25.0};
        if (b < 1 || b > 4) throw DomainError("BDFScheme: order must be in {1,2,3,4}");
        return {b, K[b - 1]};
    }
    double kappa(double h) const { return kappa_over_h * h; }
};

class HelmholtzTensorStepper {
public:
    HelmholtzTensorStepper(const GridSpec& spec, double diffusivity, double h, double adi_tol,
                           BoundaryCondition bc = {})
        : spec_(spec), diff_(diffusivity), h_(h), tol_(adi_tol), bc_(std::move(bc)) {
        spec.validate();
    }
    CoeffTensor step(const std::deque<CoeffTensor>& history, const BDFScheme& scheme, const CoeffTensor* forcing) const {
        // timestep.cpp:69-70 (forcing); the C-ABI reads spec-sized buffers, so every history entry is checked too
        if (forcing && !(forcing->spec == spec_)) throw DomainError("HelmholtzTensorStepper: forcing spec mismatch");
        if (int(history.size()) < scheme.order)
            throw DomainError("bdf_rhs: insufficient history for the requested order");  // timestep.cpp:43
        std::vector<const double*> hp;
        for (const auto& t : history) {
            if (!(t.spec == spec_)) throw DomainError("HelmholtzTensorStepper: history spec mismatch");
            hp.push_back(t.raw());
        }
        CoeffTensor out(spec_);
        ccf_ctx* c = detail::context(spec_, tol_);
        detail::check(ccf_helmholtz_step(c, hp.data(), int(hp.size()), scheme.order, forcing ? forcing->raw() : nullptr,
                                         diff_, h_, out.raw()),
                      c);
        if (bc_.kind == BoundaryCondition::Kind::dirichlet_lifted)  // timestep.cpp:84-101
            detail::add_lift_correction(out, bc_, scheme.kappa(h_) * diff_, false, tol_);
        return out;
    }

private:
    GridSpec spec_;
    double diff_, h_, tol_;
    BoundaryCondition bc_;
};

// ---- ptns.hpp:47-137
inline VectorFieldCoeffs pt_synthesize(const PTScalars& s) {
    detail::same_spec("pt_synthesize", s.lambda, s.gamma);
    VectorFieldCoeffs v(s.lambda.spec);
    ccf_ctx* c = detail::context(s.lambda.spec);
    detail::check(ccf_pt_synthesize(c, s.lambda.raw(), s.gamma.raw(), v.comp_r.raw(), v.comp_theta.raw(), v.comp_z.raw()), c);
    return v;
}
inline CoeffTensor divergence(const VectorFieldCoeffs& v);
inline PTScalars pt_decompose(const VectorFieldCoeffs& v, bool check_divergence = false, double div_tol = 1e-8) {
    detail::same_spec("pt_decompose", v.comp_r, v.comp_theta, v.comp_z);
    if (check_divergence) {  // ptns.cpp:60-67
        const double div = divergence(v).max_abs();
        const double scale = std::max(1.0, std::max({v.comp_r.max_abs(), v.comp_theta.max_abs(), v.comp_z.max_abs()}));
        if (div > div_tol * scale)
            throw NotIncompressibleError("pt_decompose: field has divergence " + std::to_string(div), div);
    }
    PTScalars s(v.comp_r.spec);
    ccf_ctx* c = detail::context(v.comp_r.spec);
    detail::check(ccf_pt_decompose(c, v.comp_r.raw(), v.comp_theta.raw(), v.comp_z.raw(), s.lambda.raw(), s.gamma.raw()), c);
    return s;
}
inline VectorFieldCoeffs curl_vector(const VectorFieldCoeffs& v) {
    detail::same_spec("curl_vector", v.comp_r, v.comp_theta, v.comp_z);
    VectorFieldCoeffs o(v.comp_r.spec);
    ccf_ctx* c = detail::context(v.comp_r.spec);
    detail::check(ccf_curl_vector(c, v.comp_r.raw(), v.comp_theta.raw(), v.comp_z.raw(), o.comp_r.raw(),
                                  o.comp_theta.raw(), o.comp_z.raw()),
                  c);
    return o;
}
inline PTScalars curl_pt(const PTScalars& s) {
    detail::same_spec("curl_pt", s.lambda, s.gamma);
    PTScalars o(s.lambda.spec);
    ccf_ctx* c = detail::context(s.lambda.spec);
    detail::check(ccf_curl_pt(c, s.lambda.raw(), s.gamma.raw(), o.lambda.raw(), o.gamma.raw()), c);
    return o;
}
inline CoeffTensor divergence(const VectorFieldCoeffs& v) {  // ptns.cpp:35-40
    CoeffTensor sum = v.comp_r;
    sum += derivative_theta(v.comp_theta);
    CoeffTensor out = derivative_r(v.comp_r);
    out += divide_r(sum);
    out += derivative_z(v.comp_z);
    return out;
}
inline PTScalars velocity_from_vorticity(const PTScalars& w, double tol = kDefaultAdiTol) {
    detail::same_spec("velocity_from_vorticity", w.lambda, w.gamma);
    PTScalars o(w.lambda.spec);
    ccf_ctx* c = detail::context(w.lambda.spec, tol);
    detail::check(ccf_velocity_from_vorticity(c, w.lambda.raw(), w.gamma.raw(), o.lambda.raw(), o.gamma.raw()), c);
    return o;
}
inline PTScalars nonlinear_term(const PTScalars& v, const PTScalars& w, bool dealias_two_thirds = false) {
    detail::same_spec("nonlinear_term", v.lambda, v.gamma, w.lambda, w.gamma);
    PTScalars o(v.lambda.spec);
    ccf_ctx* c = detail::context(v.lambda.spec);
    detail::check(ccf_nonlinear_ex(c, v.lambda.raw(), v.gamma.raw(), w.lambda.raw(), w.gamma.raw(),
                                   dealias_two_thirds ? 1 : 0, o.lambda.raw(), o.gamma.raw()),
                  c);
    return o;
}

enum class NSBootstrap { ramp, substeps };  // ptns.hpp:79-82
struct NSConfig {
    GridSpec spec;
    double reynolds = 100.0;
    double h = 1e-2;
    int order = 4;
    double adi_tol = kDefaultAdiTol;
    bool disable_nonlinear = false;   // Stokes limit
    bool dealias_two_thirds = false;
    bool compute_gamma_psi = false;   // diagnostic-only extra Poisson solve (gamma_psi())
    NSBootstrap bootstrap = NSBootstrap::ramp;
};

class NSStepper {  // state resident on the GPU between steps
public:
    NSStepper(const NSConfig& cfg, const PTScalars& omega0) : cfg_(cfg), omega_(cfg.spec) {
        // ptns.cpp:185-189
        if (!(omega0.lambda.spec == cfg.spec) || !(omega0.gamma.spec == cfg.spec))
            throw DomainError("NSStepper: initial vorticity spec mismatch");
        if (cfg.spec.m % 2 != 0) throw DomainError("NSStepper: even m required for the nonlinear pipeline");
        ctx_ = detail::context(cfg.spec, cfg.adi_tol);
        const int flags = (cfg.disable_nonlinear ? 1 : 0) | (cfg.dealias_two_thirds ? 2 : 0) | (cfg.compute_gamma_psi ? 4 : 0);
        detail::check(ccf_ns_create_ex(ctx_, cfg.reynolds, cfg.h, cfg.order, flags, omega0.lambda.raw(),
                                       omega0.gamma.raw(), &st_),
                      ctx_);
    }
    ~NSStepper() { ccf_ns_destroy(st_); }
    NSStepper(const NSStepper&) = delete;
    NSStepper& operator=(const NSStepper&) = delete;
    void step() { detail::check(ccf_ns_step(st_, 1), ctx_); }
    void steps(int k) { detail::check(ccf_ns_step(st_, k), ctx_); }
    /// Install a prebuilt history (bootstrap helpers), ptns.cpp:195-203. Newest first; nonlinear_hist[i] belongs to
    /// omega_hist[i + 1].
    void seed(const std::deque<PTScalars>& omega_hist, const std::deque<PTScalars>& nonlinear_hist, double time,
              int steps_taken) {
        if (omega_hist.empty()) throw DomainError("NSStepper::seed: empty history");
        std::vector<const double*> ol, og, nl, ng;
        for (const PTScalars& s : omega_hist) {
            if (!(s.lambda.spec == cfg_.spec) || !(s.gamma.spec == cfg_.spec))
                throw DomainError("NSStepper::seed: history spec mismatch");
            ol.push_back(s.lambda.raw());
            og.push_back(s.gamma.raw());
        }
        for (const PTScalars& s : nonlinear_hist) {
            if (!(s.lambda.spec == cfg_.spec) || !(s.gamma.spec == cfg_.spec))
                throw DomainError("NSStepper::seed: history spec mismatch");
            nl.push_back(s.lambda.raw());
            ng.push_back(s.gamma.raw());
        }
        detail::check(ccf_ns_seed(st_, int(ol.size()), ol.data(), og.data(), int(nl.size()), nl.data(), ng.data(), time,
                                  steps_taken),
                      ctx_);
        time_ = time;
        taken_ = steps_taken;
    }
    const PTScalars& omega() {
        detail::check(ccf_ns_get_omega(st_, omega_.lambda.raw(), omega_.gamma.raw(), &time_, &taken_), ctx_);
        return omega_;
    }
    double time() const { return time_; }
    const NSConfig& config() const { return cfg_; }
    PTScalars velocity() const {  // velocity scalars of the current state (fresh psi solve)
        PTScalars v(cfg_.spec);
        detail::check(ccf_ns_velocity(st_, v.lambda.raw(), v.gamma.raw()), ctx_);
        return v;
    }
    CoeffTensor gamma_psi() const {  // NSState::gamma_psi under compute_gamma_psi
        CoeffTensor g(cfg_.spec);
        detail::check(ccf_ns_gamma_psi(st_, g.raw()), ctx_);
        return g;
    }

private:
    NSConfig cfg_;
    ccf_ctx* ctx_ = nullptr;
    ccf_ns_state* st_ = nullptr;
    PTScalars omega_;
    double time_ = 0.0;
    int taken_ = 0;
};

struct NSRunResult {
    PTScalars final_omega;
    double final_time = 0.0;
    std::vector<PTScalars> snapshots;
    std::vector<double> snapshot_times;
};

// ns_run (ptns.cpp:269-324): ramp bootstrap, or NSBootstrap::substeps: [0, (b-1) h] integrated with 32 BDF2
// sub-steps per h, the sampled trajectory and its replayed nonlinear terms seeded into the full-order stepper
inline NSRunResult ns_run(const NSConfig& config, const PTScalars& initial_omega, int steps, int output_every = 0) {
    NSRunResult r;
    auto advance = [&](NSStepper& st, int first) {
        if (output_every > 0) {
            for (int s = first; s < steps; ++s) {
                st.step();
                if ((s + 1) % output_every == 0) {
                    r.snapshots.push_back(st.omega());
                    r.snapshot_times.push_back(st.time());
                }
            }
        } else if (steps > first) {
            st.steps(steps - first);  // one C-ABI call: the steady steps replay their CUDA graphs back to back
        }
        r.final_omega = st.omega();
        r.final_time = st.time();
    };
    const int b = config.order;
    const bool bootstrap = config.bootstrap == NSBootstrap::substeps && b > 1 && steps > 0;
    std::deque<PTScalars> samples{initial_omega};  // newest first
    if (bootstrap) {  // the trajectory at t = h .. (b-1) h from a BDF-min(2, b) run with 32 sub-steps per h
        constexpr int kSub = 32;
        NSConfig fine_cfg = config;
        fine_cfg.order = std::min(2, b);
        fine_cfg.h = config.h / kSub;
        fine_cfg.bootstrap = NSBootstrap::ramp;
        NSStepper fine(fine_cfg, initial_omega);  // (released before the full-order stepper takes its arenas)
        for (int level = 1; level < b; ++level) {
            fine.steps(kSub);
            samples.push_front(fine.omega());
        }
    }
    NSStepper full(config, samples.front());
    int done = 0;
    if (bootstrap) {
        std::deque<PTScalars> nl;  // N of samples[1..], newest first: the explicit extrapolation's old time levels
        if (!config.disable_nonlinear)
            for (size_t i = 1; i < samples.size(); ++i)
                nl.push_back(nonlinear_term(velocity_from_vorticity(samples[i], config.adi_tol), samples[i],
                                            config.dealias_two_thirds));
        done = b - 1;
        full.seed(samples, nl, done * config.h, done);
    }
    advance(full, done);
    return r;
}

// ---- HeatStepper / heat_run (timestep.hpp:60-111)
enum class ForcingMode { exact, lagged };  // forcing evaluated at t + h (exact) or t
struct HeatConfig {
    GridSpec spec;
    double alpha = 1.0;
    double h = 1e-2;
    int order = 4;
    double adi_tol = kDefaultAdiTol;
    ForcingMode forcing_mode = ForcingMode::exact;
    BoundaryCondition bc;
    int output_every = 0;  // 0: keep only initial and final snapshots
};
using ForcingCallback = std::function<GridField(double time)>;

class HeatStepper {  // state resident on the GPU (eigen coordinates) between steps
public:
    HeatStepper(const HeatConfig& config, const GridField& initial) : config_(config), cur_(config.spec) {
        // timestep.cpp:113-114 (the reference analyzes first, then checks the coefficient spec)
        if (!(initial.spec == config.spec)) throw DomainError("HeatStepper: initial data spec mismatch");
        init(initial.values.data(), 0);
    }
    HeatStepper(const HeatConfig& config, const CoeffTensor& initial) : config_(config), cur_(config.spec) {
        if (!(initial.spec == config.spec)) throw DomainError("HeatStepper: initial data spec mismatch");
        init(initial.raw(), 1);
    }
    ~HeatStepper() { ccf_ns_destroy(st_); }
    HeatStepper(const HeatStepper&) = delete;
    HeatStepper& operator=(const HeatStepper&) = delete;
    void step(const CoeffTensor* forcing) {
        if (forcing && !(forcing->spec == config_.spec))  // timestep.cpp:69-70
            throw DomainError("HelmholtzTensorStepper: forcing spec mismatch");
        detail::check(ccf_heat_step(st_, forcing ? forcing->raw() : nullptr, 1), ctx_);
        time_ += config_.h;
        ++steps_;
    }
    void step_with_callback(const ForcingCallback& forcing) {
        if (!forcing) return step(nullptr);
        const GridField g = forcing(config_.forcing_mode == ForcingMode::exact ? time_ + config_.h : time_);
        if (!(g.spec == config_.spec))  // analyze(g) would carry g's spec into timestep.cpp:69-70
            throw DomainError("HelmholtzTensorStepper: forcing spec mismatch");
        detail::check(ccf_heat_step(st_, g.values.data(), 0), ctx_);  // analyzed on the device
        time_ += config_.h;
        ++steps_;
    }
    const CoeffTensor& current() {
        detail::check(ccf_heat_get(st_, cur_.raw(), &time_, &steps_), ctx_);
        return cur_;
    }
    double time() const { return time_; }
    int current_order() const { return std::min(config_.order, steps_ + 1); }
    const HeatConfig& config() const { return config_; }

private:
    void init(const double* data, int kind) {
        if (config_.bc.kind == BoundaryCondition::Kind::dirichlet_lifted)
            throw ConfigError("HeatStepper: lifted boundary data is not supported by the device-resident stepper "
                              "(its state lives in the homogeneous modal basis); step HelmholtzTensorStepper with the "
                              "lifted BoundaryCondition instead");
        ctx_ = detail::context(config_.spec, config_.adi_tol);
        detail::check(ccf_heat_create(ctx_, config_.alpha, config_.h, config_.order, data, kind, &st_), ctx_);
    }
    HeatConfig config_;
    ccf_ctx* ctx_ = nullptr;
    ccf_ns_state* st_ = nullptr;
    CoeffTensor cur_;
    double time_ = 0.0;
    int steps_ = 0;
};

struct HeatRunResult {
    std::vector<GridField> snapshots;
    std::vector<double> snapshot_times;
    CoeffTensor final_coeffs;
    double final_time = 0.0;
    // timestep.cpp:102 tracks max(last_residual()) of the ADI solves. The modal solves here are exact
    // (fast diagonalization), so this is the worst relative Sylvester residual ||AXB + CXD - E|| / ||E||
    // of the solver data the run used (every BDF order's scale, both z parities; every |w| up to m = 64,
    // else |w| in {0, 1, p/4, p/2}) on seeded right-hand sides (ccf_diag_host_check, long double)
    double worst_residual = 0.0;
};

namespace detail {
inline double diag_worst_residual(const GridSpec& spec, double alpha, double h, int max_order) {
    std::vector<int> ws;
    if (spec.m <= 64) {
        for (int w = 0; w <= spec.p / 2; ++w) ws.push_back(w);
    } else {
        ws = {0, 1, spec.p / 4, spec.p / 2};
    }
    double worst = 0.0;
    for (int b = 1; b <= max_order; ++b) {
        const double scale = BDFScheme::of_order(b).kappa(h) * alpha;  // timestep.cpp:63-64
        for (int w : ws)
            for (int k0 = 0; k0 < 2; ++k0) {
                double r = 0.0;
                check(ccf_diag_host_check(spec.m, spec.n, w, scale, 0, k0, 12345u + unsigned(w), &r), nullptr);
                worst = std::max(worst, r);
            }
    }
    return worst;
}
}  // namespace detail

inline HeatRunResult heat_run(const HeatConfig& config, const GridField& initial, const ForcingCallback& forcing,
                              int steps) {  // timestep.cpp:146-170
    if (steps < 0) throw DomainError("heat_run: steps must be nonnegative");
    HeatStepper stepper(config, initial);
    HeatRunResult result;
    result.snapshots.push_back(initial);
    result.snapshot_times.push_back(0.0);
    for (int s = 0; s < steps; ++s) {
        stepper.step_with_callback(forcing);
        const bool cadence = config.output_every > 0 && (s + 1) % config.output_every == 0;
        if (cadence && s + 1 < steps) {
            result.snapshots.push_back(synthesize(stepper.current()));
            result.snapshot_times.push_back(stepper.time());
        }
    }
    result.final_coeffs = stepper.current();
    if (steps > 0) {
        result.snapshots.push_back(synthesize(result.final_coeffs));
        result.snapshot_times.push_back(stepper.time());
    }
    result.final_time = stepper.time();
    if (steps > 0) result.worst_residual = detail::diag_worst_residual(config.spec, config.alpha, config.h,
                                                                         std::min(config.order, steps));
    return result;
}

// ---- FieldFile "CCF1" (io.hpp:11-28); checksums of device data run on the GPU
inline uint32_t crc32_ieee(const uint8_t* data, size_t len) {
    unsigned c = 0;
    detail::check(ccf_crc32(data, len, &c), nullptr);
    return c;
}
inline void write_field(const std::string& path, const GridField& field) {
    detail::check(ccf_write_field(path.c_str(), 0, field.spec.m, field.spec.n, field.spec.p, field.values.data()),
                  nullptr);
}
inline void write_field(const std::string& path, const CoeffTensor& coeffs) {
    detail::check(ccf_write_field(path.c_str(), 1, coeffs.spec.m, coeffs.spec.n, coeffs.spec.p, coeffs.raw()), nullptr);
}
using FieldVariant = std::variant<GridField, CoeffTensor>;
inline FieldVariant read_field(const std::string& path) {
    int kind = 0, m = 0, n = 0, p = 0;
    detail::check(ccf_read_field_header(path.c_str(), &kind, &m, &n, &p), nullptr);
    GridSpec spec(m, n, p);
    if (kind == 0) {
        GridField f(spec);
        detail::check(ccf_read_field(path.c_str(), &kind, &m, &n, &p, f.values.data(), f.values.size()), nullptr);
        return f;
    }
    CoeffTensor t(spec);
    detail::check(ccf_read_field(path.c_str(), &kind, &m, &n, &p, t.raw(), 2 * t.data.size()), nullptr);
    return t;
}

}  // namespace cylspec
