// ============================================================================
//  CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
//  A single-threaded (optionally mode-parallel) C++20 restatement of the
//  reference `cylspec` hot path (arXiv 2206.04827 CCF spectral Navier–Stokes),
//  written from the reference's semantics, used ONLY by tests/, by
//  __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
//  --impl reference leg. The product (paper_2206_04827_b200/) never links,
//  imports or calls anything under oracle/.
//
//  Every function cites the reference file:line it restates (paths relative to
//  the reference root, e.g. proj/src/adi.cpp:150).
//
//  Third-party arithmetic the reference delegates (absent here):
//   * FFTW3 REDFT00 / complex DFT (proj/src/transform.cpp:19-60)  -> restated
//     below as a mixed-radix FFT (fft.cpp); same mathematical definition.
//   * Eigen3 GeneralizedEigenSolver (proj/src/adi.cpp:26-27)       -> delegated
//     to a registered provider callback (the Python harness supplies LAPACK
//     dggev through scipy.linalg.eigvals, the same QZ algorithm family).
//   * Eigen PartialPivLU (dense Kronecker oracle, adi.cpp:231)     -> restated
//     as a textbook partial-pivot LU.
// ============================================================================
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace oracle {

using cd = std::complex<double>;

// ---- errors: proj/include/cylspec/errors.hpp:10-40 -------------------------
struct DomainError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct SingularOperatorError : std::runtime_error {
    explicit SingularOperatorError(const std::string& w, int j = -1) : std::runtime_error(w), shift_index(j) {}
    int shift_index;
};
struct NonConvergenceError : std::runtime_error {
    NonConvergenceError(const std::string& w, std::vector<double> h) : std::runtime_error(w), history(std::move(h)) {}
    std::vector<double> history;
};
struct NotIncompressibleError : std::runtime_error {
    NotIncompressibleError(const std::string& w, double d) : std::runtime_error(w), divergence(d) {}
    double divergence;
};
struct NumericalError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---- threading knob (reference is single-threaded; >1 only for the
//      "best-effort CPU" --impl reference line) -----------------------------
void set_threads(int n);
int threads();
void parallel_for(long n, const std::function<void(long)>& body);

// ---- grid: proj/src/grid.cpp ----------------------------------------------
struct Spec {
    int m = 0, n = 0, p = 0;
    Spec() = default;
    Spec(int m_, int n_, int p_) : m(m_), n(n_), p(p_) { validate(); }
    void validate() const;                                  // grid.cpp:8-14
    long total() const { return long(m) * n * p; }
    int zero_mode() const { return p / 2; }
    int wavenumber(int l) const { return l - p / 2; }
    bool operator==(const Spec&) const = default;
};
std::vector<double> chebyshev_points(int count);           // grid.cpp:16-26
std::vector<double> fourier_points(int count);             // grid.cpp:28-34

struct Field {                                              // grid.hpp:37-50
    Spec s;
    std::vector<double> v;
    Field() = default;
    explicit Field(const Spec& sp) : s(sp), v(size_t(sp.total()), 0.0) {}
    size_t idx(int j, int k, int l) const { return (size_t(l) * s.n + k) * s.m + j; }
    double& at(int j, int k, int l) { return v[idx(j, k, l)]; }
    double at(int j, int k, int l) const { return v[idx(j, k, l)]; }
    double max_abs() const;
};

// ---- coeffs: proj/include/cylspec/coeffs.hpp, proj/src/coeffs.cpp ----------
struct Coeff {
    Spec s;
    std::vector<cd> d;
    Coeff() = default;
    explicit Coeff(const Spec& sp) : s(sp), d(size_t(sp.total()), cd(0)) {}
    size_t idx(int j, int k, int l) const { return (size_t(l) * s.n + k) * s.m + j; }
    cd& at(int j, int k, int l) { return d[idx(j, k, l)]; }
    cd at(int j, int k, int l) const { return d[idx(j, k, l)]; }
    cd* slice(int l) { return d.data() + size_t(l) * s.m * s.n; }
    const cd* slice(int l) const { return d.data() + size_t(l) * s.m * s.n; }
    double max_abs() const;
    bool all_finite() const;
    Coeff& operator+=(const Coeff& o);
    Coeff& operator-=(const Coeff& o);
    Coeff& operator*=(cd a);
};
Coeff operator+(Coeff a, const Coeff& b);
Coeff operator-(Coeff a, const Coeff& b);
enum class Parity { scalar = 0, azimuthal_flip = 1 };
void parity_project_in_place(Coeff& c, Parity p = Parity::scalar);   // coeffs.cpp:50-59
Coeff parity_project(const Coeff& c, Parity p = Parity::scalar);     // coeffs.cpp:61-65
double hermitian_symmetry_error(const Coeff& t);                     // coeffs.cpp:36-48

// ---- dense complex / real matrices (column-major) --------------------------
struct MatC {
    int r = 0, c = 0;
    std::vector<cd> a;
    MatC() = default;
    MatC(int r_, int c_) : r(r_), c(c_), a(size_t(r_) * c_, cd(0)) {}
    cd& operator()(int i, int j) { return a[size_t(j) * r + i]; }
    cd operator()(int i, int j) const { return a[size_t(j) * r + i]; }
    double norm() const;
    double max_abs() const;
};

// ---- fft (stands in for FFTW, proj/src/transform.cpp:19-60) ----------------
// out[k] = sum_j in[j] exp(sign * 2 pi i j k / n), unnormalised.
void fft(int n, const cd* in, cd* out, int sign);
// FFTW REDFT00 definition: Y_k = X_0 + (-1)^k X_{L-1} + 2 sum_{j=1}^{L-2} X_j cos(pi j k/(L-1))
void redft00(int L, const double* in, double* out);

// ---- transform: proj/src/transform.cpp -------------------------------------
Coeff analyze(const Field& f);                              // transform.cpp:122-165
Field synthesize(const Coeff& c);                           // transform.cpp:167-203
cd evaluate_at(const Coeff& c, double r, double z, double th);  // transform.cpp:205-233

// ---- calculus: proj/src/calculus.cpp ----------------------------------------
Coeff derivative_r(const Coeff& f);                         // calculus.cpp:23-32
Coeff derivative_z(const Coeff& f);                         // calculus.cpp:34-43
Coeff derivative_theta(const Coeff& f);                     // calculus.cpp:45-54
Coeff multiply_r(const Coeff& f);                           // calculus.cpp:56-69
Coeff divide_r(const Coeff& f);                             // calculus.cpp:71-97
Coeff horizontal_laplacian(const Coeff& f);                 // calculus.cpp:99-107
Coeff laplacian(const Coeff& f);                            // calculus.cpp:109-113

// ---- banded: proj/include/cylspec/banded.hpp, proj/src/banded.cpp ----------
class Banded {
public:
    Banded() = default;
    Banded(int r, int c) : rows_(r), cols_(c) {}
    static Banded identity(int n);
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    double at(int i, int j) const;                          // banded.cpp:13-20
    void set(int i, int j, double v);                       // banded.cpp:22-31
    void add(int i, int j, double v) { set(i, j, at(i, j) + v); }
    std::vector<int> offsets() const;
    int lower_bandwidth() const;
    int upper_bandwidth() const;
    Banded transposed() const;                              // banded.cpp:53-63
    Banded cropped(int r, int c) const;                     // banded.cpp:65-76
    std::vector<double> dense() const;                      // column-major rows x cols
    double max_abs() const;
    void prune(double tol = 0.0);
    Banded& operator+=(const Banded& o);
    Banded& operator-=(const Banded& o);
    Banded& operator*=(double s);
    friend Banded operator+(Banded a, const Banded& b) { return a += b; }
    friend Banded operator-(Banded a, const Banded& b) { return a -= b; }
    friend Banded operator*(const Banded& a, const Banded& b);   // banded.cpp:127-148
    MatC apply_left(const MatC& x) const;                   // banded.hpp:51-65
    MatC apply_right(const MatC& x) const;                  // banded.hpp:68-81
    const std::map<int, std::vector<double>>& bands() const { return bands_; }
private:
    int rows_ = 0, cols_ = 0;
    std::map<int, std::vector<double>> bands_;
};

class BandedLU {                                            // banded.hpp:104-153
public:
    BandedLU() = default;
    explicit BandedLU(const Banded& a) { factorize(a); }
    void factorize(const Banded& a);                        // banded.cpp:150-187
    int size() const { return n_; }
    void solve_in_place(MatC& b) const;                     // banded.hpp:117-136
    void solve_in_place_real(std::vector<double>& b, int ncols) const;
private:
    double band(int i, int j) const { return w_[size_t(i) * width_ + size_t(j - i + kl_)]; }
    double& band(int i, int j) { return w_[size_t(i) * width_ + size_t(j - i + kl_)]; }
    int n_ = 0, kl_ = 0, ku_ = 0, width_ = 0;
    std::vector<double> w_;
    std::vector<int> piv_;
};

// ---- ultraop: proj/src/ultraop.cpp ------------------------------------------
Banded build_conversion_01(int n);                          // ultraop.cpp:9-16
Banded build_conversion_12(int n);                          // ultraop.cpp:18-24
Banded build_multiplication_r(int n);                       // ultraop.cpp:30-37
Banded build_derivative_1(int n);                           // ultraop.cpp:39-44
Banded build_derivative_2(int n);                           // ultraop.cpp:46-51
struct UltraOps {                                           // ultraop.cpp:53-71
    int size = 0;
    Banded c01, c12, c02, r, r2, d1, d2;
    static const UltraOps& get(int n);
};
Banded radial_modal_laplacian(int m, int w);                // ultraop.cpp:73-81
struct ModalOperator {
    int m = 0, n = 0, wavenumber = 0;
    double scale = 0;
    Banded A, B, C, D;
    MatC apply(const MatC& x) const;                        // ultraop.cpp:83-87
};
ModalOperator assemble_modal_helmholtz(int m, int n, int w, double scale);  // ultraop.cpp:89-107
ModalOperator assemble_modal_poisson(int m, int n, int w);                  // ultraop.cpp:109-123
Banded dirichlet_recombination(int n);                      // ultraop.cpp:125-133
Banded recombine(const Banded& M);                          // ultraop.cpp:135-138

// ---- special: proj/src/special.cpp ------------------------------------------
double elliptic_K_from_kprime(double kprime);               // special.cpp:15-25
double elliptic_K(double k);                                // special.cpp:27-31
struct Jacobi { double sn, cn, dn; };
Jacobi jacobi_elliptic_from_kprime(double u, double kprime);// special.cpp:33-72
Jacobi jacobi_elliptic(double u, double k);
struct Mobius {                                             // special.cpp:80-103
    std::array<double, 4> c{1, 0, 0, 1};
    Mobius() = default;
    Mobius(double a, double b, double cc, double d);
    double operator()(double t) const { return (c[0] * t + c[1]) / (c[2] * t + c[3]); }
    Mobius inverse() const { return {c[3], -c[1], -c[2], c[0]}; }
    Mobius compose(const Mobius& g) const;
};
Mobius mobius_from_points(const std::array<double, 4>& s, const std::array<double, 4>& t);  // special.cpp:112-127

// ---- adi: proj/src/adi.cpp ------------------------------------------------
// Generalised eigenvalue provider (stands in for Eigen's QZ). Dense column-major
// n x n A and C in; alpha (complex) and beta (real) out. Returns 0 on success.
using EigProvider = int (*)(int n, const double* A, const double* C, double* alpha_re,
                            double* alpha_im, double* beta);
void set_eig_provider(EigProvider p);

struct SylvesterProblem { Banded A, B, C, D; MatC E; void check() const; };
struct ShiftPlan {
    double a = 0, b = 0, c = 0, d = 0, gamma_cr = 0, alpha_z = 0, modulus = 0, tol = 0;
    int J = 0;
    std::vector<double> u, v;
};
std::pair<double, double> spectral_bounds(const Banded& A, const Banded& C);          // adi.cpp:22-49
std::pair<double, double> spectral_bounds_gershgorin(const Banded& A, const Banded& C); // adi.cpp:51-66
ShiftPlan compute_shifts(std::pair<double, double> ca, std::pair<double, double> db, double tol);  // adi.cpp:68-104
double sylvester_residual(const SylvesterProblem& p, const MatC& x);                  // adi.cpp:106-112
struct AdiResult { MatC X; std::vector<double> history; int iterations = 0; bool converged = true; };
class AdiWorkspace {                                        // adi.cpp:114-202
public:
    AdiWorkspace(const SylvesterProblem& shape, const ShiftPlan& plan);
    AdiResult solve(const MatC& e) const;
    const ShiftPlan& plan() const { return plan_; }
private:
    ShiftPlan plan_;
    Banded A_, B_, C_, D_;
    BandedLU luBt_, luC_;
    std::vector<BandedLU> lu_shiftA_, lu_shiftBt_;
};
AdiResult adi_solve_detailed(const SylvesterProblem& p, const ShiftPlan& plan);
MatC dense_sylvester_oracle(const SylvesterProblem& p);    // adi.cpp:214-255

// ---- solvers: proj/src/solvers.cpp ----------------------------------------
struct BoundaryCondition {                                 // solvers.hpp:18-31
    bool lifted = false;
    std::optional<Coeff> lift;
};
std::pair<double, double> radial_pencil_range(int m, int w);   // solvers.cpp:15-28
std::pair<double, double> vertical_pencil_range(int n);        // solvers.cpp:30-42
class ModalSolver {                                        // solvers.cpp:46-98
public:
    ModalSolver(int m, int n, int w, double scale, bool poisson, double tol);
    MatC solve(const MatC& f_full) const;
    const ModalOperator& raw() const { return op_; }
    const SylvesterProblem& reduced_shape() const { return shape_; }
    const ShiftPlan* plan() const { return plan_ ? &*plan_ : nullptr; }
    double last_residual() const { return last_residual_; }
    int last_iterations() const { return last_iterations_; }
private:
    ModalOperator op_;
    SylvesterProblem shape_;
    Banded recomb_r_, recomb_z_;
    std::optional<ShiftPlan> plan_;
    std::unique_ptr<AdiWorkspace> adi_;
    std::unique_ptr<BandedLU> mass_lu_r_, mass_lu_zt_;
    mutable double last_residual_ = 0.0;
    mutable int last_iterations_ = 0;
};
class ModalSolverCache {                                   // solvers.cpp:100-109
public:
    ModalSolverCache(int m, int n, double tol) : m_(m), n_(n), tol_(tol) {}
    const ModalSolver& get(int w, double scale, bool poisson) const;
    int m() const { return m_; }
    int n() const { return n_; }
    double tol() const { return tol_; }
private:
    int m_, n_;
    double tol_;
    mutable std::map<std::tuple<int, double, bool>, std::unique_ptr<ModalSolver>> cache_;
    mutable std::mutex mu_;
};
MatC solve_modal_helmholtz(const ModalOperator& op, const MatC& f, const BoundaryCondition& bc, double tol);
Coeff solve_poisson_3d(const Coeff& f, const BoundaryCondition& bc, const ModalSolverCache& cache);  // solvers.cpp:142-169
Coeff solve_poisson_3d(const Coeff& f, const BoundaryCondition& bc, double tol = 1e-12);             // solvers.cpp:171-175
Coeff solve_horizontal_poisson(const Coeff& rhs);                                                     // solvers.cpp:177-203

// ---- solver statistics (oracle-side logging of ADI rounds) ------
struct AdiStats { long solves = 0; long iterations = 0; int max_rounds = 0; double worst_residual = 0; };
void adi_stats_reset();
AdiStats adi_stats();

// ---- timestep: proj/src/timestep.cpp ----------------------------------------
struct BDFScheme {                                         // timestep.cpp:5-29
    int order = 1;
    double kappa_over_h = 1.0;
    std::vector<double> w;
    static BDFScheme of_order(int b);
    double kappa(double h) const { return kappa_over_h * h; }
};
std::vector<double> imex_coefficients(int order);          // timestep.cpp:31-39
Coeff bdf_rhs(const std::deque<Coeff>& hist, const BDFScheme& s);  // timestep.cpp:41-51
class HelmholtzTensorStepper {                             // timestep.cpp:53-108
public:
    HelmholtzTensorStepper(const Spec& spec, double diffusivity, double h, double tol, BoundaryCondition bc = {});
    Coeff step(const std::deque<Coeff>& hist, const BDFScheme& s, const Coeff* forcing) const;
    double worst_residual() const { return worst_; }
private:
    Spec spec_;
    double diff_, h_;
    BoundaryCondition bc_;
    ModalSolverCache cache_;
    mutable double worst_ = 0.0;
};
using ForcingCallback = std::function<Field(double)>;
struct HeatConfig { Spec spec; double alpha = 1.0, h = 1e-2; int order = 4; double tol = 1e-12; bool exact_forcing = true; };
class HeatStepper {                                        // timestep.cpp:110-144
public:
    HeatStepper(const HeatConfig& cfg, Coeff initial);
    void step(const Coeff* forcing);
    void step_with_callback(const ForcingCallback& f);
    const Coeff& current() const { return hist_.front(); }
    double time() const { return time_; }
    int current_order() const { return std::min(cfg_.order, steps_ + 1); }
    double worst_residual() const { return stepper_.worst_residual(); }
private:
    HeatConfig cfg_;
    HelmholtzTensorStepper stepper_;
    std::deque<Coeff> hist_;
    double time_ = 0;
    int steps_ = 0;
};

// ---- ptns: proj/src/ptns.cpp ------------------------------------------------
struct PT { Coeff lambda, gamma; };
struct Vec3 { Coeff r, t, z; };
Vec3 curl_vector(const Vec3& v);                           // ptns.cpp:25-33
Coeff divergence(const Vec3& v);                           // ptns.cpp:35-40
Vec3 pt_synthesize(const PT& s);                           // ptns.cpp:42-57
PT pt_decompose(const Vec3& v, bool check_divergence = true, double div_tol = 1e-8);  // ptns.cpp:59-77
PT curl_pt(const PT& s);                                   // ptns.cpp:79-83
PT velocity_from_vorticity(const PT& omega, const ModalSolverCache& cache);          // ptns.cpp:85-91
PT nonlinear_term(const PT& v, const PT& omega, bool dealias = false);               // ptns.cpp:114-149
struct NSConfig { Spec spec; double reynolds = 100, h = 1e-2; int order = 4; double tol = 1e-12;
                  bool disable_nonlinear = false, dealias = false; };
class NSStepper {                                          // ptns.cpp:177-267
public:
    NSStepper(const NSConfig& cfg, PT omega0);
    void step();
    void seed(std::deque<PT> omega_hist, std::deque<PT> nonlinear_hist, double time, int steps_taken);  // ptns.cpp:195-203
    const PT& omega() const { return omega_.front(); }
    double time() const { return time_; }
    int steps_taken() const { return steps_; }
    PT velocity() const;
private:
    NSConfig cfg_;
    HelmholtzTensorStepper stepper_;
    ModalSolverCache poisson_cache_;
    std::deque<PT> omega_, nonlinear_;
    double time_ = 0;
    int steps_ = 0;
};

// ptns.cpp:269-324; substeps: the NSBootstrap::substeps branch (:272-311), else the ramp bootstrap
PT ns_run(const NSConfig& cfg, const PT& omega0, int steps, bool substeps, double* final_time);

// ---- io: proj/src/io.cpp:12-109 (CCF1 FieldFile) ---------------------------
uint32_t crc32_ieee(const uint8_t* data, size_t len);

}  // namespace oracle
