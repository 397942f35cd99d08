// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Banded matrices + banded LU (proj/include/cylspec/banded.hpp, proj/src/banded.cpp),
// ultraspherical operators (proj/src/ultraop.cpp), elliptic functions
// (proj/src/special.cpp).
#include <algorithm>
#include <cmath>
#include <numbers>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- Banded
Banded Banded::identity(int n) {
    Banded m(n, n);
    for (int i = 0; i < n; ++i) m.set(i, i, 1.0);
    return m;
}

double Banded::at(int i, int j) const {  // banded.cpp:13-20
    const int d = j - i;
    auto it = bands_.find(d);
    if (it == bands_.end()) return 0.0;
    const int i0 = std::max(0, -d);
    if (i < i0 || i >= i0 + int(it->second.size())) return 0.0;
    return it->second[size_t(i - i0)];
}

void Banded::set(int i, int j, double v) {  // banded.cpp:22-31
    if (i < 0 || i >= rows_ || j < 0 || j >= cols_) throw DomainError("BandedMatrix::set: index out of range");
    const int d = j - i;
    auto& vals = bands_[d];
    const int i0 = std::max(0, -d);
    const int len = std::min(rows_ - i0, cols_ - std::max(0, d));
    if (vals.empty()) vals.assign(size_t(len), 0.0);
    vals[size_t(i - i0)] = v;
}

std::vector<int> Banded::offsets() const {
    std::vector<int> o;
    for (const auto& [d, v] : bands_) o.push_back(d);
    return o;
}
int Banded::lower_bandwidth() const {
    int kl = 0;
    for (const auto& [d, v] : bands_)
        if (d < 0) kl = std::max(kl, -d);
    return kl;
}
int Banded::upper_bandwidth() const {
    int ku = 0;
    for (const auto& [d, v] : bands_)
        if (d > 0) ku = std::max(ku, d);
    return ku;
}

Banded Banded::transposed() const {  // banded.cpp:53-63
    Banded t(cols_, rows_);
    for (const auto& [d, vals] : bands_) {
        const int i0 = std::max(0, -d);
        for (int q = 0; q < int(vals.size()); ++q)
            if (vals[size_t(q)] != 0.0) t.set(i0 + q + d, i0 + q, vals[size_t(q)]);
    }
    return t;
}

Banded Banded::cropped(int r, int c) const {  // banded.cpp:65-76
    if (r > rows_ || c > cols_) throw DomainError("BandedMatrix::cropped: enlarging");
    Banded o(r, c);
    for (const auto& [d, vals] : bands_) {
        const int i0 = std::max(0, -d);
        for (int q = 0; q < int(vals.size()); ++q) {
            const int i = i0 + q, j = i + d;
            if (i < r && j < c && vals[size_t(q)] != 0.0) o.set(i, j, vals[size_t(q)]);
        }
    }
    return o;
}

std::vector<double> Banded::dense() const {
    std::vector<double> o(static_cast<size_t>(rows_) * cols_, 0.0);
    for (const auto& [d, vals] : bands_) {
        const int i0 = std::max(0, -d);
        for (int q = 0; q < int(vals.size()); ++q) o[size_t(i0 + q + d) * rows_ + (i0 + q)] = vals[size_t(q)];
    }
    return o;
}

double Banded::max_abs() const {
    double m = 0;
    for (const auto& [d, vals] : bands_)
        for (double v : vals) m = std::max(m, std::abs(v));
    return m;
}

void Banded::prune(double tol) {
    for (auto it = bands_.begin(); it != bands_.end();) {
        bool zero = true;
        for (double v : it->second)
            if (std::abs(v) > tol) {
                zero = false;
                break;
            }
        it = zero ? bands_.erase(it) : std::next(it);
    }
}

Banded& Banded::operator+=(const Banded& o) {  // banded.cpp:101-109
    if (rows_ != o.rows_ || cols_ != o.cols_) throw DomainError("BandedMatrix: size mismatch in +=");
    for (const auto& [d, vals] : o.bands_) {
        const int i0 = std::max(0, -d);
        for (int q = 0; q < int(vals.size()); ++q)
            if (vals[size_t(q)] != 0.0) add(i0 + q, i0 + q + d, vals[size_t(q)]);
    }
    return *this;
}
Banded& Banded::operator-=(const Banded& o) {
    Banded neg = o;
    neg *= -1.0;
    return (*this) += neg;
}
Banded& Banded::operator*=(double s) {
    for (auto& [d, vals] : bands_)
        for (double& v : vals) v *= s;
    return *this;
}

Banded operator*(const Banded& a, const Banded& b) {  // banded.cpp:127-148
    if (a.cols_ != b.rows_) throw DomainError("BandedMatrix: size mismatch in *");
    Banded c(a.rows_, b.cols_);
    for (const auto& [da, va] : a.bands_) {
        const int ia0 = std::max(0, -da);
        for (const auto& [db, vb] : b.bands_) {
            const int ib0 = std::max(0, -db);
            for (int t = 0; t < int(va.size()); ++t) {
                const int i = ia0 + t, k = i + da, j = k + db;
                if (j < 0 || j >= b.cols_) continue;
                if (k < ib0 || k >= ib0 + int(vb.size())) continue;
                const double prod = va[size_t(t)] * vb[size_t(k - ib0)];
                if (prod != 0.0) c.add(i, j, prod);
            }
        }
    }
    c.prune();
    return c;
}

MatC Banded::apply_left(const MatC& x) const {  // banded.hpp:51-65
    if (x.r != cols_) throw DomainError("BandedMatrix::apply_left: size mismatch");
    MatC y(rows_, x.c);
    for (const auto& [d, vals] : bands_) {
        const int i0 = std::max(0, -d), i1 = std::min(rows_, cols_ - d);
        for (int c = 0; c < x.c; ++c)
            for (int i = i0; i < i1; ++i) y(i, c) += vals[size_t(i - i0)] * x(i + d, c);
    }
    return y;
}

MatC Banded::apply_right(const MatC& x) const {  // banded.hpp:68-81
    if (x.c != rows_) throw DomainError("BandedMatrix::apply_right: size mismatch");
    MatC y(x.r, cols_);
    for (const auto& [d, vals] : bands_) {
        const int i0 = std::max(0, -d), i1 = std::min(rows_, cols_ - d);
        for (int i = i0; i < i1; ++i) {
            const double v = vals[size_t(i - i0)];
            for (int r = 0; r < x.r; ++r) y(r, i + d) += v * x(r, i);
        }
    }
    return y;
}

// ---------------------------------------------------------------- BandedLU
void BandedLU::factorize(const Banded& a) {  // banded.cpp:150-187
    if (a.rows() != a.cols()) throw DomainError("BandedLU: matrix must be square");
    n_ = a.rows();
    kl_ = a.lower_bandwidth();
    ku_ = a.upper_bandwidth();
    width_ = 2 * kl_ + ku_ + 1;
    w_.assign(size_t(n_) * width_, 0.0);
    piv_.assign(size_t(n_), 0);
    for (int i = 0; i < n_; ++i) {
        const int j0 = std::max(0, i - kl_), j1 = std::min(n_ - 1, i + ku_);
        for (int j = j0; j <= j1; ++j) band(i, j) = a.at(i, j);
    }
    for (int k = 0; k < n_; ++k) {
        int p = k;
        double pmax = std::abs(band(k, k));
        const int iend = std::min(n_ - 1, k + kl_);
        for (int i = k + 1; i <= iend; ++i) {
            const double v = std::abs(band(i, k));
            if (v > pmax) {
                pmax = v;
                p = i;
            }
        }
        if (pmax == 0.0) throw SingularOperatorError("BandedLU: singular matrix");
        piv_[size_t(k)] = p;
        if (p != k) {
            const int jend = std::min(n_ - 1, k + kl_ + ku_);
            for (int j = k; j <= jend; ++j) std::swap(band(k, j), band(p, j));
        }
        const double pivot = band(k, k);
        for (int i = k + 1; i <= iend; ++i) {
            const double m = band(i, k) / pivot;
            band(i, k) = m;
            if (m != 0.0) {
                const int jend = std::min(n_ - 1, k + kl_ + ku_);
                for (int j = k + 1; j <= jend; ++j) band(i, j) -= m * band(k, j);
            }
        }
    }
}

void BandedLU::solve_in_place(MatC& b) const {  // banded.hpp:117-136
    if (b.r != n_) throw DomainError("BandedLU::solve: size mismatch");
    for (int c = 0; c < b.c; ++c) {
        cd* x = b.a.data() + size_t(c) * b.r;
        for (int k = 0; k < n_; ++k) {
            if (piv_[size_t(k)] != k) std::swap(x[k], x[piv_[size_t(k)]]);
            const int iend = std::min(n_ - 1, k + kl_);
            for (int i = k + 1; i <= iend; ++i) x[i] -= band(i, k) * x[k];
        }
        for (int k = n_ - 1; k >= 0; --k) {
            const int jend = std::min(n_ - 1, k + kl_ + ku_);
            cd s = x[k];
            for (int j = k + 1; j <= jend; ++j) s -= band(k, j) * x[j];
            x[k] = s / band(k, k);
        }
    }
}

void BandedLU::solve_in_place_real(std::vector<double>& b, int ncols) const {
    for (int c = 0; c < ncols; ++c) {
        double* x = b.data() + size_t(c) * n_;
        for (int k = 0; k < n_; ++k) {
            if (piv_[size_t(k)] != k) std::swap(x[k], x[piv_[size_t(k)]]);
            const int iend = std::min(n_ - 1, k + kl_);
            for (int i = k + 1; i <= iend; ++i) x[i] -= band(i, k) * x[k];
        }
        for (int k = n_ - 1; k >= 0; --k) {
            const int jend = std::min(n_ - 1, k + kl_ + ku_);
            double s = x[k];
            for (int j = k + 1; j <= jend; ++j) s -= band(k, j) * x[j];
            x[k] = s / band(k, k);
        }
    }
}

// ---------------------------------------------------------------- ultraop (proj/src/ultraop.cpp)
Banded build_conversion_01(int n) {  // ultraop.cpp:9-16
    if (n < 2) throw DomainError("build_conversion_01: n >= 2 required");
    Banded m(n, n);
    m.set(0, 0, 1.0);
    for (int k = 1; k < n; ++k) m.set(k, k, 0.5);
    for (int k = 0; k + 2 < n; ++k) m.set(k, k + 2, -0.5);
    return m;
}
Banded build_conversion_12(int n) {  // ultraop.cpp:18-24
    if (n < 2) throw DomainError("build_conversion_12: n >= 2 required");
    Banded m(n, n);
    for (int k = 0; k < n; ++k) m.set(k, k, 1.0 / double(k + 1));
    for (int k = 0; k + 2 < n; ++k) m.set(k, k + 2, -1.0 / double(k + 3));
    return m;
}
Banded build_multiplication_r(int n) {  // ultraop.cpp:30-37
    if (n < 2) throw DomainError("build_multiplication_r: n >= 2 required");
    Banded m(n, n);
    for (int k = 0; k + 1 < n; ++k) m.set(k + 1, k, double(k + 1) / double(2 * (k + 2)));
    for (int k = 1; k < n; ++k) m.set(k - 1, k, double(k + 3) / double(2 * (k + 2)));
    return m;
}
Banded build_derivative_1(int n) {  // ultraop.cpp:39-44
    if (n < 3) throw DomainError("build_derivative_1: n >= 3 required");
    Banded m(n, n);
    for (int k = 0; k + 1 < n; ++k) m.set(k, k + 1, double(k + 1));
    return m;
}
Banded build_derivative_2(int n) {  // ultraop.cpp:46-51
    if (n < 3) throw DomainError("build_derivative_2: n >= 3 required");
    Banded m(n, n);
    for (int k = 0; k + 2 < n; ++k) m.set(k, k + 2, 2.0 * double(k + 2));
    return m;
}

const UltraOps& UltraOps::get(int n) {  // ultraop.cpp:53-71
    static std::mutex mu;
    static std::map<int, std::unique_ptr<UltraOps>> cache;
    std::lock_guard<std::mutex> g(mu);
    auto& s = cache[n];
    if (!s) {
        auto o = std::make_unique<UltraOps>();
        o->size = n;
        o->c01 = build_conversion_01(n);
        o->c12 = build_conversion_12(n);
        o->c02 = o->c12 * o->c01;
        o->r = build_multiplication_r(n);
        o->r2 = o->r * o->r * o->c02;
        o->d1 = build_derivative_1(n);
        o->d2 = build_derivative_2(n);
        s = std::move(o);
    }
    return *s;
}

Banded radial_modal_laplacian(int m, int w) {  // ultraop.cpp:73-81
    const UltraOps& o = UltraOps::get(m);
    Banded l = o.r * o.c12 * o.d1 + o.r * o.r * o.d2;
    Banded w2 = o.c02;
    w2 *= double(w) * double(w);
    l -= w2;
    l.prune();
    return l;
}

MatC ModalOperator::apply(const MatC& x) const {  // ultraop.cpp:83-87
    MatC out = B.apply_right(A.apply_left(x));
    if (C.rows() > 0 && C.max_abs() > 0.0) {
        MatC t = D.apply_right(C.apply_left(x));
        for (size_t i = 0; i < out.a.size(); ++i) out.a[i] += t.a[i];
    }
    return out;
}

ModalOperator assemble_modal_helmholtz(int m, int n, int w, double scale) {  // ultraop.cpp:89-107
    if (m < 4 || n < 4) throw DomainError("assemble_modal_helmholtz: sizes too small");
    const UltraOps& ro = UltraOps::get(m);
    const UltraOps& zo = UltraOps::get(n);
    ModalOperator op;
    op.m = m;
    op.n = n;
    op.wavenumber = w;
    op.scale = scale;
    Banded lap = radial_modal_laplacian(m, w);
    lap *= scale;
    op.A = ro.r2 - lap;
    op.B = zo.c02.transposed();
    op.C = ro.r2;
    op.C *= -scale;
    op.C.prune();
    op.D = zo.d2.transposed();
    return op;
}

ModalOperator assemble_modal_poisson(int m, int n, int w) {  // ultraop.cpp:109-123
    if (m < 4 || n < 4) throw DomainError("assemble_modal_poisson: sizes too small");
    const UltraOps& ro = UltraOps::get(m);
    const UltraOps& zo = UltraOps::get(n);
    ModalOperator op;
    op.m = m;
    op.n = n;
    op.wavenumber = w;
    op.scale = 1.0;
    op.A = radial_modal_laplacian(m, w);
    op.B = zo.c02.transposed();
    op.C = ro.r2;
    op.D = zo.d2.transposed();
    return op;
}

Banded dirichlet_recombination(int n) {  // ultraop.cpp:125-133
    if (n < 4) throw DomainError("dirichlet_recombination: n >= 4 required");
    Banded s(n, n - 2);
    for (int j = 0; j + 2 < n; ++j) {
        s.set(j, j, 1.0);
        s.set(j + 2, j, -1.0);
    }
    return s;
}

Banded recombine(const Banded& M) {  // ultraop.cpp:135-138
    Banded prod = M * dirichlet_recombination(M.cols());
    return prod.cropped(M.rows() - 2, M.cols() - 2);
}

// ---------------------------------------------------------------- special (proj/src/special.cpp)
static constexpr double kAgmTol = 1e-16;
static constexpr int kAgmMaxIter = 64;

double elliptic_K_from_kprime(double kp) {  // special.cpp:15-25
    if (!(kp > 0.0) || kp > 1.0) throw DomainError("elliptic_K: complementary modulus must be in (0,1]");
    double a = 1.0, b = kp;
    for (int i = 0; i < kAgmMaxIter && std::abs(a - b) > kAgmTol * a; ++i) {
        const double an = 0.5 * (a + b);
        b = std::sqrt(a * b);
        a = an;
    }
    return std::numbers::pi / (2.0 * a);
}

double elliptic_K(double k) {  // special.cpp:27-31
    if (k < 0.0 || k >= 1.0) throw DomainError("elliptic_K: modulus must satisfy 0 <= k < 1");
    return elliptic_K_from_kprime(std::sqrt((1.0 - k) * (1.0 + k)));
}

Jacobi jacobi_elliptic_from_kprime(double u, double kp) {  // special.cpp:33-72
    if (!(kp > 0.0) || kp > 1.0) throw DomainError("jacobi_elliptic: complementary modulus must be in (0,1]");
    const double k2 = std::max(0.0, (1.0 - kp) * (1.0 + kp));
    const double k = std::sqrt(k2);
    std::vector<double> a{1.0}, c{k};
    double b = kp;
    int N = 0;
    while (std::abs(c.back()) > kAgmTol * a.back() && N < kAgmMaxIter) {
        const double an = 0.5 * (a.back() + b);
        const double cn = 0.5 * (a.back() - b);
        b = std::sqrt(a.back() * b);
        a.push_back(an);
        c.push_back(cn);
        ++N;
    }
    if (N == 0) return {std::sin(u), std::cos(u), 1.0};
    double phi = std::ldexp(a[size_t(N)] * u, N);
    double phi_prev = phi;
    for (int i = N; i >= 1; --i) {
        phi_prev = phi;
        const double s = std::clamp(c[size_t(i)] / a[size_t(i)] * std::sin(phi), -1.0, 1.0);
        phi = 0.5 * (phi + std::asin(s));
    }
    Jacobi out;
    out.sn = std::sin(phi);
    out.cn = std::cos(phi);
    const double den = std::cos(phi_prev - phi);
    out.dn = std::abs(den) > 1e-12 ? out.cn / den : std::sqrt(1.0 - k2 * out.sn * out.sn);
    return out;
}

Jacobi jacobi_elliptic(double u, double k) {
    if (k < 0.0 || k >= 1.0) throw DomainError("jacobi_elliptic: modulus must satisfy 0 <= k < 1");
    return jacobi_elliptic_from_kprime(u, std::sqrt((1.0 - k) * (1.0 + k)));
}

Mobius::Mobius(double a, double b, double cc, double d) : c{a, b, cc, d} {  // special.cpp:76-79
    if (std::abs(a * d - b * cc) < 1e-300) throw DomainError("MobiusMap: zero determinant");
}

Mobius Mobius::compose(const Mobius& g) const {  // special.cpp:89-94
    const auto& f = c;
    return {f[0] * g.c[0] + f[1] * g.c[2], f[0] * g.c[1] + f[1] * g.c[3], f[2] * g.c[0] + f[3] * g.c[2],
            f[2] * g.c[1] + f[3] * g.c[3]};
}

Mobius mobius_from_points(const std::array<double, 4>& s, const std::array<double, 4>& t) {  // special.cpp:112-127
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j) {
            if (s[i] == s[j]) throw DomainError("mobius_from_points: repeated source point");
            if (t[i] == t[j]) throw DomainError("mobius_from_points: repeated target point");
        }
    auto three = [](double z1, double z2, double z3) {  // special.cpp:99-102
        return std::array<double, 4>{z2 - z3, -z1 * (z2 - z3), z2 - z1, -z3 * (z2 - z1)};
    };
    const auto a = three(s[0], s[1], s[3]);
    const auto b = three(t[0], t[1], t[3]);
    const Mobius ms(a[0], a[1], a[2], a[3]);
    const Mobius mt(b[0], b[1], b[2], b[3]);
    return mt.inverse().compose(ms);
}

}  // namespace oracle
