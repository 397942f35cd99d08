// Host setup numerics (see setup.hpp). One-time cost per context; never on the
// per-step path.
#include "setup.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <limits>
#include <numbers>

namespace ccf {

Dense matmul(const Dense& x, const Dense& y) {
    Dense z(x.r, y.c);
    for (int i = 0; i < x.r; ++i)
        for (int k = 0; k < x.c; ++k) {
            const double a = x(i, k);
            if (a == 0.0) continue;
            const double* yr = &y.a[size_t(k) * y.c];
            double* zr = &z.a[size_t(i) * z.c];
            for (int j = 0; j < y.c; ++j) zr[j] += a * yr[j];
        }
    return z;
}

Dense transpose(const Dense& x) {
    Dense t(x.c, x.r);
    for (int i = 0; i < x.r; ++i)
        for (int j = 0; j < x.c; ++j) t(j, i) = x(i, j);
    return t;
}

// ---------------------------------------------------------------- operators
Ultra::Ultra(int n_) : n(n_) {
    if (n < 4) throw Error(DOMAIN_ERROR, "Ultra: n >= 4 required");
    c01 = Dense(n, n);
    c12 = Dense(n, n);
    r = Dense(n, n);
    d1 = Dense(n, n);
    d2 = Dense(n, n);
    c01(0, 0) = 1.0;                                   // ultraop.cpp:9-16
    for (int k = 1; k < n; ++k) c01(k, k) = 0.5;
    for (int k = 0; k + 2 < n; ++k) c01(k, k + 2) = -0.5;
    for (int k = 0; k < n; ++k) c12(k, k) = 1.0 / double(k + 1);   // ultraop.cpp:18-24
    for (int k = 0; k + 2 < n; ++k) c12(k, k + 2) = -1.0 / double(k + 3);
    for (int k = 0; k + 1 < n; ++k) r(k + 1, k) = double(k + 1) / double(2 * (k + 2));  // ultraop.cpp:30-37
    for (int k = 1; k < n; ++k) r(k - 1, k) = double(k + 3) / double(2 * (k + 2));
    for (int k = 0; k + 1 < n; ++k) d1(k, k + 1) = double(k + 1);  // ultraop.cpp:39-44
    for (int k = 0; k + 2 < n; ++k) d2(k, k + 2) = 2.0 * double(k + 2);  // ultraop.cpp:46-51
    c02 = matmul(c12, c01);
    const Dense rr = matmul(r, r);
    r2 = matmul(rr, c02);
    rrc02 = r2;
    l0 = matmul(matmul(r, c12), d1);
    const Dense t = matmul(rr, d2);
    for (size_t i = 0; i < l0.a.size(); ++i) l0.a[i] += t.a[i];
}

Dense radial_laplacian(const Ultra& u, int w) {
    Dense l = u.l0;
    const double w2 = double(w) * double(w);
    for (size_t i = 0; i < l.a.size(); ++i) l.a[i] -= w2 * u.c02.a[i];
    return l;
}

Dense recombine(const Dense& M) {
    Dense o(M.r - 2, M.c - 2);
    for (int i = 0; i < M.r - 2; ++i)
        for (int j = 0; j < M.c - 2; ++j) o(i, j) = M(i, j) - M(i, j + 2);
    return o;
}

CBand compress(const Dense& M, int parity, int rows, int cols, int lo, int hi) {
    CBand b;
    b.rows = rows;
    b.lo = lo;
    b.hi = hi;
    const int w = hi - lo + 1;
    b.v.assign(size_t(rows) * w, 0.0);
    for (int a = 0; a < rows; ++a)
        for (int d = lo; d <= hi; ++d) {
            const int c = a + d;
            if (c < 0 || c >= cols) continue;
            const int i = 2 * a + parity, j = 2 * c + parity;
            if (i < M.r && j < M.c) b.v[size_t(a) * w + (d - lo)] = M(i, j);
        }
    return b;
}

// ---------------------------------------------------------------- banded LU (banded.cpp:150-187)
CLU banded_lu(const CBand& A, int kl, int ku) {
    const int n = A.rows;
    CLU f;
    f.n = n;
    f.kl = kl;
    f.ku = ku;
    const int width = 2 * kl + ku + 1;  // row i covers columns [i-kl, i+kl+ku]
    std::vector<double> w(size_t(n) * width, 0.0);
    auto band = [&](int i, int j) -> double& { return w[size_t(i) * width + size_t(j - i + kl)]; };
    for (int i = 0; i < n; ++i)
        for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) band(i, j) = A.at(i, j - i);
    f.L.assign(size_t(n) * std::max(kl, 1), 0.0);
    f.piv.assign(size_t(n), 0);
    f.U.assign(size_t(n) * (kl + ku), 0.0);
    f.inv.assign(size_t(n), 0.0);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double pmax = std::abs(band(k, k));
        const int iend = std::min(n - 1, k + kl);
        for (int i = k + 1; i <= iend; ++i)
            if (std::abs(band(i, k)) > pmax) {
                pmax = std::abs(band(i, k));
                p = i;
            }
        if (pmax == 0.0) throw Error(SINGULAR, "BandedLU: singular matrix");
        f.piv[size_t(k)] = p - k;
        const int jend = std::min(n - 1, k + kl + ku);
        if (p != k)
            for (int j = k; j <= jend; ++j) std::swap(band(k, j), band(p, j));
        const double pivot = band(k, k);
        for (int i = k + 1; i <= iend; ++i) {
            const double m = band(i, k) / pivot;
            band(i, k) = m;
            if (m != 0.0)
                for (int j = k + 1; j <= jend; ++j) band(i, j) -= m * band(k, j);
        }
    }
    for (int k = 0; k < n; ++k) {
        for (int t = 0; t < kl; ++t) f.L[size_t(k) * kl + t] = (k + 1 + t < n) ? band(k + 1 + t, k) : 0.0;
        f.inv[size_t(k)] = 1.0 / band(k, k);
        for (int t = 0; t < kl + ku; ++t) f.U[size_t(k) * (kl + ku) + t] = (k + 1 + t < n) ? band(k, k + 1 + t) : 0.0;
    }
    return f;
}

// ---------------------------------------------------------------- eigenvalues
namespace {

// Dense LU with partial pivoting, in place (row-major). Returns false if singular.
bool dense_lu(Dense& a, std::vector<int>& perm) {
    const int n = a.r;
    perm.resize(size_t(n));
    for (int i = 0; i < n; ++i) perm[size_t(i)] = i;
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
        if (a(p, k) == 0.0) return false;
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(a(k, j), a(p, j));
            std::swap(perm[size_t(k)], perm[size_t(p)]);
        }
        const double inv = 1.0 / a(k, k);
        for (int i = k + 1; i < n; ++i) {
            const double m = a(i, k) * inv;
            a(i, k) = m;
            if (m == 0.0) continue;
            for (int j = k + 1; j < n; ++j) a(i, j) -= m * a(k, j);
        }
    }
    return true;
}

// Parlett–Reinsch balancing by powers of two.
void balance(Dense& a) {
    const int n = a.r;
    bool done = false;
    while (!done) {
        done = true;
        for (int i = 0; i < n; ++i) {
            double r = 0, c = 0;
            for (int j = 0; j < n; ++j)
                if (j != i) {
                    c += std::abs(a(j, i));
                    r += std::abs(a(i, j));
                }
            if (c == 0.0 || r == 0.0) continue;
            const double s = c + r;
            double f = 1.0, g = r / 2.0;
            while (c < g) {
                f *= 2.0;
                c *= 4.0;
            }
            g = r * 2.0;
            while (c > g) {
                f /= 2.0;
                c /= 4.0;
            }
            if ((c + r) / f < 0.95 * s) {
                done = false;
                const double gi = 1.0 / f;
                for (int j = 0; j < n; ++j) a(i, j) *= gi;
                for (int j = 0; j < n; ++j) a(j, i) *= f;
            }
        }
    }
}

// Householder reduction to upper Hessenberg form.
void hessenberg(Dense& a) {
    const int n = a.r;
    std::vector<double> v(static_cast<size_t>(n));
    for (int k = 0; k + 2 < n; ++k) {
        double norm = 0;
        for (int i = k + 1; i < n; ++i) norm += a(i, k) * a(i, k);
        norm = std::sqrt(norm);
        if (norm == 0.0) continue;
        const double alpha = a(k + 1, k) > 0 ? -norm : norm;
        for (int i = 0; i < n; ++i) v[size_t(i)] = 0.0;
        v[size_t(k + 1)] = a(k + 1, k) - alpha;
        for (int i = k + 2; i < n; ++i) v[size_t(i)] = a(i, k);
        double vn = 0;
        for (int i = k + 1; i < n; ++i) vn += v[size_t(i)] * v[size_t(i)];
        if (vn == 0.0) continue;
        const double beta = 2.0 / vn;
        // A <- (I - beta v v^T) A
        for (int j = 0; j < n; ++j) {
            double s = 0;
            for (int i = k + 1; i < n; ++i) s += v[size_t(i)] * a(i, j);
            s *= beta;
            for (int i = k + 1; i < n; ++i) a(i, j) -= s * v[size_t(i)];
        }
        // A <- A (I - beta v v^T)
        for (int i = 0; i < n; ++i) {
            double s = 0;
            for (int j = k + 1; j < n; ++j) s += a(i, j) * v[size_t(j)];
            s *= beta;
            for (int j = k + 1; j < n; ++j) a(i, j) -= s * v[size_t(j)];
        }
        a(k + 1, k) = alpha;
        for (int i = k + 2; i < n; ++i) a(i, k) = 0.0;
    }
}

inline double sgn(double a, double b) { return b >= 0 ? std::abs(a) : -std::abs(a); }

// Francis double-shift QR on an upper Hessenberg matrix: eigenvalues only.
void hessenberg_qr(Dense& a, std::vector<double>& wr, std::vector<double>& wi) {
    const int n = a.r;
    wr.assign(size_t(n), 0.0);
    wi.assign(size_t(n), 0.0);
    double anorm = 0;
    for (int i = 0; i < n; ++i)
        for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::abs(a(i, j));
    int hi = n - 1, its = 0;
    double t = 0.0;
    while (hi >= 0) {
        int l = hi;
        for (; l >= 1; --l) {
            double s = std::abs(a(l - 1, l - 1)) + std::abs(a(l, l));
            if (s == 0.0) s = anorm;
            if (std::abs(a(l, l - 1)) + s == s) {
                a(l, l - 1) = 0.0;
                break;
            }
        }
        double x = a(hi, hi);
        if (l == hi) {  // one root
            wr[size_t(hi)] = x + t;
            wi[size_t(hi)] = 0.0;
            --hi;
            its = 0;
            continue;
        }
        double y = a(hi - 1, hi - 1), w = a(hi, hi - 1) * a(hi - 1, hi);
        if (l == hi - 1) {  // two roots
            const double p = 0.5 * (y - x), q = p * p + w;
            double z = std::sqrt(std::abs(q));
            x += t;
            if (q >= 0.0) {
                z = p + sgn(z, p);
                wr[size_t(hi - 1)] = wr[size_t(hi)] = x + z;
                if (z != 0.0) wr[size_t(hi)] = x - w / z;
                wi[size_t(hi - 1)] = wi[size_t(hi)] = 0.0;
            } else {
                wr[size_t(hi - 1)] = wr[size_t(hi)] = x + p;
                wi[size_t(hi - 1)] = -z;
                wi[size_t(hi)] = z;
            }
            hi -= 2;
            its = 0;
            continue;
        }
        if (its == 90) throw Error(NUMERICAL, "spectral_bounds: QR iteration did not converge");
        if (its == 10 || its == 20 || its == 40) {  // exceptional shift
            t += x;
            for (int i = 0; i <= hi; ++i) a(i, i) -= x;
            const double s = std::abs(a(hi, hi - 1)) + std::abs(a(hi - 1, hi - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
        }
        ++its;
        int mm = hi - 2;
        double p = 0, q = 0, r = 0, z = 0;
        for (; mm >= l; --mm) {
            z = a(mm, mm);
            r = x - z;
            const double s0 = y - z;
            p = (r * s0 - w) / a(mm + 1, mm) + a(mm, mm + 1);
            q = a(mm + 1, mm + 1) - z - r - s0;
            r = a(mm + 2, mm + 1);
            const double s = std::abs(p) + std::abs(q) + std::abs(r);
            p /= s;
            q /= s;
            r /= s;
            if (mm == l) break;
            const double u = std::abs(a(mm, mm - 1)) * (std::abs(q) + std::abs(r));
            const double v = std::abs(p) * (std::abs(a(mm - 1, mm - 1)) + std::abs(z) + std::abs(a(mm + 1, mm + 1)));
            if (u + v == v) break;
        }
        for (int i = mm + 2; i <= hi; ++i) {
            a(i, i - 2) = 0.0;
            if (i != mm + 2) a(i, i - 3) = 0.0;
        }
        for (int k = mm; k <= hi - 1; ++k) {
            if (k != mm) {
                p = a(k, k - 1);
                q = a(k + 1, k - 1);
                r = (k != hi - 1) ? a(k + 2, k - 1) : 0.0;
                x = std::abs(p) + std::abs(q) + std::abs(r);
                if (x != 0.0) {
                    p /= x;
                    q /= x;
                    r /= x;
                }
            }
            const double s = sgn(std::sqrt(p * p + q * q + r * r), p);
            if (s == 0.0) continue;
            if (k == mm) {
                if (l != mm) a(k, k - 1) = -a(k, k - 1);
            } else {
                a(k, k - 1) = -s * x;
            }
            p += s;
            x = p / s;
            y = q / s;
            z = r / s;
            q /= p;
            r /= p;
            for (int j = k; j <= hi; ++j) {  // row transformation
                double pp = a(k, j) + q * a(k + 1, j);
                if (k != hi - 1) {
                    pp += r * a(k + 2, j);
                    a(k + 2, j) -= pp * z;
                }
                a(k + 1, j) -= pp * y;
                a(k, j) -= pp * x;
            }
            const int imax = std::min(hi, k + 3);
            for (int i = l; i <= imax; ++i) {  // column transformation
                double pp = x * a(i, k) + y * a(i, k + 1);
                if (k != hi - 1) {
                    pp += z * a(i, k + 2);
                    a(i, k + 2) -= pp * r;
                }
                a(i, k + 1) -= pp * q;
                a(i, k) -= pp;
            }
        }
    }
}

}  // namespace

std::vector<double> eigenvalues_real_checked(const Dense& A, const Dense& Cm, double* radius, double* worst_imag) {
    const int n = A.r;
    // M = C^-1 A
    Dense lu = Cm;
    std::vector<int> perm;
    if (!dense_lu(lu, perm)) throw Error(SINGULAR, "spectral_bounds: infinite eigenvalue (singular C)");
    Dense M(n, n);
    for (int col = 0; col < n; ++col) {
        std::vector<double> x(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) x[size_t(i)] = A(perm[size_t(i)], col);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < i; ++j) x[size_t(i)] -= lu(i, j) * x[size_t(j)];
        for (int i = n - 1; i >= 0; --i) {
            for (int j = i + 1; j < n; ++j) x[size_t(i)] -= lu(i, j) * x[size_t(j)];
            x[size_t(i)] /= lu(i, i);
        }
        for (int i = 0; i < n; ++i) M(i, col) = x[size_t(i)];
    }
    balance(M);
    hessenberg(M);
    std::vector<double> wr, wi;
    hessenberg_qr(M, wr, wi);
    double rad = 0, wim = 0;
    for (int i = 0; i < n; ++i) {
        rad = std::max(rad, std::hypot(wr[size_t(i)], wi[size_t(i)]));
        wim = std::max(wim, std::abs(wi[size_t(i)]));
    }
    *radius = rad;
    *worst_imag = wim;
    return wr;
}

Range padded_range(const std::vector<Dense>& As, const std::vector<Dense>& Cs, bool q2_endpoint_pad) {
    double lo = std::numeric_limits<double>::infinity(), hi = -lo, radius = 0, worst_imag = 0;
    for (size_t b = 0; b < As.size(); ++b) {
        if (As[b].r == 0) continue;
        double rad, wim;
        auto ev = eigenvalues_real_checked(As[b], Cs[b], &rad, &wim);
        for (double e : ev) {
            lo = std::min(lo, e);
            hi = std::max(hi, e);
        }
        radius = std::max(radius, rad);
        worst_imag = std::max(worst_imag, wim);
    }
    if (worst_imag > 1e-6 * radius) throw Error(NUMERICAL, "spectral_bounds: spectrum of C^-1 A is not real");
    if (q2_endpoint_pad)  // SURVEY Q2 deviation: endpoint-relative pad (config 5 only)
        return {lo - 1e-8 * std::max(1.0, std::abs(lo)), hi + 1e-8 * std::max(1.0, std::abs(hi))};
    const double pad = 1e-8 * std::max(1.0, hi - lo) + 1e-12 * radius;  // adi.cpp:47
    return {lo - pad, hi + pad};
}

// ---------------------------------------------------------------- elliptic functions + shifts
double elliptic_K_kp(double kp) {
    if (!(kp > 0.0) || kp > 1.0) throw Error(DOMAIN_ERROR, "elliptic_K: complementary modulus must be in (0,1]");
    double a = 1.0, b = kp;
    for (int i = 0; i < 64 && std::abs(a - b) > 1e-16 * a; ++i) {
        const double an = 0.5 * (a + b);
        b = std::sqrt(a * b);
        a = an;
    }
    return std::numbers::pi / (2.0 * a);
}

double jacobi_dn_kp(double u, double kp) {
    // Descending Landen / AGM scheme (A&S 16.4) for dn(u | k), k = sqrt(1-kp^2).
    const double k2 = std::max(0.0, (1.0 - kp) * (1.0 + kp));
    double a[80], c[80];
    a[0] = 1.0;
    c[0] = std::sqrt(k2);
    double b = kp;
    int N = 0;
    while (std::abs(c[N]) > 1e-16 * a[N] && N < 64) {
        a[N + 1] = 0.5 * (a[N] + b);
        c[N + 1] = 0.5 * (a[N] - b);
        b = std::sqrt(a[N] * b);
        ++N;
    }
    if (N == 0) return 1.0;
    double phi = std::ldexp(a[N] * u, N), prev = phi;
    for (int i = N; i >= 1; --i) {
        prev = phi;
        const double s = std::clamp(c[i] / a[i] * std::sin(phi), -1.0, 1.0);
        phi = 0.5 * (phi + std::asin(s));
    }
    const double den = std::cos(prev - phi);
    const double sn = std::sin(phi);
    return std::abs(den) > 1e-12 ? std::cos(phi) / den : std::sqrt(1.0 - k2 * sn * sn);
}

Plan shift_plan(Range ca, Range db, double tol) {
    Plan p;
    p.a = ca.lo;
    p.b = ca.hi;
    p.c = db.lo;
    p.d = db.hi;
    p.tol = tol;
    if (!(p.b < p.c || p.d < p.a)) throw Error(DOMAIN_ERROR, "compute_shifts: spectral intervals overlap");
    if (!(tol > 0.0) || tol >= 1.0) throw Error(DOMAIN_ERROR, "compute_shifts: tol must be in (0,1)");
    p.gamma = std::abs(p.c - p.a) * std::abs(p.d - p.b) / (std::abs(p.c - p.b) * std::abs(p.d - p.a));
    const double g = p.gamma;
    p.alpha = -1.0 + 2.0 * g + 2.0 * std::sqrt(g * g - g);
    const double kp = 1.0 / p.alpha;
    p.modulus = std::sqrt(std::max(0.0, (1.0 - kp) * (1.0 + kp)));
    p.J = std::max(1, int(std::ceil(std::log(16.0 * g) * std::log(4.0 / tol) / (std::numbers::pi * std::numbers::pi))));
    const double K = elliptic_K_kp(kp);
    // Moebius map {-alpha,-1,1,alpha} -> {a,b,c,d} from the points 0,1,3 (special.cpp:112-127):
    // T = Mt^-1 o Ms, with M(z1,z2,z3): z -> (z-z1)(z2-z3)/((z-z3)(z2-z1)).
    auto mat = [](double z1, double z2, double z3) {
        return std::array<double, 4>{z2 - z3, -z1 * (z2 - z3), z2 - z1, -z3 * (z2 - z1)};
    };
    const auto s = mat(-p.alpha, -1.0, p.alpha);
    const auto t = mat(p.a, p.b, p.d);
    const std::array<double, 4> ti{t[3], -t[1], -t[2], t[0]};
    const std::array<double, 4> T{ti[0] * s[0] + ti[1] * s[2], ti[0] * s[1] + ti[1] * s[3], ti[2] * s[0] + ti[3] * s[2],
                                  ti[2] * s[1] + ti[3] * s[3]};
    auto apply = [&](double x) { return (T[0] * x + T[1]) / (T[2] * x + T[3]); };
    p.u.resize(size_t(p.J));
    p.v.resize(size_t(p.J));
    for (int j = 0; j < p.J; ++j) {
        const double dn = jacobi_dn_kp((2.0 * j + 1.0) / (2.0 * p.J) * K, kp);
        p.u[size_t(j)] = apply(-p.alpha * dn);
        p.v[size_t(j)] = apply(p.alpha * dn);
    }
    return p;
}

}  // namespace ccf
