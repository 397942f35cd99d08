// CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Grid, coefficient tensors, FFT stand-in for FFTW, CCF transforms, calculus.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <numbers>
#include <thread>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- threads
static int g_threads = 1;
void set_threads(int n) { g_threads = std::max(1, n); }
int threads() { return g_threads; }
void parallel_for(long n, const std::function<void(long)>& body) {
    const int t = int(std::min<long>(g_threads, n));
    if (t <= 1) {
        for (long i = 0; i < n; ++i) body(i);
        return;
    }
    std::atomic<long> next{0};
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex emu;
    for (int q = 0; q < t; ++q)
        pool.emplace_back([&] {
            for (;;) {
                const long i = next.fetch_add(1);
                if (i >= n) break;
                try {
                    body(i);
                } catch (...) {
                    std::lock_guard<std::mutex> g(emu);
                    if (!err) err = std::current_exception();
                }
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

// ---------------------------------------------------------------- grid (proj/src/grid.cpp)
void Spec::validate() const {  // grid.cpp:8-14
    if (m < 4 || n < 4) throw DomainError("GridSpec: m and n must be at least 4");
    if (p < 2 || p % 2 != 0) throw DomainError("GridSpec: p must be even and at least 2");
}

std::vector<double> chebyshev_points(int count) {  // grid.cpp:16-26
    if (count < 2) throw DomainError("chebyshev_points: need at least 2 points");
    std::vector<double> x(static_cast<size_t>(count));
    for (int j = 0; j < count; ++j) x[j] = std::cos(double(count - j - 1) * std::numbers::pi / double(count - 1));
    x.front() = -1.0;
    x.back() = 1.0;
    if (count % 2 == 1) x[size_t(count / 2)] = 0.0;
    return x;
}

std::vector<double> fourier_points(int count) {  // grid.cpp:28-34
    std::vector<double> t(static_cast<size_t>(count));
    for (int l = 0; l < count; ++l) t[l] = double(2 * l - count) * std::numbers::pi / double(count);
    return t;
}

double Field::max_abs() const {
    double r = 0;
    for (double x : v) r = std::max(r, std::abs(x));
    return r;
}

// ---------------------------------------------------------------- coeffs (proj/src/coeffs.cpp)
double Coeff::max_abs() const {
    double r = 0;
    for (const cd& c : d) r = std::max(r, std::abs(c));
    return r;
}
bool Coeff::all_finite() const {
    for (const cd& c : d)
        if (!std::isfinite(c.real()) || !std::isfinite(c.imag())) return false;
    return true;
}
Coeff& Coeff::operator+=(const Coeff& o) {
    if (!(s == o.s)) throw DomainError("CoeffTensor: spec mismatch");
    for (size_t i = 0; i < d.size(); ++i) d[i] += o.d[i];
    return *this;
}
Coeff& Coeff::operator-=(const Coeff& o) {
    if (!(s == o.s)) throw DomainError("CoeffTensor: spec mismatch");
    for (size_t i = 0; i < d.size(); ++i) d[i] -= o.d[i];
    return *this;
}
Coeff& Coeff::operator*=(cd a) {
    for (cd& c : d) c *= a;
    return *this;
}
Coeff operator+(Coeff a, const Coeff& b) { return a += b; }
Coeff operator-(Coeff a, const Coeff& b) { return a -= b; }

double hermitian_symmetry_error(const Coeff& t) {  // coeffs.cpp:36-48
    const int half = t.s.p / 2;
    double worst = 0;
    for (int l = 0; l < t.s.p; ++l) {
        const int lp = 2 * half - l;
        if (lp < 0 || lp >= t.s.p) continue;
        for (int k = 0; k < t.s.n; ++k)
            for (int j = 0; j < t.s.m; ++j) worst = std::max(worst, std::abs(t.at(j, k, l) - std::conj(t.at(j, k, lp))));
    }
    return worst;
}

void parity_project_in_place(Coeff& c, Parity parity) {  // coeffs.cpp:50-59
    const int keep = parity == Parity::scalar ? 0 : 1;
    for (int l = 0; l < c.s.p; ++l) {
        const int w = c.s.wavenumber(l);
        for (int k = 0; k < c.s.n; ++k)
            for (int j = 0; j < c.s.m; ++j)
                if ((((j + w) % 2) + 2) % 2 != keep) c.at(j, k, l) = cd(0);
    }
}
Coeff parity_project(const Coeff& c, Parity p) {
    Coeff o = c;
    parity_project_in_place(o, p);
    return o;
}

double MatC::norm() const {
    double s = 0;
    for (const cd& x : a) s += std::norm(x);
    return std::sqrt(s);
}
double MatC::max_abs() const {
    double s = 0;
    for (const cd& x : a) s = std::max(s, std::abs(x));
    return s;
}

// ---------------------------------------------------------------- FFT (stand-in for FFTW)
namespace {

struct FftPlan {
    int n = 0;
    bool pow2 = false;
    std::vector<int> rev;  // bit reversal (power-of-two sizes)
    std::vector<int> fac;
    std::vector<cd> tw;  // exp(-2 pi i k / n)
    bool blue = false;
    int nb = 0;
    std::vector<cd> chirp, bk;  // Bluestein
    std::unique_ptr<FftPlan> sub;
    explicit FftPlan(int n_);
    void exec(const cd* in, cd* out, int sign) const;
    void rec(cd* out, const cd* in, int len, int stride, int fi, int sign) const;
};

FftPlan::FftPlan(int n_) : n(n_) {
    pow2 = n >= 2 && (n & (n - 1)) == 0;
    if (pow2) {
        int lg = 0;
        while ((1 << lg) < n) ++lg;
        rev.resize(size_t(n));
        for (int i = 0; i < n; ++i) {
            int r2 = 0;
            for (int b = 0; b < lg; ++b)
                if (i & (1 << b)) r2 |= 1 << (lg - 1 - b);
            rev[size_t(i)] = r2;
        }
    }
    int r = n;
    for (int f : {4, 2, 3, 5}) {
        while (r % f == 0) {
            fac.push_back(f);
            r /= f;
        }
    }
    for (int f = 7; f * f <= r; f += 2)
        while (r % f == 0) {
            fac.push_back(f);
            r /= f;
        }
    if (r > 1) fac.push_back(r);
    const int big = *std::max_element(fac.begin(), fac.end());
    tw.resize(size_t(n));
    for (int k = 0; k < n; ++k) tw[k] = std::polar(1.0, -2.0 * std::numbers::pi * double(k) / double(n));
    if (big > 32) {
        // Bluestein for a large prime factor (generic radix is O(p^2))
        blue = true;
        nb = 1;
        while (nb < 2 * n - 1) nb *= 2;
        sub = std::make_unique<FftPlan>(nb);
        chirp.resize(size_t(n));
        for (long k = 0; k < n; ++k) {
            const long kk = (k * k) % (2L * n);
            chirp[k] = std::polar(1.0, -std::numbers::pi * double(kk) / double(n));
        }
        std::vector<cd> b(static_cast<size_t>(nb), cd(0));
        b[0] = std::conj(chirp[0]);
        for (int k = 1; k < n; ++k) b[k] = b[nb - k] = std::conj(chirp[k]);
        bk.resize(size_t(nb));
        sub->exec(b.data(), bk.data(), -1);
    }
}

void FftPlan::rec(cd* out, const cd* in, int len, int stride, int fi, int sign) const {
    const int p = fac[size_t(fi)];
    const int m = len / p;
    if (m == 1) {
        for (int q = 0; q < p; ++q) out[q] = in[size_t(q) * stride];
    } else {
        for (int q = 0; q < p; ++q) rec(out + size_t(q) * m, in + size_t(q) * stride, m, stride * p, fi + 1, sign);
    }
    // butterflies: twiddle step for this level
    const int tstep = n / len;  // W_len^x = tw[x * tstep]
    cd t[256];
    for (int k = 0; k < m; ++k) {
        for (int q = 0; q < p; ++q) {
            const cd w = tw[size_t((long(q) * k % len) * tstep)];
            t[q] = out[size_t(q) * m + k] * (sign < 0 ? w : std::conj(w));
        }
        for (int q2 = 0; q2 < p; ++q2) {
            cd acc = 0;
            for (int q = 0; q < p; ++q) {
                const cd w = tw[size_t((long(q) * q2 % p) * (n / p))];
                acc += t[q] * (sign < 0 ? w : std::conj(w));
            }
            out[size_t(q2) * m + k] = acc;
        }
    }
}

void FftPlan::exec(const cd* in, cd* out, int sign) const {
    if (pow2) {  // iterative radix-2 Cooley-Tukey
        for (int i = 0; i < n; ++i) out[rev[size_t(i)]] = in[i];
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1, step = n / len;
            for (int i = 0; i < n; i += len)
                for (int k = 0; k < half; ++k) {
                    const cd w = sign < 0 ? tw[size_t(k * step)] : std::conj(tw[size_t(k * step)]);
                    const cd a = out[i + k], b = out[i + k + half] * w;
                    out[i + k] = a + b;
                    out[i + k + half] = a - b;
                }
        }
        return;
    }
    if (!blue) {
        rec(out, in, n, 1, 0, sign);
        return;
    }
    if (sign > 0) {  // inverse via conjugation
        std::vector<cd> c(in, in + n);
        for (cd& x : c) x = std::conj(x);
        exec(c.data(), out, -1);
        for (int k = 0; k < n; ++k) out[k] = std::conj(out[k]);
        return;
    }
    thread_local std::vector<cd> a, fa;
    a.assign(size_t(nb), cd(0));
    fa.resize(size_t(nb));
    for (int k = 0; k < n; ++k) a[k] = in[k] * chirp[k];
    sub->exec(a.data(), fa.data(), -1);
    for (int k = 0; k < nb; ++k) fa[k] *= bk[k];
    sub->exec(fa.data(), a.data(), +1);
    for (int k = 0; k < n; ++k) out[k] = a[k] * (1.0 / nb) * chirp[k];
}

std::mutex g_plan_mu;
const FftPlan& plan_for(int n) {
    thread_local std::map<int, const FftPlan*> local;
    auto it = local.find(n);
    if (it != local.end()) return *it->second;
    static std::map<int, std::unique_ptr<FftPlan>> cache;
    std::lock_guard<std::mutex> g(g_plan_mu);
    auto& s = cache[n];
    if (!s) s = std::make_unique<FftPlan>(n);
    local[n] = s.get();
    return *s;
}

}  // namespace

void fft(int n, const cd* in, cd* out, int sign) { plan_for(n).exec(in, out, sign); }

void redft00(int L, const double* in, double* out) {
    // FFTW REDFT00 via the even extension of length 2(L-1).
    const int N = 2 * (L - 1);
    thread_local std::vector<cd> e, E;
    if (int(e.size()) < N) {
        e.resize(size_t(N));
        E.resize(size_t(N));
    }
    for (int j = 0; j < L; ++j) e[j] = in[j];
    for (int j = 1; j < L - 1; ++j) e[N - j] = in[j];
    fft(N, e.data(), E.data(), -1);
    for (int k = 0; k < L; ++k) out[k] = E[k].real();
}

// ---------------------------------------------------------------- transform (proj/src/transform.cpp)
namespace {

// In-place DCT-I sweep (transform.cpp:81-118). addr(q, t) gives the flat index.
template <class Addr>
void dct_sweep(std::vector<cd>& data, int len, long pencils, Addr addr, bool forward) {
    const double scale = 1.0 / double(len - 1);
    for (int part = 0; part < 2; ++part) {
        parallel_for(pencils, [&](long q) {
            std::vector<double> in(static_cast<size_t>(len)), out(static_cast<size_t>(len));
            bool nonzero = false;
            for (int t = 0; t < len; ++t) {
                const cd& c = data[addr(q, t)];
                const double v = part == 0 ? c.real() : c.imag();
                if (forward) in[len - 1 - t] = v;
                else in[t] = (t == 0 || t == len - 1) ? v : 0.5 * v;
                nonzero = nonzero || v != 0.0;
            }
            if (!nonzero) return;  // transform.cpp:101 skips all-zero pencils
            redft00(len, in.data(), out.data());
            for (int t = 0; t < len; ++t) {
                double v;
                if (forward) {
                    v = out[t] * scale;
                    if (t == 0 || t == len - 1) v *= 0.5;
                } else {
                    v = out[len - 1 - t];
                }
                cd& c = data[addr(q, t)];
                if (part == 0) c.real(v);
                else c.imag(v);
            }
        });
    }
}

}  // namespace

Coeff analyze(const Field& f) {  // transform.cpp:122-165
    const Spec& s = f.s;
    s.validate();
    for (double v : f.v)
        if (!std::isfinite(v)) throw NumericalError("analyze: non-finite input value");
    Coeff out(s);
    for (size_t i = 0; i < f.v.size(); ++i) out.d[i] = cd(f.v[i], 0.0);
    const int m = s.m, n = s.n, p = s.p;
    const long mn = long(m) * n;
    dct_sweep(out.d, m, long(n) * p, [&](long q, int t) { return size_t(q) * m + t; }, true);
    dct_sweep(out.d, n, long(m) * p, [&](long q, int t) {
        const long l = q / m, j = q % m;
        return (size_t(l) * n + t) * m + j;
    }, true);
    parallel_for(mn, [&](long q) {
        std::vector<cd> in(static_cast<size_t>(p)), X(static_cast<size_t>(p));
        for (int l = 0; l < p; ++l) in[l] = out.d[size_t(l) * mn + q];
        fft(p, in.data(), X.data(), -1);
        for (int l = 0; l < p; ++l) {
            const int w = l - p / 2;
            const int t = ((w % p) + p) % p;
            const double sign = (w % 2 == 0) ? 1.0 : -1.0;
            out.d[size_t(l) * mn + q] = X[t] * (sign / double(p));
        }
    });
    return out;
}

Field synthesize(const Coeff& c) {  // transform.cpp:167-203
    const Spec& s = c.s;
    s.validate();
    const int m = s.m, n = s.n, p = s.p;
    const long mn = long(m) * n;
    std::vector<cd> work(c.d.size());
    parallel_for(mn, [&](long q) {
        std::vector<cd> in(static_cast<size_t>(p)), X(static_cast<size_t>(p));
        for (int l = 0; l < p; ++l) {
            const int w = l - p / 2;
            const int t = ((w % p) + p) % p;
            const double sign = (w % 2 == 0) ? 1.0 : -1.0;
            in[t] = c.d[size_t(l) * mn + q] * sign;
        }
        fft(p, in.data(), X.data(), +1);
        for (int l = 0; l < p; ++l) work[size_t(l) * mn + q] = X[l];
    });
    dct_sweep(work, n, long(m) * p, [&](long q, int t) {
        const long l = q / m, j = q % m;
        return (size_t(l) * n + t) * m + j;
    }, false);
    dct_sweep(work, m, long(n) * p, [&](long q, int t) { return size_t(q) * m + t; }, false);
    Field out(s);
    for (size_t i = 0; i < work.size(); ++i) out.v[i] = work[i].real();  // transform.cpp:201 (Re only)
    return out;
}

cd evaluate_at(const Coeff& c, double r, double z, double th) {  // transform.cpp:205-233
    const int m = c.s.m, n = c.s.n, p = c.s.p;
    cd total(0);
    std::vector<cd> zs(static_cast<size_t>(n));
    for (int l = 0; l < p; ++l) {
        for (int k = 0; k < n; ++k) {
            cd b1(0), b2(0);
            for (int j = m - 1; j >= 1; --j) {
                const cd b = c.at(j, k, l) + 2.0 * r * b1 - b2;
                b2 = b1;
                b1 = b;
            }
            zs[k] = c.at(0, k, l) + r * b1 - b2;
        }
        cd b1(0), b2(0);
        for (int k = n - 1; k >= 1; --k) {
            const cd b = zs[k] + 2.0 * z * b1 - b2;
            b2 = b1;
            b1 = b;
        }
        const cd radial = zs[0] + z * b1 - b2;
        total += radial * std::polar(1.0, double(l - p / 2) * th);
    }
    return total;
}

// ---------------------------------------------------------------- calculus (proj/src/calculus.cpp)
namespace {
template <class Get, class Set>
void cheb_deriv(int len, Get get, Set set) {  // calculus.cpp:7-19
    cd next(0), next2(0);
    for (int k = len - 1; k >= 0; --k) {
        const cd ak1 = (k + 1 < len) ? get(k + 1) : cd(0);
        cd bk = next2 + 2.0 * double(k + 1) * ak1;
        if (k == 0) bk *= 0.5;
        next2 = next;
        next = bk;
        set(k, bk);
    }
}
}  // namespace

Coeff derivative_r(const Coeff& f) {  // calculus.cpp:23-32
    Coeff out(f.s);
    for (int l = 0; l < f.s.p; ++l)
        for (int k = 0; k < f.s.n; ++k)
            cheb_deriv(f.s.m, [&](int j) { return f.at(j, k, l); }, [&](int j, cd v) { out.at(j, k, l) = v; });
    return out;
}

Coeff derivative_z(const Coeff& f) {  // calculus.cpp:34-43
    Coeff out(f.s);
    for (int l = 0; l < f.s.p; ++l)
        for (int j = 0; j < f.s.m; ++j)
            cheb_deriv(f.s.n, [&](int k) { return f.at(j, k, l); }, [&](int k, cd v) { out.at(j, k, l) = v; });
    return out;
}

Coeff derivative_theta(const Coeff& f) {  // calculus.cpp:45-54
    Coeff out(f.s);
    const size_t mn = size_t(f.s.m) * f.s.n;
    for (int l = 0; l < f.s.p; ++l) {
        const cd factor = (l == 0) ? cd(0) : cd(0, double(f.s.wavenumber(l)));
        for (size_t i = 0; i < mn; ++i) out.d[size_t(l) * mn + i] = factor * f.d[size_t(l) * mn + i];
    }
    return out;
}

Coeff multiply_r(const Coeff& f) {  // calculus.cpp:56-69
    Coeff out(f.s);
    const int m = f.s.m;
    for (int l = 0; l < f.s.p; ++l)
        for (int k = 0; k < f.s.n; ++k) {
            out.at(1, k, l) += f.at(0, k, l);
            for (int j = 1; j < m; ++j) {
                const cd half = 0.5 * f.at(j, k, l);
                out.at(j - 1, k, l) += half;
                if (j + 1 < m) out.at(j + 1, k, l) += half;
            }
        }
    return out;
}

Coeff divide_r(const Coeff& f) {  // calculus.cpp:71-97 (quirk Q1: real-part synthesis)
    if (f.s.m % 2 != 0) throw DomainError("divide_r: even m required (odd m places a node at r = 0)");
    const auto r = chebyshev_points(f.s.m);
    Coeff fr(f.s), fi(f.s);
    for (size_t i = 0; i < f.d.size(); ++i) {
        fr.d[i] = cd(f.d[i].real(), 0.0);
        fi.d[i] = cd(f.d[i].imag(), 0.0);
    }
    Field re = synthesize(fr), im = synthesize(fi);
    for (int l = 0; l < f.s.p; ++l)
        for (int k = 0; k < f.s.n; ++k)
            for (int j = 0; j < f.s.m; ++j) {
                re.at(j, k, l) /= r[size_t(j)];
                im.at(j, k, l) /= r[size_t(j)];
            }
    Coeff cre = analyze(re), cim = analyze(im);
    Coeff out(f.s);
    for (size_t i = 0; i < out.d.size(); ++i) out.d[i] = cre.d[i] + cd(0, 1) * cim.d[i];
    return out;
}

Coeff horizontal_laplacian(const Coeff& f) {  // calculus.cpp:99-107
    Coeff dr = derivative_r(f);
    Coeff inner = derivative_theta(derivative_theta(f));
    inner = divide_r(inner);
    inner += dr;
    Coeff out = derivative_r(dr);
    out += divide_r(inner);
    return out;
}

Coeff laplacian(const Coeff& f) {  // calculus.cpp:109-113
    Coeff out = horizontal_laplacian(f);
    out += derivative_z(derivative_z(f));
    return out;
}

// ---------------------------------------------------------------- io (proj/src/io.cpp:12-25)
uint32_t crc32_ieee(const uint8_t* data, size_t len) {
    static const auto table = [] {
        std::array<uint32_t, 256> t{};
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int b = 0; b < 8; ++b) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[i] = c;
        }
        return t;
    }();
    uint32_t crc = 0xFFFFFFFFu;
    for (size_t i = 0; i < len; ++i) crc = table[(crc ^ data[i]) & 0xFFu] ^ (crc >> 8);
    return crc ^ 0xFFFFFFFFu;
}

}  // namespace oracle
