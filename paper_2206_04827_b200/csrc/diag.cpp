// Fast-diagonalization setup (see diag.hpp). Long double throughout; outputs rounded once.
#include "diag.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

namespace ccf {

namespace {

using R = long double;

struct LMat {
    int r = 0, c = 0;
    std::vector<R> a;
    LMat() = default;
    LMat(int r_, int c_) : r(r_), c(c_), a(size_t(r_) * c_, 0.0L) {}
    R& operator()(int i, int j) { return a[size_t(i) * c + j]; }
    R operator()(int i, int j) const { return a[size_t(i) * c + j]; }
};

// Dense storage, banded partial-pivot LU (lower bandwidth kl, upper ku before pivoting).
struct BandLU {
    int n = 0, kl = 0, ku = 0;
    LMat m;
    std::vector<int> piv;
    bool factor() {
        piv.assign(size_t(n), 0);
        const int w = kl + ku;
        for (int k = 0; k < n; ++k) {
            int p = k;
            R best = std::fabs(m(k, k));
            for (int i = k + 1; i <= std::min(n - 1, k + kl); ++i)
                if (std::fabs(m(i, k)) > best) {
                    best = std::fabs(m(i, k));
                    p = i;
                }
            if (best == 0.0L) return false;
            piv[size_t(k)] = p;
            const int jend = std::min(n - 1, k + w);
            if (p != k)
                for (int j = k; j <= jend; ++j) std::swap(m(k, j), m(p, j));
            for (int i = k + 1; i <= std::min(n - 1, k + kl); ++i) {
                const R f = m(i, k) / m(k, k);
                m(i, k) = f;
                if (f != 0.0L)
                    for (int j = k + 1; j <= jend; ++j) m(i, j) -= f * m(k, j);
            }
        }
        return true;
    }
    void solve(std::vector<R>& b) const {
        for (int k = 0; k < n; ++k) {
            const int p = piv[size_t(k)];
            if (p != k) std::swap(b[size_t(k)], b[size_t(p)]);
            for (int i = k + 1; i <= std::min(n - 1, k + kl); ++i) b[size_t(i)] -= m(i, k) * b[size_t(k)];
        }
        const int w = kl + ku;
        for (int k = n - 1; k >= 0; --k) {
            R acc = b[size_t(k)];
            for (int j = k + 1; j <= std::min(n - 1, k + w); ++j) acc -= m(k, j) * b[size_t(j)];
            b[size_t(k)] = acc / m(k, k);
        }
    }
};

// Dense partial-pivot LU solve of S X = Bm (long double), Bm overwritten with X.
bool dense_solve(LMat S, LMat& Bm) {
    const int n = S.r;
    for (int k = 0; k < n; ++k) {
        int p = k;
        for (int i = k + 1; i < n; ++i)
            if (std::fabs(S(i, k)) > std::fabs(S(p, k))) p = i;
        if (S(p, k) == 0.0L) return false;
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(S(k, j), S(p, j));
            for (int j = 0; j < Bm.c; ++j) std::swap(Bm(k, j), Bm(p, j));
        }
        for (int i = k + 1; i < n; ++i) {
            const R f = S(i, k) / S(k, k);
            if (f == 0.0L) continue;
            for (int j = k + 1; j < n; ++j) S(i, j) -= f * S(k, j);
            for (int j = 0; j < Bm.c; ++j) Bm(i, j) -= f * Bm(k, j);
        }
    }
    for (int k = n - 1; k >= 0; --k)
        for (int j = 0; j < Bm.c; ++j) {
            R acc = Bm(k, j);
            for (int i = k + 1; i < n; ++i) acc -= S(k, i) * Bm(i, j);
            Bm(k, j) = acc / S(k, k);
        }
    return true;
}

struct BandOp {  // square banded operator as dense long double with its band
    LMat m;
    int kl = 0, ku = 0;
};

// Refined eigenpairs of A v = lambda C v (real, simple spectrum): Hessenberg-QR estimates in
// double, then inverse iteration in long double (banded LU of A - sigma C, 3 + 1 iterations).
void eig_refined(const BandOp& A, const BandOp& Cm, std::vector<R>& lam, LMat& V) {
    const int n = A.m.r;
    Dense Ad(n, n), Cd(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            Ad(i, j) = double(A.m(i, j));
            Cd(i, j) = double(Cm.m(i, j));
        }
    double rad = 0.0, wim = 0.0;
    const std::vector<double> est = eigenvalues_real_checked(Ad, Cd, &rad, &wim);
    if (wim > 1e-6 * rad) throw Error(NUMERICAL, "diag: generalized spectrum is not real");
    const int kl = std::max(A.kl, Cm.kl), ku = std::max(A.ku, Cm.ku);
    lam.assign(size_t(n), 0.0L);
    V = LMat(n, n);
    std::vector<R> v(static_cast<size_t>(n)), y(static_cast<size_t>(n)), av(static_cast<size_t>(n)), cv(static_cast<size_t>(n));
    auto apply = [&](const LMat& Mx, const std::vector<R>& x, std::vector<R>& out) {
        for (int i = 0; i < n; ++i) {
            R acc = 0.0L;
            for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j) acc += Mx(i, j) * x[size_t(j)];
            out[size_t(i)] = acc;
        }
    };
    auto quotient = [&]() {
        apply(A.m, v, av);
        apply(Cm.m, v, cv);
        R num = 0.0L, den = 0.0L;
        for (int i = 0; i < n; ++i) {
            num += cv[size_t(i)] * av[size_t(i)];
            den += cv[size_t(i)] * cv[size_t(i)];
        }
        return num / den;
    };
    for (int e = 0; e < n; ++e) {
        R sigma = R(est[size_t(e)]);
        uint64_t st = 0x9E3779B97F4A7C15ull * uint64_t(e + 1);
        for (int i = 0; i < n; ++i) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            v[size_t(i)] = R(double(st >> 11) / 9007199254740992.0) - 0.5L;
        }
        for (int pass = 0; pass < 2; ++pass) {
            BandLU lu;
            lu.n = n;
            lu.kl = kl;
            lu.ku = ku;
            lu.m = LMat(n, n);
            for (int i = 0; i < n; ++i)
                for (int j = std::max(0, i - kl); j <= std::min(n - 1, i + ku); ++j)
                    lu.m(i, j) = A.m(i, j) - sigma * Cm.m(i, j);
            if (!lu.factor()) {  // exact shift: perturb
                sigma *= (1.0L + 1e-15L);
                --pass;
                continue;
            }
            for (int it = 0; it < (pass == 0 ? 3 : 1); ++it) {
                apply(Cm.m, v, y);
                lu.solve(y);
                R nrm = 0.0L;
                for (R x : y) nrm += x * x;
                nrm = std::sqrt(nrm);
                for (int i = 0; i < n; ++i) v[size_t(i)] = y[size_t(i)] / nrm;
            }
            sigma = quotient();
        }
        lam[size_t(e)] = sigma;
        for (int i = 0; i < n; ++i) V(i, e) = v[size_t(i)];
    }
    // distinctness guard: two estimates converging to one eigenpair would make V singular
    std::vector<R> sorted(lam);
    std::sort(sorted.begin(), sorted.end());
    for (int i = 1; i < n; ++i)
        if (std::fabs(sorted[size_t(i)] - sorted[size_t(i) - 1]) <= 1e-13L * std::fabs(sorted[size_t(i)]))
            throw Error(NUMERICAL, "diag: repeated generalized eigenvalue");
}

BandOp from_band(const CBand& b, int n) {  // row a: entries at a + d, d in [lo, hi]
    BandOp o;
    o.m = LMat(n, n);
    o.kl = -b.lo;
    o.ku = b.hi;
    for (int a = 0; a < n; ++a)
        for (int d = b.lo; d <= b.hi; ++d)
            if (a + d >= 0 && a + d < n) o.m(a, a + d) = R(b.at(a, d));
    return o;
}

BandOp from_band_transposed(const CBand& b, int n) {  // (b as above)^T
    BandOp o;
    o.m = LMat(n, n);
    o.kl = b.hi;
    o.ku = -b.lo;
    for (int a = 0; a < n; ++a)
        for (int d = b.lo; d <= b.hi; ++d)
            if (a + d >= 0 && a + d < n) o.m(a + d, a) = R(b.at(a, d));
    return o;
}

std::vector<double> to_double(const LMat& x) {
    std::vector<double> o(x.a.size());
    for (size_t i = 0; i < o.size(); ++i) o[i] = double(x.a[i]);
    return o;
}

}  // namespace

DiagLeft diag_left(const CBand& Ab, const CBand& Cb, const CBand& R2b, int M, int mh) {
    const BandOp A = from_band(Ab, M), Cm = from_band(Cb, M);
    std::vector<R> lam;
    LMat V;
    eig_refined(A, Cm, lam, V);
    for (int e = 0; e < M; ++e) {  // unit columns
        R nrm = 0.0L;
        for (int i = 0; i < M; ++i) nrm += V(i, e) * V(i, e);
        nrm = std::sqrt(nrm);
        for (int i = 0; i < M; ++i) V(i, e) /= nrm;
    }
    LMat CV(M, M);
    for (int i = 0; i < M; ++i)
        for (int e = 0; e < M; ++e) {
            R acc = 0.0L;
            for (int j = std::max(0, i - Cm.kl); j <= std::min(M - 1, i + Cm.ku); ++j) acc += Cm.m(i, j) * V(j, e);
            CV(i, e) = acc;
        }
    LMat PL(M, mh);  // R2m[a][y] = R2(a, y - a)
    for (int a = 0; a < M; ++a)
        for (int d = R2b.lo; d <= R2b.hi; ++d)
            if (a + d >= 0 && a + d < mh) PL(a, a + d) = R(R2b.at(a, d));
    if (!dense_solve(CV, PL)) throw Error(SINGULAR, "diag: C V is singular");
    LMat QL(mh, M);  // S_r V
    for (int a = 0; a < mh; ++a)
        for (int e = 0; e < M; ++e) QL(a, e) = (a < M ? V(a, e) : 0.0L) - (a > 0 ? V(a - 1, e) : 0.0L);
    DiagLeft out;
    out.PL = to_double(PL);
    out.PL_ld = PL.a;
    out.QL = to_double(QL);
    out.lam.resize(size_t(M));
    for (int i = 0; i < M; ++i) out.lam[size_t(i)] = double(lam[size_t(i)]);
    out.lam_ld = lam;
    return out;
}

DiagRight diag_right(const CBand& Btb, const CBand& Dtb, const CBand& C02b, int N, int nh) {
    const BandOp B = from_band_transposed(Btb, N), D = from_band_transposed(Dtb, N);
    std::vector<R> mu;
    LMat W;
    eig_refined(D, B, mu, W);
    LMat BW(N, N);
    for (int i = 0; i < N; ++i)
        for (int e = 0; e < N; ++e) {
            R acc = 0.0L;
            for (int j = std::max(0, i - B.kl); j <= std::min(N - 1, i + B.ku); ++j) acc += B.m(i, j) * W(j, e);
            BW(i, e) = acc;
        }
    for (int e = 0; e < N; ++e) {  // columns with |B^ w| = 1
        R nrm = 0.0L;
        for (int i = 0; i < N; ++i) nrm += BW(i, e) * BW(i, e);
        nrm = std::sqrt(nrm);
        for (int i = 0; i < N; ++i) {
            BW(i, e) /= nrm;
            W(i, e) /= nrm;
        }
    }
    LMat PR(nh, N);  // C02m W, C02m[x][b] = C02(b, x - b)
    for (int b = 0; b < N; ++b)
        for (int d = C02b.lo; d <= C02b.hi; ++d) {
            const int x = b + d;
            if (x < 0 || x >= nh) continue;
            const R c = R(C02b.at(b, d));
            if (c == 0.0L) continue;
            for (int e = 0; e < N; ++e) PR(x, e) += c * W(b, e);
        }
    LMat inv(N, N);
    for (int i = 0; i < N; ++i) inv(i, i) = 1.0L;
    if (!dense_solve(BW, inv)) throw Error(SINGULAR, "diag: B W is singular");
    LMat QR(N, nh);  // (B^ W)^-1 S_z^T
    for (int i = 0; i < N; ++i)
        for (int b = 0; b < nh; ++b) QR(i, b) = (b < N ? inv(i, b) : 0.0L) - (b > 0 ? inv(i, b - 1) : 0.0L);
    DiagRight out;
    out.PR = to_double(PR);
    out.QR = to_double(QR);
    out.mu.resize(size_t(N));
    for (int i = 0; i < N; ++i) out.mu[size_t(i)] = double(mu[size_t(i)]);
    out.mu_ld = mu;
    return out;
}

DiagLeft mass_left(const CBand& Ab, const CBand& R2b, int M, int mh) {
    const BandOp A = from_band(Ab, M);
    LMat PL(M, mh);  // R2m[a][y] = R2(a, y - a) (identity band: the raw right-hand side, truncated)
    for (int a = 0; a < M; ++a)
        for (int d = R2b.lo; d <= R2b.hi; ++d)
            if (a + d >= 0 && a + d < mh) PL(a, a + d) = R(R2b.at(a, d));
    if (!dense_solve(A.m, PL)) throw Error(SINGULAR, "mass solve: R2 block is singular");
    LMat QL(mh, M);  // S_r
    for (int a = 0; a < mh; ++a)
        for (int e = 0; e < M; ++e) QL(a, e) = (a == e ? 1.0L : 0.0L) - (a == e + 1 ? 1.0L : 0.0L);
    DiagLeft out;
    out.PL = to_double(PL);
    out.PL_ld = PL.a;
    out.QL = to_double(QL);
    out.lam.assign(size_t(M), 1.0);  // with mu = 0: 1 / (lambda_i + mu_j) = 1
    out.lam_ld.assign(size_t(M), 1.0L);
    return out;
}

DiagRight mass_right(const CBand& Btb, const CBand& C02b, int N, int nh) {
    // Y B^ = E  <=>  B^^T Y^T = E^T: invert Bt = B^^T and transpose
    const BandOp Bt = from_band(Btb, N);
    LMat inv(N, N);
    for (int i = 0; i < N; ++i) inv(i, i) = 1.0L;
    if (!dense_solve(Bt.m, inv)) throw Error(SINGULAR, "mass solve: C02 block is singular");
    LMat PR(nh, N);  // C02m B^^-1, C02m[x][b] = C02(b, x - b), B^^-1 = (Bt^-1)^T
    for (int b = 0; b < N; ++b)
        for (int d = C02b.lo; d <= C02b.hi; ++d) {
            const int x = b + d;
            if (x < 0 || x >= nh) continue;
            const R c = R(C02b.at(b, d));
            if (c == 0.0L) continue;
            for (int e = 0; e < N; ++e) PR(x, e) += c * inv(e, b);
        }
    LMat QR(N, nh);  // S_z^T
    for (int i = 0; i < N; ++i)
        for (int b = 0; b < nh; ++b) QR(i, b) = (b == i ? 1.0L : 0.0L) - (b == i + 1 ? 1.0L : 0.0L);
    DiagRight out;
    out.PR = to_double(PR);
    out.QR = to_double(QR);
    out.mu.assign(size_t(N), 0.0);
    out.mu_ld.assign(size_t(N), 0.0L);
    return out;
}

}  // namespace ccf
