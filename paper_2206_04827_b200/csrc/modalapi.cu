// Per-mode solver API on the device: ModalSolver::solve on a raw C2 x C2 right-hand side (any parity content, the
// mass-only pair at scale 0) and ModalOperator::apply, the pieces of solve_modal_helmholtz and of the lifted
// boundary data (proj/include/cylspec/solvers.hpp:35-82, proj/src/solvers.cpp:46-140, proj/src/ultraop.cpp:83-123).
//
// One Fourier mode's system A X B + C X D = F splits into 2 (j parity) x 2 (k parity) x 2 (re / im) real
// sub-problems. Each is solved exactly by fast diagonalization in the four-product form of diag.hpp,
//     u = QL [ (PL f PR) .* RT ] QR,
// with the raw right-hand side: PL = (C V)^-1 [I | 0] and PR = [I ; 0] W (the zero column / row is the reference's
// truncation to the top-left (m-2) x (n-2) block, solvers.cpp:81), RT = 1 / (lambda_i + mu_j) for the Poisson
// quadruple and (-1/s) / (lambda_i + mu_j - 1/s) for the Helmholtz quadruple of scale s (same eigenvectors), and
// for s = 0 the mass pair X = R2'^-1 F C02'^-T (RT = 1). The products run as batched FP64 tensor-core GEMMs
// (GemmPlan); the host only marshals the column-major complex matrix into the parity blocks.
#include <cmath>
#include <mutex>
#include <set>
#include <vector>

#include "../../include/ccf.h"
#include "context.hpp"
#include "pipeline.hpp"

namespace ccf {

Dense modal_dense_transpose(const Dense& x) {
    Dense t(x.c, x.r);
    for (int i = 0; i < x.r; ++i)
        for (int j = 0; j < x.c; ++j) t(j, i) = x(i, j);
    return t;
}

struct ModalDev {
    int m = 0, n = 0, w = 0;
    double scale = 1.0;
    bool poisson = true;
    int M = 0, N = 0, mh = 0, nh = 0, Np = 0, Mp = 0;
    Dense A, B, C, D;  // ModalOperator (ultraop.cpp:89-123), host copies for raw()
    DBuf mats, work;
    double *dF = nullptr, *dT1 = nullptr, *dZ = nullptr, *dT3 = nullptr, *dU = nullptr;  // 8 sub-problems each
    double *dX = nullptr, *dTA = nullptr, *dTC = nullptr, *dY = nullptr;                  // apply: 2 planes each
    GemmPlan g1, g2, g3, g4, a1, a2;
    std::vector<double> hF, hU, hX, hY;

    ModalDev(Ctx& c, int w_, double scale_, bool poisson_) : m(c.m), n(c.n), w(w_), scale(scale_), poisson(poisson_) {
        if (m % 2 || n % 2 || m < 4 || n < 4) throw Error(DOMAIN_ERROR, "ModalSolver: even m, n >= 4 required on the B200 path");
        if (!poisson && !(scale >= 0.0)) throw Error(DOMAIN_ERROR, "ModalSolver: scale must be >= 0");
        SizeOps& so = *c.sizeops;
        M = (m - 2) / 2; N = (n - 2) / 2; mh = m / 2; nh = n / 2;
        Np = N + (N & 1); Mp = M + (M & 1);
        const int aw = std::abs(w);
        const Dense lw = radial_laplacian(so.ur, aw);
        // ModalOperator: Poisson A = L_w, C = R2; Helmholtz A = R2 - s L_w, C = -s R2; B = C02^T, D = D2^T
        A = Dense(m, m); C = Dense(m, m);
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                A(i, j) = poisson ? lw(i, j) : so.ur.r2(i, j) - scale * lw(i, j);
                C(i, j) = poisson ? so.ur.r2(i, j) : -scale * so.ur.r2(i, j);
            }
        B = modal_dense_transpose(so.uz.c02);
        D = modal_dense_transpose(so.uz.d2);
        const bool mass = !poisson && scale == 0.0;
        // per-parity diagonalization data
        DiagLeft left[2];
        DiagRight right[2];
        CBand idM, idN;
        idM.rows = M; idM.lo = idM.hi = 0; idM.v.assign(size_t(M), 1.0);
        idN.rows = N; idN.lo = idN.hi = 0; idN.v.assign(size_t(N), 1.0);
        const Dense lrec = recombine(lw);
        for (int j0 = 0; j0 < 2; ++j0) {
            const CBand Cp = compress(so.R2rec, j0, M, M, -2, 3);
            left[j0] = mass ? mass_left(Cp, idM, M, mh) : diag_left(compress(lrec, j0, M, M, -2, 3), Cp, idM, M, mh);
        }
        for (int k0 = 0; k0 < 2; ++k0) {
            const CBand Btc = compress(so.C02recZ, k0, N, N, -1, 2);
            right[k0] = mass ? mass_right(Btc, idN, N, nh)
                             : diag_right(Btc, compress(so.D2recZ, k0, N, N, -1, 2), idN, N, nh);
        }
        // pack: per j0 [PL M x mh | QL mh x Mp], per k0 [PR nh x Np | QR N x nh], RT[j0][k0] M x Np, then the
        // apply operands A^T, C^T (m x m), B^T, D^T (n x n)
        std::vector<double> G;
        auto put = [&](const std::vector<double>& x) {
            const size_t off = G.size();
            G.insert(G.end(), x.begin(), x.end());
            if (G.size() % 2) G.push_back(0.0);
            return off;
        };
        auto padld = [](const std::vector<double>& x, int rows, int cols) {
            const int ld = cols + (cols & 1);
            std::vector<double> o(size_t(rows) * ld, 0.0);
            for (int r = 0; r < rows; ++r)
                for (int q = 0; q < cols; ++q) o[size_t(r) * ld + q] = x[size_t(r) * cols + q];
            return o;
        };
        size_t oPL[2], oQL[2], oPR[2], oQR[2], oRT[2][2];
        for (int j0 = 0; j0 < 2; ++j0) {
            oPL[j0] = put(left[j0].PL);
            oQL[j0] = put(padld(left[j0].QL, mh, M));
        }
        for (int k0 = 0; k0 < 2; ++k0) {
            oPR[k0] = put(padld(right[k0].PR, nh, N));
            oQR[k0] = put(right[k0].QR);
        }
        const long double is = (poisson || mass) ? 0.0L : 1.0L / (long double)scale;
        for (int j0 = 0; j0 < 2; ++j0)
            for (int k0 = 0; k0 < 2; ++k0) {
                std::vector<double> rt(size_t(M) * Np, 0.0);
                for (int a = 0; a < M; ++a)
                    for (int b = 0; b < N; ++b) {
                        long double v = 1.0L;
                        if (!mass) {
                            const long double den = left[j0].lam_ld[size_t(a)] + right[k0].mu_ld[size_t(b)] - is;
                            v = (poisson ? 1.0L : -is) / den;
                        }
                        rt[size_t(a) * Np + b] = double(v);
                    }
                oRT[j0][k0] = put(rt);
            }
        const size_t oAt = put(modal_dense_transpose(A).a), oCt = put(modal_dense_transpose(C).a);
        const size_t oBt = put(so.uz.c02.a), oDt = put(so.uz.d2.a);
        mats.alloc(G.size());
        CCF_H2D(mats.p, G.data(), G.size() * sizeof(double));
        const size_t per = std::max(size_t(mh) * std::max(nh, Np), size_t(M) * std::max(nh, Np));
        const size_t perE = per + (per & 1);
        const size_t plane = size_t(m) * n;
        work.alloc(5 * 8 * perE + 4 * 2 * plane);
        CCF_CUDA(cudaMemset(work.p, 0, work.n * sizeof(double)));
        dF = work.p; dT1 = dF + 8 * perE; dZ = dT1 + 8 * perE; dT3 = dZ + 8 * perE; dU = dT3 + 8 * perE;
        dX = dU + 8 * perE; dTA = dX + 2 * plane; dTC = dTA + 2 * plane; dY = dTC + 2 * plane;
        hF.assign(8 * perE, 0.0); hU.assign(8 * perE, 0.0); hX.assign(2 * plane, 0.0); hY.assign(2 * plane, 0.0);
        const double* g = mats.p;
        int sub = 0;
        for (int j0 = 0; j0 < 2; ++j0)
            for (int k0 = 0; k0 < 2; ++k0)
                for (int pl = 0; pl < 2; ++pl, ++sub) {
                    double *F = dF + sub * perE, *T1 = dT1 + sub * perE, *Z = dZ + sub * perE, *T3 = dT3 + sub * perE,
                           *U = dU + sub * perE;
                    g1.A.push_back(g + oPL[j0]); g1.B.push_back(F); g1.C.push_back(T1);      // T1 = PL f      M x nh
                    g2.A.push_back(T1); g2.B.push_back(g + oPR[k0]); g2.C.push_back(Z);      // Z = T1 PR .* RT  M x N
                    g2.DL.push_back(g + oRT[j0][k0]); g2.DR.push_back(g + oRT[j0][k0]);
                    g3.A.push_back(g + oQL[j0]); g3.B.push_back(Z); g3.C.push_back(T3);      // T3 = QL Z      mh x N
                    g4.A.push_back(T3); g4.B.push_back(g + oQR[k0]); g4.C.push_back(U);      // u = T3 QR      mh x nh
                }
        g1.M = M; g1.N = nh; g1.K = mh; g1.lda = mh; g1.ldb = nh; g1.ldc = nh;
        g2.M = M; g2.N = N; g2.K = nh; g2.lda = nh; g2.ldb = Np; g2.ldc = Np; g2.ldd = Np;
        g3.M = mh; g3.N = N; g3.K = M; g3.lda = Mp; g3.ldb = Np; g3.ldc = Np;
        g4.M = mh; g4.N = nh; g4.K = N; g4.lda = Np; g4.ldb = nh; g4.ldc = nh;
        // apply, on X^T (n x m row-major = the column-major m x n matrix): Y^T = B^T (X^T A^T) + D^T (X^T C^T)
        for (int pl = 0; pl < 2; ++pl) {
            a1.A.push_back(dX + pl * plane); a1.B.push_back(g + oAt); a1.C.push_back(dTA + pl * plane);
            a1.A.push_back(dX + pl * plane); a1.B.push_back(g + oCt); a1.C.push_back(dTC + pl * plane);
            a2.A.push_back(g + oBt); a2.B.push_back(dTA + pl * plane);
            a2.A.push_back(g + oDt); a2.B.push_back(dTC + pl * plane);
            a2.C.push_back(dY + pl * plane);
        }
        a2.tstart = {0, 2, 4};
        a1.M = n; a1.N = m; a1.K = m; a1.lda = m; a1.ldb = m; a1.ldc = m;
        a2.M = n; a2.N = m; a2.K = n; a2.lda = n; a2.ldb = m; a2.ldc = m;
        for (GemmPlan* p : {&g1, &g2, &g3, &g4, &a1, &a2}) p->upload();
        perE_ = perE;
    }
    size_t perE_ = 0;

    // f, x: m x n complex, column-major (Eigen::MatrixXcd / a CoeffTensor slice), host memory
    void solve(Ctx& c, const double* f, double* x) {
        for (size_t i = 0; i < size_t(m) * n * 2; ++i)
            if (!std::isfinite(f[i])) throw Error(NUMERICAL, "ModalSolver::solve: non-finite right-hand side");
        int sub = 0;
        for (int j0 = 0; j0 < 2; ++j0)
            for (int k0 = 0; k0 < 2; ++k0)
                for (int pl = 0; pl < 2; ++pl, ++sub) {
                    double* F = hF.data() + sub * perE_;
                    for (int a = 0; a < mh; ++a)
                        for (int b = 0; b < nh; ++b)
                            F[size_t(a) * nh + b] = f[2 * (size_t(2 * a + j0) + size_t(m) * (2 * b + k0)) + pl];
                }
        CCF_CUDA(cudaMemcpyAsync(dF, hF.data(), hF.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        g1.launch(c.stream);
        g2.launch(c.stream);
        g3.launch(c.stream);
        g4.launch(c.stream);
        c.launches += 4;
        c.gemm_flops += g1.flops() + g2.flops() + g3.flops() + g4.flops();
        CCF_CUDA(cudaMemcpyAsync(hU.data(), dU, hU.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        sub = 0;
        for (int j0 = 0; j0 < 2; ++j0)
            for (int k0 = 0; k0 < 2; ++k0)
                for (int pl = 0; pl < 2; ++pl, ++sub) {
                    const double* U = hU.data() + sub * perE_;
                    for (int a = 0; a < mh; ++a)
                        for (int b = 0; b < nh; ++b)
                            x[2 * (size_t(2 * a + j0) + size_t(m) * (2 * b + k0)) + pl] = U[size_t(a) * nh + b];
                }
    }

    // ModalOperator::apply (ultraop.cpp:83-87): y = A x B + C x D
    void apply(Ctx& c, const double* x, double* y) {
        const size_t plane = size_t(m) * n;
        for (size_t i = 0; i < plane; ++i) {
            hX[i] = x[2 * i];
            hX[plane + i] = x[2 * i + 1];
        }
        CCF_CUDA(cudaMemcpyAsync(dX, hX.data(), hX.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        a1.launch(c.stream);
        a2.launch(c.stream);
        c.launches += 2;
        CCF_CUDA(cudaMemcpyAsync(hY.data(), dY, hY.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (size_t i = 0; i < plane; ++i) {
            y[2 * i] = hY[i];
            y[2 * i + 1] = hY[plane + i];
        }
    }
};

}  // namespace ccf

struct ccf_modal {
    ccf_ctx* ctx = nullptr;
    std::unique_ptr<ccf::ModalDev> d;
};

// live handles per context: ccf_ctx_destroy releases their device data and detaches them (api.cu), so a handle
// outliving its context only reports CCF_INTERNAL_ERROR and can still be destroyed
namespace {
std::mutex g_modal_mu;
std::set<ccf_modal*> g_modals;
}  // namespace
void ccf_modal_detach_ctx(ccf_ctx* ctx) {
    std::lock_guard<std::mutex> lock(g_modal_mu);
    for (ccf_modal* h : g_modals)
        if (h->ctx == ctx) {
            h->d.reset();
            h->ctx = nullptr;
        }
}

// (api.cu)
ccf_status ccf_ctx_guard(ccf_ctx* ctx, void (*fn)(ccf::Ctx&, void*), void* user);

namespace {
template <class F>
ccf_status mguard(ccf_ctx* ctx, F&& f) {
    return ccf_ctx_guard(ctx, [](ccf::Ctx& c, void* u) { (*static_cast<F*>(u))(c); }, &f);
}
}  // namespace

extern "C" {

ccf_status ccf_modal_create(ccf_ctx* ctx, int w, double scale, int poisson, ccf_modal** out) {
    if (!out) return CCF_INTERNAL_ERROR;
    *out = nullptr;
    return mguard(ctx, [&](ccf::Ctx& c) {
        auto h = std::make_unique<ccf_modal>();
        h->ctx = ctx;
        h->d = std::make_unique<ccf::ModalDev>(c, w, scale, poisson != 0);
        std::lock_guard<std::mutex> lock(g_modal_mu);
        g_modals.insert(h.get());
        *out = h.release();
    });
}

ccf_status ccf_modal_solve(ccf_modal* h, const double* f_full, double* x) {
    if (!h || !h->ctx || !f_full || !x) return CCF_INTERNAL_ERROR;
    return mguard(h->ctx, [&](ccf::Ctx& c) { h->d->solve(c, f_full, x); });
}

ccf_status ccf_modal_apply(ccf_modal* h, const double* x, double* y) {
    if (!h || !h->ctx || !x || !y) return CCF_INTERNAL_ERROR;
    return mguard(h->ctx, [&](ccf::Ctx& c) { h->d->apply(c, x, y); });
}

ccf_status ccf_modal_operator(ccf_modal* h, int which, double* dense) {
    if (!h || !h->d || !dense || which < 0 || which > 3) return CCF_INTERNAL_ERROR;
    const ccf::Dense* ops[4] = {&h->d->A, &h->d->B, &h->d->C, &h->d->D};
    std::copy(ops[which]->a.begin(), ops[which]->a.end(), dense);
    return CCF_OK;
}

ccf_status ccf_modal_destroy(ccf_modal* h) {
    if (!h) return CCF_OK;
    {
        std::lock_guard<std::mutex> lock(g_modal_mu);
        g_modals.erase(h);
    }
    ccf_status st = CCF_OK;
    if (h->ctx) st = mguard(h->ctx, [&](ccf::Ctx&) { h->d.reset(); });
    delete h;
    return st;
}

}  // extern "C"
