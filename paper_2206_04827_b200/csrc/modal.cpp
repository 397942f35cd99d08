// Host builder for packed ADI operator blocks (see modal.hpp).
#include "modal.hpp"

#include "diag.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>

namespace ccf {

namespace {

Dense parity_block(const Dense& M, int p) {
    const int n = (M.r - p + 1) / 2;
    Dense b(n, n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) b(i, j) = M(2 * i + p, 2 * j + p);
    return b;
}

Dense scaled(const Dense& a, double s) {
    Dense o = a;
    for (double& x : o.a) x *= s;
    return o;
}

Dense axpby(double al, const Dense& a, double be, const Dense& b) {
    Dense o = a;
    for (size_t i = 0; i < o.a.size(); ++i) o.a[i] = al * a.a[i] + be * b.a[i];
    return o;
}

// right-side LU fields: [L | piv | inv | 0 | Uf0 Uf1 Uf2 | 0]
void put_right_lu(double* r, const CLU& lu, int b) {
    r[0] = lu.L[size_t(b)];
    r[1] = double(lu.piv[size_t(b)]);
    r[2] = lu.inv[size_t(b)];
    r[3] = 0.0;
    for (int q = 0; q < 3; ++q) r[4 + q] = lu.U[size_t(b) * 3 + q] * lu.inv[size_t(b)];
    r[7] = 0.0;
}

// sum of two compressed bands with identical shape
CBand cb_axpy(double al, const CBand& x, double be, const CBand& y) {
    CBand o = x;
    for (size_t i = 0; i < o.v.size(); ++i) o.v[i] = al * x.v[i] + be * y.v[i];
    return o;
}

// Spike vectors of the two-way partitioned sweeps (adi.cu, col/row_phase_spike).
// Left (column) sweep, rows k of one shift block, split row h:
//   forward  x_{k+1} -= L0[k] x_k, x_{k+2} -= L1[k] x_k: the lower part runs without the
//            contributions of x_{h-1}, x_{h-2}; true x_k = x'_k + F1[k] x_{h-1} + F2[k] x_{h-2}
//   backward z_k = inv x_k - Uf0 z_{k+1} - Uf1 z_{k+2} - Uf2 z_{k+3}: the upper part runs with
//            z_h = z_{h+1} = z_{h+2} = 0; true z_k = z'_k + G1[k] z_h + G2[k] z_{h+1} + G3[k] z_{h+2}
void add_left_spikes(double* blk, int M, int h) {
    auto f = [&](int k, int q) -> double { return blk[size_t(k) * kLeftW + q]; };
    std::vector<long double> d(size_t(M) + 3);
    for (int which = 0; which < 2; ++which) {
        std::fill(d.begin(), d.end(), 0.0L);
        if (which == 0) {
            d[size_t(h)] = -(long double)f(h - 1, 6);
            d[size_t(h) + 1] = -(long double)f(h - 1, 7);
        } else {
            d[size_t(h)] = -(long double)f(h - 2, 7);
        }
        for (int k = h; k < M; ++k) {
            d[size_t(k) + 1] -= (long double)f(k, 6) * d[size_t(k)];
            d[size_t(k) + 2] -= (long double)f(k, 7) * d[size_t(k)];
        }
        for (int k = h; k < M; ++k) blk[size_t(k) * kLeftW + 13 + which] = double(d[size_t(k)]);
    }
    for (int which = 0; which < 3; ++which) {
        std::fill(d.begin(), d.end(), 0.0L);
        d[size_t(h + which)] = 1.0L;
        for (int k = h - 1; k >= 0; --k)
            d[size_t(k)] = -(long double)f(k, 10) * d[size_t(k) + 1] - (long double)f(k, 11) * d[size_t(k) + 2] -
                           (long double)f(k, 12) * d[size_t(k) + 3];
        for (int k = 0; k < h; ++k) blk[size_t(k) * kLeftW + 13 + which] = double(d[size_t(k)]);
    }
}

// Right (row) sweep with the fused multiply g = z (v'B + D) (row k: mul fields 0..3, d = -1..2):
//   forward  x_{k+1} -= L[k] x_k -> lower half: true x_k = x'_k + F[k] x_{h-1}        (k >= h)
//   backward z_k = inv x_k - Uf0 z_{k+1} - Uf1 z_{k+2}: the upper half runs with z_h = z_{h+1} = 0,
//            true z_k = z'_k + G1[k] z_h + G2[k] z_{h+1}; its fused multiply g'_k (k <= h) then
//            differs from g_k by the rank-3 term H1[k] z_h + H2[k] z_{h+1} + H3[k] z_{h+2}.
// Fields (unpivoted rows only): [5] F (k >= h), [7] H3 (k = h), [10] H1, [11] H2 (k <= h).
void add_right_spikes(double* blk, int N, int h) {
    auto f = [&](int k, int q) -> double { return blk[size_t(k) * kRightW + q]; };
    std::vector<long double> d(size_t(N) + 3);
    std::fill(d.begin(), d.end(), 0.0L);
    d[size_t(h)] = -(long double)f(h - 1, 4);
    for (int k = h; k < N; ++k) d[size_t(k) + 1] -= (long double)f(k, 4) * d[size_t(k)];
    for (int k = h; k < N; ++k) blk[size_t(k) * kRightW + 5] = double(d[size_t(k)]);
    for (int which = 0; which < 2; ++which) {
        std::fill(d.begin(), d.end(), 0.0L);  // extended response: G[j] (j < h), unit at h + which
        d[size_t(h + which)] = 1.0L;
        for (int k = h - 1; k >= 0; --k)
            d[size_t(k)] = -(long double)f(k, 8) * d[size_t(k) + 1] - (long double)f(k, 9) * d[size_t(k) + 2];
        for (int k = 0; k <= h && k < N; ++k) {
            long double acc = 0.0L;
            for (int dd = -1; dd <= 2; ++dd) {
                const int j = k + dd;
                if (j >= 0) acc += (long double)f(k, dd + 1) * d[size_t(j)];
            }
            blk[size_t(k) * kRightW + 10 + which] = double(acc);
        }
    }
    if (h < N) blk[size_t(h) * kRightW + 7] = f(h, 3);  // H3: m_2[h] z_{h+2}
}

}  // namespace

SizeOps::SizeOps(int m_, int n_) : m(m_), n(n_), ur(m_), uz(n_) {
    R2rec = recombine(ur.r2);
    C02recZ = recombine(uz.c02);
    D2recZ = recombine(uz.d2);
}

Range radial_range(const SizeOps& so, int w, bool q2_pad) {
    const Dense lw = recombine(radial_laplacian(so.ur, w));
    std::vector<Dense> As{parity_block(lw, 0), parity_block(lw, 1)};
    std::vector<Dense> Cs{parity_block(so.R2rec, 0), parity_block(so.R2rec, 1)};
    return padded_range(As, Cs, q2_pad);
}

Range vertical_range(SizeOps& so, bool q2_pad) {
    const Dense negd2 = scaled(so.D2recZ, -1.0);
    std::vector<Dense> As{parity_block(negd2, 0), parity_block(negd2, 1)};
    std::vector<Dense> Cs{parity_block(so.C02recZ, 0), parity_block(so.C02recZ, 1)};
    return padded_range(As, Cs, q2_pad);
}

SolverSet build_solver_set(SizeOps& so, const std::vector<int>& slot_w, bool poisson, double scale, double tol,
                           std::map<int, Range>& radial_cache, bool q2_pad, double plan_margin, bool with_diag,
                           bool with_adi, bool keep_static) {
    if (!with_diag && !with_adi) throw Error(INTERNAL, "build_solver_set: nothing to build");
    const int m = so.m, n = so.n, M = (m - 2) / 2, N = (n - 2) / 2, mh = m / 2, nh = n / 2;
    const int lrows = ((M + 7) / 8) * 8 + 2, rrows = ((N + 7) / 8) * 8 + 2;  // zero-padded sweep rows
    SolverSet set;
    set.poisson = poisson;
    set.scale = scale;
    set.tol = tol;
    const int S = int(slot_w.size());
    set.plans.resize(size_t(S));
    set.slots.resize(size_t(S));

    // unique |w| -> radial ranges (parallel over wavenumbers: O(m^3) QR each)
    std::vector<int> need;
    for (int w : slot_w)
        if (with_adi && !radial_cache.count(std::abs(w))) need.push_back(std::abs(w));
    std::sort(need.begin(), need.end());
    need.erase(std::unique(need.begin(), need.end()), need.end());
    if (!need.empty()) {
        std::vector<Range> res(need.size());
        std::vector<std::string> errs(need.size());
        std::vector<int> codes(need.size(), 0);
        const int nth = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), int(need.size())));
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        for (int q = 0; q < nth; ++q)
            pool.emplace_back([&] {
                for (;;) {
                    const size_t i = next.fetch_add(1);
                    if (i >= need.size()) break;
                    try {
                        res[i] = radial_range(so, need[i], false);
                    } catch (const Error& e) {
                        codes[i] = e.status;
                        errs[i] = e.what();
                    }
                }
            });
        for (auto& th : pool) th.join();
        for (size_t i = 0; i < need.size(); ++i) {
            if (codes[i]) throw Error(codes[i], errs[i]);
            radial_cache[need[i]] = res[i];
        }
    }
    const Range vert = with_adi ? vertical_range(so, false) : Range{};

    // per |w| block cache
    std::map<int, AdiSlot> built;
    struct DiagIn {
        int aw;
        CBand A, C, R2;
    };
    std::vector<DiagIn> diag_in;
    std::vector<double>& C = set.coef;
    auto alloc = [&](size_t count) {
        const long off = long(C.size());
        C.resize(C.size() + ((count + 1) / 2) * 2, 0.0);  // 16-byte aligned blocks (bulk copies)
        return off;
    };

    // right-side operators (independent of w)
    const Dense Bt = so.C02recZ, Dt = so.D2recZ;
    CBand Btc[2], Dtc[2], C02c[2];
    for (int k0 = 0; k0 < 2; ++k0) {
        Btc[k0] = compress(Bt, k0, N, N, -1, 2);
        Dtc[k0] = compress(Dt, k0, N, N, -1, 2);
        C02c[k0] = compress(so.uz.c02, k0, N, nh, 0, 2);
    }
    for (int s = 0; s < S; ++s) {
        const int w = slot_w[size_t(s)], aw = std::abs(w);
        if (built.count(aw)) {
            set.slots[size_t(s)] = built[aw];
            for (int q = 0; q < s; ++q)
                if (std::abs(slot_w[size_t(q)]) == aw) {
                    set.plans[size_t(s)] = set.plans[size_t(q)];
                    break;
                }
            set.plans[size_t(s)].w = w;
            continue;
        }
        const int j0 = aw & 1;  // scalar class: j + w even
        if (!with_adi && !keep_static && !(with_diag && !so.diag_poisson.count(aw))) {
            // diagonalization data of this |w| already cached (the shared Poisson basis): nothing to build
            if (with_diag) diag_in.push_back({aw, CBand{}, CBand{}, CBand{}});
            AdiSlot d{};
            d.j0 = j0;
            built[aw] = d;
            set.slots[size_t(s)] = d;
            set.plans[size_t(s)].w = w;
            continue;
        }
        const Dense lw = radial_laplacian(so.ur, aw);
        Dense Af, Cf;
        if (poisson) {
            Af = lw;
            Cf = so.ur.r2;
        } else {
            Af = axpby(1.0, so.ur.r2, -scale, lw);
            Cf = scaled(so.ur.r2, -scale);
        }
        const Dense Ar = recombine(Af), Cr = recombine(Cf);
        const CBand Ac = compress(Ar, j0, M, M, -2, 3), Cc = compress(Cr, j0, M, M, -2, 3);
        const CBand R2c = compress(so.ur.r2, j0, M, mh, -1, 3);
        if (with_diag) {  // Poisson pencil bands of this |w| (shared modal basis, see SizeOps)
            const CBand Ap = compress(recombine(lw), j0, M, M, -2, 3);
            const CBand Cp = compress(so.R2rec, j0, M, M, -2, 3);
            diag_in.push_back({aw, Ap, Cp, R2c});
        }
        if (!with_adi) {  // diagonalization data only (no plan, no ADI shift blocks); the static operator
            // bands (R2, A, C | C02, B^T, D^T) are kept for host-side residual checks (diag_check_residual)
            AdiSlot d{};
            d.j0 = j0;
            if (!keep_static) {
                built[aw] = d;
                set.slots[size_t(s)] = d;
                set.plans[size_t(s)].w = w;
                continue;
            }
            d.sleft = alloc(size_t(M) * kStatW);
            d.sright0 = alloc(size_t(N) * kStatW);
            d.sright1 = alloc(size_t(N) * kStatW);
            for (int a = 0; a < M; ++a) {
                double* r = C.data() + d.sleft + size_t(a) * kStatW;
                for (int q = 0; q < 5; ++q) r[1 + q] = R2c.at(a, q - 1);
                for (int q = 0; q < 6; ++q) {
                    r[6 + q] = Ac.at(a, q - 2);
                    r[12 + q] = Cc.at(a, q - 2);
                }
            }
            for (int k0 = 0; k0 < 2; ++k0)
                for (int b = 0; b < N; ++b) {
                    double* r = C.data() + (k0 ? d.sright1 : d.sright0) + size_t(b) * kStatW;
                    for (int q = 0; q < 3; ++q) r[1 + q] = C02c[k0].at(b, q);
                    for (int q = 0; q < 4; ++q) {
                        r[12 + q] = Btc[k0].at(b, q - 1);
                        r[16 + q] = Dtc[k0].at(b, q - 1);
                    }
                }
            built[aw] = d;
            set.slots[size_t(s)] = d;
            set.plans[size_t(s)].w = w;
            continue;
        }

        const Range mu = radial_cache.at(aw);
        Range ca = poisson ? mu : Range{-1.0 / scale + mu.lo, -1.0 / scale + mu.hi};
        Plan plan;
        Range db = vert;
        try {
            plan = shift_plan(ca, vert, tol);
        } catch (const Error& e) {
            if (!(q2_pad && e.status == DOMAIN_ERROR)) throw;
            // endpoint-relative pad only where the reference intervals overlap
            const Range mu2 = radial_range(so, aw, true);
            db = vertical_range(so, true);
            ca = poisson ? mu2 : Range{-1.0 / scale + mu2.lo, -1.0 / scale + mu2.hi};
            plan = shift_plan(ca, db, tol);
        }
        // Executed shifts: the reference plan (reported through modal_plan), or with plan_margin > 1
        // the Zolotarev plan for tol / plan_margin (1-2 more shifts) so that rounding in the first
        // round does not push a slot just over tol into a second, serial round; the acceptance test
        // per round stays ||R|| / ||E|| <= tol.
        const Plan xplan = plan_margin > 1.0 ? shift_plan(ca, db, tol / plan_margin) : plan;
        const int J = xplan.J;
        AdiSlot d{};
        d.J = J;
        d.j0 = j0;
        d.left = alloc(size_t(J) * lrows * kLeftW);
        d.right0 = alloc(size_t(J) * rrows * kRightW);
        d.right1 = alloc(size_t(J) * rrows * kRightW);
        d.sleft = alloc(size_t(M) * kStatW);
        d.sright0 = alloc(size_t(N) * kStatW);
        d.sright1 = alloc(size_t(N) * kStatW);
        d.ds = alloc(size_t(J) + 1);
        // left dynamic blocks
        for (int j = 0; j < J; ++j) {
            const CBand mul = cb_axpy(xplan.u[size_t(j)], Cc, -1.0, Ac);
            const CBand sh = cb_axpy(xplan.v[size_t(j)], Cc, -1.0, Ac);
            CLU lu;
            try {
                lu = banded_lu(sh, 2, 3);
            } catch (const Error&) {
                Error e(SINGULAR, "ADI: singular (v_j C - A)");
                e.shift_index = j;
                throw e;
            }
            double* blk = C.data() + d.left + size_t(j) * lrows * kLeftW;
            for (int a = 0; a < M; ++a) {
                double* r = blk + size_t(a) * kLeftW;
                for (int q = 0; q < 6; ++q) r[q] = mul.at(a, q - 2);
                r[6] = lu.L[size_t(a) * 2];
                r[7] = lu.L[size_t(a) * 2 + 1];
                r[8] = lu.inv[size_t(a)];
                r[9] = double(lu.piv[size_t(a)]);
                if (lu.piv[size_t(a)]) d.pivot = 1;
                for (int q = 0; q < 5; ++q) r[10 + q] = lu.U[size_t(a) * 5 + q] * lu.inv[size_t(a)];
            }
            C[size_t(d.ds) + j] = xplan.u[size_t(j)] - xplan.v[size_t(j)];
        }
        // right dynamic blocks
        for (int k0 = 0; k0 < 2; ++k0) {
            const long base = k0 ? d.right1 : d.right0;
            for (int j = 0; j < J; ++j) {
                // G_{j+1} = X_{j+1} (v_{j+1} B + D); identity after the last shift (the row sweep then yields X)
                CBand mul = (j + 1 < J) ? cb_axpy(xplan.v[size_t(j + 1)], Btc[k0], 1.0, Dtc[k0]) : Btc[k0];
                if (j + 1 == J)
                    for (int b = 0; b < N; ++b)
                        for (int d = -1; d <= 2; ++d) mul.v[size_t(b) * 4 + size_t(d + 1)] = (d == 0) ? 1.0 : 0.0;
                const CBand sh = cb_axpy(xplan.u[size_t(j)], Btc[k0], 1.0, Dtc[k0]);
                CLU lu;
                try {
                    lu = banded_lu(sh, 1, 2);
                } catch (const Error&) {
                    Error e(SINGULAR, "ADI: singular (u_j B + D)");
                    e.shift_index = j;
                    throw e;
                }
                double* blk = C.data() + base + size_t(j) * rrows * kRightW;
                for (int b = 0; b < N; ++b) {
                    double* r = blk + size_t(b) * kRightW;
                    for (int q = 0; q < 4; ++q) r[q] = mul.at(b, q - 1);
                    put_right_lu(r + 4, lu, b);
                    if (lu.piv[size_t(b)]) d.pivot = 1;
                }
            }
            // static right block
            CLU lub;
            try {
                lub = banded_lu(Btc[k0], 1, 2);
            } catch (const Error&) {
                throw Error(SINGULAR, "AdiWorkspace: B is singular");
            }
            const CBand rs = cb_axpy(xplan.v[0], Btc[k0], 1.0, Dtc[k0]);
            double* blk = C.data() + (k0 ? d.sright1 : d.sright0);
            for (int b = 0; b < N; ++b) {
                double* r = blk + size_t(b) * kStatW;
                r[0] = 0.0;
                for (int q = 0; q < 3; ++q) r[1 + q] = C02c[k0].at(b, q);
                put_right_lu(r + 4, lub, b);
                if (lub.piv[size_t(b)]) d.pivot = 1;
                for (int q = 0; q < 4; ++q) {
                    r[12 + q] = Btc[k0].at(b, q - 1);
                    r[16 + q] = Dtc[k0].at(b, q - 1);
                    r[20 + q] = rs.at(b, q - 1);
                }
            }
        }
        // static left block
        {
            // C must be invertible for ADI (adi.cpp:121-124)
            try {
                (void)banded_lu(Cc, 2, 3);
            } catch (const Error&) {
                throw Error(SINGULAR, "AdiWorkspace: C is singular; ADI needs invertible C");
            }
            double* blk = C.data() + d.sleft;
            for (int a = 0; a < M; ++a) {
                double* r = blk + size_t(a) * kStatW;
                r[0] = 0.0;
                for (int q = 0; q < 5; ++q) r[1 + q] = R2c.at(a, q - 1);
                for (int q = 0; q < 6; ++q) {
                    r[6 + q] = Ac.at(a, q - 2);
                    r[12 + q] = Cc.at(a, q - 2);
                }
            }
        }
        // spike vectors for the partitioned sweeps (unpivoted slots only: the fields they
        // occupy hold pivoted fill-in otherwise, and pivoted slots keep the sequential sweeps)
        const int hc = spike_split(lrows - 2), hr = spike_split(rrows - 2);
        if (!d.pivot && hc > 0 && hr > 0 && hc < M && hr < N) {
            for (int j = 0; j < J; ++j) {
                add_left_spikes(C.data() + d.left + size_t(j) * lrows * kLeftW, M, hc);
                add_right_spikes(C.data() + d.right0 + size_t(j) * rrows * kRightW, N, hr);
                add_right_spikes(C.data() + d.right1 + size_t(j) * rrows * kRightW, N, hr);
            }
        }
        built[aw] = d;
        set.slots[size_t(s)] = d;
        set.plans[size_t(s)].w = w;
        set.plans[size_t(s)].plan = plan;
        set.plans[size_t(s)].has_plan = true;
    }
    C.resize(C.size() + 256, 0.0);  // read slack past the last block
    if (with_diag) {
        // Poisson-pencil left data per unique |w| (cached per size; parallel: O(M^3) long double each)
        std::vector<size_t> todo;
        for (size_t i = 0; i < diag_in.size(); ++i)
            if (!so.diag_poisson.count(diag_in[i].aw)) todo.push_back(i);
        std::vector<DiagLeft> fresh(todo.size());
        std::vector<std::string> errs(todo.size());
        std::vector<int> codes(todo.size(), 0);
        {
            const int nth = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), int(todo.size())));
            std::vector<std::thread> pool;
            std::atomic<size_t> next{0};
            for (int q = 0; q < nth; ++q)
                pool.emplace_back([&] {
                    for (;;) {
                        const size_t i = next.fetch_add(1);
                        if (i >= todo.size()) break;
                        const auto& di = diag_in[todo[i]];
                        try {
                            fresh[i] = diag_left(di.A, di.C, di.R2, M, mh);
                        } catch (const Error& e) {
                            codes[i] = e.status;
                            errs[i] = e.what();
                        }
                    }
                });
            for (auto& th : pool) th.join();
        }
        for (size_t i = 0; i < todo.size(); ++i)
            if (codes[i]) throw Error(codes[i], errs[i]);
        for (size_t i = 0; i < todo.size(); ++i) so.diag_poisson[diag_in[todo[i]].aw] = std::move(fresh[i]);
        // this set's left data: Poisson as cached; Helmholtz (A = R2 - s L, C = -s R2): same V,
        // lambda = nu - 1/s, PL = -(1/s) PL_Poisson
        std::vector<DiagLeft> left(diag_in.size());
        const bool mass = !poisson && scale == 0.0;
        DiagLeft mass_l[2];
        for (size_t i = 0; i < diag_in.size(); ++i) {
            const DiagLeft& P = so.diag_poisson.at(diag_in[i].aw);
            DiagLeft& L = left[i];
            if (mass) {  // scale 0 (solvers.cpp:57-62): X = R2'^-1 (R2 f C02^T) C02'^-T, no eigenpairs involved
                const int j0 = diag_in[i].aw & 1;
                if (mass_l[j0].PL.empty())
                    mass_l[j0] = mass_left(compress(so.R2rec, j0, M, M, -2, 3), compress(so.ur.r2, j0, M, mh, -1, 3), M, mh);
                L = mass_l[j0];
                continue;
            }
            L.QL = P.QL;
            if (poisson) {
                L.PL = P.PL;
                L.lam = P.lam;
                L.lam_ld = P.lam_ld;
            } else {
                const long double is = 1.0L / (long double)scale;
                L.PL.resize(P.PL_ld.size());
                for (size_t q = 0; q < P.PL_ld.size(); ++q) L.PL[q] = double(-is * P.PL_ld[q]);
                L.lam_ld.resize(P.lam_ld.size());
                L.lam.resize(P.lam_ld.size());
                for (size_t q = 0; q < P.lam_ld.size(); ++q) {
                    L.lam_ld[q] = P.lam_ld[q] - is;
                    L.lam[q] = double(L.lam_ld[q]);
                }
            }
        }
        std::vector<double>& G = set.dg;
        auto put = [&](const std::vector<double>& x) {
            const long off = long(G.size());
            G.insert(G.end(), x.begin(), x.end());
            if (G.size() % 2) G.push_back(0.0);
            return off;
        };
        // right data per k-parity (scale-independent, cached per size)
        if (!so.diag_right_ok) {
            for (int k0 = 0; k0 < 2; ++k0) so.diag_right_data[k0] = diag_right(Btc[k0], Dtc[k0], C02c[k0], N, nh);
            so.diag_right_ok = true;
        }
        DiagRight mass_r[2];
        if (mass)
            for (int k0 = 0; k0 < 2; ++k0) mass_r[k0] = mass_right(Btc[k0], C02c[k0], N, nh);
        const DiagRight* right = mass ? mass_r : so.diag_right_data;
        // QL (mh x M) and PR (nh x N) are stored with the leading dimension rounded up to even so
        // that every GEMM operand row is 16-byte aligned (cp.async pipeline)
        auto padld = [](const std::vector<double>& x, int rows, int cols) {
            const int ld = cols + (cols & 1);
            std::vector<double> o(size_t(rows) * ld, 0.0);
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < cols; ++c) o[size_t(r) * ld + c] = x[size_t(r) * cols + c];
            return o;
        };
        std::map<int, long> left_off;
        for (size_t i = 0; i < diag_in.size(); ++i) {
            const long o = put(left[i].PL);
            put(padld(left[i].QL, mh, M));
            put(left[i].lam);
            for (int k0 = 0; k0 < 2; ++k0) {  // 1 / (lambda_i + mu_j), rounded once; M x N, ld N rounded up to even
                const int ldr = N + (N & 1);
                std::vector<double> rt(size_t(M) * ldr, 0.0);
                for (int a = 0; a < M; ++a)
                    for (int b = 0; b < N; ++b)
                        rt[size_t(a) * ldr + b] =
                            double(1.0L / ((long double)left[i].lam_ld[size_t(a)] + right[k0].mu_ld[size_t(b)]));
                put(rt);
            }
            left_off[diag_in[i].aw] = o;
        }
        set.dg_left.resize(size_t(S));
        for (int s = 0; s < S; ++s) set.dg_left[size_t(s)] = left_off.at(std::abs(slot_w[size_t(s)]));
        for (int k0 = 0; k0 < 2; ++k0) {
            set.dg_right[k0] = put(padld(right[k0].PR, nh, N));
            put(right[k0].QR);
            put(right[k0].mu);
        }
        set.has_diag = true;
    }
    for (const AdiSlot& d : set.slots) {
        set.maxJ = std::max(set.maxJ, d.J);
        set.iters_per_round += d.J;
    }
    return set;
}

double diag_check_residual(const SolverSet& set, int slot, int k0, int M, int N, unsigned long long seed) {
    if (!set.has_diag) throw Error(DOMAIN_ERROR, "diag_check_residual: set has no diagonalization data");
    const int mh = M + 1, nh = N + 1, Mp = M + (M & 1), Np = N + (N & 1);
    auto even = [](long x) { return x + (x & 1); };
    const double* dg = set.dg.data();
    const long PLo = set.dg_left[size_t(slot)], QLo = PLo + long(M) * mh, LAMo = QLo + long(mh) * Mp,
               RTo = LAMo + even(M) + long(k0) * long(M) * Np;
    const long PRo = set.dg_right[k0], QRo = PRo + long(nh) * Np;
    std::vector<double> f(size_t(mh) * nh);
    unsigned long long st = seed * 0x9E3779B97F4A7C15ull + 1;
    for (double& x : f) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        x = double(st >> 11) / 9007199254740992.0 - 0.5;
    }
    auto mm = [](const double* A, int lda, const double* B, int ldb, int r, int k, int c) {
        std::vector<double> C(size_t(r) * c, 0.0);
        for (int i = 0; i < r; ++i)
            for (int q = 0; q < k; ++q) {
                const double a = A[size_t(i) * lda + q];
                if (a == 0.0) continue;
                for (int j = 0; j < c; ++j) C[size_t(i) * c + j] = std::fma(a, B[size_t(q) * ldb + j], C[size_t(i) * c + j]);
            }
        return C;
    };
    std::vector<double> T1 = mm(dg + PLo, mh, f.data(), nh, M, mh, nh);
    std::vector<double> Z = mm(T1.data(), nh, dg + PRo, Np, M, nh, N);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) Z[size_t(i) * N + j] *= dg[RTo + long(i) * Np + j];
    std::vector<double> T3 = mm(dg + QLo, Mp, Z.data(), N, mh, M, N);
    std::vector<double> u = mm(T3.data(), N, dg + QRo, nh, mh, N, nh);
    // X = S_r^-1 u S_z^-T: u[a][b] = X[a][b] - X[a-1][b] - X[a][b-1] + X[a-1][b-1] -> prefix sums
    std::vector<long double> X(size_t(M) * N, 0.0L);
    for (int a = 0; a < M; ++a)
        for (int b = 0; b < N; ++b) {
            long double v = u[size_t(a) * nh + b];
            if (a > 0) v += X[size_t(a - 1) * N + b];
            if (b > 0) v += X[size_t(a) * N + b - 1];
            if (a > 0 && b > 0) v -= X[size_t(a - 1) * N + b - 1];
            X[size_t(a) * N + b] = v;
        }
    const AdiSlot& so = set.slots[size_t(slot)];
    const double* sl = set.coef.data() + so.sleft;
    const double* sr = set.coef.data() + (k0 ? so.sright1 : so.sright0);
    auto fx = [&](int i, int j) -> long double { return (i >= 0 && i < mh && j >= 0 && j < nh) ? f[size_t(i) * nh + j] : 0.0L; };
    auto xx = [&](int i, int j) -> long double { return (i >= 0 && i < M && j >= 0 && j < N) ? X[size_t(i) * N + j] : 0.0L; };
    long double rr = 0.0L, ee = 0.0L;
    for (int a = 0; a < M; ++a)
        for (int b = 0; b < N; ++b) {
            // E = R2 f C02^T: rows via sleft 0..5 (d = -2..3), columns via sright 0..3 (d = -1..2)
            long double e = 0.0L, r = 0.0L;
            for (int dc = -1; dc <= 2; ++dc) {
                const long double cz = sr[size_t(b) * kStatW + size_t(dc + 1)];
                if (cz == 0.0L) continue;
                long double t = 0.0L;
                for (int da = -2; da <= 3; ++da) t += (long double)sl[size_t(a) * kStatW + size_t(da + 2)] * fx(a + da, b + dc);
                e += cz * t;
            }
            // A X B^ + C X D^: left rows sleft 6..11 / 12..17, right sright 12..15 / 16..19
            for (int da = -2; da <= 3; ++da) {
                const long double ca = sl[size_t(a) * kStatW + 6 + size_t(da + 2)];
                const long double cc = sl[size_t(a) * kStatW + 12 + size_t(da + 2)];
                if (ca == 0.0L && cc == 0.0L) continue;
                long double xb = 0.0L, xd = 0.0L;
                for (int dc = -1; dc <= 2; ++dc) {
                    xb += (long double)sr[size_t(b) * kStatW + 12 + size_t(dc + 1)] * xx(a + da, b + dc);
                    xd += (long double)sr[size_t(b) * kStatW + 16 + size_t(dc + 1)] * xx(a + da, b + dc);
                }
                r += ca * xb + cc * xd;
            }
            rr += (r - e) * (r - e);
            ee += e * e;
        }
    return double(std::sqrt(rr / ee));
}

}  // namespace ccf
