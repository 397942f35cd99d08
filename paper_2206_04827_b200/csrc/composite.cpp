// Composite radial operators (see composite.hpp). The pencil programs below mirror
// pencil.cu (pt_synth_kernel, curl_decomp_kernel) step by step.
#include "composite.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <thread>

namespace ccf {

namespace {

using R = long double;
using Pv = std::vector<R>;

int slot_w(int s, int p) { return s == p / 2 ? -p / 2 : s; }

// pencil.cu pen_dr: compressed parity j0 in -> 1 - j0 out
void dr(const Pv& in, Pv& out, int mh, int j0, R sg = 1.0L) {
    R b = 0.0L;
    if (j0 == 0) {
        for (int i = mh - 1; i >= 0; --i) {
            if (i + 1 < mh) b += R(4 * i + 4) * in[size_t(i) + 1];
            out[size_t(i)] = sg * b;
        }
    } else {
        for (int i = mh - 1; i >= 0; --i) {
            b += R(4 * i + 2) * in[size_t(i)];
            out[size_t(i)] = sg * (i == 0 ? 0.5L * b : b);
        }
    }
}

// pencil.cu pen_divr (Q1 D_r)
void divr(const Pv& in, Pv& out, int mh, int j0, const std::vector<double>& q) {
    if (j0 == 1) {
        R gn = 0.0L;
        for (int i = mh - 1; i >= 1; --i) {
            const R gv = 2.0L * in[size_t(i)] - gn;
            out[size_t(i)] = gv;
            gn = gv;
        }
        out[0] = in[0] - 0.5L * gn;
    } else {
        R f0 = 0.0L;
        for (int i = 0; i < mh; ++i) f0 += (i & 1) ? -in[size_t(i)] : in[size_t(i)];
        R h = 0.0L;
        out[size_t(mh) - 1] = f0 * R(q[size_t(mh) - 1]);
        for (int i = mh - 2; i >= 0; --i) {
            h = 2.0L * in[size_t(i) + 1] - h;
            out[size_t(i)] = f0 * R(q[size_t(i)]) + h;
        }
    }
}

void axpy(R a, const Pv& x, Pv& y, int mh) {
    for (int i = 0; i < mh; ++i) y[size_t(i)] += a * x[size_t(i)];
}

// pencil.cu pen_hp (horizontal Poisson, solvers.cpp:177-203)
void hp(const Pv& rhs, R sgn, Pv& out, int mh, int M, const double* hc, const double* rc) {
    Pv y(static_cast<size_t>(M) + 1, 0.0L);
    for (int a = 0; a < M; ++a) {
        const double* c = rc + a * 8;
        R acc = 0.0L;
        for (int d = -1; d <= 3; ++d) {
            const int i = a + d;
            if (i >= 0 && i < mh) acc += R(c[d + 1]) * rhs[size_t(i)];
        }
        y[size_t(a)] = sgn * acc;
    }
    for (int a = 0; a < M; ++a) {
        const double* c = hc + a * 8;
        if (c[1] == 1.0 && a + 1 < M) std::swap(y[size_t(a)], y[size_t(a) + 1]);
        if (a + 1 < M) y[size_t(a) + 1] -= R(c[0]) * y[size_t(a)];
    }
    R x1 = 0.0L, x2 = 0.0L, x3 = 0.0L;
    for (int a = M - 1; a >= 0; --a) {
        const double* c = hc + a * 8;
        R acc = y[size_t(a)] * R(c[2]) - R(c[5]) * x3 - R(c[4]) * x2 - R(c[3]) * x1;
        y[size_t(a)] = acc;
        x3 = x2;
        x2 = x1;
        x1 = acc;
    }
    R prev = 0.0L;
    for (int i = 0; i < mh; ++i) {
        const R cur = i < M ? y[size_t(i)] : 0.0L;
        out[size_t(i)] = cur - prev;
        prev = cur;
    }
}

// pt_synth_kernel for one slot: in[0..5] = (lam re, lam im, gam re, gam im, dzgam re, dzgam im),
// out[0..5] = (V_r re, im, V_t re, im, V_z re, im)
void pt_synth_program(const RadialTables& t, int s, const Pv* in, Pv* out) {
    const int mh = t.mh, p = t.p;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0s = w & 1;
    const R fw = R(w);
    const Pv &lr = in[0], &li = in[1], &gr = in[2], &gi = in[3], &zr = in[4], &zi = in[5];
    Pv s1(static_cast<size_t>(mh), 0.0L), s2(static_cast<size_t>(mh), 0.0L);
    dr(zr, out[0], mh, j0s);
    dr(zi, out[1], mh, j0s);
    if (pair) {
        divr(li, s1, mh, j0s, t.q);
        axpy(-fw, s1, out[0], mh);
    }
    dr(lr, out[2], mh, j0s, -1.0L);
    dr(li, out[3], mh, j0s, -1.0L);
    if (pair) {
        divr(zi, s1, mh, j0s, t.q);
        axpy(-fw, s1, out[2], mh);
    }
    for (int pl = 0; pl < 2; ++pl) {
        const Pv& gg = pl ? gi : gr;
        Pv& vz = out[4 + pl];
        dr(gg, s1, mh, j0s);
        dr(s1, vz, mh, 1 - j0s);
        if (pl == 0 || !pair) {
            if (pair) {
                divr(gg, s2, mh, j0s, t.q);
                axpy(-fw * fw, s2, s1, mh);
            }
            divr(s1, s2, mh, 1 - j0s, t.q);
            for (int i = 0; i < mh; ++i) vz[size_t(i)] = -(vz[size_t(i)] + s2[size_t(i)]);
        } else {
            for (int i = 0; i < mh; ++i) vz[size_t(i)] = -vz[size_t(i)];
        }
    }
}

// curl_decomp_kernel (curl path) for one slot: in[0..9] = (a_r re, im, a_t re, im, a_z re, im,
// dz a_r re, im, dz a_t re, im), out[0..3] = (gamma re, im, lambda re, im)
void curl_decomp_program(const RadialTables& t, int s, const Pv* in, Pv* out) {
    const int mh = t.mh, p = t.p, M = t.M;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0f = (w + 1) & 1, j0s = 1 - j0f;
    const R fw = R(w);
    const Pv &ari = in[1], &atr = in[2], &ati = in[3], &azr = in[4], &azi = in[5];
    const Pv &dzar = in[6], &dzai = in[7], &dzti = in[9];
    Pv ozr(static_cast<size_t>(mh), 0.0L), ozi(static_cast<size_t>(mh), 0.0L), otr(static_cast<size_t>(mh), 0.0L), oti(static_cast<size_t>(mh), 0.0L), s1(static_cast<size_t>(mh), 0.0L), s2(static_cast<size_t>(mh), 0.0L);
    dr(atr, ozr, mh, j0f);
    dr(ati, ozi, mh, j0f);
    if (pair) {
        for (int i = 0; i < mh; ++i) s1[size_t(i)] = fw * ari[size_t(i)] + atr[size_t(i)];
        divr(s1, s2, mh, j0f, t.q);
        axpy(1.0L, s2, ozr, mh);
    } else {
        divr(atr, s2, mh, j0f, t.q);
        axpy(1.0L, s2, ozr, mh);
        divr(ati, s2, mh, j0f, t.q);
        axpy(1.0L, s2, ozi, mh);
    }
    dr(azr, otr, mh, j0s);
    dr(azi, oti, mh, j0s);
    for (int i = 0; i < mh; ++i) {
        otr[size_t(i)] = dzar[size_t(i)] - otr[size_t(i)];
        oti[size_t(i)] = dzai[size_t(i)] - oti[size_t(i)];
    }
    const double* hc = t.hpc.data() + size_t(s) * M * 8;
    const double* rc = t.hpr.data() + size_t(j0s) * M * 8;
    hp(ozr, -1.0L, out[0], mh, M, hc, rc);
    hp(ozi, -1.0L, out[1], mh, M, hc, rc);
    Pv czr(static_cast<size_t>(mh), 0.0L), czi(static_cast<size_t>(mh), 0.0L);
    dr(otr, czr, mh, j0f);
    dr(oti, czi, mh, j0f);
    if (pair) {
        for (int i = 0; i < mh; ++i) s1[size_t(i)] = -fw * dzti[size_t(i)] + otr[size_t(i)];
        divr(s1, s2, mh, j0f, t.q);
        axpy(1.0L, s2, czr, mh);
    } else {
        divr(otr, s2, mh, j0f, t.q);
        axpy(1.0L, s2, czr, mh);
        divr(oti, s2, mh, j0f, t.q);
        axpy(1.0L, s2, czi, mh);
    }
    hp(czr, -1.0L, out[2], mh, M, hc, rc);
    hp(czi, -1.0L, out[3], mh, M, hc, rc);
}

// Basis injection for one slot: maps[o][i] = mh x mh matrix (row = output index, col = input index).
template <class Prog>
void slot_maps(const RadialTables& t, int s, int nin, int nout, Prog prog, std::vector<std::vector<Pv>>& maps) {
    const int mh = t.mh;
    maps.assign(size_t(nout), std::vector<Pv>(size_t(nin), Pv(size_t(mh) * mh, 0.0L)));
    std::vector<Pv> in(size_t(nin), Pv(size_t(mh), 0.0L)), out(size_t(nout), Pv(size_t(mh), 0.0L));
    for (int x = 0; x < nin; ++x)
        for (int j = 0; j < mh; ++j) {
            in[size_t(x)][size_t(j)] = 1.0L;
            for (auto& o : out) std::fill(o.begin(), o.end(), 0.0L);
            prog(t, s, in.data(), out.data());
            in[size_t(x)][size_t(j)] = 0.0L;
            for (int o = 0; o < nout; ++o)
                for (int i = 0; i < mh; ++i) maps[size_t(o)][size_t(x)][size_t(i) * mh + j] = out[size_t(o)][size_t(i)];
        }
}

bool nonzero(const Pv& a) {
    for (R v : a)
        if (v != 0.0L) return true;
    return false;
}

template <class Body>
void parallel_slots(int nslots, Body body) {
    const int nth = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), nslots));
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int q = 0; q < nth; ++q)
        pool.emplace_back([&] {
            for (;;) {
                const int s = next.fetch_add(1);
                if (s >= nslots) break;
                body(s);
            }
        });
    for (auto& th : pool) th.join();
}

struct SlotBlocks {
    std::vector<CompositeTerm> terms;  // off relative to this slot's block list
    std::vector<double> data;
};

CompositeSet assemble(const RadialTables& t, std::vector<SlotBlocks>& per) {
    CompositeSet cs;
    cs.mh = t.mh;
    cs.nslots = t.nslots;
    cs.terms.resize(size_t(t.nslots));
    size_t total = 0;
    for (auto& sb : per) total += sb.data.size();
    cs.blocks.reserve(total);
    for (int s = 0; s < t.nslots; ++s) {
        const long base = long(cs.blocks.size());
        for (CompositeTerm ct : per[size_t(s)].terms) {
            ct.off += base;
            cs.terms[size_t(s)].push_back(ct);
        }
        cs.blocks.insert(cs.blocks.end(), per[size_t(s)].data.begin(), per[size_t(s)].data.end());
    }
    return cs;
}

}  // namespace

CompositeSet build_synth_composite(const RadialTables& t) {
    const int mh = t.mh;
    std::vector<SlotBlocks> per(size_t(t.nslots));
    parallel_slots(t.nslots, [&](int s) {
        std::vector<std::vector<Pv>> maps;
        slot_maps(t, s, 6, 6, pt_synth_program, maps);
        const int w = slot_w(s, t.p);
        const int cls[3] = {1, 1, 0};  // V_r, V_theta flip class; V_z scalar class
        SlotBlocks& sb = per[size_t(s)];
        for (int o = 0; o < 6; ++o) {
            const int F = o / 2;
            const int j0 = (w + cls[F]) & 1;
            const std::vector<double>& S = t.SrT[j0];
            for (int x = 0; x < 6; ++x) {
                const Pv& Mx = maps[size_t(o)][size_t(x)];
                if (!nonzero(Mx)) continue;
                // block[jr][jj] = sum_i SrT[jr][i] * M[i][jj]
                const long off = long(sb.data.size());
                sb.data.resize(sb.data.size() + size_t(mh) * mh);
                for (int jr = 0; jr < mh; ++jr)
                    for (int jj = 0; jj < mh; ++jj) {
                        R acc = 0.0L;
                        for (int i = 0; i < mh; ++i) acc += R(S[size_t(jr) * mh + i]) * Mx[size_t(i) * mh + jj];
                        sb.data[size_t(off) + size_t(jr) * mh + jj] = double(acc);
                    }
                sb.terms.push_back({o, x, off});
            }
        }
    });
    return assemble(t, per);
}

CompositeSet build_anal_composite(const RadialTables& t) {
    const int mh = t.mh;
    std::vector<SlotBlocks> per(size_t(t.nslots));
    parallel_slots(t.nslots, [&](int s) {
        std::vector<std::vector<Pv>> maps;
        slot_maps(t, s, 10, 4, curl_decomp_program, maps);
        const int w = slot_w(s, t.p);
        const int cls[5] = {1, 1, 0, 1, 1};  // a_r, a_t, a_z, dz a_r, dz a_t
        SlotBlocks& sb = per[size_t(s)];
        for (int o = 0; o < 4; ++o)
            for (int x = 0; x < 10; ++x) {
                const Pv& Mx = maps[size_t(o)][size_t(x)];
                if (!nonzero(Mx)) continue;
                const int j0 = (w + cls[x / 2]) & 1;
                const std::vector<double>& A = t.ArT[j0];
                // block[jj][jr] = sum_i M[jj][i] * ArT[i][jr]
                const long off = long(sb.data.size());
                sb.data.resize(sb.data.size() + size_t(mh) * mh);
                for (int jj = 0; jj < mh; ++jj)
                    for (int jr = 0; jr < mh; ++jr) {
                        R acc = 0.0L;
                        for (int i = 0; i < mh; ++i) acc += Mx[size_t(jj) * mh + i] * R(A[size_t(i) * mh + jr]);
                        sb.data[size_t(off) + size_t(jj) * mh + jr] = double(acc);
                    }
                sb.terms.push_back({o, x, off});
            }
    });
    return assemble(t, per);
}

}  // namespace ccf
