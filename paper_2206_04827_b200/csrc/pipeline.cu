// NS time-step pipeline (see pipeline.hpp).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <atomic>
#include <thread>

#include <cudaTypedefs.h>

#include "pipeline.hpp"
#include "ozaki_dev.cuh"

#include <cstdlib>

namespace ccf {


namespace {

std::vector<double> cheb_points_double(int count) {  // proj/src/grid.cpp:16-26 (pinned endpoints)
    std::vector<double> x(static_cast<size_t>(count));
    for (int j = 0; j < count; ++j) x[size_t(j)] = std::cos(double(count - j - 1) * M_PI / double(count - 1));
    x.front() = -1.0;
    x.back() = 1.0;
    if (count % 2 == 1) x[size_t(count / 2)] = 0.0;
    return x;
}

// cos(pi * a / L) with exact integer reduction, long double
long double cospi_frac(long a, long L) {
    long r = a % (2 * L);
    if (r < 0) r += 2 * L;
    return cosl(3.141592653589793238462643383279502884L * (long double)r / (long double)L);
}

void upload(DBuf& d, const std::vector<double>& h) {
    d.alloc(h.size());
    CCF_H2D(d.p, h.data(), h.size() * sizeof(double));
}

unsigned blocks_for(long n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace

TransformPlan::TransformPlan(Ctx& c) {
    SetupTimer tm("transform tables");
    const int m = c.m, n = c.n, p = c.p, mh = m / 2, M = c.M;
    const long L = m - 1, Lz = n - 1;
    // r synthesis / analysis on the r > 0 half grid, per coefficient parity j0 (A operands):
    //   SrT[j0][jr][i] = T_{2i+j0}(r_{mh+jr}),  ArT[j0][i][jr] = analysis weights (values -> coefficients)
    for (int j0 = 0; j0 < 2; ++j0) {
        std::vector<double> S(size_t(mh) * mh), A(size_t(mh) * mh);
        for (int i = 0; i < mh; ++i) {
            const int k = 2 * i + j0;
            const long double eps = (k == 0 || k == m - 1) ? 0.5L : 1.0L;
            for (int jr = 0; jr < mh; ++jr) {
                const int s = mh - 1 - jr;  // descending-x index of grid point j = mh + jr
                S[size_t(jr) * mh + i] = double(cospi_frac(long(k) * s, L));
                const long double ws = (s == 0) ? 1.0L : 2.0L;
                A[size_t(i) * mh + jr] = double(eps / (long double)L * 2.0L * ws * cospi_frac(long(k) * s, L));
            }
        }
        upload(SrT[j0], S);
        upload(ArT[j0], A);
        rt.SrT[j0] = S;
        rt.ArT[j0] = A;
    }
    // z: values are kept z-parity split per r row, [E | O] with E_i / O_i the even- / odd-k parts at
    // z_{nh+i} > 0 (f(+-z_{nh+i}) = E_i +- O_i), so each z transform is two nh x nh products:
    //   SzE[q][i] = T_{2q}(z_{nh+i}), SzO[q][i] = T_{2q+1}(z_{nh+i})          (synthesis, B operands)
    //   AzE[i][q] = 2 A[2q][nh+i],   AzO[i][q] = 2 A[2q+1][nh+i]            (analysis of E' / O')
    // (A[k][kz] the analysis weights; A[k][n-1-kz] = (-1)^k A[k][kz]). Requires even n.
    {
        const int nh = n / 2;
        auto zan = [&](int k, int kz) {
            const int s = n - 1 - kz;
            const long double eps = (k == 0 || k == n - 1) ? 0.5L : 1.0L;
            const long double ws = (s == 0 || s == n - 1) ? 1.0L : 2.0L;
            return eps / (long double)Lz * ws * cospi_frac(long(k) * s, Lz);
        };
        std::vector<double> S(size_t(n) * nh), A(size_t(n) * nh);  // [SzE ; SzO], [AzE ; AzO]
        for (int par = 0; par < 2; ++par)
            for (int q = 0; q < nh; ++q)
                for (int i = 0; i < nh; ++i) {
                    const int k = 2 * q + par, kz = nh + i;
                    S[size_t(par) * nh * nh + size_t(q) * nh + i] = double(cospi_frac(long(k) * (n - 1 - kz), Lz));
                    A[size_t(par) * nh * nh + size_t(i) * nh + q] = double(2.0L * zan(k, kz));
                }
        upload(Sz, S);
        upload(Az, A);
    }
    {
        const int nh = n / 2;
        std::vector<double> S(size_t(n) * n), A(size_t(n) * n);
        for (int kz = 0; kz < n; ++kz)
            for (int q = 0; q < n; ++q) {
                const int k = kfrompos(q, nh);
                const int s = n - 1 - kz;
                S[size_t(q) * n + kz] = double(cospi_frac(long(k) * s, Lz));
                const long double eps = (k == 0 || k == n - 1) ? 0.5L : 1.0L;
                const long double ws = (s == 0 || s == n - 1) ? 1.0L : 2.0L;
                A[size_t(kz) * n + q] = double(eps / (long double)Lz * ws * cospi_frac(long(k) * s, Lz));
            }
        std::vector<double> Sf(size_t(n) * n), Af(size_t(n) * n);
        for (int kz = 0; kz < n; ++kz)
            for (int q = 0; q < n; ++q) {
                const int k = kfrompos(q, nh);
                Sf[size_t(kz) * n + k] = S[size_t(q) * n + kz];
                Af[size_t(k) * n + kz] = A[size_t(kz) * n + q];
            }
        upload(Szf, Sf);
        upload(Azf, Af);
    }
    // r: dense m x m (API transforms): values_j = sum_k c_k T_k(r_j);  c_k = sum_j A[k][j] values_j
    {
        std::vector<double> S(size_t(m) * m), A(size_t(m) * m);
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < m; ++k) {
                const int s = m - 1 - j;
                S[size_t(j) * m + k] = double(cospi_frac(long(k) * s, L));
                const long double eps = (k == 0 || k == m - 1) ? 0.5L : 1.0L;
                const long double ws = (s == 0 || s == m - 1) ? 1.0L : 2.0L;
                A[size_t(k) * m + j] = double(eps / (long double)L * ws * cospi_frac(long(k) * s, L));
            }
        upload(Rfull_S, S);
        upload(Rfull_A, A);
    }
    // q: odd coefficients of the grid interpolant of 1/r (values divided by the reference's double r_j)
    {
        const auto r = cheb_points_double(m);
        std::vector<double> qv(static_cast<size_t>(mh));
        for (int i = 0; i < mh; ++i) {
            const int k = 2 * i + 1;
            const long double eps = (k == m - 1) ? 0.5L : 1.0L;
            long double acc = 0.0L;
            for (int s = 0; s < m; ++s) {
                const int j = m - 1 - s;
                const long double ws = (s == 0 || s == m - 1) ? 1.0L : 2.0L;
                acc += ws * (1.0L / (long double)r[size_t(j)]) * cospi_frac(long(k) * s, L);
            }
            qv[size_t(i)] = double(eps / (long double)L * acc);
        }
        upload(q, qv);
        rt.q = qv;
    }
    // theta twiddles
    {
        int lg = 0;
        while ((1 << lg) < p) ++lg;
        logp = ((1 << lg) == p) ? lg : -1;
        std::vector<double> t(static_cast<size_t>(p)), tf(static_cast<size_t>(2 * p));
        for (int i = 0; i < p / 2; ++i) {
            t[size_t(2 * i)] = double(cospi_frac(2L * i, p));
            t[size_t(2 * i + 1)] = -double(cospi_frac(2L * i - p / 2, p));  // -sin(2 pi i / p)
        }
        for (int i = 0; i < p; ++i) {
            tf[size_t(2 * i)] = double(cospi_frac(2L * i, p));
            tf[size_t(2 * i + 1)] = -double(cospi_frac(2L * i - p / 2, p));
        }
        upload(tw, t);
        upload(twfull, tf);
    }
    // horizontal Poisson: LU(recombine(L_w)) per half slot (proj/src/solvers.cpp:189-195), R R C02 per parity
    {
        const Geo& g = c.gh;
        std::vector<double> hc(size_t(g.nslots) * M * 8, 0.0), hr(size_t(2) * M * 8, 0.0);
        std::atomic<int> next{0}, bad{0};
        auto work = [&] {  // per slot: O(m^2) recombination + banded LU, independent across slots
            for (int s = next.fetch_add(1); s < g.nslots; s = next.fetch_add(1)) {
                const int w = (s == p / 2) ? -p / 2 : s;
                const int j0 = ((w % 2) + 2) % 2;
                const Dense lw = recombine(radial_laplacian(c.sizeops->ur, w));
                const CBand b = compress(lw, j0, M, M, -1, 2);
                CLU lu;
                try {
                    lu = banded_lu(b, 1, 2);
                } catch (const Error&) {
                    bad = 1;
                    continue;
                }
                for (int a = 0; a < M; ++a) {
                    double* r = hc.data() + (size_t(s) * M + a) * 8;
                    r[0] = lu.L[size_t(a)];
                    r[1] = double(lu.piv[size_t(a)]);
                    r[2] = lu.inv[size_t(a)];
                    for (int t = 0; t < 3; ++t) r[3 + t] = lu.U[size_t(a) * 3 + t] * lu.inv[size_t(a)];
                }
            }
        };
        {
            const int nth = std::max(1, std::min<int>(int(std::thread::hardware_concurrency()), g.nslots));
            std::vector<std::thread> pool;
            for (int q = 0; q < nth; ++q) pool.emplace_back(work);
            for (auto& th : pool) th.join();
        }
        if (bad) throw Error(SINGULAR, "solve_horizontal_poisson: singular column system");
        for (int j0 = 0; j0 < 2; ++j0) {
            const CBand b = compress(c.sizeops->ur.r2, j0, M, mh, -1, 3);
            for (int a = 0; a < M; ++a)
                for (int d = -1; d <= 3; ++d) hr[(size_t(j0) * M + a) * 8 + size_t(d + 1)] = b.at(a, d);
        }
        upload(hpc, hc);
        upload(hpr, hr);
        rt.hpc = hc;
        rt.hpr = hr;
        rt.m = m;
        rt.mh = mh;
        rt.M = M;
        rt.p = p;
        rt.nslots = g.nslots;
    }
    // derivative_z (calculus.cpp:34-43) folded into the z transforms of the nonlinear term:
    //   (dz c)_k = sum_{k' > k, k' - k odd} 2 k' c_k' (halved for k = 0), maps parity par -> 1 - par;
    //   DzS[po][q'][i] = sum_{k = 2q + po} Dz[k][2q' + 1 - po] T_k(z_{nh+i})
    //   ADz[po][i][q]  = sum_{q'} Az_{1-po}[i][q'] Dz[2q + po][2q' + 1 - po]
    {
        const int nh = n / 2;
        auto dzm = [&](int k, int kp) -> long double {
            if (kp <= k || ((kp - k) & 1) == 0) return 0.0L;
            return (k == 0 ? 1.0L : 2.0L) * (long double)kp;
        };
        auto zan = [&](int k, int kz) {
            const int s = n - 1 - kz;
            const long double eps = (k == 0 || k == n - 1) ? 0.5L : 1.0L;
            const long double ws = (s == 0 || s == n - 1) ? 1.0L : 2.0L;
            return eps / (long double)Lz * ws * cospi_frac(long(k) * s, Lz);
        };
        std::vector<double> DS(size_t(n) * nh, 0.0), AD(size_t(n) * nh, 0.0);
        // T_k(z_{nh+i}) and the analysis weights, tabulated once (the triple loops below are O(n^3))
        std::vector<long double> Tk(size_t(n) * nh), Zk(size_t(n) * nh);
        for (int k = 0; k < n; ++k)
            for (int i = 0; i < nh; ++i) {
                Tk[size_t(k) * nh + i] = cospi_frac(long(k) * (n - 1 - (nh + i)), Lz);
                Zk[size_t(k) * nh + i] = zan(k, nh + i);
            }
        for (int po = 0; po < 2; ++po) {
            const int pi = 1 - po;
            for (int qp = 0; qp < nh; ++qp)
                for (int i = 0; i < nh; ++i) {
                    long double acc = 0.0L;
                    for (int q = 0; q < nh; ++q) {
                        const int k = 2 * q + po;
                        const long double d = dzm(k, 2 * qp + pi);
                        if (d != 0.0L) acc += d * Tk[size_t(k) * nh + i];
                    }
                    DS[size_t(po) * nh * nh + size_t(qp) * nh + i] = double(acc);
                }
            for (int i = 0; i < nh; ++i)
                for (int q = 0; q < nh; ++q) {
                    long double acc = 0.0L;
                    for (int qp = 0; qp < nh; ++qp) {
                        const long double d = dzm(2 * q + po, 2 * qp + pi);
                        if (d != 0.0L) acc += 2.0L * Zk[size_t(2 * qp + pi) * nh + i] * d;
                    }
                    AD[size_t(po) * nh * nh + size_t(i) * nh + q] = double(acc);
                }
        }
        upload(DzS, DS);
        upload(ADz, AD);
    }
}

// ---------------------------------------------------------------- GEMM plans
namespace {
// driver entry points for the TMA GEMM (no link-time libcuda dependency)
struct DriverFns {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    PFN_cuMemGetAddressRange_v3020 range = nullptr;
};
const DriverFns& drv() {
    static const DriverFns d = [] {
        DriverFns f;
        cudaDriverEntryPointQueryResult q;
        void* e = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &e, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            f.encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(e);
        e = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &e, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            f.range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(e);
        return f;
    }();
    return d;
}
// CCF_GEMM_TMA: 1 (default) = every eligible plan, 2 = single-term plans only, 0 = off (cp.async kernel)
int tma_mode() {
    static const int on = [] {
        const char* e = std::getenv("CCF_GEMM_TMA");
        return e ? std::atoi(e) : 1;
    }();
    return (drv().encode && drv().range) ? on : 0;
}
// f64 2-D map over [base, base + bytes) viewed as rows of ld doubles; box 16 x box_rows, 128-byte swizzle
bool encode_map(CUtensorMap& m, const void* base, size_t bytes, long ld, int box_rows) {
    const cuuint64_t rows = bytes / (size_t(ld) * 8);
    if (rows == 0 || rows > (1ull << 31) || ld > (1L << 31)) return false;
    cuuint64_t dims[2] = {cuuint64_t(ld), rows};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
    cuuint32_t box[2] = {16, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    return drv().encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool alloc_range(const void* p, uintptr_t& base, size_t& size) {
    CUdeviceptr b = 0;
    size_t s = 0;
    if (drv().range(&b, &s, CUdeviceptr(reinterpret_cast<uintptr_t>(p))) != CUDA_SUCCESS) return false;
    base = uintptr_t(b);
    size = s;
    return true;
}
}  // namespace

void GemmPlan::upload() {
    // multi-term plans: batches in descending term count, so that a round-robin (persistent) item
    // assignment starts with the long items (LPT order) and the launch tail holds the short ones
    if (!tstart.empty() && tstart.size() > 2) {
        const size_t nbt = tstart.size() - 1;
        std::vector<size_t> ord(nbt);
        for (size_t b = 0; b < nbt; ++b) ord[b] = b;
        std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) {
            return tstart[x + 1] - tstart[x] > tstart[y + 1] - tstart[y];
        });
        std::vector<const double*> nA, nB;
        std::vector<long> nBoff, nAoff;
        std::vector<int> nT{0};
        for (size_t b : ord)
            for (int t = tstart[b]; t < tstart[b + 1]; ++t) {
                nA.push_back(A[size_t(t)]);
                if (!B.empty()) nB.push_back(B[size_t(t)]);
                if (!Boff.empty()) nBoff.push_back(Boff[size_t(t)]);
                if (!Aoff.empty()) nAoff.push_back(Aoff[size_t(t)]);
            }
        for (size_t b : ord) nT.push_back(nT.back() + (tstart[b + 1] - tstart[b]));
        auto permute = [&](auto& v) {
            if (v.size() != nbt) return;
            auto w = v;
            for (size_t i = 0; i < nbt; ++i) w[i] = v[ord[i]];
            v = w;
        };
        permute(C);
        permute(Coff);
        permute(DL);
        permute(DR);
        A = nA;
        if (!B.empty()) B = nB;
        if (!Boff.empty()) Boff = nBoff;
        if (!Aoff.empty()) Aoff = nAoff;
        tstart = nT;
    }
    const size_t nb = std::max(C.size(), Coff.size()), na = A.size();
    // the pipelined kernel copies 16-byte chunks: A / B bases (and base-relative offsets) 16-byte
    // aligned, even leading dimensions
    if (!Aoff.empty() && !Boff.empty()) throw Error(INTERNAL, "GemmPlan: base-relative A and B together");
    pipe = (lda % 2 == 0) && (ldb % 2 == 0);
    for (size_t i = 0; i < na && pipe; ++i) {
        if (Aoff.empty() ? (reinterpret_cast<uintptr_t>(A[i]) % 16 != 0) : (Aoff[i] % 2 != 0)) pipe = false;
        if (Boff.empty() ? (reinterpret_cast<uintptr_t>(B[i]) % 16 != 0) : (Boff[i] % 2 != 0)) pipe = false;
    }
    if (!dA) {
        CCF_CUDA(cudaMalloc(&dA, std::max<size_t>(na, 1) * sizeof(void*)));
        CCF_CUDA(cudaMalloc(&dB, std::max<size_t>(na, 1) * sizeof(void*)));
        CCF_CUDA(cudaMalloc(&dC, nb * sizeof(void*)));
        if (!tstart.empty()) CCF_CUDA(cudaMalloc(&dT, tstart.size() * sizeof(int)));
    }
    if (na) {
        CCF_H2D(dA, A.data(), na * sizeof(void*));
        CCF_H2D(dB, B.data(), na * sizeof(void*));
    }
    if (!C.empty()) CCF_H2D(dC, C.data(), C.size() * sizeof(void*));
    if (!tstart.empty()) CCF_H2D(dT, tstart.data(), tstart.size() * sizeof(int));
    if (!Boff.empty()) {
        if (!dBoff) CCF_CUDA(cudaMalloc(&dBoff, Boff.size() * sizeof(long)));
        CCF_H2D(dBoff, Boff.data(), Boff.size() * sizeof(long));
    }
    if (!Aoff.empty()) {
        if (!dAoff) CCF_CUDA(cudaMalloc(&dAoff, Aoff.size() * sizeof(long)));
        CCF_H2D(dAoff, Aoff.data(), Aoff.size() * sizeof(long));
    }
    if (!Coff.empty()) {
        if (!dCoff) CCF_CUDA(cudaMalloc(&dCoff, Coff.size() * sizeof(long)));
        CCF_H2D(dCoff, Coff.data(), Coff.size() * sizeof(long));
    }
    if (!DL.empty()) {
        if (!dDL) {
            CCF_CUDA(cudaMalloc(&dDL, nb * sizeof(void*)));
            CCF_CUDA(cudaMalloc(&dDR, nb * sizeof(void*)));
        }
        CCF_H2D(dDL, DL.data(), nb * sizeof(void*));
        CCF_H2D(dDR, DR.data(), nb * sizeof(void*));
    }
    // ---- TMA variant: one map per (operand allocation, leading dimension), box origins per term
    tma = false;
    const bool kbox_ok = K % 16 == 0 || K + kzero >= ((K + 15) / 16) * 16;  // no live data in the last k-box
    if (pipe && kbox_ok && tma_mode() && (tma_mode() == 1 || tstart.empty()) && M > 64 && !A.empty()) {
        struct Key {
            uintptr_t base;
            long ld;
            int box;
        };
        std::vector<Key> keys;
        std::vector<CUtensorMap> maps;
        std::vector<int> hta(4 * na), htb(2 * na);
        bool ok = true;
        auto find = [&](const double* ptr, long ld, int box, int& idx, int& col, int& row) {
            uintptr_t b;
            size_t sz;
            if (!alloc_range(ptr, b, sz)) return false;
            idx = -1;
            for (size_t k = 0; k < keys.size(); ++k)
                if (keys[k].base == b && keys[k].ld == ld && keys[k].box == box) idx = int(k);
            if (idx < 0) {
                if (keys.size() >= ((Boff.empty() && Aoff.empty()) ? size_t(kTmaMaps) : size_t(5))) return false;  // 5..7: launch bases
                CUtensorMap m;
                if (!encode_map(m, reinterpret_cast<const void*>(b), sz, ld, box)) return false;
                keys.push_back({b, ld, box});
                maps.push_back(m);
                idx = int(keys.size()) - 1;
            }
            const uintptr_t off = (reinterpret_cast<uintptr_t>(ptr) - b) / 8;
            if (off / uintptr_t(ld) > uintptr_t(1u << 31)) return false;
            row = int(off / uintptr_t(ld));
            col = int(off % uintptr_t(ld));
            return true;
        };
        for (size_t t = 0; t < na && ok; ++t) {
            int ia = 0, ca = 0, ra = 0;
            if (Aoff.empty()) {
                ok = find(A[t], lda, 128, ia, ca, ra);
            } else {  // relative to the launch base (slot 5 + base index)
                const long o = Aoff[t] & ((1L << kBaseShift) - 1);
                ia = 5 + int(Aoff[t] >> kBaseShift);
                ra = int(o / lda);
                ca = int(o % lda);
            }
            int ib = 0, cb = 0, rb = 0;
            if (ok) {
                if (Boff.empty()) {
                    ok = find(B[t], ldb, 16, ib, cb, rb);
                } else {  // relative to the launch base (slot 5 + base index)
                    const long o = Boff[t] & ((1L << kBaseShift) - 1);
                    ib = 5 + int(Boff[t] >> kBaseShift);
                    rb = int(o / ldb);
                    cb = int(o % ldb);
                }
            }
            // a block must not wrap around the rows of its 2-D view: the boxes read columns [col, col + extent)
            // of one row (past the row end they read zeros, not the wrapped data)
            if (ok && (long(ca) + K > lda || long(cb) + N > ldb)) ok = false;
            hta[4 * t] = ia;
            hta[4 * t + 1] = ca;
            hta[4 * t + 2] = ra;
            hta[4 * t + 3] = ib;
            htb[2 * t] = cb;
            htb[2 * t + 1] = rb;
        }
        if (ok) {
            tmaps = maps;
            if (!dTA) {
                CCF_CUDA(cudaMalloc(&dTA, hta.size() * sizeof(int)));
                CCF_CUDA(cudaMalloc(&dTB, htb.size() * sizeof(int)));
            }
            CCF_H2D(dTA, hta.data(), hta.size() * sizeof(int));
            CCF_H2D(dTB, htb.data(), htb.size() * sizeof(int));
            tma = true;
        }
    }
}

void GemmPlan::launch(cudaStream_t s, const double* b0, const double* b1, double* c0, double* c1,
                      const double* b2) const {
    const unsigned nb = unsigned(std::max(C.size(), Coff.size()));
    static const bool trace = std::getenv("CCF_GEMM_TRACE") != nullptr;  // diagnostics: one line per launch
    if (trace)
        std::fprintf(stderr, "[gemm] M %d N %d K %d batches %u terms %zu flops %.4e tma %d pipe %d\n", M, N, K, nb,
                     A.size(), flops(), int(tma), int(pipe));
    GemmBatch g{dA, dB, dC, M, N, K, lda, ldb, ldc, alpha, beta, dT, dDL, dDR, dBoff, dCoff, {b0, b1, b2}, {c0, c1}, int(nb),
                ldd ? ldd : long(N), 1, dAoff};
    const bool based_ok = (reinterpret_cast<uintptr_t>(b0) % 16 == 0) && (reinterpret_cast<uintptr_t>(b1) % 16 == 0);
    if (tma && based_ok) {
        static bool tattr = false;
        static int nsm = 0;
        if (!tattr) {
            CCF_CUDA(cudaFuncSetAttribute(dgemm_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(dgemm_tma_smem())));
            int dev = 0;
            CCF_CUDA(cudaGetDevice(&dev));
            CCF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            tattr = true;
        }
        TmaMaps mp{};
        for (size_t i = 0; i < tmaps.size(); ++i) mp.m[i] = tmaps[i];
        if (!Boff.empty() || !Aoff.empty()) {  // launch bases of the base-relative operand: maps cached per base
            const bool isA = !Aoff.empty();
            const double* bases[3] = {b0, b1 ? b1 : b0, b2 ? b2 : b0};
            for (int q = 0; q < 3; ++q) {
                const double* bp = bases[q];
                bool hit = false;
                for (auto& kv : bmap_cache)
                    if (kv.first == bp) {
                        mp.m[5 + q] = kv.second;
                        hit = true;
                    }
                if (!hit) {
                    uintptr_t ab;
                    size_t sz;
                    CUtensorMap m;
                    if (!bp || !alloc_range(bp, ab, sz) ||
                        !encode_map(m, bp, sz - (reinterpret_cast<uintptr_t>(bp) - ab), isA ? lda : ldb, isA ? 128 : 16))
                        throw Error(INTERNAL, "GemmPlan: cannot build the TMA map of a launch base");
                    bmap_cache.emplace_back(bp, m);
                    mp.m[5 + q] = m;
                }
            }
        }
        const long items = long(nb) * ((M + 127) / 128) * ((N + 63) / 64);
        dgemm_tma_kernel<<<unsigned(std::min<long>(items, 2L * nsm)), 288, dgemm_tma_smem(), s>>>(
            g, mp, static_cast<const int4*>(dTA), static_cast<const int2*>(dTB));
        CCF_CUDA(cudaGetLastError());  // launch-configuration errors surface here, not as silent no-ops
    } else if (pipe && based_ok) {
        static bool attr = false;  // process-wide function attributes (same on every device)
        if (!attr) {
            CCF_CUDA(cudaFuncSetAttribute(dgemm_pipe_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(dgemm_pipe_smem(128))));
            CCF_CUDA(cudaFuncSetAttribute(dgemm_pipe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(dgemm_pipe_smem(64))));
            attr = true;
        }
        // short-K products (one term of K <= 128): 64-row tiles, 4 CTAs/SM, so tile fills overlap
        const bool small = tstart.empty() && K <= 128;
        const int bm = (small && !std::getenv("CCF_GEMM_BM128")) ? 64 : 128;
        const long items = long(nb) * ((M + bm - 1) / bm) * ((N + 63) / 64);
        // single-term batches: several consecutive items per CTA share one cp.async stream
        static int ipc_env = -1;
        if (ipc_env < 0) {
            const char* e = std::getenv("CCF_GEMM_IPC");
            ipc_env = e ? std::max(1, std::atoi(e)) : 0;
        }
        const int ipc = tstart.empty() ? (ipc_env ? ipc_env : 1) : 1;  // measured: 2 and 4 do not help
        GemmBatch gg = g;
        gg.ipc = ipc;
        const unsigned grid = unsigned((items + ipc - 1) / ipc);
        if (bm == 64) dgemm_pipe_kernel<64><<<grid, 128, dgemm_pipe_smem(64), s>>>(gg);
        else dgemm_pipe_kernel<128><<<grid, 256, dgemm_pipe_smem(128), s>>>(gg);
    } else {
        const dim3 grid(unsigned((N + 63) / 64), unsigned((M + 63) / 64), nb);
        dgemm_batched_kernel<<<grid, 128, 0, s>>>(g);
    }
}

GemmPlan::~GemmPlan() {
    if (dAoff) cudaFree(dAoff);
    if (dTA) cudaFree(dTA);
    if (dTB) cudaFree(dTB);
    if (dBoff) cudaFree(dBoff);
    if (dCoff) cudaFree(dCoff);
    if (dDL) cudaFree(dDL);
    if (dDR) cudaFree(dDR);
    if (dT) cudaFree(dT);
    if (dA) cudaFree(dA);
    if (dB) cudaFree(dB);
    if (dC) cudaFree(dC);
}

// ---------------------------------------------------------------- Pipeline
Pipeline::~Pipeline() {
    for (auto& kv : fdtasks_) cudaFree(kv.second.first);
    for (auto& kv : zrt_) cudaFree(kv.second);
    for (auto& kv : eig_rt_) cudaFree(const_cast<const double**>(kv.second));
}

Pipeline::Pipeline(Ctx& c_) : c(c_), tp(c_), T(c_.tensor_doubles(false)) {
    big_scratch(size_t(3) * T);  // pencil scratch: max(pt_synth 2 pairs x 2, curl 6 pencils per thread)
}

OzPipe& Pipeline::oz() {
    if (!oz_) oz_ = std::make_unique<OzPipe>(*this);
    return *oz_;
}

double* Pipeline::scratch(int i) {
    // mode sharding: the theta stage's inputs / outputs live in the peer-mapped exchange buffer
    if (c.sh.xbuf && i >= 6 && i < 6 + kExchangeTensors) return c.sh.xbuf + size_t(i - 6) * size_t(T);
    while (int(scr_.size()) <= i) scr_.emplace_back();
    if (scr_[size_t(i)].n < size_t(T)) scr_[size_t(i)].alloc(size_t(T));
    return scr_[size_t(i)].p;
}

double* Pipeline::big_scratch(size_t doubles) {
    if (big_.n < doubles) big_.alloc(doubles);
    return big_.p;
}

GemmPlan& Pipeline::gemm(const std::string& key, bool& fresh) {
    auto& slot = gemms_[key];
    fresh = !slot;
    if (fresh) {  // plans allocate and upload: never inside a CUDA-graph capture
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(c.stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
            throw Error(INTERNAL, "GEMM plan first built during graph capture: " + key.substr(0, key.find(':')));
    }
    if (!slot) slot = std::make_unique<GemmPlan>();
    return *slot;
}

static std::string ptr_key(const char* tag, int count, const void* const* a, const void* const* b, const int* cls) {
    std::string k(tag);
    for (int i = 0; i < count; ++i) {
        k += ":" + std::to_string(reinterpret_cast<uintptr_t>(a[i])) + "/" +
             std::to_string(reinterpret_cast<uintptr_t>(b[i]));
        if (cls) k += "/" + std::to_string(cls[i]);
    }
    return k;
}

void Pipeline::dz(const std::vector<const double*>& in, const std::vector<double*>& out) {
    const Geo& g = c.gh;
    DzBatch d{};
    d.g = g;
    d.count = int(in.size());
    for (size_t i = 0; i < in.size(); ++i) {
        d.in[i] = in[i];
        d.out[i] = out[i];
    }
    const long warps = long(g.nslots) * 2 * g.mh * d.count;
    dz_kernel<<<blocks_for(warps * 32, 256), 256, 0, c.stream>>>(d);
    ++c.launches;
}

void Pipeline::pt_synthesize(int count, const double* const* lam, const double* const* gam, double* const* vr,
                             double* const* vt, double* const* vz) {
    const Geo& g = c.gh;
    std::vector<const double*> gi(gam, gam + count);
    std::vector<double*> dzo;
    for (int i = 0; i < count; ++i) dzo.push_back(scratch(20 + i));
    dz(gi, dzo);
    PtSynth a{};
    a.g = g;
    a.count = count;
    for (int i = 0; i < count; ++i) {
        a.lam[i] = lam[i];
        a.gam[i] = gam[i];
        a.dzg[i] = dzo[size_t(i)];
        a.vr[i] = vr[i];
        a.vt[i] = vt[i];
        a.vz[i] = vz[i];
    }
    a.scratch = big_scratch(size_t(count) * g.nslots * g.n * 2 * g.mh);
    a.q = tp.q.p;
    const long n = long(count) * g.nslots * g.n;
    pt_synth_kernel<<<blocks_for(n, 64), 64, 0, c.stream>>>(a);
    ++c.launches;
}

void Pipeline::rz_synth(int count, const double* const* in, const int* cls, double* const* out) {
    const Geo& g = c.gh;
    double* tmp[8];
    for (int i = 0; i < count; ++i) tmp[i] = scratch(24 + i);
    bool fresh;
    GemmPlan& r = gemm(ptr_key("rs", count, reinterpret_cast<const void* const*>(in),
                               reinterpret_cast<const void* const*>(out), cls),
                       fresh);
    GemmPlan& z = gemm(ptr_key("zs", count, reinterpret_cast<const void* const*>(in),
                               reinterpret_cast<const void* const*>(out), cls),
                       fresh);
    if (fresh) {
        for (int t = 0; t < count; ++t)
            for (int s = 0; s < g.nslots; ++s)
                for (int pl = 0; pl < 2; ++pl) {
                    const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                    const int w = (s == g.p / 2) ? -g.p / 2 : s;
                    const int j0 = ((w + cls[t]) % 2 + 2) % 2;
                    r.A.push_back(tp.SrT[j0].p);  // [jr][jj]
                    r.B.push_back(in[t] + off);   // [jj][q]
                    r.C.push_back(tmp[t] + off);  // [jr][q]
                    for (int par = 0; par < 2; ++par) {
                        z.A.push_back(tmp[t] + off + par * g.nh);                // [jr][q of parity par]
                        z.B.push_back(tp.Sz.p + size_t(par) * g.nh * g.nh);     // [q][i]
                        z.C.push_back(out[t] + off + par * g.nh);                // [jr][E | O]
                    }
                }
        r.M = g.mh;
        r.N = g.n;
        r.K = g.mh;
        r.lda = g.mh;
        r.ldb = g.n;
        r.ldc = g.n;
        z.M = g.mh;
        z.N = g.nh;
        z.K = g.nh;
        z.lda = g.n;
        z.ldb = g.nh;
        z.ldc = g.n;
        r.upload();
        z.upload();
    }
    r.launch(c.stream);
    c.gemm_flops += r.flops();
    z.launch(c.stream);
    c.gemm_flops += z.flops();
    c.launches += 2;
}

void Pipeline::rz_analyze(int count, const double* const* in, const int* cls, double* const* out) {
    const Geo& g = c.gh;
    double* tmp[8];
    for (int i = 0; i < count; ++i) tmp[i] = scratch(24 + i);
    bool fresh;
    GemmPlan& z = gemm(ptr_key("za", count, reinterpret_cast<const void* const*>(in),
                               reinterpret_cast<const void* const*>(out), cls),
                       fresh);
    GemmPlan& r = gemm(ptr_key("ra", count, reinterpret_cast<const void* const*>(in),
                               reinterpret_cast<const void* const*>(out), cls),
                       fresh);
    if (fresh) {
        for (int t = 0; t < count; ++t)
            for (int s = 0; s < g.nslots; ++s)
                for (int pl = 0; pl < 2; ++pl) {
                    const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                    const int w = (s == g.p / 2) ? -g.p / 2 : s;
                    const int j0 = ((w + cls[t]) % 2 + 2) % 2;
                    for (int par = 0; par < 2; ++par) {
                        z.A.push_back(in[t] + off + par * g.nh);             // values [jr][E' | O']
                        z.B.push_back(tp.Az.p + size_t(par) * g.nh * g.nh);  // [i][q]
                        z.C.push_back(tmp[t] + off + par * g.nh);            // [jr][q of parity par]
                    }
                    r.A.push_back(tp.ArT[j0].p);  // [jj][jr]
                    r.B.push_back(tmp[t] + off);  // [jr][q]
                    r.C.push_back(out[t] + off);  // [jj][q]
                }
        z.M = g.mh;
        z.N = g.nh;
        z.K = g.nh;
        z.lda = g.n;
        z.ldb = g.nh;
        z.ldc = g.n;
        r.M = g.mh;
        r.N = g.n;
        r.K = g.mh;
        r.lda = g.mh;
        r.ldb = g.n;
        r.ldc = g.n;
        z.upload();
        r.upload();
    }
    z.launch(c.stream);
    c.gemm_flops += z.flops();
    r.launch(c.stream);
    c.gemm_flops += r.flops();
    c.launches += 2;
}

bool Pipeline::theta_quad_ok() const {
    const char* q = std::getenv("CCF_THETA_VARIANT");
    const char* e = std::getenv("CCF_THETA_GENERIC");
    return c.gh.p == 256 && tp.logp >= 0 && !(q && q[0] == '1' && q[1] == '6') && !(e && e[0] == '1');
}

void Pipeline::theta_cross(const double* const* v6, double* const* a3) {
    const Geo& g = c.gh;
    ThetaCross t{};  // (p not a power of two: the generic kernel's dense-DFT path)
    t.g = g;
    t.logp = tp.logp;
    if (g.n % 2) throw Error(DOMAIN_ERROR, "ccf: the z-parity split value layout needs even n");
    int tj = 8;  // points per CTA (pairs of +-z)
    const size_t nbuf = tp.logp < 0 ? 2 : 1;  // the dense-DFT path transforms out of place
    while (tj > 2 && nbuf * 3 * tj * g.p * sizeof(double2) > 100 * 1024) tj /= 2;
    if (nbuf * 3 * tj * g.p * sizeof(double2) > 200 * 1024)
        throw Error(DOMAIN_ERROR, "ccf: p too large for the theta kernel's shared-memory tile");
    t.tj = tj;
    for (int i = 0; i < 6; ++i) t.in[i] = v6[i];
    for (int i = 0; i < 3; ++i) t.out[i] = a3[i];
    t.vquad = val_quad_ ? 1 : 0;
    val_quad_ = false;
    t.tw = reinterpret_cast<const double2*>(tp.tw.p);
    t.twfull = reinterpret_cast<const double2*>(tp.twfull.p);
    // mode sharding: this rank's rows of every slot, each slot in its owner's exchange buffer
    const Shard& sh = c.sh;
    t.row0 = sh.r_lo;
    t.world = sh.world;
    for (int q = 0; q <= kMaxRanks; ++q) t.sb[q] = q <= sh.world ? sh.sb[q] : g.nslots;
    for (int q = 0; q < kMaxRanks; ++q) t.rdelta[q] = sh.rdelta[q];
    const unsigned rows = unsigned(sh.r_hi - sh.r_lo);
    if (!theta_attr_) {
        CCF_CUDA(cudaFuncSetAttribute(theta_cross_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CCF_CUDA(cudaFuncSetAttribute(theta_cross256_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(theta_cross256_smem())));
        CCF_CUDA(cudaFuncSetAttribute(theta_cross256w_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(theta_cross256w_smem(1))));
        CCF_CUDA(cudaFuncSetAttribute(theta_cross256w_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(theta_cross256w_smem(2))));
        CCF_CUDA(cudaFuncSetAttribute(theta_cross512_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(theta_cross512_smem())));
        const char* q = std::getenv("CCF_THETA_PAIRS");  // z-position pairs per CTA of the warp kernel (1 | 2)
        theta_nq_ = (q && q[0] == '1') ? 1 : 2;
        const char* v = std::getenv("CCF_THETA_VARIANT");  // "16": 16-thread FFT kernel
        theta_w_ = !(v && v[0] == '1' && v[1] == '6');
        const char* e = std::getenv("CCF_THETA_GENERIC");
        theta_generic_ = e && e[0] == '1';
        theta_attr_ = true;
    }
    if (sh.sharded() && g.p == 256 && !theta_generic_ && !theta_w_)
        throw Error(CONFIG_ERROR, "theta: the 16-thread variant (CCF_THETA_VARIANT=16) has no sharded form");
    if (t.vquad && !(g.p == 256 && !theta_generic_ && theta_w_))
        throw Error(INTERNAL, "theta: column-quad-major inputs need the warp-per-point p = 256 kernel");
    if (g.p == 256 && !theta_generic_ && theta_w_) {
        const int np = 2 * theta_nq_;
        const dim3 grid(unsigned((g.nh + np - 1) / np), rows);
        if (theta_nq_ == 2)
            theta_cross256w_kernel<2><<<grid, 256, theta_cross256w_smem(2), c.stream>>>(t);
        else
            theta_cross256w_kernel<1><<<grid, 128, theta_cross256w_smem(1), c.stream>>>(t);
    } else if (g.p == 512 && g.nslots == 257 && !theta_generic_) {
        const int tj5 = kTheta512Points;
        const dim3 grid(unsigned((g.nh + tj5 / 2 - 1) / (tj5 / 2)), rows);
        t.tj = tj5;
        theta_cross512_kernel<<<grid, kTheta512Threads, theta_cross512_smem(), c.stream>>>(t);
    } else if (g.p == 256 && !theta_generic_) {
        const int np = theta_cross256_positions();
        const dim3 grid(unsigned((g.nh + np - 1) / np), unsigned(g.mh));
        theta_cross256_kernel<<<grid, theta_cross256_threads(), theta_cross256_smem(), c.stream>>>(t);
    } else {
        const size_t smem = nbuf * 3 * tj * g.p * sizeof(double2);
        const dim3 grid(unsigned((g.nh + tj / 2 - 1) / (tj / 2)), rows);
        theta_cross_kernel<<<grid, 256, smem, c.stream>>>(t);
    }
    ++c.launches;
}

void Pipeline::curl_decompose(const double* ar, const double* at, const double* az, double* out_r, double* out_t,
                              double* out_z, double* lam, double* gam) {
    const Geo& g = c.gh;
    double* dzar = scratch(30);
    double* dzat = scratch(31);
    dz({ar, at}, {dzar, dzat});
    CurlDecomp a{};
    a.g = g;
    a.ar = ar;
    a.at = at;
    a.az = az;
    a.dzar = dzar;
    a.dzat = dzat;
    a.out_r = out_r;
    a.out_t = out_t;
    a.out_z = out_z;
    a.lam = lam;
    a.gam = gam;
    a.scratch = big_scratch(size_t(g.nslots) * g.n * 6 * g.mh);
    a.q = tp.q.p;
    a.hpc = tp.hpc.p;
    a.hpr = tp.hpr.p;
    const long n = long(g.nslots) * g.n;
    curl_decomp_kernel<<<blocks_for(n, 64), 64, 0, c.stream>>>(a);
    ++c.launches;
}

void Pipeline::ensure_composite() {
    if (comp_ready_) return;
    const char* e = std::getenv("CCF_NONLINEAR_PENCIL");
    comp_off_ = e && e[0] == '1';
    if (!comp_off_) {
        SetupTimer tm("composite operators");
        synth_ = build_synth_composite(tp.rt);
        anal_ = build_anal_composite(tp.rt);
        upload(dsynth_, synth_.blocks);
        upload(danal_, anal_.blocks);
    }
    comp_ready_ = true;
}

// Nonlinear term N = curl(v x w) in PT form (proj/src/ptns.cpp:114-149) with every radial step on
// the tensor cores:
//   Z  = z synthesis of (lambda, gamma, dz gamma) of the v and w PT pairs      (DMMA, nh x nh halves)
//   V  = per-slot composite r operators: (r-values of v_r, v_t, v_z, w_r, w_t, w_z) = sum_t C_t Z_t
//   a  = v x w pointwise in theta (register FFTs)
//   Y  = z analysis of (a_r, a_t, a_z, dz a_r, dz a_t)
//   (gamma_N, lambda_N) = per-slot composite r operators (curl + decompose + r analysis) on Y
void Pipeline::ensure_dealias(DevSet* eig) {
    const Geo& g = c.gh;
    const int m = c.m, n = c.n, nh = g.nh, mh = g.mh;
    if (!dealias_ready_) {
        const int jmax = 2 * m / 3, kmax = 2 * n / 3;  // ptns.cpp:101-103
        const long Lz = n - 1;
        auto zan = [&](int k, int kz) {
            const int s = n - 1 - kz;
            const long double eps = (k == 0 || k == n - 1) ? 0.5L : 1.0L;
            const long double ws = (s == 0 || s == n - 1) ? 1.0L : 2.0L;
            return eps / (long double)Lz * ws * cospi_frac(long(k) * s, Lz);
        };
        auto dzm = [&](int k, int kp) -> long double {
            if (kp <= k || ((kp - k) & 1) == 0) return 0.0L;
            return (k == 0 ? 1.0L : 2.0L) * (long double)kp;
        };
        // analysis with the k >= kmax coefficients dropped; dz acts on the masked coefficients
        std::vector<double> A(size_t(n) * nh, 0.0), AD(size_t(n) * nh, 0.0);
        for (int par = 0; par < 2; ++par)
            for (int i = 0; i < nh; ++i)
                for (int q = 0; q < nh; ++q)
                    if (2 * q + par < kmax) A[size_t(par) * nh * nh + size_t(i) * nh + q] = double(2.0L * zan(2 * q + par, nh + i));
        for (int po = 0; po < 2; ++po) {
            const int pi = 1 - po;
            for (int i = 0; i < nh; ++i)
                for (int q = 0; q < nh; ++q) {
                    long double acc = 0.0L;
                    for (int qp = 0; qp < nh; ++qp) {
                        if (2 * qp + pi >= kmax) continue;
                        const long double d = dzm(2 * q + po, 2 * qp + pi);
                        if (d != 0.0L) acc += 2.0L * zan(2 * qp + pi, nh + i) * d;
                    }
                    AD[size_t(po) * nh * nh + size_t(i) * nh + q] = double(acc);
                }
        }
        upload(AzD_, A);
        upload(ADzD_, AD);
        // composite curl / decompose on the r analysis with the j >= jmax coefficients dropped
        RadialTables rt = tp.rt;
        for (int j0 = 0; j0 < 2; ++j0)
            for (int i = 0; i < mh; ++i)
                if (2 * i + j0 >= jmax)
                    for (int jr = 0; jr < mh; ++jr) rt.ArT[j0][size_t(i) * mh + jr] = 0.0;
        analD_ = build_anal_composite(rt);
        upload(danalD_, analD_.blocks);
        dealias_ready_ = true;
    }
    if (eig && eigD_set_ != eig) {  // eigen-coordinate forms (as ensure_eigen)
        const int N = c.N, M = c.M, Np = N + (N & 1);
        eig_AzPD_.alloc(size_t(2) * nh * Np);
        eig_ADzPD_.alloc(size_t(2) * nh * Np);
        GemmPlan gp;
        for (int k0 = 0; k0 < 2; ++k0)
            for (int d = 0; d < 2; ++d) {
                gp.A.push_back((d ? ADzD_.p : AzD_.p) + size_t(k0) * nh * nh);
                gp.B.push_back(eig->dg + eig->host.dg_right[k0]);
                gp.C.push_back((d ? eig_ADzPD_.p : eig_AzPD_.p) + size_t(k0) * nh * Np);
            }
        gp.M = nh; gp.N = N; gp.K = nh; gp.lda = nh; gp.ldb = Np; gp.ldc = Np;
        gp.upload();
        gp.launch(c.stream);
        eig_analD_.alloc(analD_.blocks.size());
        GemmPlan ga;
        for (int s = 0; s < g.nslots; ++s)
            for (const CompositeTerm& ct : analD_.terms[size_t(s)]) {
                ga.A.push_back(eig->dg + eig->host.dg_left[size_t(s)]);
                ga.B.push_back(danalD_.p + ct.off);
                ga.C.push_back(eig_analD_.p + ct.off);
            }
        ga.M = M; ga.N = mh; ga.K = mh; ga.lda = mh; ga.ldb = mh; ga.ldc = mh;
        ga.upload();
        ga.launch(c.stream);
        CCF_CUDA(cudaStreamSynchronize(c.stream));
        eigD_set_ = eig;
    }
}

void Pipeline::nonlinear(const double* lam_v, const double* gam_v, const double* lam_w, const double* gam_w,
                         double* lam_n, double* gam_n, DevSet* eig, bool zpre, bool eigY, bool dealias) {
    ensure_composite();
    if (eig && comp_off_) throw Error(INTERNAL, "nonlinear: eigen-coordinate output needs the composite path");
    if (dealias && comp_off_) throw Error(CONFIG_ERROR, "nonlinear: 2/3 dealiasing needs the composite path");
    if (dealias) ensure_dealias(eig);
    if (comp_off_) {
        if (c.sh.sharded()) throw Error(CONFIG_ERROR, "nonlinear: the pencil path (CCF_NONLINEAR_PENCIL=1) has no sharded form");
        nonlinear_pencil(lam_v, gam_v, lam_w, gam_w, lam_n, gam_n);
        return;
    }
    const Geo& g = c.gh;
    const double* lam[2] = {lam_v, lam_w};
    const double* gam[2] = {gam_v, gam_w};
    double* Z[2][3];
    for (int pr = 0; pr < 2; ++pr)
        for (int x = 0; x < 3; ++x) Z[pr][x] = scratch(3 * pr + x);
    // the velocity's lambda is the vorticity's gamma (velocity_from_vorticity, ptns.cpp:85-91):
    // synthesize that tensor once
    const bool alias = lam_v == gam_w;
    if (alias) Z[0][0] = Z[1][1];
    double* val[6];
    for (int i = 0; i < 6; ++i) val[i] = scratch(6 + i);
    double* av[3] = {scratch(12), scratch(13), scratch(14)};
    double* Y[5];
    for (int i = 0; i < 5; ++i) Y[i] = scratch(15 + i);
    const void* keyp[8] = {lam_v, gam_v, lam_w, gam_w, lam_n, gam_n, nullptr, nullptr};
    const int cls0[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool fresh;
    // ---- z synthesis: 6 tensors, two nh x nh halves per (slot, plane)
    const int acls[8] = {int(alias), 0, 0, 0, 0, 0, 0, 0};
    if (!zpre) {  // zpre: the caller synthesized the six z tensors (eigen_ysynth)
        GemmPlan& zs = gemm(ptr_key("nzs", 4, keyp, keyp, acls), fresh);  // outputs: scratch
        if (fresh) {
            for (int pr = 0; pr < 2; ++pr)
                for (int x = 0; x < 3; ++x) {
                    if (alias && pr == 0 && x == 0) continue;
                    const double* src = x == 0 ? lam[pr] : gam[pr];
                    const double* mat = x == 2 ? tp.DzS.p : tp.Sz.p;
                    for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
                        for (int pl = 0; pl < 2; ++pl) {
                            const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                            for (int po = 0; po < 2; ++po) {
                                const int pi = x == 2 ? 1 - po : po;
                                zs.A.push_back(src + off + pi * g.nh);
                                zs.B.push_back(mat + size_t(po) * g.nh * g.nh);
                                zs.C.push_back(Z[pr][x] + off + po * g.nh);
                            }
                        }
                }
            zs.M = g.mh;
            zs.N = g.nh;
            zs.K = g.nh;
            zs.lda = g.n;
            zs.ldb = g.nh;
            zs.ldc = g.n;
            zs.upload();
        }
        zw_owner_ = nullptr;
        zs.launch(c.stream);
        c.gemm_flops += zs.flops();
    }
    // ---- composite r synthesis -> (r, z)-values of the 6 velocity / vorticity components
    // eigY: the z tensors are Y = Z (QR S_z) in eigen coordinates along r, the synthesis blocks carry QL
    const int ycls[8] = {int(eigY), 0, 0, 0, 0, 0, 0, 0};
    const bool oz_rs = eigY && oz().rsynth(Z, val);  // INT8 tensor cores (ozpipe.cu)
    val_quad_ = oz_rs && theta_quad_ok();             // (rsynth writes that layout exactly then)
    if (!oz_rs) {
    GemmPlan& rs = gemm(ptr_key(eigY ? "nrsY" : "nrs", 4, keyp, keyp, ycls), fresh);  // outputs: scratch
    if (fresh) {
        for (int pr = 0; pr < 2; ++pr)
            for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
                for (int o = 0; o < 6; ++o) {
                    rs.tstart.push_back(int(rs.A.size()));
                    for (const CompositeTerm& ct : synth_.terms[size_t(s)]) {
                        if (ct.out != o) continue;
                        rs.A.push_back((eigY ? dsynth_eig_.p : dsynth_.p) + ct.off);
                        rs.B.push_back(Z[pr][ct.in / 2] + long(s) * g.slot_stride + long(ct.in % 2) * g.plane_stride);
                    }
                    rs.C.push_back(val[3 * pr + o / 2] + long(s) * g.slot_stride + long(o % 2) * g.plane_stride);
                }
        rs.tstart.push_back(int(rs.A.size()));
        rs.M = g.mh;
        rs.N = g.n;
        rs.K = g.mh;
        rs.lda = g.mh;
        rs.ldb = g.n;
        rs.ldc = g.n;
        rs.upload();
    }
    rs.launch(c.stream);
    c.gemm_flops += rs.flops();
    c.launches += 2;
    }
    c.mark("X1_rz_synthesis");
    c.shard_sync();  // every owner's values written, every owner done with the previous step's outputs
    theta_cross(val, av);
    c.shard_sync();  // every rank's rows of the cross product stored
    c.mark("X2_theta_cross");
    // ---- z analysis of a_r, a_t, a_z and (derivative_z folded in) dz a_r, dz a_t
    // eigen mode (eig != nullptr): the z analysis carries PR of the shared modal basis, Y_x half k0 =
    // values * (Az PR)[k0] (N columns, leading dimension 2 Np), see ensure_eigen
    const int Np = c.N + (c.N & 1);
    const int ecls[8] = {eig ? 1 : 0, int(dealias), 0, 0, 0, 0, 0, 0};
    // the analysis side reads only scratch tensors: key it on the outputs
    const void* okeyp[2] = {lam_n, gam_n};
    if (eig && !dealias && oz().analyze(av, Y, lam_n, gam_n)) {  // X3 + C on the INT8 tensor cores (ozpipe.cu)
        c.mark("C_curl_decompose");
        return;
    }
    GemmPlan& za = gemm(ptr_key("nza", 2, okeyp, okeyp, ecls), fresh);
    if (fresh) {
        for (int x = 0; x < 5; ++x) {
            const double* src = av[x < 3 ? x : x - 3];
            const double* mat = dealias ? (eig ? (x >= 3 ? eig_ADzPD_.p : eig_AzPD_.p) : (x >= 3 ? ADzD_.p : AzD_.p))
                                        : (eig ? (x >= 3 ? eig_ADzP_.p : eig_AzP_.p) : (x >= 3 ? tp.ADz.p : tp.Az.p));
            const long mstride = eig ? long(g.nh) * Np : long(g.nh) * g.nh;
            for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
                for (int pl = 0; pl < 2; ++pl) {
                    const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                    for (int po = 0; po < 2; ++po) {
                        const int pi = x >= 3 ? 1 - po : po;
                        za.A.push_back(src + off + pi * g.nh);
                        za.B.push_back(mat + po * mstride);
                        za.C.push_back(eig ? Y[x] + long(s) * g.slot_stride + long(pl) * g.mh * 2 * Np + po * Np
                                           : Y[x] + off + po * g.nh);
                    }
                }
        }
        za.M = g.mh;
        za.N = eig ? c.N : g.nh;
        za.K = g.nh;
        za.lda = g.n;
        za.ldb = eig ? Np : g.nh;
        za.ldc = eig ? 2 * Np : g.n;
        za.upload();
    }
    za.launch(c.stream);
    c.gemm_flops += za.flops();
    c.launches += 1;
    c.mark("X3_rz_analysis");
    // ---- composite curl + pt_decompose + r analysis -> (gamma_N, lambda_N)
    // eigen mode: blocks PL_P A_t (M x mh) and output in the eigen layout (M x 2 Np per slot, plane)
    GemmPlan& ra = gemm(ptr_key("nra", 2, okeyp, okeyp, ecls), fresh);
    if (fresh) {
        const CompositeSet& an = dealias ? analD_ : anal_;
        const double* blocks = dealias ? (eig ? eig_analD_.p : danalD_.p) : (eig ? eig_anal_.p : danal_.p);
        for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
            for (int o = 0; o < 4; ++o) {
                ra.tstart.push_back(int(ra.A.size()));
                for (const CompositeTerm& ct : an.terms[size_t(s)]) {
                    if (ct.out != o) continue;
                    ra.A.push_back(blocks + ct.off);
                    ra.B.push_back(eig ? Y[ct.in / 2] + long(s) * g.slot_stride + long(ct.in % 2) * g.mh * 2 * Np
                                       : Y[ct.in / 2] + long(s) * g.slot_stride + long(ct.in % 2) * g.plane_stride);
                }
                ra.C.push_back(eig ? (o < 2 ? gam_n : lam_n) + eig_off(s, o % 2, 0)
                                   : (o < 2 ? gam_n : lam_n) + long(s) * g.slot_stride + long(o % 2) * g.plane_stride);
            }
        ra.tstart.push_back(int(ra.A.size()));
        ra.M = eig ? c.M : g.mh;
        ra.N = eig ? 2 * Np : g.n;
        ra.K = g.mh;
        ra.lda = g.mh;
        ra.ldb = eig ? 2 * Np : g.n;
        ra.ldc = eig ? 2 * Np : g.n;
        ra.upload();
    }
    ra.launch(c.stream);
    c.gemm_flops += ra.flops();
    c.launches += 1;
    if (dealias) {  // |w| >= 2 (p/2) / 3: the whole slot of N is zero (a is masked, curl / decompose act per slot)
        const int s0 = std::max(2 * (c.p / 2) / 3, c.sh.s_lo), s1 = c.sh.s_hi;
        if (s0 < s1) {
            const int Np = c.N + (c.N & 1);
            const long per = eig ? 2L * c.M * 2 * Np : g.slot_stride;
            const long off = eig ? eig_off(s0, 0, 0) : long(s0) * g.slot_stride;
            for (double* t : {lam_n, gam_n})
                CCF_CUDA(cudaMemsetAsync(t + off, 0, sizeof(double) * size_t(per) * size_t(s1 - s0), c.stream));
        }
    }
    c.mark("C_curl_decompose");
}

void Pipeline::nonlinear_pencil(const double* lam_v, const double* gam_v, const double* lam_w, const double* gam_w,
                                double* lam_n, double* gam_n) {
    // proj/src/ptns.cpp:114-149
    zw_owner_ = nullptr;
    double* comp[6];
    for (int i = 0; i < 6; ++i) comp[i] = scratch(i);
    const double* lam[2] = {lam_v, lam_w};
    const double* gam[2] = {gam_v, gam_w};
    double* vr[2] = {comp[0], comp[3]};
    double* vt[2] = {comp[1], comp[4]};
    double* vz[2] = {comp[2], comp[5]};
    pt_synthesize(2, lam, gam, vr, vt, vz);
    c.mark("V_pt_synthesize");
    double* val[6];
    for (int i = 0; i < 6; ++i) val[i] = scratch(6 + i);
    const int cls6[6] = {1, 1, 0, 1, 1, 0};
    rz_synth(6, comp, cls6, val);
    c.mark("X1_rz_synthesis");
    double* av[3] = {scratch(12), scratch(13), scratch(14)};
    theta_cross(val, av);
    c.mark("X2_theta_cross");
    double* ac[3] = {scratch(15), scratch(16), scratch(17)};
    const int cls3[3] = {1, 1, 0};
    rz_analyze(3, av, cls3, ac);
    c.mark("X3_rz_analysis");
    curl_decompose(ac[0], ac[1], ac[2], nullptr, nullptr, nullptr, lam_n, gam_n);
    c.mark("C_curl_decompose");
}

void Pipeline::poisson(const double* f, double w, double* u) {
    DevSet& set = c.set(false, true, 1.0);
    const double* src[1] = {f};
    const double ww[1] = {w};
    modal_solve(set, false, 1, src, ww, 1, nullptr, nullptr, 0, u, nullptr);
}

// Z[task] *= w * RT[task] (M x N, leading dimension ld) - eigen-coordinate RHS of a modal solve
__global__ void zscale_kernel(double* __restrict__ Z, long per, const double* const* __restrict__ rt, int M, int N,
                              int ld, double w) {
    const int task = blockIdx.x;
    double* z = Z + long(task) * per;
    const double* r = rt[task];
    for (int e = threadIdx.x; e < M * N; e += blockDim.x) {
        const int i = e / N, j = e - i * N;
        z[long(i) * ld + j] *= w * __ldg(r + long(i) * ld + j);
    }
}

// Poisson solve of w * lambda_omega when lambda_omega was produced by the previous Helmholtz solve in
// the shared modal basis (modal.hpp SizeOps): with u = QL Z_H QR, PL_P u PR = Z_H exactly
// (PL_P QL = I, QR PR = I), so the first two products drop out: Z_P = w Z_H .* RT_P, then
// T3 = QL Z_P, u_P = T3 QR. Returns false if the chain plans of this set do not exist yet.
bool Pipeline::modal_solve_from_z(DevSet& set, double w, double* out) {
    if (!set.host.has_diag || !set.dg || !dZ_.p) return false;
    const void* keyp[1] = {&set};
    const int ci[1] = {1};  // half spectrum, one tensor
    const std::string k3 = ptr_key("d3", 1, keyp, keyp, ci), k4 = ptr_key("d4", 1, keyp, keyp, ci);
    auto i3 = gemms_.find(k3), i4 = gemms_.find(k4);
    if (i3 == gemms_.end() || i4 == gemms_.end()) return false;
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, mh = g.mh, nh = g.nh;
    const int Mp = M + (M & 1), Np = N + (N & 1);
    const size_t per = std::max(size_t(mh) * Np, size_t(M) * std::max(nh, Np));
    const int ntask = g.nslots * 4;
    auto it = zrt_.find(&set);
    if (it == zrt_.end()) {
        auto even = [](long x) { return x + (x & 1); };
        std::vector<const double*> rt;
        for (int s = 0; s < g.nslots; ++s)
            for (int k0 = 0; k0 < 2; ++k0)
                for (int pl = 0; pl < 2; ++pl) {
                    const long PLo = set.host.dg_left[size_t(s)], QLo = PLo + long(M) * mh, LAMo = QLo + long(mh) * Mp;
                    rt.push_back(set.dg + LAMo + even(M) + long(k0) * long(M) * Np);
                }
        const double** d = nullptr;
        CCF_CUDA(cudaMalloc(&d, rt.size() * sizeof(void*)));
        CCF_H2D(d, rt.data(), rt.size() * sizeof(void*));
        it = zrt_.emplace(&set, d).first;
    }
    zscale_kernel<<<ntask, 256, 0, c.stream>>>(dZ_.p, long(per), it->second, M, N, Np, w);
    ++c.launches;
    GemmPlan& g3 = *i3->second;
    GemmPlan& g4 = *i4->second;
    g3.launch(c.stream);
    c.gemm_flops += g3.flops();
    g4.launch(c.stream, nullptr, nullptr, out, out);
    c.gemm_flops += g4.flops();
    c.launches += 2;
    z_owner_ = nullptr;  // dZ_ was scaled in place
    return true;
}

// Fast diagonalization (diag.hpp) per real sub-problem (tensor t, slot s, k-parity k0, plane):
//   T1 = PL[s] f          (M x nh)      f = sum_i w_t[i] src_t[i], rows jj, half row k0
//   Z  = (T1 PR[k0]) ./ (lam[s]_i + mu[k0]_j)
//   T3 = QL[s] Z          (mh x N)
//   u  = T3 QR[k0]        (mh x nh)  written in place into the output tensor
void Pipeline::modal_solve(DevSet& set, bool full, int ntensor, const double* const* src0, const double* w0, int n0,
                           const double* const* src1, const double* w1, int n1, double* out0, double* out1,
                           const char* rhs_mark) {
    last_z_valid_ = false;
    z_owner_ = nullptr;
    if (!set.host.has_diag || !set.dg) {
        c.run_adi(set, full, ntensor, src0, w0, n0, src1, w1, n1, out0, out1);
        return;
    }
    const Geo& g = c.geo(full);
    const int M = c.M, N = c.N, mh = g.mh, nh = g.nh;
    const long Tt = c.tensor_doubles(full);
    const double* const* srcs[2] = {src0, src1};
    const double* ws[2] = {w0, w1};
    const int ns[2] = {n0, n1};
    double* outs[2] = {out0, out1};
    const double* f[2] = {nullptr, nullptr};
    double alpha = 1.0;
    for (int t = 0; t < ntensor; ++t) {  // RHS combination (BDF history + kappa * IMEX), timestep.cpp:41-73
        if (ntensor == 1 && ns[t] == 1) {  // single source: its weight rides on the first product
            f[t] = srcs[t][0];
            alpha = ws[t][0];
            continue;
        }
        if (fcomb_[t].n < size_t(Tt)) fcomb_[t].alloc(size_t(Tt));
        Combo cb{};
        for (int i = 0; i < ns[t]; ++i) {
            cb.src[i] = srcs[t][i];
            cb.w[i] = ws[t][i];
        }
        cb.nsrc = ns[t];
        cb.out = fcomb_[t].p;
        cb.n = Tt;
        combo_kernel<<<std::min<long>(4736, (Tt + 255) / 256), 256, 0, c.stream>>>(cb);
        ++c.launches;
        f[t] = fcomb_[t].p;
    }
    // scratch sized once for the largest task list of either slot table (cached GEMM plans hold
    // pointers into it, so it must never be reallocated); leading dimensions rounded up to even
    const int Mp = M + (M & 1), Np = N + (N & 1);
    const size_t per = std::max(size_t(mh) * Np, size_t(M) * std::max(nh, Np));
    if (!dT1_.p) {
        const size_t cap = per * size_t(3 * std::max(c.gh.nslots, c.gf.nslots) * 4);  // up to 3 tensors of sub-problems
        dT1_.alloc(cap);
        dZ_.alloc(cap);
        dT3_.alloc(cap);
    }
    const void* keyp[1] = {&set};
    const int ci[1] = {int(full) * 16 + ntensor};
    // fused path: all four products per sub-problem in one CTA (tile edge 128)
    if (!fd_attr_) {
        // the fused kernel (one CTA per sub-problem, intermediates in shared memory) runs at 1 CTA/SM
        // and measured 0.47 / 0.76 ms (P / H) against 0.41 / 0.68 ms for the four pipelined GEMMs at
        // 2 CTAs/SM, so it is opt-in (CCF_FDSOLVE_FUSED=1)
        const char* e = std::getenv("CCF_FDSOLVE_FUSED");
        fd_fused_ = e && e[0] == '1';
        if (fd_fused_) CCF_CUDA(cudaFuncSetAttribute(fdsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     int(fdsolve_smem())));
        fd_attr_ = true;
    }
    const bool aligned = (reinterpret_cast<uintptr_t>(f[0]) % 16 == 0) && (ntensor < 2 || reinterpret_cast<uintptr_t>(f[1]) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(out0) % 16 == 0) && (ntensor < 2 || reinterpret_cast<uintptr_t>(out1) % 16 == 0);
    if (fd_fused_ && aligned && M <= 128 && N <= 128 && mh <= 128 && nh <= 128 && g.n % 2 == 0 && nh % 2 == 0) {
        const std::string key = ptr_key("fd", 1, keyp, keyp, ci);
        auto it = fdtasks_.find(key);
        if (it == fdtasks_.end()) {
            std::vector<FdTask> tv;
            auto even = [](long x) { return x + (x & 1); };
            const double* dg = set.dg;
            for (int t = 0; t < ntensor; ++t)
                for (int s = 0; s < g.nslots; ++s)
                    for (int k0 = 0; k0 < 2; ++k0)
                        for (int pl = 0; pl < 2; ++pl) {
                            const long PLo = set.host.dg_left[size_t(s)], QLo = PLo + long(M) * mh,
                                       LAMo = QLo + long(mh) * Mp, RTo = LAMo + even(M) + long(k0) * long(M) * Np;
                            const long PRo = set.host.dg_right[k0], QRo = PRo + long(nh) * Np;
                            FdTask tk{};
                            tk.t = t;
                            tk.off = long(s) * g.slot_stride + long(pl) * g.plane_stride + long(k0) * nh;
                            tk.PL = dg + PLo;
                            tk.PR = dg + PRo;
                            tk.RT = dg + RTo;
                            tk.QL = dg + QLo;
                            tk.QR = dg + QRo;
                            tv.push_back(tk);
                        }
            FdTask* d = nullptr;
            CCF_CUDA(cudaMalloc(&d, tv.size() * sizeof(FdTask)));
            CCF_H2D(d, tv.data(), tv.size() * sizeof(FdTask));
            it = fdtasks_.emplace(key, std::make_pair(d, int(tv.size()))).first;
        }
        if (rhs_mark) c.mark(rhs_mark);
        FdSolve fp{};
        fp.tasks = it->second.first;
        fp.fbase[0] = f[0];
        fp.fbase[1] = ntensor > 1 ? f[1] : f[0];
        fp.obase[0] = out0;
        fp.obase[1] = ntensor > 1 ? out1 : out0;
        fp.M = M;
        fp.N = N;
        fp.mh = mh;
        fp.nh = nh;
        fp.ldf = g.n;
        fp.ldpr = Np;
        fp.ldql = Mp;
        fp.ldrt = Np;
        fp.alpha = alpha;
        fdsolve_kernel<<<it->second.second, 256, fdsolve_smem(), c.stream>>>(fp);
        ++c.launches;
        last_z_valid_ = false;  // the fused kernel keeps Z on chip
        c.gemm_flops += 2.0 * double(it->second.second) *
                        (double(M) * nh * mh + double(M) * N * nh + double(mh) * N * M + double(mh) * nh * N);
        return;
    }
    bool fresh;
    GemmPlan& g1 = gemm(ptr_key("d1", 1, keyp, keyp, ci), fresh);
    GemmPlan& g2 = gemm(ptr_key("d2", 1, keyp, keyp, ci), fresh);
    GemmPlan& g3 = gemm(ptr_key("d3", 1, keyp, keyp, ci), fresh);
    GemmPlan& g4 = gemm(ptr_key("d4", 1, keyp, keyp, ci), fresh);
    if (fresh) {
        const double* dg = set.dg;
        auto even = [](long x) { return x + (x & 1); };
        long task = 0;
        for (int t = 0; t < ntensor; ++t)
            for (int s = 0; s < g.nslots; ++s)
                for (int k0 = 0; k0 < 2; ++k0)
                    for (int pl = 0; pl < 2; ++pl, ++task) {
                        // dg layout (modal.cpp): left [PL M x mh | QL mh x Mp | lam | 1/(lam+mu) x2], right [PR nh x Np | QR N x nh | mu]
                        const long PLo = set.host.dg_left[size_t(s)], QLo = PLo + long(M) * mh,
                                   LAMo = QLo + long(mh) * Mp, RTo = LAMo + even(M) + long(k0) * long(M) * Np;
                        const long PRo = set.host.dg_right[k0], QRo = PRo + long(nh) * Np;
                        const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride + long(k0) * nh;
                        const long rel = (long(t) << kBaseShift) + off;  // base t = f_t / out_t at launch
                        double* T1 = dT1_.p + size_t(task) * per;
                        double* Z = dZ_.p + size_t(task) * per;
                        double* T3 = dT3_.p + size_t(task) * per;
                        g1.A.push_back(dg + PLo);                      // PL  M x mh
                        g1.B.push_back(nullptr);
                        g1.Boff.push_back(rel);                        // f   mh x nh (ld n)
                        g1.C.push_back(T1);                            // T1  M x nh
                        g2.A.push_back(T1);
                        g2.B.push_back(dg + PRo);                      // PR  nh x N (ld Np)
                        g2.C.push_back(Z);                             // Z   M x N (ld Np)
                        g2.DL.push_back(dg + RTo);                     // 1 / (lambda_i + mu_j)
                        g2.DR.push_back(dg + RTo);
                        g3.A.push_back(dg + QLo);                      // QL  mh x M (ld Mp)
                        g3.B.push_back(Z);
                        g3.C.push_back(T3);                            // T3  mh x N (ld Np)
                        g4.A.push_back(T3);
                        g4.B.push_back(dg + QRo);                      // QR  N x nh
                        g4.Coff.push_back(rel);                        // u   mh x nh (ld n)
                    }
        g1.M = M; g1.N = nh; g1.K = mh; g1.lda = mh; g1.ldb = g.n; g1.ldc = nh;
        g2.M = M; g2.N = N; g2.K = nh; g2.lda = nh; g2.ldb = Np; g2.ldc = Np; g2.ldd = Np;
        g3.M = mh; g3.N = N; g3.K = M; g3.lda = Mp; g3.ldb = Np; g3.ldc = Np;
        g4.M = mh; g4.N = nh; g4.K = N; g4.lda = Np; g4.ldb = nh; g4.ldc = g.n;
        g1.upload();
        g2.upload();
        g3.upload();
        g4.upload();
    }
    if (rhs_mark) c.mark(rhs_mark);
    g1.alpha = alpha;
    g1.launch(c.stream, f[0], f[1]);
    c.gemm_flops += g1.flops();
    g2.launch(c.stream);
    c.gemm_flops += g2.flops();
    g3.launch(c.stream);
    c.gemm_flops += g3.flops();
    g4.launch(c.stream, nullptr, nullptr, out0, out1);
    c.gemm_flops += g4.flops();
    last_z_valid_ = !full;  // dZ_ holds Z of every task (half-spectrum task order) until the next solve
    c.launches += 4;
}

// ---------------------------------------------------------------- eigen-coordinate NS state
// Eigen layout (one tensor): E[slot][plane][i < M][k0 * Np + j] (leading dimension 2 Np, j < N used);
// Z = PL_P u PR in the modal basis shared by every solver set (modal.hpp SizeOps). With
// PL_H = -(1/s) PL_P for a Helmholtz set of scale s and PL_P QL = I, QR PR = I:
//   Poisson RHS   PL_P (-lambda_omega) PR = -Z_lambda
//   Helmholtz RHS PL_H (sum b_i omega_i + kappa sum e_i N_i) PR = -(1/s) (sum b_i Z_i + kappa sum e_i N~_i)
// so the solves reduce to (RHS .* RT) followed by the back transform u = QL Z QR, and the nonlinear
// term is produced directly as N~ = PL_P N PR (PR folded into the z analysis, PL_P into the composite
// curl/decompose blocks).
long Pipeline::eig_off(int s, int pl, int k0) const {
    const int Np = c.N + (c.N & 1);
    return (long(s) * 2 + pl) * long(c.M) * 2 * Np + long(k0) * Np;
}

template <int NS>
__global__ void __launch_bounds__(128) eigen_rhs_kernel(EigRhs a) {
    // one eigen-layout row (t, s, pl, i) per block row; 2 Np columns over the threads (16-byte pairs)
    const long rows = long(a.ntensor) * a.nslots * 2 * a.M;
    const int ld = 2 * a.Np, pairs = a.Np;  // 2 Np / 2
    for (long row = blockIdx.x; row < rows; row += gridDim.x) {
        const int t = int(row / (long(a.nslots) * 2 * a.M));
        const long rr = row - long(t) * a.nslots * 2 * a.M;  // (s * 2 + pl) * M + i
        const int i = int(rr % a.M);
        const int s = a.slo + int(rr / (2L * a.M));
        const long base = (rr + long(a.slo) * 2 * a.M) * ld;
        for (int pc = threadIdx.x; pc < pairs; pc += blockDim.x) {
            const int col = 2 * pc;
            const int k0 = col >= a.Np ? 1 : 0, j = col - k0 * a.Np;
            double2 v[NS];  // all source loads in flight before the combination
#pragma unroll
            for (int q = 0; q < NS; ++q) v[q] = __ldg(reinterpret_cast<const double2*>(a.src[t][q] + base + col));
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                acc.x = fma(a.w[q], v[q].x, acc.x);
                acc.y = fma(a.w[q], v[q].y, acc.y);
            }
            const double2 r = __ldg(reinterpret_cast<const double2*>(a.rt[s * 2 + k0] + long(i) * a.Np + j));
            double2 o;
            o.x = j < a.N ? a.factor * acc.x * r.x : 0.0;
            o.y = j + 1 < a.N ? a.factor * acc.y * r.y : 0.0;
            *reinterpret_cast<double2*>(a.out[t] + base + col) = o;
            if (a.outp && t == 0) {
                const double2 rp = __ldg(reinterpret_cast<const double2*>(a.rtp[s * 2 + k0] + long(i) * a.Np + j));
                *reinterpret_cast<double2*>(a.outp + base + col) = make_double2(-o.x * rp.x, -o.y * rp.y);
            }
            if (a.flag && !(isfinite(o.x) && isfinite(o.y))) *a.flag = 1;
        }
    }
}

// eigen_rhs_kernel fused with the back transform's row split (INT8 product path): one warp per half row
// (t, s, pl, i, k0), four columns per lane; besides the fp64 outputs it writes each half row as a row of the
// digit panel ((s - slo) 2 + pl) 2 + k0 of its tensor (ozaki.hpp: 48-bit fixed point relative to the row max,
// the same digits the row-split kernel would produce), so the split pass of the back transform disappears
template <int NS>
__global__ void __launch_bounds__(128) eigen_rhs_pan_kernel(EigRhs a) {
    const int lane = threadIdx.x & 31;
    const long hrows = long(a.ntensor) * a.nslots * 2 * a.M * 2;
    const int ld = 2 * a.Np;
    auto panel_row = [&](const double (&o)[4], int t, long pidx, int i) {  // digits of one panel row
        oz_warp_row(o, a.pan[t] + pidx * (size_t(kOzS) * 128 * kOzK), 128 * kOzK, i, a.psc[t] + pidx * 128 + i);
    };
    for (long hr = long(blockIdx.x) * 4 + (threadIdx.x >> 5); hr < hrows; hr += long(gridDim.x) * 4) {
        const int k0 = int(hr & 1);
        const long row = hr >> 1;
        const int t = int(row / (long(a.nslots) * 2 * a.M));
        const long rr = row - long(t) * a.nslots * 2 * a.M;  // ((s - slo) * 2 + pl) * M + i
        const int i = int(rr % a.M);
        const long spl = rr / a.M;                             // (s - slo) * 2 + pl
        const int s = a.slo + int(spl >> 1);
        const long base = (rr + long(a.slo) * 2 * a.M) * ld + long(k0) * a.Np;
        const int j = 4 * lane;
        double2 v[NS][2];
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            v[q][0] = __ldg(reinterpret_cast<const double2*>(a.src[t][q] + base + j));
            v[q][1] = __ldg(reinterpret_cast<const double2*>(a.src[t][q] + base + j + 2));
        }
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            acc[0] = fma(a.w[q], v[q][0].x, acc[0]);
            acc[1] = fma(a.w[q], v[q][0].y, acc[1]);
            acc[2] = fma(a.w[q], v[q][1].x, acc[2]);
            acc[3] = fma(a.w[q], v[q][1].y, acc[3]);
        }
        const double* rt = a.rt[s * 2 + k0] + long(i) * a.Np + j;
        const double2 r0 = __ldg(reinterpret_cast<const double2*>(rt)), r1 = __ldg(reinterpret_cast<const double2*>(rt + 2));
        const double rv[4] = {r0.x, r0.y, r1.x, r1.y};
        double o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] = j + u < a.N ? a.factor * acc[u] * rv[u] : 0.0;
        *reinterpret_cast<double2*>(a.out[t] + base + j) = make_double2(o[0], o[1]);
        *reinterpret_cast<double2*>(a.out[t] + base + j + 2) = make_double2(o[2], o[3]);
        if (a.flag && !(isfinite(o[0]) && isfinite(o[1]) && isfinite(o[2]) && isfinite(o[3]))) *a.flag = 1;
        const long pidx = spl * 2 + k0;
        panel_row(o, t, pidx, i);
        if (a.outp && t == 0) {
            const double* rtp = a.rtp[s * 2 + k0] + long(i) * a.Np + j;
            const double2 p0 = __ldg(reinterpret_cast<const double2*>(rtp)), p1 = __ldg(reinterpret_cast<const double2*>(rtp + 2));
            const double op[4] = {-o[0] * p0.x, -o[1] * p0.y, -o[2] * p1.x, -o[3] * p1.y};
            *reinterpret_cast<double2*>(a.outp + base + j) = make_double2(op[0], op[1]);
            *reinterpret_cast<double2*>(a.outp + base + j + 2) = make_double2(op[2], op[3]);
            panel_row(op, 2, pidx, i);
        }
    }
}

void Pipeline::ensure_eigen(DevSet& pset) {
    if (eig_set_ == &pset) return;
    SetupTimer tm("eigen-coordinate operators");
    ensure_composite();
    if (comp_off_ || !pset.host.has_diag || !pset.dg) throw Error(INTERNAL, "ensure_eigen: no shared modal basis");
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, mh = g.mh, nh = g.nh;
    const int Mp = M + (M & 1), Np = N + (N & 1);
    (void)Mp;
    auto even = [](long x) { return x + (x & 1); };
    // (Az PR)[k0], (ADz PR)[k0]: nh x Np each
    eig_AzP_.alloc(size_t(2) * nh * Np);
    eig_ADzP_.alloc(size_t(2) * nh * Np);
    {
        GemmPlan gp;
        for (int k0 = 0; k0 < 2; ++k0)
            for (int d = 0; d < 2; ++d) {
                gp.A.push_back((d ? tp.ADz.p : tp.Az.p) + size_t(k0) * nh * nh);
                gp.B.push_back(pset.dg + pset.host.dg_right[k0]);
                gp.C.push_back((d ? eig_ADzP_.p : eig_AzP_.p) + size_t(k0) * nh * Np);
            }
        gp.M = nh; gp.N = N; gp.K = nh; gp.lda = nh; gp.ldb = Np; gp.ldc = Np;
        CCF_CUDA(cudaMemsetAsync(eig_AzP_.p, 0, eig_AzP_.n * sizeof(double), c.stream));
        CCF_CUDA(cudaMemsetAsync(eig_ADzP_.p, 0, eig_ADzP_.n * sizeof(double), c.stream));
        gp.upload();
        gp.launch(c.stream);
        CCF_CUDA(cudaStreamSynchronize(c.stream));
    }
    // PL_P[s] A_t for every composite curl/decompose block (M x mh, ld mh)
    eig_anal_.alloc(anal_.blocks.size());
    {
        GemmPlan gp;
        for (int s = 0; s < g.nslots; ++s)
            for (const CompositeTerm& ct : anal_.terms[size_t(s)]) {
                gp.A.push_back(pset.dg + pset.host.dg_left[size_t(s)]);
                gp.B.push_back(danal_.p + ct.off);
                gp.C.push_back(eig_anal_.p + ct.off);
            }
        gp.M = M; gp.N = mh; gp.K = mh; gp.lda = mh; gp.ldb = mh; gp.ldc = mh;
        CCF_CUDA(cudaMemsetAsync(eig_anal_.p, 0, eig_anal_.n * sizeof(double), c.stream));
        gp.upload();
        gp.launch(c.stream);
        CCF_CUDA(cudaStreamSynchronize(c.stream));
    }
    // C_t QL[s] for every composite synthesis block (mh x M in the mh x mh slot, pad column zero):
    // sum_t C_t (u_t S_z) = sum_t (C_t QL) (Z_t QS), see eigen_ysynth
    dsynth_eig_.alloc(synth_.blocks.size());
    {
        GemmPlan gp;
        for (int s = 0; s < g.nslots; ++s)
            for (const CompositeTerm& ct : synth_.terms[size_t(s)]) {
                gp.A.push_back(dsynth_.p + ct.off);
                gp.B.push_back(pset.dg + pset.host.dg_left[size_t(s)] + long(M) * mh);  // QL mh x M (ld Mp)
                gp.C.push_back(dsynth_eig_.p + ct.off);
            }
        gp.M = mh; gp.N = M; gp.K = mh; gp.lda = mh; gp.ldb = Mp; gp.ldc = mh;
        gp.upload();
        gp.launch(c.stream);
        CCF_CUDA(cudaStreamSynchronize(c.stream));
    }
    // QS[k0] = QR[k0] Sz[k0], QD[k0] = QR[k0] DzS[1 - k0] (N x nh): u_k0 Sz = T3 QS, the dz synthesis
    // of the same half lands in value half 1 - k0
    eig_QS_.alloc(size_t(2) * N * nh);
    eig_QD_.alloc(size_t(2) * N * nh);
    {
        GemmPlan gp;
        for (int k0 = 0; k0 < 2; ++k0)
            for (int d = 0; d < 2; ++d) {
                gp.A.push_back(pset.dg + pset.host.dg_right[k0] + long(nh) * Np);  // QR N x nh
                gp.B.push_back(d ? tp.DzS.p + size_t(1 - k0) * nh * nh : tp.Sz.p + size_t(k0) * nh * nh);
                gp.C.push_back((d ? eig_QD_.p : eig_QS_.p) + size_t(k0) * N * nh);
            }
        gp.M = N; gp.N = nh; gp.K = nh; gp.lda = nh; gp.ldb = nh; gp.ldc = nh;
        gp.upload();
        gp.launch(c.stream);
        CCF_CUDA(cudaStreamSynchronize(c.stream));
    }
    eig_set_ = &pset;
    (void)even;
}

// z-synthesized tensors in eigen coordinates along r: for each tensor t and requested output,
// Y_S = Z_t QS[k0] into value half k0, Y_D = Z_t QD[k0] into half 1 - k0 (M rows of each mh-row
// block, ld n). u_t S_z = QL Y_S, so the composite synthesis with the QL-folded blocks
// (dsynth_eig_) consumes Y directly: one product per output instead of QL Z then T3 QS.
// Z_t is base-relative (ring slots): bases z[0..ntensor).
void Pipeline::eigen_ysynth(int ntensor, const double* const* z, double* const* outS, double* const* outD) {
    if (oz().ysynth(ntensor, z, outS, outD)) return;  // INT8 tensor cores (ozpipe.cu)
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, nh = g.nh;
    const int Np = N + (N & 1);
    const void* okey[6] = {outS[0], outD[0], ntensor > 1 ? outS[1] : nullptr, ntensor > 1 ? outD[1] : nullptr,
                           ntensor > 2 ? outS[2] : nullptr, ntensor > 2 ? outD[2] : nullptr};
    const int ci6[6] = {ntensor, ntensor, ntensor, ntensor, ntensor, ntensor};
    bool fresh;
    GemmPlan& ys = gemm(ptr_key("eys", 6, okey, okey, ci6), fresh);
    if (fresh) {
        for (int t = 0; t < ntensor; ++t)
            for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
                for (int k0 = 0; k0 < 2; ++k0)
                    for (int pl = 0; pl < 2; ++pl) {
                        const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                        const long zo = (long(t) << kBaseShift) + eig_off(s, pl, k0);  // Z_t: M x N (ld 2 Np)
                        if (outS[t]) {
                            ys.A.push_back(nullptr);
                            ys.Aoff.push_back(zo);
                            ys.B.push_back(eig_QS_.p + size_t(k0) * N * nh);
                            ys.C.push_back(outS[t] + off + long(k0) * nh);
                        }
                        if (outD[t]) {
                            ys.A.push_back(nullptr);
                            ys.Aoff.push_back(zo);
                            ys.B.push_back(eig_QD_.p + size_t(k0) * N * nh);
                            ys.C.push_back(outD[t] + off + long(1 - k0) * nh);
                        }
                    }
        ys.M = M; ys.N = nh; ys.K = N; ys.lda = 2 * Np; ys.ldb = nh; ys.ldc = g.n;
        ys.kzero = Np - N;  // Z's pad column is zero (eigen_rhs / to_eigen)
        ys.upload();
    }
    ys.launch(c.stream, z[0], ntensor > 1 ? z[1] : z[0], nullptr, nullptr, ntensor > 2 ? z[2] : z[0]);
    c.gemm_flops += ys.flops();
    ++c.launches;
}

const double* const* Pipeline::eig_rt(DevSet& set) {
    auto it = eig_rt_.find(&set);
    if (it != eig_rt_.end()) return it->second;
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, mh = g.mh;
    const int Mp = M + (M & 1), Np = N + (N & 1);
    auto even = [](long x) { return x + (x & 1); };
    std::vector<const double*> rt;
    for (int s = 0; s < g.nslots; ++s)
        for (int k0 = 0; k0 < 2; ++k0) {
            const long PLo = set.host.dg_left[size_t(s)], QLo = PLo + long(M) * mh, LAMo = QLo + long(mh) * Mp;
            rt.push_back(set.dg + LAMo + even(M) + long(k0) * long(M) * Np);
        }
    const double** d = nullptr;
    CCF_CUDA(cudaMalloc(&d, rt.size() * sizeof(void*)));
    CCF_H2D(d, rt.data(), rt.size() * sizeof(void*));
    eig_rt_.emplace(&set, d);
    return d;
}

void Pipeline::eigen_rhs(DevSet& set, int ntensor, const double* const* s0, const double* const* s1, const double* w,
                         int nsrc, double factor, double* out0, double* out1, double* outp, DevSet* pset,
                         int* flag, bool panels) {
    EigRhs a{};
    if (outp) {
        a.outp = outp;
        a.rtp = eig_rt(*pset);
    }
    a.flag = flag;
    for (int q = 0; q < nsrc; ++q) {
        a.src[0][q] = s0[q];
        a.src[1][q] = ntensor > 1 ? s1[q] : s0[q];
        a.w[q] = w[q];
    }
    a.nsrc = nsrc;
    a.ntensor = ntensor;
    a.out[0] = out0;
    a.out[1] = ntensor > 1 ? out1 : out0;
    a.rt = eig_rt(set);
    a.factor = factor;
    a.M = c.M;
    a.N = c.N;
    a.Np = c.N + (c.N & 1);
    a.slo = c.sh.s_lo;  // mode sharding: the owned slots only
    a.nslots = c.sh.s_hi - c.sh.s_lo;
    const long rows = long(a.nslots) * 2 * a.M * ntensor;
    const unsigned grid = unsigned(std::min<long>(rows, 148L * 16));
    if (panels && ntensor == 2 && outp && a.Np == 128 && oz().rhs_panels(out0, out1, outp, a)) {
        const unsigned gp = unsigned(std::min<long>((rows * 2 + 3) / 4, 148L * 16));
        switch (nsrc) {
            case 1: eigen_rhs_pan_kernel<1><<<gp, 128, 0, c.stream>>>(a); break;
            case 2: eigen_rhs_pan_kernel<2><<<gp, 128, 0, c.stream>>>(a); break;
            case 3: eigen_rhs_pan_kernel<3><<<gp, 128, 0, c.stream>>>(a); break;
            case 4: eigen_rhs_pan_kernel<4><<<gp, 128, 0, c.stream>>>(a); break;
            case 5: eigen_rhs_pan_kernel<5><<<gp, 128, 0, c.stream>>>(a); break;
            case 6: eigen_rhs_pan_kernel<6><<<gp, 128, 0, c.stream>>>(a); break;
            case 7: eigen_rhs_pan_kernel<7><<<gp, 128, 0, c.stream>>>(a); break;
            case 8: eigen_rhs_pan_kernel<8><<<gp, 128, 0, c.stream>>>(a); break;
            default: throw Error(INTERNAL, "eigen_rhs: source count out of range");
        }
        CCF_CUDA(cudaGetLastError());
        ++c.launches;
        return;
    }
    switch (nsrc) {
        case 1: eigen_rhs_kernel<1><<<grid, 128, 0, c.stream>>>(a); break;
        case 2: eigen_rhs_kernel<2><<<grid, 128, 0, c.stream>>>(a); break;
        case 3: eigen_rhs_kernel<3><<<grid, 128, 0, c.stream>>>(a); break;
        case 4: eigen_rhs_kernel<4><<<grid, 128, 0, c.stream>>>(a); break;
        case 5: eigen_rhs_kernel<5><<<grid, 128, 0, c.stream>>>(a); break;
        case 6: eigen_rhs_kernel<6><<<grid, 128, 0, c.stream>>>(a); break;
        case 7: eigen_rhs_kernel<7><<<grid, 128, 0, c.stream>>>(a); break;
        case 8: eigen_rhs_kernel<8><<<grid, 128, 0, c.stream>>>(a); break;
        default: throw Error(INTERNAL, "eigen_rhs: source count out of range");
    }
    ++c.launches;
}

// u_t = QL Z_t QR for Z_t in the eigen layout (z0, z1) -> coefficient tensors (out0, out1)
void Pipeline::eigen_back(DevSet& set, int ntensor, const double* z0, const double* z1, double* out0, double* out1) {
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, mh = g.mh, nh = g.nh;
    const int Mp = M + (M & 1), Np = N + (N & 1);
    const size_t per = std::max(size_t(mh) * Np, size_t(M) * std::max(nh, Np));
    if (!dT1_.p) {
        const size_t cap = per * size_t(3 * std::max(c.gh.nslots, c.gf.nslots) * 4);  // up to 3 tensors of sub-problems
        dT1_.alloc(cap);
        dZ_.alloc(cap);
        dT3_.alloc(cap);
    }
    const void* keyp[1] = {&set};
    const int ci[1] = {ntensor};
    bool fresh;
    GemmPlan& e3 = gemm(ptr_key("e3", 1, keyp, keyp, ci), fresh);
    GemmPlan& e4 = gemm(ptr_key("e4", 1, keyp, keyp, ci), fresh);
    if (fresh) {
        const double* dg = set.dg;
        long task = 0;
        for (int t = 0; t < ntensor; ++t)
            for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
                for (int k0 = 0; k0 < 2; ++k0)
                    for (int pl = 0; pl < 2; ++pl, ++task) {
                        const long PLo = set.host.dg_left[size_t(s)], QLo = PLo + long(M) * mh;
                        const long PRo = set.host.dg_right[k0], QRo = PRo + long(nh) * Np;
                        double* T3 = dT3_.p + size_t(task) * per;
                        e3.A.push_back(dg + QLo);                                       // QL  mh x M (ld Mp)
                        e3.B.push_back(nullptr);
                        e3.Boff.push_back((long(t) << kBaseShift) + eig_off(s, pl, k0));  // Z   M x N (ld 2 Np)
                        e3.C.push_back(T3);                                             // T3  mh x N (ld Np)
                        e4.A.push_back(T3);
                        e4.B.push_back(dg + QRo);                                       // QR  N x nh
                        e4.Coff.push_back((long(t) << kBaseShift) + long(s) * g.slot_stride + long(pl) * g.plane_stride +
                                          long(k0) * nh);                               // u   mh x nh (ld n)
                    }
        e3.M = mh; e3.N = N; e3.K = M; e3.lda = Mp; e3.ldb = 2 * Np; e3.ldc = Np;
        e3.kzero = Mp - M;  // QL's pad column is zero (modal.cpp padld)
        e4.M = mh; e4.N = nh; e4.K = N; e4.lda = Np; e4.ldb = nh; e4.ldc = g.n;
        e3.upload();
        e4.upload();
    }
    e3.launch(c.stream, z0, ntensor > 1 ? z1 : z0);
    c.gemm_flops += e3.flops();
    e4.launch(c.stream, nullptr, nullptr, out0, ntensor > 1 ? out1 : out0);
    c.gemm_flops += e4.flops();
    c.launches += 2;
}

// Z = PL_P u PR (no RT) for one coefficient tensor -> eigen layout (initial NS state)
void Pipeline::to_eigen(DevSet& pset, const double* u, double* z) {
    const Geo& g = c.gh;
    const int M = c.M, N = c.N, mh = g.mh, nh = g.nh;
    const int Np = N + (N & 1);
    const size_t per = std::max(size_t(mh) * Np, size_t(M) * std::max(nh, Np));
    if (!dT1_.p) {
        const size_t cap = per * size_t(3 * std::max(c.gh.nslots, c.gf.nslots) * 4);  // up to 3 tensors of sub-problems
        dT1_.alloc(cap);
        dZ_.alloc(cap);
        dT3_.alloc(cap);
    }
    GemmPlan t1, t2;
    long task = 0;
    for (int s = c.sh.s_lo; s < c.sh.s_hi; ++s)
        for (int k0 = 0; k0 < 2; ++k0)
            for (int pl = 0; pl < 2; ++pl, ++task) {
                double* T1 = dT1_.p + size_t(task) * per;
                t1.A.push_back(pset.dg + pset.host.dg_left[size_t(s)]);
                t1.B.push_back(u + long(s) * g.slot_stride + long(pl) * g.plane_stride + long(k0) * nh);
                t1.C.push_back(T1);
                t2.A.push_back(T1);
                t2.B.push_back(pset.dg + pset.host.dg_right[k0]);
                t2.C.push_back(z + eig_off(s, pl, k0));
            }
    t1.M = M; t1.N = nh; t1.K = mh; t1.lda = mh; t1.ldb = g.n; t1.ldc = nh;
    t2.M = M; t2.N = N; t2.K = nh; t2.lda = nh; t2.ldb = Np; t2.ldc = 2 * Np;
    CCF_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * size_t(g.nslots) * 2 * M * 2 * Np, c.stream));
    t1.upload();
    t2.upload();
    t1.launch(c.stream);
    t2.launch(c.stream);
    CCF_CUDA(cudaStreamSynchronize(c.stream));
    c.launches += 2;
}

void Pipeline::decompose(const double* vr, const double* vt, const double* vz, double* lam, double* gam) {
    const Geo& g = c.gh;
    CurlDecomp a{};
    a.g = g;
    a.decompose_only = 1;
    a.ar = vr;
    a.at = vt;
    a.az = vz;
    a.lam = lam;
    a.gam = gam;
    a.scratch = big_scratch(size_t(g.nslots) * g.n * 6 * g.mh);
    a.q = tp.q.p;
    a.hpc = tp.hpc.p;
    a.hpr = tp.hpr.p;
    const long n = long(g.nslots) * g.n;
    curl_decomp_kernel<<<blocks_for(n, 64), 64, 0, c.stream>>>(a);
    ++c.launches;
}

void Pipeline::hpoisson(const double* rhs, double* u) {
    const Geo& g = c.gh;
    HpArgs a{g, rhs, u, big_scratch(size_t(g.nslots) * g.n * g.mh), tp.hpc.p, tp.hpr.p};
    hp_kernel<<<blocks_for(long(g.nslots) * g.n, 64), 64, 0, c.stream>>>(a);
    ++c.launches;
}

void Pipeline::scale(double* x, double a) {
    Combo cb{};
    cb.src[0] = x;
    cb.w[0] = a;
    cb.nsrc = 1;
    cb.out = x;
    cb.n = T;
    combo_kernel<<<std::min<long>(4736, (T + 255) / 256), 256, 0, c.stream>>>(cb);
    ++c.launches;
}

void Pipeline::calculus(int op, int cls, const double* in, double* out) {
    const Geo& g = c.gh;
    if (op == 1 || op == 6) {  // d/dz ; laplacian = hlap + dzz
        if (op == 1) {
            dz({in}, {out});
            return;
        }
        double* t1 = scratch(32);
        double* t2 = scratch(33);
        dz({in}, {t1});
        dz({t1}, {t2});
        CalcArgs a{g, 5, cls, in, out, big_scratch(size_t(g.nslots) * g.n * 3 * g.mh), tp.q.p};
        calc_kernel<<<blocks_for(long(g.nslots) * g.n, 64), 64, 0, c.stream>>>(a);
        Combo cb{};
        cb.src[0] = out;
        cb.w[0] = 1.0;
        cb.src[1] = t2;
        cb.w[1] = 1.0;
        cb.nsrc = 2;
        cb.out = out;
        cb.n = T;
        combo_kernel<<<std::min<long>(4736, (T + 255) / 256), 256, 0, c.stream>>>(cb);
        c.launches += 2;
        return;
    }
    if (op != 0 && op != 2 && op != 4 && op != 5) throw Error(DOMAIN_ERROR, "ccf_calculus: unknown op");
    CalcArgs a{g, op, cls, in, out, big_scratch(size_t(g.nslots) * g.n * 3 * g.mh), tp.q.p};
    calc_kernel<<<blocks_for(long(g.nslots) * g.n, 64), 64, 0, c.stream>>>(a);
    ++c.launches;
}

// Full (parity-agnostic, full-spectrum) transforms for arbitrary real fields.
void Pipeline::analyze_full(const double* values, double* coeffs) {
    const int m = c.m, n = c.n, p = c.p;
    const long nv = long(m) * n * p;
    double* v = big_scratch(size_t(4) * nv);  // v | t | complex (2 nv)
    double* t = v + nv;
    double* z = v + 2 * nv;
    c.load_values(values, v);
    CCF_CUDA(cudaMemsetAsync(c.ws.flag, 0, sizeof(int), c.stream));
    finite_check_kernel<<<std::min<long>(1184, (nv + 255) / 256), 256, 0, c.stream>>>(v, nv, c.ws.flag);
    int f = 0;
    CCF_CUDA(cudaMemcpyAsync(&f, c.ws.flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (f) throw Error(NUMERICAL, "analyze: non-finite input value");
    GemmPlan r, zz;
    for (int l = 0; l < p; ++l) {
        r.A.push_back(v + long(l) * m * n);  // [k][j] slice, r-analysis on the right
        r.B.push_back(tp.Rfull_A.p);         // B = A_r^T: (j, k) -> A[k][j]
        r.C.push_back(t + long(l) * m * n);
        zz.A.push_back(tp.Azf.p);
        zz.B.push_back(t + long(l) * m * n);
        zz.C.push_back(v + long(l) * m * n);
    }
    // Rfull_A is stored as A[k][j]; the right operand needs B[j][k] = A[k][j] -> use the transposed copy
    r.B.assign(size_t(p), full_rT());
    r.M = n; r.N = m; r.K = m; r.lda = m; r.ldb = m; r.ldc = m;
    zz.M = n; zz.N = m; zz.K = n; zz.lda = n; zz.ldb = m; zz.ldc = m;
    r.upload();
    zz.upload();
    r.launch(c.stream);
    c.gemm_flops += r.flops();
    zz.launch(c.stream);
    c.gemm_flops += zz.flops();
    real_to_complex_kernel<<<std::min<long>(4736, (nv + 255) / 256), 256, 0, c.stream>>>(v, z, nv);
    double* dst = coeffs;
    const bool host = !c.is_device_ptr(coeffs);
    if (host) dst = t;  // reuse t (+ next nv) as the complex output staging (t..t+2nv overlaps z? no: z = v+2nv)
    double* outc = host ? big2(size_t(2) * nv) : coeffs;
    theta_dft_full_kernel<<<unsigned(long(m) * n), 128, size_t(p) * sizeof(double2), c.stream>>>(
        z, outc, m, n, p, -1, reinterpret_cast<const double2*>(tp.twfull.p));
    c.launches += 5;
    if (host) CCF_CUDA(cudaMemcpyAsync(coeffs, outc, sizeof(double) * 2 * nv, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
}

void Pipeline::synthesize_full(const double* coeffs, double* values) {
    const int m = c.m, n = c.n, p = c.p;
    const long nv = long(m) * n * p;
    double* v = big_scratch(size_t(4) * nv);
    double* t = v + nv;
    double* z = v + 2 * nv;  // complex, 2 nv
    if (c.is_device_ptr(coeffs))
        CCF_CUDA(cudaMemcpyAsync(z, coeffs, sizeof(double) * 2 * nv, cudaMemcpyDeviceToDevice, c.stream));
    else
        CCF_CUDA(cudaMemcpyAsync(z, coeffs, sizeof(double) * 2 * nv, cudaMemcpyHostToDevice, c.stream));
    double* zc = big2(size_t(2) * nv);
    theta_dft_full_kernel<<<unsigned(long(m) * n), 128, size_t(p) * sizeof(double2), c.stream>>>(
        z, zc, m, n, p, +1, reinterpret_cast<const double2*>(tp.twfull.p));
    complex_re_kernel<<<std::min<long>(4736, (nv + 255) / 256), 256, 0, c.stream>>>(zc, v, nv);
    GemmPlan zz, r;
    for (int l = 0; l < p; ++l) {
        zz.A.push_back(tp.Szf.p);
        zz.B.push_back(v + long(l) * m * n);
        zz.C.push_back(t + long(l) * m * n);
        r.A.push_back(t + long(l) * m * n);
        r.B.push_back(full_sT());
        r.C.push_back(v + long(l) * m * n);
    }
    zz.M = n; zz.N = m; zz.K = n; zz.lda = n; zz.ldb = m; zz.ldc = m;
    r.M = n; r.N = m; r.K = m; r.lda = m; r.ldb = m; r.ldc = m;
    zz.upload();
    r.upload();
    zz.launch(c.stream);
    c.gemm_flops += zz.flops();
    r.launch(c.stream);
    c.gemm_flops += r.flops();
    c.launches += 4;
    c.store_values(v, values);
    c.sync();
}

const double* Pipeline::full_rT() {  // B[j][k] = A_r[k][j]
    if (!rAT_.p) {
        const int m = c.m;
        std::vector<double> A(size_t(m) * m), AT(size_t(m) * m);
        CCF_CUDA(cudaMemcpy(A.data(), tp.Rfull_A.p, A.size() * 8, cudaMemcpyDeviceToHost));
        for (int k = 0; k < m; ++k)
            for (int j = 0; j < m; ++j) AT[size_t(j) * m + k] = A[size_t(k) * m + j];
        upload(rAT_, AT);
    }
    return rAT_.p;
}

const double* Pipeline::full_sT() {  // B[k][j] = S_r[j][k]
    if (!rST_.p) {
        const int m = c.m;
        std::vector<double> S(size_t(m) * m), ST(size_t(m) * m);
        CCF_CUDA(cudaMemcpy(S.data(), tp.Rfull_S.p, S.size() * 8, cudaMemcpyDeviceToHost));
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < m; ++k) ST[size_t(k) * m + j] = S[size_t(j) * m + k];
        upload(rST_, ST);
    }
    return rST_.p;
}

double* Pipeline::big2(size_t doubles) {
    if (big2_.n < doubles) big2_.alloc(doubles);
    return big2_.p;
}

// ---------------------------------------------------------------- NS state
NSState::~NSState() {
    for (auto g : graphs)
        if (g) cudaGraphExecDestroy(g);
    if (dflag) cudaFree(dflag);
}

static void bdf_table(int b, double* koh, double w[4]) {  // proj/src/timestep.cpp:5-29
    static const double K[4] = {1.0, 2.0 / 3.0, 6.0 / 11.0, 12.0 / 25.0};
    static const double W[4][4] = {{1.0, 0, 0, 0},
                                   {4.0 / 3.0, -1.0 / 3.0, 0, 0},
                                   {18.0 / 11.0, -9.0 / 11.0, 2.0 / 11.0, 0},
                                   {48.0 / 25.0, -36.0 / 25.0, 16.0 / 25.0, -3.0 / 25.0}};
    *koh = K[b - 1];
    for (int i = 0; i < 4; ++i) w[i] = W[b - 1][i];
}

static void imex_table(int b, double w[4]) {  // proj/src/timestep.cpp:31-39
    static const double W[4][4] = {{1, 0, 0, 0}, {2, -1, 0, 0}, {3, -3, 1, 0}, {4, -6, 4, -1}};
    for (int i = 0; i < 4; ++i) w[i] = W[b - 1][i];
}

void NSState::enqueue(int b, int eo, int cur, int out, int nnew) {
    // proj/src/ptns.cpp:217-267
    Pipeline& P = *pl;
    Ctx& c = P.c;
    const double* lw = lam[cur].p;
    const double* gw = gam[cur].p;
    double koh, bw[4], iw[4] = {0, 0, 0, 0};
    bdf_table(b, &koh, bw);
    if (eo > 0) imex_table(eo, iw);
    const double kappa = koh * h;
    const double scale = kappa * (1.0 / reynolds);
    if (eigen) {
        // eigen-coordinate step (see Pipeline::eig_off): every modal solve is (RHS .* RT) + back transform,
        // and the back transforms produce the nonlinear term's z-synthesized inputs directly in eigen
        // coordinates along r (Pipeline::eigen_ysynth, QL folded into the synthesis blocks); omega
        // itself is reconstructed on demand (NSState::omega_coeff)
        DevSet& pset = c.set(false, true, 1.0);
        if (!disable_nonlinear) {
            c.mark("start");
            if (coeff_first) {
                // initial data: omega_0 need not lie in the range of QL PL, so the first nonlinear term runs on
                // the coefficient-space omega_0 and psi = QL Z_P QR, exactly as the reference
                if (zp_head != cur) {
                    const double* zs[1] = {zl[cur].p};
                    const double wm1[1] = {-1.0};
                    P.eigen_rhs(pset, 1, zs, zs, wm1, 1, 1.0, zpsi.p, zpsi.p);  // Z_P = -Z_lambda .* RT_P
                    zp_head = cur;
                }
                double* lpsi = P.scratch(18);
                P.eigen_back(pset, 1, zpsi.p, zpsi.p, lpsi, lpsi);
                c.mark("P_poisson_solve");
                P.nonlinear(gw, lpsi, lw, gw, nl[nnew].p, ng[nnew].p, &pset, false, false, dealias);  // N~ = PL_P N PR
            } else {
                // velocity_from_vorticity (ptns.cpp:85-91): lambda_v = gamma_omega (scratch 4), gamma_v = lambda_psi
                // (scratch 1, 2). In the steady state the previous step's Helmholtz back transform produced
                // them from Z_P; otherwise (displaced scratch) solve here.
                if (!(zv_head == cur && P.zw_owner_ == this)) {
                    velocity(cur);
                    c.mark("P_poisson_solve");
                }
                P.nonlinear(P.scratch(4), P.scratch(1), P.scratch(3), P.scratch(4), nl[nnew].p, ng[nnew].p, &pset,
                            true, true, dealias);  // N~ = PL_P N PR
            }
        }
        const double* sl[kMaxSrc];
        const double* sg[kMaxSrc];
        double wl[kMaxSrc];
        int ns = 0;
        for (int i = 0; i < b; ++i) {
            sl[ns] = zl[(cur + i) % 5].p;
            sg[ns] = zg[(cur + i) % 5].p;
            wl[ns++] = bw[i];
        }
        for (int i = 0; i < eo; ++i) {
            sl[ns] = nl[(nnew + i) % 5].p;
            sg[ns] = ng[(nnew + i) % 5].p;
            wl[ns++] = kappa * iw[i];
        }
        if (forced) {  // HeatStepper forcing: rhs += kappa * F (timestep.cpp:71-73), F~ = PL_P F PR
            sl[ns] = zf.p;
            sg[ns] = zf.p;
            wl[ns++] = kappa;
        }
        DevSet& set = c.set(false, false, scale);
        if (c.prof_events.empty()) c.mark("start");
        // PL_H = -(1/s) PL_P; the same pass leaves the next step's Poisson RHS Z_P = -Z_lambda .* RT_P and
        // raises the non-finite flag
        P.eigen_rhs(set, scalar ? 1 : 2, sl, sg, wl, ns, -1.0 / scale, zl[out].p, zg[out].p,
                    disable_nonlinear ? nullptr : zpsi.p, &pset, dflag, !disable_nonlinear);
        c.mark("H_rhs_combine");
        if (!disable_nonlinear) {
            zp_head = out;
            zsynth_omega(out);  // omega's and (next step's Poisson solve) the velocity's z tensors
            c.mark("H_helmholtz_solve");
        }
        return;
    } else {
        if (!disable_nonlinear) {
            double* lpsi = P.scratch(18);
            c.mark("start");
            // velocity_from_vorticity, ptns.cpp:85-91: lambda_psi = Poisson3D(-lambda_omega); after the first
            // step lambda_omega comes from our Helmholtz solve in the shared modal basis (modal_solve_from_z)
            if (!(zvalid && P.z_owner_ == this && P.modal_solve_from_z(c.set(false, true, 1.0), -1.0, lpsi)))
                P.poisson(lw, -1.0, lpsi);
            c.mark("P_poisson_solve");
            P.nonlinear(gw, lpsi, lw, gw, nl[nnew].p, ng[nnew].p, nullptr, false, false, dealias);  // nonlinear_term(v, omega)
        }
        const double* sl[kMaxSrc];
        const double* sg[kMaxSrc];
        double wl[kMaxSrc];
        int ns = 0;
        for (int i = 0; i < b; ++i) {
            sl[ns] = lam[(cur + i) % 5].p;
            sg[ns] = gam[(cur + i) % 5].p;
            wl[ns++] = bw[i];
        }
        for (int i = 0; i < eo; ++i) {  // kappa * sum_i imex_i N_i  (ptns.cpp:235-245, timestep.cpp:71-73)
            sl[ns] = nl[(nnew + i) % 5].p;
            sg[ns] = ng[(nnew + i) % 5].p;
            wl[ns++] = kappa * iw[i];
        }
        if (forced) {
            sl[ns] = fh.p;
            sg[ns] = fh.p;
            wl[ns++] = kappa;
        }
        DevSet& set = c.set(false, false, scale);
        if (c.prof_events.empty()) c.mark("start");
        if (scalar)
            P.modal_solve(set, false, 1, sl, wl, ns, nullptr, nullptr, 0, lam[out].p, nullptr, "H_rhs_combine");
        else
            P.modal_solve(set, false, 2, sl, wl, ns, sg, wl, ns, lam[out].p, gam[out].p, "H_rhs_combine");
        c.mark("H_helmholtz_solve");
        zvalid = P.last_z_valid_;  // Z of lambda_omega(out) stays in dZ_ (shared modal basis) for the next P
        if (zvalid) P.z_owner_ = this;
    }
    const long T = P.T;
    finite_check_kernel<<<std::min<long>(1184, (T + 255) / 256), 256, 0, c.stream>>>(lam[out].p, T, dflag);
    if (!scalar) finite_check_kernel<<<std::min<long>(1184, (T + 255) / 256), 256, 0, c.stream>>>(gam[out].p, T, dflag);
    c.launches += scalar ? 1 : 2;
}

// the nonlinear term's omega inputs (z synthesis of lambda_omega, gamma_omega, dz gamma_omega) into
// scratch 3..5, from the eigen state of ring slot r
// solve_poisson_3d(-lambda_omega) of ring slot r in eigen coordinates and the velocity's z tensors
// (scratch 1, 2)
void NSState::velocity(int r) {
    Pipeline& P = *pl;
    DevSet& pset = P.c.set(false, true, 1.0);
    if (zp_head != r) {  // Z_P = -Z_lambda .* RT_P
        const double* zs[1] = {zl[r].p};
        const double wm1[1] = {-1.0};
        P.eigen_rhs(pset, 1, zs, zs, wm1, 1, 1.0, zpsi.p, zpsi.p);
        zp_head = r;
    }
    const double* zz[1] = {zpsi.p};
    double* oS[1] = {P.scratch(1)};
    double* oD[1] = {P.scratch(2)};
    P.eigen_ysynth(1, zz, oS, oD);
    zv_head = r;
}

void NSState::zsynth_omega(int r) {
    // lambda_omega -> S (scratch 3); gamma_omega -> S, dz S (4, 5); with a valid Z_P of the same slot also
    // lambda_psi -> S, dz S (1, 2), i.e. the next nonlinear term's velocity: one launch (eigen_ysynth)
    Pipeline& P = *pl;
    const bool vel = zp_head == r;
    const double* z[3] = {zl[r].p, zg[r].p, zpsi.p};
    double* oS[3] = {P.scratch(3), P.scratch(4), P.scratch(1)};
    double* oD[3] = {nullptr, P.scratch(5), P.scratch(2)};
    P.eigen_ysynth(vel ? 3 : 2, z, oS, oD);
    zv_head = vel ? r : -1;
    P.zw_owner_ = this;
}

// NSStepper::velocity(): (lambda_v, gamma_v) = (gamma_omega, Poisson3D(-lambda_omega)) of the current state
void NSState::velocity_coeff(double* lam_v, double* gam_v) {
    Pipeline& P = *pl;
    Ctx& c = P.c;
    omega_coeff();
    CCF_CUDA(cudaMemcpyAsync(lam_v, gam[head].p, sizeof(double) * size_t(P.T), cudaMemcpyDeviceToDevice, c.stream));
    if (!eigen) {
        P.poisson(lam[head].p, -1.0, gam_v);
        return;
    }
    DevSet& pset = c.set(false, true, 1.0);
    if (ztmp.n < size_t(P.T)) ztmp.alloc(size_t(P.T));
    const double* zs[1] = {zl[head].p};
    const double wm1[1] = {-1.0};
    P.eigen_rhs(pset, 1, zs, zs, wm1, 1, 1.0, ztmp.p, ztmp.p);  // -Z_lambda .* RT_P
    P.eigen_back(pset, 1, ztmp.p, ztmp.p, gam_v, gam_v);
}

// gamma_psi = Poisson3D(-gamma_omega) of the omega the last step started from (ptns.cpp:248-253)
void NSState::gamma_psi_coeff(double* out) {
    Pipeline& P = *pl;
    Ctx& c = P.c;
    if (steps == 0) throw Error(DOMAIN_ERROR, "NSStepper: gamma_psi is computed from the first step on");
    const int prev = (head + 1) % 5;
    if (!eigen) {
        P.poisson(gam[prev].p, -1.0, out);
        return;
    }
    DevSet& pset = c.set(false, true, 1.0);
    if (ztmp.n < size_t(P.T)) ztmp.alloc(size_t(P.T));
    const double* zs[1] = {zg[prev].p};
    const double wm1[1] = {-1.0};
    P.eigen_rhs(pset, 1, zs, zs, wm1, 1, 1.0, ztmp.p, ztmp.p);
    P.eigen_back(pset, 1, ztmp.p, ztmp.p, out, out);
}

// coefficient-space omega of the newest ring slot (eigen mode keeps only Z between steps)
void NSState::omega_coeff() {
    if (!eigen || coeff_head == head) return;
    pl->eigen_back(pl->c.set(false, true, 1.0), scalar ? 1 : 2, zl[head].p, zg[head].p, lam[head].p, gam[head].p);
    coeff_head = head;
}

// NSStepper::seed (ptns.cpp:195-203): install a prebuilt history (reference-layout coefficient tensors on the
// host or the device, newest first). nonlinear_hist[i] belongs to omega_hist[i + 1]: the next step pushes
// N(omega_hist[0]) in front (ptns.cpp:232). Only the entries a step can read are kept (<= 4 of each).
void NSState::seed(int n_omega, const double* const* lam_h, const double* const* gam_h, int n_nl,
                   const double* const* nl_l, const double* const* nl_g, double t, int steps_taken) {
    Pipeline& P = *pl;
    Ctx& c = P.c;
    if (n_omega < 1) throw Error(DOMAIN_ERROR, "NSStepper::seed: empty history");
    if (scalar) throw Error(CONFIG_ERROR, "NSStepper::seed: not an NS stepper");
    const int no = std::min(n_omega, 4);
    const int nn = disable_nonlinear ? 0 : std::min(std::max(n_nl, 0), 4);
    DevSet* pset = eigen ? &c.set(false, true, 1.0) : nullptr;
    for (int i = 0; i < no; ++i) {
        const int r = (head + i) % 5;
        c.load_coeff(lam_h[i], lam[r].p, false, 0, 0);
        c.load_coeff(gam_h[i], gam[r].p, false, 0, 1);
        if (eigen) {
            P.to_eigen(*pset, lam[r].p, zl[r].p);
            P.to_eigen(*pset, gam[r].p, zg[r].p);
        }
    }
    if (nn > 0 && eigen && ctmp.n < size_t(P.T)) ctmp.alloc(size_t(P.T));
    for (int i = 0; i < nn; ++i) {
        const int r = (nhead + i) % 5;
        if (eigen) {  // N~ = PL_P N PR
            c.load_coeff(nl_l[i], ctmp.p, false, 0, 0);
            P.to_eigen(*pset, ctmp.p, nl[r].p);
            c.load_coeff(nl_g[i], ctmp.p, false, 0, 1);
            P.to_eigen(*pset, ctmp.p, ng[r].p);
        } else {
            c.load_coeff(nl_l[i], nl[r].p, false, 0, 0);
            c.load_coeff(nl_g[i], ng[r].p, false, 0, 1);
        }
    }
    c.sync();
    ocount = no;
    ncount = std::min(nn, order);
    time = t;
    steps = steps_taken;
    coeff_head = head;
    coeff_first = true;
    zp_head = zv_head = -1;
    zvalid = false;
    if (P.zw_owner_ == this) P.zw_owner_ = nullptr;
}

void NSState::step_once() {
    Ctx& c = pl->c;
    // bdf_rhs (timestep.cpp:41-42)
    if (ocount < std::min(order, steps + 1))
        throw Error(DOMAIN_ERROR, "bdf_rhs: insufficient history for the requested order");
    // scratch 3..5 may have been reused (another stepper, a standalone nonlinear call) since our last step
    if (eigen && !disable_nonlinear && !coeff_first && pl->zw_owner_ != this) {
        zsynth_omega(head);
        if (zv_head != head) velocity(head);  // a replayed graph has no Poisson stage
    }
    // coefficient-space state: dZ_ may have been reused (another stepper, a standalone solve) since our last step
    if (!eigen && zvalid && pl->z_owner_ != this) zvalid = false;
    const int b = std::min(order, steps + 1);
    const int out = (head + 4) % 5;
    const int nnew = (nhead + 4) % 5;
    const int ncnt = disable_nonlinear ? 0 : std::min(ncount + 1, order);
    const int eo = disable_nonlinear ? 0 : std::min(b, ncnt);
    const bool steady = (b == order) && (disable_nonlinear || ncount == order);
    const int key = head * 5 + nhead;
    // host-mode rank barriers synchronise inside the step: no graph capture
    if (use_graphs && steady && phase_warm[key] && c.sh.mode != Shard::HOST && !forced && !coeff_first &&
        (!graphs[key] || !graph_z[key] || zvalid)) {
        if (!graphs[key]) {
            graph_z[key] = !eigen && !disable_nonlinear && zvalid;
            cudaGraph_t g;
            const long l0 = c.launches;
            CCF_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
            enqueue(b, eo, head, out, nnew);
            CCF_CUDA(cudaStreamEndCapture(c.stream, &g));
            CCF_CUDA(cudaGraphInstantiate(&graphs[key], g, 0));
            CCF_CUDA(cudaGraphDestroy(g));
            launches_per_step = c.launches - l0;
            c.launches = l0;
        }
        CCF_CUDA(cudaGraphLaunch(graphs[key], c.stream));
        c.launches += launches_per_step;
    } else {
        const long l0 = c.launches;
        enqueue(b, eo, head, out, nnew);
        if (steady) launches_per_step = c.launches - l0;
        phase_warm[key] = true;
    }
    if (!eigen && !disable_nonlinear && zvalid) pl->z_owner_ = this;  // (graph replays skip enqueue)
    head = out;
    coeff_head = eigen ? -1 : head;
    if (eigen && !disable_nonlinear) zp_head = zv_head = out;  // (graph replays skip enqueue)
    if (!disable_nonlinear) {
        nhead = nnew;
        ncount = ncnt;
    }
    ocount = std::min(ocount + 1, order);
    coeff_first = false;
    ++steps;
    time += h;
}

}  // namespace ccf
