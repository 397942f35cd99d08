// CTA-pair INT8 GEMM (csrc/ozaki.cu, oz_pair_kernel: tcgen05.mma.cta_group::2) against a long-double host
// product, and its speed:
//   oz_pair_check npair nt kind amn decay [reps]
// Pair item i computes, for rank r = 0, 1 (batch b = 2 i + r), C_b = sum_t A_bt Bt_t^T with A_bt 128 x 128 and
// Bt_t 128 x 128 (rows = output columns, K contiguous); every item shares the nt B blocks, split with one scale
// per row over the nt blocks (the composite-operator layout). amn = 1: A is given as A^T (K x M row-major) and
// split into MN-major panels with one scale per tile (the panel-output layout of the NS products).
// kind 0: fp64 rows, 1: fp64 transposed (C^T), 2: MN-major panel tiles (timing only). Exit 1 if the error
// exceeds 1e-12 of max |C|.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ozaki.hpp"
#include "pipeline.hpp"

using namespace ccf;
extern "C" void ccf_debug_pz_trace_dump(int n);

int main(int argc, char** argv) {
    if (argc < 6) return 2;
    const int np = atoi(argv[1]), nt = atoi(argv[2]), kind = atoi(argv[3]), amn = atoi(argv[4]);
    const double decay = atof(argv[5]);
    const int reps = argc > 6 ? atoi(argv[6]) : 0;
    const int nb = 2 * np, M = 128, N = 128, K = 128;
    std::mt19937_64 rng(11);
    std::uniform_real_distribution<double> u(-1, 1);
    const size_t bsz = size_t(M) * K;
    std::vector<double> hA(bsz * nb * nt), hB(bsz * nt);  // hA[(b nt + t)]: A (M x K) or A^T (K x M) if amn
    for (int bt = 0; bt < nb * nt; ++bt)
        for (int i = 0; i < M; ++i)
            for (int k = 0; k < K; ++k) {
                const double v = u(rng) * std::pow(decay, i + k) * (1 + bt % 3);
                hA[bt * bsz + (amn ? size_t(k) * M + i : size_t(i) * K + k)] = v;
            }
    for (int t = 0; t < nt; ++t)
        for (int j = 0; j < N; ++j)
            for (int k = 0; k < K; ++k) hB[t * bsz + j * K + k] = u(rng) * std::pow(decay, j + k) * std::pow(10.0, t % 3);
    DBuf A(hA.size()), B(hB.size()), C(size_t(M) * N * nb);
    cudaMemcpy(A.p, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B.p, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(C.p, 0, C.n * 8);
    const size_t pan = oz_panel_bytes(128);
    const long sl = long(oz_slice_bytes(128));
    DBuf PA((pan * nb * nt + 7) / 8), PB((pan * nt + 7) / 8), SA(size_t(128) * nb * nt), SB(128), PE(size_t(nb) * nt);
    DBuf PO(kind == 2 ? (pan * nb + 7) / 8 : 1), POE(nb);
    int* pe = reinterpret_cast<int*>(PE.p);
    auto pa = [&](int bt) { return reinterpret_cast<uint8_t*>(PA.p) + pan * bt; };
    auto pb = [&](int t) { return reinterpret_cast<uint8_t*>(PB.p) + pan * t; };
    OzSplitPlan sa, sb;
    sa.mn = amn != 0;
    for (int bt = 0; bt < nb * nt; ++bt)
        sa.jobs.push_back(amn ? oz_job(A.p + bt * bsz, M, M, K, pa(bt), SA.p + 128 * bt, sl, 128, pe + bt)
                              : oz_job(A.p + bt * bsz, K, M, K, pa(bt), SA.p + 128 * bt, sl, 128));
    {  // the nt B blocks: one job, shared row scales
        OzSplitJob j = oz_job(B.p, K, N, K, pb(0), SB.p, sl, 128);
        j.nsrc = nt;
        for (int t = 0; t < nt; ++t) {
            j.src[t] = B.p + t * bsz;
            j.dst[t] = pb(t);
        }
        sb.jobs.push_back(j);
    }
    OzPairPlan g;
    g.a_mn = amn != 0;
    g.b_res = std::getenv("CCF_OZ_BRES") && std::atoi(std::getenv("CCF_OZ_BRES"));  // (nt = 1: one B tile)
    for (int i = 0; i < np; ++i) {
        OzPItem it{};
        it.t0 = int(g.terms.size());
        for (int t = 0; t < nt; ++t) {
            OzPTerm T{};
            for (int r = 0; r < 2; ++r) {
                const int bt = (2 * i + r) * nt + t;
                T.a[r] = pa(bt);
                T.sa[r] = amn ? nullptr : SA.p + 128 * bt;
                T.pe[r] = amn ? pe + bt : nullptr;
            }
            T.b = pb(t);
            T.astride = sl;
            T.bstride = sl;
            g.terms.push_back(T);
        }
        it.t1 = int(g.terms.size());
        it.m[0] = it.m[1] = M;
        it.n = N;
        it.kind = kind;
        it.alpha = 1.0;
        it.sb = SB.p;
        it.ldc = kind == 1 ? M : N;
        for (int r = 0; r < 2; ++r) {
            it.c[r] = C.p + size_t(2 * i + r) * M * N;
            if (kind == 2) {
                it.pdst[r] = reinterpret_cast<uint8_t*>(PO.p) + pan * (2 * i + r);
                it.ppe[r] = reinterpret_cast<int*>(POE.p) + 2 * i + r;
            }
        }
        it.pstride = sl;
        g.items.push_back(it);
    }
    sa.upload();
    sb.upload();
    g.upload();
    sa.launch(nullptr);
    sb.launch(nullptr);
    g.launch(nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        std::printf("CUDA error %s\n", cudaGetErrorString(e));
        return 1;
    }
    std::vector<double> hC(C.n);
    cudaMemcpy(hC.data(), C.p, hC.size() * 8, cudaMemcpyDeviceToHost);
    double worst = 0;
    int nbad = 0;
    const int ncheck = kind == 2 ? 0 : std::min(nb, 64);
    for (int b = 0; b < ncheck; ++b) {
        double err = 0, mx = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long double s = 0;
                for (int t = 0; t < nt; ++t)
                    for (int k = 0; k < K; ++k) {
                        const double a = hA[(size_t(b) * nt + t) * bsz + (amn ? size_t(k) * M + i : size_t(i) * K + k)];
                        s += (long double)a * hB[t * bsz + j * K + k];
                    }
                const double got = hC[size_t(b) * M * N + (kind == 1 ? size_t(j) * M + i : size_t(i) * N + j)];
                err = std::max(err, std::fabs(double(s) - got));
                mx = std::max(mx, std::fabs(double(s)));
            }
        worst = std::max(worst, err / mx);
        nbad += err / mx > 1e-12;
    }
    std::printf("oz pair np %d nt %d kind %d amn %d decay %.2f: max rel err %.3e, bad tiles %d of %d checked\n", np, nt, kind,
                amn, decay, worst, nbad, ncheck);
    if (reps > 0) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int w = 0; w < 3; ++w) g.launch(nullptr);
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) g.launch(nullptr);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float tg;
        cudaEventElapsedTime(&tg, e0, e1);
        if (std::getenv("CCF_OZ_MODE") && (std::atoi(std::getenv("CCF_OZ_MODE")) & 4)) ccf_debug_pz_trace_dump(60);
        const double fl = 2.0 * M * N * K * nt * nb;
        std::printf("  pair gemm %.4f ms (%.1f TFLOP/s fp64-equiv, %.0f TOPS int8)  %s\n", tg / reps,
                    fl / (tg / reps * 1e-3) / 1e12, 26.0 * fl / (tg / reps * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return (worst < 1e-12) ? 0 : 1;
}
