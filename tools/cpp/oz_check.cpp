// Ozaki INT8 tcgen05 GEMM (csrc/ozaki.cu) against a long-double host product, and its speed against
// the FP64 DMMA GEMM (GemmPlan) on the same batch:
//   oz_check M N K nbatch nterms decay [reps]
// C_b = sum_t A_bt (M x K, row-major) B_bt (K x N, row-major); A rows split directly (A side), B split
// with the transpose (B side), as in the NS step. decay: entries ~ U(-1,1) * decay^(i + k) so rows and
// columns span several decades (spectral data). Prints max |C - C_ref| / max |C_ref| per batch (worst)
// and timings; exit 1 if the error exceeds 1e-12.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "ozaki.hpp"
#include "pipeline.hpp"

using namespace ccf;

int main(int argc, char** argv) {
    if (argc < 7) return 2;
    const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), nb = atoi(argv[4]), nt = atoi(argv[5]);
    const double decay = atof(argv[6]);
    const int reps = argc > 7 ? atoi(argv[7]) : 0;
    const int shared = argc > 8 ? atoi(argv[8]) : 0;  // 1: every term reads batch 0's panels (L2-resident operands)
    const int Np = ((N + kOzNT - 1) / kOzNT) * kOzNT;  // B panel rows
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> u(-1, 1);
    const size_t asz = size_t(M) * K, bsz = size_t(K) * N;
    std::vector<double> hA(asz * nb * nt), hB(bsz * nb * nt);
    for (int bt = 0; bt < nb * nt; ++bt) {
        for (int i = 0; i < M; ++i)
            for (int k = 0; k < K; ++k) hA[bt * asz + i * K + k] = u(rng) * std::pow(decay, i + k) * (1 + bt % 3);
        for (int k = 0; k < K; ++k)
            for (int j = 0; j < N; ++j) hB[bt * bsz + k * N + j] = u(rng) * std::pow(decay, k + (j % 128)) * std::pow(10.0, bt % 5);
    }
    DBuf A(hA.size()), B(hB.size()), C(size_t(M) * N * nb), C2(size_t(M) * N * nb);
    cudaMemcpy(A.p, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B.p, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
    // panels: A: 128 rows per (b, t); B: Np rows per (b, t)
    const size_t pa = oz_panel_bytes(128), pb = oz_panel_bytes(Np);
    DBuf PA((pa * nb * nt + 7) / 8), PB((pb * nb * nt + 7) / 8), SA(size_t(128) * nb * nt), SB(size_t(Np) * nb * nt);
    DBuf PE(size_t(nb) * nt * (Np / 128));  // plane exponents (ints) [b][t][tile]
    int* pe = reinterpret_cast<int*>(PE.p);
    cudaMemset(PA.p, 0, PA.n * 8);
    cudaMemset(PB.p, 0, PB.n * 8);
    OzSplitPlan sa, sb;
    sb.transpose = true;
    sb.mn = std::getenv("CCF_OZ_MN") && std::atoi(std::getenv("CCF_OZ_MN"));
    OzGemmPlan g;
    for (int bt = 0; bt < nb * nt; ++bt) {
        uint8_t* pA = reinterpret_cast<uint8_t*>(PA.p) + pa * bt;
        sa.jobs.push_back(oz_job(A.p + bt * asz, long(K), M, K, pA, SA.p + 128 * bt, long(oz_slice_bytes(128)), 128));
        const int bs = shared ? bt % nt : bt;
        // the terms of one batch share B column scales (one split job over the batch's nt B blocks)
        const int b0 = (bs / nt) * nt;
        // shared 2: only B is shared (A distinct per batch, like the back transforms / z analysis)
        const int as = shared == 2 ? bt : bs;
        g.terms.push_back({reinterpret_cast<uint8_t*>(PA.p) + pa * as, reinterpret_cast<uint8_t*>(PB.p) + pb * bs,
                           SA.p + 128 * as, SB.p + long(Np) * b0, long(oz_slice_bytes(Np)), pe + size_t(bs) * (Np / 128)});
    }
    for (int b = 0; b < nb; ++b) {
        OzSplitJob j = oz_job(B.p + size_t(b) * nt * bsz, long(N), N, K, reinterpret_cast<uint8_t*>(PB.p) + pb * b * nt,
                              SB.p + long(Np) * b * nt, long(oz_slice_bytes(Np)), Np, pe + size_t(b) * nt * (Np / 128));
        j.nsrc = nt;
        for (int t = 0; t < nt; ++t) {
            j.src[t] = B.p + (size_t(b) * nt + t) * bsz;
            j.dst[t] = reinterpret_cast<uint8_t*>(PB.p) + pb * (size_t(b) * nt + t);
        }
        sb.jobs.push_back(j);
    }
    // CCF_OZ_PANEL=1: every tile is written as an MN-major B panel tile (the X3 / H epilogue) instead of fp64
    // (timing only: the check is skipped)
    const bool panel_out = std::getenv("CCF_OZ_PANEL") && std::atoi(std::getenv("CCF_OZ_PANEL"));
    const int ntile = (N + kOzNT - 1) / kOzNT;
    DBuf PO(panel_out ? (size_t(nb) * ntile * oz_panel_bytes(128) + 7) / 8 : 1), POE(size_t(nb) * ntile);
    for (int b = 0; b < nb; ++b)
        for (int n0 = 0; n0 < N; n0 += kOzNT) {
            OzItem it{b * nt, (b + 1) * nt, n0, M, std::min(kOzNT, N - n0), 0, C.p + size_t(b) * M * N + n0, long(N), 1.0};
            if (panel_out) {
                const size_t ti = size_t(b) * ntile + n0 / kOzNT;
                it.pdst = reinterpret_cast<uint8_t*>(PO.p) + ti * oz_panel_bytes(128);
                it.pstride = long(oz_slice_bytes(128));
                it.ppe = reinterpret_cast<int*>(POE.p) + ti;
            }
            g.items.push_back(it);
        }
    g.b_mn = sb.mn;
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
    double worst = 0, worst_bound = 0;
    int nbad = 0, firstbad = -1;
    for (int b = 0; b < (panel_out || std::getenv("CCF_OZ_NOCHECK") ? 0 : nb); ++b) {
        double err = 0, mx = 0, bound = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long double s = 0, sabs = 0;
                for (int t = 0; t < nt; ++t) {
                    const size_t bt = size_t(b) * nt + t;
                    for (int k = 0; k < K; ++k) {
                        const long double p = (long double)hA[bt * asz + i * K + k] * hB[bt * bsz + k * N + j];
                        s += p;
                        sabs += fabsl(p);
                    }
                }
                const double d = std::fabs(double(s) - hC[size_t(b) * M * N + i * N + j]);
                err = std::max(err, d);
                mx = std::max(mx, std::fabs(double(s)));
                if (sabs > 0) bound = std::max(bound, d / double(sabs));
            }
        worst = std::max(worst, err / mx);
        if (err / mx > 1e-12) {
            if (firstbad < 0) firstbad = b;
            ++nbad;
        }
        worst_bound = std::max(worst_bound, bound);
    }
    if (panel_out) worst = worst_bound = 0;  // (no fp64 output to check)
    std::printf("oz M %d N %d K %d nb %d nt %d decay %.2f: max rel err %.3e (vs sum|ab| %.3e), bad batches %d (first %d)\n", M,
                N, K, nb, nt, decay, worst, worst_bound, nbad, firstbad);
    if (reps > 0) {  // speed: split + GEMM vs the DMMA GemmPlan on the same batch
        GemmPlan d;
        for (int b = 0; b < nb; ++b) {
            d.tstart.push_back(int(d.A.size()));
            for (int t = 0; t < nt; ++t) {
                d.A.push_back(A.p + (size_t(b) * nt + t) * asz);
                d.B.push_back(B.p + (size_t(b) * nt + t) * bsz);
            }
            d.C.push_back(C2.p + size_t(b) * M * N);
        }
        d.tstart.push_back(int(d.A.size()));
        if (nt == 1) d.tstart.clear();
        d.M = M; d.N = N; d.K = K; d.lda = K; d.ldb = N; d.ldc = N;
        d.upload();
        cudaEvent_t e0, e1, e2, e3;
        cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
        for (int w = 0; w < 3; ++w) { sa.launch(nullptr); sb.launch(nullptr); g.launch(nullptr); d.launch(nullptr); }
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) { sa.launch(nullptr); sb.launch(nullptr); }
        cudaEventRecord(e1);
        for (int r = 0; r < reps; ++r) g.launch(nullptr);
        cudaEventRecord(e2);
        for (int r = 0; r < reps; ++r) d.launch(nullptr);
        cudaEventRecord(e3);
        cudaDeviceSynchronize();
        float ts, tg, td;
        cudaEventElapsedTime(&ts, e0, e1);
        cudaEventElapsedTime(&tg, e1, e2);
        cudaEventElapsedTime(&td, e2, e3);
        if (std::getenv("CCF_OZ_MODE") && (std::atoi(std::getenv("CCF_OZ_MODE")) & 4)) oz_trace_dump();
        const double fl = 2.0 * M * N * K * nt * nb;
        std::printf("  split %.4f ms, oz gemm %.4f ms (%.1f TFLOP/s fp64-equiv), dmma gemm %.4f ms (%.1f TFLOP/s)  %s\n",
                    ts / reps, tg / reps, fl / (tg / reps * 1e-3) / 1e12, td / reps, fl / (td / reps * 1e-3) / 1e12,
                    cudaGetErrorString(cudaGetLastError()));
    }
    return (worst < 1e-12 || shared) ? 0 : 1;
}
