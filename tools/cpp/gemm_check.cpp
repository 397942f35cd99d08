// Batched-GEMM launcher check (GemmPlan, csrc/pipeline.cu) against a host reference on random data:
//   gemm_check M N K lda ldb ldc nbatch [bcol]   (bcol: column offset of every B block inside its rows)
// Prints the max relative error and which kernel variant the plan selected.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "pipeline.hpp"

int main(int argc, char** argv) {
    if (argc < 8) return 2;
    const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]);
    const long lda = atol(argv[4]), ldb = atol(argv[5]), ldc = atol(argv[6]);
    const int nb = atoi(argv[7]);
    const int bcol = argc > 8 ? atoi(argv[8]) : 0;
    // blocks start on whole rows of their leading dimension (as every operand on the library's path)
    const size_t asz = size_t(M + 1) * lda, bsz = size_t(K + 1) * ldb, csz = size_t(M + 1) * ldc;
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> u(-1, 1);
    std::vector<double> hA(asz * nb), hB(bsz * nb);
    for (double& x : hA) x = u(rng);
    for (double& x : hB) x = u(rng);
    ccf::DBuf A(hA.size()), B(hB.size()), C(csz * nb);
    cudaMemcpy(A.p, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B.p, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
    ccf::GemmPlan g;
    for (int b = 0; b < nb; ++b) {
        g.A.push_back(A.p + b * asz);
        g.B.push_back(B.p + b * bsz + bcol);
        g.C.push_back(C.p + b * csz);
    }
    g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
    g.upload();
    g.launch(nullptr);
    cudaDeviceSynchronize();
    std::vector<double> hC(C.n);
    cudaMemcpy(hC.data(), C.p, hC.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int b = 0; b < nb; ++b)
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                long double s = 0;
                for (int k = 0; k < K; ++k) s += (long double)hA[b * asz + i * lda + k] * hB[b * bsz + bcol + k * ldb + j];
                err = std::max(err, std::fabs(double(s) - hC[b * csz + i * ldc + j]));
                mx = std::max(mx, std::fabs(double(s)));
            }
    std::printf("M %d N %d K %d lda %ld ldb %ld ldc %ld nb %d: tma %d pipe %d rel err %.3e  %s\n", M, N, K, lda, ldb, ldc,
                nb, int(g.tma), int(g.pipe), err / mx, cudaGetErrorString(cudaGetLastError()));
    return err / mx < 1e-12 ? 0 : 1;
}
