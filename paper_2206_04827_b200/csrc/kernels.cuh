// Kernel declarations shared between the .cu translation units and the host driver.
#pragma once

#include <cuda_runtime.h>

#include "ccf_device.cuh"

namespace ccf {

// adi.cu
__global__ void adi_kernel(const AdiParams P);
struct RoundCheck {
    int ntensor, nslots, round;
    double tol;
    double* res2;
    double* e2;
    int* active;
    double* history;
    int* rounds;
    int* err;
    const int* J;          // per slot
    unsigned long long* iters;  // executed sub-problem iterations (4 sub-problems per (tensor, slot))
};
__global__ void adi_round_check(RoundCheck c);

// layout.cu
__global__ void ref_to_h_kernel(const double* __restrict__ ref, double* __restrict__ out, Geo g, int full, int cls);
__global__ void h_to_ref_kernel(const double* __restrict__ in, double* __restrict__ ref, Geo g, int full, int cls);
__global__ void finite_check_kernel(const double* __restrict__ x, long n, int* flag);
struct Combo {
    const double* src[kMaxSrc];
    double w[kMaxSrc];
    int nsrc;
    double* out;
    long n;
};
__global__ void combo_kernel(Combo c);

}  // namespace ccf
