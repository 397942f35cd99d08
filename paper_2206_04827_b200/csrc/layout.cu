// Layout conversion between the reference tensor layout (complex interleaved,
// (l*n+k)*m+j, all p slices; proj/include/cylspec/coeffs.hpp:16-45) and the
// device-resident half-spectrum parity-compressed layout (ccf_device.cuh).
// Also: finite guards (proj/src/solvers.cpp:145, transform.cpp:125) and the
// pointwise BDF/IMEX combinations.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ccf {

__device__ __forceinline__ int slot_of_l(int l, int p, bool full) {
    if (full) return l;
    if (l == 0) return p / 2;
    return l >= p / 2 ? l - p / 2 : p / 2 - l;
}

__device__ __forceinline__ int w_of_slot(int s, int p, bool full) {
    if (full) return s - p / 2;
    return s == p / 2 ? -p / 2 : s;
}

__device__ __forceinline__ int parity_j0(int w, int cls) { return ((w + cls) % 2 + 2) % 2; }

// ref (interleaved complex) -> compressed. One thread per compressed element.
__global__ void ref_to_h_kernel(const double* __restrict__ ref, double* __restrict__ out, Geo g, int full, int cls) {
    const long total = long(g.nslots) * g.slot_stride;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const int k = kfrompos(int(i % g.n), g.nh);
        const long r = i / g.n;
        const int jj = int(r % g.mh);
        const long r2 = r / g.mh;
        const int plane = int(r2 % 2);
        const int s = int(r2 / 2);
        int l;
        if (full) l = s;
        else l = (s == g.p / 2) ? 0 : s + g.p / 2;
        const int w = l - g.p / 2;
        const int j = 2 * jj + parity_j0(w, cls);
        out[i] = ref[2 * ((long(l) * g.n + k) * g.m + j) + plane];
    }
}

// compressed -> ref (interleaved complex), Hermitian completion in half mode.
__global__ void h_to_ref_kernel(const double* __restrict__ in, double* __restrict__ ref, Geo g, int full, int cls,
                                int accumulate) {
    const long total = long(g.p) * g.n * g.m;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const int j = int(i % g.m);
        const long r = i / g.m;
        const int k = int(r % g.n);
        const int l = int(r / g.n);
        const int w = l - g.p / 2;
        const int j0 = parity_j0(w, cls);
        double re = 0.0, im = 0.0;
        if (((j - j0) & 1) == 0) {
            const int s = slot_of_l(l, g.p, full);
            const long off = long(s) * g.slot_stride + long((j - j0) / 2) * g.n + kpos(k, g.nh);
            re = in[off];
            im = in[off + g.plane_stride];
            if (!full && l != 0 && l < g.p / 2) im = -im;  // w < 0: conjugate partner
        }
        if (accumulate) {
            ref[2 * i] += re;
            ref[2 * i + 1] += im;
        } else {
            ref[2 * i] = re;
            ref[2 * i + 1] = im;
        }
    }
}

__global__ void finite_check_kernel(const double* __restrict__ x, long n, int* flag) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        if (!isfinite(x[i])) {
            atomicExch(flag, 1);
            return;
        }
}

__global__ void real_to_complex_kernel(const double* __restrict__ in, double* __restrict__ out, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        out[2 * i] = in[i];
        out[2 * i + 1] = 0.0;
    }
}

__global__ void complex_re_kernel(const double* __restrict__ in, double* __restrict__ out, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        out[i] = in[2 * i];
}

// out = sum_i w_i * src_i  (BDF history / IMEX extrapolation combinations,
// proj/src/timestep.cpp:41-51, proj/src/ptns.cpp:235-245)
__global__ void combo_kernel(Combo c) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < c.n; i += long(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int q = 0; q < c.nsrc; ++q) acc = fma(c.w[q], c.src[q][i], acc);
        c.out[i] = acc;
    }
}

}  // namespace ccf
