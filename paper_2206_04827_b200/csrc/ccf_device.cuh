// Shared device-side definitions for the B200 CCF kernels (sm_100a).
//
// Data layout in HBM ("CCF-H", half-spectrum, parity-compressed, k fastest):
//   tensor[slot][plane][jj][k']  plane 0 = Re, 1 = Im;  jj in [0,m/2), k' = (k&1)*n/2 + k/2
//   (rows of n along z with the even-k then odd-k halves, so a thread per (slot, k) walking jj
//   -- the radial recurrences -- coalesces across the warp, and each ADI k-parity block is a
//   contiguous half-row)
//   slot s < p/2  -> wavenumber w = s ; slot p/2 -> Nyquist w = -p/2 (reference slice l = 0)
//   coefficient (j, k) of slot s lives at jj = (j - j0)/2 where j0 = (w + cls) mod 2,
//   cls = 0 for scalar-parity fields (j+w even), 1 for azimuthal-flip fields
//   (proj/src/coeffs.cpp:50-59). The opposite-parity coefficients are identically
//   zero on the whole hot path, so they are not stored.
// A "full" slot table (slot = reference slice l, w = l - p/2) is also supported
// for API calls on non-Hermitian input.
#pragma once

#include <cstdint>

namespace ccf {

constexpr int kMaxSrc = 8;

// Per (solver set, slot) descriptor of the packed operator blocks (offsets in doubles).
struct AdiSlot {
    int J;        // shifts per round
    int j0;       // j-parity of the (scalar-class) unknowns of this slot
    int pivot;    // 1 if any banded LU of this slot row-swaps (selects the pivoted kernel path)
    int pad_;
    long left;    // J x (Mpad+2) x 16 : [mul(uC-A) -2..3 | L0 L1 | inv | piv | Uf0..Uf4 | 0]
                  //   unpivoted slots: fields 13..15 carry the spike vectors of the split
                  //   sweep (rows >= hc: F1 F2 ; rows < hc: G1 G2 G3), see adi.cu
    long right0;  // J x (Npad+2) x 12 (k-parity 0): [mul -1..2 | L | piv | inv | 0 | Uf0..Uf2 | 0]
                  //   unpivoted slots: field 7 = F (rows >= hr) / G1 (rows < hr), field 11 = G2
    long right1;  // J x N x 12  (k-parity 1)
    long sleft;   // M x 24      : [R2 -2..3 (first 0) | A -2..3 | C -2..3 | pad 6]
    long sright0; // N x 24      : [C02 -1..2 (first 0) | LU(B^T) as the right block fields 4..11 |
                  //                B^T -1..2 | D^T -1..2 | restart mul (v_0 B + D)^T -1..2]
    long sright1;
    long ds;      // J : u_j - v_j
};
constexpr int kLeftW = 16, kRightW = 12, kStatW = 24;

// Two-way partitioned sweeps (SPIKE): split row of a padded sweep length (multiple of 8),
// 0 = no split. Shared by the host builder (spike vectors) and the kernel.
__host__ __device__ inline int spike_split(int pad) { return pad >= 16 ? (pad / 16) * 8 : 0; }

struct AdiTask {
    int tensor, slot, k0, plane;
};

// Tensor geometry in the compressed layout.
struct Geo {
    int m, n, p, mh, nh, nslots;
    int M, N;           // (m-2)/2, (n-2)/2: reduced (Dirichlet-recombined) sizes per parity
    long plane_stride;  // n * mh
    long slot_stride;   // 2 * n * mh
};

// position of z-index k inside a row (parity split) and its inverse
__host__ __device__ __forceinline__ int kpos(int k, int nh) { return (k & 1) * nh + (k >> 1); }
__host__ __device__ __forceinline__ int kfrompos(int q, int nh) { return q < nh ? 2 * q : 2 * (q - nh) + 1; }

struct AdiParams {
    Geo g;
    int M, N, pitch, round, ntasks;
    const double* coef;
    const AdiSlot* slots;
    const AdiTask* tasks;
    const double* src[2][kMaxSrc];
    double wsrc[2][kMaxSrc];
    int nsrc[2];
    double* out[2];
    double* eprime;  // ntasks x estride scratch, rows padded to Mpad (multiple of 8)
    double* escr;    // ntasks x estride: E (residual)
    double* xscr;    // ntasks x estride: X of the last round (restart)
    long estride;    // doubles per task (Mpad * N rounded to even)
    int Mpad, Npad;  // M, N rounded up to multiples of 8 (zero-padded sweeps)
    int lanes;       // threads per line set: max(M, N) rounded up to a warp multiple
    int hc, hr;      // split row / column of the partitioned sweeps (0: sequential sweeps, lanes threads)
    int lrows, rrows;  // rows per left / right shift block (Mpad + 2, Npad + 2)
    double* res2;    // [2][nslots]
    double* e2;      // [2][nslots]
    const int* active;  // [2][nslots]
};

}  // namespace ccf
