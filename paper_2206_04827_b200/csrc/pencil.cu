// Radial / axial pencil operators of the poloidal-toroidal machinery, per Fourier
// slot, on the parity-compressed half-spectrum layout (ccf_device.cuh):
//   derivative_r / derivative_z   proj/src/calculus.cpp:7-43   (O(m) backward recurrences)
//   derivative_theta              proj/src/calculus.cpp:45-54
//   divide_r                      proj/src/calculus.cpp:71-97  (quirk Q1, see below)
//   pt_synthesize                 proj/src/ptns.cpp:42-57      (stage V of the NS step)
//   curl_vector + pt_decompose    proj/src/ptns.cpp:25-33,59-77 (stage C)
//   solve_horizontal_poisson      proj/src/solvers.cpp:177-203
//
// divide_r (Q1). The reference divides in value space after a full synthesis that
// keeps only the real part, separately for Re c and Im c. For a Hermitian tensor this
// is exactly the r-only operator D_r applied to Re c for 0 < w < p/2 (the imaginary
// part is dropped), and to both parts for w = 0 and the Nyquist slice. D_r itself is
// the interpolant of f(r_j)/r_j on the doubled grid (no r = 0 node for even m):
//   f odd in r : exact polynomial division, g_{k-1} = 2 f_k - g_{k+1}      (O(m))
//   f even     : f(0) * q + (f - f(0))/r, q = interpolant of 1/r_j          (O(m))
// which is what analyze(synthesize(f)/r) computes, without any transform.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace ccf {

namespace {

// A pencil along jj: element i at p[i * s] (s = n for tensor rows, = #threads for scratch,
// so consecutive threads touch consecutive addresses in both cases).
struct Pen {
    double* p;
    long s;
    __device__ __forceinline__ double& operator[](int i) const { return p[long(i) * s]; }
};
struct CPen {
    const double* p;
    long s;
    __device__ __forceinline__ double operator[](int i) const { return __ldg(p + long(i) * s); }
};

// b = d/dr a on a compressed pencil: in parity j0 -> out parity 1-j0 (calculus.cpp:7-19).
template <class I>
__device__ __forceinline__ void pen_dr(I in, Pen out, int mh, int j0, double sg = 1.0) {
    double b = 0.0;
    if (j0 == 0) {
        for (int i = mh - 1; i >= 0; --i) {
            if (i + 1 < mh) b = fma(double(4 * i + 4), in[i + 1], b);
            out[i] = sg * b;
        }
    } else {
        for (int i = mh - 1; i >= 0; --i) {
            b = fma(double(4 * i + 2), in[i], b);
            out[i] = sg * (i == 0 ? 0.5 * b : b);
        }
    }
}

// out = D_r(in): divide by r in value space, compressed parity j0 -> 1-j0.
template <class I>
__device__ __forceinline__ void pen_divr(I in, Pen out, int mh, int j0, const double* __restrict__ q) {
    if (j0 == 1) {  // odd -> even: exact division
        double gn = 0.0;
        for (int i = mh - 1; i >= 1; --i) {
            const double gv = fma(2.0, in[i], -gn);
            out[i] = gv;
            gn = gv;
        }
        out[0] = fma(-0.5, gn, in[0]);
    } else {  // even -> odd: f(0) q + (f - f(0)) / r
        double f0 = 0.0;
        for (int i = 0; i < mh; ++i) f0 += (i & 1) ? -in[i] : in[i];
        double h = 0.0;
        out[mh - 1] = f0 * q[mh - 1];
        for (int i = mh - 2; i >= 0; --i) {
            h = fma(2.0, in[i + 1], -h);
            out[i] = fma(f0, q[i], h);
        }
    }
}

template <class I>
__device__ __forceinline__ void pen_axpy(double a, I x, Pen y, int mh) {
    for (int i = 0; i < mh; ++i) y[i] = fma(a, x[i], y[i]);
}
__device__ __forceinline__ void pen_zero(Pen y, int mh) {
    for (int i = 0; i < mh; ++i) y[i] = 0.0;
}

__device__ __forceinline__ int slot_w(int s, int p) { return s == p / 2 ? -p / 2 : s; }

// Horizontal Poisson on one compressed pencil (solvers.cpp:177-203):
//   cols = (R R C02) rhs, reduced = top (m-2) rows, LU(recombine(L_w)) solve, u = S y.
// hc: M rows x 8 [L, piv, inv, Uf0, Uf1, Uf2, 0, 0]; rc: M rows x 8 [RRC02 -1..3, 0, 0, 0].
template <class I>
__device__ __forceinline__ void pen_hp(I rhs, double sgn, Pen out, Pen y, int mh, int M, const double* __restrict__ hc,
                                       const double* __restrict__ rc) {
    for (int a = 0; a < M; ++a) {
        const double* c = rc + a * 8;
        double acc = 0.0;
        for (int d = -1; d <= 3; ++d) {
            const int i = a + d;
            if (i >= 0 && i < mh) acc = fma(c[d + 1], rhs[i], acc);
        }
        y[a] = sgn * acc;
    }
    for (int a = 0; a < M; ++a) {
        const double* c = hc + a * 8;
        if (c[1] == 1.0 && a + 1 < M) {
            const double t = y[a];
            y[a] = y[a + 1];
            y[a + 1] = t;
        }
        if (a + 1 < M) y[a + 1] = fma(-c[0], y[a], y[a + 1]);
    }
    double x1 = 0.0, x2 = 0.0, x3 = 0.0;
    for (int a = M - 1; a >= 0; --a) {
        const double* c = hc + a * 8;
        double acc = y[a] * c[2];
        acc = fma(-c[5], x3, acc);
        acc = fma(-c[4], x2, acc);
        acc = fma(-c[3], x1, acc);
        y[a] = acc;
        x3 = x2;
        x2 = x1;
        x1 = acc;
    }
    double prev = 0.0;
    for (int i = 0; i < mh; ++i) {
        const double cur = i < M ? y[i] : 0.0;
        out[i] = cur - prev;
        prev = cur;
    }
}

}  // namespace

// d/dz along k for compressed tensors (calculus.cpp:34-43), one warp per row (slot, plane, jj).
// The recurrence b_k = b_{k+2} + 2(k+1) a_{k+1} (b_0 halved) is a suffix sum over the opposite
// parity half of the row:  b_{2q} = S_odd(q),  b_{2q+1} = S_even(q+1), with
// S_odd(i) = sum_{i' >= i} 2(2i'+1) a_{2i'+1},  S_even(i) = sum_{i' >= i} 4 i' a_{2i'};
// warp suffix scans over coalesced 32-element chunks of the contiguous half rows.
__global__ void __launch_bounds__(256) dz_kernel(DzBatch d) {
    const Geo& g = d.g;
    const int n = g.n, nh = g.nh;
    const long rows_per = long(g.nslots) * 2 * g.mh;
    const long wid = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= rows_per * d.count) return;
    const int t = int(wid / rows_per);
    const long row = wid % rows_per;
    const double* __restrict__ in = d.in[t] + row * n;
    double* __restrict__ out = d.out[t] + row * n;
    for (int half = 0; half < 2; ++half) {  // half 0: outputs b_even from a_odd; half 1: b_odd from a_even
        double carry = 0.0;
        const int nchunk = (nh + 31) / 32;
        for (int ch = nchunk - 1; ch >= 0; --ch) {
            const int i = ch * 32 + lane;
            double c = 0.0;
            if (i < nh) {
                if (half == 0) c = 2.0 * double(2 * i + 1) * in[nh + i];  // a_{2i+1}
                else c = 4.0 * double(i) * in[i];                          // a_{2i}
            }
            double v = c;
            for (int o = 1; o < 32; o <<= 1) {
                const double u = __shfl_down_sync(0xffffffffu, v, o);
                if (lane + o < 32) v += u;
            }
            const double total = __shfl_sync(0xffffffffu, v, 0);
            const double S = v + carry;  // suffix sum from i to the end
            if (i < nh) {
                if (half == 0) out[i] = (i == 0) ? 0.5 * S : S;  // b_{2i}
                else out[nh + i] = S - c;                        // b_{2i+1} = S_even(i+1)
            }
            carry += total;
        }
    }
}

// Thread mapping of the pencil kernels: idx -> (t, slot, q) with q the position inside the
// row (k = kfrompos(q)); consecutive threads touch consecutive addresses of every pencil.
struct PIdx {
    int t, s, q, k;
};
__device__ __forceinline__ PIdx pidx(long idx, const Geo& g) {
    const long per = long(g.nslots) * g.n;
    PIdx r;
    r.t = int(idx / per);
    r.s = int((idx % per) / g.n);
    r.q = int(idx % g.n);
    r.k = kfrompos(r.q, g.nh);
    return r;
}

// Stage V: pt_synthesize for `count` PT pairs (ptns.cpp:42-57), thread per (pair, slot, k).
//   V_r = D(dth lam) + dr(dz gam), V_t = D(dth dz gam) - dr lam, V_z = -(dr dr gam + D(dr gam + D(dth dth gam)))
__global__ void pt_synth_kernel(PtSynth a) {
    const Geo& g = a.g;
    const long NT = long(a.count) * g.nslots * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= NT) return;
    const PIdx ix = pidx(idx, g);
    const int t = ix.t, s = ix.s;
    const int mh = g.mh, p = g.p;
    const long n = g.n;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);  // Q1: D_r keeps Re only
    const int j0s = w & 1;                      // scalar-class parity of lam, gam, dz gam
    const long o = long(s) * g.slot_stride + ix.q, oi = o + g.plane_stride;
    const CPen lr{a.lam[t] + o, n}, li{a.lam[t] + oi, n}, gr{a.gam[t] + o, n}, gi{a.gam[t] + oi, n};
    const CPen zr{a.dzg[t] + o, n}, zi{a.dzg[t] + oi, n};
    const Pen vrr{a.vr[t] + o, n}, vri{a.vr[t] + oi, n}, vtr{a.vt[t] + o, n}, vti{a.vt[t] + oi, n};
    const Pen vzr{a.vz[t] + o, n}, vzi{a.vz[t] + oi, n};
    const Pen s1{a.scratch + idx, NT}, s2{a.scratch + NT * mh + idx, NT};
    const double fw = double(w);
    // V_r
    pen_dr(zr, vrr, mh, j0s);
    pen_dr(zi, vri, mh, j0s);
    if (pair) {
        pen_divr(li, s1, mh, j0s, a.q);  // D(dth lam).re = -w D(lam.im)
        pen_axpy(-fw, s1, vrr, mh);
    }
    // V_t
    pen_dr(lr, vtr, mh, j0s, -1.0);
    pen_dr(li, vti, mh, j0s, -1.0);
    if (pair) {
        pen_divr(zi, s1, mh, j0s, a.q);  // D(dth dz gam).re = -w D(dz gam.im)
        pen_axpy(-fw, s1, vtr, mh);
    }
    // V_z (real plane, then imaginary plane)
    for (int pl = 0; pl < 2; ++pl) {
        const CPen gg = pl ? gi : gr;
        const Pen vz = pl ? vzi : vzr;
        pen_dr(gg, s1, mh, j0s);      // dr gam            (flip class)
        pen_dr(s1, vz, mh, 1 - j0s);  // dr dr gam         (scalar class)
        if (pl == 0 || !pair) {
            // inner = dr gam + D(dth dth gam) ; dth dth gam = -w^2 gam (0 for w = 0 / Nyquist)
            if (pair) {
                pen_divr(gg, s2, mh, j0s, a.q);
                pen_axpy(-fw * fw, s2, s1, mh);
            }
            pen_divr(s1, s2, mh, 1 - j0s, a.q);  // D(inner)
            for (int i = 0; i < mh; ++i) vz[i] = -(vz[i] + s2[i]);
        } else {
            for (int i = 0; i < mh; ++i) vz[i] = -vz[i];
        }
    }
}

// Stage C: curl_vector (ptns.cpp:25-33) of a = (a_r, a_t, a_z) followed by pt_decompose
// without the divergence check (ptns.cpp:59-77, as called from nonlinear_term):
//   out_z = dr a_t + D(a_t - dth a_r);  out_t = dz a_r - dr a_z;  out_r = D(dth a_z) - dz a_t
//   gamma = HP(-out_z);  lambda = HP(-(dr out_t + D(out_t - dth out_r)))
// decompose_only: (a_r, a_t, a_z) are already (v_r, v_t, v_z) (API pt_decompose).
__global__ void curl_decomp_kernel(CurlDecomp a) {
    const Geo& g = a.g;
    const long NT = long(g.nslots) * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= NT) return;
    const PIdx ix = pidx(idx, g);
    const int s = ix.s;
    const int mh = g.mh, p = g.p;
    const long n = g.n;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0f = (w + 1) & 1;  // flip-class parity (a_r, a_t, out_r, out_t)
    const int j0s = 1 - j0f;
    const long o = long(s) * g.slot_stride + ix.q, oi = o + g.plane_stride;
    const double fw = double(w);
    auto spen = [&](int i) { return Pen{a.scratch + NT * mh * i + idx, NT}; };
    const Pen s1 = spen(0), s2 = spen(1);
    Pen ozr = spen(2), ozi = spen(3), otr = spen(4), oti = spen(5);
    if (a.out_z) {
        ozr = Pen{a.out_z + o, n};
        ozi = Pen{a.out_z + oi, n};
    }
    if (a.out_t) {
        otr = Pen{a.out_t + o, n};
        oti = Pen{a.out_t + oi, n};
    }
    const CPen arr{a.ar + o, n}, ari{a.ar + oi, n}, atr{a.at + o, n}, ati{a.at + oi, n}, azr{a.az + o, n},
        azi{a.az + oi, n};
    const bool dec = a.decompose_only != 0;
    if (dec) {
        for (int i = 0; i < mh; ++i) {
            ozr[i] = azr[i];
            ozi[i] = azi[i];
            otr[i] = atr[i];
            oti[i] = ati[i];
        }
    } else {
        const CPen dzar{a.dzar + o, n}, dzai{a.dzar + oi, n}, dztr{a.dzat + o, n}, dzti{a.dzat + oi, n};
        // out_z
        pen_dr(atr, ozr, mh, j0f);
        pen_dr(ati, ozi, mh, j0f);
        if (pair) {
            for (int i = 0; i < mh; ++i) s1[i] = fma(fw, ari[i], atr[i]);  // (a_t - dth a_r).re
            pen_divr(s1, s2, mh, j0f, a.q);
            pen_axpy(1.0, s2, ozr, mh);
        } else {
            pen_divr(atr, s2, mh, j0f, a.q);
            pen_axpy(1.0, s2, ozr, mh);
            pen_divr(ati, s2, mh, j0f, a.q);
            pen_axpy(1.0, s2, ozi, mh);
        }
        // out_t = dz a_r - dr a_z
        pen_dr(azr, otr, mh, j0s);
        pen_dr(azi, oti, mh, j0s);
        for (int i = 0; i < mh; ++i) {
            otr[i] = dzar[i] - otr[i];
            oti[i] = dzai[i] - oti[i];
        }
        // out_r (API only): re = D(dth a_z).re - dz a_t.re, im = D(dth a_z).im - dz a_t.im
        if (a.out_r) {
            const Pen orr{a.out_r + o, n}, ori{a.out_r + oi, n};
            if (pair) {
                pen_divr(azi, s1, mh, j0s, a.q);
                for (int i = 0; i < mh; ++i) {
                    orr[i] = -fw * s1[i] - dztr[i];
                    ori[i] = -dzti[i];
                }
            } else {
                for (int i = 0; i < mh; ++i) {
                    orr[i] = -dztr[i];
                    ori[i] = -dzti[i];
                }
            }
        }
    }
    if (!a.lam) return;
    const double* hc = a.hpc + long(s) * g.M * 8;
    const double* rc = a.hpr + long(j0s) * g.M * 8;
    const Pen gr{a.gam + o, n}, gi{a.gam + oi, n}, lr{a.lam + o, n}, li{a.lam + oi, n};
    // gamma = HP(-out_z)
    pen_hp(ozr, -1.0, gr, s1, mh, g.M, hc, rc);
    pen_hp(ozi, -1.0, gi, s1, mh, g.M, hc, rc);
    // cz = dr out_t + D(out_t - dth out_r); (dth out_r).re = -w out_r.im
    const Pen czr = spen(2), czi = spen(3);
    pen_dr(otr, czr, mh, j0f);
    pen_dr(oti, czi, mh, j0f);
    if (pair) {
        // out_r.im = v_r.im (decompose) or -dz a_t.im (curl path)
        if (dec) {
            for (int i = 0; i < mh; ++i) s1[i] = fma(fw, ari[i], otr[i]);
        } else {
            const CPen dzti{a.dzat + oi, n};
            for (int i = 0; i < mh; ++i) s1[i] = fma(-fw, dzti[i], otr[i]);
        }
        pen_divr(s1, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, czr, mh);
    } else {
        pen_divr(otr, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, czr, mh);
        pen_divr(oti, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, czi, mh);
    }
    pen_hp(czr, -1.0, lr, s1, mh, g.M, hc, rc);
    pen_hp(czi, -1.0, li, s1, mh, g.M, hc, rc);
}

// Standalone horizontal Poisson (API), thread per (slot, k).
__global__ void hp_kernel(HpArgs a) {
    const Geo& g = a.g;
    const long NT = long(g.nslots) * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= NT) return;
    const PIdx ix = pidx(idx, g);
    const int w = slot_w(ix.s, g.p);
    const int j0s = w & 1;
    const long o = long(ix.s) * g.slot_stride + ix.q;
    const double* hc = a.hpc + long(ix.s) * g.M * 8;
    const double* rc = a.hpr + long(j0s) * g.M * 8;
    const Pen y{a.scratch + idx, NT};
    for (int pl = 0; pl < 2; ++pl)
        pen_hp(CPen{a.in + o + pl * g.plane_stride, g.n}, 1.0, Pen{a.out + o + pl * g.plane_stride, g.n}, y, g.mh,
               g.M, hc, rc);
}

// Generic per-slot calculus on one compressed class (API calculus.hpp), thread per (slot, k):
// op 0 dr, 2 dtheta, 4 divide_r (Q1), 5 horizontal_laplacian.
__global__ void calc_kernel(CalcArgs a) {
    const Geo& g = a.g;
    const long NT = long(g.nslots) * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= NT) return;
    const PIdx ix = pidx(idx, g);
    const int s = ix.s;
    const int mh = g.mh, p = g.p;
    const long n = g.n;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0 = (w + a.cls) & 1;
    const long o = long(s) * g.slot_stride + ix.q, oi = o + g.plane_stride;
    const CPen xr{a.in + o, n}, xi{a.in + oi, n};
    const Pen yr{a.out + o, n}, yi{a.out + oi, n};
    const Pen s1{a.scratch + idx, NT}, s2{a.scratch + NT * mh + idx, NT}, s3{a.scratch + 2 * NT * mh + idx, NT};
    const double fw = double(w);
    switch (a.op) {
        case 0:
            pen_dr(xr, yr, mh, j0);
            pen_dr(xi, yi, mh, j0);
            break;
        case 2:
            for (int i = 0; i < mh; ++i) {
                const double re = xr[i], im = xi[i];
                yr[i] = s == p / 2 ? 0.0 : -fw * im;
                yi[i] = s == p / 2 ? 0.0 : fw * re;
            }
            break;
        case 4:
            pen_divr(xr, yr, mh, j0, a.q);
            if (pair) pen_zero(yi, mh);
            else pen_divr(xi, yi, mh, j0, a.q);
            break;
        case 5: {  // dr dr f + D(dr f + D(dth dth f))
            for (int pl = 0; pl < 2; ++pl) {
                const CPen x = pl ? xi : xr;
                const Pen y = pl ? yi : yr;
                pen_dr(x, s1, mh, j0);
                pen_dr(s1, y, mh, 1 - j0);
                if (!(pl == 0 || !pair)) continue;
                if (pair) {
                    pen_divr(x, s2, mh, j0, a.q);
                    pen_axpy(-fw * fw, s2, s1, mh);
                }
                pen_divr(s1, s3, mh, 1 - j0, a.q);
                pen_axpy(1.0, s3, y, mh);
            }
            break;
        }
        default:
            break;
    }
}

}  // namespace ccf
