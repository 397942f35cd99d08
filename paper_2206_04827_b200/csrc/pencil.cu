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

// b = d/dr a on a compressed pencil: in parity j0 -> out parity 1-j0 (calculus.cpp:7-19).
__device__ __forceinline__ void pen_dr(const double* __restrict__ in, double* __restrict__ out, int mh, int j0,
                                       double sg = 1.0) {
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
__device__ __forceinline__ void pen_divr(const double* __restrict__ in, double* __restrict__ out, int mh, int j0,
                                         const double* __restrict__ q) {
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

__device__ __forceinline__ void pen_axpy(double a, const double* __restrict__ x, double* __restrict__ y, int mh) {
    for (int i = 0; i < mh; ++i) y[i] = fma(a, x[i], y[i]);
}
__device__ __forceinline__ void pen_scale(double a, const double* __restrict__ x, double* __restrict__ y, int mh) {
    for (int i = 0; i < mh; ++i) y[i] = a * x[i];
}
__device__ __forceinline__ void pen_zero(double* __restrict__ y, int mh) {
    for (int i = 0; i < mh; ++i) y[i] = 0.0;
}

__device__ __forceinline__ int slot_w(int s, int p) { return s == p / 2 ? -p / 2 : s; }

// Horizontal Poisson on one compressed pencil (solvers.cpp:177-203):
//   cols = (R R C02) rhs, reduced = top (m-2) rows, LU(recombine(L_w)) solve, u = S y.
// hc: M rows x 8 [L, piv, inv, Uf0, Uf1, Uf2, 0, 0]; rc: M rows x 8 [RRC02 -1..3, 0, 0, 0].
__device__ __forceinline__ void pen_hp(const double* __restrict__ rhs, double sgn, double* __restrict__ out,
                                       double* __restrict__ y, int mh, int M, const double* __restrict__ hc,
                                       const double* __restrict__ rc) {
    // forward: y = L^-1 P (R R C02 rhs)
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
    for (int a = M - 1; a >= 0; --a) {
        const double* c = hc + a * 8;
        double acc = y[a] * c[2];
        for (int t = 0; t < 3; ++t)
            if (a + 1 + t < M) acc = fma(-c[3 + t], y[a + 1 + t], acc);
        y[a] = acc;
    }
    for (int i = 0; i < mh; ++i) out[i] = (i < M ? y[i] : 0.0) - (i >= 1 && i - 1 < M ? y[i - 1] : 0.0);
}

}  // namespace

// d/dz along k for compressed tensors (calculus.cpp:34-43): thread per (slot, plane, jj).
__global__ void dz_kernel(DzBatch d) {
    const Geo& g = d.g;
    const long per = long(g.nslots) * 2 * g.mh;
    const long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (i >= per * d.count) return;
    const int t = int(i / per);
    const long r = i % per;
    const int jj = int(r % g.mh);
    const long sp = r / g.mh;  // slot * 2 + plane
    const double* __restrict__ in = d.in[t] + sp * g.plane_stride + jj;
    double* __restrict__ out = d.out[t] + sp * g.plane_stride + jj;
    double next = 0.0, next2 = 0.0;
    for (int k = g.n - 1; k >= 0; --k) {
        const double ak1 = (k + 1 < g.n) ? in[long(k + 1) * g.mh] : 0.0;
        double bk = fma(2.0 * double(k + 1), ak1, next2);
        if (k == 0) bk *= 0.5;
        next2 = next;
        next = bk;
        out[long(k) * g.mh] = bk;
    }
}

// Stage V: pt_synthesize for `count` PT pairs (ptns.cpp:42-57), thread per (pair, slot, k).
//   V_r = D(dth lam) + dr(dz gam), V_t = D(dth dz gam) - dr lam, V_z = -(dr dr gam + D(dr gam + D(dth dth gam)))
__global__ void pt_synth_kernel(PtSynth a) {
    const Geo& g = a.g;
    const long per = long(g.nslots) * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= per * a.count) return;
    const int t = int(idx / per);
    const int s = int((idx % per) / g.n), k = int(idx % g.n);
    const int mh = g.mh, p = g.p;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);  // Q1: D_r keeps Re only
    const int j0s = w & 1;                      // scalar-class parity of lam, gam, dz gam
    const long o = long(s) * g.slot_stride + long(k) * mh, oi = o + g.plane_stride;
    const double *lr = a.lam[t] + o, *li = a.lam[t] + oi;
    const double *gr = a.gam[t] + o, *gi = a.gam[t] + oi;
    const double *zr = a.dzg[t] + o, *zi = a.dzg[t] + oi;
    double *vrr = a.vr[t] + o, *vri = a.vr[t] + oi;
    double *vtr = a.vt[t] + o, *vti = a.vt[t] + oi;
    double *vzr = a.vz[t] + o, *vzi = a.vz[t] + oi;
    double* s1 = a.scratch + idx * 2 * mh;
    double* s2 = s1 + mh;
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
        const double* gg = pl ? gi : gr;
        double* vz = pl ? vzi : vzr;
        pen_dr(gg, s1, mh, j0s);            // dr gam            (flip class)
        pen_dr(s1, vz, mh, 1 - j0s);        // dr dr gam         (scalar class)
        const bool dr_active = (pl == 0) || !pair;
        if (dr_active) {
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
// Optional outputs: the curl components (API curl_vector) and/or the PT scalars.
__global__ void curl_decomp_kernel(CurlDecomp a) {
    const Geo& g = a.g;
    const long per = long(g.nslots) * g.n;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= per) return;
    const int s = int(idx / g.n), k = int(idx % g.n);
    const int mh = g.mh, p = g.p;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0f = (w + 1) & 1;  // flip-class parity (a_r, a_t, out_r, out_t)
    const int j0s = 1 - j0f;
    const long o = long(s) * g.slot_stride + long(k) * mh, oi = o + g.plane_stride;
    const double fw = double(w);
    double* sc = a.scratch + idx * 6 * mh;
    double *s1 = sc, *s2 = sc + mh, *ozr = sc + 2 * mh, *ozi = sc + 3 * mh, *otr = sc + 4 * mh, *oti = sc + 5 * mh;
    if (a.out_z) {
        ozr = a.out_z + o;
        ozi = a.out_z + oi;
    }
    if (a.out_t) {
        otr = a.out_t + o;
        oti = a.out_t + oi;
    }
    const double *arr = a.ar + o, *ari = a.ar + oi, *atr = a.at + o, *ati = a.at + oi, *azr = a.az + o,
                 *azi = a.az + oi;
    const double *dzar = a.dzar ? a.dzar + o : nullptr, *dzai = a.dzar ? a.dzar + oi : nullptr;
    const double *dztr = a.dzat ? a.dzat + o : nullptr, *dzti = a.dzat ? a.dzat + oi : nullptr;
    double ori_buf = 0.0;
    (void)ori_buf;
    const double* vri = nullptr;  // out_r.im source for the decomposition
    if (a.decompose_only) {
        // pt_decompose(v) with v = (ar, at, az): out_z := v_z, out_t := v_t, out_r.im := v_r.im
        for (int i = 0; i < mh; ++i) {
            ozr[i] = azr[i];
            ozi[i] = azi[i];
            otr[i] = atr[i];
            oti[i] = ati[i];
        }
        vri = ari;
    } else {
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
            double *orr = a.out_r + o, *ori = a.out_r + oi;
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
    // gamma = HP(-out_z)
    pen_hp(ozr, -1.0, a.gam + o, s1, mh, g.M, hc, rc);
    pen_hp(ozi, -1.0, a.gam + oi, s1, mh, g.M, hc, rc);
    // cz = dr out_t + D(out_t - dth out_r);  (dth out_r).re = -w out_r.im = w dz a_t.im
    pen_dr(otr, ozr, mh, j0f);  // reuse the out_z storage as cz
    pen_dr(oti, ozi, mh, j0f);
    if (pair) {
        // (out_t - dth out_r).re = out_t.re + w out_r.im ; out_r.im = -dz a_t.im on the curl path
        if (vri)
            for (int i = 0; i < mh; ++i) s1[i] = fma(fw, vri[i], otr[i]);
        else
            for (int i = 0; i < mh; ++i) s1[i] = fma(-fw, dzti[i], otr[i]);
        pen_divr(s1, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, ozr, mh);
    } else {
        pen_divr(otr, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, ozr, mh);
        pen_divr(oti, s2, mh, j0f, a.q);
        pen_axpy(1.0, s2, ozi, mh);
    }
    pen_hp(ozr, -1.0, a.lam + o, s1, mh, g.M, hc, rc);
    pen_hp(ozi, -1.0, a.lam + oi, s1, mh, g.M, hc, rc);
}

// Standalone horizontal Poisson (API), thread per (slot, k).
__global__ void hp_kernel(HpArgs a) {
    const Geo& g = a.g;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= long(g.nslots) * g.n) return;
    const int s = int(idx / g.n), k = int(idx % g.n);
    const int w = slot_w(s, g.p);
    const int j0s = w & 1;
    const long o = long(s) * g.slot_stride + long(k) * g.mh;
    const double* hc = a.hpc + long(s) * g.M * 8;
    const double* rc = a.hpr + long(j0s) * g.M * 8;
    double* y = a.scratch + idx * g.mh;
    for (int pl = 0; pl < 2; ++pl) pen_hp(a.in + o + pl * g.plane_stride, 1.0, a.out + o + pl * g.plane_stride, y, g.mh, g.M, hc, rc);
}

// Generic per-slot calculus on one compressed class (API calculus.hpp), thread per (slot, k):
// op 0 dr, 2 dtheta, 4 divide_r (Q1), 5 horizontal_laplacian, 7 -laplacian-without-dzz helper.
__global__ void calc_kernel(CalcArgs a) {
    const Geo& g = a.g;
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= long(g.nslots) * g.n) return;
    const int s = int(idx / g.n), k = int(idx % g.n);
    const int mh = g.mh, p = g.p;
    const int w = slot_w(s, p);
    const bool pair = (w != 0 && s != p / 2);
    const int j0 = (w + a.cls) & 1;
    const long o = long(s) * g.slot_stride + long(k) * mh, oi = o + g.plane_stride;
    const double *xr = a.in + o, *xi = a.in + oi;
    double *yr = a.out + o, *yi = a.out + oi;
    double* s1 = a.scratch + idx * 3 * mh;
    double *s2 = s1 + mh, *s3 = s2 + mh;
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
                const double* x = pl ? xi : xr;
                double* y = pl ? yi : yr;
                pen_dr(x, s1, mh, j0);
                pen_dr(s1, y, mh, 1 - j0);
                const bool act = pl == 0 || !pair;
                if (!act) continue;
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
