// The NS step's dense product stages on the INT8 tensor cores (Ozaki splitting, ozaki.hpp):
//   H   eigen back transforms Y = Z (QR S_z), Z (QR D_z S_z)           (Pipeline::eigen_ysynth)
//   X1  composite r synthesis of the six velocity / vorticity fields    (Pipeline::nonlinear, eigY)
//   X3  z analysis of the cross product (PR folded in)                  (Pipeline::nonlinear, eig)
//   C   composite curl / decompose / r analysis (PL_P folded in)        (Pipeline::nonlinear, eig)
// Constant operands (QS / QD, AzP / ADzP, the composite blocks) are split once; the data operands are
// split every step by the split kernels (rows for an A operand, transposed columns for a B operand).
// The data B operands (X1, C) are split with one power-of-two scale per (plane, 128-column tile) and
// unit column scales (the row scales of every term's A carry the plane scale): one pass, no column
// scales to share between the terms of an output tile.
// Enabled at m = n = 256 (every reduction is one 128-long panel); CCF_OZAKI=0 selects the FP64 DMMA
// GEMMs (transform.cu). Plans are keyed by their pointers like the GemmPlans and never built inside a
// CUDA-graph capture (the stage then falls back to the DMMA path).
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"
#include "ozaki.hpp"
#include "pipeline.hpp"

namespace ccf {

struct OzPipe::Stage {
    OzSplitPlan split;
    OzGemmPlan gemm;
};

namespace {
uint8_t* bytes(DBuf& b) { return reinterpret_cast<uint8_t*>(b.p); }
int* ints(DBuf& b) { return reinterpret_cast<int*>(b.p); }
void alloc_bytes(DBuf& b, size_t n) { b.alloc((n + 7) / 8); }
bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}
std::string key_of(const char* tag, std::initializer_list<const void*> ptrs) {
    std::string k(tag);
    for (const void* p : ptrs) k += ":" + std::to_string(reinterpret_cast<uintptr_t>(p));
    return k;
}
constexpr size_t kPanel128 = size_t(kOzS) * 128 * kOzK;  // bytes of a 128-row panel
constexpr size_t kPanel256 = 2 * kPanel128;               // a 256-row panel (two column tiles)
}  // namespace

OzPipe::OzPipe(Pipeline& p) : P(p) {
    const Geo& g = P.c.gh;
    const char* e = std::getenv("CCF_OZAKI");
    const bool want = !(e && e[0] == '0');
    const int Np = P.c.N + (P.c.N & 1);
    on = want && g.mh == 128 && g.nh == 128 && g.n == 256 && P.c.M <= 128 && P.c.N <= 128 && Np == 128;
    const char* m = std::getenv("CCF_OZ_STAGES");  // diagnostics: bit 0 H, bit 1 X1, bit 2 X3 + C
    mask = m ? std::atoi(m) : 7;
}
OzPipe::~OzPipe() = default;

// MN-major B panels (256 rows = two 128-column tiles per (slot, plane)) standing for an fp64 tensor
// of the pipeline: written by the producing product's epilogue, read by the next product
OzPipe::Panels& OzPipe::panels(const double* buf) {
    Panels& p = panels_[buf];
    const int ns = P.c.sh.s_hi - P.c.sh.s_lo;
    const size_t bytes_needed = size_t(ns) * 2 * kPanel256;
    if (p.pan.n * 8 < bytes_needed) {
        alloc_bytes(p.pan, bytes_needed);
        p.pe.alloc(size_t(ns) * 2);  // [slot][plane][2 tiles] ints
    }
    return p;
}

OzPipe::Stage* OzPipe::stage(const std::string& key, bool& fresh) {
    auto& s = stages_[key];
    fresh = !s;
    if (fresh) {
        if (capturing(P.c.stream)) {
            stages_.erase(key);
            return nullptr;
        }
        s = std::make_unique<Stage>();
    }
    return s.get();
}

bool OzPipe::ensure_const() {
    if (const_set_ == P.eig_set_) return true;
    if (capturing(P.c.stream) || !P.eig_set_) return false;
    const Geo& g = P.c.gh;
    const int M = P.c.M, N = P.c.N, mh = g.mh, nh = g.nh;
    const int Np = N + (N & 1);
    // panel map: QS[2], QD[2], AzP[2], ADzP[2], then the X1 (synthesis) and C (analysis) blocks
    const size_t nsyn = P.synth_.blocks.size() / size_t(mh * mh), nana = P.anal_.blocks.size() / size_t(mh * mh);
    const size_t npan = 8 + nsyn + nana;
    alloc_bytes(cpan_, npan * kPanel128);
    csc_.alloc(npan * 128);
    cpe_.alloc(8);  // plane exponents of the 8 transposed (B) panels, one tile each
    CCF_CUDA(cudaMemsetAsync(cpan_.p, 0, cpan_.n * 8, P.c.stream));
    OzSplitPlan rows, cols;
    cols.transpose = true;  // B panels: K-major, one scale per column (the constant operators keep full precision)
    auto pan = [&](size_t i) { return bytes(cpan_) + i * kPanel128; };
    auto sc = [&](size_t i) { return csc_.p + i * 128; };
    auto cpe = [&](size_t i) { return ints(cpe_) + i; };
    const long st = long(oz_slice_bytes(128));
    for (int k0 = 0; k0 < 2; ++k0) {
        // B operands (rows = output columns, K = reduction index): QS / QD are N x nh (K = j), AzP / ADzP nh x Np (K = q)
        cols.jobs.push_back(oz_job(P.eig_QS_.p + size_t(k0) * N * nh, nh, nh, N, pan(k0), sc(k0), st, 128, cpe(k0)));
        cols.jobs.push_back(oz_job(P.eig_QD_.p + size_t(k0) * N * nh, nh, nh, N, pan(2 + k0), sc(2 + k0), st, 128, cpe(2 + k0)));
        cols.jobs.push_back(oz_job(P.eig_AzP_.p + size_t(k0) * nh * Np, Np, N, nh, pan(4 + k0), sc(4 + k0), st, 128, cpe(4 + k0)));
        cols.jobs.push_back(oz_job(P.eig_ADzP_.p + size_t(k0) * nh * Np, Np, N, nh, pan(6 + k0), sc(6 + k0), st, 128, cpe(6 + k0)));
    }
    // A operands: composite synthesis blocks (mh x mh, QL folded: the pad column is zero) and the PL_P-folded
    // curl / decompose blocks (M x mh); panel index 8 + block offset / mh^2
    for (size_t b = 0; b < nsyn; ++b)
        rows.jobs.push_back(oz_job(P.dsynth_eig_.p + b * mh * mh, mh, mh, mh, pan(8 + b), sc(8 + b), st, 128));
    for (size_t b = 0; b < nana; ++b)
        rows.jobs.push_back(oz_job(P.eig_anal_.p + b * mh * mh, mh, M, mh, pan(8 + nsyn + b), sc(8 + nsyn + b), st, 128));
    rows.upload();
    cols.upload();
    rows.launch(P.c.stream);
    cols.launch(P.c.stream);
    CCF_CUDA(cudaStreamSynchronize(P.c.stream));
    syn0_ = 8;
    ana0_ = 8 + nsyn;
    const_set_ = P.eig_set_;
    stages_.clear();  // plans reference the panels of the previous modal basis
    return true;
}

// ---- H: Y_S[t] = Z_t QS[k0] into value half k0, Y_D[t] = Z_t QD[k0] into half 1 - k0 (Pipeline::eigen_ysynth)
bool OzPipe::ysynth(int ntensor, const double* const* z, double* const* outS, double* const* outD) {
    for (int t = 0; t < ntensor; ++t) {  // a DMMA fallback writes fp64 tensors
        if (outS[t]) panel_only_.erase(outS[t]);
        if (outD[t]) panel_only_.erase(outD[t]);
    }
    if (!on || !(mask & 1) || !(mask & 2) || !ensure_const()) return false;
    const Geo& g = P.c.gh;
    const int M = P.c.M, N = P.c.N, nh = g.nh;
    const int s_lo = P.c.sh.s_lo, s_hi = P.c.sh.s_hi, ns = s_hi - s_lo;
    const void* z1 = ntensor > 1 ? z[1] : nullptr;
    const void* z2 = ntensor > 2 ? z[2] : nullptr;
    const void* o1 = ntensor > 1 ? outS[1] : nullptr;
    const void* o2 = ntensor > 2 ? outS[2] : nullptr;
    const void* d1 = ntensor > 1 ? outD[1] : nullptr;
    const void* d2 = ntensor > 2 ? outD[2] : nullptr;
    bool fresh;
    Stage* sp = stage(key_of("ys_split", {z[0], z1, z2}), fresh);
    if (!sp) return false;
    // data panels: (t, slot, pl, k0), 128 rows each
    const size_t need = size_t(3) * ns * 4 * kPanel128;
    if (fresh) {
        if (ysp_.n * 8 < need) {
            alloc_bytes(ysp_, need);
            ysc_.alloc(size_t(3) * ns * 4 * 128);
            CCF_CUDA(cudaMemsetAsync(ysp_.p, 0, ysp_.n * 8, P.c.stream));
        }
        for (int t = 0; t < ntensor; ++t)
            for (int s = s_lo; s < s_hi; ++s)
                for (int pl = 0; pl < 2; ++pl)
                    for (int k0 = 0; k0 < 2; ++k0) {
                        const size_t i = ((size_t(t) * ns + (s - s_lo)) * 2 + pl) * 2 + k0;
                        sp->split.jobs.push_back(oz_job(z[t] + P.eig_off(s, pl, k0), 2 * 128, M, N, bytes(ysp_) + i * kPanel128,
                                                        ysc_.p + i * 128, long(oz_slice_bytes(128)), 128));
                    }
        sp->split.upload();
    }
    Stage* gp = stage(key_of("ys_gemm", {outS[0], outD[0], o1, d1, o2, d2, reinterpret_cast<const void*>(size_t(ntensor))}),
                      fresh);
    if (!gp) return false;
    if (fresh) {
        for (int t = 0; t < ntensor; ++t)
            for (int s = s_lo; s < s_hi; ++s)
                for (int pl = 0; pl < 2; ++pl)
                    for (int k0 = 0; k0 < 2; ++k0) {
                        const size_t i = ((size_t(t) * ns + (s - s_lo)) * 2 + pl) * 2 + k0;
                        const long off = long(s) * g.slot_stride + long(pl) * g.plane_stride;
                        for (int dd = 0; dd < 2; ++dd) {
                            double* out = dd ? outD[t] : outS[t];
                            if (!out) continue;
                            const int cp = dd ? 2 + k0 : k0;  // QD[k0] / QS[k0] panel
                            const int t0 = int(gp->gemm.terms.size());
                            gp->gemm.terms.push_back({bytes(ysp_) + i * kPanel128, bytes(cpan_) + size_t(cp) * kPanel128,
                                                      ysc_.p + i * 128, csc_.p + size_t(cp) * 128, long(oz_slice_bytes(128)),
                                                      ints(cpe_) + cp});
                            OzItem item{t0, t0 + 1, 0, M, nh, 0, out + off + long(dd ? 1 - k0 : k0) * nh, long(g.n), 1.0};
                            // the value half of this tile as the X1 product's B panel tile (no fp64 tensor)
                            Panels& pp = panels(out);
                            const size_t pi = size_t(s - s_lo) * 2 + pl;
                            const int h = dd ? 1 - k0 : k0;
                            item.pdst = bytes(pp.pan) + pi * kPanel256 + size_t(h) * 128 * kOzK;
                            item.pstride = long(oz_slice_bytes(256));
                            item.ppe = ints(pp.pe) + pi * 2 + h;
                            gp->gemm.items.push_back(item);
                        }
                    }
        gp->gemm.tag = "H";
        gp->gemm.upload();
    }
    const bool written = rhs_split_ == key_of("ys_split", {z[0], z1, z2});  // by the RHS pass just before
    rhs_split_.clear();
    if (!written) sp->split.launch(P.c.stream);
    P.c.mark("H_z_split");
    gp->gemm.launch(P.c.stream);
    P.c.gemm_flops += gp->gemm.flops;
    P.c.launches += written ? 1 : 2;
    for (int t = 0; t < ntensor; ++t) {  // these tensors now exist as panels only (rsynth reads them)
        if (outS[t]) panel_only_.insert(outS[t]);
        if (outD[t]) panel_only_.insert(outD[t]);
    }
    return true;
}

bool OzPipe::rhs_panels(const double* z0, const double* z1, const double* z2, EigRhs& a) {
    rhs_split_.clear();
    if (!on || !(mask & 1) || !(mask & 2) || const_set_ != P.eig_set_ || !z0 || !z1 || !z2) return false;
    const std::string key = key_of("ys_split", {z0, z1, z2});
    if (!stages_.count(key) || !stages_[key]) return false;  // built by ysynth's first (eager) call
    const int ns = P.c.sh.s_hi - P.c.sh.s_lo;
    for (int t = 0; t < 3; ++t) {  // panel index ((t ns + s - s_lo) 2 + pl) 2 + k0, as in ysynth
        a.pan[t] = bytes(ysp_) + size_t(t) * ns * 4 * kPanel128;
        a.psc[t] = ysc_.p + size_t(t) * ns * 4 * 128;
    }
    rhs_split_ = key;
    return true;
}

// ---- X1: val[3 pr + o/2] plane o%2 = sum_terms (C_t QL)(Y[pr][in]) (composite synthesis, eigen rows)
bool OzPipe::rsynth(double* const (&Z)[2][3], double* const* val) {
    bool all_panels = true;
    for (int pr = 0; pr < 2; ++pr)
        for (int x = 0; x < 3; ++x) all_panels &= panel_only_.count(Z[pr][x]) > 0;
    if (!on || !(mask & 2) || !ensure_const()) {
        if (all_panels) throw Error(INTERNAL, "OzPipe: the X1 inputs exist as INT8 panels only");
        return false;
    }
    if (!all_panels) return false;  // (fp64 inputs: the DMMA plan)
    const Geo& g = P.c.gh;
    const int mh = g.mh;
    const int s_lo = P.c.sh.s_lo, s_hi = P.c.sh.s_hi;
    bool fresh;
    const bool quad = P.theta_quad_ok();  // (the pipeline passes the layout to theta_cross)
    Stage* sp = stage(key_of(quad ? "rsq" : "rs", {Z[0][0], Z[0][1], Z[0][2], Z[1][0], Z[1][1], Z[1][2], val[0], val[3]}), fresh);
    if (!sp) throw Error(INTERNAL, "OzPipe: X1 plan first built during a graph capture");
    if (fresh) {
        // item order (s, o, nt, pr): the four items that read one composite block (and the items that read
        // one input panel) are adjacent, so they run concurrently on neighbouring CTAs and share it through L2;
        // the kernel's upload() only regroups them by term count (stable)
        for (int s = s_lo; s < s_hi; ++s)
            for (int o = 0; o < 6; ++o)
                for (int nt = 0; nt < 2; ++nt)
                    for (int pr = 0; pr < 2; ++pr) {
                        const int t0 = int(sp->gemm.terms.size());
                        for (const CompositeTerm& ct : P.synth_.terms[size_t(s)]) {
                            if (ct.out != o) continue;
                            const size_t bi = size_t(syn0_) + size_t(ct.off) / size_t(mh * mh);
                            Panels& pp = panels(Z[pr][ct.in / 2]);
                            const size_t pi = size_t(s - s_lo) * 2 + ct.in % 2;
                            sp->gemm.terms.push_back({bytes(cpan_) + bi * kPanel128, bytes(pp.pan) + pi * kPanel256,
                                                      csc_.p + bi * 128, nullptr, long(oz_slice_bytes(256)), ints(pp.pe) + pi * 2});
                        }
                        // (an output no block feeds is an item without terms: the kernel stores zeros)
                        const int t1 = int(sp->gemm.terms.size());
                        double* plane = val[3 * pr + o / 2] + long(s) * g.slot_stride + long(o % 2) * g.plane_stride;
                        OzItem item{t0, t1, nt * 128, mh, 128, 0, plane + nt * 128, long(g.n), 1.0};
                        if (quad) {  // column-quad-major values for the theta kernel (Pipeline::val_quad_)
                            item.cq = 4L * mh;
                            item.c = plane + long(nt * 128 / 4) * item.cq;
                        }
                        sp->gemm.items.push_back(item);
                    }
        sp->gemm.b_mn = true;
        sp->gemm.tag = "X1";
        sp->gemm.upload();
    }
    sp->gemm.launch(P.c.stream);
    P.c.gemm_flops += sp->gemm.flops;
    P.c.launches += 1;
    return true;
}

// ---- X3 + C: Y[x] = av (Az PR) per half, then N~ = sum_terms (PL_P A_t) Y[in] (eigen layout outputs)
bool OzPipe::analyze(double* const* av, double* const* Y, double* lam_n, double* gam_n) {
    if (!on || !(mask & 4) || !ensure_const()) return false;
    const Geo& g = P.c.gh;
    const int M = P.c.M, mh = g.mh, nh = g.nh;
    const int Np = P.c.N + (P.c.N & 1);
    const int s_lo = P.c.sh.s_lo, s_hi = P.c.sh.s_hi, ns = s_hi - s_lo;
    bool fresh;
    // C: B = the Y planes (rows = r rows jr = K, columns k0 Np + j) as MN-major panels, written by X3's epilogue
    const size_t pb = kPanel256;
    auto rpan = [&](int s, int in) { return bytes(rap_) + (size_t(s - s_lo) * 10 + in) * pb; };
    if (rap_.n * 8 < size_t(ns) * 10 * pb) {
        alloc_bytes(rap_, size_t(ns) * 10 * pb);
        rape_.alloc(size_t(ns) * 10);  // [slot][10 planes][2 tiles] ints
    }
    // X3: A = av rows (slot, plane, r row) x one z half; B = AzP / ADzP [po]
    Stage* za = stage(key_of("za", {av[0], av[1], av[2], Y[0], Y[4]}), fresh);
    if (!za) return false;
    if (fresh) {
        const size_t need = size_t(3) * ns * 4 * kPanel128;
        if (zap_.n * 8 < need) {
            alloc_bytes(zap_, need);
            zasc_.alloc(size_t(3) * ns * 4 * 128);
        }
        auto idx = [&](int f, int s, int pl, int pi) { return ((size_t(f) * ns + (s - s_lo)) * 2 + pl) * 2 + pi; };
        for (int f = 0; f < 3; ++f)
            for (int s = s_lo; s < s_hi; ++s)
                for (int pl = 0; pl < 2; ++pl)
                    for (int pi = 0; pi < 2; ++pi) {
                        const size_t i = idx(f, s, pl, pi);
                        za->split.jobs.push_back(oz_job(av[f] + long(s) * g.slot_stride + long(pl) * g.plane_stride + pi * nh, g.n,
                                                        mh, nh, bytes(zap_) + i * kPanel128, zasc_.p + i * 128,
                                                        long(oz_slice_bytes(128)), 128));
                    }
        for (int x = 0; x < 5; ++x)
            for (int s = s_lo; s < s_hi; ++s)
                for (int pl = 0; pl < 2; ++pl)
                    for (int po = 0; po < 2; ++po) {
                        const int f = x < 3 ? x : x - 3, pi = x >= 3 ? 1 - po : po;
                        const size_t i = idx(f, s, pl, pi);
                        const int cp = (x >= 3 ? 6 : 4) + po;  // ADzP / AzP [po]
                        const int t0 = int(za->gemm.terms.size());
                        za->gemm.terms.push_back({bytes(zap_) + i * kPanel128, bytes(cpan_) + size_t(cp) * kPanel128, zasc_.p + i * 128,
                                                  csc_.p + size_t(cp) * 128, long(oz_slice_bytes(128)), ints(cpe_) + cp});
                        OzItem item{t0, t0 + 1, 0, mh, Np, 0, Y[x] + long(s) * g.slot_stride + long(pl) * mh * 2 * Np + long(po) * Np,
                                    long(2 * Np), 1.0};
                        // ra's B plane in = 2 x + pl, column tile po (no fp64 Y tensor)
                        item.pdst = rpan(s, 2 * x + pl) + size_t(po) * 128 * kOzK;
                        item.pstride = long(oz_slice_bytes(256));
                        item.ppe = ints(rape_) + size_t(s - s_lo) * 20 + (2 * x + pl) * 2 + po;
                        za->gemm.items.push_back(item);
                    }
        za->split.upload();
        za->gemm.tag = "X3";
        za->gemm.upload();
    }
    Stage* ra = stage(key_of("ra_gemm", {Y[0], lam_n, gam_n}), fresh);
    if (!ra) return false;
    if (fresh) {
        for (int s = s_lo; s < s_hi; ++s)
            for (int o = 0; o < 4; ++o)
                for (int nt = 0; nt < 2; ++nt) {
                    const int t0 = int(ra->gemm.terms.size());
                    for (const CompositeTerm& ct : P.anal_.terms[size_t(s)]) {
                        if (ct.out != o) continue;
                        const size_t bi = size_t(ana0_) + size_t(ct.off) / size_t(mh * mh);
                        ra->gemm.terms.push_back({bytes(cpan_) + bi * kPanel128, rpan(s, ct.in), csc_.p + bi * 128,
                                                  nullptr, long(oz_slice_bytes(256)),
                                                  ints(rape_) + size_t(s - s_lo) * 20 + ct.in * 2});
                    }
                    const int t1 = int(ra->gemm.terms.size());
                    ra->gemm.b_mn = true;
                    ra->gemm.items.push_back({t0, t1, nt * 128, M, 128, 0,
                                              (o < 2 ? gam_n : lam_n) + P.eig_off(s, o % 2, 0) + nt * 128, long(2 * Np), 1.0});
                }
        ra->gemm.tag = "C";
        ra->gemm.upload();
    }
    za->split.launch(P.c.stream);
    P.c.mark("X3_av_split");
    za->gemm.launch(P.c.stream);
    P.c.gemm_flops += za->gemm.flops;
    P.c.mark("X3_rz_analysis");
    ra->gemm.launch(P.c.stream);
    P.c.gemm_flops += ra->gemm.flops;
    P.c.launches += 3;
    return true;
}

}  // namespace ccf
