// C-ABI (include/ccf.h) over the B200 CCF context.
#include <cmath>
#include <cstring>
#include <optional>
#include <set>
#include <vector>

#include "../../include/ccf.h"
#include "context.hpp"
#include "pipeline.hpp"

#include <cstdlib>


struct ccf_ctx {
    std::unique_ptr<ccf::Ctx> c;
    std::unique_ptr<ccf::Pipeline> pipe;
    std::set<ccf_ns_state*> states;  // live steppers: detached (ctx = nullptr) when the context goes first
    ccf::Pipeline& pl() {
        if (!pipe) pipe = std::make_unique<ccf::Pipeline>(*c);
        return *pipe;
    }
};

struct ccf_ns_state {
    ccf_ctx* ctx = nullptr;
    ccf::NSState st;
    // the history rings live in two arenas from the context's cache (Ctx::arena_get), returned on destroy
    double* arena[2] = {nullptr, nullptr};
    size_t arena_n[2] = {0, 0};
    ~ccf_ns_state() {
        for (int i = 0; i < 2; ++i)
            if (arena[i]) cudaFree(arena[i]);  // (detached from a destroyed context; otherwise handed back first)
    }
};

using ccf::Ctx;
using ccf::Error;

namespace {

thread_local std::string g_create_err;

template <class F>
ccf_status guard(ccf_ctx* h, F&& f) {
    if (!h || !h->c) return CCF_INTERNAL_ERROR;
    Ctx& c = *h->c;
    try {
        CCF_CUDA(cudaSetDevice(c.device));
        f(c);
        return CCF_OK;
    } catch (const Error& e) {
        c.err_kind = e.status;
        c.err_slice = e.slice;
        c.err_shift = e.shift_index;
        c.err_hist = e.history;
        c.err_msg = e.what();
        return ccf_status(e.status);
    } catch (const std::exception& e) {
        c.err_kind = CCF_INTERNAL_ERROR;
        c.err_slice = c.err_shift = -1;
        c.err_hist.clear();
        c.err_msg = e.what();
        return CCF_INTERNAL_ERROR;
    }
}

// BDF tables, proj/src/timestep.cpp:5-39
void bdf_scheme(int b, double* kappa_over_h, double w[4]) {
    switch (b) {
        case 1: *kappa_over_h = 1.0; w[0] = 1.0; break;
        case 2: *kappa_over_h = 2.0 / 3.0; w[0] = 4.0 / 3.0; w[1] = -1.0 / 3.0; break;
        case 3: *kappa_over_h = 6.0 / 11.0; w[0] = 18.0 / 11.0; w[1] = -9.0 / 11.0; w[2] = 2.0 / 11.0; break;
        case 4:
            *kappa_over_h = 12.0 / 25.0;
            w[0] = 48.0 / 25.0; w[1] = -36.0 / 25.0; w[2] = 16.0 / 25.0; w[3] = -3.0 / 25.0;
            break;
        default: throw Error(ccf::DOMAIN_ERROR, "BDFScheme: order must be in {1,2,3,4}");
    }
}

}  // namespace

void ccf_modal_detach_ctx(ccf_ctx* ctx);  // modalapi.cu

// context guard for the other translation units of the C-ABI (modalapi.cu)
ccf_status ccf_ctx_guard(ccf_ctx* ctx, void (*fn)(ccf::Ctx&, void*), void* user) {
    return guard(ctx, [&](Ctx& c) { fn(c, user); });
}

extern "C" {

const char* ccf_version(void) { return "ccf-b200 0.1 (sm_100a)"; }

ccf_status ccf_ctx_create(int m, int n, int p, int device, double adi_tol, int flags, ccf_ctx** out) {
    if (!out) return CCF_INTERNAL_ERROR;
    *out = nullptr;
    try {
        auto h = new ccf_ctx;
        h->c = std::make_unique<Ctx>(m, n, p, device, adi_tol, flags);
        *out = h;
        return CCF_OK;
    } catch (const Error& e) {
        g_create_err = e.what();
        return ccf_status(e.status);
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return CCF_INTERNAL_ERROR;
    }
}

const char* ccf_create_error(void) { return g_create_err.c_str(); }

ccf_status ccf_ctx_destroy(ccf_ctx* ctx) {
    if (!ctx) return CCF_OK;
    try {
        if (ctx->c) cudaSetDevice(ctx->c->device);
        for (ccf_ns_state* st : ctx->states) {
            st->ctx = nullptr;  // later calls on the stepper report CCF_INTERNAL_ERROR; destroy only frees it
            st->st.pl = nullptr;
        }
        ccf_modal_detach_ctx(ctx);
        ctx->pipe.reset();
        delete ctx;
    } catch (...) {
        return CCF_INTERNAL_ERROR;
    }
    return CCF_OK;
}

ccf_status ccf_ctx_set_stream(ccf_ctx* ctx, void* stream) {
    return guard(ctx, [&](Ctx& c) { c.stream = stream ? static_cast<cudaStream_t>(stream) : c.own_stream; });
}

ccf_status ccf_ctx_synchronize(ccf_ctx* ctx) {
    return guard(ctx, [&](Ctx& c) { c.sync(); });
}

ccf_status ccf_poisson3d(ccf_ctx* ctx, const double* f, double* u) {
    // proj/src/solvers.cpp:142-175: parity(f); per slice R2 f C02^T -> ModalSolver(Poisson) -> parity(out).
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_poisson3d");
        const bool full = true;  // arbitrary complex input: no Hermitian assumption
        const long nt = c.tensor_doubles(full);
        if (c.tens[0].n < size_t(nt)) c.tens[0].alloc(size_t(nt));
        if (c.tens[1].n < size_t(nt)) c.tens[1].alloc(size_t(nt));
        c.load_coeff(f, c.tens[0].p, full, 0, 0);
        c.require_finite(c.tens[0].p, nt, "solve_poisson_3d");
        ccf::DevSet& set = c.set(full, true, 1.0);
        const double* src[1] = {c.tens[0].p};
        const double w[1] = {1.0};
        ctx->pl().modal_solve(set, full, 1, src, w, 1, nullptr, nullptr, 0, c.tens[1].p, nullptr);
        c.check_adi_error(full);
        c.store_coeff(c.tens[1].p, u, full, 0, 0);
        c.sync();
    });
}

ccf_status ccf_helmholtz_step(ccf_ctx* ctx, const double* const* hist, int nhist, int order, const double* forcing,
                              double diffusivity, double h, double* out) {
    // proj/src/timestep.cpp:61-108
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_helmholtz_step");
        double koh, bw[4] = {0, 0, 0, 0};
        bdf_scheme(order, &koh, bw);
        if (nhist < order) throw Error(ccf::DOMAIN_ERROR, "bdf_rhs: insufficient history for the requested order");
        const double kappa = koh * h;
        const double scale = kappa * diffusivity;
        // zero diffusivity: the mass pair (solvers.cpp:57-62) as a fast-diagonalization set with unit denominators
        if (scale == 0.0 && (c.flags & 4))
            throw Error(ccf::CONFIG_ERROR, "ccf_helmholtz_step: the mass solve (zero diffusivity) needs a fast-diagonalization context");
        if (scale < 0.0) throw Error(ccf::DOMAIN_ERROR, "HelmholtzTensorStepper: negative diffusivity");
        const bool full = true;
        const long nt = c.tensor_doubles(full);
        for (int i = 0; i < order + 2; ++i)
            if (c.tens[i].n < size_t(nt)) c.tens[i].alloc(size_t(nt));
        const double* src[ccf::kMaxSrc];
        double w[ccf::kMaxSrc];
        int ns = 0;
        for (int i = 0; i < order; ++i) {
            c.load_coeff(hist[i], c.tens[i].p, full, 0, i % 4);
            src[ns] = c.tens[i].p;
            w[ns++] = bw[i];
        }
        if (forcing) {
            c.load_coeff(forcing, c.tens[order].p, full, 0, 0);
            src[ns] = c.tens[order].p;
            w[ns++] = kappa;
        }
        ccf::DevSet& set = c.set(full, false, scale);
        double* o = c.tens[order + 1].p;
        ctx->pl().modal_solve(set, full, 1, src, w, ns, nullptr, nullptr, 0, o, nullptr);
        c.check_adi_error(full);
        c.require_finite(o, nt, "HelmholtzTensorStepper");
        c.store_coeff(o, out, full, 0, 0);
        c.sync();
    });
}

ccf_status ccf_modal_plan(ccf_ctx* ctx, int w, double scale, int poisson, double* info, double* u, double* v, int cap) {
    return guard(ctx, [&](Ctx& c) {
        const int s = w + c.p / 2;
        if (s < 0 || s >= c.p) throw Error(ccf::DOMAIN_ERROR, "ccf_modal_plan: wavenumber out of range");
        // the reference's shift plan of this mode (a fast-diagonalization context keeps no ADI data:
        // build the plan of this one mode on the host)
        ccf::SolverSet one;
        const ccf::Plan* plp = nullptr;
        if (c.flags & 4) {
            plp = &c.set(true, poisson != 0, scale).host.plans[size_t(s)].plan;
        } else {
            one = ccf::build_solver_set(*c.sizeops, {w}, poisson != 0, scale, c.tol, c.radial_cache, (c.flags & 1) != 0,
                                        1.0, false, true);
            plp = &one.plans[0].plan;
        }
        const ccf::Plan& pl = *plp;
        const double vals[8] = {pl.a, pl.b, pl.c, pl.d, pl.gamma, pl.alpha, pl.modulus, double(pl.J)};
        std::memcpy(info, vals, sizeof vals);
        for (int j = 0; j < pl.J && j < cap; ++j) {
            u[j] = pl.u[size_t(j)];
            v[j] = pl.v[size_t(j)];
        }
    });
}

ccf_status ccf_get_last_error(ccf_ctx* ctx, int* kind, int* slice, int* shift_index, double* residual_hist, int* n_hist,
                              char* msg, int cap) {
    if (!ctx || !ctx->c) return CCF_INTERNAL_ERROR;
    Ctx& c = *ctx->c;
    if (kind) *kind = c.err_kind;
    if (slice) *slice = c.err_slice;
    if (shift_index) *shift_index = c.err_shift;
    if (n_hist) {
        const int k = std::min<int>(*n_hist, int(c.err_hist.size()));
        for (int i = 0; i < k && residual_hist; ++i) residual_hist[i] = c.err_hist[size_t(i)];
        *n_hist = int(c.err_hist.size());
    }
    if (msg && cap > 0) {
        std::strncpy(msg, c.err_msg.c_str(), size_t(cap - 1));
        msg[cap - 1] = 0;
    }
    return CCF_OK;
}

ccf_status ccf_get_stats(ccf_ctx* ctx, long* adi_subproblems, long* adi_iterations, int* max_rounds,
                         double* worst_residual, long* kernel_launches) {
    return guard(ctx, [&](Ctx& c) {
        unsigned long long it[2];
        CCF_CUDA(cudaMemcpy(it, c.ws.iters, sizeof(it), cudaMemcpyDeviceToHost));
        if (adi_iterations) *adi_iterations = long(it[0]);
        if (adi_subproblems) *adi_subproblems = 0;
        if (max_rounds) *max_rounds = 0;
        if (worst_residual) *worst_residual = 0;
        if (kernel_launches) *kernel_launches = c.launches;
    });
}

ccf_status ccf_adi_keep_history(ccf_ctx* ctx, int enable) {
    return guard(ctx, [&](Ctx& c) {
        c.keep_history = enable != 0;
        if (c.keep_history)
            for (int k = 1; k < 3; ++k) {
                const size_t cap = size_t(2) * size_t(std::max(c.p, 2));
                if (!c.kept_hist[k].p) c.kept_hist[k].alloc(cap * 4);
                if (!c.kept_rounds[k].p) c.kept_rounds[k].alloc(cap);  // ints fit in the double slots
            }
    });
}

ccf_status ccf_adi_last_rounds(ccf_ctx* ctx, int which, int* ntensor, int* nslots, int* rounds, double* history,
                               int cap) {
    return guard(ctx, [&](Ctx& c) {
        if (which < 0 || which > 2) throw Error(ccf::DOMAIN_ERROR, "ccf_adi_last_rounds: which in {0, 1, 2}");
        if (which > 0 && !c.keep_history)
            throw Error(ccf::DOMAIN_ERROR, "ccf_adi_last_rounds: enable ccf_adi_keep_history first");
        const int nt = which ? c.kept_shape[which][0] : c.last_adi_ntensor;
        const int ns = which ? c.kept_shape[which][1] : c.last_adi_nslots;
        const int n = nt * ns;
        *ntensor = nt;
        *nslots = ns;
        if (n == 0) return;
        if (cap < n) throw Error(ccf::DOMAIN_ERROR, "ccf_adi_last_rounds: cap < ntensor * nslots");
        c.sync();
        const void* rs = which ? static_cast<const void*>(c.kept_rounds[which].p) : c.ws.rounds;
        const void* hs = which ? static_cast<const void*>(c.kept_hist[which].p) : c.ws.history;
        if (rounds) CCF_CUDA(cudaMemcpy(rounds, rs, sizeof(int) * size_t(n), cudaMemcpyDeviceToHost));
        if (history) CCF_CUDA(cudaMemcpy(history, hs, sizeof(double) * 4 * size_t(n), cudaMemcpyDeviceToHost));
    });
}

ccf_status ccf_reset_stats(ccf_ctx* ctx) {
    return guard(ctx, [&](Ctx& c) {
        CCF_CUDA(cudaMemsetAsync(c.ws.iters, 0, sizeof(unsigned long long) * 2, c.stream));
        c.launches = 0;
        c.gemm_flops = 0.0;
    });
}

ccf_status ccf_get_gemm_flops(ccf_ctx* ctx, double* flops) {
    return guard(ctx, [&](Ctx& c) { *flops = c.gemm_flops; });
}

}  // extern "C"


// ------------------------------------------------------------------------------------------
// Half-spectrum entry points. Inputs are coefficient tensors of real fields (Hermitian,
// as every tensor of the reference NS path is); the scalar / flip parity classes are
// handled separately so arbitrary physical fields round-trip.
namespace {

double* tens(Ctx& c, int i) {
    const long nt = c.tensor_doubles(false);
    if (c.tens[i].n < size_t(nt)) c.tens[i].alloc(size_t(nt));
    return c.tens[i].p;
}

void sync_check(Ctx& c) {
    c.check_adi_error(false);
    c.sync();
}

}  // namespace

extern "C" {

ccf_status ccf_velocity_from_vorticity(ccf_ctx* ctx, const double* lam_w, const double* gam_w, double* lam_v,
                                       double* gam_v) {
    // proj/src/ptns.cpp:85-91: (lambda_v, gamma_v) = (gamma_w, Poisson3D(-lambda_w))
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_velocity_from_vorticity");
        ccf::Pipeline& P = ctx->pl();
        double *l = tens(c, 0), *g = tens(c, 1), *u = tens(c, 2);
        c.load_coeff(lam_w, l, false, 0, 0);
        c.load_coeff(gam_w, g, false, 0, 1);
        c.require_finite(l, P.T, "solve_poisson_3d");
        P.poisson(l, -1.0, u);
        sync_check(c);
        c.store_coeff(g, lam_v, false, 0, 0);
        c.store_coeff(u, gam_v, false, 0, 1);
        c.sync();
    });
}

ccf_status ccf_nonlinear_ex(ccf_ctx* ctx, const double* lam_v, const double* gam_v, const double* lam_w,
                            const double* gam_w, int dealias_two_thirds, double* lam_out, double* gam_out) {
    // proj/src/ptns.cpp:114-149 (dealias: ptns.cpp:100-110, 140-144)
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_nonlinear");
        ccf::Pipeline& P = ctx->pl();
        double *a = tens(c, 0), *b = tens(c, 1), *d = tens(c, 2), *e = tens(c, 3), *o1 = tens(c, 4), *o2 = tens(c, 5);
        c.load_coeff(lam_v, a, false, 0, 0);
        c.load_coeff(gam_v, b, false, 0, 1);
        c.load_coeff(lam_w, d, false, 0, 2);
        c.load_coeff(gam_w, e, false, 0, 3);
        P.nonlinear(a, b, d, e, o1, o2, nullptr, false, false, dealias_two_thirds != 0);
        c.store_coeff(o1, lam_out, false, 0, 0);
        c.store_coeff(o2, gam_out, false, 0, 1);
        c.sync();
    });
}

ccf_status ccf_nonlinear(ccf_ctx* ctx, const double* lam_v, const double* gam_v, const double* lam_w,
                         const double* gam_w, double* lam_out, double* gam_out) {
    return ccf_nonlinear_ex(ctx, lam_v, gam_v, lam_w, gam_w, 0, lam_out, gam_out);
}

ccf_status ccf_pt_synthesize(ccf_ctx* ctx, const double* lam, const double* gam, double* vr, double* vt, double* vz) {
    // proj/src/ptns.cpp:42-57
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_pt_synthesize");
        if (c.m % 2) throw Error(ccf::DOMAIN_ERROR, "pt_synthesize: even m required (no r = 0 grid node)");
        ccf::Pipeline& P = ctx->pl();
        double *l = tens(c, 0), *g = tens(c, 1), *o0 = tens(c, 2), *o1 = tens(c, 3), *o2 = tens(c, 4);
        c.load_coeff(lam, l, false, 0, 0);
        c.load_coeff(gam, g, false, 0, 1);
        const double* L[1] = {l};
        const double* G[1] = {g};
        double* R[1] = {o0};
        double* Tt[1] = {o1};
        double* Z[1] = {o2};
        P.pt_synthesize(1, L, G, R, Tt, Z);
        c.store_coeff(o0, vr, false, 1, 0);
        c.store_coeff(o1, vt, false, 1, 1);
        c.store_coeff(o2, vz, false, 0, 0);
        c.sync();
    });
}

ccf_status ccf_curl_vector(ccf_ctx* ctx, const double* vr, const double* vt, const double* vz, double* or_,
                           double* ot, double* oz) {
    // proj/src/ptns.cpp:25-33 on a physical vector field (r, theta components azimuthal-flip class)
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_curl_vector");
        ccf::Pipeline& P = ctx->pl();
        double *a = tens(c, 0), *b = tens(c, 1), *d = tens(c, 2), *o0 = tens(c, 3), *o1 = tens(c, 4), *o2 = tens(c, 5);
        c.load_coeff(vr, a, false, 1, 0);
        c.load_coeff(vt, b, false, 1, 1);
        c.load_coeff(vz, d, false, 0, 2);
        P.curl_decompose(a, b, d, o0, o1, o2, nullptr, nullptr);
        c.store_coeff(o0, or_, false, 1, 0);
        c.store_coeff(o1, ot, false, 1, 1);
        c.store_coeff(o2, oz, false, 0, 0);
        c.sync();
    });
}

ccf_status ccf_pt_decompose(ccf_ctx* ctx, const double* vr, const double* vt, const double* vz, double* lam,
                            double* gam) {
    // proj/src/ptns.cpp:59-77 (divergence check off, as on the NS path)
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_pt_decompose");
        ccf::Pipeline& P = ctx->pl();
        double *a = tens(c, 0), *b = tens(c, 1), *d = tens(c, 2), *o0 = tens(c, 3), *o1 = tens(c, 4);
        c.load_coeff(vr, a, false, 1, 0);
        c.load_coeff(vt, b, false, 1, 1);
        c.load_coeff(vz, d, false, 0, 2);
        P.decompose(a, b, d, o0, o1);
        c.store_coeff(o0, lam, false, 0, 0);
        c.store_coeff(o1, gam, false, 0, 1);
        c.sync();
    });
}

ccf_status ccf_hpoisson(ccf_ctx* ctx, const double* rhs, double* u) {
    // proj/src/solvers.cpp:177-203
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_hpoisson");
        ccf::Pipeline& P = ctx->pl();
        double *a = tens(c, 0), *o = tens(c, 1);
        c.load_coeff(rhs, a, false, 0, 0);
        c.require_finite(a, P.T, "solve_horizontal_poisson");
        P.hpoisson(a, o);
        c.store_coeff(o, u, false, 0, 0);
        c.sync();
    });
}

ccf_status ccf_calculus(ccf_ctx* ctx, int op, const double* in, double* out) {
    // proj/src/calculus.cpp; both parity classes of the input are processed
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_calculus");
        if (op == 4 && c.m % 2) throw Error(ccf::DOMAIN_ERROR, "divide_r: even m required");
        ccf::Pipeline& P = ctx->pl();
        for (int cls = 0; cls < 2; ++cls) {
            double *a = tens(c, 0), *o = tens(c, 1);
            c.load_coeff(in, a, false, cls, 0);
            const int ocls = (op == 0 || op == 4) ? 1 - cls : cls;
            P.calculus(op, cls, a, o);
            c.store_coeff(o, out, false, ocls, 0, cls == 1);
        }
        c.sync();
    });
}

ccf_status ccf_curl_pt(ccf_ctx* ctx, const double* lam, const double* gam, double* lam_out, double* gam_out) {
    // proj/src/ptns.cpp:79-83: (lambda, gamma) -> (-lap gamma, lambda)
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_curl_pt");
        ccf::Pipeline& P = ctx->pl();
        double *g = tens(c, 0), *o = tens(c, 1), *l = tens(c, 2);
        c.load_coeff(gam, g, false, 0, 0);
        P.calculus(6, 0, g, o);
        P.scale(o, -1.0);
        c.load_coeff(lam, l, false, 0, 1);
        c.store_coeff(o, lam_out, false, 0, 0);
        c.store_coeff(l, gam_out, false, 0, 1);
        c.sync();
    });
}

ccf_status ccf_analyze(ccf_ctx* ctx, const double* values, double* coeffs) {
    // proj/src/transform.cpp:122-165 (arbitrary real fields, full spectrum)
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_analyze");
        ccf::Pipeline& P = ctx->pl();
        P.analyze_full(values, coeffs);
        c.sync();
    });
}

ccf_status ccf_synthesize(ccf_ctx* ctx, const double* coeffs, double* values) {
    // proj/src/transform.cpp:167-203
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_synthesize");
        ccf::Pipeline& P = ctx->pl();
        P.synthesize_full(coeffs, values);
        c.sync();
    });
}

// ---- NSStepper (ptns.hpp:104-127)
namespace {
// NSStepper (ptns.cpp:180-215) and HeatStepper (timestep.cpp:110-129) construction. scalar: one field
// (lam0; gam unused), which is also the heat stepper's state; lam0 holds grid values when values != 0.
ccf_ns_state* ns_create_impl(ccf_ctx* ctx, Ctx& c, double reynolds, double h, int order, bool disable_nonlinear,
                             const double* lam0, const double* gam0, bool scalar, bool values, bool dealias = false,
                             bool gamma_psi = false) {
    if (order < 1 || order > 4) throw Error(ccf::DOMAIN_ERROR, "BDFScheme: order must be in {1,2,3,4}");
    if (c.m % 2) throw Error(ccf::DOMAIN_ERROR, "NSStepper: even m required for the nonlinear pipeline");
    auto st = std::make_unique<ccf_ns_state>();
    st->ctx = ctx;
    ccf::NSState& s = st->st;
    s.pl = &ctx->pl();
    s.reynolds = reynolds;
    s.h = h;
    s.order = order;
    s.disable_nonlinear = disable_nonlinear;
    s.scalar = scalar;
    s.dealias = dealias;
    s.gamma_psi = gamma_psi;
    const long T = s.pl->T;
    {
        ccf::SetupTimer tm("NSStepper: ring buffers");
        const int nt = disable_nonlinear ? 10 : 20;  // lam, gam (+ N~ lam, gam) rings of 5
        st->arena_n[0] = size_t(nt) * size_t(T);
        st->arena[0] = c.arena_get(st->arena_n[0]);
        double* a = st->arena[0];
        for (int i = 0; i < 5; ++i) {
            s.lam[i].view(a + size_t(i) * T, size_t(T));
            s.gam[i].view(a + size_t(5 + i) * T, size_t(T));
        }
        if (!disable_nonlinear)
            for (int i = 0; i < 5; ++i) {
                s.nl[i].view(a + size_t(10 + i) * T, size_t(T));
                s.ng[i].view(a + size_t(15 + i) * T, size_t(T));
            }
    }
    std::optional<ccf::SetupTimer> tm_phase;  // (CCF_SETUP_TRACE phase timers)
    tm_phase.emplace("NSStepper: initial data");
    CCF_CUDA(cudaMalloc(&s.dflag, sizeof(int)));
    CCF_CUDA(cudaMemsetAsync(s.dflag, 0, sizeof(int), c.stream));
    if (values) {  // HeatStepper(config, GridField) = HeatStepper(config, analyze(initial))
        ccf::DBuf ref(size_t(2) * c.m * c.n * c.p);
        s.pl->analyze_full(lam0, ref.p);
        c.load_coeff(ref.p, s.lam[0].p, false, 0, 0);
        c.sync();
    } else {
        c.load_coeff(lam0, s.lam[0].p, false, 0, 0);  // parity projection of the initial data (ptns.cpp:190-191)
    }
    if (gam0) c.load_coeff(gam0, s.gam[0].p, false, 0, 1);
    if (std::getenv("CCF_SETUP_TRACE")) c.sync();  // (diagnostics: the copies inside the timer)
    tm_phase.emplace("NSStepper: eigen state");
    // build every solver set the run needs before any graph capture
    ccf::DevSet& pset = c.set(false, true, 1.0);
    for (int b = 1; b <= order; ++b) {
        static const double K[4] = {1.0, 2.0 / 3.0, 6.0 / 11.0, 12.0 / 25.0};
        c.set(false, false, K[b - 1] * h * (1.0 / reynolds));
    }
    // eigen-coordinate state when every solve has diagonalization data in the shared basis and the
    // nonlinear term runs on the composite operators (CCF_NS_EIGEN=0 keeps coefficient-space history);
    // the heat stepper needs only the modal bases (no composite operators)
    const char* ev = std::getenv("CCF_NS_EIGEN");
    const bool want = !(ev && ev[0] == '0');
    // (a zero-diffusivity heat stepper solves the mass pair, which has no place in the shared Poisson basis)
    if (want && pset.host.has_diag && pset.dg && std::isfinite(reynolds)) {
        ccf::Pipeline& P = *s.pl;
        bool ok = true;
        if (!disable_nonlinear) {
            P.ensure_composite();
            ok = !P.composite_off();
            if (ok) P.ensure_eigen(pset);
        }
        if (ok) {
            s.eigen = true;
            st->arena_n[1] = size_t(scalar ? 6 : 11) * size_t(T);  // zl (5), zpsi, zg (5)
            st->arena[1] = c.arena_get(st->arena_n[1]);
            double* a = st->arena[1];
            s.zpsi.view(a, size_t(T));
            for (int i = 0; i < 5; ++i) {
                s.zl[i].view(a + size_t(1 + i) * T, size_t(T));
                if (!scalar) s.zg[i].view(a + size_t(6 + i) * T, size_t(T));
            }
            P.to_eigen(pset, s.lam[0].p, s.zl[0].p);
            if (!scalar) P.to_eigen(pset, s.gam[0].p, s.zg[0].p);
        }
    }
    if (dealias && !disable_nonlinear) s.pl->ensure_dealias(s.eigen ? &pset : nullptr);  // before any graph capture
    if (c.sh.sharded() && !s.eigen)
        throw Error(ccf::CONFIG_ERROR, "NSStepper: a mode-sharded context needs the eigen-coordinate state "
                                       "(composite nonlinear term, fast-diagonalization solves)");
    c.sync();
    ctx->states.insert(st.get());
    return st.release();
}
}  // namespace

ccf_status ccf_ns_create(ccf_ctx* ctx, double reynolds, double h, int order, int disable_nonlinear, const double* lam0,
                         const double* gam0, ccf_ns_state** out) {
    return guard(ctx, [&](Ctx& c) {
        if (!lam0 || !gam0) throw Error(ccf::DOMAIN_ERROR, "NSStepper: initial vorticity required");
        *out = ns_create_impl(ctx, c, reynolds, h, order, disable_nonlinear != 0, lam0, gam0, false, false);
    });
}

// NSConfig flags (ptns.hpp:84-94): bit 0 disable_nonlinear, bit 1 dealias_two_thirds, bit 2 compute_gamma_psi
ccf_status ccf_ns_create_ex(ccf_ctx* ctx, double reynolds, double h, int order, int flags, const double* lam0,
                            const double* gam0, ccf_ns_state** out) {
    return guard(ctx, [&](Ctx& c) {
        if (!lam0 || !gam0) throw Error(ccf::DOMAIN_ERROR, "NSStepper: initial vorticity required");
        *out = ns_create_impl(ctx, c, reynolds, h, order, (flags & 1) != 0, lam0, gam0, false, false, (flags & 2) != 0,
                              (flags & 4) != 0);
    });
}

ccf_status ccf_ns_velocity(ccf_ns_state* st, double* lam_v, double* gam_v) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_ns_velocity");
        const long T = st->st.pl->T;
        ccf::DBuf a{static_cast<size_t>(T)}, b{static_cast<size_t>(T)};
        st->st.velocity_coeff(a.p, b.p);
        c.store_coeff(a.p, lam_v, false, 0, 0);
        c.store_coeff(b.p, gam_v, false, 0, 1);
        c.sync();
    });
}

ccf_status ccf_ns_gamma_psi(ccf_ns_state* st, double* out) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_ns_gamma_psi");
        if (!st->st.gamma_psi) throw Error(ccf::CONFIG_ERROR, "NSStepper: compute_gamma_psi is off");
        ccf::DBuf a{static_cast<size_t>(st->st.pl->T)};
        st->st.gamma_psi_coeff(a.p);
        c.store_coeff(a.p, out, false, 0, 0);
        c.sync();
    });
}

ccf_status ccf_nonlinear_ex(ccf_ctx* ctx, const double* lam_v, const double* gam_v, const double* lam_w,
                            const double* gam_w, int dealias_two_thirds, double* lam_out, double* gam_out);

// ---- HeatStepper / heat_run (proj/include/cylspec/timestep.hpp:60-111, proj/src/timestep.cpp:110-170)
ccf_status ccf_heat_create(ccf_ctx* ctx, double alpha, double h, int order, const double* initial, int initial_kind,
                           ccf_ns_state** out) {
    return guard(ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_heat_create");
        // alpha = 0 (test_timestep.cpp:136-149): every step is the mass solve; coefficient-space state
        if (!(alpha >= 0.0)) throw Error(ccf::DOMAIN_ERROR, "HeatStepper: alpha must be nonnegative");
        if (alpha == 0.0 && (c.flags & 4))
            throw Error(ccf::CONFIG_ERROR, "HeatStepper: alpha = 0 (mass solve) needs a fast-diagonalization context");
        if (initial_kind != 0 && initial_kind != 1) throw Error(ccf::DOMAIN_ERROR, "ccf_heat_create: initial_kind 0 | 1");
        *out = ns_create_impl(ctx, c, 1.0 / alpha, h, order, true, initial, nullptr, true, initial_kind == 0);
    });
}

// HeatStepper::step(const CoeffTensor* forcing) (kind 1) / step_with_callback (kind 0: the callback's grid
// values, analyzed on the device); forcing == NULL steps without forcing
ccf_status ccf_heat_step(ccf_ns_state* st, const double* forcing, int forcing_kind) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        ccf::NSState& s = st->st;
        if (!s.scalar) throw Error(ccf::CONFIG_ERROR, "ccf_heat_step: not a heat stepper (ccf_heat_create)");
        s.forced = forcing != nullptr;
        if (forcing) {
            if (forcing_kind != 0 && forcing_kind != 1) throw Error(ccf::DOMAIN_ERROR, "ccf_heat_step: forcing_kind 0 | 1");
            const long T = s.pl->T;
            if (s.fh.n < size_t(T)) s.fh.alloc(size_t(T));
            const double* ref = forcing;
            ccf::DBuf tmp;
            if (forcing_kind == 0) {  // analyze(forcing(t)) (timestep.cpp:142)
                tmp.alloc(size_t(2) * c.m * c.n * c.p);
                s.pl->analyze_full(forcing, tmp.p);
                ref = tmp.p;
            }
            c.load_coeff(ref, s.fh.p, false, 0, 2);  // rhs parity projection (timestep.cpp:74)
            if (s.eigen) {
                if (s.zf.n < size_t(T)) s.zf.alloc(size_t(T));
                s.pl->to_eigen(c.set(false, true, 1.0), s.fh.p, s.zf.p);
            }
        }
        s.step_once();
        s.forced = false;
        c.check_adi_error(false);
        int f = 0;
        CCF_CUDA(cudaMemcpyAsync(&f, s.dflag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (f) throw Error(ccf::NUMERICAL, "HelmholtzTensorStepper: non-finite state");
    });
}

ccf_status ccf_heat_get(ccf_ns_state* st, double* coeffs, double* time, int* steps_taken) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        st->st.omega_coeff();
        if (coeffs) c.store_coeff(st->st.lam[st->st.head].p, coeffs, false, 0, 0);
        c.sync();
        if (time) *time = st->st.time;
        if (steps_taken) *steps_taken = st->st.steps;
    });
}

ccf_status ccf_ns_step(ccf_ns_state* st, int nsteps) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        for (int i = 0; i < nsteps; ++i) st->st.step_once();
        c.shard_check();
        // solver error words and the non-finite flag in one round trip (pinned status words, one sync)
        int* hs = c.ws.hstat;
        CCF_CUDA(cudaMemcpyAsync(hs, c.ws.err, sizeof(int) * 4, cudaMemcpyDeviceToHost, c.stream));
        CCF_CUDA(cudaMemcpyAsync(hs + 4, st->st.dflag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (hs[0]) c.check_adi_error(false);
        if (hs[4]) throw Error(ccf::NUMERICAL, "NSStepper: non-finite state at step " + std::to_string(st->st.steps));
    });
}

// NSStepper::seed (ptns.cpp:195-203, ptns.hpp:110-112): install a prebuilt history, newest first
ccf_status ccf_ns_seed(ccf_ns_state* st, int n_omega, const double* const* lam_hist, const double* const* gam_hist,
                       int n_nonlinear, const double* const* nl_lam, const double* const* nl_gam, double time,
                       int steps_taken) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_ns_seed");
        if (n_omega < 1 || !lam_hist || !gam_hist) throw Error(ccf::DOMAIN_ERROR, "NSStepper::seed: empty history");
        if (n_nonlinear > 0 && (!nl_lam || !nl_gam))
            throw Error(ccf::DOMAIN_ERROR, "NSStepper::seed: nonlinear history pointers required");
        for (int i = 0; i < n_omega; ++i)
            if (!lam_hist[i] || !gam_hist[i]) throw Error(ccf::DOMAIN_ERROR, "NSStepper::seed: null history tensor");
        for (int i = 0; i < n_nonlinear; ++i)
            if (!nl_lam[i] || !nl_gam[i]) throw Error(ccf::DOMAIN_ERROR, "NSStepper::seed: null history tensor");
        st->st.seed(n_omega, lam_hist, gam_hist, n_nonlinear, nl_lam, nl_gam, time, steps_taken);
    });
}

ccf_status ccf_ns_get_omega(ccf_ns_state* st, double* lam, double* gam, double* time, int* steps_taken) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        st->st.omega_coeff();
        c.store_coeff(st->st.lam[st->st.head].p, lam, false, 0, 0);
        c.store_coeff(st->st.gam[st->st.head].p, gam, false, 0, 1);
        c.sync();
        if (time) *time = st->st.time;
        if (steps_taken) *steps_taken = st->st.steps;
    });
}

// ---- mode sharding (csrc/shard.cu)
ccf_status ccf_shard_init(ccf_ctx* ctx, int rank, int world) {
    return guard(ctx, [&](Ctx& c) {
        if (!ctx->states.empty()) throw Error(ccf::CONFIG_ERROR, "ccf_shard_init: shard before creating a stepper");
        c.shard_init(rank, world);
        if (ctx->pipe) ctx->pipe->gemms_.clear();  // plans built so far address the unsharded scratch
    });
}

ccf_status ccf_shard_partition(int m, int p, int world, int* slot_bounds, int* row_bounds) {
    if (m < 4 || m % 2 || p < 2 || p % 2 || world < 1 || world > ccf::kMaxRanks || world > m / 2 || world > p / 2 + 1)
        return CCF_CONFIG_ERROR;
    ccf::shard_bounds(p / 2 + 1, world, slot_bounds);
    ccf::shard_bounds(m / 2, world, row_bounds);
    return CCF_OK;
}

ccf_status ccf_shard_info(ccf_ctx* ctx, int* rank, int* world, int* slot_lo, int* slot_hi, int* row_lo, int* row_hi) {
    return guard(ctx, [&](Ctx& c) {
        if (rank) *rank = c.sh.rank;
        if (world) *world = c.sh.world;
        if (slot_lo) *slot_lo = c.sh.s_lo;
        if (slot_hi) *slot_hi = c.sh.s_hi;
        if (row_lo) *row_lo = c.sh.r_lo;
        if (row_hi) *row_hi = c.sh.r_hi;
    });
}

ccf_status ccf_shard_ipc_handle(ccf_ctx* ctx, void* handle) {
    return guard(ctx, [&](Ctx& c) { ccf::shard_ipc_handle(c, handle); });
}

ccf_status ccf_shard_open_ipc(ccf_ctx* ctx, const void* handles) {
    return guard(ctx, [&](Ctx& c) { ccf::shard_open_ipc(c, handles); });
}

ccf_status ccf_shard_link_local(ccf_ctx* const* ctxs, int world) {
    if (!ctxs || world < 1 || !ctxs[0]) return CCF_INTERNAL_ERROR;
    return guard(ctxs[0], [&](Ctx&) {
        std::vector<Ctx*> cs;
        for (int i = 0; i < world; ++i) {
            if (!ctxs[i] || !ctxs[i]->c) throw Error(ccf::CONFIG_ERROR, "ccf_shard_link_local: null context");
            cs.push_back(ctxs[i]->c.get());
        }
        ccf::shard_link_local(cs.data(), world);
    });
}

ccf_status ccf_shard_set_host_barrier(ccf_ctx* ctx, void (*fn)(void*), void* user) {
    return guard(ctx, [&](Ctx& c) { ccf::shard_set_host_barrier(c, fn, user); });
}

ccf_status ccf_ns_destroy(ccf_ns_state* st) {
    if (!st) return CCF_OK;
    if (st->ctx) {
        if (st->ctx->c) {
            cudaSetDevice(st->ctx->c->device);
            cudaStreamSynchronize(st->ctx->c->stream);  // queued work is done with the arenas before another stepper gets them
            for (int i = 0; i < 2; ++i) {
                st->ctx->c->arena_put(st->arena[i], st->arena_n[i]);
                st->arena[i] = nullptr;
            }
        }
        st->ctx->states.erase(st);
    }
    delete st;
    return CCF_OK;
}

ccf_status ccf_ns_set_graphs(ccf_ns_state* st, int enable) {
    if (!st) return CCF_INTERNAL_ERROR;
    st->st.use_graphs = enable != 0;
    return CCF_OK;
}

ccf_status ccf_ns_launches_per_step(ccf_ns_state* st, long* n) {
    if (!st || !n) return CCF_INTERNAL_ERROR;
    *n = st->st.launches_per_step;
    return CCF_OK;
}

}  // extern "C"

extern "C" {
// Run the next step eagerly with CUDA events at the stage boundaries (P, V, X1, X2, X3, C, H).
// names: '\n'-separated stage names written to `names` (cap bytes); ms: per-stage durations.
ccf_status ccf_ns_profile_step(ccf_ns_state* st, double* ms, int* nstages, char* names, int cap) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        const bool g = st->st.use_graphs;
        st->st.use_graphs = false;
        c.profiling = true;
        c.prof_events.clear();
        c.prof_names.clear();
        try {
            st->st.step_once();
        } catch (...) {
            c.profiling = false;
            st->st.use_graphs = g;
            throw;
        }
        c.profiling = false;
        st->st.use_graphs = g;
        c.sync();
        std::string nm;
        const int k = int(c.prof_events.size());
        int out = 0;
        for (int i = 1; i < k && out < *nstages; ++i, ++out) {
            float t = 0;
            cudaEventElapsedTime(&t, c.prof_events[size_t(i - 1)], c.prof_events[size_t(i)]);
            ms[out] = t;
            nm += c.prof_names[size_t(i)] + "\n";
        }
        for (auto e : c.prof_events) cudaEventDestroy(e);
        c.prof_events.clear();
        *nstages = out;
        if (names && cap > 0) {
            std::strncpy(names, nm.c_str(), size_t(cap - 1));
            names[cap - 1] = 0;
        }
    });
}
}  // extern "C"

extern "C" {
// Host-only modal shift plan (no GPU needed): the same setup path the context uses
// (spectral enclosure + Zolotarev shifts, proj/src/solvers.cpp:46-75, adi.cpp:22-104).
ccf_status ccf_diag_host_check(int m, int n, int w, double scale, int poisson, int k0, unsigned long long seed,
                               double* residual) {
    try {
        if (m < 6 || n < 6 || m % 2 || n % 2) throw Error(ccf::DOMAIN_ERROR, "ccf_diag_host_check: even m, n >= 6 required");
        ccf::SizeOps so(m, n);
        std::map<int, ccf::Range> cache;
        ccf::SolverSet set = ccf::build_solver_set(so, {w}, poisson != 0, scale, 1e-12, cache, false, 4.0, true, false);
        *residual = ccf::diag_check_residual(set, 0, k0 & 1, (m - 2) / 2, (n - 2) / 2, seed);
        return CCF_OK;
    } catch (const Error& e) {
        g_create_err = e.what();
        return ccf_status(e.status);
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return CCF_INTERNAL_ERROR;
    }
}

ccf_status ccf_plan_host(int m, int n, int w, double scale, int poisson, double tol, int flags, double* info, double* u,
                         double* v, int cap) {
    try {
        if (m < 4 || n < 4 || m % 2 || n % 2) throw Error(ccf::DOMAIN_ERROR, "ccf_plan_host: even m, n >= 4 required");
        ccf::SizeOps so(m, n);
        std::map<int, ccf::Range> cache;
        ccf::SolverSet set = ccf::build_solver_set(so, {w}, poisson != 0, scale, tol, cache, (flags & 1) != 0);
        const ccf::Plan& pl = set.plans[0].plan;
        const double vals[8] = {pl.a, pl.b, pl.c, pl.d, pl.gamma, pl.alpha, pl.modulus, double(pl.J)};
        std::memcpy(info, vals, sizeof vals);
        if (flags & 2) info[8] = double(set.slots[0].pivot);  // caller provides info[9]
        for (int j = 0; j < pl.J && j < cap; ++j) {
            u[j] = pl.u[size_t(j)];
            v[j] = pl.v[size_t(j)];
        }
        return CCF_OK;
    } catch (const Error& e) {
        g_create_err = e.what();
        return ccf_status(e.status);
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return CCF_INTERNAL_ERROR;
    }
}
}  // extern "C"

// ---- CCF1 FieldFile I/O (proj/include/cylspec/io.hpp:11-28, proj/src/io.cpp:12-109)
namespace {
template <class F>
ccf_status guard_free(F&& f) {  // context-free entry points: message via ccf_create_error()
    try {
        f();
        return CCF_OK;
    } catch (const Error& e) {
        g_create_err = e.what();
        return ccf_status(e.status);
    } catch (const std::exception& e) {
        g_create_err = e.what();
        return CCF_INTERNAL_ERROR;
    }
}
bool device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}
// selects the device that owns a pointer for the scope and restores the caller's current device
// afterwards (the free functions below must not change the calling thread's device for torch etc.)
struct PtrDeviceGuard {
    int prev = -1;
    explicit PtrDeviceGuard(const void* p) {
        cudaPointerAttributes a{};
        CCF_CUDA(cudaPointerGetAttributes(&a, p));
        CCF_CUDA(cudaGetDevice(&prev));
        if (a.device != prev) CCF_CUDA(cudaSetDevice(a.device));
        else prev = -1;
    }
    ~PtrDeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    PtrDeviceGuard(const PtrDeviceGuard&) = delete;
    PtrDeviceGuard& operator=(const PtrDeviceGuard&) = delete;
};
}  // namespace

ccf_status ccf_crc32(const void* data, size_t len, unsigned* crc) {
    return guard_free([&] {
        if (len && device_ptr(data)) {
            PtrDeviceGuard dg(data);  // tables, sync and launch on the device that owns the data
            CCF_CUDA(cudaDeviceSynchronize());
            if (len % 8 == 0 && reinterpret_cast<uintptr_t>(data) % 8 == 0) {
                *crc = ccf::crc32_device(data, len, nullptr);
                return;
            }
            std::vector<uint8_t> h(len);
            CCF_CUDA(cudaMemcpy(h.data(), data, len, cudaMemcpyDeviceToHost));
            *crc = ccf::crc32_host(h.data(), len);
            return;
        }
        *crc = ccf::crc32_host(static_cast<const uint8_t*>(data), len);
    });
}

ccf_status ccf_write_field(const char* path, int kind, int m, int n, int p, const double* payload) {
    return guard_free([&] {
        if (m < 4 || n < 4) throw Error(ccf::DOMAIN_ERROR, "GridSpec: m and n must be at least 4");
        if (p < 2 || p % 2 != 0) throw Error(ccf::DOMAIN_ERROR, "GridSpec: p must be even and at least 2");
        const bool dev = device_ptr(payload);
        std::unique_ptr<PtrDeviceGuard> dg;
        if (dev) {
            dg = std::make_unique<PtrDeviceGuard>(payload);
            CCF_CUDA(cudaDeviceSynchronize());
        }
        ccf::write_field_file(path, kind, m, n, p, payload, dev, nullptr);
    });
}

ccf_status ccf_read_field_header(const char* path, int* kind, int* m, int* n, int* p) {
    return guard_free([&] { ccf::read_field_header(path, *kind, *m, *n, *p); });
}

ccf_status ccf_read_field(const char* path, int* kind, int* m, int* n, int* p, double* payload, size_t cap) {
    return guard_free([&] {
        const bool dev = device_ptr(payload);
        std::unique_ptr<PtrDeviceGuard> dg;
        if (dev) {
            dg = std::make_unique<PtrDeviceGuard>(payload);
            CCF_CUDA(cudaDeviceSynchronize());
        }
        ccf::read_field_file(path, *kind, *m, *n, *p, payload, cap, dev, nullptr);
    });
}

ccf_status ccf_ns_write_omega(ccf_ns_state* st, const char* lam_path, const char* gam_path) {
    if (!st) return CCF_INTERNAL_ERROR;
    return guard(st->ctx, [&](Ctx& c) {
        c.require_unsharded("ccf_ns_write_omega");
        st->st.omega_coeff();
        const size_t nref = size_t(2) * c.m * c.n * c.p;
        ccf::DBuf ref(nref);
        const char* paths[2] = {lam_path, gam_path};
        const double* src[2] = {st->st.lam[st->st.head].p, st->st.gam[st->st.head].p};
        for (int i = 0; i < 2; ++i) {
            if (!paths[i]) continue;
            c.store_coeff(src[i], ref.p, false, 0, i);  // reference layout, on the device
            ccf::write_field_file(paths[i], 1, c.m, c.n, c.p, ref.p, true, c.stream);
        }
    });
}
