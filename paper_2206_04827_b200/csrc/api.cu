// C-ABI (include/ccf.h) over the B200 CCF context.
#include <cstring>
#include <vector>

#include "../../include/ccf.h"
#include "context.hpp"


struct ccf_ctx {
    std::unique_ptr<ccf::Ctx> c;
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
        const bool full = true;  // arbitrary complex input: no Hermitian assumption
        const long nt = c.tensor_doubles(full);
        if (c.tens[0].n < size_t(nt)) c.tens[0].alloc(size_t(nt));
        if (c.tens[1].n < size_t(nt)) c.tens[1].alloc(size_t(nt));
        c.load_coeff(f, c.tens[0].p, full, 0, 0);
        c.require_finite(c.tens[0].p, nt, "solve_poisson_3d");
        ccf::DevSet& set = c.set(full, true, 1.0);
        const double* src[1] = {c.tens[0].p};
        const double w[1] = {1.0};
        c.run_adi(set, full, 1, src, w, 1, nullptr, nullptr, 0, c.tens[1].p, nullptr);
        c.check_adi_error(full);
        c.store_coeff(c.tens[1].p, u, full, 0, 0);
        c.sync();
    });
}

ccf_status ccf_helmholtz_step(ccf_ctx* ctx, const double* const* hist, int nhist, int order, const double* forcing,
                              double diffusivity, double h, double* out) {
    // proj/src/timestep.cpp:61-108
    return guard(ctx, [&](Ctx& c) {
        double koh, bw[4] = {0, 0, 0, 0};
        bdf_scheme(order, &koh, bw);
        if (nhist < order) throw Error(ccf::DOMAIN_ERROR, "bdf_rhs: insufficient history for the requested order");
        const double kappa = koh * h;
        const double scale = kappa * diffusivity;
        if (scale == 0.0) throw Error(ccf::DOMAIN_ERROR, "ccf_helmholtz_step: zero diffusivity (mass solve) is not supported on the B200 path");
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
        c.run_adi(set, full, 1, src, w, ns, nullptr, nullptr, 0, o, nullptr);
        c.check_adi_error(full);
        c.require_finite(o, nt, "HelmholtzTensorStepper");
        c.store_coeff(o, out, full, 0, 0);
        c.sync();
    });
}

ccf_status ccf_modal_plan(ccf_ctx* ctx, int w, double scale, int poisson, double* info, double* u, double* v, int cap) {
    return guard(ctx, [&](Ctx& c) {
        ccf::DevSet& set = c.set(true, poisson != 0, scale);
        const int s = w + c.p / 2;
        if (s < 0 || s >= c.p) throw Error(ccf::DOMAIN_ERROR, "ccf_modal_plan: wavenumber out of range");
        const ccf::Plan& pl = set.host.plans[size_t(s)].plan;
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

ccf_status ccf_reset_stats(ccf_ctx* ctx) {
    return guard(ctx, [&](Ctx& c) {
        CCF_CUDA(cudaMemset(c.ws.iters, 0, sizeof(unsigned long long) * 2));
        c.launches = 0;
    });
}

}  // extern "C"

// ---- entry points not yet wired (return an explicit error instead of a CPU fallback)
#define CCF_TODO(sig)                                                                            \
    ccf_status sig {                                                                             \
        return guard(ctx, [&](Ctx&) { throw Error(ccf::INTERNAL, "ccf: entry point not implemented yet"); }); \
    }
extern "C" {
CCF_TODO(ccf_analyze(ccf_ctx* ctx, const double*, double*))
CCF_TODO(ccf_synthesize(ccf_ctx* ctx, const double*, double*))
CCF_TODO(ccf_calculus(ccf_ctx* ctx, int, const double*, double*))
CCF_TODO(ccf_hpoisson(ccf_ctx* ctx, const double*, double*))
CCF_TODO(ccf_pt_synthesize(ccf_ctx* ctx, const double*, const double*, double*, double*, double*))
CCF_TODO(ccf_pt_decompose(ccf_ctx* ctx, const double*, const double*, const double*, double*, double*))
CCF_TODO(ccf_curl_vector(ccf_ctx* ctx, const double*, const double*, const double*, double*, double*, double*))
CCF_TODO(ccf_curl_pt(ccf_ctx* ctx, const double*, const double*, double*, double*))
CCF_TODO(ccf_velocity_from_vorticity(ccf_ctx* ctx, const double*, const double*, double*, double*))
CCF_TODO(ccf_nonlinear(ccf_ctx* ctx, const double*, const double*, const double*, const double*, double*, double*))
CCF_TODO(ccf_ns_create(ccf_ctx* ctx, double, double, int, int, const double*, const double*, ccf_ns_state**))
ccf_status ccf_ns_step(ccf_ns_state*, int) { return CCF_INTERNAL_ERROR; }
ccf_status ccf_ns_get_omega(ccf_ns_state*, double*, double*, double*, int*) { return CCF_INTERNAL_ERROR; }
ccf_status ccf_ns_destroy(ccf_ns_state*) { return CCF_OK; }
}
