// Host-side context implementation: device memory, solver-set cache
// (ModalSolverCache, proj/src/solvers.cpp:100-109), ADI round driver.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <cstdio>
#include <cstring>

#include "context.hpp"

namespace ccf {

void DBuf::alloc(size_t count) {
    if (p && own) cudaFree(p);
    own = true;
    p = nullptr;
    n = count;
    if (count) {
        CCF_CUDA(cudaMalloc(&p, count * sizeof(double)));
        // zero-filled: pad columns of every tensor are defined (the TMA GEMM reads them at K edges).
        // cudaMemset runs on the legacy default stream, which the library's non-blocking streams do
        // not wait for: complete it here, or a kernel writing the fresh buffer could be overtaken
        CCF_CUDA(cudaMemset(p, 0, count * sizeof(double)));
        CCF_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
}
void DBuf::view(double* ptr, size_t count) {
    if (p && own) cudaFree(p);
    p = ptr;
    n = count;
    own = false;
}
DBuf::~DBuf() {
    if (p && own) cudaFree(p);
}
DBuf& DBuf::operator=(DBuf&& o) noexcept {
    if (this != &o) {
        if (p && own) cudaFree(p);
        p = o.p;
        n = o.n;
        own = o.own;
        o.p = nullptr;
        o.n = 0;
        o.own = true;
    }
    return *this;
}

DevSet::~DevSet() {
    if (coef) cudaFree(coef);
    if (slots) cudaFree(slots);
    if (J) cudaFree(J);
    if (dg) cudaFree(dg);
    for (auto* t : tasks)
        if (t) cudaFree(t);
}

static Geo make_geo(int m, int n, int p, int nslots) {
    Geo g{};
    g.m = m;
    g.n = n;
    g.p = p;
    g.mh = m / 2;
    g.nh = n / 2;
    g.nslots = nslots;
    g.M = (m - 2) / 2;
    g.N = (n - 2) / 2;
    g.plane_stride = long(n) * (m / 2);
    g.slot_stride = 2 * g.plane_stride;
    return g;
}

Ctx::Ctx(int m_, int n_, int p_, int device_, double tol_, int flags_)
    : m(m_), n(n_), p(p_), device(device_), flags(flags_), tol(tol_) {
    if (m < 4 || n < 4) throw Error(DOMAIN_ERROR, "GridSpec: m and n must be at least 4");
    if (p < 2 || p % 2 != 0) throw Error(DOMAIN_ERROR, "GridSpec: p must be even and at least 2");
    if (m % 2 || n % 2) throw Error(DOMAIN_ERROR, "ccf: the B200 path requires even m and n (parity-compressed layout)");
    const bool adi = (flags & 4) != 0;  // the ADI kernel (single-CTA tile) is the modal solver
    if (adi && (m > 320 || n > 320)) throw Error(DOMAIN_ERROR, "ccf: m, n <= 320 with the ADI solver (single-CTA tile)");
    if (m > 2050 || n > 2050) throw Error(DOMAIN_ERROR, "ccf: m, n <= 2050");
    if (!(tol > 0.0) || tol >= 1.0) throw Error(DOMAIN_ERROR, "compute_shifts: tol must be in (0,1)");
    CCF_CUDA(cudaSetDevice(device));
    CCF_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
    stream = own_stream;
    gh = make_geo(m, n, p, p / 2 + 1);
    gf = make_geo(m, n, p, p);
    sh.s_hi = gh.nslots;
    sh.r_hi = gh.mh;
    M = (m - 2) / 2;
    N = (n - 2) / 2;
    Mpad = ((M + 7) / 8) * 8;
    Npad = ((N + 7) / 8) * 8;
    pitch = (Npad + 4) | 1;
    estride = ((long(Mpad) * N + 1) / 2) * 2;
    if (adi && std::max(M, N) > 256) throw Error(DOMAIN_ERROR, "ccf: (m-2)/2, (n-2)/2 <= 256 with the ADI solver");
    sizeops = std::make_unique<SizeOps>(m, n);
    // workspace
    const int cap = p;  // max slots (full mode)
    ws.cap_slots = cap;
    CCF_CUDA(cudaMalloc(&ws.res2, sizeof(double) * 2 * cap));
    CCF_CUDA(cudaMalloc(&ws.e2, sizeof(double) * 2 * cap));
    CCF_CUDA(cudaMalloc(&ws.history, sizeof(double) * 2 * cap * 4));
    CCF_CUDA(cudaMalloc(&ws.active, sizeof(int) * 2 * cap));
    CCF_CUDA(cudaMalloc(&ws.rounds, sizeof(int) * 2 * cap));
    CCF_CUDA(cudaMalloc(&ws.err, sizeof(int) * 4));
    CCF_CUDA(cudaMalloc(&ws.flag, sizeof(int) * 4));
    CCF_CUDA(cudaMalloc(&ws.iters, sizeof(unsigned long long) * 2));
    CCF_CUDA(cudaHostAlloc(&ws.hstat, sizeof(int) * 8, cudaHostAllocDefault));
    CCF_CUDA(cudaMemset(ws.err, 0, sizeof(int) * 4));
    CCF_CUDA(cudaMemset(ws.iters, 0, sizeof(unsigned long long) * 2));
    CCF_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    if (adi) {  // ADI round scratch and the single-CTA tile's shared memory
        ws.eprime.alloc(size_t(2) * cap * 4 * size_t(estride));
        ws.escr.alloc(size_t(2) * cap * 4 * size_t(estride));
        ws.xscr.alloc(size_t(2) * cap * 4 * size_t(estride));
        int optin = 0;
        CCF_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        const size_t stat = adi_static_smem();
        const size_t need = adi_smem_bytes();
        if (need + stat > size_t(optin))
            throw Error(DOMAIN_ERROR, "ccf: ADI tile exceeds shared memory (m, n too large for the single-CTA kernel)");
        CCF_CUDA(adi_set_smem(int(optin - stat)));
    }
}

double* Ctx::arena_get(size_t count) {
    double* p = nullptr;
    for (size_t i = 0; i < arena_cache.size(); ++i)
        if (arena_cache[i].first == count) {
            p = arena_cache[i].second;
            arena_cache.erase(arena_cache.begin() + long(i));
            break;
        }
    if (!p) CCF_CUDA(cudaMalloc(&p, count * sizeof(double)));
    CCF_CUDA(cudaMemsetAsync(p, 0, count * sizeof(double), stream));
    return p;
}

void Ctx::arena_put(double* p, size_t count) {
    if (p) arena_cache.push_back({count, p});
}

Ctx::~Ctx() {
    for (auto& a : arena_cache) cudaFree(a.second);
    arena_cache.clear();
    shard_close();
    sets.clear();
    cudaFree(ws.res2);
    cudaFree(ws.e2);
    cudaFree(ws.history);
    cudaFree(ws.active);
    cudaFree(ws.rounds);
    cudaFree(ws.err);
    cudaFree(ws.flag);
    cudaFree(ws.iters);
    if (ws.hstat) cudaFreeHost(ws.hstat);
    if (own_stream) cudaStreamDestroy(own_stream);
}

int Ctx::adi_lanes() const { return ((std::max(M, N) + 31) / 32) * 32; }

bool Ctx::adi_split() const {
    const int hc = spike_split(Mpad), hr = spike_split(Npad);
    return hc > 0 && hr > 0 && hc < M && hr < N && 2 * adi_lanes() <= 512;
}

size_t Ctx::adi_smem_bytes() const {
    const long rows = Mpad + 6;
    const long ysize = ((rows * pitch + 1) / 2) * 2;
    const long rings = adi_split() ? 6 : 3;
    const long total = ysize + long(Mpad + 2) * kLeftW + long(Npad + 2) * kRightW + rings * 8 * N + 4L * adi_lanes();
    return size_t(total) * sizeof(double);
}

void Ctx::sync() { CCF_CUDA(cudaStreamSynchronize(stream)); }

bool Ctx::is_device_ptr(const void* ptr) const {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

DevSet& Ctx::set(bool full, bool poisson, double scale) {
    auto key = std::make_tuple(int(full), int(poisson), poisson ? 1.0 : scale);
    auto it = sets.find(key);
    if (it != sets.end()) return *it->second;
    const Geo& g = geo(full);
    std::vector<int> slot_w(size_t(g.nslots));
    for (int s = 0; s < g.nslots; ++s) slot_w[size_t(s)] = full ? s - p / 2 : (s == p / 2 ? -p / 2 : s);
    SetupTimer tm(poisson ? "solver set (Poisson)" : "solver set (Helmholtz)");
    auto ds = std::make_unique<DevSet>();
    // flags bit1: execute the reference's shift counts (no tail-avoidance margin)
    // flags bit2: solve with the ADI kernel (the reference algorithm) instead of fast diagonalization
    // the ADI data (enclosures, shift plans, factor blocks) only when the ADI kernel is the solver
    ds->host = build_solver_set(*sizeops, slot_w, poisson, scale, tol, radial_cache, (flags & 1) != 0,
                                (flags & 2) ? 1.0 : 4.0, (flags & 4) == 0, (flags & 4) != 0, false);
    const SolverSet& h = ds->host;
    if (h.has_diag) {
        CCF_CUDA(cudaMalloc(&ds->dg, h.dg.size() * sizeof(double)));
        CCF_H2D(ds->dg, h.dg.data(), h.dg.size() * sizeof(double));
    }
    CCF_CUDA(cudaMalloc(&ds->coef, h.coef.size() * sizeof(double)));
    CCF_H2D(ds->coef, h.coef.data(), h.coef.size() * sizeof(double));
    CCF_CUDA(cudaMalloc(&ds->slots, h.slots.size() * sizeof(AdiSlot)));
    CCF_H2D(ds->slots, h.slots.data(), h.slots.size() * sizeof(AdiSlot));
    std::vector<int> J(h.slots.size());
    for (size_t s = 0; s < J.size(); ++s) J[s] = h.slots[s].J;
    CCF_CUDA(cudaMalloc(&ds->J, J.size() * sizeof(int)));
    CCF_H2D(ds->J, J.data(), J.size() * sizeof(int));
    // tasks: longest slots first (load balance of the J-heterogeneous batch)
    std::vector<int> order(size_t(g.nslots));
    for (int s = 0; s < g.nslots; ++s) order[size_t(s)] = s;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return J[size_t(a)] > J[size_t(b)]; });
    for (int nt = 1; nt <= 2; ++nt) {
        std::vector<AdiTask> tasks;
        for (int s : order)
            for (int t = 0; t < nt; ++t)
                for (int k0 = 0; k0 < 2; ++k0)
                    for (int pl = 0; pl < 2; ++pl) tasks.push_back({t, s, k0, pl});
        ds->ntasks[nt - 1] = int(tasks.size());
        CCF_CUDA(cudaMalloc(&ds->tasks[nt - 1], tasks.size() * sizeof(AdiTask)));
        CCF_H2D(ds->tasks[nt - 1], tasks.data(), tasks.size() * sizeof(AdiTask));
    }
    DevSet& ref = *ds;
    sets[key] = std::move(ds);
    return ref;
}

void Ctx::run_adi(DevSet& set, bool full, int ntensor, const double* const* src0, const double* w0, int n0,
                  const double* const* src1, const double* w1, int n1, double* out0, double* out1) {
    if (!(flags & 4) || set.host.maxJ == 0)
        throw Error(INTERNAL, "run_adi: this context solves by fast diagonalization (no ADI data; flag bit 2)");
    const Geo& g = geo(full);
    last_adi_kind = set.host.poisson ? "Poisson" : "Helmholtz";
    last_adi_ntensor = ntensor;
    last_adi_nslots = g.nslots;
    AdiParams P{};
    P.g = g;
    P.M = M;
    P.N = N;
    P.pitch = pitch;
    P.ntasks = set.ntasks[ntensor - 1];
    P.coef = set.coef;
    P.slots = set.slots;
    P.tasks = set.tasks[ntensor - 1];
    P.nsrc[0] = n0;
    P.nsrc[1] = n1;
    for (int i = 0; i < n0; ++i) {
        P.src[0][i] = src0[i];
        P.wsrc[0][i] = w0[i];
    }
    for (int i = 0; i < n1; ++i) {
        P.src[1][i] = src1[i];
        P.wsrc[1][i] = w1[i];
    }
    P.out[0] = out0;
    P.out[1] = out1;
    P.eprime = ws.eprime.p;
    P.estride = estride;
    P.escr = ws.escr.p;
    P.xscr = ws.xscr.p;
    P.Mpad = Mpad;
    P.Npad = Npad;
    P.lrows = Mpad + 2;
    P.rrows = Npad + 2;
    P.lanes = adi_lanes();
    P.hc = adi_split() ? spike_split(Mpad) : 0;
    P.hr = adi_split() ? spike_split(Npad) : 0;
    P.res2 = ws.res2;
    P.e2 = ws.e2;
    P.active = ws.active;
    const int nts = ntensor * g.nslots;
    adi_init_kernel<<<(nts + 127) / 128, 128, 0, stream>>>(ws.active, ws.res2, ws.e2, nts);
    ++launches;
    const int threads = adi_split() ? 2 * adi_lanes() : adi_lanes();
    const size_t smem = adi_smem_bytes();
    RoundCheck rc{};
    rc.ntensor = ntensor;
    rc.nslots = g.nslots;
    rc.tol = tol;
    rc.res2 = ws.res2;
    rc.e2 = ws.e2;
    rc.active = ws.active;
    rc.history = ws.history;
    rc.rounds = ws.rounds;
    rc.err = ws.err;
    rc.J = set.J;
    rc.iters = ws.iters;
    for (int round = 0; round < 4; ++round) {
        P.round = round;
        adi_launch(P, threads, smem, stream);
        rc.round = round;
        adi_round_check<<<(nts + 127) / 128, 128, 0, stream>>>(rc);
        launches += 2;
    }
    if (keep_history) {  // diagnostics: per-kind copy of the round bookkeeping (ccf_adi_last_rounds)
        const int k = set.host.poisson ? 1 : 2;
        kept_shape[k][0] = ntensor;
        kept_shape[k][1] = g.nslots;
        CCF_CUDA(cudaMemcpyAsync(kept_rounds[k].p, ws.rounds, sizeof(int) * size_t(nts), cudaMemcpyDeviceToDevice, stream));
        CCF_CUDA(cudaMemcpyAsync(kept_hist[k].p, ws.history, sizeof(double) * 4 * size_t(nts), cudaMemcpyDeviceToDevice,
                                 stream));
    }
    CCF_CUDA(cudaGetLastError());
}

void Ctx::check_adi_error(bool full) {
    int e[4];
    CCF_CUDA(cudaMemcpyAsync(e, ws.err, sizeof(e), cudaMemcpyDeviceToHost, stream));
    sync();
    if (e[0] == 0) return;
    const Geo& g = geo(full);
    std::vector<double> hist(4);
    CCF_CUDA(cudaMemcpy(hist.data(), ws.history + size_t(e[1] * g.nslots + e[2]) * 4, sizeof(double) * 4,
                        cudaMemcpyDeviceToHost));
    CCF_CUDA(cudaMemsetAsync(ws.err, 0, sizeof(int) * 4, stream));
    const int s = e[2];
    const int l = full ? s : (s == p / 2 ? 0 : s + p / 2);
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.3e", hist[3]);
    Error err(NON_CONVERGENCE, std::string("modal solve failed for Fourier slice ") + std::to_string(l) + " (" +
                                   last_adi_kind + "): ADI did not converge: relative residual " + buf +
                                   " after 4 rounds");
    err.slice = l;
    err.history = hist;
    throw err;
}

void Ctx::require_finite(const double* dptr, long count, const char* what) {
    CCF_CUDA(cudaMemsetAsync(ws.flag, 0, sizeof(int), stream));
    finite_check_kernel<<<std::min<long>(1184, (count + 255) / 256), 256, 0, stream>>>(dptr, count, ws.flag);
    ++launches;
    int f = 0;
    CCF_CUDA(cudaMemcpyAsync(&f, ws.flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
    sync();
    if (f) throw Error(NUMERICAL, std::string(what) + ": non-finite right-hand side");
}

void Ctx::load_coeff(const double* ref, double* dst, bool full, int cls, int slot) {
    const long nref = 2L * m * n * p;
    const double* dref = ref;
    if (!is_device_ptr(ref)) {
        if (stage_in[slot].n < size_t(nref)) stage_in[slot].alloc(size_t(nref));
        if (full) {
            CCF_CUDA(cudaMemcpyAsync(stage_in[slot].p, ref, sizeof(double) * nref, cudaMemcpyHostToDevice, stream));
        } else {  // the half spectrum reads only slices l = 0 (Nyquist) and l >= p/2 (w >= 0): copy just those
            const long sl = 2L * n * m;
            CCF_CUDA(cudaMemcpyAsync(stage_in[slot].p, ref, sizeof(double) * sl, cudaMemcpyHostToDevice, stream));
            CCF_CUDA(cudaMemcpyAsync(stage_in[slot].p + sl * (p / 2), ref + sl * (p / 2), sizeof(double) * sl * (p - p / 2),
                                     cudaMemcpyHostToDevice, stream));
        }
        dref = stage_in[slot].p;
    }
    const Geo& g = geo(full);
    const long total = long(g.nslots) * g.slot_stride;
    ref_to_h_kernel<<<std::min<long>(4736, (total + 255) / 256), 256, 0, stream>>>(dref, dst, g, int(full), cls);
    ++launches;
}

void Ctx::store_coeff(const double* src, double* ref, bool full, int cls, int slot, bool accumulate) {
    const long nref = 2L * m * n * p;
    double* dref = ref;
    const bool host = !is_device_ptr(ref);
    if (host) {
        if (stage_out[slot].n < size_t(nref)) stage_out[slot].alloc(size_t(nref));
        dref = stage_out[slot].p;
        if (accumulate)
            CCF_CUDA(cudaMemcpyAsync(dref, ref, sizeof(double) * nref, cudaMemcpyHostToDevice, stream));
    }
    const Geo& g = geo(full);
    const long total = long(p) * n * m;
    h_to_ref_kernel<<<std::min<long>(4736, (total + 255) / 256), 256, 0, stream>>>(src, dref, g, int(full), cls, int(accumulate));
    ++launches;
    if (host) CCF_CUDA(cudaMemcpyAsync(ref, dref, sizeof(double) * nref, cudaMemcpyDeviceToHost, stream));
}

void Ctx::load_values(const double* vals, double* dst) {
    const long nv = long(m) * n * p;
    if (is_device_ptr(vals)) CCF_CUDA(cudaMemcpyAsync(dst, vals, sizeof(double) * nv, cudaMemcpyDeviceToDevice, stream));
    else CCF_CUDA(cudaMemcpyAsync(dst, vals, sizeof(double) * nv, cudaMemcpyHostToDevice, stream));
}

void Ctx::store_values(const double* src, double* vals) {
    const long nv = long(m) * n * p;
    if (is_device_ptr(vals)) CCF_CUDA(cudaMemcpyAsync(vals, src, sizeof(double) * nv, cudaMemcpyDeviceToDevice, stream));
    else CCF_CUDA(cudaMemcpyAsync(vals, src, sizeof(double) * nv, cudaMemcpyDeviceToHost, stream));
}

}  // namespace ccf
