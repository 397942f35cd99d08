// Host-side context of the B200 CCF library (behind include/ccf.h).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "ccf_device.cuh"
#include "kernels.cuh"
#include "modal.hpp"
#include "setup.hpp"

namespace ccf {

#define CCF_CUDA(x)                                                                                          \
    do {                                                                                                     \
        cudaError_t _e = (x);                                                                                \
        if (_e != cudaSuccess) throw ::ccf::Error(::ccf::CUDA_ERR, std::string("CUDA: ") + cudaGetErrorString(_e) + \
                                                                     " at " __FILE__ ":" + std::to_string(__LINE__)); \
    } while (0)

// Device buffer (RAII).
struct DBuf {
    double* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count);
    ~DBuf();
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept;
};

// Packed solver set resident on the device.
struct DevSet {
    SolverSet host;
    double* coef = nullptr;
    AdiSlot* slots = nullptr;
    int* J = nullptr;
    AdiTask* tasks[2] = {nullptr, nullptr};  // for 1 and 2 tensors
    int ntasks[2] = {0, 0};
    double* dg = nullptr;  // fast-diagonalization matrices (host.dg), when built
    ~DevSet();
};

struct Workspace {  // ADI round bookkeeping
    DBuf eprime, escr, xscr;
    double *res2 = nullptr, *e2 = nullptr, *history = nullptr;
    int *active = nullptr, *rounds = nullptr, *err = nullptr, *flag = nullptr;
    unsigned long long* iters = nullptr;
    int cap_slots = 0;
};

struct Ctx {
    int m, n, p, device, flags;
    double tol;
    cudaStream_t stream = nullptr, own_stream = nullptr;
    Geo gh{}, gf{};  // half-spectrum and full-spectrum slot tables
    int M, N, pitch, Mpad, Npad;
    long estride;
    size_t adi_smem_bytes() const;
    int adi_lanes() const;
    bool adi_split() const;
    std::unique_ptr<SizeOps> sizeops;
    std::map<int, Range> radial_cache;
    std::map<std::tuple<int, int, double>, std::unique_ptr<DevSet>> sets;  // (full, poisson, scale)
    Workspace ws;
    DBuf stage_in[4], stage_out[2];
    DBuf tens[16];  // generic device scratch tensors (compressed layout, full size)
    long launches = 0;
    const char* last_adi_kind = "";
    int last_adi_ntensor = 0, last_adi_nslots = 0;  // shape of ws.rounds / ws.history of the last ADI run
    bool keep_history = false;  // diagnostics: keep the last Poisson (1) / Helmholtz (2) round bookkeeping
    DBuf kept_hist[3], kept_rounds[3];
    int kept_shape[3][2] = {};
    // optional stage profiling: events recorded at stage boundaries when enabled
    bool profiling = false;
    double gemm_flops = 0.0;  // FP64 tensor-core flops of the GEMM launches enqueued since reset_stats
    std::vector<cudaEvent_t> prof_events;
    std::vector<std::string> prof_names;
    void mark(const char* name) {
        if (!profiling) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, stream);
        prof_events.push_back(e);
        prof_names.push_back(name);
    }
    // last error
    int err_kind = 0, err_slice = -1, err_shift = -1;
    std::vector<double> err_hist;
    std::string err_msg;

    Ctx(int m, int n, int p, int device, double tol, int flags);
    ~Ctx();
    const Geo& geo(bool full) const { return full ? gf : gh; }
    long tensor_doubles(bool full) const { return long(geo(full).nslots) * geo(full).slot_stride; }
    DevSet& set(bool full, bool poisson, double scale);
    // Run the batched ADI for 1 or 2 tensors that share the solver set.
    // srcs[t]: sum_i w_i * src_i forms the modal RHS of tensor t; out[t] compressed output.
    void run_adi(DevSet& set, bool full, int ntensor, const double* const* src0, const double* w0, int n0,
                 const double* const* src1, const double* w1, int n1, double* out0, double* out1);
    void check_adi_error(bool full);  // synchronises and raises NonConvergenceError
    bool is_device_ptr(const void* p) const;
    // Reference-layout coefficient tensor (host or device) -> compressed device tensor.
    void load_coeff(const double* ref, double* dst, bool full, int cls, int slot);
    void store_coeff(const double* src, double* ref, bool full, int cls, int slot, bool accumulate = false);
    void load_values(const double* vals, double* dst);  // reference-layout real field -> device
    void store_values(const double* src, double* vals);
    void require_finite(const double* dptr, long n, const char* what);
    void sync();
};

}  // namespace ccf
