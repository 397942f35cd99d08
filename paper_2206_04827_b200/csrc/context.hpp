// Host-side context of the B200 CCF library (behind include/ccf.h).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
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

// Synchronous host -> device copy. cudaMemcpy from pageable memory may return before the DMA lands,
// and it runs on the legacy default stream, which the library's non-blocking streams do not wait
// for: complete it before returning.
#define CCF_H2D(dst, src, bytes)                                                       \
    do {                                                                               \
        CCF_CUDA(cudaMemcpy((dst), (src), (bytes), cudaMemcpyHostToDevice));           \
        CCF_CUDA(cudaStreamSynchronize(cudaStreamLegacy));                             \
    } while (0)

// Setup-phase timer (CCF_SETUP_TRACE=1: one stderr line per phase).
struct SetupTimer {
    const char* what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit SetupTimer(const char* w) : what(w) {}
    ~SetupTimer() {
        static const bool on = std::getenv("CCF_SETUP_TRACE") != nullptr;
        if (on)
            std::fprintf(stderr, "[setup] %-28s %.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
};

// Device buffer (RAII).
struct DBuf {
    double* p = nullptr;
    size_t n = 0;
    bool own = true;  // false: a view into memory owned elsewhere (a stepper arena)
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count);
    void view(double* ptr, size_t count);
    ~DBuf();
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), own(o.own) { o.p = nullptr; o.n = 0; o.own = true; }
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
    int* hstat = nullptr;  // pinned host copy of {err[4], stepper flag}: one sync per status read (ccf_ns_step)
};

// Mode sharding of the NS step over the GPUs of one node (csrc/shard.cu).
// Every rank keeps full-extent tensors (same layout, same offsets on every rank) and computes the
// half-spectrum slots [s_lo, s_hi) in every per-mode stage. The only exchange is the theta stage:
// rank r transforms the radial rows [r_lo, r_hi) of all slots, reading each slot's (r,z)-values
// straight from the owning rank's exchange buffer and storing the cross product back into it
// (NVLink peer loads / stores at the same offset; no pack, no copy). Two rank barriers per step
// (before and after the theta stage) order those accesses.
constexpr int kMaxRanks = 8;
constexpr int kShardHandleBytes = 128;  // include/ccf.h CCF_SHARD_HANDLE_BYTES
constexpr int kExchangeTensors = 9;  // pipeline scratch 6..14: the six theta inputs and three outputs
struct HostBarrier;                  // in-process barrier of linked contexts (shard.cu)
struct Shard {
    int rank = 0, world = 1;
    int s_lo = 0, s_hi = 0;  // owned half-spectrum slots
    int r_lo = 0, r_hi = 0;  // owned theta rows (r > 0 grid rows jr)
    int sb[kMaxRanks + 1] = {}, rb[kMaxRanks + 1] = {};  // slot / row bounds of every rank
    double* xbuf = nullptr;      // exchange allocation: kExchangeTensors tensors, then the barrier flags
    unsigned* flags = nullptr;   // kMaxRanks arrival counters in xbuf, written by the peers
    unsigned* epoch = nullptr;   // device barrier epoch (device-resident: CUDA-graph replay safe)
    int* err = nullptr;          // barrier timeout flag
    long rdelta[kMaxRanks] = {};             // doubles from xbuf to rank r's exchange buffer (as mapped here)
    unsigned* peer_flags[kMaxRanks] = {};    // rank r's flag array (as mapped here)
    void* ipc_open[kMaxRanks] = {};          // cudaIpcOpenMemHandle mappings to close
    enum Mode { NONE = 0, DEVICE = 1, HOST = 2 } mode = NONE;
    void (*host_fn)(void*) = nullptr;        // HOST mode: caller-provided rank barrier
    void* host_user = nullptr;
    std::shared_ptr<HostBarrier> local;      // HOST mode between linked contexts of one process
    bool sharded() const { return world > 1; }
    long slot_delta(int s) const {
        int r = 0;
        while (r + 1 < world && s >= sb[r + 1]) ++r;
        return rdelta[r];
    }
};

struct Ctx {
    int m, n, p, device, flags;
    Shard sh;
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

    // stepper state arenas: a stepper's history rings live in one block, which a destroyed stepper returns
    // here and the next stepper of the context reuses (no cudaMalloc / cudaFree per stepper: ~0.4 ms per
    // 68 MB tensor at 256^3, i.e. most of a fresh stepper's creation time)
    std::vector<std::pair<size_t, double*>> arena_cache;
    double* arena_get(size_t count);  // zero-filled on this context's stream
    void arena_put(double* p, size_t count);

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
    // mode sharding (shard.cu)
    void shard_init(int rank, int world);
    void shard_sync();              // rank barrier on the stream (no-op unsharded)
    void shard_check();             // synchronises; raises a barrier timeout
    void shard_close();
    void require_unsharded(const char* what) const;
};

// CCF1 FieldFile I/O (fieldio.cu, proj/src/io.cpp:12-109)
uint32_t crc32_host(const uint8_t* data, size_t len);
uint32_t crc32_device(const void* dptr, size_t nbytes, cudaStream_t stream);
void write_field_file(const std::string& path, int kind, int m, int n, int p, const double* payload, bool device,
                      cudaStream_t stream);
void read_field_header(const std::string& path, int& kind, int& m, int& n, int& p);
void read_field_file(const std::string& path, int& kind, int& m, int& n, int& p, double* out, size_t cap, bool device,
                     cudaStream_t stream);
// contiguous partition of count items over world ranks: rank r owns [bounds[r], bounds[r+1])
void shard_bounds(int count, int world, int* bounds);
// peer connection of sharded contexts (shard.cu)
void shard_ipc_handle(Ctx& c, void* out);           // kShardHandleBytes: IPC handle + offset of the exchange buffer
void shard_open_ipc(Ctx& c, const void* handles);   // world x kShardHandleBytes (own entry ignored); DEVICE barriers
void shard_link_local(Ctx* const* cs, int world);   // ranks of one process on one device; HOST barriers
void shard_set_host_barrier(Ctx& c, void (*fn)(void*), void* user);

}  // namespace ccf
