// Mode sharding of the NS step over the GPUs of one node.
//
// Partition: rank r owns the contiguous half-spectrum slots [sb[r], sb[r+1]) in every per-mode
// stage (Poisson / Helmholtz eigen-coordinate solves, z transforms, composite radial operators:
// all independent per Fourier mode, proj/src/ptns.cpp:217-267 has no coupling between modes
// outside the pointwise product) and the radial value rows [rb[r], rb[r+1]) in the theta stage
// (theta FFT x cross product x theta FFT, which couples all modes at one (r, z) point).
//
// Exchange: the six theta inputs and three outputs live in one "exchange" allocation per rank with
// identical offsets on every rank. The theta kernel of rank r reads slot s of its rows from the
// owning rank's allocation and stores the cross product's spectrum there (peer loads / stores over
// NVLink through CUDA IPC mappings; rdelta[q] = mapped base of rank q - own base). The transpose is
// therefore fused into the FFT kernel: no pack, no all-to-all buffer, no extra HBM pass.
//
// Ordering: two rank barriers per step, before the theta stage (every owner's inputs written, every
// owner done reading the previous step's outputs) and after it (every output stored). DEVICE mode:
// a one-warp kernel on the stream (release store of the epoch into each peer's flag slot, acquire
// spin on the own slots), graph-capturable, epoch kept on the device. HOST mode: stream
// synchronisation + a host barrier (caller callback, or an in-process barrier between linked
// contexts), used to emulate ranks on one GPU without device-side waiting between them.
#include <chrono>
#include <cstring>
#include <condition_variable>
#include <mutex>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "context.hpp"

namespace ccf {

struct HostBarrier {
    std::mutex mu;
    std::condition_variable cv;
    int n, waiting = 0;
    long gen = 0;
    explicit HostBarrier(int n_) : n(n_) {}
    bool wait(double timeout_s) {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++waiting == n) {
            waiting = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        return cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g; });
    }
};

namespace {

struct BarrierArgs {
    unsigned* peer_flags[kMaxRanks];
    unsigned* my_flags;
    unsigned* epoch;
    int* err;
    int rank, world;
};

// lane q: signal arrival of this rank in rank q's flag slot [rank], then wait for rank q's
// arrival in the own slot [q]. Bounded spin (~10 s): a lost peer sets err instead of hanging.
__global__ void shard_barrier_kernel(BarrierArgs b) {
    __shared__ unsigned e;
    if (threadIdx.x == 0) e = *b.epoch + 1u;
    __syncthreads();
    const int q = threadIdx.x;
    if (q < b.world) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(b.peer_flags[q] + b.rank), "r"(e) : "memory");
        const unsigned* f = b.my_flags + q;
        const long long t0 = clock64();
        for (;;) {
            unsigned v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if (int(v - e) >= 0) break;
            if (clock64() - t0 > 20000000000LL) {  // ~10 s at 1.97 GHz
                atomicExch(b.err, 1);
                break;
            }
            __nanosleep(32);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *b.epoch = e;
}

}  // namespace

void shard_bounds(int count, int world, int* bounds) {
    for (int r = 0; r <= world; ++r) bounds[r] = int((long(r) * count) / world);
}

void Ctx::shard_init(int rank, int world) {
    if (sh.xbuf) throw Error(CONFIG_ERROR, "ccf_shard_init: context already sharded");
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
        throw Error(CONFIG_ERROR, "ccf_shard_init: need 0 <= rank < world <= 8");
    const Geo& g = gh;
    if (world > g.nslots || world > g.mh) throw Error(CONFIG_ERROR, "ccf_shard_init: more ranks than Fourier slots or rows");
    sh.rank = rank;
    sh.world = world;
    shard_bounds(g.nslots, world, sh.sb);
    shard_bounds(g.mh, world, sh.rb);
    sh.s_lo = sh.sb[rank];
    sh.s_hi = sh.sb[rank + 1];
    sh.r_lo = sh.rb[rank];
    sh.r_hi = sh.rb[rank + 1];
    if (world == 1) return;
    const size_t T = size_t(tensor_doubles(false));
    const size_t bytes = T * kExchangeTensors * sizeof(double) + 256;
    CCF_CUDA(cudaMalloc(&sh.xbuf, bytes));
    CCF_CUDA(cudaMemset(sh.xbuf, 0, bytes));
    sh.flags = reinterpret_cast<unsigned*>(sh.xbuf + T * kExchangeTensors);
    CCF_CUDA(cudaMalloc(&sh.epoch, 64));
    CCF_CUDA(cudaMemset(sh.epoch, 0, 64));
    CCF_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // before any use on the library's stream
    sh.err = reinterpret_cast<int*>(sh.epoch + 4);
    for (int r = 0; r < kMaxRanks; ++r) {
        sh.rdelta[r] = 0;
        sh.peer_flags[r] = sh.flags;
    }
}

void Ctx::shard_sync() {
    if (!sh.sharded()) return;
    if (sh.mode == Shard::DEVICE) {
        BarrierArgs b{};
        for (int q = 0; q < kMaxRanks; ++q) b.peer_flags[q] = sh.peer_flags[q];
        b.my_flags = sh.flags;
        b.epoch = sh.epoch;
        b.err = sh.err;
        b.rank = sh.rank;
        b.world = sh.world;
        shard_barrier_kernel<<<1, 32, 0, stream>>>(b);
        ++launches;
    } else if (sh.mode == Shard::HOST) {
        CCF_CUDA(cudaStreamSynchronize(stream));
        if (sh.local) {
            if (!sh.local->wait(120.0)) throw Error(INTERNAL, "shard: host barrier timed out (a linked rank stopped)");
        } else if (sh.host_fn) {
            sh.host_fn(sh.host_user);
        }
    } else {
        throw Error(CONFIG_ERROR, "shard: peers not connected (ccf_shard_open_ipc / ccf_shard_link_local)");
    }
}

void Ctx::shard_check() {
    if (!sh.sharded() || !sh.err) return;
    CCF_CUDA(cudaStreamSynchronize(stream));
    int e = 0;
    CCF_CUDA(cudaMemcpy(&e, sh.err, sizeof(int), cudaMemcpyDeviceToHost));
    if (e) throw Error(INTERNAL, "shard: device barrier timed out (a peer rank stopped)");
}

void Ctx::shard_close() {
    for (int r = 0; r < kMaxRanks; ++r)
        if (sh.ipc_open[r]) {
            cudaIpcCloseMemHandle(sh.ipc_open[r]);
            sh.ipc_open[r] = nullptr;
        }
    if (sh.xbuf) cudaFree(sh.xbuf);
    if (sh.epoch) cudaFree(sh.epoch);
    sh.xbuf = nullptr;
    sh.epoch = nullptr;
    sh.local.reset();
}

void Ctx::require_unsharded(const char* what) const {
    if (sh.sharded())
        throw Error(CONFIG_ERROR, std::string(what) + ": a mode-sharded context runs the NS / heat stepper only");
}

// ---- peer connection (C-ABI helpers in api.cu)

// handle blob (kShardHandleBytes): [0, 64) cudaIpcMemHandle_t of the allocation holding the exchange
// buffer, [64, 72) byte offset of the buffer inside it (the runtime may place a cudaMalloc inside a
// larger driver allocation, and an opened handle maps that allocation's base)
void shard_ipc_handle(Ctx& c, void* out) {
    if (!c.sh.xbuf) throw Error(CONFIG_ERROR, "ccf_shard_ipc_handle: context not sharded");
    static PFN_cuMemGetAddressRange_v3020 range = [] {
        void* e = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &e, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            e = nullptr;
        return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(e);
    }();
    if (!range) throw Error(CUDA_ERR, "ccf_shard_ipc_handle: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, CUdeviceptr(reinterpret_cast<uintptr_t>(c.sh.xbuf))) != CUDA_SUCCESS)
        throw Error(CUDA_ERR, "ccf_shard_ipc_handle: cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    CCF_CUDA(cudaIpcGetMemHandle(&h, c.sh.xbuf));
    const unsigned long long off = reinterpret_cast<uintptr_t>(c.sh.xbuf) - uintptr_t(base);
    std::memset(out, 0, kShardHandleBytes);
    std::memcpy(out, &h, sizeof(h));
    std::memcpy(static_cast<char*>(out) + 64, &off, sizeof(off));
}

void shard_open_ipc(Ctx& c, const void* handles) {
    Shard& s = c.sh;
    if (!s.xbuf) throw Error(CONFIG_ERROR, "ccf_shard_open_ipc: context not sharded");
    const size_t T = size_t(c.tensor_doubles(false));
    for (int r = 0; r < s.world; ++r) {
        if (r == s.rank) continue;
        cudaIpcMemHandle_t h;
        unsigned long long off = 0;
        const char* blob = static_cast<const char*>(handles) + size_t(r) * kShardHandleBytes;
        std::memcpy(&h, blob, sizeof(h));
        std::memcpy(&off, blob + 64, sizeof(off));
        void* p = nullptr;
        CCF_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        s.ipc_open[r] = p;
        double* base = reinterpret_cast<double*>(static_cast<char*>(p) + off);
        s.rdelta[r] = long(base - s.xbuf);
        s.peer_flags[r] = reinterpret_cast<unsigned*>(base + T * kExchangeTensors);
    }
    s.rdelta[s.rank] = 0;
    s.peer_flags[s.rank] = s.flags;
    s.mode = Shard::DEVICE;
}

void shard_link_local(Ctx* const* cs, int world) {
    auto bar = std::make_shared<HostBarrier>(world);
    for (int i = 0; i < world; ++i) {
        Shard& s = cs[i]->sh;
        if (!s.xbuf || s.world != world || s.rank != i)
            throw Error(CONFIG_ERROR, "ccf_shard_link_local: contexts must be sharded as ranks 0..world-1 of world");
        if (cs[i]->device != cs[0]->device)
            throw Error(CONFIG_ERROR, "ccf_shard_link_local: linked contexts share one device");
        for (int r = 0; r < world; ++r) {
            s.rdelta[r] = long(cs[r]->sh.xbuf - s.xbuf);
            s.peer_flags[r] = cs[r]->sh.flags;
        }
        s.local = bar;
        s.mode = Shard::HOST;
    }
}

void shard_set_host_barrier(Ctx& c, void (*fn)(void*), void* user) {
    if (!c.sh.xbuf) throw Error(CONFIG_ERROR, "ccf_shard_set_host_barrier: context not sharded");
    c.sh.host_fn = fn;
    c.sh.host_user = user;
    c.sh.local.reset();
    c.sh.mode = fn ? Shard::HOST : Shard::DEVICE;
}

}  // namespace ccf
