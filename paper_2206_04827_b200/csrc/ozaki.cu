// FP64 GEMMs on the INT8 tensor cores (tcgen05.mma kind::i8 + TMEM), see ozaki.hpp.
#include <algorithm>
#include <climits>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "context.hpp"
#include "ozaki.hpp"
#include "ozaki_dev.cuh"

namespace ccf {
namespace {

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// Digit d (byte 5 - d of X) of four fixed-point values held as fma(x, 2^(47-e), 1.5 2^52) doubles, packed into one
// word (value u in byte u): X bytes 0-3 are the low word, bytes 4-5 the low half of the high word
__device__ __forceinline__ uint32_t oz_digit_word(const double* xb, int d) {
    const int hiw = d < 2;
    const uint32_t k = hiw ? uint32_t(1 - d) : uint32_t(5 - d);  // byte within the word
    uint32_t w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = uint32_t(hiw ? __double2hiint(xb[u]) : __double2loint(xb[u]));
    const uint32_t sel = k | ((4u + k) << 4);
    return __byte_perm(__byte_perm(w[0], w[1], sel), __byte_perm(w[2], w[3], sel), 0x5410);
}

// A-side split: one warp per panel row, lane l holds reduction indices 4l .. 4l + 3 (oz_warp_row)
__global__ void __launch_bounds__(256) oz_split_rows_kernel(const OzSplitJob* __restrict__ jobs) {
    const OzSplitJob& J = jobs[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= J.rows_pad) return;
    const double* src = J.src[0] + long(r) * J.ld + 4 * lane;
    const int nrows = J.nrows, ncols = J.ncols;
    double v[4];
    if (r < nrows && 4 * lane + 4 <= ncols && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(src)), b = __ldg(reinterpret_cast<const double2*>(src + 2));
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = (r < nrows && 4 * lane + u < ncols) ? __ldg(src + u) : 0.0;
    }
    oz_warp_row(v, J.dst[0], J.stride, r, J.sc + r);
}

// B-side split with transpose: CTA = (job, 128-row tile of the panel), thread = panel row = source
// column (loads coalesced over the columns). Per plane: the tile max 2^e_p (CTA reduction); per row:
// the common max of the normalised planes 2^e_r; digits of x 2^-e_p relative to 2^e_r are staged as
// the swizzled panel image in shared memory and stored with bulk copies (16 KB per slice).
constexpr int kSplitThreads = 128;
size_t oz_split_cols_smem() { return size_t(kOzS) * 128 * kOzK + 1024; }
__global__ void __launch_bounds__(kSplitThreads) oz_split_cols_kernel(const OzSplitJob* __restrict__ jobs) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* stage = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ double red[kOzGroup][kSplitThreads / 32];
    const OzSplitJob& J = jobs[blockIdx.y];
    const int tile = blockIdx.x, ntiles = J.rows_pad / 128;
    if (tile >= ntiles) return;
    const int rl = threadIdx.x, r = tile * 128 + rl, lane = rl & 31, wid = rl >> 5;
    const bool live = r < J.nrows;
    const int nsrc = J.nsrc, ncols = J.ncols;
    const long ld = J.ld;
    double m[kOzGroup];
#pragma unroll
    for (int g = 0; g < kOzGroup; ++g) {
        m[g] = 0.0;
        if (g < nsrc && live) {
            const double* src = J.src[g] + r;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int k = 0;
            for (; k + 4 <= ncols; k += 4) {
                a0 = fmax(a0, fabs(__ldg(src + long(k) * ld)));
                a1 = fmax(a1, fabs(__ldg(src + long(k + 1) * ld)));
                a2 = fmax(a2, fabs(__ldg(src + long(k + 2) * ld)));
                a3 = fmax(a3, fabs(__ldg(src + long(k + 3) * ld)));
            }
            for (; k < ncols; ++k) a0 = fmax(a0, fabs(__ldg(src + long(k) * ld)));
            m[g] = fmax(fmax(a0, a1), fmax(a2, a3));
        }
        double w = m[g];
#pragma unroll
        for (int o = 16; o; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (lane == 0) red[g][wid] = w;
    }
    __syncthreads();
    int ep[kOzGroup];
    double sig = 0.0;
#pragma unroll
    for (int g = 0; g < kOzGroup; ++g) {
        const double pm = fmax(fmax(red[g][0], red[g][1]), fmax(red[g][2], red[g][3]));
        ep[g] = pm > 0.0 ? oz_exponent(pm) : 0;
        if (g < nsrc) sig = fmax(sig, ldexp(m[g], -ep[g]));
    }
    const int er = sig > 0.0 ? oz_exponent(sig) : 0;
    if (rl < nsrc && J.pe) J.pe[rl * ntiles + tile] = ep[rl];
    for (int g = 0; g < nsrc; ++g) {
        const double* src = J.src[g] + r;
        const int E = er + ep[g];
#pragma unroll 1
        for (int kc = 0; kc < kOzK / 16; ++kc) {
            uint32_t w[kOzS][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                long long X[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = 16 * kc + 4 * q + u;
                    const double x = (live && k < ncols) ? __ldg(src + long(k) * ld) : 0.0;
                    X[u] = sig > 0.0 ? oz_fixed(x, E) : 0;
                }
#pragma unroll
                for (int d = 0; d < kOzS; ++d)
                    w[d][q] = oz_digit(X[0], d) | (oz_digit(X[1], d) << 8) | (oz_digit(X[2], d) << 16) | (oz_digit(X[3], d) << 24);
            }
            const uint32_t off = oz_swz(rl, 16 * kc);
#pragma unroll
            for (int d = 0; d < kOzS; ++d)
                *reinterpret_cast<uint4*>(stage + size_t(d) * 128 * kOzK + off) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staged image -> async proxy (bulk store)
        __syncthreads();
        if (rl == 0) {
            for (int d = 0; d < kOzS; ++d)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 J.dst[g] + size_t(d) * J.stride + size_t(tile) * 128 * kOzK),
                             "r"(uint32_t(__cvta_generic_to_shared(stage + size_t(d) * 128 * kOzK))), "r"(uint32_t(128 * kOzK))
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // stage free for the next plane
        }
        __syncthreads();
    }
    J.sc[r] = sig > 0.0 ? ldexp(1.0, er) : 0.0;
    if (rl == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before exit
}

// B-side split into the MN-major panel layout (slice of a 128-column tile: 128 k-rows of 128 column
// bytes, row k at oz_swz(k, n); tcgen05 reads it with b_major = MN): no transpose, so a CTA (512
// threads) holds the whole (plane, tile) in registers (warp = 8 k-rows, lane = 4 columns; loads and
// stores fully coalesced), reduces its max 2^e (pe[plane * tiles + tile]) and writes the digits
// relative to 2^e in one pass. Column scales sc = 1 (absolute accuracy 2^-48 of the tile max).
constexpr int kMnThreads = 512;
__global__ void __launch_bounds__(kMnThreads) oz_split_mn_kernel(const OzSplitJob* __restrict__ jobs) {
    __shared__ double red[kMnThreads / 32];
    const OzSplitJob& J = jobs[blockIdx.y / kOzGroup];
    const int g = blockIdx.y % kOzGroup, tile = blockIdx.x, ntiles = J.rows_pad / 128;
    if (g >= J.nsrc || tile >= ntiles) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n0 = tile * 128 + 4 * lane;  // this lane's 4 columns
    const int ncols = J.ncols, nrows = J.nrows;
    const double* src = J.src[g] + n0;
    double v[8][4];
    double mx = 0.0;
    const bool vec = n0 + 4 <= nrows && ((reinterpret_cast<uintptr_t>(src) | uintptr_t(J.ld * 8)) & 15) == 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = wid * 8 + i;
        if (k < ncols && vec) {
            const double2 a = __ldg(reinterpret_cast<const double2*>(src + long(k) * J.ld));
            const double2 b = __ldg(reinterpret_cast<const double2*>(src + long(k) * J.ld + 2));
            v[i][0] = a.x; v[i][1] = a.y; v[i][2] = b.x; v[i][3] = b.y;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[i][u] = (k < ncols && n0 + u < nrows) ? __ldg(src + long(k) * J.ld + u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) mx = fmax(mx, fabs(v[i][u]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red[wid] = mx;
    __syncthreads();
    mx = red[0];
#pragma unroll
    for (int w = 1; w < kMnThreads / 32; ++w) mx = fmax(mx, red[w]);
    const int e = mx > 0.0 ? oz_exponent(mx) : 0;
    const double scale = mx > 0.0 ? ldexp(1.0, 47 - e) : 0.0;
    uint8_t* dst = J.dst[g] + size_t(tile) * 128 * kOzK;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = wid * 8 + i;
        uint32_t w[kOzS];
        oz_pack4(v[i], scale, w);
        const uint32_t off = oz_mn32(k, 4 * lane);
#pragma unroll
        for (int d = 0; d < kOzS; ++d) *reinterpret_cast<uint32_t*>(dst + size_t(d) * J.stride + off) = w[d];
    }
    if (threadIdx.x == 0 && J.pe) J.pe[g * ntiles + tile] = e;
    if (g == 0 && threadIdx.x < 128) J.sc[tile * 128 + threadIdx.x] = 1.0;
}

// ---------------------------------------------------------------- tcgen05 / mbarrier primitives
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nOZW:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra OZW;\n}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// K-major, 128-byte swizzle, 1024 B between 8-row atoms, sm_100 descriptor version 1
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}
// kind::i8, D = s32, M = 128, N = kOzNT, K-major A and B; signedness per digit (digit 0 signed)
__host__ __device__ constexpr uint32_t oz_idesc(int asig, int bsig) {
    return (2u << 4) | (uint32_t(asig) << 7) | (uint32_t(bsig) << 10) | (uint32_t(kOzNT >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

constexpr uint32_t kSlice = 128 * kOzK;  // 16 KB: one digit slice of a 128-row panel block
constexpr uint32_t kPair = 2 * kSlice;   // A_d and B_d of one term
constexpr int kBufs = 6;                 // pair buffers: one term (the next term's pairs load as this one's leave)
constexpr int kSlots = 4;                // TMEM accumulator ring: 4 x 128 columns
constexpr int kLevels = 7;               // L = d + d' <= 6: 26 digit-pair products
constexpr int kEpiWarps = 16;            // warpgroups 1-4: 4 per TMEM lane quadrant
constexpr int kCols = 128 * 4 / kEpiWarps;  // output columns per epilogue thread (32)
constexpr int kCtlWarps = 4;              // warpgroup 0: warp 0 producer, warp 1 MMA issuer
constexpr int kThreads = 32 * (kCtlWarps + kEpiWarps);
constexpr int kEpi0 = 32 * kCtlWarps;      // first epilogue thread
// register budget: the register file is split between the 4 SM sub-partitions (16384 each) and 5 warps
// share one, so the launch gets 96 per thread; warpgroup 0 releases to kRegsCtl and the epilogue takes
// kRegsEpi (setmaxnreg; per sub-partition: 1 control + 4 epilogue warps)
constexpr int kRegsLaunch = (65536 / kThreads) / 8 * 8;
constexpr int kRegsCtl = 56;
constexpr int kRegsEpi = ((kRegsLaunch * kThreads - kRegsCtl * 128) / (32 * kEpiWarps)) / 8 * 8;
static_assert(kRegsCtl * 128 + kRegsEpi * 32 * kEpiWarps <= kRegsLaunch * kThreads, "setmaxnreg beyond the CTA pool");
static_assert((kRegsCtl + kRegsEpi * (kEpiWarps / 4)) * 32 <= 16384, "setmaxnreg beyond an SM sub-partition");
constexpr size_t kSmemBufs = size_t(kBufs) * kPair;

__device__ unsigned long long g_oz_trace[8192];  // diagnostics (CCF_OZ_MODE bit 2): block 0 event times
__device__ __forceinline__ unsigned long long oz_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define OZ_TRACE(idx)                                                                     \
    do {                                                                                  \
        if ((mode & 4) && blockIdx.x == 0 && (idx) < 8192) g_oz_trace[(idx)] = oz_now(); \
    } while (0)

// low word of a K-major / MN-major 128-byte-swizzle descriptor (start address >> 4, LBO 16 B); the high
// word (SBO 1024 B, sm_100 version 1, layout 2) is the same for every operand slice
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr) { return ((saddr >> 4) & 0x3FFFu) | (1u << 16); }
constexpr uint32_t kDescHi = (1024u >> 4) | (1u << 14) | (2u << 29);
// MN-major B panels (oz_mn32): SWIZZLE_32B, LBO 4096 B between column quarters, SBO 256 B between 8-row atoms
constexpr uint32_t kDescHiMn = (256u >> 4) | (1u << 14) | (6u << 29);
constexpr uint32_t kLboMn = (4096u >> 4) << 16;
__device__ __forceinline__ uint32_t sdesc_lo_mn(uint32_t saddr) { return ((saddr >> 4) & 0x3FFFu) | kLboMn; }
__device__ __forceinline__ void mma_i8_lo(uint32_t tmem_d, uint32_t alo, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n.reg .b64 ad, bd;\n.reg .pred p;\n"
        "mov.b64 ad, {%1, %6};\nmov.b64 bd, {%2, %3};\nsetp.ne.b32 p, %5, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], ad, bd, %4, p;\n}\n" ::"r"(tmem_d),
        "r"(alo), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc), "n"(kDescHi));
}
// the products of level L: pairs (d, L - d), 4 K-steps each, straight-line (descriptors precomputed per term)
template <int L>
__device__ __forceinline__ void oz_issue_level(uint32_t acc, const uint32_t (&alo)[kOzS], const uint32_t (&blo)[kOzS], int bmn) {
    constexpr int d0 = L > kOzS - 1 ? L - (kOzS - 1) : 0, d1 = L < kOzS - 1 ? L : kOzS - 1;
    const uint32_t bstep = bmn ? 64u : 2u;  // 32 k-rows of 32 B (MN-major, 32B swizzle) or 32 bytes, >> 4
    const uint32_t mnbit = bmn ? (1u << 16) : 0u;
    const uint32_t bhi = bmn ? kDescHiMn : kDescHi;
#pragma unroll
    for (int d = d0; d <= d1; ++d) {
        const uint32_t id = oz_idesc(d == 0, L - d == 0) | mnbit;
#pragma unroll
        for (int k = 0; k < kOzK / 32; ++k)
            mma_i8_lo(acc, alo[d] + 2 * k, blo[L - d] + bstep * k, bhi, id, (d == d0 && k == 0) ? 0u : 1u);
    }
}

// ring position of digit pair d within a term (load / release order 5, 4, 3, 2, 1, 0) and its inverse
__device__ __forceinline__ int oz_pos_of(int d) { return d == 0 ? kOzS - 1 : kOzS - 1 - d; }
__device__ __forceinline__ int oz_digit_at(int i) { return i == kOzS - 1 ? 0 : kOzS - 1 - i; }

struct OzBars {
    uint64_t full[kBufs], empty[kBufs], accfull[kSlots], accempty[kSlots];
    uint64_t sbfull[2], sbempty[2];  // column scales of the tiles in flight (two slots)
    alignas(16) double red[2][16];  // per-warp tile maxima (panel outputs, read as uint4), double-buffered by item parity
    uint32_t tmem_base;
};
constexpr size_t kSbBytes = 128 * sizeof(double);
constexpr size_t kBarsBytes = (sizeof(OzBars) + 127) / 128 * 128;
// item slots (two, bulk-copy targets): the OzItem (80 B) + a has-column-scales flag, then the 128 column scales
constexpr size_t kItemSlot = 128 + kSbBytes;
static_assert(sizeof(OzItem) + sizeof(int) <= 128 && sizeof(OzItem) % 16 == 0, "item slot");


// Persistent: one CTA per SM walks 128 x 128 output tiles (items). Warpgroup 0: warp 0 producer,
// warp 1 MMA issuer (registers released with setmaxnreg); warpgroups 1-4: epilogue (registers raised;
// 4 warps per TMEM lane quadrant, 32 columns each). The six digit-slice pairs (A_d, B_d) of a term
// stream through a ring of seven 32 KB buffers in the order d = 5, 4, 3, 2, 1, 0. The MMA thread issues
// the levels in DESCENDING order (level L = all pairs d + d' = L, 4 K-steps each, M = N = 128) into a
// 4-slot TMEM ring, so pair d is last used at level d: pairs leave the ring in the order they entered
// and the next term's pairs 5..1 load while the current term runs its low levels (level 6 of a term
// needs pairs 1..5, level 5 adds pair 0). The epilogue warps drain each level as it completes: each
// int32 is converted exactly (1.5 2^52 bit trick) and accumulated with the row's weight 2^-(14 + 8L) x
// row scale (two FP64 instructions per element and level); column scales, shared by an item's terms,
// multiply the tile once; then the tile is stored as fp64 (256-bit stores) or, for a product feeding
// another one, as that product's MN-major B panel tile (digits relative to the tile max, CTA-wide).
// N = 128 per instruction keeps the tensor pipe at ~4 POPS (N = 64 costs ~60 cycles per instruction,
// tools/microbench/i8mma.cu).
// D4: the first drain of a term takes levels 6..3 at once (fewer conversions; the MMA cannot run ahead during
// it): faster for single-term items, slower for multi-term ones, so the plan picks it
template <bool D4>
__global__ void __launch_bounds__(kThreads, 1) oz_gemm_kernel(const OzTerm* __restrict__ terms,
                                                              const OzItem* __restrict__ items, int nitems, int mode,
                                                              int bmn) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    // no room for alignment slack (6 x 32 KB + barriers + 2 KB of column scales nearly fill the 227 KB): the
    // dynamic window of a kernel without static shared memory starts 1024-byte aligned
    if (su32(dsm) & 1023) __trap();
    uint8_t* sm = dsm;
    OzBars& bar = *reinterpret_cast<OzBars*>(sm + kSmemBufs);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kBufs; ++i) {
            mbar_init(&bar.full[i], 1);
            mbar_init(&bar.empty[i], 1);
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&bar.accfull[i], 1);
            mbar_init(&bar.accempty[i], kEpiWarps);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar.sbfull[i], 1);
            mbar_init(&bar.sbempty[i], kEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint8_t* islot = sm + kSmemBufs + kBarsBytes;  // item slots [2]
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&bar.tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = bar.tmem_base;

    if (warp < kCtlWarps) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsCtl));
        if (warp == 0) {  // ---------------- producer: per item its header + column scales, then the terms' pairs
            if (lane == 0) {
                uint32_t pc = 0;  // pair counter over all terms (buffer pc % 7, use (pc / 7))
                uint32_t ic = 0;  // item counter (slot ic & 1)
                // the next term's descriptor is loaded one step ahead (dependent global loads)
                int it = blockIdx.x;
                int ct0 = 0, ct1 = 0, cn0 = 0;
                if (it < nitems) {
                    ct0 = items[it].t0;
                    ct1 = items[it].t1;
                    cn0 = items[it].n0;
                }
                OzTerm T = ct1 > ct0 ? terms[ct0] : OzTerm{};
                for (; it < nitems; it += gridDim.x, ++ic) {
                    const int t0 = ct0, t1 = ct1, n0 = cn0;
                    const int itn = it + int(gridDim.x);
                    if (itn < nitems) {
                        ct0 = items[itn].t0;
                        ct1 = items[itn].t1;
                        cn0 = items[itn].n0;
                    }
                    const double* sbp = t1 > t0 ? T.sb : nullptr;  // column scales: the first term's B row scales
                    for (int t = t0; t < t1; ++t) {
                        const OzTerm Tc = T;
                        const int tn = t + 1 < t1 ? t + 1 : (itn < nitems && ct1 > ct0 ? ct0 : -1);
                        if (tn >= 0) T = terms[tn];
                        const uint8_t* bsrc = Tc.b + size_t(n0) * kOzK;
                        for (int i = 0; i < kOzS; ++i, ++pc) {  // digit pairs in release order 5, 4, 3, 2, 1, 0
                            const int d = oz_digit_at(i);
                            const uint32_t b = pc % kBufs, use = pc / kBufs;
                            mbar_wait(&bar.empty[b], (use & 1) ^ 1);
                            OZ_TRACE(pc);
                            mbar_expect(&bar.full[b], kPair);
                            bulk_g2s(sm + size_t(b) * kPair, Tc.a + size_t(d) * kSlice, kSlice, &bar.full[b]);
                            bulk_g2s(sm + size_t(b) * kPair + kSlice, bsrc + size_t(d) * Tc.bstride, kSlice, &bar.full[b]);
                        }
                    }
                    // item slot: the item (read by the epilogue at the end of the tile) and its column scales, after
                    // the item's pairs (the slot of item ic - 2 is released only when that tile is stored)
                    {
                        const uint32_t k = ic & 1;
                        mbar_wait(&bar.sbempty[k], ((ic >> 1) & 1) ^ 1);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // epilogue reads -> next bulk write
                        uint8_t* slot = islot + k * kItemSlot;
                        *reinterpret_cast<int*>(slot + sizeof(OzItem)) = sbp != nullptr;
                        mbar_expect(&bar.sbfull[k], uint32_t(sizeof(OzItem)) + (sbp ? uint32_t(kSbBytes) : 0u));
                        bulk_g2s(slot, items + it, uint32_t(sizeof(OzItem)), &bar.sbfull[k]);
                        if (sbp) bulk_g2s(slot + 128, sbp + n0, uint32_t(kSbBytes), &bar.sbfull[k]);
                        OZ_TRACE(3968 + ic);
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {  // ---------------- MMA issuer
            if (lane == 0) {
                uint32_t pc = 0, g = 0;
                const uint32_t s0 = su32(sm);
                int n0t = 0, n1t = 0;  // the next item's term range (one item ahead)
                if (int(blockIdx.x) < nitems) {
                    n0t = items[blockIdx.x].t0;
                    n1t = items[blockIdx.x].t1;
                }
                for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
                    const int nterm = n1t - n0t;
                    if (it + int(gridDim.x) < nitems) {
                        n0t = items[it + gridDim.x].t0;
                        n1t = items[it + gridDim.x].t1;
                    }
                    for (int t = 0; t < nterm; ++t, pc += kOzS) {
                        // this term's ring buffers: position i (digit pair oz_digit_at(i)) in buffer (pc + i) mod 7
                        const uint32_t p0 = pc % kBufs, u0 = pc / kBufs;
                        uint32_t alo[kOzS], blo[kOzS], fb[kOzS], fph[kOzS];
#pragma unroll
                        for (int i = 0; i < kOzS; ++i) {
                            const uint32_t b = p0 + i >= kBufs ? p0 + i - kBufs : p0 + i;
                            const int d = oz_digit_at(i);
                            alo[d] = sdesc_lo(s0 + b * kPair);
                            blo[d] = bmn ? sdesc_lo_mn(s0 + b * kPair + kSlice) : sdesc_lo(s0 + b * kPair + kSlice);
                            fb[i] = b;
                            fph[i] = (u0 + (p0 + i >= kBufs ? 1 : 0)) & 1;
                        }
                        // levels 6 .. 0 (level 6 needs digit pairs 1..5 = ring positions 0..4, level 5 adds pair 0);
                        // digit pair L is last used at level L: pairs leave the ring in load order
                        auto level = [&](auto Lc) {
                            constexpr int L = decltype(Lc)::value;
                            if (L == kLevels - 1)
                                for (int i = 0; i < kOzS - 1; ++i) mbar_wait(&bar.full[fb[i]], fph[i]);
                            if (L == kLevels - 2) mbar_wait(&bar.full[fb[kOzS - 1]], fph[kOzS - 1]);
                            OZ_TRACE(1024 + g);
                            const uint32_t slot = g % kSlots;
                            mbar_wait(&bar.accempty[slot], ((g / kSlots) & 1) ^ 1);
                            OZ_TRACE(2048 + g);
                            tc_after();
                            if (!(mode & 2)) oz_issue_level<L>(tmem + slot * 128, alo, blo, bmn);
                            if (g < 512) OZ_TRACE(2560 + g);
                            tc_commit(&bar.accfull[slot]);
                            if (L < kOzS) tc_commit(&bar.empty[fb[oz_pos_of(L)]]);
                            ++g;
                        };
                        level(std::integral_constant<int, 6>{});
                        level(std::integral_constant<int, 5>{});
                        level(std::integral_constant<int, 4>{});
                        level(std::integral_constant<int, 3>{});
                        level(std::integral_constant<int, 2>{});
                        level(std::integral_constant<int, 1>{});
                        level(std::integral_constant<int, 0>{});
                    }
                }
            }
            __syncwarp();
        }
    } else {  // ---------------- epilogue: warpgroups 1-4; TMEM lane quadrant warp % 4, 32-column part
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
        // epilogue warp w: TMEM lane quadrant w % 4 (the warp's hardware access rule), column part (w - 4) / 4
        const int q = warp & 3, half = (warp - kCtlWarps) >> 2;  // half: column part 0..3
        const int row = q * 32 + lane;
        const uint32_t tq = tmem + (uint32_t(q * 32) << 16) + uint32_t(half * kCols);
        uint32_t g = 0, ic = 0, ipar = 0;
        // a term's row factor (A row scale x the B plane's tile normalisation), loaded one term ahead
        // The row factor of a term (A row scale x the B plane's tile normalisation) is prefetched in two
        // stages, a term ahead, so no dependent global load stalls the drains: the next term's pointers at
        // the start of a term, their values after its first drain. Item headers are loaded two items ahead.
        auto hdr = [&](int i, int& a, int& b, int& c) {
            if (i < nitems) {
                a = items[i].t0;
                b = items[i].t1;
                c = items[i].n0;
            } else {
                a = b = c = 0;
            }
        };
        int h1t0, h1t1, h1n0, h2t0, h2t1, h2n0;  // the next item's and the one after's headers
        hdr(int(blockIdx.x), h1t0, h1t1, h1n0);
        hdr(int(blockIdx.x + gridDim.x), h2t0, h2t1, h2n0);
        // raw next-term factor: the A row scale and the B plane exponent, combined only when the term starts
        // (the power of two by integer ops), so the loads never stall the drains they overlap
        double fsa = 0.0;
        int fpe = 0;
        if (h1t1 > h1t0) {
            const double* sap = terms[h1t0].sa;
            const int* pep = terms[h1t0].pe;
            fsa = __ldg(sap + row);
            fpe = pep ? __ldg(pep + h1n0 / 128) : 0;
        }
        for (int it = blockIdx.x; it < nitems; it += gridDim.x, ++ic) {
            const int t0 = h1t0, t1 = h1t1, n0 = h1n0;
            h1t0 = h2t0;
            h1t1 = h2t1;
            h1n0 = h2n0;
            hdr(it + 2 * int(gridDim.x), h2t0, h2t1, h2n0);
            const uint32_t k = ic & 1;
            const uint8_t* slot = islot + k * kItemSlot;
            double acc[kCols];
#pragma unroll
            for (int j = 0; j < kCols; ++j) acc[j] = 0.0;
            for (int t = t0; t < t1; ++t) {
                const double sa = fsa * __longlong_as_double((long long)(fpe + 1023) << 52);
                // the next term: t + 1 of this item, else the next item's first (if it has terms)
                const bool inner = t + 1 < t1;
                const int nx = inner ? t + 1 : (h1t1 > h1t0 ? h1t0 : -1);
                const int nxn0 = inner ? n0 : h1n0;
                const double* nsap = nullptr;
                const int* npep = nullptr;
                if (nx >= 0) {  // stage 1: pointers
                    nsap = terms[nx].sa;
                    npep = terms[nx].pe;
                }
                auto drain = [&](int L, int nl) {
                    const uint32_t sl0 = g % kSlots, sl1 = (g + 1) % kSlots, sl2 = (g + 2) % kSlots;
                    mbar_wait(&bar.accfull[sl0], (g / kSlots) & 1);
                    if (nl > 1) {
                        mbar_wait(&bar.accfull[sl1], ((g + 1) / kSlots) & 1);
                        mbar_wait(&bar.accfull[sl2], ((g + 2) / kSlots) & 1);
                    }
                    if (warp == kCtlWarps && lane == 0) OZ_TRACE(3072 + g);  // (diagnostics: CCF_OZ_MODE bit 2)
                    tc_after();
                    if (!(mode & 1)) {
                        const double f = sa * ldexp(1.0, -14 - 8 * L);  // row scale x level weight (powers of 2)
#pragma unroll
                        for (int c = 0; c < kCols / 8; ++c) {
                            uint32_t v0[8], v1[8], v2[8];
                            tmem_ld8(tq + sl0 * 128 + uint32_t(c * 8), v0);  // level L
                            if (nl > 1) {
                                tmem_ld8(tq + sl1 * 128 + uint32_t(c * 8), v1);  // L - 1
                                tmem_ld8(tq + sl2 * 128 + uint32_t(c * 8), v2);  // L - 2
                            }
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const long long y = nl > 1 ? (long long)int(v2[j]) * 65536 + (long long)int(v1[j]) * 256 + int(v0[j])
                                                           : (long long)int(v0[j]);
                                // int64 (|y| < 2^51) -> fp64 exactly: bits(1.5 2^52) + y, minus 1.5 2^52
                                const double x = __hiloint2double(int(uint32_t(y >> 32) + 0x43380000u), int(uint32_t(y))) -
                                                 6755399441055744.0;
                                acc[c * 8 + j] = fma(x, f, acc[c * 8 + j]);
                            }
                        }
                    }
                    tc_before();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&bar.accempty[sl0]);
                        if (nl > 1) {
                            mbar_arrive(&bar.accempty[sl1]);
                            mbar_arrive(&bar.accempty[sl2]);
                        }
                    }
                    g += nl;
                };
                // levels 6, 5, 4, 3 in one drain: y = P3 2^24 + P4 2^16 + P5 2^8 + P6 (|y| < 2^51), 4-column chunks
                auto drain4 = [&](int L) {
                    uint32_t sl[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        sl[u] = (g + u) % kSlots;
                        mbar_wait(&bar.accfull[sl[u]], ((g + u) / kSlots) & 1);
                    }
                    tc_after();
                    if (!(mode & 1)) {
                        const double f = sa * ldexp(1.0, -14 - 8 * L);
#pragma unroll
                        for (int c = 0; c < kCols / 4; ++c) {
                            uint32_t v[4][4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                                             : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3])
                                             : "r"(tq + sl[u] * 128 + uint32_t(c * 4)));
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const long long y = (long long)int(v[3][j]) * 16777216 + (long long)int(v[2][j]) * 65536 +
                                                    (long long)int(v[1][j]) * 256 + int(v[0][j]);
                                const double x = __hiloint2double(int(uint32_t(y >> 32) + 0x43380000u), int(uint32_t(y))) -
                                                 6755399441055744.0;
                                acc[c * 4 + j] = fma(x, f, acc[c * 4 + j]);
                            }
                        }
                    }
                    tc_before();
                    __syncwarp();
                    if (lane == 0)
                        for (int u = 0; u < 4; ++u) mbar_arrive(&bar.accempty[sl[u]]);
                    g += 4;
                };
                if (D4) {
                    drain4(6);
                    if (nx >= 0) {  // stage 2
                        fsa = __ldg(nsap + row);
                        fpe = npep ? __ldg(npep + nxn0 / 128) : 0;
                    }
                    drain(2, 3);
                } else {
                    drain(6, 3);
                    if (nx >= 0) {  // stage 2
                        fsa = __ldg(nsap + row);
                        fpe = npep ? __ldg(npep + nxn0 / 128) : 0;
                    }
                    drain(3, 3);
                    drain(0, 1);
                }
            }
            if (warp == kCtlWarps && lane == 0) OZ_TRACE(3584 + (it - blockIdx.x) / gridDim.x);
            mbar_wait(&bar.sbfull[k], (ic >> 1) & 1);  // the item slot: the item and its column scales
            if (warp == kCtlWarps && lane == 0) OZ_TRACE(4032 + ic);
            const OzItem& I = *reinterpret_cast<const OzItem*>(slot);
            if (t1 > t0 && *reinterpret_cast<const int*>(slot + sizeof(OzItem))) {  // column scales
                const uint32_t sba = su32(slot + 128) + 8u * uint32_t(half * kCols);  // broadcast shared loads
#pragma unroll
                for (int j = 0; j < kCols; j += 2) {
                    double sx, sy;
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(sx), "=d"(sy) : "r"(sba + 8u * j));
                    acc[j] *= sx;
                    acc[j + 1] *= sy;
                }
                if (I.flags & kOzItemAlpha) {
                    const double al = I.alpha;
#pragma unroll
                    for (int j = 0; j < kCols; ++j) acc[j] *= al;
                }
            }
            if (warp == kCtlWarps && lane == 0) OZ_TRACE(3712 + (it - blockIdx.x) / gridDim.x);
            if (I.pdst) {  // the tile as the next product's MN-major B panel tile: digits relative to the tile max
                // tile max exponent from the high words of |acc| (the exponent lives there): integer max, no FP64 ops
                if (!(I.flags & kOzItemFull)) {  // ragged tile: rows >= m and columns >= n become zero digits
                    const int nv = row < I.m ? I.n - half * kCols : 0;
#pragma unroll
                    for (int j = 0; j < kCols; ++j) acc[j] = j < nv ? acc[j] : 0.0;
                }
                uint32_t hx = 0;
#pragma unroll
                for (int j = 0; j < kCols; ++j) hx = max(hx, uint32_t(__double2hiint(acc[j])) & 0x7FFFFFFFu);
#pragma unroll
                for (int o = 16; o; o >>= 1) hx = max(hx, __shfl_xor_sync(0xffffffffu, hx, o));
                if (lane == 0) reinterpret_cast<uint32_t*>(bar.red[ipar])[warp - kCtlWarps] = hx;
                asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");  // the epilogue warps only
                const uint4* rp = reinterpret_cast<const uint4*>(bar.red[ipar]);
#pragma unroll
                for (int w = 0; w < kEpiWarps / 4; ++w) {
                    const uint4 r4 = rp[w];
                    hx = max(max(hx, r4.x), max(r4.y, max(r4.z, r4.w)));
                }
                ipar ^= 1;
                const int e = oz_tile_exponent(hx);
                const double scale = hx ? ldexp(1.0, 47 - e) : 0.0;
                // in place: acc[j] -> the bits of fma(acc[j], 2^(47 - e), 1.5 2^52), whose low 48 bits are the
                // two's-complement fixed-point value X (|X| < 2^47 by the choice of e)
#pragma unroll
                for (int j = 0; j < kCols; ++j) acc[j] = fma(acc[j], scale, 6755399441055744.0);
                // per digit slice: this thread's 32 columns = one 32-byte sector of its 128-byte panel row
                // (chunks 2i, 2i + 1 of the row swizzle land in one aligned sector), one 256-bit store each
                const uint32_t off = oz_mn32(row, half * kCols) & ~31u;  // 32 rows of a quarter: 1 KB per instruction
                const bool swp = ((row >> 2) & 1) != 0;
                if (!(mode & 32)) {
#pragma unroll
                    for (int d = 0; d < kOzS; ++d) {
                        uint32_t wd[8];
#pragma unroll
                        for (int q8 = 0; q8 < 8; ++q8) wd[q8] = oz_digit_word(acc + 4 * q8, d);
                        const uint64_t a0 = uint64_t(wd[0]) | (uint64_t(wd[1]) << 32), a1 = uint64_t(wd[2]) | (uint64_t(wd[3]) << 32);
                        const uint64_t b0 = uint64_t(wd[4]) | (uint64_t(wd[5]) << 32), b1 = uint64_t(wd[6]) | (uint64_t(wd[7]) << 32);
                        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(I.pdst + size_t(d) * I.pstride + off),
                                     "l"(swp ? b0 : a0), "l"(swp ? b1 : a1), "l"(swp ? a0 : b0), "l"(swp ? a1 : b1)
                                     : "memory");
                    }
                }
                if (threadIdx.x == kEpi0 && I.ppe) *I.ppe = e;
            } else if (row < I.m && !(mode & 8) && I.cq) {  // column-quad major: lane = row, 1 KB per instruction
                const long cq = I.cq;
                double* cb = I.c + long(half * (kCols / 4)) * cq + long(row) * 4;
                const int nv = I.n - half * kCols;
#pragma unroll
                for (int j = 0; j < kCols; j += 4) {
                    if (j + 4 <= nv)
                        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(cb + (j / 4) * cq), "d"(acc[j]),
                                     "d"(acc[j + 1]), "d"(acc[j + 2]), "d"(acc[j + 3])
                                     : "memory");
                    else
                        for (int u = 0; u < 4; ++u)
                            if (j + u < nv) cb[(j / 4) * cq + u] = acc[j + u];
                }
            } else if (row < I.m && !(mode & 8)) {
                double* crow = I.c + long(row) * I.ldc + half * kCols;
                const int nv = I.n - half * kCols;
                if (nv >= kCols && ((reinterpret_cast<uintptr_t>(crow) & 31) == 0)) {
#pragma unroll
                    for (int j = 0; j < kCols; j += 4)
                        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(crow + j), "d"(acc[j]), "d"(acc[j + 1]),
                                     "d"(acc[j + 2]), "d"(acc[j + 3])
                                     : "memory");
                } else {
#pragma unroll
                    for (int j = 0; j < kCols; ++j)
                        if (j < nv) crow[j] = acc[j];
                }
            }
            if (warp == kCtlWarps && lane == 0) OZ_TRACE(3840 + (it - blockIdx.x) / gridDim.x);
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar.sbempty[k]);  // item slot read
        }
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}


}  // namespace

void oz_trace_dump() {  // diagnostics (CCF_OZ_MODE bit 2): block 0's event times, ns from the first
    std::vector<unsigned long long> t(8192);
    cudaMemcpyFromSymbol(t.data(), g_oz_trace, 8192 * 8);
    const unsigned long long t0 = t[0];
    for (int i = 0; i < 48; ++i)
        std::printf("level %2d: pair-issue %7lld  mma-start %7lld  mma-go %7lld  issued %7lld  epi-got %7lld\n", i,
                    i < 1024 && t[i] ? (long long)(t[i] - t0) : -1, t[1024 + i] ? (long long)(t[1024 + i] - t0) : -1,
                    t[2048 + i] ? (long long)(t[2048 + i] - t0) : -1, t[2560 + i] ? (long long)(t[2560 + i] - t0) : -1,
                    t[3072 + i] ? (long long)(t[3072 + i] - t0) : -1);
    for (int i = 0; i < 6; ++i)
        std::printf("tile %d: drained %7lld  sb-copied %7lld  sb-got %7lld  scaled %7lld  stored %7lld\n", i,
                    (long long)(t[3584 + i] - t0), (long long)(t[3968 + i] - t0), (long long)(t[4032 + i] - t0),
                    (long long)(t[3712 + i] - t0), (long long)(t[3840 + i] - t0));
    for (int i = 0; i < 8; ++i) {  // per epilogue warp: tile max start / after the epilogue barrier / stores done
        if (!t[4096 + i * 16]) continue;
        for (int k = 0; k < 3; ++k) {
            std::printf("tile %d %s:", i, k == 0 ? "pre-max" : k == 1 ? "bar-out" : "stored ");
            for (int w = 0; w < 16; ++w) {
                const unsigned long long v = t[4096 + 128 * k + i * 16 + w];
                std::printf(" %6lld", v ? (long long)(v - t0) : -1);
            }
            std::printf("\n");
        }
    }
}

size_t oz_smem_bytes() { return kSmemBufs + kBarsBytes + 2 * kItemSlot; }

void OzSplitPlan::upload() {
    maxrows = 0;
    for (const OzSplitJob& j : jobs) {
        if (j.ncols > kOzK || j.nrows > j.rows_pad || j.rows_pad % 8 || j.nsrc < 1 || j.nsrc > kOzGroup ||
            (!transpose && !mn && j.nsrc != 1) || ((transpose || mn) && j.rows_pad % 128))
            throw Error(INTERNAL, "OzSplitPlan: bad job shape");
        maxrows = std::max(maxrows, j.rows_pad);
    }
    if (d) cudaFree(d);
    d = nullptr;
    if (jobs.empty()) return;
    CCF_CUDA(cudaMalloc(&d, jobs.size() * sizeof(OzSplitJob)));
    CCF_H2D(d, jobs.data(), jobs.size() * sizeof(OzSplitJob));
}

void OzSplitPlan::launch(cudaStream_t s) const {
    if (jobs.empty()) return;
    if (mn) {
        const dim3 grid(unsigned(maxrows / 128), unsigned(jobs.size() * kOzGroup));
        oz_split_mn_kernel<<<grid, kMnThreads, 0, s>>>(d);
    } else if (transpose) {
        static bool attr = false;
        if (!attr) {
            CCF_CUDA(cudaFuncSetAttribute(oz_split_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(oz_split_cols_smem())));
            attr = true;
        }
        const dim3 grid(unsigned(maxrows / 128), unsigned(jobs.size()));
        oz_split_cols_kernel<<<grid, kSplitThreads, oz_split_cols_smem(), s>>>(d);
    } else {
        const dim3 grid(unsigned((maxrows + 7) / 8), unsigned(jobs.size()));
        oz_split_rows_kernel<<<grid, 256, 0, s>>>(d);
    }
    CCF_CUDA(cudaGetLastError());
}

OzSplitPlan::~OzSplitPlan() {
    if (d) cudaFree(d);
}

void OzGemmPlan::upload() {
    if (dterms) cudaFree(dterms);
    if (ditems) cudaFree(ditems);
    dterms = nullptr;
    ditems = nullptr;
    flops = 0.0;
    for (OzItem& it : items) {
        it.flags = (it.alpha != 1.0 ? kOzItemAlpha : 0) | (it.m == 128 && it.n == kOzNT ? kOzItemFull : 0);
        if (it.t0 < 0 || it.t1 > int(terms.size()) || it.t0 > it.t1 || it.n0 % kOzNT || it.m > 128 || it.n > kOzNT)
            throw Error(INTERNAL, "OzGemmPlan: bad item");
        flops += 2.0 * it.m * it.n * kOzK * (it.t1 - it.t0);
    }
    single_term = std::all_of(items.begin(), items.end(), [](const OzItem& x) { return x.t1 - x.t0 <= 1; });
    // long items first (persistent round-robin assignment)
    std::stable_sort(items.begin(), items.end(), [](const OzItem& x, const OzItem& y) { return x.t1 - x.t0 > y.t1 - y.t0; });
    if (terms.empty() || items.empty()) return;
    CCF_CUDA(cudaMalloc(&dterms, terms.size() * sizeof(OzTerm)));
    CCF_CUDA(cudaMalloc(&ditems, items.size() * sizeof(OzItem)));
    CCF_H2D(dterms, terms.data(), terms.size() * sizeof(OzTerm));
    CCF_H2D(ditems, items.data(), items.size() * sizeof(OzItem));
}

void OzGemmPlan::launch(cudaStream_t s) const {
    if (items.empty()) return;
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        CCF_CUDA(cudaGetDevice(&dev));
        CCF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        CCF_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(oz_smem_bytes())));
        CCF_CUDA(cudaFuncSetAttribute(oz_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(oz_smem_bytes())));
    }
    const unsigned grid = unsigned(std::min<size_t>(items.size(), size_t(nsm)));
    static const int mode0 = std::getenv("CCF_OZ_MODE") ? std::atoi(std::getenv("CCF_OZ_MODE")) : 0;  // diagnostics
    static const char* trace_tag = std::getenv("CCF_OZ_TRACE");  // trace (mode bit 2) only the plan with this tag
    const int mode = (trace_tag && tag && std::strcmp(trace_tag, tag) != 0) ? (mode0 & ~4) : mode0;
    if (single_term)
        oz_gemm_kernel<true><<<grid, kThreads, oz_smem_bytes(), s>>>(dterms, ditems, int(items.size()), mode, int(b_mn));
    else
        oz_gemm_kernel<false><<<grid, kThreads, oz_smem_bytes(), s>>>(dterms, ditems, int(items.size()), mode, int(b_mn));
    CCF_CUDA(cudaGetLastError());
}

OzGemmPlan::~OzGemmPlan() {
    if (dterms) cudaFree(dterms);
    if (ditems) cudaFree(ditems);
}

}  // namespace ccf

// diagnostics entry point (not part of include/ccf.h): print block 0's trace of the last traced launch
extern "C" void ccf_debug_oz_trace_dump() { ccf::oz_trace_dump(); }

