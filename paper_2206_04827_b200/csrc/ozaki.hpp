// FP64 products on the INT8 tensor cores (tcgen05.mma kind::i8, TMEM accumulators): Ozaki splitting.
//
// B200 has no FP64 tcgen05 kind; its FP64 DMMA path peaks at ~37 TFLOP/s, while the INT8 tcgen05
// path runs at ~4.2 POPS (tools/microbench/i8mma.cu). Every dense product of the NS step is an FP64
// GEMM with K = 128 (one parity half of a Chebyshev / eigen index), so each operand row is split
// into S = 6 two's-complement 8-bit digits relative to a power-of-two row scale:
//
//   x = s * 2^-7 * (c0 + sum_{d=1..5} c_d 2^-8d),  c0 signed int8, c_d unsigned uint8,  s = 2^e > max|row|
//
// (48 significant bits, rounding error 2^-48 s). A product row . column is then
//   sum_L 2^-(14 + 8L) P_L,  P_L = sum_{d + d' = L} (A_d B_d'^T)   (L = 0..6, 26 int8 GEMMs, int32-exact)
// streamed level by level through a ring of TMEM accumulators and combined in FP64 by the epilogue. The dropped
// levels L >= 7 and the 2^-49 rounding of the digits bound the error by a few 1e-15 of
// (row scale) x (column scale) x K, i.e. FP64-GEMM-like accuracy (tools/cpp/oz_check.cpp).
//
// Operands live in "panels": a matrix of R rows x K = 128 columns stored as S slices, each slice the
// 128-byte-swizzled K-major shared-memory image of the rows (row r at (r/8)*1024 + (r%8)*128, 16-byte
// chunk c at position c ^ (r%8)), so the GEMM moves every slice with one bulk copy; plus one double
// scale per row. A term of a product is (A panel, 128 rows) x (B panel rows = output columns).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace ccf {

constexpr int kOzS = 6;            // digits per operand
constexpr int kOzK = 128;          // reduction length of one panel (bytes per panel row)
constexpr int kOzNT = 128;         // output columns per tile (one 128-column TMEM accumulator slot)

inline size_t oz_slice_bytes(int rows) { return size_t(rows) * kOzK; }
inline size_t oz_panel_bytes(int rows) { return size_t(kOzS) * oz_slice_bytes(rows); }

struct OzTerm {
    const uint8_t* a;   // A panel (128 rows)
    const uint8_t* b;   // B panel (rb rows, the output columns)
    const double* sa;   // 128 row scales of A
    const double* sb;   // rb row scales of B, or null (MN-major / tile-scaled B panels: unit column scales)
    long bstride;       // bytes per B slice (rb * 128)
    const int* pe;      // B plane exponent per 128-row tile of the B panel (transposed splits)
};

constexpr int kOzItemAlpha = 1;  // alpha != 1
constexpr int kOzItemFull = 2;   // m = 128 and n = kOzNT (no row / column guards in the epilogue)
struct alignas(16) OzItem {  // one 128 x 128 output tile; every term of an item has the same B (column) scales
    int t0, t1;         // terms [t0, t1)
    int n0;             // first B-panel row (output column) of the tile
    int m, n;           // valid rows / columns of the tile
    int flags;          // (set by OzGemmPlan::upload: kOzItemAlpha, kOzItemFull)
    double* c;          // tile origin in the output (row-major, ldc)
    long ldc;
    double alpha;       // (ignored when the terms carry no column scales: alpha = 1)
    // optional: write the tile (rows = K of the next product, columns = its output columns) as that
    // product's MN-major B panel tile instead of fp64: slice d at pdst + d * pstride, tile exponent -> *ppe.
    // MN-major slices use the canonical SWIZZLE_32B form (ozaki_dev.cuh oz_mn32): column quarters 4 KB apart,
    // so a warp of the epilogue (32 rows of one quarter) stores 1 KB contiguous per instruction
    uint8_t* pdst = nullptr;
    long pstride = 0;
    int* ppe = nullptr;
    // optional fp64 column-quad-major output: element (row, col) at c + (col / 4) * cq + row * 4 + col % 4
    // (cq = 4 x rows of the tensor): a warp's store instruction then covers 1 KB contiguous
    long cq = 0;
};

// Split jobs: fp64 source -> panel slices + row scales.
//  rows: source rows are panel rows (row r at src + r * ld, K contiguous values), the A-side layout
//  cols: source columns are panel rows (value (k, r) at src + k * ld + r), transposed into K-major
//  A transpose job splits up to kOzGroup sources ("planes") with ONE scale per panel row: per 128-row
//  tile every plane is first normalised by a power of two 2^e_p (its max over the tile, written to
//  pe[p * tiles + tile]), then the panel row scale is the common max of the normalised planes. The B
//  operands of one output tile's terms share the row scales (OzItem); each term carries its plane's
//  2^e_p as a factor of its A row scale, so a small plane keeps its own precision.
constexpr int kOzGroup = 10;
struct OzSplitJob {
    const double* src[kOzGroup];
    uint8_t* dst[kOzGroup];  // panel bases
    int nsrc;
    long ld;
    int nrows, ncols;   // valid panel rows / reduction length (<= 128; the rest is zero)
    double* sc;         // row scales
    long stride;        // bytes per slice (panel rows * 128)
    int rows_pad;       // panel rows written (>= nrows, multiple of 8; transposed: multiple of 128)
    int* pe;            // transposed: plane exponents [nsrc][rows_pad / 128]
};
inline OzSplitJob oz_job(const double* src, long ld, int nrows, int ncols, uint8_t* dst, double* sc, long stride,
                         int rows_pad, int* pe = nullptr) {
    OzSplitJob j{};
    j.pe = pe;
    j.src[0] = src;
    j.dst[0] = dst;
    j.nsrc = 1;
    j.ld = ld;
    j.nrows = nrows;
    j.ncols = ncols;
    j.sc = sc;
    j.stride = stride;
    j.rows_pad = rows_pad;
    return j;
}

struct OzSplitPlan {
    std::vector<OzSplitJob> jobs;
    bool transpose = false;
    bool mn = false;          // B data in the MN-major panel layout (src rows = K, columns = panel rows): one
                              // scale per (plane, 128-column tile), row scales 1; read with OzGemmPlan::b_mn
    OzSplitJob* d = nullptr;
    int maxrows = 0;
    void upload();
    void launch(cudaStream_t s) const;
    ~OzSplitPlan();
};

struct OzGemmPlan {
    std::vector<OzTerm> terms;
    std::vector<OzItem> items;
    OzTerm* dterms = nullptr;
    OzItem* ditems = nullptr;
    double flops = 0.0;  // FP64-equivalent 2 M N K per term and tile
    bool b_mn = false;   // B panels in the MN-major layout (OzSplitPlan::mn)
    bool single_term = false;  // (set by upload: every item has at most one term -> the 4-level first drain)
    const char* tag = nullptr;  // diagnostics label (CCF_OZ_TRACE)
    void upload();
    void launch(cudaStream_t s) const;
    ~OzGemmPlan();
};

size_t oz_smem_bytes();
void oz_trace_dump();

}  // namespace ccf
