// Device helpers of the INT8 digit representation (ozaki.hpp), shared by the product kernels (ozaki.cu) and
// the producers that write digit panels directly (the NS step's RHS pass, pipeline.cu).
#pragma once

#include <cstdint>

#include "ozaki.hpp"

namespace ccf {

// byte offset of (row r, reduction byte k) in a 128-byte-swizzled K-major slice
__host__ __device__ __forceinline__ uint32_t oz_swz(int r, int k) {
    return uint32_t(r >> 3) * 1024u + uint32_t(r & 7) * 128u + ((uint32_t((k >> 4) ^ (r & 7)) << 4) | uint32_t(k & 15));
}

// byte offset of (k-row k, column byte n) in an MN-major slice of 128 k-rows x 128 columns, laid out as the
// tcgen05 canonical MN-major SWIZZLE_32B form: four 32-column quarters 4 KB apart (LBO), each 128 rows of 32 bytes
// (8-row atoms of 256 B, SBO), 16-byte halves swapped on row bit 2. A product epilogue writing a tile as the
// next product's B operand then stores one contiguous kilobyte per warp instruction (32 rows of one quarter).
__host__ __device__ __forceinline__ uint32_t oz_mn32(int k, int n) {
    return uint32_t(n >> 5) * 4096u + uint32_t(k) * 32u + ((uint32_t(((n >> 4) & 1) ^ ((k >> 2) & 1))) << 4) + uint32_t(n & 15);
}

// ---------------------------------------------------------------- digits
// s = 2^e with max|row| < s; X = rint(x 2^(47 - e)) in [-2^47, 2^47): 48-bit two's complement,
// digit 0 = signed top byte, digits 1..5 = unsigned lower bytes (ozaki.hpp)
__device__ __forceinline__ int oz_exponent(double maxabs) {
    int e = 0;
    frexp(maxabs, &e);  // maxabs = f 2^e, f in [0.5, 1): maxabs < 2^e
    return e;
}
__device__ __forceinline__ long long oz_fixed(double x, int e) {
    long long X = __double2ll_rn(ldexp(x, 47 - e));
    return X > (1LL << 47) - 1 ? (1LL << 47) - 1 : X;
}
__device__ __forceinline__ uint32_t oz_digit(long long X, int d) {
    return d == 0 ? uint32_t(int(X >> 40)) & 255u : uint32_t(X >> (40 - 8 * d)) & 255u;
}

// The digits of four values as six packed words (word d holds digit d of value u in byte u): scale
// 2^(47 - e) and round with one FMA against 1.5 2^52 (exact: |x 2^(47-e)| < 2^47), so the low 48 bits
// of the double ARE the two's-complement integer X, whose bytes 5..0 are digits 0..5 (digit 0 signed).
// Byte transposes with PRMT: 12 per four values.
__device__ __forceinline__ void oz_pack4(const double (&x)[4], double scale, uint32_t (&w)[kOzS]) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const double y = fma(x[u], scale, 6755399441055744.0);
        lo[u] = uint32_t(__double2loint(y));
        hi[u] = uint32_t(__double2hiint(y)) - 0x43380000u;  // X = bits(y) - bits(1.5 2^52)
        if (hi[u] == 0x8000u) {  // X = 2^47 (a rounded maximum): clamp to 2^47 - 1
            hi[u] = 0x7FFFu;
            lo[u] = 0xFFFFFFFFu;
        }
    }
    const uint32_t a = __byte_perm(lo[0], lo[1], 0x5140), b = __byte_perm(lo[2], lo[3], 0x5140);
    const uint32_t c = __byte_perm(lo[0], lo[1], 0x7362), d = __byte_perm(lo[2], lo[3], 0x7362);
    const uint32_t e = __byte_perm(hi[0], hi[1], 0x5140), f = __byte_perm(hi[2], hi[3], 0x5140);
    w[0] = __byte_perm(e, f, 0x7632);  // byte 5 of X
    w[1] = __byte_perm(e, f, 0x5410);  // byte 4
    w[2] = __byte_perm(c, d, 0x7632);  // byte 3
    w[3] = __byte_perm(c, d, 0x5410);  // byte 2
    w[4] = __byte_perm(a, b, 0x7632);  // byte 1
    w[5] = __byte_perm(a, b, 0x5410);  // byte 0
}

// Clamp-free variant for scales from oz_tile_exponent (|x scale| < 2^47 after rounding by construction)
__device__ __forceinline__ void oz_pack4_nc(const double (&x)[4], double scale, uint32_t (&w)[kOzS]) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const double y = fma(x[u], scale, 6755399441055744.0);
        lo[u] = uint32_t(__double2loint(y));
        hi[u] = uint32_t(__double2hiint(y));  // bytes 0-1 = X bytes 4-5 (the magic's low half word is 0)
    }
    const uint32_t a = __byte_perm(lo[0], lo[1], 0x5140), b = __byte_perm(lo[2], lo[3], 0x5140);
    const uint32_t c = __byte_perm(lo[0], lo[1], 0x7362), d = __byte_perm(lo[2], lo[3], 0x7362);
    const uint32_t e = __byte_perm(hi[0], hi[1], 0x5140), f = __byte_perm(hi[2], hi[3], 0x5140);
    w[0] = __byte_perm(e, f, 0x7632);
    w[1] = __byte_perm(e, f, 0x5410);
    w[2] = __byte_perm(c, d, 0x7632);
    w[3] = __byte_perm(c, d, 0x5410);
    w[4] = __byte_perm(a, b, 0x7632);
    w[5] = __byte_perm(a, b, 0x5410);
}

// Exponent of a set whose largest |value| has the high word hx: e with max < (hx + 1, 0) <= 2^e, so that
// max 2^(47 - e) rounds below 2^47 (the usual e of the max; one more only when the high-word mantissa is all ones)
__device__ __forceinline__ int oz_tile_exponent(uint32_t hx) { return hx ? oz_exponent(__hiloint2double(int(hx + 1), 0)) : 0; }

// One 128-value panel row held by a warp (four values per lane, lane l = reduction bytes 4l .. 4l + 3): digits
// relative to the row max into the six slices (row r, stride bytes apart), the row scale 2^e (0 for a zero row)
__device__ __forceinline__ void oz_warp_row(const double (&v)[4], uint8_t* dst, long stride, int r, double* sc) {
    const int lane = threadIdx.x & 31;
    uint32_t hx = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) hx = max(hx, uint32_t(__double2hiint(v[u])) & 0x7FFFFFFFu);
#pragma unroll
    for (int o = 16; o; o >>= 1) hx = max(hx, __shfl_xor_sync(0xffffffffu, hx, o));
    const int e = oz_tile_exponent(hx);
    uint32_t w[kOzS];
    oz_pack4_nc(v, hx ? ldexp(1.0, 47 - e) : 0.0, w);
    const uint32_t off = oz_swz(r, 4 * lane);
#pragma unroll
    for (int d = 0; d < kOzS; ++d) *reinterpret_cast<uint32_t*>(dst + size_t(d) * stride + off) = w[d];
    if (lane == 0) *sc = hx ? ldexp(1.0, e) : 0.0;
}

}  // namespace ccf
