// CCF1 FieldFile I/O (reference proj/src/io.cpp:12-109, proj/include/cylspec/io.hpp:11-28):
//   "CCF1" | version u32 | kind u8 (0 real grid values, 1 complex coefficients) | m, n, p u32 |
//   payload f64 LE in (l, k, j) order (complex interleaved) | CRC-32/IEEE of the payload bytes u32
//
// Device payloads (snapshots of the device-resident NS state, fields produced on the GPU) are
// checksummed on the GPU: the payload is read once from HBM and only the file bytes cross PCIe.
// CRC-32 is affine over GF(2): with the raw register update R (init 0, no final xor),
//   raw(A || B) = raw(A) * x^(8|B|)  xor  raw(B)        (mod P, reflected)
//   crc(M)      = raw(M) xor (0xFFFFFFFF * x^(8|M|)) xor 0xFFFFFFFF
// and leading zero bytes leave raw() unchanged. The stream is therefore front-padded with zeros to
// a whole number of uniform chunks; each thread folds one 64-byte chunk with slicing-by-8 tables
// in shared memory, and chunk CRCs are merged pairwise up a tree whose shift at every level is one
// constant x^(8 * chunk * 2^level) — fully parallel, two passes over HBM-resident data at most.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "context.hpp"

namespace ccf {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;  // reflected CRC-32/IEEE polynomial
constexpr int kChunk = 64;               // bytes per thread
constexpr int kThreads = 256;            // chunks merged per block per level

__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {  // a * b mod P (reflected)
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

uint32_t x8n(unsigned long long n) {  // x^(8 n) mod P
    uint32_t r = 1u << 31, sq = 1u << 23;  // x^0, x^8
    while (n) {
        if (n & 1) r = multmodp(sq, r);
        sq = multmodp(sq, sq);
        n >>= 1;
    }
    return r;
}

struct Tables {
    uint32_t t[8][256];
};

const Tables& host_tables() {
    static const Tables T = [] {
        Tables x{};
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int b = 0; b < 8; ++b) c = (c & 1) ? kPoly ^ (c >> 1) : c >> 1;
            x.t[0][i] = c;
        }
        for (int k = 1; k < 8; ++k)
            for (int i = 0; i < 256; ++i) x.t[k][i] = (x.t[k - 1][i] >> 8) ^ x.t[0][x.t[k - 1][i] & 0xFF];
        return x;
    }();
    return T;
}

// merge kThreads consecutive raw CRCs (uniform segment length) held in s[] -> s[0]
__device__ inline void tree_merge(uint32_t* s, const uint32_t* shift) {
    for (int lv = 0, w = 1; w < kThreads; ++lv, w <<= 1) {
        __syncthreads();
        const int t = threadIdx.x;
        if ((t & (2 * w - 1)) == 0) s[t] = multmodp(shift[lv], s[t]) ^ s[t + w];
    }
    __syncthreads();
}

// level 0: thread g folds padded bytes [64 g, 64 g + 64) (padded byte i = payload byte i - pad, zero before)
__global__ void __launch_bounds__(kThreads) crc_chunks_kernel(const unsigned long long* __restrict__ words, long nwords,
                                                              long padw, const Tables* __restrict__ tab,
                                                              const uint32_t* __restrict__ shift,
                                                              uint32_t* __restrict__ out) {
    __shared__ uint32_t T[8][256];
    __shared__ uint32_t s[kThreads];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&T[0][0])[i] = (&tab->t[0][0])[i];
    __syncthreads();
    const long g = long(blockIdx.x) * kThreads + threadIdx.x;
    uint32_t crc = 0;
#pragma unroll
    for (int u = 0; u < kChunk / 8; ++u) {
        const long w = g * (kChunk / 8) + u - padw;
        const unsigned long long v = (w >= 0 && w < nwords) ? __ldg(words + w) ^ crc : (unsigned long long)crc;
        crc = T[7][v & 0xFF] ^ T[6][(v >> 8) & 0xFF] ^ T[5][(v >> 16) & 0xFF] ^ T[4][(v >> 24) & 0xFF] ^
              T[3][(v >> 32) & 0xFF] ^ T[2][(v >> 40) & 0xFF] ^ T[1][(v >> 48) & 0xFF] ^ T[0][v >> 56];
    }
    s[threadIdx.x] = crc;
    tree_merge(s, shift);
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

// higher levels: merge kThreads segment CRCs per block (front-padded with zero CRCs)
__global__ void __launch_bounds__(kThreads) crc_merge_kernel(const uint32_t* __restrict__ in, long n, long pad,
                                                             const uint32_t* __restrict__ shift,
                                                             uint32_t* __restrict__ out) {
    __shared__ uint32_t s[kThreads];
    const long i = long(blockIdx.x) * kThreads + threadIdx.x - pad;
    s[threadIdx.x] = (i >= 0 && i < n) ? in[i] : 0u;
    tree_merge(s, shift);
    if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

}  // namespace

uint32_t crc32_host(const uint8_t* data, size_t len) {  // proj/src/io.cpp:12-25 (slicing-by-8 on the host)
    const Tables& T = host_tables();
    uint32_t crc = 0xFFFFFFFFu;
    size_t i = 0;
    for (; i + 8 <= len; i += 8) {
        unsigned long long v;
        std::memcpy(&v, data + i, 8);
        v ^= crc;
        crc = T.t[7][v & 0xFF] ^ T.t[6][(v >> 8) & 0xFF] ^ T.t[5][(v >> 16) & 0xFF] ^ T.t[4][(v >> 24) & 0xFF] ^
              T.t[3][(v >> 32) & 0xFF] ^ T.t[2][(v >> 40) & 0xFF] ^ T.t[1][(v >> 48) & 0xFF] ^ T.t[0][v >> 56];
    }
    for (; i < len; ++i) crc = T.t[0][(crc ^ data[i]) & 0xFF] ^ (crc >> 8);
    return crc ^ 0xFFFFFFFFu;
}

// CRC-32/IEEE of nbytes (multiple of 8, 8-byte aligned) of device memory, on stream
uint32_t crc32_device(const void* dptr, size_t nbytes, cudaStream_t stream) {
    if (nbytes == 0) return 0;
    if (nbytes % 8 || reinterpret_cast<uintptr_t>(dptr) % 8)
        throw Error(DOMAIN_ERROR, "crc32_device: payload must be whole, aligned doubles");
    const Tables* dtab = nullptr;
    const long nwords = long(nbytes / 8);
    const long chunks = (long(nbytes) + kChunk - 1) / kChunk;
    const long blocks0 = (chunks + kThreads - 1) / kThreads;
    const long padw = blocks0 * kThreads * (kChunk / 8) - nwords;
    // passes: level 0 (chunks -> blocks0), then merges by kThreads until one value remains
    std::vector<long> counts{blocks0};
    while (counts.back() > 1) counts.push_back((counts.back() + kThreads - 1) / kThreads);
    const int npass = int(counts.size());
    std::vector<uint32_t> hshift(size_t(npass) * 8);
    unsigned long long seg = kChunk;  // bytes per leaf of the pass
    for (int ps = 0; ps < npass; ++ps) {
        for (int lv = 0; lv < 8; ++lv) hshift[size_t(ps) * 8 + lv] = x8n(seg << lv);
        seg *= kThreads;
    }
    {  // slicing-by-8 tables, once per device
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        int dev = 0;
        CCF_CUDA(cudaGetDevice(&dev));
        static Tables* per_dev[64] = {};
        if (dev < 0 || dev >= 64) throw Error(INTERNAL, "crc32_device: device index");
        if (!per_dev[dev]) {
            CCF_CUDA(cudaMalloc(&per_dev[dev], sizeof(Tables)));
            CCF_H2D(per_dev[dev], &host_tables(), sizeof(Tables));
        }
        dtab = per_dev[dev];
    }
    long total = 0;
    for (long c : counts) total += c;
    uint32_t* buf = nullptr;  // per-call scratch: the passes' outputs, then the shift constants
    CCF_CUDA(cudaMallocAsync(&buf, sizeof(uint32_t) * size_t(total + 1 + npass * 8), stream));
    uint32_t* dshift = buf + total + 1;
    CCF_CUDA(cudaMemcpyAsync(dshift, hshift.data(), sizeof(uint32_t) * hshift.size(), cudaMemcpyHostToDevice, stream));
    uint32_t* cur = buf;
    crc_chunks_kernel<<<unsigned(blocks0), kThreads, 0, stream>>>(
        static_cast<const unsigned long long*>(dptr), nwords, padw, dtab, dshift, cur);
    for (int ps = 1; ps < npass; ++ps) {
        uint32_t* nxt = cur + counts[size_t(ps) - 1];
        const long pad = counts[size_t(ps)] * kThreads - counts[size_t(ps) - 1];
        crc_merge_kernel<<<unsigned(counts[size_t(ps)]), kThreads, 0, stream>>>(cur, counts[size_t(ps) - 1], pad,
                                                                                dshift + ps * 8, nxt);
        cur = nxt;
    }
    uint32_t raw = 0;
    CCF_CUDA(cudaMemcpyAsync(&raw, cur, sizeof(uint32_t), cudaMemcpyDeviceToHost, stream));
    CCF_CUDA(cudaFreeAsync(buf, stream));
    CCF_CUDA(cudaStreamSynchronize(stream));
    return raw ^ multmodp(x8n(nbytes), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
}

// ---- FieldFile (io.cpp:42-109)

namespace {
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(uint8_t(v >> (8 * i)));
}
uint32_t get_u32(const uint8_t* p) { return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24; }
}  // namespace

void write_field_file(const std::string& path, int kind, int m, int n, int p, const double* payload, bool device,
                      cudaStream_t stream) {
    if (kind != 0 && kind != 1) throw Error(FIELDFILE_ERR, "FieldFile: unknown kind");
    const size_t count = size_t(m) * n * p * (kind == 1 ? 2 : 1);
    const size_t nbytes = count * 8;
    std::vector<uint8_t> head;
    head.insert(head.end(), {'C', 'C', 'F', '1'});
    put_u32(head, 1);  // kFieldFileVersion
    head.push_back(uint8_t(kind));
    put_u32(head, uint32_t(m));
    put_u32(head, uint32_t(n));
    put_u32(head, uint32_t(p));
    uint32_t crc;
    const uint8_t* bytes = reinterpret_cast<const uint8_t*>(payload);
    std::vector<uint8_t> staged;
    if (device) {
        crc = crc32_device(payload, nbytes, stream);
        staged.resize(nbytes);
        CCF_CUDA(cudaMemcpyAsync(staged.data(), payload, nbytes, cudaMemcpyDeviceToHost, stream));
        CCF_CUDA(cudaStreamSynchronize(stream));
        bytes = staged.data();
    } else {
        crc = crc32_host(bytes, nbytes);
    }
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw Error(FIELDFILE_ERR, "FieldFile: cannot open for writing: " + path);
    std::vector<uint8_t> tail;
    put_u32(tail, crc);
    const bool ok = std::fwrite(head.data(), 1, head.size(), f) == head.size() &&
                    (nbytes == 0 || std::fwrite(bytes, 1, nbytes, f) == nbytes) &&
                    std::fwrite(tail.data(), 1, 4, f) == 4;
    const bool closed = std::fclose(f) == 0;
    if (!ok || !closed) throw Error(FIELDFILE_ERR, "FieldFile: write failed: " + path);
}

void read_field_header(const std::string& path, int& kind, int& m, int& n, int& p) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Error(FIELDFILE_ERR, "FieldFile: cannot open: " + path);
    uint8_t h[21];
    const size_t got = std::fread(h, 1, 21, f);
    std::fclose(f);
    if (got < 4 || std::memcmp(h, "CCF1", 4) != 0) throw Error(FIELDFILE_ERR, "FieldFile: bad magic");
    if (got < 21) throw Error(FIELDFILE_ERR, "FieldFile: truncated header");
    const uint32_t version = get_u32(h + 4);
    if (version != 1) throw Error(FIELDFILE_ERR, "FieldFile: unsupported version " + std::to_string(version));
    kind = h[8];
    if (kind != 0 && kind != 1) throw Error(FIELDFILE_ERR, "FieldFile: unknown kind");
    m = int(get_u32(h + 9));
    n = int(get_u32(h + 13));
    p = int(get_u32(h + 17));
    // GridSpec::validate (proj/src/grid.cpp:8-14)
    if (m < 4 || n < 4) throw Error(DOMAIN_ERROR, "GridSpec: m and n must be at least 4");
    if (p < 2 || p % 2 != 0) throw Error(DOMAIN_ERROR, "GridSpec: p must be even and at least 2");
}

// payload into out (host or device, count doubles); verifies the CRC (on the GPU for device output)
void read_field_file(const std::string& path, int& kind, int& m, int& n, int& p, double* out, size_t cap, bool device,
                     cudaStream_t stream) {
    read_field_header(path, kind, m, n, p);
    const size_t count = size_t(m) * n * p * (kind == 1 ? 2 : 1);
    if (count > cap) throw Error(DOMAIN_ERROR, "FieldFile: output buffer too small");
    const size_t nbytes = count * 8;
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw Error(FIELDFILE_ERR, "FieldFile: cannot open: " + path);
    std::fseek(f, 21, SEEK_SET);
    std::vector<uint8_t> buf(nbytes + 4);
    const size_t got = std::fread(buf.data(), 1, nbytes + 4, f);
    std::fclose(f);
    if (got < nbytes) throw Error(FIELDFILE_ERR, "FieldFile: truncated payload");
    if (got < nbytes + 4) throw Error(FIELDFILE_ERR, "FieldFile: truncated header");  // io.cpp get_u32 message
    const uint32_t crc = get_u32(buf.data() + nbytes);
    uint32_t actual;
    if (device) {
        CCF_CUDA(cudaMemcpyAsync(out, buf.data(), nbytes, cudaMemcpyHostToDevice, stream));
        actual = crc32_device(out, nbytes, stream);  // synchronises the stream (the copy is complete)
    } else {
        std::memcpy(out, buf.data(), nbytes);
        actual = crc32_host(buf.data(), nbytes);
    }
    if (crc != actual) throw Error(FIELDFILE_ERR, "FieldFile: CRC mismatch");
}

}  // namespace ccf
