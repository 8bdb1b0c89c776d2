// .hgi payload of a generated hologram on the device (
// reference writer: cghkit/serialio.py:167-185 save_field). The payload is
// the row-major complex128 field, little-endian (re, im) float64 pairs, and
// the header carries zlib's CRC-32 of those bytes.
//
// A hologram takes only state values, so the payload is expanded from the
// index plane on the device (16 B/px written once, then one D2H copy), and
// the CRC is computed from the index plane without reading the payload back:
// the raw (unconditioned) CRC register is linear over GF(2), so appending a
// 16-byte record r to a stream with register c gives S16(c) ^ K[r], where
// S16 is "advance by 16 zero bytes" (a fixed 32x32 bit matrix, applied with
// four 256-entry byte tables) and K[r] is the raw CRC of the record alone.
// Chunks of records are folded the same way with S_{chunk bytes}. Leading
// zero bytes do not change a raw CRC, so the plane is front-padded to whole
// chunks. zlib's conditioning is applied on the host:
//   crc32(data) = raw(data) ^ S_len(0xFFFFFFFF) ^ 0xFFFFFFFF.
#include <algorithm>
#include <array>

#include "runtime.cuh"

namespace cgh {

constexpr uint32_t kCrcPoly = 0xEDB88320u;   // reflected CRC-32 (zlib)
constexpr int kCrcChunk = 256;               // records per thread chunk
constexpr int kCrcBlock = 256;               // chunks per block fold

using Mat32 = std::array<uint32_t, 32>;      // column j = image of bit j

static uint32_t mat_apply(const Mat32& m, uint32_t v) {
    uint32_t r = 0;
    for (int j = 0; j < 32; ++j)
        if (v >> j & 1u) r ^= m[j];
    return r;
}

static Mat32 mat_mul(const Mat32& a, const Mat32& b) {   // a o b
    Mat32 r;
    for (int j = 0; j < 32; ++j) r[j] = mat_apply(a, b[j]);
    return r;
}

// advance the raw register by one zero byte
static uint32_t zero_byte(uint32_t c) {
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ kCrcPoly : c >> 1;
    return c;
}

// S_n: advance by n zero bytes (square-and-multiply on the 32x32 matrix)
static Mat32 shift_matrix(uint64_t n) {
    Mat32 one, res;
    for (int j = 0; j < 32; ++j) {
        one[j] = zero_byte(1u << j);
        res[j] = 1u << j;
    }
    while (n) {
        if (n & 1) res = mat_mul(one, res);
        one = mat_mul(one, one);
        n >>= 1;
    }
    return res;
}

// four byte tables: S(c) = T[0][c & 255] ^ T[1][c >> 8 & 255] ^ T[2][..] ^ T[3][c >> 24]
static void byte_tables(const Mat32& m, uint32_t* t /* 4 x 256 */) {
    for (int k = 0; k < 4; ++k)
        for (int b = 0; b < 256; ++b) t[k * 256 + b] = mat_apply(m, uint32_t(b) << (8 * k));
}

// raw CRC of bytes (register starting at 0)
static uint32_t raw_crc(const unsigned char* p, size_t n, uint32_t c = 0) {
    for (size_t i = 0; i < n; ++i) {
        c ^= p[i];
        for (int k = 0; k < 8; ++k) c = (c & 1u) ? (c >> 1) ^ kCrcPoly : c >> 1;
    }
    return c;
}

__device__ __forceinline__ uint32_t tab_apply(const uint32_t* t, uint32_t c) {
    return t[c & 255u] ^ t[256 + (c >> 8 & 255u)] ^ t[512 + (c >> 16 & 255u)] ^ t[768 + (c >> 24)];
}

// payload[p] = states[idx[p]] (complex128 as two doubles). An index outside
// the table (the reference's states[indices] raises IndexError) sets *bad and
// is not read.
__global__ void hgi_expand_kernel(const void* __restrict__ idx, int idx_bytes, long long n,
                                  const double2* __restrict__ states, int n_states, double2* __restrict__ out,
                                  unsigned* __restrict__ bad) {
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const int k = idx_bytes == 1 ? int(static_cast<const uint8_t*>(idx)[p]) : static_cast<const int32_t*>(idx)[p];
        if (k < 0 || k >= n_states) {
            *bad = 1u;
            continue;
        }
        out[p] = states[k];
    }
}

// Raw CRC per chunk of kCrcChunk records, folded per block of kCrcBlock
// chunks (fixed order). Record q of the front-padded stream is pixel q - pad
// (a zero record for q < pad). k_rec: raw CRC of each state's 16 bytes.
__global__ void __launch_bounds__(kCrcBlock) hgi_crc_kernel(const void* __restrict__ idx, int idx_bytes, long long n,
                                                            long long pad, const uint32_t* __restrict__ k_rec,
                                                            int n_states, const uint32_t* __restrict__ s16_g,
                                                            const uint32_t* __restrict__ sch_g,
                                                            uint32_t* __restrict__ block_crc,
                                                            unsigned* __restrict__ bad) {
    __shared__ uint32_t s16[1024], sch[1024], part[kCrcBlock];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        s16[i] = s16_g[i];
        sch[i] = sch_g[i];
    }
    __syncthreads();
    const long long q0 = ((long long)blockIdx.x * kCrcBlock + threadIdx.x) * kCrcChunk;
    uint32_t c = 0;
    for (int r = 0; r < kCrcChunk; ++r) {
        const long long p = q0 + r - pad;
        uint32_t kr = 0;
        if (p >= 0 && p < n) {
            const int k = idx_bytes == 1 ? int(static_cast<const uint8_t*>(idx)[p]) : static_cast<const int32_t*>(idx)[p];
            if (k >= 0 && k < n_states) kr = k_rec[k];
            else *bad = 1u;
        }
        c = tab_apply(s16, c) ^ kr;
    }
    part[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t b = 0;
        for (int j = 0; j < kCrcBlock; ++j) b = tab_apply(sch, b) ^ part[j];
        block_crc[blockIdx.x] = b;
    }
}

}  // namespace cgh

using namespace cgh;

extern "C" {

int cgh_crc32_combine(uint32_t crc1, uint32_t crc2, int64_t len2, uint32_t* out) {
    // zlib crc32_combine: with crc(X) = raw(X) ^ S_|X|(F) ^ F (F = 0xFFFFFFFF)
    // and raw(A||B) = S_|B|(raw(A)) ^ raw(B), the conditioning terms cancel:
    // crc(A||B) = S_|B|(crc(A)) ^ crc(B).
    if (!out || len2 < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    const Mat32 s = shift_matrix(uint64_t(len2));
    *out = mat_apply(s, crc1) ^ crc2;
    return CGH_OK;
}

int cgh_hgi_payload(int32_t device, const void* idx, int32_t idx_bytes, int64_t count, const double* states,
                    int32_t n_states, double* out_payload, uint32_t* out_crc) {
    if (!idx || !states || count < 0 || n_states < 1 || (idx_bytes != 1 && idx_bytes != 4) || !out_crc)
        return fail(CGH_ERR_VALUE, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    if (device < 0 || device >= ndev) return fail(CGH_ERR_VALUE, "device %d out of range", device);
    CGH_CUDA(cudaSetDevice(device));
    // host tables: K (raw CRC of each state's record), S16, S_chunk, S_block
    std::vector<uint32_t> k(static_cast<size_t>(n_states) + 0);
    for (int i = 0; i < n_states; ++i) k[i] = raw_crc(reinterpret_cast<const unsigned char*>(states + 2 * i), 16);
    std::vector<uint32_t> tabs(3 * 1024);
    byte_tables(shift_matrix(16), tabs.data());
    byte_tables(shift_matrix(uint64_t(16) * kCrcChunk), tabs.data() + 1024);
    const long long per_block = (long long)kCrcChunk * kCrcBlock;
    const long long nblocks = std::max<long long>(1, (count + per_block - 1) / per_block);
    const long long pad = nblocks * per_block - count;
    cudaStream_t st;
    CGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void *d_idx = nullptr, *d_states = nullptr, *d_k = nullptr, *d_tabs = nullptr, *d_blk = nullptr, *d_pay = nullptr;
    auto cleanup = [&]() {
        void* ps[] = {d_idx, d_states, d_k, d_tabs, d_blk, d_pay};
        for (void* p : ps)
            if (p) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    };
#define HGI_CUDA(call)                                                                                    \
    do {                                                                                                  \
        cudaError_t e_ = (call);                                                                          \
        if (e_ != cudaSuccess) {                                                                          \
            cleanup();                                                                                    \
            return fail(e_ == cudaErrorMemoryAllocation ? CGH_ERR_MEMORY : CGH_ERR_CUDA, "%s: %s", #call, \
                        cudaGetErrorString(e_));                                                          \
        }                                                                                                 \
    } while (0)
    const size_t ib = size_t(count) * idx_bytes;
    HGI_CUDA(cudaMallocAsync(&d_idx, std::max<size_t>(ib, 16), st));
    HGI_CUDA(cudaMallocAsync(&d_states, size_t(n_states) * 16, st));
    HGI_CUDA(cudaMallocAsync(&d_k, size_t(n_states) * 4, st));
    HGI_CUDA(cudaMallocAsync(&d_tabs, tabs.size() * 4, st));
    HGI_CUDA(cudaMallocAsync(&d_blk, size_t(nblocks) * 4 + 16, st));
    unsigned* d_bad = reinterpret_cast<unsigned*>(static_cast<char*>(d_blk) + size_t(nblocks) * 4);
    HGI_CUDA(cudaMemsetAsync(d_bad, 0, 4, st));
    HGI_CUDA(cudaMemcpyAsync(d_idx, idx, ib, cudaMemcpyHostToDevice, st));
    HGI_CUDA(cudaMemcpyAsync(d_states, states, size_t(n_states) * 16, cudaMemcpyHostToDevice, st));
    HGI_CUDA(cudaMemcpyAsync(d_k, k.data(), size_t(n_states) * 4, cudaMemcpyHostToDevice, st));
    HGI_CUDA(cudaMemcpyAsync(d_tabs, tabs.data(), tabs.size() * 4, cudaMemcpyHostToDevice, st));
    hgi_crc_kernel<<<unsigned(nblocks), kCrcBlock, 0, st>>>(d_idx, idx_bytes, count, pad, static_cast<uint32_t*>(d_k),
                                                            n_states, static_cast<uint32_t*>(d_tabs),
                                                            static_cast<uint32_t*>(d_tabs) + 1024,
                                                            static_cast<uint32_t*>(d_blk), d_bad);
    HGI_CUDA(cudaGetLastError());
    if (out_payload && count > 0) {
        HGI_CUDA(cudaMallocAsync(&d_pay, size_t(count) * 16, st));
        hgi_expand_kernel<<<grid_for(count), 256, 0, st>>>(d_idx, idx_bytes, count, static_cast<double2*>(d_states),
                                                          n_states, static_cast<double2*>(d_pay), d_bad);
        HGI_CUDA(cudaGetLastError());
        HGI_CUDA(cudaMemcpyAsync(out_payload, d_pay, size_t(count) * 16, cudaMemcpyDeviceToHost, st));
    }
    std::vector<uint32_t> blk(static_cast<size_t>(nblocks) + 1);
    HGI_CUDA(cudaMemcpyAsync(blk.data(), d_blk, size_t(nblocks) * 4 + 4, cudaMemcpyDeviceToHost, st));
    HGI_CUDA(cudaStreamSynchronize(st));
    cleanup();
    if (blk[size_t(nblocks)] != 0u) return fail(CGH_ERR_VALUE, "index outside the state table (%d states)", n_states);
#undef HGI_CUDA
    // fold the block registers (each covers per_block records) and condition
    std::vector<uint32_t> sb(1024);
    byte_tables(shift_matrix(uint64_t(16) * per_block), sb.data());
    uint32_t raw = 0;
    for (long long b = 0; b < nblocks; ++b) {
        const uint32_t c = raw;
        raw = sb[c & 255u] ^ sb[256 + (c >> 8 & 255u)] ^ sb[512 + (c >> 16 & 255u)] ^ sb[768 + (c >> 24)];
        raw ^= blk[size_t(b)];
    }
    const uint32_t init = mat_apply(shift_matrix(uint64_t(count) * 16), 0xFFFFFFFFu);
    *out_crc = raw ^ init ^ 0xFFFFFFFFu;
    return CGH_OK;
}

}  // extern "C"

// ---- full-plane rank-1 replay update (cghkit/propagation.py:205-218,
// SURVEY.md §8(f) #4): replay[u][v] += delta / sqrt(HW) * w_H^(m u) * w_W^(n v),
// with the exponents reduced mod H / W into long-double-built 1-D tables.
namespace cgh {
__global__ void delta_update_kernel(double2* __restrict__ R, int H, int W, int m, int n, double2 d,
                                    const double2* __restrict__ rt, const double2* __restrict__ ct) {
    const long long total = (long long)H * W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (long long)gridDim.x * blockDim.x) {
        const int u = int(p / W), v = int(p - (long long)u * W);
        const double2 a = rt[(long long)m * u % H], b = ct[(long long)n * v % W];
        const double2 w = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
        R[p].x += d.x * w.x - d.y * w.y;
        R[p].y += d.x * w.y + d.y * w.x;
    }
}
}  // namespace cgh

extern "C" int cgh_delta_replay_update(int32_t device, double* replay, int32_t h, int32_t w, int32_t m, int32_t n,
                                       double delta_re, double delta_im) {
    if (!replay || h < 1 || w < 1) return fail(CGH_ERR_VALUE, "bad arguments");
    if (m < 0 || m >= h || n < 0 || n >= w) return fail(CGH_ERR_VALUE, "pixel (%d, %d) outside %dx%d", m, n, h, w);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    if (device < 0 || device >= ndev) return fail(CGH_ERR_VALUE, "device %d out of range", device);
    CGH_CUDA(cudaSetDevice(device));
    std::vector<double> rt, ct;
    twiddle_table(h, rt);
    twiddle_table(w, ct);
    const size_t n_el = size_t(h) * w;
    double2 *d_r = nullptr, *d_rt = nullptr, *d_ct = nullptr;
    CGH_CUDA(cudaMalloc(&d_r, n_el * 16));
    CGH_CUDA(cudaMalloc(&d_rt, size_t(h) * 16));
    CGH_CUDA(cudaMalloc(&d_ct, size_t(w) * 16));
    cudaMemcpy(d_r, replay, n_el * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rt, rt.data(), size_t(h) * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ct, ct.data(), size_t(w) * 16, cudaMemcpyHostToDevice);
    const double s = 1.0 / std::sqrt(double(h) * double(w));
    delta_update_kernel<<<grid_for((long)n_el), 256>>>(d_r, h, w, m, n, make_double2(delta_re * s, delta_im * s), d_rt, d_ct);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(replay, d_r, n_el * 16, cudaMemcpyDeviceToHost);
    cudaFree(d_r);
    cudaFree(d_rt);
    cudaFree(d_ct);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "delta replay update: %s", cudaGetErrorString(e));
    return CGH_OK;
}
