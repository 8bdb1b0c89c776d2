// Runtime dispatch (line length, mode) -> templated pass kernels, and the
// element-wise helper kernels (target preparation, field conversion).
#pragma once
#include "pass_kernels.cuh"

namespace cgh {

constexpr int kMinLog2 = 1;    // N = 2
constexpr int kMaxLog2 = 12;   // N = 4096

template <class T, int N>
cudaError_t row_dispatch(int mode, const PassArgs<T>& a, int frames, cudaStream_t st);
template <class T, int N>
cudaError_t col_dispatch(int mode, const PassArgs<T>& a, int frames, cudaStream_t st);

template <class T>
cudaError_t launch_row(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st);
template <class T>
cudaError_t launch_col(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st);
template <class T>
int row_grid_blocks(int N, int H);
template <class T>
int col_grid_blocks(int N, int W);

// Non-power-of-two line lengths (anysize.cu): the same row/column pass modes
// with Bluestein line DFTs; one CTA per line. The line's twiddle table
// (PassArgs tw_row / tw_col) is then the packed Bluestein table of
// blue_pack_table: chirp [N] | chirp-filter spectrum [M] | exp(-2 pi i k / M) [M].
template <class T>
cudaError_t launch_row_any(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st);
template <class T>
cudaError_t launch_col_any(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st);
int blue_length(int n);
constexpr int kMaxAnyLine = 4096;   // non-power-of-two sides of GS plans

// ---------------------------------------------------------------- prep
// Build the uncentred (ifftshifted) target amplitude with the mask folded in
// as the sign bit, the hologram-plane beam amplitude, and optionally the
// shifted complex target; reduce [count_in_mask, sum_mask t^2,
// nonfinite_in_mask, nonfinite_anywhere, nonfinite_beam].
struct PrepStats {
    double* partials;
    unsigned* counter;
    double* out;   // 5 doubles
};

template <class T>
__global__ void prep_kernel(const double* __restrict__ tc, const uint8_t* __restrict__ mask,
                            const double* __restrict__ ic, int H, int W, T* __restrict__ tgt,
                            T* __restrict__ beam, cx<T>* __restrict__ shifted, PrepStats ps) {
    const long total = long(H) * W;
    double cnt = 0, den = 0, nfm = 0, nfa = 0, nfb = 0;
    for (long p = long(blockIdx.x) * blockDim.x + threadIdx.x; p < total; p += long(gridDim.x) * blockDim.x) {
        // planes are < 2^31 pixels (cgh_plan_create): 32-bit division, no modulo
        const unsigned pu = unsigned(p), uu = pu / unsigned(W);
        const int u = int(uu), v = int(pu - uu * unsigned(W));
        int uc = u + H / 2, vc = v + W / 2;
        if (uc >= H) uc -= H;
        if (vc >= W) vc -= W;
        const long pc = long(uc) * W + vc;
        const double re = tc[2 * pc], im = tc[2 * pc + 1];
        const double t = hypot(re, im);
        const bool in = mask[pc] != 0;
        const bool fin = isfinite(re) && isfinite(im);
        if (in) {
            cnt += 1.0;
            den += t * t;
            if (!fin) nfm += 1.0;
        }
        if (!fin) nfa += 1.0;
        T tt = T(t);
        tgt[p] = in ? tt : -tt;   // -0.0 for dark pixels outside the mask
        if (shifted) shifted[p] = mk<T>(T(re), T(im));
        if (beam) {
            const double br = ic[2 * p], bi = ic[2 * p + 1];
            if (!(isfinite(br) && isfinite(bi))) nfb += 1.0;
            beam[p] = T(hypot(br, bi));
        }
    }
    __shared__ double sh[32 * 5];
    double acc[5] = {cnt, den, nfm, nfa, nfb};
#pragma unroll
    for (int q = 0; q < 5; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int q = 0; q < 5; ++q) sh[q * 32 + warp] = acc[q];
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 5; ++q) {
            double s = 0;
            for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
            ps.partials[q * gridDim.x + blockIdx.x] = s;
        }
        __threadfence();
        last = atomicAdd(ps.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        // the whole last block sums the partials (strided per thread, then a
        // fixed shuffle/warp tree: deterministic); one thread summing up to
        // 2368 x 5 partials serially took most of the kernel's time
        __threadfence();
        double tot[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double s = 0;
            for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(&ps.partials[q * gridDim.x + b]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            tot[q] = s;
        }
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 5; ++q) sh[q * 32 + warp] = tot[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < 5; ++q) {
                double s = 0;
                for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
                ps.out[q] = s;
            }
            *ps.counter = 0u;
        }
    }
}

// complex128 host-layout field -> working precision, optional ifftshift of the
// input (inverse centred transform), optional Fresnel pre-multiply by q.
template <class T>
__global__ void load_field_kernel(const double* __restrict__ in, cx<T>* __restrict__ out, int H, int W,
                                  int shift, const cx<T>* __restrict__ qr, const cx<T>* __restrict__ qc,
                                  unsigned* __restrict__ nonfinite) {
    const long total = long(H) * W;
    for (long p = long(blockIdx.x) * blockDim.x + threadIdx.x; p < total; p += long(gridDim.x) * blockDim.x) {
        const int u = int(p / W), v = int(p - long(u) * W);
        long src = p;
        if (shift) src = long((u + H / 2) % H) * W + (v + W / 2) % W;
        const double re = in[2 * src], im = in[2 * src + 1];
        if (!(isfinite(re) && isfinite(im))) atomicAdd(nonfinite, 1u);
        cx<T> z = mk<T>(T(re), T(im));
        if (qr) z = cmul(z, cmul(qr[u], qc[v]));
        out[p] = z;
    }
}

// working precision -> complex128, optional fftshift of the output (forward
// centred transform), optional post-multiply by conj(q) (inverse Fresnel).
template <class T>
__global__ void store_field_kernel(const cx<T>* __restrict__ in, double* __restrict__ out, int H, int W,
                                   int shift, const cx<T>* __restrict__ qr, const cx<T>* __restrict__ qc) {
    const long total = long(H) * W;
    for (long p = long(blockIdx.x) * blockDim.x + threadIdx.x; p < total; p += long(gridDim.x) * blockDim.x) {
        const int u = int(p / W), v = int(p - long(u) * W);
        long dst = p;
        if (shift) dst = long((u + H / 2) % H) * W + (v + W / 2) % W;   // np.fft.fftshift, odd sides too
        cx<T> z = in[p];
        if (qr) z = cmulc(z, cmul(qr[u], qc[v]));
        out[2 * dst] = double(z.x);
        out[2 * dst + 1] = double(z.y);
    }
}

// Pixel field from an index plane: states[idx] (* q).
template <class T>
__global__ void field_from_index_kernel(const void* __restrict__ idx, int idx_bytes, SchemeDev s,
                                        cx<T>* __restrict__ out, int H, int W, const cx<T>* __restrict__ qr,
                                        const cx<T>* __restrict__ qc) {
    const long total = long(H) * W;
    for (long p = long(blockIdx.x) * blockDim.x + threadIdx.x; p < total; p += long(gridDim.x) * blockDim.x) {
        const int u = int(p / W), v = int(p - long(u) * W);
        const int k = idx_bytes == 1 ? int(static_cast<const uint8_t*>(idx)[p]) : static_cast<const int32_t*>(idx)[p];
        cx<T> z = state_value<T>(s, k);
        if (qr) z = cmul(z, cmul(qr[u], qc[v]));
        out[p] = z;
    }
}

}  // namespace cgh
