// Kernel bodies for the row / column passes (instantiated per precision and
// line length in pass_fp32.cu / pass_fp64.cu).
#pragma once
#include "passes.cuh"

namespace cgh {

// Shared scratch for reductions (doubles), placed after the FFT exchange area.
constexpr int kRedWords = 32 * 4;

template <class T>
__device__ __forceinline__ double* red_scratch(unsigned char* smem, size_t fft_bytes) {
    return reinterpret_cast<double*>(smem + ((fft_bytes + 15) & ~size_t(15)));
}

// Random-phase start value of hologram pixel index p (row-major draw p).
template <class T>
__device__ __forceinline__ cx<T> unit_phase(Pcg64& g) {
    if constexpr (sizeof(T) == 8) {
        const double u = pcg_next_double(g);
        const double theta = 6.283185307179586 * u;   // 2.0 * np.pi * u
        double s, c;
        sincos(theta, &s, &c);
        return mk<T>(c, s);
    } else {
        float s, c;
        sincospif(pcg_next_halfturns(g), &s, &c);   // angle / pi in [-1, 1)
        return mk<T>(c, s);
    }
}

// ============================================================== row kernel
// Launch bound = the CTA size launch_row_n uses (max(TF, 256) threads: one
// 4096-point complex128 line takes 512 threads at 8 elements each).
// complex128 rows at 256 threads ask ptxas for 3 resident CTAs per SM (80
// registers; 24 warps instead of 16): C3 fp64 53.1 -> 51.2 ms per 200
// iterations on B200. 0 = no minimum (the default bound).
#ifndef CGH_F64_ROW_MINB
#define CGH_F64_ROW_MINB 3
#endif
template <class T, int N>
struct RowBounds {
    static constexpr int THREADS = LineShape<T, N>::TF >= 256 ? LineShape<T, N>::TF : 256;
    static constexpr int MINB = (sizeof(T) == 8 && THREADS == 256) ? CGH_F64_ROW_MINB : 0;
};
template <class T, int N, int MODE>
__global__ void __launch_bounds__(RowBounds<T, N>::THREADS, RowBounds<T, N>::MINB) row_kernel(PassArgs<T> a) {
    using Sh = LineShape<T, N>;
    constexpr int E = Sh::E, TF = Sh::TF;
    constexpr int WORDS = line_words<T, N>();
    extern __shared__ __align__(16) unsigned char smem[];
    const int lines = blockDim.x / TF;
    const int li = threadIdx.x / TF, t = threadIdx.x - li * TF;
    const int m = blockIdx.x * lines + li;
    const bool active = m < a.H;
    T* sre = reinterpret_cast<T*>(smem) + li * 2 * WORDS;
    T* sim = sre + WORDS;
    double* rs = red_scratch<T>(smem, size_t(lines) * 2 * WORDS * sizeof(T));
    const long foff = long(blockIdx.y) * a.frame_stride;
    cx<T>* row = a.data + foff + long(m) * N;
    cx<T> v[E];

    if constexpr (MODE == ROW_FWD || MODE == ROW_INV || MODE == ROW_HOLO) {
#pragma unroll
        for (int r = 0; r < E; ++r) v[r] = active ? row[t + r * TF] : mk<T>(0, 0);
        if constexpr (MODE == ROW_FWD) {
            LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_row);
        } else {
            LineFft<T, N, +1>::run(v, sre, sim, t, a.tw_row);
        }
        if constexpr (MODE == ROW_HOLO) {
            if (active) {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = holo_project<T>(a, v[r], m, t + r * TF, 0);
            }
            LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_row);
        } else if (a.scale != T(1)) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
        }
        if (active) {
#pragma unroll
            for (int r = 0; r < E; ++r) row[t + r * TF] = v[r];
        }
    } else if constexpr (MODE == ROW_INIT || MODE == ROW_OSPR_GEN) {
        // Each thread generates a contiguous chunk of E draws of this row,
        // stages it in shared memory, then reads back the strided layout.
        Pcg64 g;
        long first;
        int uc = m;
        if constexpr (MODE == ROW_INIT) {
            g = a.rng;
            first = long(m) * N + long(t) * E;
        } else {
            g = a.frame_rng[a.frame0 + blockIdx.y];
            uc = (m + a.H / 2) % a.H;             // centred row feeding uncentred row m
            first = long(uc) * N + long(t) * E;
        }
        if (active) {
            pcg_advance(g, uint64_t(first));
#pragma unroll 4
            for (int e = 0; e < E; ++e) {
                cx<T> z = unit_phase<T>(g);
                int pos = t * E + e;   // column index in draw order
                T amp;
                if constexpr (MODE == ROW_INIT) {
                    amp = a.beam ? a.beam[long(m) * N + pos] : T(1);
                } else {
                    pos = (pos + N / 2) % N;          // uncentred column
                    amp = fabs(a.tgt[long(m) * N + pos]);
                }
                const int p = padx<T>(pos);
                cx<T> h = mk(amp * z.x, amp * z.y);
                if constexpr (MODE == ROW_INIT) h = beam_zero_signs(amp, h);
                sre[p] = h.x;
                sim[p] = h.y;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int p = padx<T>(t + r * TF);
            v[r] = mk(sre[p], sim[p]);
        }
        if constexpr (MODE == ROW_INIT) {
            if (active) {
                const bool fres = a.q_row != nullptr;
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int n = t + r * TF;
                    cx<T> h = v[r];
                    if (a.field_out) a.field_out[long(m) * N + n] = h;
                    if (a.quantize) {
                        const int k = quantize_index<T>(a.scheme, h);
                        if (a.idx_out) {
                            const long p = long(m) * N + n;
                            if (a.idx_bytes == 1) static_cast<uint8_t*>(a.idx_out)[p] = (uint8_t)k;
                            else static_cast<int32_t*>(a.idx_out)[p] = k;
                        }
                        h = state_value<T>(a.scheme, k);
                    }
                    if (fres) h = cmul(h, cmul(a.q_row[m], a.q_col[n]));
                    v[r] = h;
                }
            }
            LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_row);
        } else {
            LineFft<T, N, +1>::run(v, sre, sim, t, a.tw_row);
        }
        if (active) {
#pragma unroll
            for (int r = 0; r < E; ++r) row[t + r * TF] = v[r];
        }
    } else if constexpr (MODE == ROW_OSPR_ACC) {
        // Row m of every frame in [frame0, frame0+frames): forward row FFT,
        // accumulate |R|^2, per-frame masked error sums of sqrt(I / i).
        __shared__ double blk[3 * 64 + 2];
        T inten[E];
        const long pix0 = long(m) * N;
#pragma unroll
        for (int r = 0; r < E; ++r)
            inten[r] = (active && a.load_intensity) ? a.intensity[pix0 + t + r * TF] : T(0);
        T tv[E];
#pragma unroll
        for (int r = 0; r < E; ++r) tv[r] = active ? a.tgt[pix0 + t + r * TF] : T(-0.0);
        for (int f = 0; f < a.frames; ++f) {
            cx<T>* fr = a.data + long(f) * a.frame_stride + pix0;
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = active ? fr[t + r * TF] : mk<T>(0, 0);
            LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_row);
            const T inv_n = T(1) / T(a.frame0 + f + 1);
            T sdd = 0, spp = 0, spd = 0;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const cx<T> R = v[r] * a.scale;
                inten[r] += R.x * R.x + R.y * R.y;
                if (!signbit(tv[r])) {
                    const T p = dev_sqrt<T>(inten[r] * inv_n);
                    const T d = p - tv[r];
                    sdd += d * d;
                    spp += p * p;
                    spd += p * d;
                }
            }
            double acc[3] = {double(sdd), double(spp), double(spd)};
            block_reduce<3>(acc, rs);
            if (threadIdx.x == 0) {
                blk[3 * f + 0] = acc[0];
                blk[3 * f + 1] = acc[1];
                blk[3 * f + 2] = acc[2];
            }
        }
        const bool tail = (a.frame0 + a.frames == a.nframes_total);
        int nq = 3 * a.frames;
        if (tail) {
            const T inv_n = T(1) / T(a.nframes_total);
            T sin_ = 0, sall = 0;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const T p2 = inten[r] * inv_n;   // perceived^2
                const T p = dev_sqrt<T>(p2);
                const T pp = p * p;
                sall += pp;
                if (!signbit(tv[r])) sin_ += pp;
            }
            double acc[2] = {double(sin_), double(sall)};
            block_reduce<2>(acc, rs);
            if (threadIdx.x == 0) {
                blk[nq + 0] = acc[0];
                blk[nq + 1] = acc[1];
            }
            nq += 2;
        }
        if (a.store_intensity && active) {
#pragma unroll
            for (int r = 0; r < E; ++r) a.intensity[pix0 + t + r * TF] = inten[r];
        }
        // publish and let the last block finish
        const int nblocks = gridDim.x;
        __shared__ int last;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < nq; ++q) a.red.partials[long(q) * nblocks + blockIdx.x] = blk[q];
            __threadfence();
            last = (atomicAdd(a.red.counter, 1u) == unsigned(nblocks - 1));
        }
        __syncthreads();
        if (last) {
            __threadfence();
            const double denom = *a.red.denom;
            for (int f = 0; f < a.frames; ++f) {
                const double sdd = sum_partials(a.red, 3 * f + 0, nblocks, rs);
                const double spp = sum_partials(a.red, 3 * f + 1, nblocks, rs);
                const double spd = sum_partials(a.red, 3 * f + 2, nblocks, rs);
                if (threadIdx.x == 0) a.red.out[a.frame0 + f] = error_from_sums(sdd, spp, spd, denom, a.red.rescale);
            }
            if (tail) {
                const double sin_ = sum_partials(a.red, 3 * a.frames + 0, nblocks, rs);
                const double sall = sum_partials(a.red, 3 * a.frames + 1, nblocks, rs);
                if (threadIdx.x == 0)
                    a.red.out[a.nframes_total] = sall == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : sin_ / sall;
            }
            if (threadIdx.x == 0) *a.red.counter = 0u;
        }
    }
}

// =========================================================== column kernel
// (CGH_COL_LB_THREADS / CGH_COL_LB_MINB: A/B builds of the complex128 column pass)
#ifndef CGH_COL_LB_THREADS
#define CGH_COL_LB_THREADS 512
#define CGH_COL_LB_MINB 0
#endif
template <class T, int N, int MODE>
__global__ void __launch_bounds__(CGH_COL_LB_THREADS, CGH_COL_LB_MINB) col_kernel(PassArgs<T> a) {
    using Sh = LineShape<T, N>;
    constexpr int E = Sh::E, TF = Sh::TF;
    constexpr int WORDS = line_words<T, N>();
    extern __shared__ __align__(16) unsigned char smem[];
    const int C = blockDim.x / TF;
    const int t = threadIdx.x / C, c = threadIdx.x - t * C;
    const int n = blockIdx.x * C + c;
    const bool active = n < a.W;
    T* sre = reinterpret_cast<T*>(smem) + c * 2 * WORDS;
    T* sim = sre + WORDS;
    double* rs = red_scratch<T>(smem, size_t(C) * 2 * WORDS * sizeof(T));
    const long foff = long(blockIdx.y) * a.frame_stride;
    cx<T>* col = a.data + foff + n;
    const long W = a.W;
    cx<T> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = active ? col[long(t + r * TF) * W] : mk<T>(0, 0);

    if constexpr (MODE == COL_FWD || MODE == COL_INV) {
        if constexpr (MODE == COL_FWD) LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_col);
        else LineFft<T, N, +1>::run(v, sre, sim, t, a.tw_col);
        if (a.scale != T(1)) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
        }
    } else if constexpr (MODE == COL_HOLO) {
        LineFft<T, N, +1>::run(v, sre, sim, t, a.tw_col);
        if (active) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = holo_project<T>(a, v[r], t + r * TF, n, foff);
        }
        LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_col);
    } else {   // COL_GS, COL_FINAL
        LineFft<T, N, -1>::run(v, sre, sim, t, a.tw_col);
        T sdd = 0, srr = 0, srd = 0, sall = 0;
        const T gain = a.gain;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int u = t + r * TF;
            const cx<T> R = v[r] * a.scale;
            const T r2 = R.x * R.x + R.y * R.y;
            const T rr = dev_sqrt<T>(r2);
            const T tt = active ? a.tgt[long(u) * W + n] : T(-0.0);
            sall += active ? r2 : T(0);
            cx<T> out = R;
            if (!signbit(tt)) {
                const T d = rr - tt;
                sdd += d * d;
                srr += r2;
                srd += rr * d;
                if constexpr (MODE == COL_GS) {
                    T want = tt + gain * (tt - rr);
                    want = want > T(0) ? want : T(0);
                    if (rr > T(0)) {
                        const T s = want / rr;
                        out = mk(R.x * s, R.y * s);
                    } else {
                        out = mk(want, T(0));
                    }
                }
            }
            v[r] = out;
        }
        if constexpr (MODE == COL_GS) LineFft<T, N, +1>::run(v, sre, sim, t, a.tw_col);
        double acc[4] = {double(sdd), double(srr), double(srd), double(sall)};
        block_reduce<4>(acc, rs);
        const int nblocks = gridDim.x;
        if (publish_partials<4>(a.red, acc, nblocks, blockIdx.x)) {
            const double s_dd = sum_partials(a.red, 0, nblocks, rs);
            const double s_rr = sum_partials(a.red, 1, nblocks, rs);
            const double s_rd = sum_partials(a.red, 2, nblocks, rs);
            const double s_all = sum_partials(a.red, 3, nblocks, rs);
            if (threadIdx.x == 0) {
                a.red.out[0] = error_from_sums(s_dd, s_rr, s_rd, *a.red.denom, a.red.rescale);
                a.red.out[1] = s_all == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : s_rr / s_all;
                *a.red.counter = 0u;
            }
        }
        if constexpr (MODE == COL_FINAL) return;
    }
    if (active) {
#pragma unroll
        for (int r = 0; r < E; ++r) col[long(t + r * TF) * W] = v[r];
    }
}

// ================================================================ launch
template <class T, int N>
struct LaunchShape {
    static constexpr int TF = LineShape<T, N>::TF;
    static int row_lines(int H) {
        int lines = TF >= 256 ? 1 : 256 / TF;
        return lines;
    }
    static int col_cols(int W) {
        // 512 threads per CTA: C columns side by side across lanes
        // (CGH_FP64_COLS overrides it for complex128 lines, A/B builds)
#ifdef CGH_FP64_COLS
        if (sizeof(T) == 8 && N >= 1024) return CGH_FP64_COLS;
#endif
        return TF >= 512 ? 1 : 512 / TF;
    }
};

template <class T, int N>
size_t row_smem(int lines) {
    return ((size_t(lines) * 2 * line_words<T, N>() * sizeof(T) + 15) & ~size_t(15)) + kRedWords * sizeof(double);
}

template <class T, int N, int MODE>
cudaError_t launch_row_n(const PassArgs<T>& a, int frames, cudaStream_t st) {
    const int lines = LaunchShape<T, N>::row_lines(a.H);
    const size_t sm = row_smem<T, N>(lines);
    auto k = row_kernel<T, N, MODE>;
    if (sm > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.H + lines - 1) / lines, MODE == ROW_OSPR_ACC ? 1 : frames);
    k<<<grid, lines * LineShape<T, N>::TF, sm, st>>>(a);
    return cudaGetLastError();
}

template <class T, int N, int MODE>
cudaError_t launch_col_n(const PassArgs<T>& a, int frames, cudaStream_t st) {
    const int C = LaunchShape<T, N>::col_cols(a.W);
    const size_t sm = row_smem<T, N>(C);
    auto k = col_kernel<T, N, MODE>;
    if (sm > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + C - 1) / C, frames);
    k<<<grid, C * LineShape<T, N>::TF, sm, st>>>(a);
    return cudaGetLastError();
}

template <class T, int N>
int row_blocks(int H) {
    const int lines = LaunchShape<T, N>::row_lines(H);
    return (H + lines - 1) / lines;
}
template <class T, int N>
int col_blocks(int W) {
    const int C = LaunchShape<T, N>::col_cols(W);
    return (W + C - 1) / C;
}

}  // namespace cgh
