// Line passes over a rank's slab of a row-distributed N x N GS run (config C6,
// SURVEY.md §8(e)): both GS passes run as row passes, the corner turn between
// them is a block transpose plus one all-to-all.
//
// Slab layout ("segmented rows"): a rank owns R = N/G lines of N points,
// stored as G segments of S = N/G points, segment-major:
//     element (line i, position n)  at  ((n / S) * R + i) * S + (n % S).
// Block g of the slab ([R][S], contiguous) is exactly the chunk exchanged with
// rank g, so transposing every block and calling all_to_all_single turns the
// hologram-plane row slab into the replay-plane column slab (and back) in the
// same layout. For G = 1 this is plain row-major.
//
// Per line the arithmetic is the generic row/column pass of pass_kernels.cuh
// (same LineFft, twiddle tables, projection and snapping), so fields and index
// planes equal the single-GPU generic path bit for bit; only the order of the
// error sums differs (per-rank block sums, all-reduced once per run).
#pragma once
#include "pass_kernels.cuh"

namespace cgh {

enum SlabMode {
    SLAB_INIT = 0,    // random-phase start (global row-major draws) [-> snap] -> forward line FFT
    SLAB_HOLO = 1,    // inverse -> hologram projection [-> snap] -> forward   (row pass of GS)
    SLAB_GS = 2,      // forward -> error sums + replay projection -> inverse  (column pass of GS)
    SLAB_FINAL = 3,   // forward -> error + efficiency sums (no store)
    SLAB_INV = 4,     // inverse, scaled (backpropagation start)
};

template <class T, int N>
struct SlabShape {
    // 16384-point fp32 lines: 32 points per thread (512 threads, 128 registers)
    // instead of 16 (1024 threads would cap registers at 64 and spill)
    static constexpr int E = (sizeof(T) == 4 && N >= 16384) ? 32 : LineShape<T, N>::E;
    static constexpr int TF = N / E;
    static constexpr int THREADS = TF >= 256 ? TF : 256;
    static constexpr int LINES = THREADS / TF;
    static constexpr int WORDS = line_words<T, N>();
    static constexpr size_t SMEM = size_t(LINES) * 2 * WORDS * sizeof(T) + 16 + 32 * 4 * sizeof(double);
};

template <class T>
struct SlabArgs {
    cx<T>* data;          // segmented slab
    int R, logS;          // local lines, log2(segment length)
    int line0;            // global index of local line 0
    const T* tgt;         // SLAB_GS/FINAL: [R][N] ifftshifted |T| of this rank's columns, sign = outside mask
    PassArgs<T> p;        // beam ([R][N]), q_row (offset by line0), q_col, scheme, idx_out ([R][N]), quantize
    T gain, scale;
    Pcg64 rng;
    ReduceArgs red;       // out[0..3] = S_dd, S_rr, S_rd, S_all of this rank
};

template <class T, int N, int MODE>
__global__ void __launch_bounds__(SlabShape<T, N>::THREADS) slab_kernel(SlabArgs<T> a) {
    constexpr int mode = MODE;
    using Sh = SlabShape<T, N>;
    constexpr int E = Sh::E, TF = Sh::TF, WORDS = Sh::WORDS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int li = threadIdx.x / TF, t = threadIdx.x - li * TF;
    const int i = blockIdx.x * Sh::LINES + li;
    const bool active = i < a.R;
    T* sre = reinterpret_cast<T*>(smem) + li * 2 * WORDS;
    T* sim = sre + WORDS;
    double* rs = red_scratch<T>(smem, size_t(Sh::LINES) * 2 * WORDS * sizeof(T));
    const int S = 1 << a.logS;
    auto at = [&](int n) -> long { return (long((n >> a.logS)) * a.R + i) * S + (n & (S - 1)); };
    cx<T> v[E];

    if constexpr (mode == SLAB_INIT) {
        // thread t draws the contiguous chunk [t*E, t*E+E) of global row line0+i
        // (row-major over the full plane, algorithms.py:132), staged through smem
        if (active) {
            Pcg64 g = a.rng;
            pcg_advance(g, uint64_t(long(a.line0 + i) * N + long(t) * E));
#pragma unroll 4
            for (int e = 0; e < E; ++e) {
                const cx<T> z = unit_phase<T>(g);
                const int pos = t * E + e;
                const T amp = a.p.beam ? a.p.beam[long(i) * N + pos] : T(1);
                const int q = padx<T>(pos);
                sre[q] = amp * z.x;
                sim[q] = amp * z.y;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int q = padx<T>(t + r * TF);
            v[r] = mk(sre[q], sim[q]);
        }
        if (active) {
            const bool fres = a.p.q_row != nullptr;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int n = t + r * TF;
                cx<T> h = v[r];
                if (a.p.quantize) {
                    const int k = quantize_index<T>(a.p.scheme, h);
                    if (a.p.idx_out) {
                        const long q = long(i) * N + n;
                        if (a.p.idx_bytes == 1) static_cast<uint8_t*>(a.p.idx_out)[q] = (uint8_t)k;
                        else static_cast<int32_t*>(a.p.idx_out)[q] = k;
                    }
                    h = state_value<T>(a.p.scheme, k);
                }
                if (fres) h = cmul(h, cmul(a.p.q_row[i], a.p.q_col[n]));
                v[r] = h;
            }
        }
        LineFft<T, N, -1, E>::run(v, sre, sim, t, a.p.tw_row);
    } else {
#pragma unroll
        for (int r = 0; r < E; ++r) v[r] = active ? a.data[at(t + r * TF)] : mk<T>(0, 0);
        if constexpr (mode == SLAB_HOLO) {
            LineFft<T, N, +1, E>::run(v, sre, sim, t, a.p.tw_row);
            if (active) {
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = holo_project<T>(a.p, v[r], i, t + r * TF, 0);
            }
            LineFft<T, N, -1, E>::run(v, sre, sim, t, a.p.tw_row);
        } else if constexpr (mode == SLAB_INV) {
            LineFft<T, N, +1, E>::run(v, sre, sim, t, a.p.tw_row);
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
        } else {   // SLAB_GS, SLAB_FINAL (pass_kernels.cuh COL_GS / COL_FINAL per line)
            LineFft<T, N, -1, E>::run(v, sre, sim, t, a.p.tw_row);
            T sdd = 0, srr = 0, srd = 0, sall = 0;
            const T gain = a.gain;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int u = t + r * TF;
                const cx<T> Rv = v[r] * a.scale;
                const T r2 = Rv.x * Rv.x + Rv.y * Rv.y;
                const T rr = dev_sqrt<T>(r2);
                const T tt = active ? a.tgt[long(i) * N + u] : T(-0.0);
                sall += active ? r2 : T(0);
                cx<T> out = Rv;
                if (!signbit(tt)) {
                    const T d = rr - tt;
                    sdd += d * d;
                    srr += r2;
                    srd += rr * d;
                    if constexpr (mode == SLAB_GS) {
                        T want = tt + gain * (tt - rr);
                        want = want > T(0) ? want : T(0);
                        if (rr > T(0)) {
                            const T s = want / rr;
                            out = mk(Rv.x * s, Rv.y * s);
                        } else {
                            out = mk(want, T(0));
                        }
                    }
                }
                v[r] = out;
            }
            if constexpr (mode == SLAB_GS) LineFft<T, N, +1, E>::run(v, sre, sim, t, a.p.tw_row);
            double acc[4] = {double(sdd), double(srr), double(srd), double(sall)};
            block_reduce<4>(acc, rs);
            const int nblocks = gridDim.x;
            if (publish_partials<4>(a.red, acc, nblocks, blockIdx.x)) {
                const double s0 = sum_partials(a.red, 0, nblocks, rs);
                const double s1 = sum_partials(a.red, 1, nblocks, rs);
                const double s2 = sum_partials(a.red, 2, nblocks, rs);
                const double s3 = sum_partials(a.red, 3, nblocks, rs);
                if (threadIdx.x == 0) {
                    a.red.out[0] = s0;
                    a.red.out[1] = s1;
                    a.red.out[2] = s2;
                    a.red.out[3] = s3;
                    *a.red.counter = 0u;
                }
            }
            if constexpr (mode == SLAB_FINAL) return;
        }
    }
    if (active) {
#pragma unroll
        for (int r = 0; r < E; ++r) a.data[at(t + r * TF)] = v[r];
    }
}

// dst[g] = transpose(src[g]) for the G square blocks [S][S] of a slab (32 x 32
// tiles through shared memory, one padding column against bank conflicts).
template <class T>
__global__ void __launch_bounds__(256) slab_transpose_kernel(const cx<T>* __restrict__ src, cx<T>* __restrict__ dst,
                                                             int S) {
    __shared__ cx<T> tile[32][33];
    const long blk = long(blockIdx.z) * S * S;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += 8) {
        const int y = y0 + k, x = x0 + threadIdx.x;
        if (y < S && x < S) tile[k][threadIdx.x] = src[blk + long(y) * S + x];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += 8) {
        const int y = x0 + k, x = y0 + threadIdx.x;   // dst row = src column
        if (y < S && x < S) dst[blk + long(y) * S + x] = tile[threadIdx.x][k];
    }
}

template <class T, int N, int MODE>
cudaError_t slab_launch_m(const SlabArgs<T>& a, cudaStream_t st) {
    using Sh = SlabShape<T, N>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(slab_kernel<T, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Sh::SMEM));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int grid = (a.R + Sh::LINES - 1) / Sh::LINES;
    slab_kernel<T, N, MODE><<<grid, Sh::THREADS, Sh::SMEM, st>>>(a);
    return cudaGetLastError();
}

template <class T, int N>
cudaError_t slab_launch_n(const SlabArgs<T>& a, int mode, cudaStream_t st) {
    switch (mode) {
        case SLAB_INIT: return slab_launch_m<T, N, SLAB_INIT>(a, st);
        case SLAB_HOLO: return slab_launch_m<T, N, SLAB_HOLO>(a, st);
        case SLAB_GS: return slab_launch_m<T, N, SLAB_GS>(a, st);
        case SLAB_FINAL: return slab_launch_m<T, N, SLAB_FINAL>(a, st);
        case SLAB_INV: return slab_launch_m<T, N, SLAB_INV>(a, st);
        default: return cudaErrorInvalidValue;
    }
}

template <class T, int N>
constexpr int slab_blocks(int R) {
    return (R + SlabShape<T, N>::LINES - 1) / SlabShape<T, N>::LINES;
}

}  // namespace cgh

#define CGH_SLAB_INSTANTIATE(T, N) \
    namespace cgh {                \
    template cudaError_t slab_launch_n<T, N>(const SlabArgs<T>&, int, cudaStream_t); \
    }
#define CGH_SLAB_EXTERN(T, N) \
    namespace cgh {           \
    extern template cudaError_t slab_launch_n<T, N>(const SlabArgs<T>&, int, cudaStream_t); \
    }
