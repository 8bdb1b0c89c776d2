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
#include <algorithm>
#include <type_traits>

#include "launch.cuh"
#include "pass_kernels.cuh"

namespace cgh {

enum SlabMode {
    SLAB_INIT = 0,    // random-phase start (global row-major draws) [-> snap] -> forward line FFT
    SLAB_HOLO = 1,    // inverse -> hologram projection [-> snap] -> forward   (row pass of GS)
    SLAB_GS = 2,      // forward -> error sums + replay projection -> inverse  (column pass of GS)
    SLAB_FINAL = 3,   // forward -> error + efficiency sums (no store)
    SLAB_INV = 4,     // inverse, scaled (backpropagation start)
    SLAB_HOLO_SNAP = 5,   // internal: SLAB_HOLO with snapping (chosen by slab_launch_n when quantize is set)
    SLAB_FWD = 6,     // forward, unscaled (transform-only: line FFT checks against numpy.fft.fft)
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
    // fp32: two-level twiddle table in shared memory (fp64 parity mode keeps
    // the exact N-entry table of the generic passes)
    static constexpr bool SPLIT_TW = sizeof(T) == 4 && N >= 1024;
    static constexpr int TW_SH = (ilog2(N) + 1) / 2;
    static constexpr int TW_WORDS = SPLIT_TW ? ((N >> TW_SH) + (1 << TW_SH)) : 0;
    static constexpr size_t FFT_BYTES = size_t(LINES) * 2 * WORDS * sizeof(T);
    static constexpr size_t TW_OFF = (FFT_BYTES + 16 + 32 * 4 * sizeof(double) + 15) / 16 * 16;
    // per-thread fp64 error-sum slots (kept out of registers across the FFTs)
    static constexpr size_t ACC_OFF = (TW_OFF + size_t(TW_WORDS) * sizeof(cx<T>) + 15) / 16 * 16;
    static constexpr size_t SMEM = ACC_OFF + 4 * size_t(THREADS) * sizeof(double);
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

template <class T, int N, int DIR>
__device__ __forceinline__ void slab_fft(cx<T> (&v)[SlabShape<T, N>::E], T* sre, T* sim, int t,
                                         const unsigned char* smem, const cx<T>* tw) {
    using Sh = SlabShape<T, N>;
    if constexpr (Sh::SPLIT_TW) {
        const cx<T>* tws = reinterpret_cast<const cx<T>*>(smem + Sh::TW_OFF);
        LineFft<T, N, DIR, Sh::E>::run(v, sre, sim, t, TwSplit<T>{tws, tws + (N >> Sh::TW_SH), Sh::TW_SH});
    } else {
        LineFft<T, N, DIR, Sh::E>::run(v, sre, sim, t, tw);
    }
}

// Persistent: CTA b transforms line groups b, b + gridDim.x, ... (tables set
// up once per CTA). An L2 bulk prefetch of each CTA's next line was measured
// to double the pass's DRAM traffic (prefetched lines evicted before use) and
// to cost 5% at 16384^2, so lines are loaded on demand.
template <class T, int N, int MODE>
__global__ void __launch_bounds__(SlabShape<T, N>::THREADS) slab_kernel(SlabArgs<T> a) {
    using Sh = SlabShape<T, N>;
    constexpr int mode = MODE;
    constexpr int E = Sh::E, TF = Sh::TF, WORDS = Sh::WORDS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int li = threadIdx.x / TF, t = threadIdx.x - li * TF;
    T* sre = reinterpret_cast<T*>(smem) + li * 2 * WORDS;
    T* sim = sre + WORDS;
    double* rs = red_scratch<T>(smem, Sh::FFT_BYTES);
    const int S = 1 << a.logS;

    if constexpr (Sh::SPLIT_TW) {
        cx<T>* tws = reinterpret_cast<cx<T>*>(smem + Sh::TW_OFF);
        constexpr int NH = N >> Sh::TW_SH, NL = 1 << Sh::TW_SH;
        for (int k = threadIdx.x; k < NH + NL; k += blockDim.x)
            tws[k] = k < NH ? ldg_cx(a.p.tw_row + (k << Sh::TW_SH)) : ldg_cx(a.p.tw_row + (k - NH));
    }
    // SLAB_GS / SLAB_FINAL: this thread's sums over its lines, slot q at acc[q * THREADS]
    double* acc_sh = reinterpret_cast<double*>(smem + Sh::ACC_OFF) + threadIdx.x;
    if constexpr (mode == SLAB_GS || mode == SLAB_FINAL) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc_sh[q * Sh::THREADS] = 0.0;
    }

    for (int base = blockIdx.x * Sh::LINES; base < a.R; base += gridDim.x * Sh::LINES) {
        const int i = base + li;
        const bool active = i < a.R;
        auto at = [&](int n) -> long { return (long((n >> a.logS)) * a.R + i) * S + (n & (S - 1)); };
        __syncthreads();   // shared line buffers / twiddles ready, previous line done
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
                    const cx<T> h = beam_zero_signs(amp, mk(amp * z.x, amp * z.y));
                    sre[q] = h.x;
                    sim[q] = h.y;
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
            slab_fft<T, N, -1>(v, sre, sim, t, smem, a.p.tw_row);
        } else {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = active ? a.data[at(t + r * TF)] : mk<T>(0, 0);
            if constexpr (mode == SLAB_HOLO || mode == SLAB_HOLO_SNAP) {
                // the snapping code stays out of the iteration kernel (its
                // 32-fold unrolled quantizer cost instruction-cache misses)
                slab_fft<T, N, +1>(v, sre, sim, t, smem, a.p.tw_row);
                if (active) {
                    if (mode == SLAB_HOLO && !a.p.q_row && !a.p.beam) {
                        // Fourier, uniform beam: h = x/|x| (0 -> 1), holo_project's arithmetic with amp = 1
#pragma unroll
                        for (int r = 0; r < E; ++r) {
                            const T mag2 = v[r].x * v[r].x + v[r].y * v[r].y;
                            T inv;
                            if constexpr (sizeof(T) == 4) inv = rsqrtf(mag2);
                            else inv = T(1) / dev_sqrt<T>(mag2);
                            v[r] = mag2 > T(0) ? mk(v[r].x * inv, v[r].y * inv) : mk<T>(1, 0);
                        }
                    } else {
#pragma unroll
                        for (int r = 0; r < E; ++r)
                            v[r] = holo_project<T, mode == SLAB_HOLO_SNAP>(a.p, v[r], i, t + r * TF, 0);
                    }
                }
                slab_fft<T, N, -1>(v, sre, sim, t, smem, a.p.tw_row);
            } else if constexpr (mode == SLAB_INV) {
                slab_fft<T, N, +1>(v, sre, sim, t, smem, a.p.tw_row);
#pragma unroll
                for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
            } else if constexpr (mode == SLAB_FWD) {
                slab_fft<T, N, -1>(v, sre, sim, t, smem, a.p.tw_row);
            } else {   // SLAB_GS, SLAB_FINAL (pass_kernels.cuh COL_GS / COL_FINAL per line)
                slab_fft<T, N, -1>(v, sre, sim, t, smem, a.p.tw_row);
                const T gain = a.gain;
                T sdd = 0, srr = 0, srd = 0, sall = 0;
                if constexpr (sizeof(T) == 4) {
                    // branchless fp32 form of the fast column pass (fast_col_gs):
                    // |R| = r2 * rsqrt(r2), projection scale = want * rsqrt(r2)
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        const int u = t + r * TF;
                        const cx<T> Rv = v[r] * a.scale;
                        const float r2 = Rv.x * Rv.x + Rv.y * Rv.y;
                        const float ri = rsqrtf(r2);                 // inf at 0
                        const float rr = r2 > 0.0f ? r2 * ri : 0.0f;
                        const float tt = active ? a.tgt[long(i) * N + u] : -0.0f;
                        const bool in = !signbit(tt);
                        const float d = rr - tt;
                        sall += active ? r2 : 0.0f;
                        sdd += in ? d * d : 0.0f;
                        srr += in ? r2 : 0.0f;
                        srd += in ? rr * d : 0.0f;
                        if constexpr (mode == SLAB_GS) {
                            const float want = fmaxf(tt + gain * (tt - rr), 0.0f);
                            const bool pos = r2 > 0.0f;
                            const float kk = in ? (pos ? want * ri : 0.0f) : 1.0f;
                            v[r] = mk(Rv.x * kk + ((in && !pos) ? want : 0.0f), Rv.y * kk);
                        }
                    }
                } else {
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
                                    const T sc = want / rr;
                                    out = mk(Rv.x * sc, Rv.y * sc);
                                } else {
                                    out = mk(want, T(0));
                                }
                            }
                        }
                        v[r] = out;
                    }
                }
                acc_sh[0] += double(sdd);
                acc_sh[Sh::THREADS] += double(srr);
                acc_sh[2 * Sh::THREADS] += double(srd);
                acc_sh[3 * Sh::THREADS] += double(sall);
                if constexpr (mode == SLAB_GS) slab_fft<T, N, +1>(v, sre, sim, t, smem, a.p.tw_row);
            }
        }
        if (mode != SLAB_FINAL && active) {
            // store addresses recomputed from an opaque copy of the line index so
            // the compiler does not keep the E load addresses live across the FFTs
            int io;
            asm volatile("mov.b32 %0, %1;" : "=r"(io) : "r"(i));
            const int So = 1 << a.logS;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int n = t + r * TF;
                a.data[(long((n >> a.logS)) * a.R + io) * So + (n & (So - 1))] = v[r];
            }
        }
    }
    if constexpr (mode == SLAB_GS || mode == SLAB_FINAL) {
        double acc[4] = {acc_sh[0], acc_sh[Sh::THREADS], acc_sh[2 * Sh::THREADS], acc_sh[3 * Sh::THREADS]};
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

// Corner turn fused with the exchange: block g of the local slab is
// transposed through shared memory and stored straight into dst.p[g] (another
// rank's receive buffer over NVLink peer mappings, another virtual rank's
// buffer, or the local buffer when G = 1).
constexpr int kMaxTurnBlocks = 64;
template <class T>
struct TurnTargets {
    cx<T>* p[kMaxTurnBlocks];
};

// TL x TL tiles (64 for complex64: 512-B row segments on both sides, which
// keeps DRAM pages open longer than 32-wide tiles; 32 for complex128 to stay
// within static shared memory), 256 threads.
template <class T>
constexpr int turn_tile() { return sizeof(T) == 4 ? 64 : 32; }

template <class T>
__global__ void __launch_bounds__(256) slab_turn_kernel(const cx<T>* __restrict__ src, TurnTargets<T> dst, int S) {
    constexpr int TL = turn_tile<T>();
    __shared__ cx<T> tile[TL][TL + 1];
    const int g = blockIdx.z;
    const cx<T>* s = src + long(g) * S * S;
    cx<T>* d = dst.p[g];
    const int x0 = blockIdx.x * TL, y0 = blockIdx.y * TL;
#pragma unroll
    for (int k = threadIdx.y; k < TL; k += 8)
#pragma unroll
        for (int c = 0; c < TL; c += 32) {
            const int y = y0 + k, x = x0 + c + threadIdx.x;
            if (y < S && x < S) tile[k][c + threadIdx.x] = s[long(y) * S + x];
        }
    __syncthreads();
#pragma unroll
    for (int k = threadIdx.y; k < TL; k += 8)
#pragma unroll
        for (int c = 0; c < TL; c += 32) {
            const int y = x0 + k, x = y0 + c + threadIdx.x;
            if (y < S && x < S) d[long(y) * S + x] = tile[c + threadIdx.x][k];
        }
}

template <class T, int N, int MODE>
cudaError_t slab_launch_m(const SlabArgs<T>& a, cudaStream_t st) {
    using Sh = SlabShape<T, N>;
    if (cudaError_t e = ensure_smem_attr<slab_kernel<T, N, MODE>>(Sh::SMEM); e != cudaSuccess) return e;
    // persistent grid: CTAs resident at once, capped by the line groups
    const int resident = resident_ctas<slab_kernel<T, N, MODE>>(Sh::THREADS, Sh::SMEM);
    const int grid = std::min(resident, (a.R + Sh::LINES - 1) / Sh::LINES);
    slab_kernel<T, N, MODE><<<grid, Sh::THREADS, Sh::SMEM, st>>>(a);
    return cudaGetLastError();
}

template <class T, int N>
cudaError_t slab_launch_n(const SlabArgs<T>& a, int mode, cudaStream_t st) {
    switch (mode) {
        case SLAB_INIT: return slab_launch_m<T, N, SLAB_INIT>(a, st);
        case SLAB_HOLO:
            return a.p.quantize ? slab_launch_m<T, N, SLAB_HOLO_SNAP>(a, st) : slab_launch_m<T, N, SLAB_HOLO>(a, st);
        case SLAB_GS: return slab_launch_m<T, N, SLAB_GS>(a, st);
        case SLAB_FINAL: return slab_launch_m<T, N, SLAB_FINAL>(a, st);
        case SLAB_INV: return slab_launch_m<T, N, SLAB_INV>(a, st);
        case SLAB_FWD: return slab_launch_m<T, N, SLAB_FWD>(a, st);
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
