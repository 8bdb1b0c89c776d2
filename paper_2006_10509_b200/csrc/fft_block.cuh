// Register/shared-memory FFT of one line (row or column) of N points.
//
// Layout contract ("strided-natural"): the TF = N/E threads that own a line
// each hold E elements, thread t holding v[r] = x[t + r*TF]. run_fft()
// consumes and produces that layout, so a forward transform can feed an
// inverse transform register-to-register (the replay-plane projection of GS
// sits between them) and global loads/stores are unit stride across t.
//
// Algorithm: Stockham auto-sort, radix E (E in {2,4,8,16}) per stage with a
// smaller final radix when log2(N) is not a multiple of log2(E). Butterflies
// are fully unrolled with compile-time roots of unity; inter-stage twiddles
// come from an N-entry table tw[k] = exp(-2 pi i k / N) built in fp64 on the
// host (conjugated for the inverse). Stages exchange through shared memory
// stored as split re/im arrays with one pad word per 128 bytes (complex64) or
// as padded interleaved double2 (complex128).
#pragma once
#include <type_traits>
#include "cx.cuh"

namespace cgh {

// ---------------------------------------------------------------- radix DFTs
// In-place DFT of R points v[0], v[S], ..., v[(R-1)S]; natural-order output.
template <int R, int DIR, int S, class T>
struct Dft;

template <int DIR, int S, class T>
struct Dft<1, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>*) {}
};

template <int DIR, int S, class T>
struct Dft<2, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>* v) {
        cx<T> a = v[0], b = v[S];
        v[0] = a + b;
        v[S] = a - b;
    }
};

template <int DIR, int S, class T>
struct Dft<4, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>* v) {
        cx<T> a = v[0] + v[2 * S], b = v[0] - v[2 * S];
        cx<T> c = v[S] + v[3 * S], d = rot90<DIR>(v[S] - v[3 * S]);
        v[0] = a + c;
        v[2 * S] = a - c;
        v[S] = b + d;
        v[3 * S] = b - d;
    }
};

// complex64: b +- DIR i d as one FFMA2 each (the swap and the signs are
// operand modifiers), the other butterflies as FADD2
template <int DIR, int S>
struct Dft<4, DIR, S, float> {
    __device__ __forceinline__ static void run(cx<float>* v) {
        const cx<float> a = v[0] + v[2 * S], b = v[0] - v[2 * S];
        const cx<float> c = v[S] + v[3 * S], d = v[S] - v[3 * S];
        v[0] = a + c;
        v[2 * S] = a - c;
        // DIR < 0: b + (d.y, -d.x) ; DIR > 0: b + (-d.y, d.x)
        const float sp = DIR < 0 ? 1.0f : -1.0f;
        const unsigned long long ds = f2::pack(mk(d.y, d.x)), bb = f2::pack(b);
        v[S] = f2::unpack(f2::fma(ds, f2::pack(mk(sp, -sp)), bb));
        v[3 * S] = f2::unpack(f2::fma(ds, f2::pack(mk(-sp, sp)), bb));
    }
};

// R = R1 * R2 split ("four-step in registers"): n = R2*n1 + n2, k = k1 + R1*k2.
template <int R1, int R2, int DIR, int S, class T>
struct DftSplit {
    template <int N2>
    __device__ __forceinline__ static void inner(cx<T>* v) {
        if constexpr (N2 < R2) {
            Dft<R1, DIR, S * R2, T>::run(v + S * N2);   // over n1, stride R2
            twiddle<N2, 1>(v);
            inner<N2 + 1>(v);
        }
    }
    template <int N2, int K1>
    __device__ __forceinline__ static void twiddle(cx<T>* v) {
        if constexpr (K1 < R1) {
            v[S * (N2 + R2 * K1)] = mul_root<T, DIR, long(N2) * K1, long(R1) * R2>(v[S * (N2 + R2 * K1)]);
            twiddle<N2, K1 + 1>(v);
        }
    }
    template <int K1>
    __device__ __forceinline__ static void outer(cx<T>* v) {
        if constexpr (K1 < R1) {
            Dft<R2, DIR, S, T>::run(v + S * R2 * K1);   // over n2, contiguous block
            outer<K1 + 1>(v);
        }
    }
    __device__ __forceinline__ static void run(cx<T>* v) {
        inner<0>(v);
        outer<0>(v);
        // element (k1, k2) now at index R2*k1 + k2; natural index k1 + R1*k2
        cx<T> tmp[R1 * R2];
#pragma unroll
        for (int i = 0; i < R1 * R2; ++i) tmp[i] = v[S * i];
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) v[S * (k1 + R1 * k2)] = tmp[R2 * k1 + k2];
    }
};

template <int DIR, int S, class T>
struct Dft<8, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>* v) { DftSplit<2, 4, DIR, S, T>::run(v); }
};
template <int DIR, int S, class T>
struct Dft<16, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>* v) { DftSplit<4, 4, DIR, S, T>::run(v); }
};
template <int DIR, int S, class T>
struct Dft<32, DIR, S, T> {
    __device__ __forceinline__ static void run(cx<T>* v) { DftSplit<4, 8, DIR, S, T>::run(v); }
};

// --------------------------------------------------------------- line FFT
__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// Twiddle sources: the N-entry global table tw[k] = exp(-2 pi i k / N), or a
// two-level shared-memory table (w^k = hi[k >> sh] * lo[k & (2^sh - 1)], two
// tables of sqrt(N) entries; one extra rounding) for long lines whose N-entry
// table does not stay in L1.
template <class T>
struct TwSplit {
    const cx<T>* hi;
    const cx<T>* lo;
    int sh;
};
template <class T>
__device__ __forceinline__ cx<T> tw_at(const cx<T>* __restrict__ tw, int k) {
    return ldg_cx(tw + k);
}
template <class T>
__device__ __forceinline__ cx<T> tw_at(const TwSplit<T>& s, int k) {
    return cmul(s.hi[k >> s.sh], s.lo[k & ((1 << s.sh) - 1)]);
}

// Elements per thread for a line of N points at precision T.
// (complex128 at 4 points per thread, 512-thread lines: C3 fp64 74 vs 53 ms)
template <class T, int N>
struct LineShape {
    static constexpr int EMAX = sizeof(T) == 8 ? 8 : 16;
    static constexpr int E = N < EMAX ? N : EMAX;
    static constexpr int TF = N / E;   // threads per line
};

// Shared-memory words per line (split re/im, padded). complex128 lines are
// exchanged as interleaved double2 (one 16-B access per element, half the
// shared-memory instructions of split 8-B re/im words) with one pad element
// per 8 (128 B): the same 2 * line_words doubles hold either layout.
template <class T>
__host__ __device__ constexpr int pad_unit() { return sizeof(T) == 8 ? 8 : 128 / int(sizeof(T)); }
__device__ __forceinline__ int padc2(int i) { return i + (i >> 3); }
template <class T>
__device__ __forceinline__ int padx(int i) { return i + i / pad_unit<T>(); }
// (complex128: the +4 makes a line's double2 region span 4 mod 8 16-B slots,
// so the lanes of two lines interleaved in one warp (column passes) fall in
// opposite halves of the banks)
template <class T, int N>
__host__ __device__ constexpr int line_words() { return N + N / pad_unit<T>() + (sizeof(T) == 8 ? 4 : 1); }

template <class T, int N, int DIR, int EE = LineShape<T, N>::E>
struct LineFft {
    static constexpr int E = EE;   // elements per thread (default LineShape)
    static constexpr int TF = N / E;

    template <int NS, class TWS>
    __device__ __forceinline__ static void stages(cx<T> (&v)[E], T* sre, T* sim, int t, const TWS& tw) {
        constexpr int R = (N / NS >= E) ? E : N / NS;
        constexpr int NB = E / R;
        // v[b*R + r] = x_s[j + r*N/R], j = t + b*TF
        if constexpr (NS > 1) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int j = t + b * TF;
                const int jm = j & (NS - 1);
                if constexpr (std::is_same<TWS, TwSplit<T>>::value) {
                    // split table: look up w^r for r = 1, 5, 9, ... and step the
                    // three powers in between by w (at most 3 extra roundings;
                    // a quarter of the shared-memory lookups)
                    const int k = jm * (N / (NS * R));
                    const cx<T> w1 = tw_at<T>(tw, k);
                    cx<T> w = w1;
#pragma unroll
                    for (int r = 1; r < R; ++r) {
                        if (r > 1) w = (r & 3) == 1 ? tw_at<T>(tw, k * r) : cmul(w, w1);
                        v[b * R + r] = DIR < 0 ? cmul(v[b * R + r], w) : cmulc(v[b * R + r], w);
                    }
                } else {
#pragma unroll
                    for (int r = 1; r < R; ++r) {
                        cx<T> w = tw_at<T>(tw, jm * r * (N / (NS * R)));
                        v[b * R + r] = DIR < 0 ? cmul(v[b * R + r], w) : cmulc(v[b * R + r], w);
                    }
                }
            }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) Dft<R, DIR, 1, T>::run(&v[b * R]);

        if constexpr (NS * R == N) {
            // last stage: output X[t + b*TF + r*N/R] = strided index (b + r*NB)
            if constexpr (NB > 1) {
                cx<T> tmp[E];
#pragma unroll
                for (int i = 0; i < E; ++i) tmp[i] = v[i];
#pragma unroll
                for (int b = 0; b < NB; ++b)
#pragma unroll
                    for (int r = 0; r < R; ++r) v[b + r * NB] = tmp[b * R + r];
            }
        } else {
            __syncthreads();
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int j = t + b * TF;
                const int base = (j / NS) * NS * R + (j & (NS - 1));
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if constexpr (sizeof(T) == 8) {
                        reinterpret_cast<double2*>(sre)[padc2(base + r * NS)] =
                            make_double2(v[b * R + r].x, v[b * R + r].y);
                    } else {
                        const int p = padx<T>(base + r * NS);
                        sre[p] = v[b * R + r].x;
                        sim[p] = v[b * R + r].y;
                    }
                }
            }
            __syncthreads();
            constexpr int R2 = (N / (NS * R) >= E) ? E : N / (NS * R);
            constexpr int NB2 = E / R2;
#pragma unroll
            for (int b = 0; b < NB2; ++b)
#pragma unroll
                for (int r = 0; r < R2; ++r) {
                    if constexpr (sizeof(T) == 8) {
                        const double2 z = reinterpret_cast<const double2*>(sre)[padc2(t + b * TF + r * (N / R2))];
                        v[b * R2 + r] = mk<T>(z.x, z.y);
                    } else {
                        const int p = padx<T>(t + b * TF + r * (N / R2));
                        v[b * R2 + r] = mk(sre[p], sim[p]);
                    }
                }
            stages<NS * R>(v, sre, sim, t, tw);
        }
    }

    // Transform one line held in strided-natural layout (unscaled).
    __device__ __forceinline__ static void run(cx<T> (&v)[E], T* sre, T* sim, int t, const cx<T>* __restrict__ tw) {
        stages<1>(v, sre, sim, t, tw);
    }
    __device__ __forceinline__ static void run(cx<T> (&v)[E], T* sre, T* sim, int t, const TwSplit<T>& tw) {
        stages<1>(v, sre, sim, t, tw);
    }
};

}  // namespace cgh
