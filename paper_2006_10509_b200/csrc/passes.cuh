// Row and column passes of the 2-D transforms with the GS / OSPR pointwise
// work fused in.
//
// Image layout in HBM: row-major H x W complex<T> (T = float | double), the
// replay plane kept UNCENTRED (the reference's fftshift/ifftshift are folded
// into a pre-shifted target plane, built once per run by prep_target).
//
// Row pass (line = image row, W points, TF_W threads per row, several rows per
// CTA) and column pass (line = image column, H points, TF_H threads per
// column, C columns per CTA with the C columns adjacent across lanes so every
// load/store instruction touches C*sizeof(cx<T>) contiguous bytes per row).
#pragma once
#include "cx.cuh"
#include "fft_block.cuh"
#include "pcg64.cuh"

namespace cgh {

// ------------------------------------------------------------------ params
struct SchemeDev {
    int kind;        // 0 phase-only, 1 amplitude-only, 2 multi-amp
    int n;           // number of states
    double offset;   // phase-only: phase_offset
    double step;     // phase-only: 2*pi/levels (as numpy computes it)
    const double* states64;  // interleaved complex128 states (device)
    const float* states32;   // interleaved complex64 states (device)
};

struct ReduceArgs {
    double* partials;     // [nq][nblocks]
    unsigned* counter;    // zero-initialised ticket
    double* out;          // destination of the reduced values / error
    const double* denom;  // masked sum of t^2 (device scalar)
    int rescale;
};

template <class T>
struct PassArgs {
    cx<T>* data;              // frames of H*W
    long frame_stride;        // elements between frames
    int H, W;
    const T* tgt;             // ifftshifted |target|, sign bit = outside mask
    const T* beam;            // |illumination| (H*W, hologram plane) or nullptr
    const cx<T>* tw_row;      // W-entry exp(-2 pi i k / W)
    const cx<T>* tw_col;      // H-entry exp(-2 pi i k / H)
    const cx<T>* q_row;       // Fresnel factor per row m (H entries) or nullptr
    const cx<T>* q_col;       // Fresnel factor per column n (W entries)
    SchemeDev scheme;
    T gain;
    T scale;                  // 1/sqrt(H*W)
    int quantize;             // hologram projection snaps to the state set
    void* idx_out;            // index plane(s) (frame stride H*W) or nullptr
    cx<T>* field_out;         // hologram-plane field before snapping (H*W) or nullptr
    int idx_bytes;            // 1 or 4
    Pcg64 rng;                // GS init stream (already at draw 0)
    const Pcg64* frame_rng;   // OSPR: per-frame streams
    int frame0, frames;       // OSPR accumulation range [frame0, frame0+frames)
    int nframes_total;        // OSPR total frames of the run (for efficiency)
    T* intensity;             // OSPR carried intensity (H*W) or nullptr
    int load_intensity, store_intensity;
    ReduceArgs red;
};

// ------------------------------------------------------------------ helpers
template <class T>
__device__ __forceinline__ T dev_sqrt(T x) { return sqrt(x); }
template <>
__device__ __forceinline__ float dev_sqrt<float>(float x) { return sqrtf(x); }

template <class T>
__device__ __forceinline__ cx<T> state_value(const SchemeDev& s, int i) {
    if constexpr (sizeof(T) == 8) return mk<T>(s.states64[2 * i], s.states64[2 * i + 1]);
    else return mk<T>(s.states32[2 * i], s.states32[2 * i + 1]);
}

// numpy's float np.mod: result takes the sign of the divisor.
template <class T>
__device__ __forceinline__ T py_mod(T a, T b) {
    T m = fmod(a, b);
    if (m != T(0)) {
        if ((b < T(0)) != (m < T(0))) m += b;
    } else {
        m = copysign(T(0), b);
    }
    return m;
}

// Nearest state index (slm.py:86-108 in working precision T).
template <class T>
__device__ __forceinline__ int quantize_index(const SchemeDev& s, cx<T> z) {
    if (s.kind == 0) {
        const int L = s.n;
        const T ang = atan2(z.y, z.x);
        const T frac = py_mod<T>((ang - T(s.offset)) / T(s.step), T(L));
        const T lowf = floor(frac);
        const T rem = frac - lowf;
        // 0 <= frac < L, so 32-bit integer wrap-around gives the same indices
        // as the 64-bit form (and avoids 64-bit % on the GPU)
        const int low = int(lowf);
        const int high = low + 1 == L ? 0 : low + 1;
        int pick = rem < T(0.5) ? low : high;
        if (rem == T(0.5)) pick = low < high ? low : high;
        if (pick >= L) pick -= L;
        if (pick < 0) pick += L;
        return pick;
    }
    // generic nearest by Euclidean distance, first minimum wins
    int best = 0;
    T bd = T(0);
    if (s.kind == 1) {
        // real states k/(L-1): the nearest is a neighbour of x*(L-1)
        const int L = s.n;
        T pos = z.x * T(L - 1);
        int k0 = (int)floor(fmin(fmax(pos, T(0)), T(L - 1)));
        int lo = k0 > 0 ? k0 - 1 : 0, hi = k0 + 2 < L ? k0 + 2 : L - 1;
        best = lo;
        cx<T> sv = state_value<T>(s, lo);
        bd = hypot(z.x - sv.x, z.y - sv.y);
        for (int k = lo + 1; k <= hi; ++k) {
            sv = state_value<T>(s, k);
            T d = hypot(z.x - sv.x, z.y - sv.y);
            if (d < bd) {
                bd = d;
                best = k;
            }
        }
        return best;
    }
    cx<T> sv = state_value<T>(s, 0);
    bd = hypot(z.x - sv.x, z.y - sv.y);
    for (int k = 1; k < s.n; ++k) {
        sv = state_value<T>(s, k);
        T d = hypot(z.x - sv.x, z.y - sv.y);
        if (d < bd) {
            bd = d;
            best = k;
        }
    }
    return best;
}

// numpy's (beam + 0j) * e for a phasor e = (c, s) (algorithms.py:135,184,501:
// a real beam array times a complex array): (b c - 0 s, b s + 0 c). Given
// h = (b c, b s) this differs only where b == 0: the zero components then take
// their signs from IEEE zero addition, e.g. e in the second quadrant gives
// -0 + 0i, whose angle is pi (quantize_indices snaps it to the level at pi).
template <class T>
__device__ __forceinline__ cx<T> beam_zero_signs(T amp, cx<T> h) {
    return amp == T(0) ? mk(h.x - h.y, h.y + h.x) : h;
}

// Hologram-plane projection at pixel (m, n) of x = inverse-transform value
// (unscaled): h = beam * exp(i angle(x conj q)) [-> snap] -> h q.
// Mirrors algorithms.py:181-184 / 500-501 (propagate_inverse, angle, quantize).
// SNAP = false compiles out the snapping and field-export branches (callers
// that know a.quantize == 0 and a.field_out == nullptr).
template <class T, bool SNAP = true>
__device__ __forceinline__ cx<T> holo_project(const PassArgs<T>& a, cx<T> x, int m, int n, long frame_off) {
    cx<T> q;
    const bool fres = a.q_row != nullptr;
    if (fres) {
        q = cmul(a.q_row[m], a.q_col[n]);
        x = cmulc(x, q);
    }
    const T amp = a.beam ? a.beam[(long)m * a.W + n] : T(1);
    const T mag2 = x.x * x.x + x.y * x.y;
    cx<T> h;
    if (mag2 > T(0)) {
        T inv;
        if constexpr (sizeof(T) == 4) inv = amp * rsqrtf(mag2);   // as the fast row pass
        else inv = amp / dev_sqrt<T>(mag2);
        h = mk(x.x * inv, x.y * inv);
    } else {
        h = mk(amp, T(0));
    }
    if (SNAP) h = beam_zero_signs(amp, h);
    if (SNAP && a.field_out) a.field_out[(long)m * a.W + n] = h;
    if (SNAP && a.quantize) {
        const int k = quantize_index<T>(a.scheme, h);
        if (a.idx_out) {
            const long p = frame_off + (long)m * a.W + n;
            if (a.idx_bytes == 1) static_cast<uint8_t*>(a.idx_out)[p] = (uint8_t)k;
            else static_cast<int32_t*>(a.idx_out)[p] = k;
        }
        h = state_value<T>(a.scheme, k);
    }
    if (fres) h = cmul(h, q);
    return h;
}

// Deterministic block reduction of NQ doubles (fixed shuffle tree + fixed
// warp order). Result valid in thread 0.
template <int NQ>
__device__ __forceinline__ void block_reduce(double (&v)[NQ], double* sh /* >= 32*NQ */) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) sh[q * 32 + warp] = v[q];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double x = lane < nw ? sh[q * 32 + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
            v[q] = x;
        }
    }
}

// Publish this block's NQ partial sums; returns true in the block that
// arrives last (all partials then visible), with its ticket reset.
template <int NQ>
__device__ __forceinline__ bool publish_partials(const ReduceArgs& r, const double (&v)[NQ], int nblocks, int bid) {
    __shared__ int last;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) r.partials[(long)q * nblocks + bid] = v[q];
        __threadfence();
        const unsigned ticket = atomicAdd(r.counter, 1u);
        last = (ticket == unsigned(nblocks - 1));
    }
    __syncthreads();
    if (last) __threadfence();
    return last != 0;
}

// Fixed-order sum of quantity q over all blocks (whole block participates).
__device__ __forceinline__ double sum_partials(const ReduceArgs& r, int q, int nblocks, double* sh) {
    double acc[1] = {0.0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) acc[0] += __ldcg(&r.partials[(long)q * nblocks + b]);
    block_reduce<1>(acc, sh);
    __shared__ double bc;
    if (threadIdx.x == 0) bc = acc[0];
    __syncthreads();
    double out = bc;
    __syncthreads();
    return out;
}

// Masked amplitude error from the four sums (propagation.py:164-192):
// S_dd = sum d^2, S_rr = sum r^2, S_rd = sum r d (d = r - t, over the mask).
__device__ __forceinline__ double error_from_sums(double sdd, double srr, double srd, double denom, int rescale) {
    double num = sdd;
    if (rescale && srr > 0.0) num = sdd - (srd * srd) / srr;
    return num / denom;
}

// ------------------------------------------------------------------ modes
enum RowMode {
    ROW_FWD = 0,        // plain forward row FFT (fft2 API), optional scale
    ROW_INV = 1,        // plain inverse row FFT, optional scale
    ROW_HOLO = 2,       // inverse -> hologram projection -> forward  (GS, requantize)
    ROW_INIT = 3,       // random-phase start field -> projection -> forward
    ROW_OSPR_GEN = 4,   // random-phase sub-target (replay plane) -> inverse
    ROW_OSPR_ACC = 5,   // forward -> intensity accumulate -> per-frame error
};
enum ColMode {
    COL_FWD = 0,        // plain forward column FFT (fft2 API), optional scale
    COL_INV = 1,        // plain inverse column FFT
    COL_GS = 2,         // forward -> error sums + replay projection -> inverse
    COL_FINAL = 3,      // forward -> error + efficiency sums (no store)
    COL_HOLO = 4,       // inverse -> hologram projection (+index) -> forward (OSPR K2)
};

}  // namespace cgh
