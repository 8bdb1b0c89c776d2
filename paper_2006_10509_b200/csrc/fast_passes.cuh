// Pipelined GS passes for complex64 (the fp32 fast path, N in 256..4096).
//
// Persistent CTAs (one per SM, 512 threads) pull line tiles from a dynamic
// tile counter. Each tile is brought into shared memory by the bulk-copy /
// tensor-memory accelerator (rows: one 1-D cp.async.bulk of LINES contiguous
// rows; columns: a 2-D tensor map box of C columns x 256 rows, repeated down
// the column) with two tile slots, so the next tile streams in from HBM/L2
// while the current one is transformed. The per-thread Stockham twiddles are
// loaded once per kernel into registers and shared by the forward and inverse
// transforms; the exchange buffer is the tile slot itself (padded layout).
//
// Row pass (hologram plane, non-snapping iterations): inverse row FFT ->
// h = beam * x / |x| -> forward row FFT. The Fresnel chirp cancels exactly in
// this projection (|q| = 1: beam e^{i arg(x conj q)} q = beam x/|x|), so it is
// applied only where x == 0 (reference: arg 0 -> beam * q).
// Column pass (replay plane): forward column FFT -> masked error sums and
// amplitude projection -> inverse column FFT.
#pragma once
#include "passes.cuh"
#include "tma.cuh"

namespace cgh {

constexpr int kFastThreads = 512;
constexpr int kFastBoxRows = 256;

__device__ __forceinline__ int padc(int i) { return i + (i >> 4); }   // 1 float2 per 16 (128 B)

template <int N>
struct FastShape {
    static constexpr int E = 16;
    static constexpr int TF = N / E;
    static constexpr int LINES = kFastThreads / TF;       // lines per tile
    // padded line (float2): 1 word per 16, plus 4 so that lines c = 0..3 of a
    // column tile start in different banks (LW = 4 mod 16)
    static constexpr int LW = N + N / 16 + 4;
    static constexpr int R1 = (N / 16 >= 16) ? 16 : N / 16;   // stage-2 radix
    static constexpr int NS2 = 16 * R1;
    static constexpr int R2 = N / NS2;                     // stage-3 radix (1 = none)
};

template <int N>
struct FastTw {
    cx<float> w1[16];   // stage 2 (NS = 16)
    cx<float> w2[16];   // stage 3 (NS = 16*R1)
};

template <int N>
__device__ __forceinline__ void fast_tw_init(FastTw<N>& tw, int t, const cx<float>* __restrict__ table) {
    using S = FastShape<N>;
    {
        constexpr int NS = 16, R = S::R1, NB = 16 / R;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = t + b * S::TF;
                tw.w1[b * R + r] = ldg_cx(table + (j & (NS - 1)) * r * (N / (NS * R)));
            }
    }
    if constexpr (S::R2 > 1) {
        constexpr int NS = S::NS2, R = S::R2, NB = 16 / R;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int j = t + b * S::TF;
                tw.w2[b * R + r] = ldg_cx(table + (j & (NS - 1)) * r * (N / (NS * R)));
            }
    }
}

// compile-time offset K added to a padded index whose base is 16-aligned in
// the low bits (K % 16 == 0) or has base % 16 == 0 and K < 16
template <int K>
__device__ __forceinline__ constexpr int padk() { return K + K / 16; }

// One Stockham stage (index algebra in fft_block.cuh). `pt` = padc(t): every
// read address is pt + constant, every write address padc(base_b) + constant.
template <int N, int DIR, int NS, int R, bool LAST>
__device__ __forceinline__ void fast_stage(cx<float> (&v)[16], float2* sm, int t, int pt, const cx<float>* tw) {
    using S = FastShape<N>;
    constexpr int NB = 16 / R;
    if constexpr (NS > 1) {
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int r = 1; r < R; ++r)
                v[b * R + r] = DIR < 0 ? cmul(v[b * R + r], tw[b * R + r]) : cmulc(v[b * R + r], tw[b * R + r]);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) Dft<R, DIR, 1, float>::run(&v[b * R]);
    if constexpr (LAST) {
        if constexpr (NB > 1) {
            cx<float> tmp[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) tmp[i] = v[i];
#pragma unroll
            for (int b = 0; b < NB; ++b)
#pragma unroll
                for (int r = 0; r < R; ++r) v[b + r * NB] = tmp[b * R + r];
        }
    } else {
        __syncthreads();
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int j = t + b * S::TF;
            float2* wp = sm + padc((j / NS) * NS * R + (j & (NS - 1)));
#pragma unroll
            for (int r = 0; r < R; ++r) wp[r * NS + (r * NS) / 16] = make_float2(v[b * R + r].x, v[b * R + r].y);
        }
        __syncthreads();
        constexpr int RN = (N / (NS * R) >= 16) ? 16 : N / (NS * R);   // next radix
        constexpr int NBN = 16 / RN;
        const float2* rp = sm + pt;
#pragma unroll
        for (int b = 0; b < NBN; ++b)
#pragma unroll
            for (int r = 0; r < RN; ++r) {
                const float2 z = rp[(b * S::TF + r * (N / RN)) + (b * S::TF + r * (N / RN)) / 16];
                v[b * RN + r] = mk(z.x, z.y);
            }
    }
}

template <int N, int DIR>
__device__ __forceinline__ void fast_fft(cx<float> (&v)[16], float2* sm, int t, int pt, const FastTw<N>& tw) {
    using S = FastShape<N>;
    fast_stage<N, DIR, 1, 16, false>(v, sm, t, pt, nullptr);
    if constexpr (S::R2 > 1) {
        fast_stage<N, DIR, 16, S::R1, false>(v, sm, t, pt, tw.w1);
        fast_stage<N, DIR, S::NS2, S::R2, true>(v, sm, t, pt, tw.w2);
    } else {
        fast_stage<N, DIR, 16, S::R1, true>(v, sm, t, pt, tw.w1);
    }
}

struct FastArgs {
    float2* data;                 // H x W complex64, row-major
    int H, W;
    const float* beam;            // |illumination| (H*W) or nullptr
    const cx<float>* tw_row;      // W-entry table
    const cx<float>* tw_col;      // H-entry table
    const cx<float>* q_row;       // Fresnel factors (zero-magnitude fallback) or nullptr
    const cx<float>* q_col;
    const float* tgt_tiled;       // [W/C][H][C] shifted |T|, sign = outside mask
    float gain, scale;
    unsigned* tile_ctr;           // [0] tile counter, [1] finished CTAs
    ReduceArgs red;
};

// Tiles are assigned statically: CTA b handles tiles b, b + G, b + 2G, ...
template <int N>
struct FastSlots {
    static constexpr int ROW = FastShape<N>::LINES * FastShape<N>::LW;                            // float2
    static constexpr int COL = FastShape<N>::LINES * FastShape<N>::LW + FastShape<N>::LINES * N / 2;   // + target tile
};

// ================================================================ rows
template <int N>
__global__ void __launch_bounds__(kFastThreads, 1) fast_row_holo(FastArgs a) {
    using S = FastShape<N>;
    constexpr int TF = S::TF, LINES = S::LINES, LW = S::LW, SLOT = FastSlots<N>::ROW;
    constexpr uint32_t TILE_BYTES = uint32_t(LINES) * N * 8u;
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[2];
    const int tid = threadIdx.x, li = tid / TF, t = tid - li * TF;
    const int pt = padc(t);
    const int ntiles = a.H / LINES, G = gridDim.x;
    FastTw<N> tw;
    fast_tw_init<N>(tw, t, a.tw_row);
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_fence_init();
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int tile = blockIdx.x + s * G;
            if (tile < ntiles) {
                mbar_expect_tx(&full[s], TILE_BYTES);
                bulk_g2s(fsm + s * SLOT, a.data + size_t(tile) * LINES * N, TILE_BYTES, &full[s]);
            }
        }
    }
    __syncthreads();
    for (int it = 0;; ++it) {
        const int s = it & 1;
        const int tile = blockIdx.x + it * G;
        if (tile >= ntiles) break;
        float2* buf = fsm + s * SLOT;
        const int m = tile * LINES + li;
        mbar_wait(&full[s], (it >> 1) & 1);
        cx<float> v[16];
        const float2* src = buf + li * N + t;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = src[r * TF];
            v[r] = mk(z.x, z.y);
        }
        float2* line = buf + li * LW;
        fast_fft<N, +1>(v, line, t, pt, tw);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float amp = a.beam ? __ldg(a.beam + size_t(m) * N + t + r * TF) : 1.0f;
            const float m2 = v[r].x * v[r].x + v[r].y * v[r].y;
            if (m2 > 0.0f) {
                const float k = amp * rsqrtf(m2);
                v[r] = mk(v[r].x * k, v[r].y * k);
            } else {
                cx<float> h = mk(amp, 0.0f);
                if (a.q_row) h = cmul(h, cmul(a.q_row[m], a.q_col[t + r * TF]));
                v[r] = h;
            }
        }
        fast_fft<N, -1>(v, line, t, pt, tw);
        float2* dst = a.data + size_t(m) * N + t;
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * TF] = make_float2(v[r].x, v[r].y);
        fence_proxy_async();
        __syncthreads();
        const int nt = tile + 2 * G;
        if (tid == 0 && nt < ntiles) {
            mbar_expect_tx(&full[s], TILE_BYTES);
            bulk_g2s(buf, a.data + size_t(nt) * LINES * N, TILE_BYTES, &full[s]);
        }
    }
}

// ============================================================= columns
template <int N>
__global__ void __launch_bounds__(kFastThreads, 1) fast_col_gs(FastArgs a, const __grid_constant__ CUtensorMap tmap) {
    using S = FastShape<N>;
    constexpr int TF = S::TF, C = S::LINES, LW = S::LW, SLOT = FastSlots<N>::COL;
    constexpr uint32_t TILE_BYTES = uint32_t(C) * N * 8u;
    constexpr uint32_t TGT_BYTES = uint32_t(C) * N * 4u;
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ double rsh[32 * 4];
    const int tid = threadIdx.x, t = tid / C, c = tid - t * C;
    const int pt = padc(t);
    const int ntiles = a.W / C, G = gridDim.x;
    FastTw<N> tw;
    fast_tw_init<N>(tw, t, a.tw_col);
    auto issue = [&](int s, int tile) {
        mbar_expect_tx(&full[s], TILE_BYTES + TGT_BYTES);
#pragma unroll 1
        for (int y = 0; y < N; y += kFastBoxRows)
            tma_g2s_2d(fsm + s * SLOT + y * C, &tmap, 2 * tile * C, y, &full[s]);
        bulk_g2s(fsm + s * SLOT + C * LW, a.tgt_tiled + size_t(tile) * N * C, TGT_BYTES, &full[s]);
    };
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_fence_init();
#pragma unroll
        for (int s = 0; s < 2; ++s)
            if (blockIdx.x + s * G < ntiles) issue(s, blockIdx.x + s * G);
    }
    __syncthreads();
    double acc[4] = {0, 0, 0, 0};
    const float gain = a.gain, scale = a.scale;
    for (int it = 0;; ++it) {
        const int s = it & 1;
        const int tile = blockIdx.x + it * G;
        if (tile >= ntiles) break;
        float2* buf = fsm + s * SLOT;
        const float* tg = reinterpret_cast<const float*>(buf + C * LW) + t * C + c;
        mbar_wait(&full[s], (it >> 1) & 1);
        cx<float> v[16];
        const float2* src = buf + t * C + c;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = src[r * TF * C];
            v[r] = mk(z.x, z.y);
        }
        float2* line = buf + c * LW;
        fast_fft<N, -1>(v, line, t, pt, tw);
        float sdd = 0.f, srr = 0.f, srd = 0.f, sall = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float x = v[r].x * scale, y = v[r].y * scale;
            const float r2 = x * x + y * y;
            const float tt = tg[r * TF * C];
            const bool in = !signbit(tt);
            const float rr = sqrtf(r2);
            const float d = rr - tt;
            sall += r2;
            sdd += in ? d * d : 0.0f;
            srr += in ? r2 : 0.0f;
            srd += in ? rr * d : 0.0f;
            const float want = fmaxf(tt + gain * (tt - rr), 0.0f);
            const bool pos = rr > 0.0f;
            const float k = in ? (pos ? __fdividef(want, rr) : 0.0f) : 1.0f;
            v[r] = mk(x * k + ((in && !pos) ? want : 0.0f), y * k);
        }
        acc[0] += sdd;
        acc[1] += srr;
        acc[2] += srd;
        acc[3] += sall;
        fast_fft<N, +1>(v, line, t, pt, tw);
        float2* dst = a.data + size_t(tile) * C + c + size_t(t) * a.W;
        const size_t step = size_t(TF) * a.W;
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * step] = make_float2(v[r].x, v[r].y);
        fence_proxy_async();
        __syncthreads();
        const int nt = tile + 2 * G;
        if (tid == 0 && nt < ntiles) issue(s, nt);
    }
    block_reduce<4>(acc, rsh);
    const int nblocks = gridDim.x;
    if (publish_partials<4>(a.red, acc, nblocks, blockIdx.x)) {
        const double s_dd = sum_partials(a.red, 0, nblocks, rsh);
        const double s_rr = sum_partials(a.red, 1, nblocks, rsh);
        const double s_rd = sum_partials(a.red, 2, nblocks, rsh);
        const double s_all = sum_partials(a.red, 3, nblocks, rsh);
        if (threadIdx.x == 0) {
            a.red.out[0] = error_from_sums(s_dd, s_rr, s_rd, *a.red.denom, a.red.rescale);
            a.red.out[1] = s_all == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : s_rr / s_all;
            *a.red.counter = 0u;
        }
    }
}

// [W/C][H][C] copy of the row-major shifted target
__global__ void tile_target_kernel(const float* __restrict__ tgt, float* __restrict__ out, int H, int W, int C) {
    const long long total = (long long)H * W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total;
         p += (long long)gridDim.x * blockDim.x) {
        const int u = int(p / W), n = int(p - (long long)u * W);
        out[((long long)(n / C) * H + u) * C + (n % C)] = tgt[p];
    }
}

}  // namespace cgh
