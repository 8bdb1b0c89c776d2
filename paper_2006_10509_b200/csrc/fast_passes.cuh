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

constexpr int kFastBoxRows = 256;
constexpr long long kRowStagger = 4096;   // cycles; see fast_row_holo

// Start odd line groups kRowStagger cycles late (see fast_row_holo).
__device__ __forceinline__ void stagger_group(int g) {
    if (g & 1) {
        const long long t0 = clock64();
        while (clock64() - t0 < kRowStagger) {
        }
    }
}

__device__ __forceinline__ int padc(int i) { return i + (i >> 4); }   // 1 float2 per 16 (128 B)

template <int N, int TH>
struct FastShape {
    static constexpr int E = 16;
    static constexpr int TF = N / E;
    static constexpr int LINES = TH / TF;                  // lines per tile
    // padded line (float2): 1 word per 16, plus a stagger so that the lines
    // of a column tile interleaved in one warp start in disjoint bank ranges
    // (4 lines: LW = 4 mod 16; 2 lines: LW = 8 mod 16)
    static constexpr int LW = N + N / 16 + (LINES == 2 ? 8 : 4);
    static constexpr int R1 = (N / 16 >= 16) ? 16 : N / 16;   // stage-2 radix
    static constexpr int NS2 = 16 * R1;
    static constexpr int R2 = N / NS2;                     // stage-3 radix (1 = none)
};

// Per-thread Stockham twiddles in compact form: for each butterfly only the
// powers w, w^2, w^4, w^8 of its base root (exp(-2 pi i (j mod NS)/(NS R)))
// are kept in registers; w^r is formed from them with at most 3 complex
// products (<= ~4 ulp). Keeping all 29 twiddles made ptxas rematerialise them
// as global loads inside the butterflies (ncu: long-scoreboard stalls).
template <int N, int TH>
struct FastTw {
    cx<float> p1[4];        // stage 2 (NS = 16): powers 1, 2, 4, 8
    cx<float> p2[16 / 2][3];   // stage 3: per butterfly b, powers 1, 2, 4 (R2 <= 8) or see p2x
    cx<float> p2x[4];       // stage 3 with R2 == 16 (N = 4096): powers 1, 2, 4, 8 (NB = 1)
};

template <int N, int TH>
__device__ __forceinline__ void fast_tw_init(FastTw<N, TH>& tw, int t, const cx<float>* __restrict__ table) {
    using S = FastShape<N, TH>;
    {
        constexpr int NS = 16, R = S::R1;
        const int jm = t & (NS - 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) tw.p1[k] = ldg_cx(table + ((jm << k) * (N / (NS * R))) % N);
    }
    if constexpr (S::R2 > 1) {
        constexpr int NS = S::NS2, R = S::R2, NB = 16 / R;
        if constexpr (R == 16) {
            const int jm = t & (NS - 1);
#pragma unroll
            for (int k = 0; k < 4; ++k) tw.p2x[k] = ldg_cx(table + ((jm << k) * (N / (NS * R))) % N);
        } else {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                const int jm = (t + b * S::TF) & (NS - 1);
#pragma unroll
                for (int k = 0; k < 3; ++k) tw.p2[b][k] = ldg_cx(table + ((jm << k) * (N / (NS * R))) % N);
            }
        }
    }
}

// w^r from the stored powers (r compile-time, 1 <= r < 16)
template <int R>
__device__ __forceinline__ cx<float> pow_from(const cx<float>* p) {
    cx<float> w = mk(1.0f, 0.0f);
    bool first = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if ((R >> k) & 1) {
            w = first ? p[k] : cmul(w, p[k]);
            first = false;
        }
    }
    return w;
}

// compile-time offset K added to a padded index whose base is 16-aligned in
// the low bits (K % 16 == 0) or has base % 16 == 0 and K < 16
template <int K>
__device__ __forceinline__ constexpr int padk() { return K + K / 16; }

// One Stockham stage (index algebra in fft_block.cuh). `pt` = padc(t): every
// read address is pt + constant, every write address padc(base_b) + constant.
// named barrier over the threads sharing one exchange buffer
__device__ __forceinline__ void group_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Twiddle sources: per-thread registers (RegTw) or a shared-memory table
// laid out [r][j mod NS] (SmemTw; lanes read consecutive entries).
// compact register powers: stage with NB butterflies per thread, powers per b
struct PowTw {
    const cx<float>* p;   // p[b * stride + k]
    int stride;
};
struct RegTw {};

template <int DIR, int R, int NB, int RR>
__device__ __forceinline__ void apply_pow(cx<float> (&v)[16], const cx<float>* p, int b) {
    if constexpr (RR < R) {
        const cx<float> w = pow_from<RR>(p);
        v[b * R + RR] = DIR < 0 ? cmul(v[b * R + RR], w) : cmulc(v[b * R + RR], w);
        apply_pow<DIR, R, NB, RR + 1>(v, p, b);
    }
}

template <int DIR, int R, int NB>
__device__ __forceinline__ void apply_tw(cx<float> (&v)[16], const PowTw& tw, int) {
#pragma unroll
    for (int b = 0; b < NB; ++b) apply_pow<DIR, R, NB, 1>(v, tw.p + b * tw.stride, b);
}
template <int DIR, int R, int NB>
__device__ __forceinline__ void apply_tw(cx<float> (&v)[16], const RegTw&, int) {}
template <int NS_, int TF_>
struct SmemTw {
    const float2* tab;   // this stage's table [r][j mod NS]
};
template <int DIR, int R, int NB, int NS_, int TF_>
__device__ __forceinline__ void apply_tw(cx<float> (&v)[16], const SmemTw<NS_, TF_>& tw, int t) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int r = 1; r < R; ++r) {
            const float2 z = tw.tab[r * NS_ + ((t + b * TF_) & (NS_ - 1))];
            const cx<float> w = mk(z.x, z.y);
            v[b * R + r] = DIR < 0 ? cmul(v[b * R + r], w) : cmulc(v[b * R + r], w);
        }
}

template <int N, int TH, int DIR, int NS, int R, bool LAST, class TW, bool PRE = true>
__device__ __forceinline__ void fast_stage(cx<float> (&v)[16], float2* sm, int t, int pt, const TW& tw, int bid,
                                           int bcount) {
    using S = FastShape<N, TH>;
    constexpr int NB = 16 / R;
    if constexpr (NS > 1) apply_tw<DIR, R, NB>(v, tw, t);
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
    } else if (bid >= 0) {   // bid < 0: exchange skipped (timing experiments only)
        if constexpr (PRE) group_sync(bid, bcount);   // PRE = false: caller alternates buffers
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const int j = t + b * S::TF;
            float2* wp = sm + padc((j / NS) * NS * R + (j & (NS - 1)));
#pragma unroll
            for (int r = 0; r < R; ++r) wp[r * NS + (r * NS) / 16] = make_float2(v[b * R + r].x, v[b * R + r].y);
        }
        group_sync(bid, bcount);
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

template <int N, int TH, int DIR>
__device__ __forceinline__ void fast_fft(cx<float> (&v)[16], float2* sm, int t, int pt, const FastTw<N, TH>& tw,
                                         int bid = 0, int bcount = TH) {
    using S = FastShape<N, TH>;
    fast_stage<N, TH, DIR, 1, 16, false>(v, sm, t, pt, RegTw{}, bid, bcount);
    if constexpr (S::R2 > 1) {
        fast_stage<N, TH, DIR, 16, S::R1, false>(v, sm, t, pt, PowTw{tw.p1, 0}, bid, bcount);
        if constexpr (S::R2 == 16)
            fast_stage<N, TH, DIR, S::NS2, S::R2, true>(v, sm, t, pt, PowTw{tw.p2x, 0}, bid, bcount);
        else
            fast_stage<N, TH, DIR, S::NS2, S::R2, true>(v, sm, t, pt, PowTw{&tw.p2[0][0], 3}, bid, bcount);
    } else {
        fast_stage<N, TH, DIR, 16, S::R1, true>(v, sm, t, pt, PowTw{tw.p1, 0}, bid, bcount);
    }
}

// Number of shared-memory exchanges in one transform (2 for N > 256).
template <int N, int TH>
constexpr int fast_exchanges() { return FastShape<N, TH>::R2 > 1 ? 2 : 1; }

// Ping-pong variant: exchange e goes to buffer e & 1 with a single barrier
// (after the writes). A write into a buffer is safe once a barrier has passed
// after that buffer's last read, which holds when the caller keeps the
// buffers alternating across consecutive transforms.
template <int N, int TH, int DIR>
__device__ __forceinline__ void fast_fft_pp(cx<float> (&v)[16], float2* b0, float2* b1, int t, int pt,
                                            const FastTw<N, TH>& tw, int bid, int bcount) {
    using S = FastShape<N, TH>;
    if constexpr (S::R2 > 1) {
        fast_stage<N, TH, DIR, 1, 16, false, RegTw, false>(v, b0, t, pt, RegTw{}, bid, bcount);
        fast_stage<N, TH, DIR, 16, S::R1, false, PowTw, false>(v, b1, t, pt, PowTw{tw.p1, 0}, bid, bcount);
        if constexpr (S::R2 == 16)
            fast_stage<N, TH, DIR, S::NS2, S::R2, true>(v, b1, t, pt, PowTw{tw.p2x, 0}, bid, bcount);
        else
            fast_stage<N, TH, DIR, S::NS2, S::R2, true>(v, b1, t, pt, PowTw{&tw.p2[0][0], 3}, bid, bcount);
    } else {
        fast_stage<N, TH, DIR, 1, 16, false, RegTw, false>(v, b0, t, pt, RegTw{}, bid, bcount);
        fast_stage<N, TH, DIR, 16, S::R1, true>(v, b0, t, pt, PowTw{tw.p1, 0}, bid, bcount);
    }
}

// Shared-memory twiddle tables: stage 2 [R1][16], stage 3 [R2][NS2] (float2).
template <int N, int TH>
struct TwTables {
    using S = FastShape<N, TH>;
    static constexpr int T2 = S::R1 * 16;
    static constexpr int T3 = S::R2 > 1 ? S::R2 * S::NS2 : 0;
    static constexpr int WORDS = (T2 + T3 + 15) / 16 * 16;
    __device__ static void load(float2* tab, const cx<float>* __restrict__ table) {
        for (int i = threadIdx.x; i < T2; i += blockDim.x) {
            const int r = i / 16, jm = i % 16;
            const cx<float> z = ldg_cx(table + jm * r * (N / (16 * S::R1)));
            tab[i] = make_float2(z.x, z.y);
        }
        for (int i = threadIdx.x; i < T3; i += blockDim.x) {
            const int r = i / S::NS2, jm = i % S::NS2;
            const cx<float> z = ldg_cx(table + jm * r * (N / (S::NS2 * S::R2)));
            tab[T2 + i] = make_float2(z.x, z.y);
        }
    }
};

template <int N, int TH, int DIR>
__device__ __forceinline__ void fast_fft_s(cx<float> (&v)[16], float2* sm, int t, int pt, const float2* tab, int bid,
                                           int bcount) {
    using S = FastShape<N, TH>;
    fast_stage<N, TH, DIR, 1, 16, false>(v, sm, t, pt, RegTw{}, bid, bcount);
    if constexpr (S::R2 > 1) {
        fast_stage<N, TH, DIR, 16, S::R1, false>(v, sm, t, pt, SmemTw<16, S::TF>{tab}, bid, bcount);
        fast_stage<N, TH, DIR, S::NS2, S::R2, true>(v, sm, t, pt, SmemTw<S::NS2, S::TF>{tab + TwTables<N, TH>::T2},
                                                   bid, bcount);
    } else {
        fast_stage<N, TH, DIR, 16, S::R1, true>(v, sm, t, pt, SmemTw<16, S::TF>{tab}, bid, bcount);
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
    int debug;                    // experiments: 1 = no transforms, 2 = no loads/stores
};

// Programmatic dependent launch: the prologue (twiddles, barriers) of pass
// k+1 overlaps the tail of pass k; data is touched only after the wait.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Dynamic tile scheduling: thread 0 claims the tile for a slot one iteration
// early (the atomic's latency hides behind the transform); the last CTA to
// finish resets the counter for the next launch.
template <int N, int TH>
struct FastSlots {
    using S = FastShape<N, TH>;
    // float2 words per slot, rounded to 128 B (TMA destination alignment)
    static constexpr int ROW = (S::LINES * S::LW + 15) / 16 * 16;
    static constexpr int COL = (S::LINES * S::LW + S::LINES * N / 2 + 15) / 16 * 16;   // + target tile
};

__device__ __forceinline__ void finish_ctas(unsigned* ctr) {
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
            ctr[0] = 0u;
            ctr[1] = 0u;
        }
    }
}

// ================================================================ rows
// Each group of TF threads (one image row) runs its own two-slot bulk-copy
// pipeline with its own barriers and claims rows independently, so the
// groups of a CTA drift apart and overlap exchange and arithmetic phases.
template <int N, int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) fast_row_holo(FastArgs a) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, GROUPS = S::LINES, LW = S::LW;
    constexpr int SLOT = (LW + 15) / 16 * 16;   // one padded line, 128-B aligned
    constexpr uint32_t LINE_BYTES = uint32_t(N) * 8u;
    constexpr bool TWO = fast_exchanges<N, TH>() == 2;
    static_assert(TF % 32 == 0, "row groups must be whole warps");
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[GROUPS][2];
    __shared__ int lineq[GROUPS][2];
    const int tid = threadIdx.x, g = tid / TF, t = tid - g * TF;
    const bool lead = (t == 0);
    const int pt = padc(t);
    const int nlines = a.H;
    const int bid = 1 + g;
    const int fb = bid;
    float2* slots = fsm + g * 3 * SLOT;   // [slot 0][slot 1][exchange X]
    float2* xb = slots + 2 * SLOT;
    FastTw<N, TH> tw;
    fast_tw_init<N, TH>(tw, t, a.tw_row);
    if (lead) {
        mbar_init(&full[g][0], 1);
        mbar_init(&full[g][1], 1);
        mbar_fence_init();
    }
    pdl_wait();
    auto issue = [&](int s, int m) {
        if (a.debug & 2) {
            mbar_expect_tx(&full[g][s], 0);
        } else {
            mbar_expect_tx(&full[g][s], LINE_BYTES);
            bulk_g2s(slots + s * SLOT, a.data + size_t(m) * N, LINE_BYTES, &full[g][s]);
        }
    };
    if (lead) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int m = int(atomicAdd(a.tile_ctr, 1u));
            lineq[g][s] = m;
            if (m < nlines) issue(s, m);
        }
    }
    group_sync(bid, TF);
    // Odd row groups start ~2 us (a quarter of a line) late. Identical groups
    // launched together stay phase-aligned, so all of an SM's groups would hit
    // their shared-memory exchanges at the same time; offset, one group's
    // exchange overlaps another's butterflies (row pass 29.5 -> 27.6 us at
    // 2048^2; 2 and 4 us measured equal, 8 us worse).
    stagger_group(g);
    unsigned next = 0;
    if (lead) next = atomicAdd(a.tile_ctr, 1u);   // refill of slot 1 after line 0
    for (int it = 0;; ++it) {
        const int s = it & 1;
        const int m = lineq[g][s];
        if (m >= nlines) break;
        float2* line = slots + s * SLOT;
        mbar_wait(&full[g][s], (it >> 1) & 1);
        cx<float> v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = line[t + r * TF];
            v[r] = mk(z.x, z.y);
        }
        // Exchange buffers alternate X, line, X, line (X, line for one-exchange
        // sizes). The first exchange barrier also retires every read of the
        // other slot (previous line), so its refill is issued right after it.
        fast_stage<N, TH, +1, 1, 16, false, RegTw, false>(v, xb, t, pt, RegTw{}, fb, TF);
        if (it > 0 && lead) {
            const int nm = int(next);
            lineq[g][s ^ 1] = nm;
            if (nm < nlines) issue(s ^ 1, nm);
            next = atomicAdd(a.tile_ctr, 1u);
        }
        if constexpr (TWO) {
            fast_stage<N, TH, +1, 16, S::R1, false, PowTw, false>(v, line, t, pt, PowTw{tw.p1, 0}, fb, TF);
            if constexpr (S::R2 == 16)
                fast_stage<N, TH, +1, S::NS2, S::R2, true>(v, line, t, pt, PowTw{tw.p2x, 0}, fb, TF);
            else
                fast_stage<N, TH, +1, S::NS2, S::R2, true>(v, line, t, pt, PowTw{&tw.p2[0][0], 3}, fb, TF);
        } else {
            fast_stage<N, TH, +1, 16, S::R1, true>(v, xb, t, pt, PowTw{tw.p1, 0}, fb, TF);
        }
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
        if constexpr (TWO) fast_fft_pp<N, TH, -1>(v, xb, line, t, pt, tw, fb, TF);
        else fast_fft_pp<N, TH, -1>(v, line, xb, t, pt, tw, fb, TF);
        float2* dst = a.data + size_t(m) * N + t;
        if (!(a.debug & 2)) {
#pragma unroll
            for (int r = 0; r < 16; ++r) dst[r * TF] = make_float2(v[r].x, v[r].y);
        }
        fence_proxy_async();   // generic accesses to this slot before its async refill
    }
    pdl_trigger();
    __syncthreads();
    finish_ctas(a.tile_ctr);
}

// Row pass, occupancy variant: twiddles from a shared table, one slot per
// row group (latency hidden by more resident groups instead of a second slot).
template <int N, int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) fast_row_holo_s(FastArgs a) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, GROUPS = S::LINES, LW = S::LW;
    constexpr int SLOT = (LW + 15) / 16 * 16;
    constexpr uint32_t LINE_BYTES = uint32_t(N) * 8u;
    static_assert(TF % 32 == 0, "row groups must be whole warps");
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[GROUPS];
    __shared__ int lineq[GROUPS];
    const int tid = threadIdx.x, g = tid / TF, t = tid - g * TF;
    const bool lead = (t == 0);
    const int pt = padc(t);
    const int nlines = a.H;
    const int bid = 1 + g;
    float2* tab = fsm;
    float2* line = fsm + TwTables<N, TH>::WORDS + g * SLOT;
    TwTables<N, TH>::load(tab, a.tw_row);
    if (lead) {
        mbar_init(&full[g], 1);
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    if (lead) {
        const int m = int(atomicAdd(a.tile_ctr, 1u));
        lineq[g] = m;
        if (m < nlines) {
            mbar_expect_tx(&full[g], LINE_BYTES);
            bulk_g2s(line, a.data + size_t(m) * N, LINE_BYTES, &full[g]);
        }
    }
    group_sync(bid, TF);
    for (int it = 0;; ++it) {
        const int m = lineq[g];
        if (m >= nlines) break;
        unsigned next = 0;
        if (lead) next = atomicAdd(a.tile_ctr, 1u);
        mbar_wait(&full[g], it & 1);
        cx<float> v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = line[t + r * TF];
            v[r] = mk(z.x, z.y);
        }
        fast_fft_s<N, TH, +1>(v, line, t, pt, tab, bid, TF);
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
        fast_fft_s<N, TH, -1>(v, line, t, pt, tab, bid, TF);
        fence_proxy_async();
        group_sync(bid, TF);
        if (lead) {
            const int nm = int(next);
            lineq[g] = nm;
            if (nm < nlines) {
                mbar_expect_tx(&full[g], LINE_BYTES);
                bulk_g2s(line, a.data + size_t(nm) * N, LINE_BYTES, &full[g]);
            }
        }
        float2* dst = a.data + size_t(m) * N + t;
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * TF] = make_float2(v[r].x, v[r].y);
        group_sync(bid, TF);
    }
    pdl_trigger();
    __syncthreads();
    finish_ctas(a.tile_ctr);
}

// ============================================================= columns
// The target tile arrives pre-divided by the transform scale, so the replay
// projection works on unscaled column-FFT outputs; sums are rescaled once.
// MODE bit 0: rescale sums (S_rr, S_rd); bit 1: feedback gain != 0.
template <int N, int TH, int MINB, int MODE>
__global__ void __launch_bounds__(TH, MINB) fast_col_gs(FastArgs a, const __grid_constant__ CUtensorMap tmap) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, C = S::LINES, LW = S::LW, SLOT = FastSlots<N, TH>::COL;
    constexpr bool RESCALE = (MODE & 1) != 0, GAIN = (MODE & 2) != 0;
    constexpr uint32_t TILE_BYTES = uint32_t(C) * N * 8u;
    constexpr uint32_t TGT_BYTES = uint32_t(C) * N * 4u;
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ int tileq[2];
    __shared__ double rsh[32 * 4];
    const int tid = threadIdx.x, t = tid / C, c = tid - t * C;
    const int pt = padc(t);
    const int ntiles = a.W / C;
    FastTw<N, TH> tw;
    fast_tw_init<N, TH>(tw, t, a.tw_col);
    auto issue = [&](int s, int tile) {
        if (a.debug & 2) {   // timing experiment: no tile traffic
            mbar_expect_tx(&full[s], 0);
            return;
        }
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
    }
    pdl_wait();
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int tile = int(atomicAdd(a.tile_ctr, 1u));
            tileq[s] = tile;
            if (tile < ntiles) issue(s, tile);
        }
    }
    __syncthreads();
    const float gain = a.gain;
    const double sc2 = double(a.scale) * double(a.scale);
    for (int it = 0;; ++it) {
        const int s = it & 1;
        const int tile = tileq[s];
        if (tile >= ntiles) break;
        unsigned next = 0;
        if (tid == 0) next = atomicAdd(a.tile_ctr, 1u);
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
        fast_fft<N, TH, -1>(v, line, t, pt, tw);
        float sdd = 0.f, srr = 0.f, srd = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float x = v[r].x, y = v[r].y;
            const float r2 = x * x + y * y;
            const float ri = rsqrtf(r2);                       // inf at 0
            const float rr = r2 > 0.0f ? r2 * ri : 0.0f;
            const float tt = tg[r * TF * C];
            const bool in = !signbit(tt);
            const float d = rr - tt;
            sdd += in ? d * d : 0.0f;
            if constexpr (RESCALE) {
                srr += in ? r2 : 0.0f;
                srd += in ? rr * d : 0.0f;
            }
            float want = tt;
            if constexpr (GAIN) want = fmaxf(tt + gain * (tt - rr), 0.0f);
            const bool pos = r2 > 0.0f;
            const float k = in ? (pos ? want * ri : 0.0f) : 1.0f;
            v[r] = mk(x * k + ((in && !pos) ? want : 0.0f), y * k);
        }
        // per-tile sums -> global slot of this tile (fixed-order total at the end,
        // independent of which CTA claimed which tile)
        {
            double ts[3] = {double(sdd), double(srr), double(srd)};
            block_reduce<3>(ts, rsh);
            if (tid == 0) {
                a.red.partials[3 * size_t(tile) + 0] = ts[0] * sc2;
                a.red.partials[3 * size_t(tile) + 1] = ts[1] * sc2;
                a.red.partials[3 * size_t(tile) + 2] = ts[2] * sc2;
            }
        }
        fast_fft<N, TH, +1>(v, line, t, pt, tw);
        float2* dst = a.data + size_t(tile) * C + c + size_t(t) * a.W;
        const size_t step = size_t(TF) * a.W;
        if (!(a.debug & 2)) {
#pragma unroll
            for (int r = 0; r < 16; ++r) dst[r * step] = make_float2(v[r].x, v[r].y);
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            const int nt = int(next);
            tileq[s] = nt;
            if (nt < ntiles) issue(s, nt);
        }
    }
    pdl_trigger();
    __shared__ int last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = (atomicAdd(a.red.counter, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        const int lane = tid & 31, warp = tid >> 5;
        if (warp < 3) {
            double v = 0;
            for (int b = lane; b < ntiles; b += 32) v += __ldcg(&a.red.partials[3 * size_t(b) + warp]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) rsh[warp] = v;
        }
        __syncthreads();
        if (tid == 0) {
            a.red.out[0] = error_from_sums(rsh[0], rsh[1], rsh[2], *a.red.denom, RESCALE ? a.red.rescale : 0);
            a.red.out[1] = 0.0;   // efficiency is reported by the final (generic) pass only
            *a.red.counter = 0u;
            a.tile_ctr[0] = 0u;
            a.tile_ctr[1] = 0u;
        }
    }
}

// ====================================================== OSPR hologram columns
// K2 of OSPR (algorithms.py:500-503): per (subframe, column tile): inverse
// column FFT -> x conj(q) -> beam x/|x| -> snap (index plane) -> state q ->
// forward column FFT. Frames are stacked vertically in one tensor map.
struct FastHoloArgs {
    float2* data;                 // frames x H x W complex64
    int H, W, frames;
    const float* beam;
    const cx<float>* tw_col;
    const cx<float>* q_row;       // Fresnel factors or nullptr
    const cx<float>* q_col;
    SchemeDev scheme;
    uint8_t* idx;                 // frames x H x W, index planes (uint8 only)
    int binary;                   // PhaseOnly(2, offset 0): snap by the sign of Re
    unsigned* tile_ctr;
};

// PLAIN: binary scheme (PhaseOnly(2), offset 0), no illumination, Fourier
// propagation — the beam loads, chirp products and their null checks compile
// out, the two state values sit in registers. Same arithmetic as the general
// path for those inputs (bitwise identical planes).
template <int N, int TH, int MINB, bool PLAIN = false>
__global__ void __launch_bounds__(TH, MINB) fast_col_holo(FastHoloArgs a, const __grid_constant__ CUtensorMap tmap) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, C = S::LINES, LW = S::LW;
    constexpr int SLOT = (C * LW + 15) / 16 * 16;
    constexpr uint32_t TILE_BYTES = uint32_t(C) * N * 8u;
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[2];
    __shared__ int tileq[2];
    __shared__ float2 sst[256];   // state table (uint8 index planes: <= 256 states)
    const int tid = threadIdx.x, t = tid / C, c = tid - t * C;
    for (int k = tid; k < a.scheme.n && k < 256; k += TH) {
        const cx<float> z = state_value<float>(a.scheme, k);
        sst[k] = make_float2(z.x, z.y);
    }
    const int pt = padc(t);
    const int cgroups = a.W / C;
    const int ntiles = a.frames * cgroups;
    FastTw<N, TH> tw;
    fast_tw_init<N, TH>(tw, t, a.tw_col);
    auto issue = [&](int s, int tile) {
        const int f = tile / cgroups, cg = tile - f * cgroups;
        mbar_expect_tx(&full[s], TILE_BYTES);
#pragma unroll 1
        for (int y = 0; y < N; y += kFastBoxRows)
            tma_g2s_2d(fsm + s * SLOT + y * C, &tmap, 2 * cg * C, f * N + y, &full[s]);
    };
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_fence_init();
    }
    pdl_wait();
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            const int tile = int(atomicAdd(a.tile_ctr, 1u));
            tileq[s] = tile;
            if (tile < ntiles) issue(s, tile);
        }
    }
    __syncthreads();
    const bool fres = !PLAIN && a.q_row != nullptr;
    float2 st0 = make_float2(0.0f, 0.0f), st1 = st0;
    if constexpr (PLAIN) {
        st0 = sst[0];
        st1 = sst[1];
    }
    for (int it = 0;; ++it) {
        const int s = it & 1;
        const int tile = tileq[s];
        if (tile >= ntiles) break;
        unsigned next = 0;
        if (tid == 0) next = atomicAdd(a.tile_ctr, 1u);
        const int f = tile / cgroups, cg = tile - f * cgroups;
        const int n = cg * C + c;
        float2* buf = fsm + s * SLOT;
        mbar_wait(&full[s], (it >> 1) & 1);
        cx<float> v[16];
        const float2* src = buf + t * C + c;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = src[r * TF * C];
            v[r] = mk(z.x, z.y);
        }
        float2* line = buf + c * LW;
        fast_fft<N, TH, +1>(v, line, t, pt, tw);
        uint8_t* ip = a.idx + size_t(f) * N * a.W + n;
        if constexpr (PLAIN) {
            // amp = 1: h = x / |x| (1 + 0i for x = 0); k by the sign of Re h,
            // the reference formula when Re h == 0
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const cx<float> x = v[r];
                const float m2 = x.x * x.x + x.y * x.y;
                cx<float> h;
                if (m2 > 0.0f) {
                    const float k = rsqrtf(m2);
                    h = mk(x.x * k, x.y * k);
                } else {
                    h = mk(1.0f, 0.0f);
                }
                const int k = h.x != 0.0f ? (h.x < 0.0f ? 1 : 0) : quantize_index<float>(a.scheme, h);
                ip[size_t(t + r * TF) * a.W] = uint8_t(k);
                const float2 z = k ? st1 : st0;
                v[r] = mk(z.x, z.y);
            }
        }
        const cx<float> qn = fres ? a.q_col[n] : mk(1.0f, 0.0f);
#pragma unroll
        for (int r = 0; r < (PLAIN ? 0 : 16); ++r) {
            const int m = t + r * TF;
            cx<float> x = v[r];
            cx<float> q = mk(1.0f, 0.0f);
            if (fres) {
                q = cmul(a.q_row[m], qn);
                x = cmulc(x, q);
            }
            const float amp = a.beam ? __ldg(a.beam + size_t(m) * a.W + n) : 1.0f;
            const float m2 = x.x * x.x + x.y * x.y;
            cx<float> h;
            if (m2 > 0.0f) {
                const float k = amp * rsqrtf(m2);
                h = mk(x.x * k, x.y * k);
            } else {
                h = mk(amp, 0.0f);
            }
            h = beam_zero_signs(amp, h);
            int k;
            // PhaseOnly(2, 0): |arg| > pi/2 <=> Re < 0; Re == 0 (a zero beam's
            // signed zeros, or arg = +-pi/2 ties) takes the reference formula
            if (a.binary && h.x != 0.0f) k = h.x < 0.0f ? 1 : 0;
            else k = quantize_index<float>(a.scheme, h);
            ip[size_t(m) * a.W] = uint8_t(k);
            const float2 z = sst[k];   // shared copy: no dependent global load per pixel
            cx<float> sv = mk(z.x, z.y);
            if (fres) sv = cmul(sv, q);
            v[r] = sv;
        }
        fast_fft<N, TH, -1>(v, line, t, pt, tw);
        float2* dst = a.data + size_t(f) * N * a.W + n + size_t(t) * a.W;
        const size_t step = size_t(TF) * a.W;
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * step] = make_float2(v[r].x, v[r].y);
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            const int nt = int(next);
            tileq[s] = nt;
            if (nt < ntiles) issue(s, nt);
        }
    }
    pdl_trigger();
    __syncthreads();
    finish_ctas(a.tile_ctr);
}

// ============================================== OSPR replay rows: K1 and K3
// Jump of k steps of the PCG64 LCG as an affine map s -> A s + inc * G
// (A = MULT^k, G = sum_{i<k} MULT^i), independent of the stream increment.
struct LcgJump {
    u128 A, G;
};
__device__ __forceinline__ LcgJump lcg_jump(uint64_t k) {
    u128 acc_m = 1, acc_g = 0, cur_m = pcg_mult(), cur_g = 1;
    while (k) {
        if (k & 1) {
            acc_g = acc_g * cur_m + cur_g;
            acc_m *= cur_m;
        }
        cur_g = (cur_m + 1) * cur_g;
        cur_m *= cur_m;
        k >>= 1;
    }
    LcgJump j;
    j.A = acc_m;
    j.G = acc_g;
    return j;
}

// Start state of every (subframe, centred row) line: stream advanced by uc*W.
__global__ void ospr_line_states(const Pcg64* __restrict__ frame_rng, int frame0, int frames, int H, int W,
                                 Pcg64* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= frames * H) return;
    const int f = i / H, uc = i - f * H;
    Pcg64 g = frame_rng[frame0 + f];
    pcg_advance(g, uint64_t(uc) * uint64_t(W));
    out[i] = g;
}

struct FastOsprArgs {
    float2* data;                 // frames x H x W
    int H, W, frames;             // frames in this group (local index)
    int frame0, nframes_total;
    const float* tgt;             // row-major shifted |T|, sign = outside mask
    const Pcg64* line_state;      // [frames][H] line start states
    const cx<float>* tw_row;
    float scale;
    float* intensity;             // carried |R|^2 (H*W) or nullptr
    int load_intensity, store_intensity;
    double* line_part;            // K3: [frames*3 + 2][H] per-line partial sums
    unsigned* tile_ctr;
};

// sqrt.approx (one MUFU op, <= 2 ulp) for K3's perceived amplitudes: they
// only enter the error / efficiency sums, whose tolerance is 1e-3 relative
// (the IEEE sqrtf carried a slow-path branch per element: 12% of K3's stall
// samples were branch instructions, profiles/r02_ncu_ospr_c2_full.json)
__device__ __forceinline__ float sqrt_fast(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// K1: random-phase sub-target of row u (uncentred) -> inverse row FFT.
template <int N, int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) fast_ospr_gen(FastOsprArgs a) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, LW = S::LW;
    constexpr int SLOT = (LW + 15) / 16 * 16;
    static_assert(TF % 32 == 0, "row groups must be whole warps");
    extern __shared__ __align__(128) float2 fsm[];
    const int tid = threadIdx.x, g = tid / TF, t = tid - g * TF;
    const int pt = padc(t);
    const int bid = 1 + g;
    float2* line = fsm + g * SLOT;
    __shared__ int lineq[8];
    FastTw<N, TH> tw;
    fast_tw_init<N, TH>(tw, t, a.tw_row);
    // this thread's chunk of 16 draws in the row, as two chains of 8 (draws
    // 16t.. and 16t+8..): two independent 128-bit LCG recurrences per step
    // (the single chain was latency bound on its IMAD/IADD3 carries)
    const LcgJump jt = lcg_jump(uint64_t(16) * t), jt8 = lcg_jump(uint64_t(16) * t + 8);
    pdl_wait();
    stagger_group(g);
    const int nlines = a.frames * a.H;
    for (;;) {
        if (t == 0) lineq[g] = int(atomicAdd(a.tile_ctr, 1u));
        group_sync(bid, TF);
        const int ln = lineq[g];
        if (ln >= nlines) break;
        const int f = ln / a.H, u = ln - f * a.H;
        const int uc = (u + a.H / 2) % a.H;
        const Pcg64 s0 = a.line_state[f * a.H + uc];
        Pcg64 ga, gb;
        ga.state = jt.A * s0.state + s0.inc * jt.G;
        gb.state = jt8.A * s0.state + s0.inc * jt8.G;
        ga.inc = gb.inc = s0.inc;
        ga.has_uint32 = gb.has_uint32 = 0;
        ga.uinteger = gb.uinteger = 0;
        // uncentred columns of centred 16t..16t+15: 16 contiguous amplitudes
        const int p0 = (16 * t + N / 2) & (N - 1);
        const float4* t4 = reinterpret_cast<const float4*>(a.tgt + size_t(u) * N + p0);
        float amp[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 z = __ldg(t4 + q);
            amp[4 * q] = z.x;
            amp[4 * q + 1] = z.y;
            amp[4 * q + 2] = z.z;
            amp[4 * q + 3] = z.w;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float sa, ca, sb, cb;
            // angle / pi in [-1, 1); SFU sine / cosine (abs. error < 4e-7 on [-pi, pi])
            __sincosf(3.14159265358979f * pcg_next_halfturns(ga), &sa, &ca);
            __sincosf(3.14159265358979f * pcg_next_halfturns(gb), &sb, &cb);
            const float aa = fabsf(amp[e]), ab = fabsf(amp[e + 8]);
            line[padc(p0 + e)] = make_float2(aa * ca, aa * sa);
            line[padc(p0 + e + 8)] = make_float2(ab * cb, ab * sb);
        }
        group_sync(bid, TF);
        cx<float> v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const float2 z = line[pt + r * TF + (r * TF) / 16];
            v[r] = mk(z.x, z.y);
        }
        fast_fft<N, TH, +1>(v, line, t, pt, tw, bid, TF);
        float2* dst = a.data + (size_t(f) * a.H + u) * N + t;
#pragma unroll
        for (int r = 0; r < 16; ++r) dst[r * TF] = make_float2(v[r].x, v[r].y);
        group_sync(bid, TF);
    }
    pdl_trigger();
    __syncthreads();
    finish_ctas(a.tile_ctr);
}

// K3: row u of every subframe in the group: forward row FFT, running
// intensity sum, per-frame masked error partials of sqrt(I / i) -> per-line
// slots (fixed-order totals in ospr_line_reduce). Twiddles from a shared table.
template <int N, int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) fast_ospr_acc(FastOsprArgs a) {
    using S = FastShape<N, TH>;
    constexpr int TF = S::TF, LW = S::LW, GROUPS = S::LINES;
    constexpr int SLOT = (LW + 15) / 16 * 16;
    constexpr uint32_t LINE_BYTES = uint32_t(N) * 8u;
    constexpr int WPG = TF / 32;   // warps per group
    static_assert(TF % 32 == 0, "row groups must be whole warps");
    extern __shared__ __align__(128) float2 fsm[];
    __shared__ __align__(8) uint64_t full[GROUPS][2];
    __shared__ int lineq[GROUPS];
    __shared__ double wsum[GROUPS][WPG][3];
    const int tid = threadIdx.x, g = tid / TF, t = tid - g * TF;
    const int lane = t & 31, wg = t >> 5;
    const int pt = padc(t);
    const int bid = 1 + g;
    float2* tab = fsm;
    float2* slots = fsm + TwTables<N, TH>::WORDS + g * 2 * SLOT;
    TwTables<N, TH>::load(tab, a.tw_row);
    if (t == 0) {
        mbar_init(&full[g][0], 1);
        mbar_init(&full[g][1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    pdl_wait();
    stagger_group(g);
    const size_t fstride = size_t(a.H) * N;
    int uses[2] = {0, 0};
    for (;;) {
        if (t == 0) lineq[g] = int(atomicAdd(a.tile_ctr, 1u));
        group_sync(bid, TF);
        const int u = lineq[g];
        if (u >= a.H) break;
        const float* trow = a.tgt + size_t(u) * N + t;
        float tv[16], inten[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            tv[r] = trow[r * TF];
            inten[r] = a.load_intensity ? a.intensity[size_t(u) * N + t + r * TF] : 0.0f;
        }
        if (t == 0) {
#pragma unroll
            for (int s = 0; s < 2; ++s)
                if (s < a.frames) {
                    mbar_expect_tx(&full[g][s], LINE_BYTES);
                    bulk_g2s(slots + s * SLOT, a.data + size_t(s) * fstride + size_t(u) * N, LINE_BYTES, &full[g][s]);
                }
        }
        for (int f = 0; f < a.frames; ++f) {
            const int s = f & 1;
            float2* line = slots + s * SLOT;
            mbar_wait(&full[g][s], uses[s] & 1);
            uses[s] += 1;
            cx<float> v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float2 z = line[t + r * TF];
                v[r] = mk(z.x, z.y);
            }
            fast_fft_s<N, TH, -1>(v, line, t, pt, tab, bid, TF);
            const float inv_n = 1.0f / float(a.frame0 + f + 1);
            float sdd = 0.f, spp = 0.f, spd = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float x = v[r].x * a.scale, y = v[r].y * a.scale;
                inten[r] += x * x + y * y;
                const bool in = !signbit(tv[r]);
                const float p = sqrt_fast(inten[r] * inv_n);
                const float d = p - tv[r];
                sdd += in ? d * d : 0.f;
                spp += in ? p * p : 0.f;
                spd += in ? p * d : 0.f;
            }
            double w3[3] = {double(sdd), double(spp), double(spd)};
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w3[q] += __shfl_xor_sync(0xffffffffu, w3[q], o);
            if (lane == 0) {
                wsum[g][wg][0] = w3[0];
                wsum[g][wg][1] = w3[1];
                wsum[g][wg][2] = w3[2];
            }
            fence_proxy_async();
            group_sync(bid, TF);
            if (t == 0) {
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    double acc = 0;
                    for (int w = 0; w < WPG; ++w) acc += wsum[g][w][q];
                    a.line_part[(size_t(3 * f + q)) * a.H + u] = acc;
                }
                if (f + 2 < a.frames) {
                    mbar_expect_tx(&full[g][s], LINE_BYTES);
                    bulk_g2s(line, a.data + size_t(f + 2) * fstride + size_t(u) * N, LINE_BYTES, &full[g][s]);
                }
            }
            group_sync(bid, TF);
        }
        if (a.frame0 + a.frames == a.nframes_total) {
            const float inv_n = 1.0f / float(a.nframes_total);
            float sin_ = 0.f, sall = 0.f;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const float p = sqrt_fast(inten[r] * inv_n);
                const float pp = p * p;
                sall += pp;
                sin_ += !signbit(tv[r]) ? pp : 0.f;
            }
            double w2[2] = {double(sin_), double(sall)};
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w2[q] += __shfl_xor_sync(0xffffffffu, w2[q], o);
            if (lane == 0) {
                wsum[g][wg][0] = w2[0];
                wsum[g][wg][1] = w2[1];
            }
            group_sync(bid, TF);
            if (t == 0) {
                for (int q = 0; q < 2; ++q) {
                    double acc = 0;
                    for (int w = 0; w < WPG; ++w) acc += wsum[g][w][q];
                    a.line_part[(size_t(3 * a.frames + q)) * a.H + u] = acc;
                }
            }
        }
        if (a.store_intensity) {
#pragma unroll
            for (int r = 0; r < 16; ++r) a.intensity[size_t(u) * N + t + r * TF] = inten[r];
        }
        group_sync(bid, TF);
    }
    pdl_trigger();
    __syncthreads();
    finish_ctas(a.tile_ctr);
}

// Fixed-order totals of the per-line partials: one CTA per quantity.
__global__ void ospr_line_reduce(const double* __restrict__ line_part, int H, int frames, int frame0, int tail,
                                 int nframes_total, const double* __restrict__ denom, int rescale,
                                 double* __restrict__ out) {
    // block f < frames: frame error; block == frames: efficiency (tail only)
    const int f = blockIdx.x;
    __shared__ double sh[32 * 3];
    const int nq = (f < frames) ? 3 : 2;
    double acc[3] = {0, 0, 0};
    for (int u = threadIdx.x; u < H; u += blockDim.x)
        for (int q = 0; q < nq; ++q) acc[q] += line_part[size_t(3 * f + q) * H + u];
    block_reduce<3>(acc, sh);
    if (threadIdx.x == 0) {
        if (f < frames) out[frame0 + f] = error_from_sums(acc[0], acc[1], acc[2], *denom, rescale);
        else if (tail) out[nframes_total] = acc[1] == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : acc[0] / acc[1];
    }
}

// [W/C][H][C] copy of the row-major shifted target
__global__ void tile_target_kernel(const float* __restrict__ tgt, float* __restrict__ out, int H, int W, int C,
                                   float inv_scale) {
    const long long total = (long long)H * W;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total;
         p += (long long)gridDim.x * blockDim.x) {
        const int u = int(p / W), n = int(p - (long long)u * W);
        out[((long long)(n / C) * H + u) * C + (n % C)] = tgt[p] * inv_scale;   // sign (mask) preserved
    }
}

}  // namespace cgh
