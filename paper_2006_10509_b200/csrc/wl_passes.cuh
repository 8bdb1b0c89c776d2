// Warp-line GS passes for complex64 planes of 2048 x 2048 (config C3).
//
// One warp owns one line (a row in the hologram-plane pass, a column in the
// replay-plane pass) for the whole pass. The line lives in shared memory
// (16 KB, XOR-swizzled, no padding), so a CTA of 14 warps keeps 14 lines on
// chip: 148 SMs x 14 = 2072 >= 2048 lines, i.e. every line of a pass is
// resident at once (one wave, no tail) and the warps of a CTA never wait for
// each other except around the two stages they share with their group.
//
// Transforms (N = 2048 = 16 * 16 * 8), in place in shared memory:
//   first transform: decimation in frequency, natural order in, digit-reversed
//     order out: stage A (radix 16, stride 128, twiddle w^(j f1)), stage B
//     (radix 16, stride 8 inside each 128-block, twiddle w_128^(j' f2)),
//     stage C (radix 8 on 8 contiguous points). Position p then holds
//     frequency (p >> 7) + 16 ((p >> 3) & 15) + 256 (p & 7).
//   pointwise projection on the digit-reversed points (target / beam tables
//     are stored in that order, fp_perm_kernel), then the second transform as
//     decimation in time (stages C', B', A' mirrored), natural order out.
// Stages B..B' touch only the warp's own line (__syncwarp between stages);
// stage A reads the line from HBM/L2 and stage A' writes it back, both done
// jointly by a group of 4 (or 2) warps on 4 (2) adjacent lines, so every
// global access of a warp instruction covers whole 32-B sectors: the plane is
// stored column-tiled, element (m, n) at ((n >> 2) * N + m) * 4 + (n & 3)
// ("T4": 4 columns x N rows per 32 KB tile), so 4 adjacent columns of a row
// are one sector and 4 adjacent rows of a 4-column tile one 128-B line.
//
// Work: a CTA holds 3 quads (4 lines each) and 1 pair (2 lines); per round a
// grid of G CTAs covers 3G quads plus G pairs (the pairs take half a quad
// each). At G = 148: 444 + 74 = 518 >= 512 quads, one round.
//
// Arithmetic: packed complex64 (pcx.cuh, one f32x2 instruction per complex
// add / subtract, two per complex product): the passes are issue-bound, and
// the packed form halves the issue slots of the butterflies and twiddles.
#pragma once
#include "fft_block.cuh"
#include "passes.cuh"
#include "pcx.cuh"

namespace cgh {
namespace wl {

// programmatic dependent launch (as fast_passes.cuh)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr int N = 2048;
constexpr int NQUAD = N / 4;              // 4-line groups per pass
constexpr int LINES = 14;                 // line slots per CTA: 3 quads + 1 pair
// 16 warps: 4 per quad (one line each) and 4 for the pair (two per line, each
// half a line), so every SM sub-partition (warp w on SMSP w % 4) carries 3.5
// lines of work
constexpr int WARPS = 16;
constexpr int THREADS = 32 * WARPS;
constexpr size_t LINE_BYTES = size_t(N) * 8;
// slot g at g * (16 KB + 32 B): the 4 lines of a quad start 32 B apart in the
// bank space, so the joint stages (4 lines x 8 consecutive points per warp
// instruction) hit every bank pair exactly twice
constexpr size_t SLOT_BYTES = LINE_BYTES + 32;
// after the slots: stage-B twiddles w_128^(j' f) as [f - 1][j'] (15 x 8), each
// stored as {wx, wy, -wy, wy} (the broadcast and the pair of a packed product)
constexpr size_t TWB_OFF = size_t(LINES) * SLOT_BYTES;
constexpr size_t TWB_ENTRY = 16;
constexpr size_t SMEM = TWB_OFF + 15 * 8 * TWB_ENTRY;

enum { ROW = 0, COL = 1 };

// Timing experiments only (wrong results), compiled in with -DCGHB200_WL_DEBUG:
// Args::debug bit 0 skips stages B..B', bit 1 replaces the HBM/L2 traffic.
#ifdef CGHB200_WL_DEBUG
constexpr bool kDebug = true;
#else
constexpr bool kDebug = false;
#endif

__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 15); }

// swz(j + 128 f) for 0 <= j < 128: (j ^ ((j >> 4) & 7)) ^ 8 (f & 1), + 128 f.
// The base is taken through an opaque copy so the compiler recomputes it per
// chunk instead of keeping all stage-A addresses of the line live.
struct SwzA {
    int b0, b1;
    __device__ __forceinline__ explicit SwzA(int j) {
        int jj;
        asm volatile("mov.b32 %0, %1;" : "=r"(jj) : "r"(j));
        b0 = jj ^ ((jj >> 4) & 7);
        b1 = b0 ^ 8;
    }
    __device__ __forceinline__ int operator()(int f) const { return ((f & 1) ? b1 : b0) + 128 * f; }
};

__device__ __forceinline__ float2* slot(float2* sm, int g) {
    return reinterpret_cast<float2*>(reinterpret_cast<char*>(sm) + size_t(g) * SLOT_BYTES);
}

// T4 index of element (row m, column n).
__device__ __forceinline__ long t4(int m, int n) { return (long((n >> 2)) * N + m) * 4 + (n & 3); }

// T4 index step between points x and x + 128 of a line: rows (ROW pass: line
// = row, points along n) jump 32 tiles, columns (COL) 128 rows of a tile.
template <int PASS>
constexpr long kStep128 = PASS == 1 ? 128L * 4 : 32L * N * 4;
template <int PASS>
__device__ __forceinline__ long t4_line(int line, int x) { return PASS == 1 ? t4(x, line) : t4(line, x); }

// Natural frequency index of digit-reversed position p (see header).
__host__ __device__ __forceinline__ int natural(int p) { return (p >> 7) + 16 * ((p >> 3) & 15) + 256 * (p & 7); }

struct Args {
    float2* data;              // T4 plane
    const float* tgt_perm;     // COL: [N][N], column n, digit-reversed row position p; |T|*sqrt(HW), sign = outside mask
    const float* beam_perm;    // ROW: [N][N], row m, digit-reversed column position p; |illumination| (or nullptr)
    const cx<float>* tw;       // N-entry table exp(-2 pi i k / N)
    const cx<float>* q_row;    // Fresnel factors (zero-magnitude fallback of the row pass) or nullptr
    const cx<float>* q_col;
    float gain;
    float scale;               // 1/sqrt(HW)
    double* line_sums;         // COL: [N][3] per-line partial sums
    ReduceArgs red;
    long long* stamps;         // timing experiments: [grid][WARPS][8] globaltimer / clock64 pairs, or nullptr
    int no_stagger;            // timing experiments: both half-CTAs load at once
    int debug;                 // timing experiments (wrong results): 1 = skip stages B..B', 2 = no HBM/L2 traffic
};

// timing experiments (CGHB200_WL_STAMPS): lane 0 of each warp records the
// global timer and the SM clock at stage boundaries of its first round
__device__ __forceinline__ void stamp(const Args& a, int w, int mark) {
    if (a.stamps && (threadIdx.x & 31) == 0) {
        long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        long long* p = a.stamps + ((long(blockIdx.x) * WARPS + w) * 8 + mark) * 2;
        p[0] = g;
        p[1] = clock64();
    }
}

using pk::pc;

__device__ __forceinline__ unsigned saddr(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }

// global / shared 64-bit accesses of one complex64 value
__device__ __forceinline__ pc ldcg_pc(const float2* p) {
    return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ void stcg_pc(float2* p, pc v) { __stcg(reinterpret_cast<unsigned long long*>(p), v); }
__device__ __forceinline__ pc ldg_pc(const cx<float>* p) {
    return __ldg(reinterpret_cast<const unsigned long long*>(p));
}

// group geometry of warp `w` (0..15). Quads (groups 0..2): warp wi of the
// group owns line wi. Pair (group 3): warps wi = 2h + sub; sub picks the line,
// h the half: chunks [2h, 2h + 2) of the joint stages and of stages B / B',
// [4h, 4h + 4) of stage C (a half line, positions [1024 h, 1024 h + 1024),
// is self-contained from stage B to B').
template <int PASS>
struct Role {
    int grp, wi;       // group 0..2 quads, 3 pair; warp in group (0..3)
    int s, j0;         // joint stages: this thread's line in the group and butterfly base
    int own;           // slot / line offset in the group of this warp's stages B..B'
    int h;             // half (pair) or -1 (quad: whole line)
    __device__ Role(int w, int l) {
        grp = w >> 2;
        wi = w & 3;
        if (grp < 3) {
            h = -1;
            own = wi;
            if (PASS == COL) {
                s = l & 3;
                j0 = 8 * wi + (l >> 2);
            } else {
                s = (l >> 2) & 3;
                j0 = 8 * wi + 4 * (l >> 4) + (l & 3);
            }
        } else {
            h = wi >> 1;
            own = wi & 1;
            if (PASS == COL) {
                s = l & 1;
                j0 = 16 * (wi & 1) + (l >> 1);
            } else {
                s = (l >> 2) & 1;
                j0 = 16 * (wi & 1) + 4 * (l >> 3) + (l & 3);
            }
        }
    }
    __device__ int a_beg() const { return h < 0 ? 0 : 2 * h; }
    __device__ int a_cnt() const { return h < 0 ? 4 : 2; }
};

__device__ __forceinline__ void group_bar(int grp) {
    asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
}

// first line of this group in round `rb` (quads), or -1 if none
__device__ __forceinline__ int group_line0(int grp, int rb) {
    const int G = gridDim.x;
    if (grp < 3) {
        const int q = rb + 3 * blockIdx.x + grp;
        return q < NQUAD ? 4 * q : -1;
    }
    const int pairs = G & ~1;
    if (int(blockIdx.x) >= pairs) return -1;
    const int u = 2 * (rb + 3 * G) + blockIdx.x;   // pair unit: quad u >> 1, half u & 1
    return (u >> 1) < NQUAD ? 2 * u : -1;
}
__device__ __forceinline__ int round_len() {
    const int G = gridDim.x;
    return 3 * G + (G & ~1) / 2;
}

// t[f - 1] = tw[(base * f) mod N], f = 1..15 (loaded per stage: only the
// stage's own twiddles are live)
__device__ __forceinline__ void load_tw(pc (&t)[15], const cx<float>* __restrict__ tw, int base) {
#pragma unroll
    for (int f = 1; f < 16; ++f) t[f - 1] = ldg_pc(tw + ((base * f) & (N - 1)));
}

// ---- stage A (joint): load 16 points of butterfly j, radix 16, twiddle, store
template <int PASS, int D>
__device__ __forceinline__ void load_a(pc (&u)[16], const float2* __restrict__ data, int line, int j,
                                       int dbg = 0) {
    if (kDebug && (dbg & 2)) {
#pragma unroll
        for (int k = 0; k < 16; ++k) u[k] = pk::make(float(j), float(k));
        return;
    }
    const float2* p = data + t4_line<PASS>(line, j);
    // ROW: the 16 points are 2 MB apart: four base pointers 8 MB apart keep
    // every offset inside the immediate range
    const float2* pb[4];
    pb[0] = p;
#pragma unroll
    for (int q = 1; q < 4; ++q) {
        long off = 4 * kStep128<PASS>;
        if (PASS == ROW) asm volatile("" : "+l"(off));
        pb[q] = pb[q - 1] + off;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
        u[k] = ldcg_pc(PASS == ROW ? pb[k >> 2] + (k & 3) * kStep128<PASS> : p + k * kStep128<PASS>);
}

// w_64^f factors that advance the stage-A twiddles from chunk c to c + 1
// (j -> j + 32: w^(j f) -> w^(j f) w^(32 f)), table (forward) convention
template <int F = 1>
__device__ __forceinline__ void advance_tw(pc (&twA)[15]) {
    if constexpr (F < 16) {
        twA[F - 1] = pk::mul_root<-1, F, 64>(twA[F - 1]);
        advance_tw<F + 1>(twA);
    }
}

// ---- stage A (joint): per chunk c, butterfly j = j0 + 32 c: load its 16
// points (x = j + 128 k) from HBM/L2, radix 16, twiddle w^(j f), store to
// the line's slot. One code copy for the four chunks (instruction cache).
template <int PASS, int D>
__device__ __forceinline__ void stage_a(float2* line_sm, const float2* __restrict__ data, int line, int j0,
                                        pc (&twA)[15], int dbg, int cbeg, int cend) {
    // chunk c + 1's 16 loads are issued before chunk c is transformed, so the
    // L2 latency is paid once per stage instead of once per chunk
    pc nxt[16];
    load_a<PASS, D>(nxt, data, line, j0 + 32 * cbeg, dbg);
#pragma unroll 1
    for (int c = cbeg; c < cend; ++c) {
        const int j = j0 + 32 * c;
        pc u[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) u[k] = nxt[k];
        if (c + 1 < cend) load_a<PASS, D>(nxt, data, line, j + 32, dbg);
        pk::Dft<16, D, 1>::run(u);
#pragma unroll
        for (int f = 1; f < 16; ++f) u[f] = pk::cmul_d<D>(u[f], twA[f - 1]);
        const SwzA sa(j);
        pc* lp = reinterpret_cast<pc*>(line_sm);
#pragma unroll
        for (int f = 0; f < 16; ++f) lp[sa(f)] = u[f];
        if (c + 1 < cend) advance_tw(twA);
    }
}

// ---- stage A' (joint): load the 16 spectrum blocks of butterfly j, twiddle,
// radix 16, store to HBM/L2
template <int PASS, int D>
__device__ __forceinline__ void stage_a2(const float2* line_sm, float2* __restrict__ data, int line, int j0,
                                         pc (&twA)[15], int dbg, int cbeg, int cend) {
#pragma unroll 1
    for (int c = cbeg; c < cend; ++c) {
        const int j = j0 + 32 * c;
        pc u[16];
        const SwzA sa(j);
        const pc* lp = reinterpret_cast<const pc*>(line_sm);
#pragma unroll
        for (int f = 0; f < 16; ++f) u[f] = lp[sa(f)];
#pragma unroll
        for (int f = 1; f < 16; ++f) u[f] = pk::cmul_d<D>(u[f], twA[f - 1]);
        pk::Dft<16, D, 1>::run(u);
        if (c + 1 < cend) advance_tw(twA);
        float2* p = data + t4_line<PASS>(line, j);
        if (kDebug && (dbg & 2)) {   // timing: arithmetic kept, no stores
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (pk::re(u[k]) == 1234.5f) stcg_pc(p, u[k]);
            continue;
        }
        float2* pb[4];
        pb[0] = p;
#pragma unroll
        for (int q = 1; q < 4; ++q) {
            long off = 4 * kStep128<PASS>;
            if (PASS == ROW) asm volatile("" : "+l"(off));
            pb[q] = pb[q - 1] + off;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            stcg_pc(PASS == ROW ? pb[k >> 2] + (k & 3) * kStep128<PASS> : p + k * kStep128<PASS>, u[k]);
    }
}

// ---- shared-memory access with precomputed swizzled addresses
template <int OFF>
__device__ __forceinline__ pc lds(unsigned a) {
    pc v;
    asm volatile("ld.shared.b64 %0, [%1+%2];" : "=l"(v) : "r"(a), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ void sts(unsigned a, pc v) {
    asm volatile("st.shared.b64 [%0+%1], %2;" ::"r"(a), "n"(OFF), "l"(v) : "memory");
}
// stage-B twiddle entry {wx, wy, -wy, wy}: the broadcast wx and the pair wn
template <int OFF>
__device__ __forceinline__ void lds_tw(unsigned a, float& wx, pc& wn) {
    pc w0;
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2+%3];" : "=l"(w0), "=l"(wn) : "r"(a), "n"(OFF));
    wx = pk::re(w0);
}

// ---- stage B / B' (own line): radix 16 on stride 8 inside each 128-block.
// Butterfly (blk, j') of chunk c (blk = 4c + lane/8, j' = lane % 8) reads
// i = 128 blk + j' + 8k; with L = 8 ((lane >> 3) & 1) + j' its swizzled
// position is 128 blk + 16 (k >> 1) + (L ^ (8 (k & 1) + (k >> 1))): 16
// lane-dependent addresses, advanced by 4 KB per chunk; each access is one
// instruction with an immediate offset.
struct AddrB {
    unsigned r[16];
    __device__ __forceinline__ AddrB(const float2* line_sm, int lane) {
        const unsigned base = saddr(line_sm) + 8u * 128u * unsigned(lane >> 3);
        const int L = 8 * ((lane >> 3) & 1) + (lane & 7);
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] = base + 8u * unsigned(L ^ (8 * (k & 1) + (k >> 1)));
    }
    __device__ __forceinline__ void next() {
#pragma unroll
        for (int k = 0; k < 16; ++k) r[k] += 4096u;
    }
};

template <int OFF = 0, int K = 0>
__device__ __forceinline__ void ld16_b(pc (&u)[16], const AddrB& ad) {
    if constexpr (K < 16) {
        u[K] = lds<OFF + 128 * (K >> 1)>(ad.r[K]);
        ld16_b<OFF, K + 1>(u, ad);
    }
}
template <int OFF = 0, int K = 0>
__device__ __forceinline__ void st16_b(const pc (&u)[16], const AddrB& ad) {
    if constexpr (K < 16) {
        sts<OFF + 128 * (K >> 1)>(ad.r[K], u[K]);
        st16_b<OFF, K + 1>(u, ad);
    }
}

// twiddles of stage B from the shared table (lane j' reads row f: 8 distinct
// entries per instruction), applied to two chunks (one table read each)
template <int D, int F = 1>
__device__ __forceinline__ void twiddle_b2(pc (&u)[16], pc (&v)[16], unsigned tb) {
    if constexpr (F < 16) {
        float wx;
        pc wn;
        lds_tw<8 * int(TWB_ENTRY) * (F - 1)>(tb, wx, wn);
        u[F] = pk::cmul_d<D>(u[F], wx, wn);
        v[F] = pk::cmul_d<D>(v[F], wx, wn);
        twiddle_b2<D, F + 1>(u, v, tb);
    }
}

// FIRST: DIF stage (butterfly, then twiddle); else DIT stage (twiddle, then butterfly)
template <int D, bool FIRST>
__device__ __forceinline__ void stage_b_any(float2* line_sm, int lane, unsigned tb, int cbeg, int cend) {
    AddrB ad(line_sm, lane);
    for (int c = 0; c < cbeg; ++c) ad.next();
    // two chunks per step (their butterflies are independent): twice the
    // instruction-level parallelism per warp; chunk counts are even
#pragma unroll 1
    for (int c = cbeg; c < cend; c += 2) {
        pc u[16], v[16];
        ld16_b<0>(u, ad);
        ld16_b<4096>(v, ad);
        if constexpr (FIRST) {
            pk::Dft<16, D, 1>::run(u);
            pk::Dft<16, D, 1>::run(v);
        }
        twiddle_b2<D>(u, v, tb);
        if constexpr (!FIRST) {
            pk::Dft<16, D, 1>::run(u);
            pk::Dft<16, D, 1>::run(v);
        }
        st16_b<0>(u, ad);
        st16_b<4096>(v, ad);
        ad.next();
        ad.next();
    }
}
__device__ __forceinline__ unsigned twb_addr(const float2* wsm, int lane) {
    return saddr(reinterpret_cast<const char*>(wsm) + TWB_OFF) + unsigned(TWB_ENTRY) * unsigned(lane & 7);
}
template <int D>
__device__ __forceinline__ void stage_b(float2* line_sm, int lane, unsigned tb, int cbeg, int cend) {
    stage_b_any<D, true>(line_sm, lane, tb, cbeg, cend);
}
template <int D>
__device__ __forceinline__ void stage_b2(float2* line_sm, int lane, unsigned tb, int cbeg, int cend) {
    stage_b_any<D, false>(line_sm, lane, tb, cbeg, cend);
}
// fill the stage-B table (whole CTA, before the first pass)
__device__ __forceinline__ void init_twb(float2* wsm, const cx<float>* __restrict__ tw) {
    float4* t = reinterpret_cast<float4*>(reinterpret_cast<char*>(wsm) + TWB_OFF);
    for (int i = threadIdx.x; i < 120; i += blockDim.x) {
        const int f = i / 8 + 1, jp = i % 8;
        const cx<float> z = ldg_cx(tw + ((16 * jp * f) & (N - 1)));
        t[i] = make_float4(z.x, z.y, -z.y, z.y);
    }
}

// ---- stage C addresses: butterfly b = lane + 32c reads i = 8b + e, whose
// swizzled position is 8 (b ^ x3) + (e ^ x7) with x = (lane >> 1) & 15,
// x3 = x >> 3, x7 = x & 7: 8 lane-dependent addresses + 2048 B per chunk.
struct AddrC {
    unsigned r[8];
    __device__ __forceinline__ AddrC(const float2* line_sm, int lane) {
        const int x = (lane >> 1) & 15;
        const unsigned base = saddr(line_sm) + 8u * 8u * unsigned(lane ^ (x >> 3));
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = base + 8u * unsigned(e ^ (x & 7));
    }
    __device__ __forceinline__ void next() {
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] += 2048u;
    }
};
template <int OFF = 0, int E = 0>
__device__ __forceinline__ void ld8_c(pc (&u)[8], const AddrC& ad) {
    if constexpr (E < 8) {
        u[E] = lds<OFF>(ad.r[E]);
        ld8_c<OFF, E + 1>(u, ad);
    }
}
template <int OFF = 0, int E = 0>
__device__ __forceinline__ void st8_c(const pc (&u)[8], const AddrC& ad) {
    if constexpr (E < 8) {
        sts<OFF>(ad.r[E], u[E]);
        st8_c<OFF, E + 1>(u, ad);
    }
}

// ---- stage C pointwise step on the 8 spectrum points of one chunk (digit-
// reversed positions p0 .. p0 + 7, target / beam values tv)
template <int PASS, int MODE>
__device__ __forceinline__ void project8(const Args& a, pc (&u)[8], const float (&tv)[8], const float* tp, int p0,
                                         int myline, float& sdd, float& srr, float& srd) {
    constexpr bool RESCALE = (MODE & 1) != 0, GAIN = (MODE & 2) != 0, FULL = (MODE & 4) != 0;
    if constexpr (PASS == COL && FULL) {
        // every pixel inside the metric mask (MODE bit 2): no mask selects
        const float gain = a.gain;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float x = pk::re(u[e]), y = pk::im(u[e]);
            const float r2 = x * x + y * y;
            const bool pos = r2 > 0.0f;
            const float ri = pos ? rsqrtf(r2) : 0.0f;
            const float rr = r2 * ri;
            const float tt = tv[e];
            const float d = rr - tt;
            sdd = fmaf(d, d, sdd);
            if constexpr (RESCALE) {
                srr += r2;
                srd = fmaf(rr, d, srd);
            }
            float want = tt;
            if constexpr (GAIN) want = fmaxf(tt + gain * (tt - rr), 0.0f);
            const float k = want * ri;
            const pc sc = pk::mul(u[e], pk::bc(k));
            u[e] = pos ? sc : pk::make(want, pk::im(sc));
        }
    } else if constexpr (PASS == COL) {
        const float gain = a.gain;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float x = pk::re(u[e]), y = pk::im(u[e]);
            const float r2 = x * x + y * y;
            const float ri = rsqrtf(r2);   // inf at 0
            const float rr = r2 > 0.0f ? r2 * ri : 0.0f;
            const float tt = tv[e];
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
            u[e] = pk::make(x * k + ((in && !pos) ? want : 0.0f), y * k);
        }
    } else {
        unsigned zero = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float amp = tv[e];
            const float x = pk::re(u[e]), y = pk::im(u[e]);
            const float m2 = x * x + y * y;
            const float k = amp * rsqrtf(m2);
            if (m2 > 0.0f) u[e] = pk::mul(u[e], pk::bc(k));
            else zero |= 1u << e;
        }
        if (zero) {   // exact zeros: arg 0 -> beam (* q for Fresnel), as fast_row_holo
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if ((zero >> e) & 1u) {
                    cx<float> h = mk(tp ? tp[p0 + e] : 1.0f, 0.0f);
                    if (a.q_row) h = cmul(h, cmul(a.q_row[myline], a.q_col[natural(p0 + e)]));
                    u[e] = pk::from(h);
                }
        }
    }
}

__device__ __forceinline__ void unpack8(float (&t)[8], float4 lo, float4 hi) {
    t[0] = lo.x; t[1] = lo.y; t[2] = lo.z; t[3] = lo.w;
    t[4] = hi.x; t[5] = hi.y; t[6] = hi.z; t[7] = hi.w;
}

// ---- stage C (own line): radix 8, projection, radix 8 (second transform),
// two chunks per step (independent: twice the instruction-level parallelism
// per warp; chunk counts are even)
template <int PASS, int MODE>
__device__ __forceinline__ void stage_c_chunks(const Args& a, AddrC& ad, const float* tp, int lane, int myline,
                                               float& sdd, float& srr, float& srd, int cbeg, int cend) {
    constexpr int D1 = PASS == COL ? -1 : +1;
    constexpr int D2 = -D1;
    for (int C = 0; C < cbeg; ++C) ad.next();
    // the target (beam) values of the next chunk pair are loaded while this
    // pair is transformed (one L2 latency per stage)
    float4 n[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) n[q] = make_float4(1.f, 1.f, 1.f, 1.f);
    if (tp) {
        const float4* t4p = reinterpret_cast<const float4*>(tp + 8 * lane + 256 * cbeg);
        n[0] = __ldg(t4p);
        n[1] = __ldg(t4p + 1);
        n[2] = __ldg(t4p + 64);
        n[3] = __ldg(t4p + 65);
    }
#pragma unroll 1
    for (int C = cbeg; C < cend; C += 2) {
        const int p0 = 8 * lane + 256 * C;
        pc u[8], v[8];
        ld8_c<0>(u, ad);
        ld8_c<2048>(v, ad);
        float tu[8], tw[8];
        unpack8(tu, n[0], n[1]);
        unpack8(tw, n[2], n[3]);
        if (tp && C + 2 < cend) {
            const float4* t4p = reinterpret_cast<const float4*>(tp + p0 + 512);
            n[0] = __ldg(t4p);
            n[1] = __ldg(t4p + 1);
            n[2] = __ldg(t4p + 64);
            n[3] = __ldg(t4p + 65);
        }
        pk::Dft<8, D1, 1>::run(u);
        pk::Dft<8, D1, 1>::run(v);
        project8<PASS, MODE>(a, u, tu, tp, p0, myline, sdd, srr, srd);
        project8<PASS, MODE>(a, v, tw, tp, p0 + 256, myline, sdd, srr, srd);
        pk::Dft<8, D2, 1>::run(u);
        pk::Dft<8, D2, 1>::run(v);
        st8_c<0>(u, ad);
        st8_c<2048>(v, ad);
        ad.next();
        ad.next();
    }
}

// ---- one pass over all lines of the plane (every CTA: its static share)
// PASS == COL (replay plane, line = column n): forward -> error sums +
//   amplitude projection (fast_col_gs arithmetic; MODE bit 0 rescale sums,
//   bit 1 feedback gain) -> inverse; per-line sums to line_sums[n][3].
// PASS == ROW (hologram plane, line = row m): inverse -> beam * x / |x| (zero:
//   beam * q, as fast_row_holo) -> forward.
template <int PASS, int MODE>
__device__ __forceinline__ void pass_body(const Args& a, float2* wsm, double* line_sums) {
    constexpr int D1 = PASS == COL ? -1 : +1;
    constexpr int D2 = -D1;
    constexpr bool RESCALE = (MODE & 1) != 0, GAIN = (MODE & 2) != 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Role<PASS> ro(w, lane);
    const int slot0 = 4 * ro.grp;                 // first slot of the group (pair: 12)
    float2* own = slot(wsm, slot0 + ro.own);
    float sdd = 0.f, srr = 0.f, srd = 0.f;
    __shared__ double pair_part[2][3];            // pair, half 1: partial sums per line
    const int a0 = ro.a_beg(), a1 = a0 + ro.a_cnt();
    const int b0 = ro.h < 0 ? 0 : 2 * ro.h, b1 = ro.h < 0 ? 4 : b0 + 2;
    const int c0 = ro.h < 0 ? 0 : 4 * ro.h, c1 = ro.h < 0 ? 8 : c0 + 4;

    // Optional stagger (CGHB200_WL_STAGGER): the second half-CTA (quad 2 +
    // pair) starts loading only when the first (quads 0, 1) has its lines on
    // chip, so one half's memory traffic overlaps the other's arithmetic.
    const bool h2 = ro.grp >= 2;
    for (int rb = 0; rb < NQUAD; rb += round_len()) {
        const int line0 = group_line0(ro.grp, rb);
        const int line = line0 + ro.s;            // this thread's line in the joint stages
        float2* gsm = slot(wsm, slot0 + ro.s);    // its slot
        const int myline = line0 + ro.own;        // this warp's line in stages B..B'

        if (h2 && !a.no_stagger) asm volatile("bar.sync 5, %0;" ::"r"(THREADS) : "memory");
        if (line0 >= 0) {
            pc twA[15];
            load_tw(twA, a.tw, ro.j0 + 32 * a0);
            stage_a<PASS, D1>(gsm, a.data, line, ro.j0, twA, a.debug, a0, a1);
        }
        if (!h2 && !a.no_stagger) asm volatile("bar.arrive 5, %0;" ::"r"(THREADS) : "memory");
        if (line0 < 0) continue;                  // uniform per group
        stamp(a, w, 2);
        group_bar(ro.grp);
        stamp(a, w, 3);
        if (!(kDebug && (a.debug & 1))) stage_b<D1>(own, lane, twb_addr(wsm, lane), b0, b1);
        stamp(a, w, 4);
        __syncwarp();

        // stage C, projection, stage C' on 8 contiguous points per butterfly
        const float* tp = nullptr;
        if constexpr (PASS == COL) tp = a.tgt_perm + long(myline) * N;
        else tp = a.beam_perm ? a.beam_perm + long(myline) * N : nullptr;
        {
            AddrC ad(own, lane);
            if (!(kDebug && (a.debug & 1)))
                stage_c_chunks<PASS, MODE>(a, ad, tp, lane, myline, sdd, srr, srd, c0, c1);
        }
        stamp(a, w, 5);
        __syncwarp();
        if (!(kDebug && (a.debug & 1))) stage_b2<D2>(own, lane, twb_addr(wsm, lane), b0, b1);
        stamp(a, w, 6);
        double s3[3] = {0.0, 0.0, 0.0};
        if constexpr (PASS == COL) {
            s3[0] = double(sdd);
            s3[1] = double(srr);
            s3[2] = double(srd);
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s3[q] += __shfl_xor_sync(0xffffffffu, s3[q], o);
            if (ro.h == 1 && lane == 0)
#pragma unroll
                for (int q = 0; q < 3; ++q) pair_part[ro.own][q] = s3[q];
            sdd = srr = srd = 0.f;
        }
        group_bar(ro.grp);
        if constexpr (PASS == COL) {
            if (ro.h <= 0 && lane == 0) {   // quad warp, or the pair's first half (+ second, fixed order)
                const double sc2 = double(a.scale) * double(a.scale);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const double v = ro.h == 0 ? s3[q] + pair_part[ro.own][q] : s3[q];
                    line_sums[3 * long(myline) + q] = v * sc2;
                }
            }
        }
        {
            pc twA[15];
            load_tw(twA, a.tw, ro.j0 + 32 * a0);
            stage_a2<PASS, D2>(gsm, a.data, line, ro.j0, twA, a.debug, a0, a1);
        }
        stamp(a, w, 7);
        if (rb + round_len() < NQUAD) group_bar(ro.grp);   // the slots are reused by the next round
    }
}

// fixed-order total of the 2048 per-line sums (one warp per quantity q < 3)
__device__ __forceinline__ double line_total(const double* __restrict__ line_sums, int q, int lane) {
    double v = 0;
    for (int b = lane; b < N; b += 32) v += __ldcg(&line_sums[3 * long(b) + q]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One pass per launch (programmatic dependent launch chains the passes).
template <int PASS, int MODE>
__global__ void __launch_bounds__(THREADS, 1) wl_pass(Args a) {
    constexpr bool RESCALE = (MODE & 1) != 0;
    extern __shared__ __align__(128) float2 wsm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    stamp(a, w, 0);
    init_twb(wsm, a.tw);
    __syncthreads();
    pdl_wait();
    stamp(a, w, 1);
    pass_body<PASS, MODE>(a, wsm, a.line_sums);
    pdl_trigger();
    if constexpr (PASS == COL) {
        // error of this iteration in the CTA that finishes last
        __shared__ int last;
        __shared__ double rsh[3];
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            last = (atomicAdd(a.red.counter, 1u) == gridDim.x - 1);
        }
        __syncthreads();
        if (last) {
            __threadfence();
            if (w < 3) {
                const double v = line_total(a.line_sums, w, lane);
                if (lane == 0) rsh[w] = v;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                a.red.out[0] = error_from_sums(rsh[0], rsh[1], rsh[2], *a.red.denom, RESCALE ? a.red.rescale : 0);
                a.red.out[1] = 0.0;
                *a.red.counter = 0u;
            }
        }
    }
}

// Grid-wide barrier of a cooperative launch (every CTA resident): a monotone
// arrival counter, released by the last arrival's increment.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// The GS iteration loop in one persistent cooperative launch: iterations
// 0..iters-1 run the replay-plane pass (errors of iteration k from
// line_sums + k*3N, reduced afterwards by wl_trace_kernel), iterations
// 0..iters-2 the hologram-plane pass (the last one snaps: generic pass).
// Grid barriers replace the kernel boundaries.
template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) wl_loop(Args a, int iters, unsigned* bar) {
    extern __shared__ __align__(128) float2 wsm[];
    init_twb(wsm, a.tw);
    __syncthreads();
    unsigned target = 0;
    // timing experiments: warp 0 of every CTA stamps pass begin / end of
    // iterations 0..7: stamps[((k * 2 + pass) * 1024 + cta) * 2 + {0, 1}]
    auto lstamp = [&](int k, int pass, int end) {
        if (a.stamps && threadIdx.x == 0 && k < 8) {
            long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            a.stamps[((long(k) * 2 + pass) * 1024 + blockIdx.x) * 2 + end] = g;
        }
    };
    Args b = a;
    b.stamps = nullptr;
    for (int k = 0; k < iters; ++k) {
        lstamp(k, 1, 0);
        pass_body<COL, MODE>(b, wsm, a.line_sums + long(k) * 3 * N);
        lstamp(k, 1, 1);
        if (k == iters - 1) break;
        grid_sync(bar, target);
        lstamp(k, 0, 0);
        pass_body<ROW, 0>(b, wsm, nullptr);
        lstamp(k, 0, 1);
        grid_sync(bar, target);
    }
}

// errors of iterations 0..iters-1 of a wl_loop launch: out[2k] (as wl_pass)
__global__ void wl_trace_kernel(const double* __restrict__ line_sums, int iters, const double* __restrict__ denom,
                                int rescale, double* __restrict__ out) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double rsh[3];
    for (int k = blockIdx.x; k < iters; k += gridDim.x) {
        if (w < 3) {
            const double v = line_total(line_sums + long(k) * 3 * N, w, lane);
            if (lane == 0) rsh[w] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            out[2 * k] = error_from_sums(rsh[0], rsh[1], rsh[2], *denom, rescale);
            out[2 * k + 1] = 0.0;
        }
        __syncthreads();
    }
}

// row-major <-> T4 (to_t4 = 1: row-major src -> T4 dst)
__global__ void relayout_kernel(const float2* __restrict__ src, float2* __restrict__ dst, int to_t4) {
    const long total = long(N) * N;
    for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        // i enumerates T4 order: coalesced on the T4 side, 32-B sectors on the row-major side
        const int n = int((i >> 2) / N) * 4 + int(i & 3);
        const int m = int((i >> 2) % N);
        const long r = long(m) * N + n;
        if (to_t4) dst[i] = __ldcg(src + r);
        else dst[r] = __ldcg(src + i);
    }
}

// digit-reversed per-line tables: out[line][p] = scale * in[...natural(p)...]
// transposed = 1: in is row-major [H][W] indexed (natural row, line column)
// (target for the column pass); 0: (line row, natural column) (beam).
__global__ void perm_table_kernel(const float* __restrict__ in, float* __restrict__ out, float scale, int transposed) {
    const long total = long(N) * N;
    for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const int line = int(i / N), p = int(i % N);
        const int k = natural(p);
        const float v = transposed ? in[long(k) * N + line] : in[long(line) * N + k];
        out[i] = v * scale;
    }
}

}  // namespace wl
}  // namespace cgh
