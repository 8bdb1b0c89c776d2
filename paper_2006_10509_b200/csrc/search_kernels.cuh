// Persistent incremental pixel search: simulated annealing and direct binary
// search (algorithms.py:208-467, kernels/_core.pyx:20-83), float64.
//
// The masked, uncentred replay R_m, the target amplitude t_m (and the packed
// mask positions for partial masks) are split into one contiguous slice per
// CTA; one CTA per SM, launched cooperatively. Slices live in shared memory
// when they fit (1024^2 full mask: 24 MB over 148 SMs) else in global/L2.
//
// Every CTA runs the same numpy-stream emulation (thread 0) so all CTAs take
// identical decisions without a broadcast. One proposal (SA) or one window of
// W candidate pixels (DBS) costs one sweep over the slice — the previous
// accepted commit is applied in the same sweep — and one grid barrier: per-CTA
// partial sums are published, every CTA reduces them in the same fixed order.
#pragma once
#include "passes.cuh"

namespace cgh {

struct SearchState {
    Pcg64 rng;              // SA proposal stream
    double temperature;
    double error_num;       // running unscaled error numerator
    double warm_total;      // SA warm-up accumulator
    long long executed;     // SA: proposals done; DBS: visits done in this pass
    long long commits;      // DBS: commits in this pass
    long long logged;       // log entries written
    unsigned long long bar; // monotonic grid-barrier counter
    int pend;               // pending commit (applied during the next sweep)
    int pend_m, pend_n, pend_j;
    double pend_re, pend_im;
    int window;             // DBS speculation window
    int warm_left;          // SA warm-up proposals still to run
};

struct SearchArgs {
    int H, W, logH, logW;
    int pow2;                    // both sides powers of two (index masks), else division / modulo
    long long M;                 // masked elements
    int full;                    // positions implicit (full mask, row-major)
    double2* R;                  // [M] replay at mask positions (global copy)
    const double* t;             // [M]
    const uint32_t* pos;         // [M] (mu << 16) | mv, or nullptr when full
    const double2* rt;           // [H] exp(-2 pi i k / H)
    const double2* ct;           // [W] exp(-2 pi i k / W) / sqrt(H W)
    const double2* qr;           // Fresnel factors (H) or nullptr
    const double2* qc;           // (W)
    const double2* states;       // [L]
    int L;
    void* idx;                   // index plane (H*W), idx_bytes
    int idx_bytes;
    SearchState* st;
    double* partials;            // [2][G][NQ] phase-flagged 16-B slots (grid_reduce)
    int resident;                // slices in shared memory
    double denom;
    // SA
    long long k_end;             // run proposals until executed == k_end
    long long interval;          // checkpoint interval
    double alpha;                // cooling factor
    double* trace;               // checkpoint values (device-visible)
    long long* trace_k;
    long long* trace_len;        // running number of trace entries
    int write_trace;             // in-kernel checkpoints (no rescale)
    // DBS
    const long long* order;      // pass permutation or nullptr (raster)
    long long p_end;             // visits in this pass
    int wmax;
    // full-mask power-of-two planes with W <= 1024: a thread's columns repeat
    // with period colp = max(1, W / kSearchThreads) (0: generic sweep)
    int colp;
    long long* probe;            // SA stage clock sums of block 0 (diagnostics) or nullptr
    // decision log
    long long log_cap;
    long long* log_pixel;
    int* log_level;
    unsigned char* log_accept;
    double* log_change;
};

constexpr int kSearchThreads = 512;
constexpr int kMaxWindow = 32;      // DBS pixels per round
constexpr int kMaxLevels = 8;       // DBS levels evaluated per pixel in-kernel

__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ int read_index(const SearchArgs& a, long long p) {
    return a.idx_bytes == 1 ? int(static_cast<const uint8_t*>(a.idx)[p]) : static_cast<const int32_t*>(a.idx)[p];
}

__device__ __forceinline__ void write_index(const SearchArgs& a, long long p, int v) {
    if (a.idx_bytes == 1) static_cast<uint8_t*>(a.idx)[p] = (uint8_t)v;
    else static_cast<int32_t*>(a.idx)[p] = v;
}

// delta = (s_j - s_cur) * q[m, n]   (algorithms.py:253-257)
__device__ __forceinline__ double2 level_delta(const SearchArgs& a, int m, int n, int j, int cur) {
    const double2 sj = a.states[j], sc = a.states[cur];
    double2 d = make_double2(sj.x - sc.x, sj.y - sc.y);
    if (a.qr) d = dmul(d, dmul(a.qr[m], a.qc[n]));
    return d;
}

// Grid barrier on a monotonic counter (all CTAs co-resident: cooperative launch).
__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1ull);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Block sum of NQ doubles; result broadcast to all threads (fixed order).
template <int NQ>
__device__ __forceinline__ void block_sum_bcast(double (&v)[NQ], double* sh) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) sh[q * 32 + warp] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double s = 0;
        for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
        v[q] = s;
    }
}

// Publish per-CTA partials [nq], grid barrier, sum over CTAs in fixed order.
//
// The barrier is carried by the partials themselves: a value is stored as two
// 64-bit words (low half | phase << 32, high half | phase << 32). Aligned
// 64-bit stores are single-copy atomic, so a reader that sees the phase in
// both words holds the value: no counter atomics and no fences. Slots
// alternate by phase parity (a CTA cannot run two phases ahead of a reader: it
// needs that reader's next partial first). The buffer is zeroed per run and
// phases start at 1. Nothing else crosses CTAs inside an SA launch: commits
// are written to the index plane by every CTA (identical values), so each CTA
// reads back its own writes. (SA only; DBS uses grid_reduce_counter below.)
constexpr int kMaxSlotsPerLane = 8;   // G <= 256 CTAs

__device__ __forceinline__ void publish_slot(unsigned long long* p, double v, unsigned ph) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long w0 = (bits & 0xffffffffull) | (static_cast<unsigned long long>(ph) << 32);
    const unsigned long long w1 = (bits >> 32) | (static_cast<unsigned long long>(ph) << 32);
    asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}

__device__ __forceinline__ void load_slot(const unsigned long long* p, unsigned long long& w0, unsigned long long& w1) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
}

// First half: threads q < nq publish vals[q] (every thread holds vals, or
// vals is shared memory written before a __syncthreads). Advances phase.
__device__ __forceinline__ unsigned long long* grid_publish(const SearchArgs& a, const double* vals, int nq,
                                                           unsigned long long& phase) {
    unsigned long long* buf =
        reinterpret_cast<unsigned long long*>(a.partials) + ((phase & 1ull) * (size_t)gridDim.x * nq) * 2;
    phase += 1;
    if (threadIdx.x < nq) publish_slot(buf + ((size_t)blockIdx.x * nq + threadIdx.x) * 2, vals[threadIdx.x], unsigned(phase));
    return buf;
}

// Second half: warp w reduces quantities q = w, w + nwarps, ...: lane l polls
// CTAs l, l+32, ... together, sums them in that order, then a fixed shuffle
// tree; totals in sh_out[q]. Ends with __syncthreads.
__device__ __forceinline__ void grid_collect(const unsigned long long* buf, int nq, unsigned long long phase,
                                             double* sh_out) {
    const int G = gridDim.x;
    const unsigned ph = unsigned(phase);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = warp; q < nq; q += nw) {
        double v[kMaxSlotsPerLane];
        unsigned need = 0;
#pragma unroll
        for (int i = 0; i < kMaxSlotsPerLane; ++i)
            if (lane + 32 * i < G) need |= 1u << i;
        // round-robin over the lane's outstanding slots, volatile (.SYS)
        // accesses. Measured on B200 at the C4 SA sweep (block 0 clock64,
        // CGHB200_SA_PROBE): this form ~5.4k cycles per barrier (113k
        // proposals/s); all slots loaded per round before the checks ~7.9k;
        // spinning on one slot before the next ~9k (91k proposals/s);
        // relaxed.gpu instead of volatile ~9.4k
        while (need) {
#pragma unroll
            for (int i = 0; i < kMaxSlotsPerLane; ++i)
                if (need & (1u << i)) {
                    unsigned long long w0, w1;
                    load_slot(buf + ((size_t)(lane + 32 * i) * nq + q) * 2, w0, w1);
                    if (unsigned(w0 >> 32) == ph && unsigned(w1 >> 32) == ph) {
                        v[i] = __longlong_as_double(static_cast<long long>((w0 & 0xffffffffull) | (w1 << 32)));
                        need &= ~(1u << i);
                    }
                }
        }
        double s = 0;
#pragma unroll
        for (int i = 0; i < kMaxSlotsPerLane; ++i)
            if (lane + 32 * i < G) s += v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sh_out[q] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ void grid_reduce(const SearchArgs& a, const double* vals, int nq,
                                            unsigned long long& phase, double* sh_out) {
    const unsigned long long* buf = grid_publish(a, vals, nq, phase);
    grid_collect(buf, nq, phase, sh_out);
}

// DBS keeps the fenced counter barrier (grid_sync on st->bar): with the
// phase-flagged partials above, DBS at 128^2 and 256^2 hung on B200 (64^2,
// 512^2 and 1024^2 completed; cause not found), and DBS pays one barrier per
// window of up to 32 pixels, so the flagged form buys it little. Partials are
// plain doubles [2][G][nq] here.
__device__ __forceinline__ void grid_reduce_counter(const SearchArgs& a, const double* vals, int nq,
                                                    unsigned long long& phase, double* sh_out) {
    const int G = gridDim.x;
    double* buf = a.partials + (phase & 1ull) * (size_t)G * nq;
    if (threadIdx.x < nq) buf[(size_t)blockIdx.x * nq + threadIdx.x] = vals[threadIdx.x];
    phase += 1;
    grid_sync(&a.st->bar, phase * (unsigned long long)G);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int q = warp; q < nq; q += nw) {
        double s = 0;
        for (int b = lane; b < G; b += 32) s += __ldcg(&buf[(size_t)b * nq + q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) sh_out[q] = s;
    }
    __syncthreads();
}

struct Slice {
    long long begin, count;
    double2* R;
    const double* t;
    const uint32_t* pos;
};

__device__ __forceinline__ void element_pos(const SearchArgs& a, const Slice& s, long long li, int& mu, int& mv) {
    if (a.full) {
        const long long e = s.begin + li;
        mu = int(e >> a.logW);
        mv = int(e & (a.W - 1));
    } else {
        const uint32_t p = s.pos[li];
        mu = int(p >> 16);
        mv = int(p & 0xFFFF);
    }
}

// twiddle product row_tw[m][mu] * col_tw[n][mv] from the 1-D tables
template <bool P2>
__device__ __forceinline__ double2 tw_of(const double2* rt, const double2* ct, const SearchArgs& a, int m, int n, int mu,
                                         int mv) {
    if constexpr (P2) return dmul(rt[(m * mu) & (a.H - 1)], ct[(n * mv) & (a.W - 1)]);
    else return dmul(rt[(m * mu) % a.H], ct[(n * mv) % a.W]);
}

__device__ __forceinline__ double dabs(double2 z) { return sqrt(z.x * z.x + z.y * z.y); }

}  // namespace cgh
