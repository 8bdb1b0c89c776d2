// SA / DBS runners (algorithms.py:208-467) and the reference-kernel seam
// (kernels/_core.pyx:20-83) on the device. Host loop + persistent kernels.
#include <algorithm>
#include <cmath>

#include "runtime.cuh"
#include "search_kernels.cuh"

namespace cgh {

// ============================================================ kernels
struct SmemLayout {
    double2* rt;
    double2* ct;
    double2* R;
    double* t;
    uint32_t* pos;
    double* scratch;   // >= 32 * 8 doubles
};

__device__ __forceinline__ SmemLayout carve(const SearchArgs& a, unsigned char* base, const Slice& s) {
    SmemLayout L;
    size_t off = 0;
    L.rt = reinterpret_cast<double2*>(base + off);
    off += sizeof(double2) * a.H;
    L.ct = reinterpret_cast<double2*>(base + off);
    off += sizeof(double2) * a.W;
    L.R = reinterpret_cast<double2*>(base + off);
    off += sizeof(double2) * (a.resident ? s.count : 0);
    L.t = reinterpret_cast<double*>(base + off);
    off += sizeof(double) * (a.resident ? s.count : 0);
    L.pos = reinterpret_cast<uint32_t*>(base + off);
    off += sizeof(uint32_t) * ((a.resident && !a.full) ? s.count : 0);
    off = (off + 15) & ~size_t(15);
    L.scratch = reinterpret_cast<double*>(base + off);
    return L;
}

// Load tables (and the slice when resident) into shared memory.
__device__ __forceinline__ Slice prologue(const SearchArgs& a, SmemLayout& L, unsigned char* base) {
    Slice s;
    const long long G = gridDim.x, b = blockIdx.x;
    s.begin = a.M * b / G;
    s.count = a.M * (b + 1) / G - s.begin;
    L = carve(a, base, s);
    for (int i = threadIdx.x; i < a.H; i += blockDim.x) L.rt[i] = a.rt[i];
    for (int i = threadIdx.x; i < a.W; i += blockDim.x) L.ct[i] = a.ct[i];
    if (a.resident) {
        for (long long i = threadIdx.x; i < s.count; i += blockDim.x) {
            L.R[i] = a.R[s.begin + i];
            L.t[i] = a.t[s.begin + i];
            if (!a.full) L.pos[i] = a.pos[s.begin + i];
        }
        s.R = L.R;
        s.t = L.t;
        s.pos = L.pos;
    } else {
        s.R = a.R + s.begin;
        s.t = a.t + s.begin;
        s.pos = a.full ? nullptr : a.pos + s.begin;
    }
    __syncthreads();
    return s;
}

__device__ __forceinline__ void epilogue(const SearchArgs& a, const Slice& s) {
    __syncthreads();
    if (a.resident)
        for (long long i = threadIdx.x; i < s.count; i += blockDim.x) a.R[s.begin + i] = s.R[i];
}

struct Bcast {
    int m, n, j, cur, go, pend, pm, pn;
    double dre, dim, pre, pim;
};

// ---------------------------------------------------------------- SA
// A proposal drawn by thread 0 ahead of time (algorithms.py:334-340):
// pixel, raw level draw, stream state after the draws, prefetched index.
struct Draw {
    Pcg64 g;
    int m, n, jraw;
};

__device__ __forceinline__ void draw_ahead(const SearchArgs& a, Pcg64 g, Draw& d) {
    const uint32_t p = pcg_integers(g, uint64_t(a.H) * uint64_t(a.W));
    d.m = a.pow2 ? int(p >> a.logW) : int(p / uint32_t(a.W));
    d.n = a.pow2 ? int(p & (a.W - 1)) : int(p % uint32_t(a.W));
    d.jraw = int(pcg_integers(g, uint64_t(a.L - 1)));
    d.g = g;
}

__device__ __forceinline__ double2 level_delta_s(const SearchArgs& a, const double2* st_s, int m, int n, int j, int cur) {
    const double2 sj = a.L <= 64 ? st_s[j] : a.states[j], sc = a.L <= 64 ? st_s[cur] : a.states[cur];
    double2 d = make_double2(sj.x - sc.x, sj.y - sc.y);
    if (a.qr) d = dmul(d, dmul(a.qr[m], a.qc[n]));
    return d;
}

// One SA sweep on a full-mask power-of-two plane (a.colp = COLP): thread
// tid's elements li = tid + 512 r lie in columns (begin + tid + 512 r) mod W,
// which repeat with period COLP, so the column twiddles ct[n mv mod W] of the
// proposal (and pending) pixel are gathered once per sweep into registers —
// in shared memory those gathers conflict up to 8-way for even n. The row
// twiddle rt[m mu mod H] is one address per warp (broadcast). Terms and their
// order are those of the generic sweep (same products, same accumulation).
template <int COLP>
__device__ __forceinline__ double sa_sweep_cols(const SearchArgs& a, const Slice& s, const SmemLayout& L, int m,
                                                int n, double2 d, bool pend, int pm, int pn, double2 pd) {
    // (generic s.R / s.t accesses: the same sweep through L.R / L.t compiles to
    // LDS/STS but measured ~20% slower at C4 on B200 — 92k vs 113k proposals/s)
    double2* const Rs = s.R;
    const double* const ts = s.t;
    const int tid = threadIdx.x, Hm = a.H - 1, Wm = a.W - 1;
    double2 cw[COLP], cp[COLP];
#pragma unroll
    for (int p = 0; p < COLP; ++p) {
        const int mv = int((s.begin + tid + (long long)kSearchThreads * p) & Wm);
        cw[p] = L.ct[(n * mv) & Wm];
        cp[p] = pend ? L.ct[(pn * mv) & Wm] : make_double2(0.0, 0.0);
    }
    double acc = 0.0;
    for (long long li = tid; li < s.count; li += (long long)COLP * kSearchThreads) {
#pragma unroll
        for (int p = 0; p < COLP; ++p) {
            const long long l = li + (long long)kSearchThreads * p;
            if (COLP == 1 || l < s.count) {
                const int mu = int((s.begin + l) >> a.logW);
                double2 R = Rs[l];
                if (pend) {
                    const double2 u = dmul(pd, dmul(L.rt[(pm * mu) & Hm], cp[p]));
                    R.x += u.x;
                    R.y += u.y;
                    Rs[l] = R;
                }
                const double2 u = dmul(d, dmul(L.rt[(m * mu) & Hm], cw[p]));
                const double2 R1 = make_double2(R.x + u.x, R.y + u.y);
                const double t = ts[l];
                const double d0 = dabs(R) - t, d1 = dabs(R1) - t;
                acc += d1 * d1 - d0 * d0;
            }
        }
    }
    return acc;
}

// P2: both sides powers of two (table indices by mask, not modulo)
template <bool P2>
__global__ void __launch_bounds__(kSearchThreads, 1) sa_kernel(SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    SmemLayout L;
    const Slice s = prologue(a, L, smem);
    __shared__ Bcast bc;
    __shared__ SearchState st;
    __shared__ double red[8];
    __shared__ double2 st_s[64];
    if (threadIdx.x < 64 && threadIdx.x < a.L) st_s[threadIdx.x] = a.states[threadIdx.x];
    if (threadIdx.x == 0) st = *a.st;
    __syncthreads();
    unsigned long long phase = st.bar / gridDim.x;
    const bool lead = (blockIdx.x == 0 && threadIdx.x == 0);
    // thread 0 state (shared memory: keeps the sweep's registers free): the
    // next proposal for both outcomes of the Metropolis draw
    __shared__ Draw nxA, nxB;
    __shared__ Pcg64 g_after_u;
    __shared__ double u_next;
    __shared__ int have_next, c1_m, c1_n, c1_j;   // c1: commit of the previous proposal (may not be visible yet)
    if (threadIdx.x == 0) {
        u_next = 0.0;
        have_next = 0;
        c1_m = -1;
        c1_n = -1;
        c1_j = 0;
    }
    // prefetched index of the drawn pixels; trace entries written so far; proposals
    // to the next checkpoint (thread 0 / the drawing thread 32 only)
    __shared__ int idxA, idxB;
    __shared__ long long trace_n, to_check;
    if (threadIdx.x == 0) {
        idxA = 0;
        idxB = 0;
        trace_n = a.write_trace ? *a.trace_len : 0;
        to_check = a.interval - st.executed % a.interval;
    }
    // optional stage timing of block 0 (CGHB200_SA_PROBE): clock64 sums
    __shared__ long long tp[8], tprev;
    if (threadIdx.x < 8) tp[threadIdx.x] = 0;
    const bool probe = a.probe != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    auto mark = [&](int k) {
        if (probe) {
            const long long t = clock64();
            if (k > 0) tp[k] += t - tprev;
            tprev = t;
        }
    };
    for (;;) {
        mark(0);
        if (threadIdx.x == 0) {
            bc.pend = st.pend;
            bc.pm = st.pend_m;
            bc.pn = st.pend_n;
            bc.pre = st.pend_re;
            bc.pim = st.pend_im;
            const bool warm = st.warm_left > 0;
            bc.go = warm || st.executed < a.k_end;
            if (bc.go) {
                Draw cur_d;
                int cur;
                if (!have_next) {
                    draw_ahead(a, st.rng, cur_d);
                    cur = read_index(a, (long long)cur_d.m * a.W + cur_d.n);
                } else {
                    cur_d = nxA;   // branch chosen at the last decision is stored in nxA
                    cur = idxA;
                }
                st.rng = cur_d.g;
                if (st.pend && st.pend_m == cur_d.m && st.pend_n == cur_d.n) cur = st.pend_j;   // commit k-1
                else if (c1_m == cur_d.m && c1_n == cur_d.n) cur = c1_j;                      // commit k-2
                int j = cur_d.jraw;
                if (j >= cur) j += 1;
                const double2 d = level_delta_s(a, st_s, cur_d.m, cur_d.n, j, cur);
                bc.m = cur_d.m;
                bc.n = cur_d.n;
                bc.j = j;
                bc.cur = cur;
                bc.dre = d.x;
                bc.dim = d.y;
            }
        }
        __syncthreads();
        mark(1);
        if (!bc.go) break;
        mark(2);
        const int m = bc.m, n = bc.n, pm = bc.pm, pn = bc.pn;
        const double2 d = make_double2(bc.dre, bc.dim), pd = make_double2(bc.pre, bc.pim);
        const bool pend = bc.pend != 0;
        double acc[1] = {0.0};
        if (P2 && a.resident && a.colp == 1) acc[0] = sa_sweep_cols<1>(a, s, L, m, n, d, pend, pm, pn, pd);
        else if (P2 && a.resident && a.colp == 2) acc[0] = sa_sweep_cols<2>(a, s, L, m, n, d, pend, pm, pn, pd);
        else
            for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
                int mu, mv;
                element_pos(a, s, li, mu, mv);
                double2 R = s.R[li];
                if (pend) {
                    const double2 u = dmul(pd, tw_of<P2>(L.rt, L.ct, a, pm, pn, mu, mv));
                    R.x += u.x;
                    R.y += u.y;
                    s.R[li] = R;
                }
                const double2 u = dmul(d, tw_of<P2>(L.rt, L.ct, a, m, n, mu, mv));
                const double2 R1 = make_double2(R.x + u.x, R.y + u.y);
                const double t = s.t[li];
                const double d0 = dabs(R) - t, d1 = dabs(R1) - t;
                acc[0] += d1 * d1 - d0 * d0;
            }
        mark(3);
        block_sum_bcast<1>(acc, L.scratch);
        mark(4);
        {
            const unsigned long long* buf = grid_publish(a, acc, 1, phase);
            if (threadIdx.x == 32) {
                // draw proposal k+1 for both outcomes of the Metropolis draw while
                // warp 0 waits for the other CTAs' partials
                Draw dA, dB;
                draw_ahead(a, st.rng, dA);
                const int iA = read_index(a, (long long)dA.m * a.W + dA.n);
                Pcg64 gb = st.rng;
                u_next = pcg_next_double(gb);
                g_after_u = gb;
                draw_ahead(a, gb, dB);
                const int iB = read_index(a, (long long)dB.m * a.W + dB.n);
                nxA = dA;
                nxB = dB;
                idxA = iA;
                idxB = iB;
                have_next = 1;
            }
            grid_collect(buf, 1, phase, red);
        }
        mark(5);
        if (threadIdx.x == 0) {
            const double change = red[0];
            // the commit applied in this sweep (k-1) becomes "k-2" for the next draw
            if (st.pend) {
                c1_m = st.pend_m;
                c1_n = st.pend_n;
                c1_j = st.pend_j;
            } else {
                c1_m = -1;
            }
            st.pend = 0;
            bool drew = false;
            if (st.warm_left > 0) {
                st.warm_total += fabs(change) / a.denom;
                st.warm_left -= 1;
                if (st.warm_left == 0) st.temperature = st.warm_total / 100.0;
            } else {
                const double x = change / a.denom;
                bool ok = x < 0.0;
                if (!ok && st.temperature > 0.0) {
                    drew = true;   // rng.random() (algorithms.py:388-389)
                    ok = u_next < exp(-x / st.temperature);
                }
                if (ok) {
                    st.error_num += change;
                    st.pend = 1;
                    st.pend_m = bc.m;
                    st.pend_n = bc.n;
                    st.pend_j = bc.j;
                    st.pend_re = bc.dre;
                    st.pend_im = bc.dim;
                    // every CTA writes the commit: its own later reads then see it
                    write_index(a, (long long)bc.m * a.W + bc.n, bc.j);
                }
                if (lead && st.executed < a.log_cap) {
                    a.log_pixel[st.executed] = (long long)bc.m * a.W + bc.n;
                    a.log_level[st.executed] = bc.j;
                    a.log_accept[st.executed] = ok ? 1 : 0;
                }
                st.temperature *= a.alpha;
                st.executed += 1;
                if (--to_check == 0) {
                    to_check = a.interval;
                    if (a.write_trace && lead) {
                        const long long c = trace_n++;
                        a.trace[c] = st.error_num / a.denom;
                        a.trace_k[c] = st.executed;
                        *a.trace_len = c + 1;
                    }
                }
            }
            if (drew) {
                st.rng = g_after_u;   // the Metropolis draw is consumed
                nxA = nxB;            // and the next proposal follows it
                idxA = idxB;
            }
            // st.rng is replaced by the chosen draw's stream state at the top
        }
        __syncthreads();
        mark(6);
        if (probe) tp[7] += 1;
    }
    if (probe)
        for (int k = 1; k < 8; ++k) a.probe[k] += tp[k];
    // the stream state to persist: proposals drawn ahead are not consumed
    // (st.rng holds the state after the last consumed draws)
    if (st.pend) {
        const double2 pd = make_double2(st.pend_re, st.pend_im);
        for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
            int mu, mv;
            element_pos(a, s, li, mu, mv);
            const double2 u = dmul(pd, tw_of<P2>(L.rt, L.ct, a, st.pend_m, st.pend_n, mu, mv));
            s.R[li].x += u.x;
            s.R[li].y += u.y;
        }
    }
    epilogue(a, s);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        SearchState out = st;
        out.pend = 0;
        out.bar = phase * gridDim.x;
        *a.st = out;
    }
}

// ---------------------------------------------------------------- DBS
// Window of up to kMaxWindow pixels evaluated against the current state; the
// first improving pixel is committed, later pixels are re-evaluated.
template <bool P2>
__global__ void __launch_bounds__(kSearchThreads, 1) dbs_kernel(SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    SmemLayout L;
    const Slice s = prologue(a, L, smem);
    __shared__ SearchState st;
    __shared__ int nwin, wm[kMaxWindow], wn[kMaxWindow], wcur[kMaxWindow], go;
    __shared__ long long wp[kMaxWindow];
    __shared__ double2 wd[kMaxWindow * kMaxLevels];
    __shared__ unsigned char wvalid[kMaxWindow * kMaxLevels];
    __shared__ double red[kMaxWindow * kMaxLevels];
    __shared__ int pend;
    __shared__ int pm, pn;
    __shared__ double2 pdel;
    const int NQMAX = a.wmax * a.L;
    double* wsum = L.scratch;   // [16 warps][wmax * L]
    if (threadIdx.x == 0) st = *a.st;
    __syncthreads();
    unsigned long long phase = st.bar / gridDim.x;
    const bool lead = (blockIdx.x == 0 && threadIdx.x == 0);
    const int Lv = a.L;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) {
            pend = st.pend;
            pm = st.pend_m;
            pn = st.pend_n;
            pdel = make_double2(st.pend_re, st.pend_im);
            const long long left = a.p_end - st.executed;
            go = left > 0;
            int w = int(std::min<long long>(left, (long long)st.window));
            nwin = w;
            for (int k = 0; k < w; ++k) {
                const long long p = a.order ? a.order[st.executed + k] : st.executed + k;
                const int m = a.pow2 ? int(p >> a.logW) : int(p / a.W);
                const int n = a.pow2 ? int(p & (a.W - 1)) : int(p % a.W);
                wp[k] = p;
                wm[k] = m;
                wn[k] = n;
                const int cur = read_index(a, p);
                wcur[k] = cur;
                for (int j = 0; j < Lv; ++j) {
                    const double2 dl = level_delta(a, m, n, j, cur);
                    wd[k * Lv + j] = dl;
                    wvalid[k * Lv + j] = !(dl.x == 0.0 && dl.y == 0.0);   // _core.pyx:71-72 skips zero deltas
                }
            }
        }
        __syncthreads();
        if (!go) break;
        const int W = nwin, NQ = W * Lv;
        const bool has_pend = pend != 0;
        // apply the pending commit once
        if (has_pend) {
            for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
                int mu, mv;
                element_pos(a, s, li, mu, mv);
                const double2 u = dmul(pdel, tw_of<P2>(L.rt, L.ct, a, pm, pn, mu, mv));
                s.R[li].x += u.x;
                s.R[li].y += u.y;
            }
            __syncthreads();
        }
        if (Lv == 2) {
            // binary schemes: one valid level per candidate (the other state).
            // Candidates in chunks of 8 share one pass over the slice, so R, t
            // and |R| are read/computed once per element per chunk; each
            // candidate's per-thread sum has the same terms in the same order
            // as the per-candidate loop below (identical decisions).
            constexpr int KC = 8;
            for (int k0 = 0; k0 < W; k0 += KC) {
                double acc[KC];
#pragma unroll
                for (int kk = 0; kk < KC; ++kk) acc[kk] = 0.0;
                for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
                    int mu, mv;
                    element_pos(a, s, li, mu, mv);
                    const double2 R = s.R[li];
                    const double t = s.t[li];
                    const double d0 = dabs(R) - t;
                    const double b0 = d0 * d0;
#pragma unroll
                    for (int kk = 0; kk < KC; ++kk) {
                        const int k = k0 + kk;
                        if (k < W) {
                            const int jv = wvalid[k * 2] ? 0 : 1;
                            if (wvalid[k * 2 + jv]) {
                                const double2 w = tw_of<P2>(L.rt, L.ct, a, wm[k], wn[k], mu, mv);
                                const double2 u = dmul(wd[k * 2 + jv], w);
                                const double d1 = dabs(make_double2(R.x + u.x, R.y + u.y)) - t;
                                acc[kk] += d1 * d1 - b0;
                            }
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < KC; ++kk) {
                    const int k = k0 + kk;
                    if (k < W) {
                        double v = acc[kk];
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        if (lane == 0) {
                            const int jv = wvalid[k * 2] ? 0 : 1;
                            wsum[warp * NQMAX + k * 2 + jv] = v;
                            wsum[warp * NQMAX + k * 2 + (1 - jv)] = 0.0;
                        }
                    }
                }
            }
        }
        for (int k = 0; k < (Lv == 2 ? 0 : W); ++k) {
            double acc[kMaxLevels];
#pragma unroll
            for (int j = 0; j < kMaxLevels; ++j) acc[j] = 0.0;
            const int m = wm[k], n = wn[k];
            for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
                int mu, mv;
                element_pos(a, s, li, mu, mv);
                const double2 R = s.R[li];
                const double t = s.t[li];
                const double2 w = tw_of<P2>(L.rt, L.ct, a, m, n, mu, mv);
                const double d0 = dabs(R) - t;
                const double b0 = d0 * d0;
#pragma unroll
                for (int j = 0; j < kMaxLevels; ++j) {
                    if (j < Lv && wvalid[k * Lv + j]) {
                        const double2 u = dmul(wd[k * Lv + j], w);
                        const double d1 = dabs(make_double2(R.x + u.x, R.y + u.y)) - t;
                        acc[j] += d1 * d1 - b0;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kMaxLevels; ++j) {
                if (j < Lv) {
                    double v = acc[j];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                    if (lane == 0) wsum[warp * NQMAX + k * Lv + j] = v;
                }
            }
        }
        __syncthreads();
        double* part = wsum + nw * NQMAX;
        for (int q = threadIdx.x; q < NQ; q += blockDim.x) {
            double v = 0;
            for (int w2 = 0; w2 < nw; ++w2) v += wsum[w2 * NQMAX + q];
            part[q] = v;
        }
        __syncthreads();
        grid_reduce_counter(a, part, NQ, phase, red);
        if (threadIdx.x == 0) {
            st.pend = 0;
            int advanced = W;
            for (int k = 0; k < W; ++k) {
                // best_delta (_core.pyx:47-83): strict '<' from 0.0, lowest index wins
                int bj = -1;
                double bc = 0.0;
                for (int j = 0; j < Lv; ++j) {
                    if (!wvalid[k * Lv + j]) continue;
                    const double c = red[k * Lv + j];
                    if (c < bc) {
                        bc = c;
                        bj = j;
                    }
                }
                const bool took = bj >= 0 && bc < 0.0;
                if (lead && st.logged < a.log_cap) {
                    a.log_pixel[st.logged] = wp[k];
                    a.log_level[st.logged] = took ? bj : -1;
                    a.log_change[st.logged] = bc;
                    st.logged += 1;
                }
                if (took) {
                    st.error_num += bc;
                    st.commits += 1;
                    st.pend = 1;
                    st.pend_m = wm[k];
                    st.pend_n = wn[k];
                    st.pend_j = bj;
                    st.pend_re = wd[k * Lv + bj].x;
                    st.pend_im = wd[k * Lv + bj].y;
                    if (blockIdx.x == 0) write_index(a, wp[k], bj);
                    advanced = k + 1;
                    break;
                }
            }
            st.executed += advanced;
            // window policy: grow while nothing commits, shrink after an early commit
            int nwin2 = st.pend ? std::max(1, 2 * advanced) : 2 * W;
            st.window = std::min(std::max(nwin2, 1), a.wmax);
        }
        __syncthreads();
    }
    if (st.pend) {
        const double2 pd = make_double2(st.pend_re, st.pend_im);
        for (long long li = threadIdx.x; li < s.count; li += blockDim.x) {
            int mu, mv;
            element_pos(a, s, li, mu, mv);
            const double2 u = dmul(pd, tw_of<P2>(L.rt, L.ct, a, st.pend_m, st.pend_n, mu, mv));
            s.R[li].x += u.x;
            s.R[li].y += u.y;
        }
    }
    epilogue(a, s);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        SearchState out = st;
        out.pend = 0;
        out.bar = phase * gridDim.x;
        *a.st = out;
    }
}

// ------------------------------------------------------- setup helpers
// per-block in-mask counts (block of 1024 pixels)
__global__ void mask_count_kernel(const double* __restrict__ tgt, long long n, int* __restrict__ counts) {
    __shared__ int c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    const long long base = (long long)blockIdx.x * 1024;
    int local = 0;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const long long p = base + i;
        if (p < n && !signbit(tgt[p])) local += 1;
    }
    atomicAdd(&c, local);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

// scatter masked elements in row-major order (one warp-serial pass per block)
__global__ void mask_scatter_kernel(const double* __restrict__ tgt, const double2* __restrict__ rep, long long n, int W,
                                    int logW, const long long* __restrict__ offsets, double2* __restrict__ R,
                                    double* __restrict__ t, uint32_t* __restrict__ pos) {
    const long long base = (long long)blockIdx.x * 1024;
    __shared__ int flags[1024];
    __shared__ int scan[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        const long long p = base + i;
        flags[i] = (p < n && !signbit(tgt[p])) ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i < 1024; ++i) {
            scan[i] = acc;
            acc += flags[i];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        if (!flags[i]) continue;
        const long long p = base + i;
        const long long o = offsets[blockIdx.x] + scan[i];
        R[o] = rep[p];
        t[o] = fabs(tgt[p]);
        pos[o] = (uint32_t(p / W) << 16) | uint32_t(p % W);   // any W (logW unused)
    }
}

// fixed-order sums over the masked elements: [sum (|R|-t)^2, sum |R|^2, sum |R| t]
// and, with scale > 0, sum (scale |R| - t)^2 in slot 3.
__global__ void search_sums_kernel(const double2* __restrict__ R, const double* __restrict__ t, long long M,
                                   double scale, double* __restrict__ partials, unsigned* __restrict__ counter,
                                   double* __restrict__ out) {
    double acc[4] = {0, 0, 0, 0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
        const double r = hypot(R[i].x, R[i].y);
        const double d = r - t[i];
        acc[0] += d * d;
        acc[1] += r * r;
        acc[2] += r * t[i];
        const double e = scale * r - t[i];
        acc[3] += e * e;
    }
    __shared__ double sh[32 * 4];
    block_reduce<4>(acc, sh);
    ReduceArgs ra;
    ra.partials = partials;
    ra.counter = counter;
    if (publish_partials<4>(ra, acc, gridDim.x, blockIdx.x)) {
        double v[4];
        for (int q = 0; q < 4; ++q) v[q] = sum_partials(ra, q, gridDim.x, sh);
        if (threadIdx.x == 0) {
            for (int q = 0; q < 4; ++q) out[q] = v[q];
            *counter = 0u;
        }
    }
}

// ------------------------------------------- reference-kernel seam kernels
// delta_error / best_delta over caller arrays (row_tw / col_tw rows given).
__global__ void seam_eval_kernel(const double2* __restrict__ Rm, const double* __restrict__ tm,
                                 const double2* __restrict__ rtw, const double2* __restrict__ ctw,
                                 const int32_t* __restrict__ mu, const int32_t* __restrict__ mv, long long n,
                                 const double2* __restrict__ deltas, int levels, double* __restrict__ partials,
                                 unsigned* __restrict__ counter, double* __restrict__ out) {
    // one level per blockIdx.y
    const int j = blockIdx.y;
    const double2 dl = deltas[j];
    double acc[1] = {0.0};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 w = dmul(rtw[mu[i]], ctw[mv[i]]);
        const double2 u = dmul(dl, w);
        const double2 R = Rm[i];
        const double d0 = dabs(R) - tm[i];
        const double d1 = dabs(make_double2(R.x + u.x, R.y + u.y)) - tm[i];
        acc[0] += d1 * d1 - d0 * d0;
    }
    __shared__ double sh[32];
    block_reduce<1>(acc, sh);
    if (threadIdx.x == 0) partials[(size_t)j * gridDim.x + blockIdx.x] = acc[0];
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (last && threadIdx.x < levels) {
        __threadfence();
        double s = 0;
        for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(&partials[(size_t)threadIdx.x * gridDim.x + b]);
        out[threadIdx.x] = s;
    }
    if (last && threadIdx.x == 0) *counter = 0u;
}

__global__ void seam_commit_kernel(double2* __restrict__ Rm, const double2* __restrict__ rtw,
                                   const double2* __restrict__ ctw, const int32_t* __restrict__ mu,
                                   const int32_t* __restrict__ mv, long long n, double2 dl) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 u = dmul(dl, dmul(rtw[mu[i]], ctw[mv[i]]));
        Rm[i].x += u.x;
        Rm[i].y += u.y;
    }
}

// DBS window: W pixels x L levels <= kMaxWindow*kMaxLevels/4 partial sums
inline int dbs_wmax(int L) { return std::max(1, std::min(kMaxWindow, 64 / std::max(1, L))); }
inline int dbs_nq(int L) { return dbs_wmax(L) * std::max(1, L); }

// ============================================================ host side
struct SearchRun {
    cgh_plan* P;
    long long M = 0;
    bool full = false;
    double2* R = nullptr;      // device
    double* t = nullptr;
    uint32_t* pos = nullptr;
    double2* rt = nullptr;     // 1-D tables (fp64)
    double2* ct = nullptr;
    SearchState* st = nullptr;
    double* partials = nullptr;
    double* sums = nullptr;    // 4
    double* trace = nullptr;   // device (mapped host)
    long long* trace_k = nullptr;
    long long* trace_len = nullptr;
    int grid = 0;
    int resident = 0;
    size_t smem = 0;
    DevBuf scratch;
};

static int search_alloc(SearchRun& S, size_t bytes, void** out) {
    (void)S;
    CGH_CUDA(cudaMallocAsync(out, bytes, S.P->st));
    return CGH_OK;
}

// Initial index plane + uncentred replay + masked gather (algorithms.py:217-251).
static int search_setup(SearchRun& S, int init_mode, const cgh_pcg64& rng0, bool dbs) {
    cgh_plan* P = S.P;
    const long long n = (long long)P->H * P->W;
    CGH_TRY(ensure(P, P->data, size_t(n) * 16));
    CGH_TRY(ensure(P, P->idx, size_t(n) * P->idx_bytes));
    const int nb = std::max(row_grid_blocks<double>(P->W, P->H), col_grid_blocks<double>(P->H, P->W));
    CGH_TRY(ensure(P, P->partials, size_t(std::max(nb, 4096)) * 8 * sizeof(double)));
    PassArgs<double> a = base_args<double>(P);
    a.rng = to_pcg(rng0);
    a.quantize = 1;
    a.idx_out = P->idx.p;
    P->idx_frames = 1;
    if (init_mode == CGH_INIT_RANDOM_PHASE) {
        CGH_TRY(run_row<double>(P, ROW_INIT, a, 1));
    } else {
        if (!P->stage_valid)
            return fail(CGH_ERR_VALUE, "backpropagation start needs the complex target (cgh_plan_set_target)");
        load_field_kernel<double><<<grid_for(n), 256, 0, P->st>>>(static_cast<const double*>(P->stage.p), a.data, P->H,
                                                                  P->W, 1, nullptr, nullptr,
                                                                  static_cast<unsigned*>(P->counter.p) + 8);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        PassArgs<double> b = a;
        b.quantize = 0;
        b.idx_out = nullptr;
        CGH_TRY(run_col<double>(P, COL_INV, b, 1));
        CGH_TRY(run_row<double>(P, ROW_HOLO, a, 1));
    }
    // data = rowFFT(states[idx] q); column FFT with the unitary scale -> replay
    a.scale = 1.0 / std::sqrt(double(n));
    CGH_TRY(run_col<double>(P, COL_FWD, a, 1));

    S.M = (long long)P->count_in;
    // full masks use implicit row-major positions (shift / mask); other planes
    // carry packed positions
    S.full = (S.M == n) && is_pow2(P->H) && is_pow2(P->W);
    if (S.full) {
        S.R = static_cast<double2*>(P->data.p);
        S.t = static_cast<double*>(P->tgt.p);
    } else {
        const int blocks = int((n + 1023) / 1024);
        int* counts = nullptr;
        long long* offs = nullptr;
        CGH_TRY(search_alloc(S, sizeof(int) * blocks, reinterpret_cast<void**>(&counts)));
        CGH_TRY(search_alloc(S, sizeof(long long) * blocks, reinterpret_cast<void**>(&offs)));
        mask_count_kernel<<<blocks, 256, 0, P->st>>>(static_cast<const double*>(P->tgt.p), n, counts);
        std::vector<int> hc(blocks);
        CGH_CUDA(cudaMemcpyAsync(hc.data(), counts, sizeof(int) * blocks, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        std::vector<long long> ho(blocks);
        long long acc = 0;
        for (int b = 0; b < blocks; ++b) {
            ho[b] = acc;
            acc += hc[b];
        }
        CGH_CUDA(cudaMemcpyAsync(offs, ho.data(), sizeof(long long) * blocks, cudaMemcpyHostToDevice, P->st));
        CGH_TRY(search_alloc(S, sizeof(double2) * std::max<long long>(acc, 1), reinterpret_cast<void**>(&S.R)));
        CGH_TRY(search_alloc(S, sizeof(double) * std::max<long long>(acc, 1), reinterpret_cast<void**>(&S.t)));
        CGH_TRY(search_alloc(S, sizeof(uint32_t) * std::max<long long>(acc, 1), reinterpret_cast<void**>(&S.pos)));
        int logW = 0;
        while ((1 << logW) < P->W) ++logW;
        mask_scatter_kernel<<<blocks, 256, 0, P->st>>>(static_cast<const double*>(P->tgt.p),
                                                       static_cast<const double2*>(P->data.p), n, P->W, logW, offs,
                                                       S.R, S.t, S.pos);
        P->launches += 2;
        CGH_CUDA(cudaGetLastError());
        CGH_CUDA(cudaFreeAsync(counts, P->st));
        CGH_CUDA(cudaFreeAsync(offs, P->st));
        S.M = acc;
    }
    // 1-D DFT tables: row exp(-2 pi i k/H); column exp(-2 pi i k/W)/sqrt(HW)
    CGH_TRY(search_alloc(S, sizeof(double2) * P->H, reinterpret_cast<void**>(&S.rt)));
    CGH_TRY(search_alloc(S, sizeof(double2) * P->W, reinterpret_cast<void**>(&S.ct)));
    {
        const long double pi = 3.141592653589793238462643383279502884L;
        std::vector<double2> r(P->H), c(P->W);
        for (int k = 0; k < P->H; ++k) {
            long double ang = -2.0L * pi * (long double)k / (long double)P->H;
            r[k] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        const long double sc = 1.0L / sqrtl((long double)P->H * (long double)P->W);
        for (int k = 0; k < P->W; ++k) {
            long double ang = -2.0L * pi * (long double)k / (long double)P->W;
            c[k] = make_double2((double)(cosl(ang) * sc), (double)(sinl(ang) * sc));
        }
        CGH_CUDA(cudaMemcpyAsync(S.rt, r.data(), sizeof(double2) * P->H, cudaMemcpyHostToDevice, P->st));
        CGH_CUDA(cudaMemcpyAsync(S.ct, c.data(), sizeof(double2) * P->W, cudaMemcpyHostToDevice, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
    }
    CGH_TRY(search_alloc(S, sizeof(SearchState), reinterpret_cast<void**>(&S.st)));
    CGH_TRY(search_alloc(S, sizeof(double) * 8, reinterpret_cast<void**>(&S.sums)));
    // persistent grid: one CTA per SM
    int dev = P->dev, sms = 0;
    CGH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int optin = 0;
    CGH_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    long long per = (S.M + sms - 1) / sms;
    const size_t tables = sizeof(double2) * (P->H + P->W);
    const int nq = dbs_nq(P->nstates);
    const size_t scratch = dbs ? sizeof(double) * ((kSearchThreads / 32) + 1) * nq + 64 : sizeof(double) * 32 * 8 + 64;
    const size_t slice = size_t(per) * (16 + 8 + (S.full ? 0 : 4));
    const size_t static_smem = 8 * 1024;
    S.resident = (tables + slice + scratch + static_smem + 64 <= size_t(optin)) ? 1 : 0;
    S.smem = tables + (S.resident ? slice : 0) + scratch + 64;
    if (S.smem + static_smem > size_t(optin))
        return fail(CGH_ERR_UNSUPPORTED, "search tables for %dx%d exceed shared memory", P->H, P->W);
    S.grid = std::max(1, (int)std::min<long long>(sms, std::max<long long>(S.M, 1)));
    // phase-flagged partials (search_kernels.cuh grid_reduce): 16 B per value,
    // two parities, zeroed so no stale flag matches a phase of this run
    const size_t pbytes = size_t(16) * 2 * S.grid * kMaxWindow * kMaxLevels;
    CGH_TRY(search_alloc(S, pbytes, reinterpret_cast<void**>(&S.partials)));
    CGH_CUDA(cudaMemsetAsync(S.partials, 0, pbytes, P->st));
    return CGH_OK;
}

static void search_free(SearchRun& S) {
    cudaStream_t st = S.P->st;
    if (!S.full) {
        if (S.R) cudaFreeAsync(S.R, st);
        if (S.t) cudaFreeAsync(S.t, st);
        if (S.pos) cudaFreeAsync(S.pos, st);
    }
    void* ps[] = {S.rt, S.ct, S.st, S.sums, S.partials};
    for (void* p : ps)
        if (p) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
}

// sums over the masked replay: [sum d^2, sum r^2, sum r t, sum (scale r - t)^2]
static int search_sums(SearchRun& S, double scale, double out[4]) {
    cgh_plan* P = S.P;
    const int grid = grid_for(std::max<long long>(S.M, 1));
    search_sums_kernel<<<grid, 256, 0, P->st>>>(S.R, S.t, S.M, scale, static_cast<double*>(P->partials.p),
                                                static_cast<unsigned*>(P->counter.p), S.sums);
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    CGH_CUDA(cudaMemcpyAsync(out, S.sums, sizeof(double) * 4, cudaMemcpyDeviceToHost, P->st));
    CGH_CUDA(cudaStreamSynchronize(P->st));
    return CGH_OK;
}

// reported_error (algorithms.py:296-303)
static int reported_error(SearchRun& S, double error_num, double denom, int rescale, double* out) {
    if (!rescale) {
        *out = error_num / denom;
        return CGH_OK;
    }
    double v[4];
    CGH_TRY(search_sums(S, 1.0, v));
    const double s = v[1] > 0.0 ? v[2] / v[1] : 1.0;
    CGH_TRY(search_sums(S, s, v));
    *out = v[3] / denom;
    return CGH_OK;
}

static SearchArgs search_args(SearchRun& S) {
    cgh_plan* P = S.P;
    SearchArgs a;
    memset(&a, 0, sizeof(a));
    a.H = P->H;
    a.W = P->W;
    while ((1 << a.logH) < P->H) ++a.logH;
    while ((1 << a.logW) < P->W) ++a.logW;
    a.pow2 = (is_pow2(P->H) && is_pow2(P->W)) ? 1 : 0;
    a.M = S.M;
    a.full = S.full ? 1 : 0;
    a.R = S.R;
    a.t = S.t;
    a.pos = S.pos;
    a.rt = S.rt;
    a.ct = S.ct;
    a.qr = P->prop_kind == CGH_FRESNEL ? static_cast<const double2*>(P->q_row.p) : nullptr;
    a.qc = P->prop_kind == CGH_FRESNEL ? static_cast<const double2*>(P->q_col.p) : nullptr;
    a.states = static_cast<const double2*>(P->states64.p);
    a.L = P->nstates;
    a.idx = P->idx.p;
    a.idx_bytes = P->idx_bytes;
    a.st = S.st;
    a.partials = S.partials;
    a.resident = S.resident;
    a.denom = P->denom;
    if (a.pow2 && a.full && P->W <= 1024) a.colp = std::max(1, P->W / kSearchThreads);
    return a;
}

static int launch_search(SearchRun& S, bool dbs, SearchArgs& a) {
    cgh_plan* P = S.P;
    void* fn = a.pow2 ? (dbs ? (void*)dbs_kernel<true> : (void*)sa_kernel<true>)
                      : (dbs ? (void*)dbs_kernel<false> : (void*)sa_kernel<false>);
    CGH_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S.smem)));
    void* args[] = {&a};
    if (P->profiling) CGH_TRY(prof_mark(P, dbs ? 17 : 16, true));
    CGH_CUDA(cudaLaunchCooperativeKernel(fn, dim3(S.grid), dim3(kSearchThreads), args, S.smem, P->st));
    if (P->profiling) CGH_TRY(prof_mark(P, dbs ? 17 : 16, false));
    P->launches += 1;
    return CGH_OK;
}

// final report: reported error + efficiency of the full replay (algorithms.py:309-328)
static int search_final(SearchRun& S, double error_num, int rescale, double* final_err, double* eff) {
    cgh_plan* P = S.P;
    CGH_TRY(reported_error(S, error_num, P->denom, rescale, final_err));
    const long long n = (long long)P->H * P->W;
    PassArgs<double> a = base_args<double>(P);
    // the replay buffer may alias data (full mask): rebuild the field from indices
    SchemeDev sd = a.scheme;
    field_from_index_kernel<double><<<grid_for(n), 256, 0, P->st>>>(P->idx.p, P->idx_bytes, sd, a.data, P->H, P->W,
                                                                    a.q_row, a.q_col);
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    a.scale = 1.0;
    CGH_TRY(run_row<double>(P, ROW_FWD, a, 1));
    CGH_TRY(ensure_res(P, 8));
    a.red.out = P->res_d;
    CGH_TRY(run_col<double>(P, COL_FINAL, a, 1));
    CGH_CUDA(cudaStreamSynchronize(P->st));
    volatile double* r = P->res_h;
    *eff = r[1];
    if (std::isnan(*eff)) return fail(CGH_ERR_ZERO_FIELD, "replay field is zero");
    return CGH_OK;
}

struct TraceOut {
    int64_t* k;
    double* v;
    int64_t cap;
    int64_t len = 0;
    int push(int64_t kk, double vv) {
        if (k && v) {
            if (len >= cap) return fail(CGH_ERR_VALUE, "trace capacity %lld exceeded", (long long)cap);
            k[len] = kk;
            v[len] = vv;
        }
        len += 1;
        return CGH_OK;
    }
};

static int audit_call(SearchRun& S, const cgh_callbacks* cb, int64_t k, double inc) {
    cgh_plan* P = S.P;
    const long long n = (long long)P->H * P->W;
    std::vector<int32_t> idx(n);
    if (P->idx_bytes == 4) {
        CGH_CUDA(cudaMemcpyAsync(idx.data(), P->idx.p, n * 4, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
    } else {
        std::vector<uint8_t> b(n);
        CGH_CUDA(cudaMemcpyAsync(b.data(), P->idx.p, n, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        for (long long i = 0; i < n; ++i) idx[i] = b[i];
    }
    cb->audit(cb->user, k, inc, idx.data());
    return CGH_OK;
}

static int sa_exec(cgh_plan* P, const cgh_sa_params* sp, int64_t* tk, double* tv, int64_t cap, cgh_report* rep,
                   const cgh_callbacks* cb) {
    GateLock gate(P->dev, true);   // grid-barrier kernels: the device to this run (runtime.cuh)
    if (P->prec != CGH_FP64) return fail(CGH_ERR_VALUE, "search runs need an fp64 plan");
    if (sp->init_mode != CGH_INIT_RANDOM_PHASE && sp->init_mode != CGH_INIT_BACKPROPAGATE)
        return fail(CGH_ERR_VALUE, "unknown init mode %d", sp->init_mode);
    if (sp->init_mode == CGH_INIT_BACKPROPAGATE && P->nf_all > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf");
    if (P->denom == 0) return fail(CGH_ERR_ZERO_TARGET, "target is zero inside the mask");
    const long launches0 = P->launches;
    CGH_CUDA(cudaEventRecord(P->ev0, P->st));
    SearchRun S;
    S.P = P;
    struct Guard {
        SearchRun* s;
        ~Guard() { search_free(*s); }
    } guard{&S};
    CGH_TRY(search_setup(S, sp->init_mode, sp->rng, false));
    double sums[4];
    CGH_TRY(search_sums(S, 1.0, sums));
    const double error0 = sums[0];
    // proposal stream: PCG64(seed) after the H*W start-phase draws (random init)
    Pcg64 g = to_pcg(sp->rng);
    if (sp->init_mode == CGH_INIT_RANDOM_PHASE) pcg_advance(g, uint64_t(P->H) * uint64_t(P->W));
    SearchState st0;
    memset(&st0, 0, sizeof(st0));
    st0.rng = g;
    st0.error_num = error0;
    st0.temperature = sp->initial_temperature;
    const bool auto_t = !(sp->initial_temperature >= 0);   // None or < 0 (algorithms.py:369-375)
    st0.warm_left = auto_t ? 100 : 0;
    st0.window = 1;
    CGH_CUDA(cudaMemcpyAsync(S.st, &st0, sizeof(st0), cudaMemcpyHostToDevice, P->st));
    TraceOut tr{tk, tv, cap};
    double first;
    CGH_TRY(reported_error(S, error0, P->denom, P->rescale, &first));
    CGH_TRY(tr.push(0, first));
    const bool has_cb = cb && (cb->cancel || cb->progress || cb->audit);
    if (cb && cb->progress) cb->progress(cb->user, 0, first);
    const long long proposals = std::max<long long>(0, sp->proposals);
    const long long interval = std::max<long long>(1, proposals / 1000);
    const bool chunked = has_cb || P->rescale;
    CGH_TRY(ensure_res(P, size_t(proposals / interval + 8) * 2 + 8));
    // device-visible trace buffers (mapped host memory)
    double* tr_v = P->res_h;
    long long* tr_k = reinterpret_cast<long long*>(P->res_h + (proposals / interval + 4));
    long long* tr_len = reinterpret_cast<long long*>(P->res_h + 2 * (proposals / interval + 4) + 2);
    *tr_len = 0;
    SearchArgs a = search_args(S);
    a.interval = interval;
    a.alpha = sp->cooling_factor;
    a.trace = P->res_d;
    a.trace_k = reinterpret_cast<long long*>(P->res_d + (proposals / interval + 4));
    a.trace_len = reinterpret_cast<long long*>(P->res_d + 2 * (proposals / interval + 4) + 2);
    a.write_trace = chunked ? 0 : 1;
    long long* dprobe = nullptr;
    if (getenv("CGHB200_SA_PROBE")) {
        CGH_TRY(search_alloc(S, sizeof(long long) * 8, reinterpret_cast<void**>(&dprobe)));
        CGH_CUDA(cudaMemsetAsync(dprobe, 0, sizeof(long long) * 8, P->st));
        a.probe = dprobe;
    }
    // decision log buffers
    long long* dlog_p = nullptr;
    int* dlog_l = nullptr;
    unsigned char* dlog_a = nullptr;
    const long long lcap = std::min<long long>(std::max<long long>(0, sp->log_cap), proposals);
    if (lcap > 0) {
        CGH_TRY(search_alloc(S, sizeof(long long) * lcap + sizeof(int) * lcap + lcap + 64, reinterpret_cast<void**>(&dlog_p)));
        dlog_l = reinterpret_cast<int*>(dlog_p + lcap);
        dlog_a = reinterpret_cast<unsigned char*>(dlog_l + lcap);
    }
    a.log_cap = lcap;
    a.log_pixel = dlog_p;
    a.log_level = dlog_l;
    a.log_accept = dlog_a;
    long long executed = 0;
    bool stop = false;
    double error_num = error0;
    if (!chunked) {
        a.k_end = proposals;
        CGH_TRY(launch_search(S, false, a));
        SearchState sh;
        CGH_CUDA(cudaMemcpyAsync(&sh, S.st, sizeof(sh), cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        executed = sh.executed;
        error_num = sh.error_num;
        volatile long long* vl = tr_len;
        for (long long c = 0; c < *vl; ++c) CGH_TRY(tr.push(tr_k[c], tr_v[c]));
    } else {
        while (executed < proposals) {
            if (cancelled(cb)) {
                stop = true;
                break;
            }
            a.k_end = std::min(proposals, (executed / interval + 1) * interval);
            CGH_TRY(launch_search(S, false, a));
            SearchState sh;
            CGH_CUDA(cudaMemcpyAsync(&sh, S.st, sizeof(sh), cudaMemcpyDeviceToHost, P->st));
            CGH_CUDA(cudaStreamSynchronize(P->st));
            executed = sh.executed;
            error_num = sh.error_num;
            if (executed % interval == 0) {
                double e;
                CGH_TRY(reported_error(S, error_num, P->denom, P->rescale, &e));
                CGH_TRY(tr.push(executed, e));
                if (cb && cb->progress) cb->progress(cb->user, executed, e);
                if (cb && cb->audit) CGH_TRY(audit_call(S, cb, executed, error_num / P->denom));
            }
        }
    }
    // _final_report
    double final_err, eff;
    CGH_TRY(search_final(S, error_num, P->rescale, &final_err, &eff));
    const double last = tr.len > 0 && tv ? tv[tr.len - 1] : first;
    if (tr.len == 0 || last != final_err) {
        CGH_TRY(tr.push(executed, final_err));
        if (cb && cb->progress) cb->progress(cb->user, executed, final_err);
    }
    if (lcap > 0 && sp->log_pixel) {
        CGH_CUDA(cudaMemcpyAsync(sp->log_pixel, dlog_p, sizeof(long long) * lcap, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaMemcpyAsync(sp->log_level, dlog_l, sizeof(int) * lcap, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaMemcpyAsync(sp->log_accept, dlog_a, lcap, cudaMemcpyDeviceToHost, P->st));
    }
    if (dlog_p) CGH_CUDA(cudaFreeAsync(dlog_p, P->st));
    if (dprobe) {
        long long hp[8];
        CGH_CUDA(cudaMemcpyAsync(hp, dprobe, sizeof(hp), cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        const double it = hp[7] > 0 ? double(hp[7]) : 1.0;
        fprintf(stderr, "[sa probe] %lld sweeps, cycles per sweep: top %.0f draw %.0f sweep %.0f block-sum %.0f "
                "grid-reduce %.0f decide %.0f\n", hp[7], hp[1] / it, hp[2] / it, hp[3] / it, hp[4] / it, hp[5] / it,
                hp[6] / it);
        CGH_CUDA(cudaFreeAsync(dprobe, P->st));
    }
    CGH_CUDA(cudaEventRecord(P->ev1, P->st));
    CGH_CUDA(cudaEventSynchronize(P->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, P->ev0, P->ev1);
    if (rep) {
        rep->final_error = final_err;
        rep->efficiency = eff;
        rep->iterations_executed = executed;
        rep->termination = stop ? CGH_CANCELLED : CGH_COMPLETED;
        rep->trace_len = tr.len;
        rep->kernel_launches = P->launches - launches0;
        rep->device_ms = ms;
    }
    return CGH_OK;
}

static int dbs_exec(cgh_plan* P, const cgh_dbs_params* dp, int64_t* tk, double* tv, int64_t cap, cgh_report* rep,
                    const cgh_callbacks* cb) {
    GateLock gate(P->dev, true);   // grid-barrier kernels: the device to this run (runtime.cuh)
    if (P->prec != CGH_FP64) return fail(CGH_ERR_VALUE, "search runs need an fp64 plan");
    if (dp->init_mode != CGH_INIT_RANDOM_PHASE && dp->init_mode != CGH_INIT_BACKPROPAGATE)
        return fail(CGH_ERR_VALUE, "unknown init mode %d", dp->init_mode);
    if (dp->init_mode == CGH_INIT_BACKPROPAGATE && P->nf_all > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf");
    if (P->denom == 0) return fail(CGH_ERR_ZERO_TARGET, "target is zero inside the mask");
    if (P->nstates > kMaxLevels) return fail(CGH_ERR_UNSUPPORTED, "DBS implements up to %d levels", kMaxLevels);
    if (dp->scan_random && dp->max_passes > 0 && !dp->pass_rng) return fail(CGH_ERR_VALUE, "pass streams missing");
    const long launches0 = P->launches;
    CGH_CUDA(cudaEventRecord(P->ev0, P->st));
    SearchRun S;
    S.P = P;
    struct Guard {
        SearchRun* s;
        ~Guard() { search_free(*s); }
    } guard{&S};
    CGH_TRY(search_setup(S, dp->init_mode, dp->rng, true));
    double sums[4];
    CGH_TRY(search_sums(S, 1.0, sums));
    double error_num = sums[0];
    SearchState st0;
    memset(&st0, 0, sizeof(st0));
    st0.error_num = error_num;
    st0.window = 1;
    CGH_CUDA(cudaMemcpyAsync(S.st, &st0, sizeof(st0), cudaMemcpyHostToDevice, P->st));
    TraceOut tr{tk, tv, cap};
    double first;
    CGH_TRY(reported_error(S, error_num, P->denom, P->rescale, &first));
    CGH_TRY(tr.push(0, first));
    if (cb && cb->progress) cb->progress(cb->user, 0, first);
    const long long n = (long long)P->H * P->W;
    long long* order = nullptr;
    std::vector<int64_t> perm;
    if (dp->scan_random) {
        CGH_TRY(search_alloc(S, sizeof(long long) * n, reinterpret_cast<void**>(&order)));
        perm.resize(n);
    }
    SearchArgs a = search_args(S);
    a.order = order;
    a.p_end = n;
    a.wmax = dbs_wmax(P->nstates);
    long long* dlog_p = nullptr;
    int* dlog_l = nullptr;
    double* dlog_c = nullptr;
    const long long lcap = std::max<long long>(0, dp->log_cap);
    if (lcap > 0) {
        CGH_TRY(search_alloc(S, (sizeof(long long) + sizeof(int) + sizeof(double)) * lcap + 64, reinterpret_cast<void**>(&dlog_p)));
        dlog_c = reinterpret_cast<double*>(dlog_p + lcap);
        dlog_l = reinterpret_cast<int*>(dlog_c + lcap);
    }
    a.log_cap = lcap;
    a.log_pixel = dlog_p;
    a.log_level = dlog_l;
    a.log_change = dlog_c;
    int passes = 0;
    bool stop = false, converged = false;
    long long logged = 0;
    for (int pass = 0; pass < dp->max_passes; ++pass) {
        if (cancelled(cb)) {
            stop = true;
            break;
        }
        if (dp->scan_random) {
            CGH_TRY(cgh_permutation(&dp->pass_rng[pass], n, perm.data()));
            CGH_CUDA(cudaMemcpyAsync(order, perm.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, P->st));
        }
        SearchState sh;
        CGH_CUDA(cudaMemcpyAsync(&sh, S.st, sizeof(sh), cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        sh.executed = 0;
        sh.commits = 0;
        sh.logged = logged;
        CGH_CUDA(cudaMemcpyAsync(S.st, &sh, sizeof(sh), cudaMemcpyHostToDevice, P->st));
        CGH_TRY(launch_search(S, true, a));
        CGH_CUDA(cudaMemcpyAsync(&sh, S.st, sizeof(sh), cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));
        error_num = sh.error_num;
        logged = sh.logged;
        passes += 1;
        if (sh.commits > 0) {
            double e;
            CGH_TRY(reported_error(S, error_num, P->denom, P->rescale, &e));
            CGH_TRY(tr.push(passes, e));
            if (cb && cb->progress) cb->progress(cb->user, passes, e);
            if (cb && cb->audit) CGH_TRY(audit_call(S, cb, passes, error_num / P->denom));
        } else {
            converged = true;
            break;
        }
    }
    double final_err, eff;
    CGH_TRY(search_final(S, error_num, P->rescale, &final_err, &eff));
    const double last = tv && tr.len > 0 ? tv[tr.len - 1] : first;
    if (tr.len == 0 || last != final_err) {
        CGH_TRY(tr.push(passes, final_err));
        if (cb && cb->progress) cb->progress(cb->user, passes, final_err);
    }
    if (lcap > 0 && dp->log_pixel) {
        const long long nl = std::min(lcap, logged);
        CGH_CUDA(cudaMemcpyAsync(dp->log_pixel, dlog_p, sizeof(long long) * nl, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaMemcpyAsync(dp->log_level, dlog_l, sizeof(int) * nl, cudaMemcpyDeviceToHost, P->st));
        CGH_CUDA(cudaMemcpyAsync(dp->log_change, dlog_c, sizeof(double) * nl, cudaMemcpyDeviceToHost, P->st));
        for (long long i = nl; i < lcap; ++i) dp->log_level[i] = -2;   // not reached
    }
    if (dlog_p) CGH_CUDA(cudaFreeAsync(dlog_p, P->st));
    if (order) CGH_CUDA(cudaFreeAsync(order, P->st));
    CGH_CUDA(cudaEventRecord(P->ev1, P->st));
    CGH_CUDA(cudaEventSynchronize(P->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, P->ev0, P->ev1);
    if (rep) {
        rep->final_error = final_err;
        rep->efficiency = eff;
        rep->iterations_executed = passes;
        rep->termination = stop ? CGH_CANCELLED : (converged ? CGH_CONVERGED : CGH_COMPLETED);
        rep->trace_len = tr.len;
        rep->kernel_launches = P->launches - launches0;
        rep->device_ms = ms;
    }
    return CGH_OK;
}

static int seam_prep(int32_t device, cudaStream_t* st) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    CGH_CUDA(cudaSetDevice(device));
    CGH_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    return CGH_OK;
}

}  // namespace cgh

using namespace cgh;

extern "C" {

int cgh_sa_run(const cgh_problem* pb, const cgh_sa_params* sp, const double* target, const uint8_t* mask,
               const double* illumination, void* out_idx, int64_t* trace_k, double* trace_v, int64_t trace_cap,
               cgh_report* rep, const cgh_callbacks* cb) {
    if (!pb || !sp) return fail(CGH_ERR_VALUE, "null argument");
    cgh_problem p = *pb;
    p.precision = CGH_FP64;
    cgh_plan* P = nullptr;
    CGH_TRY(cgh_plan_create(&p, &P));
    struct G {
        cgh_plan* p;
        ~G() { cgh_plan_destroy(p); }
    } g{P};
    CGH_TRY(plan_upload_target(P, target, mask, illumination));
    cgh_report r{};
    CGH_TRY(sa_exec(P, sp, trace_k, trace_v, trace_cap, &r, cb));
    if (rep) *rep = r;
    if (out_idx) CGH_TRY(cgh_plan_download_idx(P, out_idx, 1));
    return CGH_OK;
}

int cgh_dbs_run(const cgh_problem* pb, const cgh_dbs_params* dp, const double* target, const uint8_t* mask,
                const double* illumination, void* out_idx, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                cgh_report* rep, const cgh_callbacks* cb) {
    if (!pb || !dp) return fail(CGH_ERR_VALUE, "null argument");
    cgh_problem p = *pb;
    p.precision = CGH_FP64;
    cgh_plan* P = nullptr;
    CGH_TRY(cgh_plan_create(&p, &P));
    struct G {
        cgh_plan* p;
        ~G() { cgh_plan_destroy(p); }
    } g{P};
    CGH_TRY(plan_upload_target(P, target, mask, illumination));
    cgh_report r{};
    CGH_TRY(dbs_exec(P, dp, trace_k, trace_v, trace_cap, &r, cb));
    if (rep) *rep = r;
    if (out_idx) CGH_TRY(cgh_plan_download_idx(P, out_idx, 1));
    return CGH_OK;
}

int cgh_plan_sa(cgh_plan* plan, const cgh_sa_params* sp, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                cgh_report* rep, const cgh_callbacks* cb) {
    if (!plan || !sp) return fail(CGH_ERR_VALUE, "null argument");
    CGH_CUDA(cudaSetDevice(plan->dev));
    return sa_exec(plan, sp, trace_k, trace_v, trace_cap, rep, cb);
}

int cgh_plan_dbs(cgh_plan* plan, const cgh_dbs_params* dp, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                 cgh_report* rep, const cgh_callbacks* cb) {
    if (!plan || !dp) return fail(CGH_ERR_VALUE, "null argument");
    CGH_CUDA(cudaSetDevice(plan->dev));
    return dbs_exec(plan, dp, trace_k, trace_v, trace_cap, rep, cb);
}

// kernels/_core.pyx:20-34
int cgh_delta_error(int32_t device, const double* replay_m, const double* target_m, const double* row_tw,
                    const double* col_tw, const int32_t* mu, const int32_t* mv, int64_t count, int32_t h, int32_t w,
                    double delta_re, double delta_im, double* out) {
    double d[2] = {delta_re, delta_im};
    int64_t bi = 0;
    double bc = 0;
    (void)bi;
    (void)bc;
    // evaluate a single level through the best_delta machinery
    cudaStream_t st;
    CGH_TRY(seam_prep(device, &st));
    const size_t n = size_t(std::max<int64_t>(count, 0));
    char* buf = nullptr;
    const int grid = grid_for(std::max<int64_t>(count, 1));
    const size_t bytes = n * 16 + n * 8 + n * 8 + size_t(h) * 16 + size_t(w) * 16 + 16 + size_t(grid) * 8 + 64 + 64;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st);
    if (e == cudaSuccess) {
        double2* R = reinterpret_cast<double2*>(buf);
        double* t = reinterpret_cast<double*>(R + n);
        int32_t* m_ = reinterpret_cast<int32_t*>(t + n);
        int32_t* v_ = m_ + n;
        double2* rtw = reinterpret_cast<double2*>(v_ + n);
        double2* ctw = rtw + h;
        double2* dl = ctw + w;
        double* part = reinterpret_cast<double*>(dl + 1);
        double* res = part + grid;
        unsigned* ctr = reinterpret_cast<unsigned*>(res + 4);
        cudaMemcpyAsync(R, replay_m, n * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(t, target_m, n * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(m_, mu, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(v_, mv, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(rtw, row_tw, size_t(h) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(ctw, col_tw, size_t(w) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dl, d, 16, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(ctr, 0, 16, st);
        cudaMemsetAsync(res, 0, 32, st);
        seam_eval_kernel<<<dim3(grid, 1), 256, 0, st>>>(R, t, rtw, ctw, m_, v_, (long long)n, dl, 1, part, ctr, res);
        cudaMemcpyAsync(out, res, 8, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(buf, st);
        e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "delta_error: %s", cudaGetErrorString(e));
    return CGH_OK;
}

// kernels/_core.pyx:37-44
int cgh_commit_update(int32_t device, double* replay_m, const double* row_tw, const double* col_tw, const int32_t* mu,
                      const int32_t* mv, int64_t count, int32_t h, int32_t w, double delta_re, double delta_im) {
    cudaStream_t st;
    CGH_TRY(seam_prep(device, &st));
    const size_t n = size_t(std::max<int64_t>(count, 0));
    char* buf = nullptr;
    const size_t bytes = n * 16 + n * 8 + size_t(h) * 16 + size_t(w) * 16 + 64;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st);
    if (e == cudaSuccess) {
        double2* R = reinterpret_cast<double2*>(buf);
        int32_t* m_ = reinterpret_cast<int32_t*>(R + n);
        int32_t* v_ = m_ + n;
        double2* rtw = reinterpret_cast<double2*>(v_ + n);
        double2* ctw = rtw + h;
        cudaMemcpyAsync(R, replay_m, n * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(m_, mu, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(v_, mv, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(rtw, row_tw, size_t(h) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(ctw, col_tw, size_t(w) * 16, cudaMemcpyHostToDevice, st);
        if (n) seam_commit_kernel<<<grid_for(count), 256, 0, st>>>(R, rtw, ctw, m_, v_, (long long)n, make_double2(delta_re, delta_im));
        cudaMemcpyAsync(replay_m, R, n * 16, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(buf, st);
        e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "commit_update: %s", cudaGetErrorString(e));
    return CGH_OK;
}

// kernels/_core.pyx:47-83
int cgh_best_delta(int32_t device, const double* replay_m, const double* target_m, const double* row_tw,
                   const double* col_tw, const int32_t* mu, const int32_t* mv, int64_t count, int32_t h, int32_t w,
                   const double* deltas, int64_t levels, int64_t* best_index, double* best_change) {
    if (levels < 0 || levels > 256) return fail(CGH_ERR_UNSUPPORTED, "best_delta implements up to 256 levels");
    cudaStream_t st;
    CGH_TRY(seam_prep(device, &st));
    const size_t n = size_t(std::max<int64_t>(count, 0));
    const int L = int(std::max<int64_t>(levels, 1));
    char* buf = nullptr;
    const int grid = grid_for(std::max<int64_t>(count, 1));
    const size_t bytes = n * 16 + n * 8 + n * 8 + size_t(h) * 16 + size_t(w) * 16 + size_t(L) * 16 +
                         size_t(grid) * L * 8 + size_t(L) * 8 + 64;
    std::vector<double> sums(L, 0.0);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st);
    if (e == cudaSuccess) {
        double2* R = reinterpret_cast<double2*>(buf);
        double* t = reinterpret_cast<double*>(R + n);
        int32_t* m_ = reinterpret_cast<int32_t*>(t + n);
        int32_t* v_ = m_ + n;
        double2* rtw = reinterpret_cast<double2*>(v_ + n);
        double2* ctw = rtw + h;
        double2* dl = ctw + w;
        double* part = reinterpret_cast<double*>(dl + L);
        double* res = part + size_t(grid) * L;
        unsigned* ctr = reinterpret_cast<unsigned*>(res + L);
        cudaMemcpyAsync(R, replay_m, n * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(t, target_m, n * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(m_, mu, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(v_, mv, n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(rtw, row_tw, size_t(h) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(ctw, col_tw, size_t(w) * 16, cudaMemcpyHostToDevice, st);
        if (levels) cudaMemcpyAsync(dl, deltas, size_t(levels) * 16, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(ctr, 0, 16, st);
        cudaMemsetAsync(res, 0, size_t(L) * 8, st);
        if (levels) seam_eval_kernel<<<dim3(grid, L), 256, 0, st>>>(R, t, rtw, ctw, m_, v_, (long long)n, dl, L, part, ctr, res);
        cudaMemcpyAsync(sums.data(), res, size_t(L) * 8, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(buf, st);
        e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "best_delta: %s", cudaGetErrorString(e));
    int64_t bj = -1;
    double bcv = 0.0;
    for (int64_t j = 0; j < levels; ++j) {
        if (deltas[2 * j] == 0.0 && deltas[2 * j + 1] == 0.0) continue;
        if (sums[j] < bcv) {
            bcv = sums[j];
            bj = j;
        }
    }
    *best_index = bj;
    *best_change = bcv;
    return CGH_OK;
}

}  // extern "C"
