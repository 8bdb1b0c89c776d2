// Host side of the warp-line 2048^2 GS passes (wl_passes.cuh).
#include "launch.cuh"
#include "runtime.cuh"
#include "wl_passes.cuh"
#include "wl_ospr.cuh"

namespace cgh {

struct WlState {
    DevBuf t4, tgt_perm, beam_perm, line_sums, stamps, bar;
    const void* tgt_src = nullptr;
    const void* beam_src = nullptr;
    bool beam_ready = false;
    // OSPR: row-ordered target table, column-ordered beam table, line states,
    // intensity, digit-reversed index bytes, per-row sums
    DevBuf o_tgt, o_beam, o_states, o_inten, o_idx, o_sums, o_jumps;
    const void* o_tgt_src = nullptr;
    bool o_beam_ready = false;
};

static WlState* wl_state(cgh_plan* P) { return static_cast<WlState*>(P->wlst); }

bool wl_eligible(cgh_plan* P) {
    if (P->prec != CGH_FP32 || P->H != wl::N || P->W != wl::N) return false;
    if (getenv("CGHB200_NO_FAST") || getenv("CGHB200_NO_WL")) return false;
    return true;
}

void wl_free(cgh_plan* P) {
    WlState* S = wl_state(P);
    if (!S) return;
    DevBuf* bufs[] = {&S->t4,      &S->tgt_perm, &S->beam_perm, &S->line_sums, &S->stamps, &S->bar,
                      &S->o_tgt,   &S->o_beam,   &S->o_states,  &S->o_inten,   &S->o_idx,   &S->o_sums,
                      &S->o_jumps};
    for (DevBuf* b : bufs)
        if (b->p) cudaFreeAsync(b->p, P->st);
    delete S;
    P->wlst = nullptr;
}

void wl_invalidate_target(cgh_plan* P) {
    WlState* S = wl_state(P);
    if (S) {
        S->tgt_src = nullptr;
        S->beam_ready = false;
        S->o_tgt_src = nullptr;
        S->o_beam_ready = false;
    }
}

// Device buffers and the digit-reversed target / beam tables of this plan.
int wl_prepare(cgh_plan* P) {
    WlState* S = wl_state(P);
    if (!S) {
        S = new WlState();
        P->wlst = S;
    }
    const long long n = (long long)wl::N * wl::N;
    CGH_TRY(ensure(P, S->t4, size_t(n) * 8));
    CGH_TRY(ensure(P, S->line_sums, size_t(wl::N) * 3 * sizeof(double)));
    if (S->tgt_src != P->tgt.p || !S->tgt_perm.p) {
        CGH_TRY(ensure(P, S->tgt_perm, size_t(n) * 4));
        const float inv_scale = float(std::sqrt(double(P->H) * double(P->W)));
        wl::perm_table_kernel<<<grid_for(n), 256, 0, P->st>>>(static_cast<const float*>(P->tgt.p),
                                                             static_cast<float*>(S->tgt_perm.p), inv_scale, 1);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        S->tgt_src = P->tgt.p;
        S->beam_ready = false;
    }
    if (P->has_beam && !S->beam_ready) {
        CGH_TRY(ensure(P, S->beam_perm, size_t(n) * 4));
        wl::perm_table_kernel<<<grid_for(n), 256, 0, P->st>>>(static_cast<const float*>(P->beam.p),
                                                             static_cast<float*>(S->beam_perm.p), 1.0f, 0);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        S->beam_ready = true;
    }
    return CGH_OK;
}

int wl_relayout(cgh_plan* P, int to_t4) {
    WlState* S = wl_state(P);
    const float2* src = static_cast<const float2*>(to_t4 ? P->data.p : S->t4.p);
    float2* dst = static_cast<float2*>(to_t4 ? S->t4.p : P->data.p);
    wl::relayout_kernel<<<grid_for(long(wl::N) * wl::N), 256, 0, P->st>>>(src, dst, to_t4);
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

template <int PASS, int MODE>
static cudaError_t wl_launch_m(cgh_plan* P, const wl::Args& w) {
    if (cudaError_t e = ensure_smem_attr<wl::wl_pass<PASS, MODE>>(wl::SMEM); e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->dev);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max(1, sms));
    cfg.blockDim = dim3(wl::THREADS);
    cfg.dynamicSmemBytes = wl::SMEM;
    cfg.stream = P->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wl::wl_pass<PASS, MODE>, w);
}

static wl::Args wl_args(cgh_plan* P, const PassArgs<float>& a) {
    WlState* S = wl_state(P);
    wl::Args w;
    w.data = static_cast<float2*>(S->t4.p);
    w.tgt_perm = static_cast<const float*>(S->tgt_perm.p);
    w.beam_perm = P->has_beam ? static_cast<const float*>(S->beam_perm.p) : nullptr;
    w.tw = a.tw_row;
    w.q_row = a.q_row;
    w.q_col = a.q_col;
    w.gain = a.gain;
    w.scale = a.scale;
    w.line_sums = static_cast<double*>(S->line_sums.p);
    w.red = a.red;
    w.stamps = nullptr;
    w.no_stagger = getenv("CGHB200_WL_STAGGER") ? 0 : 1;   // measured: no gain
    const char* dbg = getenv("CGHB200_WL_DEBUG");
    w.debug = dbg ? atoi(dbg) : 0;
    return w;
}

// timing experiments: stamps of the last launch of each pass type
static int wl_stamp_buf(cgh_plan* P, wl::Args& w, int pass) {
    if (!P->profiling || !getenv("CGHB200_WL_STAMPS")) return CGH_OK;
    WlState* S = wl_state(P);
    const size_t per = size_t(1024) * wl::WARPS * 8 * 2;   // up to 1024 CTAs
    CGH_TRY(ensure(P, S->stamps, 2 * per * sizeof(long long)));
    w.stamps = static_cast<long long*>(S->stamps.p) + size_t(pass) * per;
    return CGH_OK;
}

int wl_col(cgh_plan* P, const PassArgs<float>& a) {
    wl::Args w = wl_args(P, a);
    CGH_TRY(wl_stamp_buf(P, w, wl::COL));
    const int mode = (P->rescale ? 1 : 0) | (a.gain != 0.0f ? 2 : 0);
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_GS, true));
    cudaError_t e;
    switch (mode) {
        case 0: e = wl_launch_m<wl::COL, 0>(P, w); break;
        case 1: e = wl_launch_m<wl::COL, 1>(P, w); break;
        case 2: e = wl_launch_m<wl::COL, 2>(P, w); break;
        default: e = wl_launch_m<wl::COL, 3>(P, w); break;
    }
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_GS, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "warp-line column pass: %s", cudaGetErrorString(e));
    return CGH_OK;
}

int wl_row(cgh_plan* P, const PassArgs<float>& a) {
    wl::Args w = wl_args(P, a);
    CGH_TRY(wl_stamp_buf(P, w, wl::ROW));
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_HOLO, true));
    const cudaError_t e = wl_launch_m<wl::ROW, 0>(P, w);
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_HOLO, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "warp-line row pass: %s", cudaGetErrorString(e));
    return CGH_OK;
}

template <int MODE>
static cudaError_t wl_loop_m(cgh_plan* P, const wl::Args& w, int iters, unsigned* bar) {
    if (cudaError_t e = ensure_smem_attr<wl::wl_loop<MODE>>(wl::SMEM); e != cudaSuccess) return e;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->dev);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max(1, sms));   // one CTA per SM: all resident (cooperative launch checks)
    cfg.blockDim = dim3(wl::THREADS);
    cfg.dynamicSmemBytes = wl::SMEM;
    cfg.stream = P->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, wl::wl_loop<MODE>, w, iters, bar);
}

// Iterations 0..iters-1 of run_gs in one persistent launch (replay-plane
// passes of all of them, hologram-plane passes of all but the last), then the
// per-iteration errors into P->res_d[2k].
int wl_gs_loop(cgh_plan* P, const PassArgs<float>& a, int iters) {
    WlState* S = wl_state(P);
    CGH_TRY(ensure(P, S->line_sums, size_t(std::max(iters, 1)) * 3 * wl::N * sizeof(double)));
    CGH_TRY(ensure(P, S->bar, 64));
    CGH_CUDA(cudaMemsetAsync(S->bar.p, 0, 4, P->st));
    wl::Args w = wl_args(P, a);
    w.line_sums = static_cast<double*>(S->line_sums.p);
    CGH_TRY(wl_stamp_buf(P, w, 0));
    // MODE bit 2: every pixel inside the metric mask (the projection drops its mask selects)
    const bool full = P->count_in == double(P->H) * double(P->W);
    const int mode = (P->rescale ? 1 : 0) | (a.gain != 0.0f ? 2 : 0) | (full ? 4 : 0);
    if (P->profiling) CGH_TRY(prof_mark(P, 16 + 7, true));
    cudaError_t e;
    unsigned* bar = static_cast<unsigned*>(S->bar.p);
    switch (mode) {
        case 0: e = wl_loop_m<0>(P, w, iters, bar); break;
        case 1: e = wl_loop_m<1>(P, w, iters, bar); break;
        case 2: e = wl_loop_m<2>(P, w, iters, bar); break;
        case 3: e = wl_loop_m<3>(P, w, iters, bar); break;
        case 4: e = wl_loop_m<4>(P, w, iters, bar); break;
        case 5: e = wl_loop_m<5>(P, w, iters, bar); break;
        case 6: e = wl_loop_m<6>(P, w, iters, bar); break;
        default: e = wl_loop_m<7>(P, w, iters, bar); break;
    }
    if (P->profiling) CGH_TRY(prof_mark(P, 16 + 7, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "warp-line GS loop: %s", cudaGetErrorString(e));
    wl::wl_trace_kernel<<<std::min(iters, 148), 96, 0, P->st>>>(w.line_sums, iters, a.red.denom, P->rescale ? 1 : 0,
                                                               P->res_d);
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

// Opt-in (CGHB200_WL_OSPR=1): measured on B200 at 2048^2 x 24 binary, the
// loop takes 1.54 ms + 0.25 ms of table / permute kernels against 1.62 ms for
// the batched fast passes (fast_ospr_gen / fast_col_holo / fast_ospr_acc):
// OSPR's per-pixel PCG64 draws and snapping, not its plane traffic, bound both
// (DESIGN.md section 3.2), so the default stays with the batched passes.
bool wl_ospr_eligible(cgh_plan* P) {
    return wl_eligible(P) && getenv("CGHB200_WL_OSPR") != nullptr;
}

// All S subframes of run_ospr in one persistent launch (wl_ospr.cuh), then
// the per-subframe errors / efficiency into P->res_d[0..S] and the index
// planes into P->idx (row-major, S frames). a.frame_rng holds the S streams.
int wl_ospr_run(cgh_plan* P, const PassArgs<float>& a, int S_frames) {
    WlState* S = wl_state(P);
    if (!S) {
        S = new WlState();
        P->wlst = S;
    }
    const long long n = (long long)wl::N * wl::N;
    CGH_TRY(ensure(P, S->t4, size_t(n) * 8));
    CGH_TRY(ensure(P, S->bar, 64));
    if (S->o_tgt_src != P->tgt.p || !S->o_tgt.p) {
        CGH_TRY(ensure(P, S->o_tgt, size_t(n) * 4));
        wl::perm_table_kernel<<<grid_for(n), 256, 0, P->st>>>(static_cast<const float*>(P->tgt.p),
                                                             static_cast<float*>(S->o_tgt.p), 1.0f, 0);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        S->o_tgt_src = P->tgt.p;
        S->o_beam_ready = false;
    }
    if (P->has_beam && !S->o_beam_ready) {
        CGH_TRY(ensure(P, S->o_beam, size_t(n) * 4));
        wl::perm_table_kernel<<<grid_for(n), 256, 0, P->st>>>(static_cast<const float*>(P->beam.p),
                                                             static_cast<float*>(S->o_beam.p), 1.0f, 1);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        S->o_beam_ready = true;
    }
    CGH_TRY(ensure(P, S->o_states, sizeof(Pcg64) * size_t(S_frames) * wl::N));
    CGH_TRY(ensure(P, S->o_inten, size_t(n) * 4));
    CGH_TRY(ensure(P, S->o_idx, size_t(n) * S_frames));
    CGH_TRY(ensure(P, S->o_sums, sizeof(double) * (size_t(S_frames) * wl::N * 3 + size_t(wl::N) * 2)));
    const int lines = S_frames * wl::N;
    wl::ospr_line_states_kernel<<<(lines + 255) / 256, 256, 0, P->st>>>(a.frame_rng, S_frames,
                                                                       static_cast<Pcg64*>(S->o_states.p));
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    CGH_CUDA(cudaMemsetAsync(S->bar.p, 0, 4, P->st));
    wl::OsprArgs o;
    o.data = static_cast<float2*>(S->t4.p);
    o.tgt_row = static_cast<const float*>(S->o_tgt.p);
    o.beam_col = P->has_beam ? static_cast<const float*>(S->o_beam.p) : nullptr;
    o.line_state = static_cast<const Pcg64*>(S->o_states.p);
    o.inten = static_cast<float*>(S->o_inten.p);
    o.idx_perm = static_cast<uint8_t*>(S->o_idx.p);
    o.sums = static_cast<double*>(S->o_sums.p);
    o.tw = a.tw_row;
    o.q_row = a.q_row;
    o.q_col = a.q_col;
    o.scheme = a.scheme;
    o.binary = (P->scheme_kind == CGH_SCHEME_PHASE && P->nstates == 2 && P->offset == 0.0) ? 1 : 0;
    o.scale = a.scale;
    o.S = S_frames;
    // LCG jumps (host-computed, as jump_of): by 256, by 2, and by every first column
    auto host_jump = [](uint64_t k) {
        wl::Jump j;
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
        j.A = acc_m;
        j.G = acc_g;
        return j;
    };
    if (!S->o_jumps.p) {
        std::vector<wl::Jump> jt(wl::kJumps);
        for (int c = 0; c < wl::kJumps; ++c) jt[c] = host_jump(uint64_t(c));
        CGH_TRY(ensure(P, S->o_jumps, sizeof(wl::Jump) * jt.size()));
        CGH_CUDA(cudaMemcpyAsync(S->o_jumps.p, jt.data(), sizeof(wl::Jump) * jt.size(), cudaMemcpyHostToDevice, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));   // jt is a temporary
    }
    o.jumps = static_cast<const wl::Jump*>(S->o_jumps.p);
    o.j256 = host_jump(256);
    o.j2 = host_jump(2);
    if (cudaError_t e = ensure_smem_attr<wl::ospr_loop>(wl::SMEM); e != cudaSuccess)
        return fail(CGH_ERR_CUDA, "warp-line OSPR: %s", cudaGetErrorString(e));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->dev);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(std::max(1, sms));
    cfg.blockDim = dim3(wl::THREADS);
    cfg.dynamicSmemBytes = wl::SMEM;
    cfg.stream = P->st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (P->profiling) CGH_TRY(prof_mark(P, 22, true));
    const cudaError_t e = cudaLaunchKernelEx(&cfg, wl::ospr_loop, o, static_cast<unsigned*>(S->bar.p));
    if (P->profiling) CGH_TRY(prof_mark(P, 22, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "warp-line OSPR loop: %s", cudaGetErrorString(e));
    wl::ospr_trace_kernel<<<std::min(S_frames + 1, 148), 96, 0, P->st>>>(o.sums, S_frames, a.red.denom,
                                                                        P->rescale ? 1 : 0, P->res_d);
    wl::ospr_idx_kernel<<<4 * sms, 256, 0, P->st>>>(o.idx_perm, static_cast<uint8_t*>(P->idx.p), S_frames);
    P->launches += 2;
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

}  // namespace cgh

extern "C" int cgh_debug_wl_stamps(cgh_plan* plan, int64_t* out, int64_t cap) {
    using namespace cgh;
    if (!plan || !out) return fail(CGH_ERR_VALUE, "bad arguments");
    WlState* S = wl_state(plan);
    if (!S || !S->stamps.p) return fail(CGH_ERR_VALUE, "no warp-line stamps recorded (CGHB200_WL_STAMPS + profiling)");
    CGH_CUDA(cudaSetDevice(plan->dev));
    CGH_CUDA(cudaStreamSynchronize(plan->st));
    const size_t n = std::min<size_t>(size_t(cap), S->stamps.cap / sizeof(long long));
    CGH_CUDA(cudaMemcpy(out, S->stamps.p, n * sizeof(long long), cudaMemcpyDeviceToHost));
    return CGH_OK;
}
