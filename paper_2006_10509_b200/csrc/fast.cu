// Host side of the pipelined complex64 GS passes (fast_passes.cuh).
#include <cudaTypedefs.h>

#include "fast_passes.cuh"
#include "launch.cuh"
#include "runtime.cuh"

namespace cgh {

struct FastState {
    CUtensorMap tmap;           // data as float32 [H][2W], box {2C, 256}
    const void* tmap_ptr = nullptr;
    int H = 0, W = 0;
    CUtensorMap tmap_frames;    // OSPR frames stacked: float32 [F*H][2W]
    const void* tmapf_ptr = nullptr;
    int tmapf_rows = 0;
    int tmapf_c = 0;
    DevBuf tgt_tiled, ctr, line_state, line_part;
    const void* tgt_src = nullptr;
};

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Launch configurations: rows 256 threads x 2 CTAs/SM (2 rows per tile);
// columns 512 threads x 1 CTA/SM (4 columns = 32 B per row segment) or, with
// CGHB200_COL_TH=256, 256 x 2 (2 columns).
constexpr int kRowTH = 256, kRowMinB = 2;

static int col_th() {
    static int v = 0;
    if (!v) {
        const char* e = getenv("CGHB200_COL_TH");
        v = (e && atoi(e) == 256) ? 256 : 512;
    }
    return v;
}

static int fast_lines_th(int n, int th) {
    switch (n) {
        case 256: return th / (256 / 16);
        case 512: return th / (512 / 16);
        case 1024: return th / (1024 / 16);
        case 2048: return th / (2048 / 16);
        case 4096: return th / (4096 / 16);
        default: return 0;
    }
}

bool fast_eligible(cgh_plan* P) {
    if (P->prec != CGH_FP32) return false;
    const int lr = fast_lines_th(P->W, kRowTH), lc = fast_lines_th(P->H, col_th());
    if (lr < 1 || lc < 1 || P->W < 512) return false;   // row groups are whole warps (W >= 512)
    if (P->H < lr || P->W < lc) return false;
    if (getenv("CGHB200_NO_FAST")) return false;
    return encode_fn() != nullptr;
}

void fast_free(cgh_plan* P) {
    FastState* F = static_cast<FastState*>(P->fast);
    if (!F) return;
    if (F->tgt_tiled.p) cudaFreeAsync(F->tgt_tiled.p, P->st);
    if (F->line_state.p) cudaFreeAsync(F->line_state.p, P->st);
    if (F->line_part.p) cudaFreeAsync(F->line_part.p, P->st);
    if (F->ctr.p) cudaFreeAsync(F->ctr.p, P->st);
    delete F;
    P->fast = nullptr;
}

// Tensor map over the data buffer, tiled target, tile counters.
int fast_prepare(cgh_plan* P) {
    FastState* F = static_cast<FastState*>(P->fast);
    if (!F) {
        F = new FastState();
        P->fast = F;
    }
    const int C = fast_lines_th(P->H, col_th());
    if (F->tmap_ptr != P->data.p || F->H != P->H || F->W != P->W) {
        cuuint64_t dims[2] = {cuuint64_t(2) * P->W, cuuint64_t(P->H)};
        cuuint64_t strides[1] = {cuuint64_t(P->W) * 8};
        cuuint32_t box[2] = {cuuint32_t(2 * C), cuuint32_t(std::min(kFastBoxRows, P->H))};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = encode_fn()(&F->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, P->data.p, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(CGH_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
        F->tmap_ptr = P->data.p;
        F->H = P->H;
        F->W = P->W;
    }
    if (!F->ctr.p) {
        CGH_TRY(ensure(P, F->ctr, 64));
        CGH_CUDA(cudaMemsetAsync(F->ctr.p, 0, 64, P->st));
    }
    if (F->tgt_src != P->tgt.p || !F->tgt_tiled.p) {
        const long long n = (long long)P->H * P->W;
        CGH_TRY(ensure(P, F->tgt_tiled, size_t(n) * 4));
        const float inv_scale = float(std::sqrt(double(P->H) * double(P->W)));
        tile_target_kernel<<<grid_for(n), 256, 0, P->st>>>(static_cast<const float*>(P->tgt.p),
                                                          static_cast<float*>(F->tgt_tiled.p), P->H, P->W, C,
                                                          inv_scale);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        F->tgt_src = P->tgt.p;
    }
    return CGH_OK;
}

void fast_invalidate_target(cgh_plan* P) {
    FastState* F = static_cast<FastState*>(P->fast);
    if (F) F->tgt_src = nullptr;
}

static FastArgs fast_args(cgh_plan* P, const PassArgs<float>& a) {
    FastState* F = static_cast<FastState*>(P->fast);
    FastArgs f;
    f.data = reinterpret_cast<float2*>(a.data);
    f.H = P->H;
    f.W = P->W;
    f.beam = a.beam;
    f.tw_row = a.tw_row;
    f.tw_col = a.tw_col;
    f.q_row = a.q_row;
    f.q_col = a.q_col;
    f.tgt_tiled = static_cast<const float*>(F->tgt_tiled.p);
    f.gain = a.gain;
    f.scale = a.scale;
    f.tile_ctr = static_cast<unsigned*>(F->ctr.p);
    f.red = a.red;
    const char* dbg = getenv("CGHB200_FAST_DEBUG");
    f.debug = dbg ? atoi(dbg) : 0;
    return f;
}

static int sm_count(int dev) {
    static int cached[64] = {0};
    if (!cached[dev & 63]) cudaDeviceGetAttribute(&cached[dev & 63], cudaDevAttrMultiProcessorCount, dev);
    return cached[dev & 63];
}

template <class K, class... Args>
static cudaError_t launch_pdl(K kernel, int grid, int block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

template <int N, int MINB>
static cudaError_t row_launch_s(cgh_plan* P, const FastArgs& f) {
    using S = FastShape<N, kRowTH>;
    const size_t smem = (size_t(TwTables<N, kRowTH>::WORDS) + size_t(S::LINES) * ((S::LW + 15) / 16 * 16)) * sizeof(float2);
    auto k = fast_row_holo_s<N, kRowTH, MINB>;
    if (cudaError_t e = ensure_smem_attr<fast_row_holo_s<N, kRowTH, MINB>>(smem); e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(MINB * sm_count(P->dev), P->H / S::LINES));
    return launch_pdl(k, grid, kRowTH, smem, P->st, f);
}

static int row_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("CGHB200_ROW_VARIANT");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <int N>
static cudaError_t row_launch(cgh_plan* P, const FastArgs& f) {
    if (row_variant() == 3) return row_launch_s<N, 3>(P, f);
    if (row_variant() == 4) return row_launch_s<N, 4>(P, f);
    using S = FastShape<N, kRowTH>;
    const size_t smem = size_t(3) * S::LINES * ((S::LW + 15) / 16 * 16) * sizeof(float2);
    auto k = fast_row_holo<N, kRowTH, kRowMinB>;
    if (cudaError_t e = ensure_smem_attr<fast_row_holo<N, kRowTH, kRowMinB>>(smem); e != cudaSuccess) return e;
    const int tiles = P->H / S::LINES;   // row groups per CTA = S::LINES
    const int grid = std::max(1, std::min(kRowMinB * sm_count(P->dev), tiles));
    return launch_pdl(k, grid, kRowTH, smem, P->st, f);
}

template <int N, int TH, int MINB, int MODE>
static cudaError_t col_launch_m(cgh_plan* P, const FastArgs& f) {
    using S = FastShape<N, TH>;
    FastState* F = static_cast<FastState*>(P->fast);
    const size_t smem = size_t(2) * FastSlots<N, TH>::COL * sizeof(float2);
    auto k = fast_col_gs<N, TH, MINB, MODE>;
    if (cudaError_t e = ensure_smem_attr<fast_col_gs<N, TH, MINB, MODE>>(smem); e != cudaSuccess) return e;
    const int tiles = P->W / S::LINES;
    const int grid = std::max(1, std::min(MINB * sm_count(P->dev), tiles));
    return launch_pdl(k, grid, TH, smem, P->st, f, F->tmap);
}

template <int N, int TH, int MINB>
static cudaError_t col_launch_th(cgh_plan* P, const FastArgs& f, int mode) {
    switch (mode) {
        case 0: return col_launch_m<N, TH, MINB, 0>(P, f);
        case 1: return col_launch_m<N, TH, MINB, 1>(P, f);
        case 2: return col_launch_m<N, TH, MINB, 2>(P, f);
        default: return col_launch_m<N, TH, MINB, 3>(P, f);
    }
}

template <int N>
static cudaError_t col_launch(cgh_plan* P, const FastArgs& f) {
    const int mode = (P->rescale ? 1 : 0) | (f.gain != 0.0f ? 2 : 0);
    if (col_th() == 256) return col_launch_th<N, 256, 2>(P, f, mode);
    return col_launch_th<N, 512, 1>(P, f, mode);
}

static int encode_2d(CUtensorMap* m, void* ptr, int W, int rows, int C, int box_rows) {
    cuuint64_t dims[2] = {cuuint64_t(2) * W, cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(W) * 8};
    cuuint32_t box[2] = {cuuint32_t(2 * C), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CGH_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
    return CGH_OK;
}

bool fast_ospr_eligible(cgh_plan* P) {
    if (P->prec != CGH_FP32 || P->idx_bytes != 1 || !is_pow2(P->H) || !is_pow2(P->W)) return false;
    const int lc = fast_lines_th(P->H, 512);
    if (lc < 1 || P->W < lc || P->H < 512 || P->W < 512 || P->W > 4096) return false;
    if (getenv("CGHB200_NO_FAST")) return false;
    return encode_fn() != nullptr;
}

// OSPR K2 CTA shape for H <= 1024: 256 threads x 2 CTAs/SM (default; the two
// CTAs' exchange barriers do not align: C2 K2 232 -> 197 us, 512^2 88 -> 58 us)
// or, with CGHB200_HOLO_TH=512, 512 threads x 1 CTA/SM (the shape H >= 2048
// always uses: 256 threads there would mean 2-column tiles, 16-B TMA rows).
static int holo_th() {
    static int th = [] {
        const char* e = getenv("CGHB200_HOLO_TH");
        return (e && atoi(e) == 512) ? 512 : 256;
    }();
    return th;
}

template <int N, int TH, int MINB>
static cudaError_t holo_launch_th(cgh_plan* P, const FastHoloArgs& h, const CUtensorMap& map) {
    using S = FastShape<N, TH>;
    const size_t smem = size_t(2) * ((S::LINES * S::LW + 15) / 16 * 16) * sizeof(float2);
    const int tiles = h.frames * (P->W / S::LINES);
    const int grid = std::max(1, std::min(MINB * sm_count(P->dev), tiles));
    if (h.binary && !h.beam && !h.q_row) {
        auto k = fast_col_holo<N, TH, MINB, true>;
        if (cudaError_t e = ensure_smem_attr<fast_col_holo<N, TH, MINB, true>>(smem); e != cudaSuccess) return e;
        return launch_pdl(k, grid, TH, smem, P->st, h, map);
    }
    auto k = fast_col_holo<N, TH, MINB>;
    if (cudaError_t e = ensure_smem_attr<fast_col_holo<N, TH, MINB>>(smem); e != cudaSuccess) return e;
    return launch_pdl(k, grid, TH, smem, P->st, h, map);
}

template <int N>
static cudaError_t holo_launch(cgh_plan* P, const FastHoloArgs& h, const CUtensorMap& map) {
    if constexpr (N <= 1024) {
        if (holo_th() == 256) return holo_launch_th<N, 256, 2>(P, h, map);
    }
    return holo_launch_th<N, 512, 1>(P, h, map);
}

// OSPR K2 over `frames` stacked frames in the data buffer (capacity `cap` frames).
int fast_ospr_holo(cgh_plan* P, const PassArgs<float>& a, int frames, int cap, uint8_t* idx_out) {
    FastState* F = static_cast<FastState*>(P->fast);
    if (!F) {
        F = new FastState();
        P->fast = F;
    }
    if (!F->ctr.p) {
        CGH_TRY(ensure(P, F->ctr, 64));
        CGH_CUDA(cudaMemsetAsync(F->ctr.p, 0, 64, P->st));
    }
    const int C = fast_lines_th(P->H, P->H <= 1024 ? holo_th() : 512);
    if (F->tmapf_ptr != P->data.p || F->tmapf_rows != cap * P->H || F->tmapf_c != C) {
        CGH_TRY(encode_2d(&F->tmap_frames, P->data.p, P->W, cap * P->H, C, std::min(kFastBoxRows, P->H)));
        F->tmapf_ptr = P->data.p;
        F->tmapf_rows = cap * P->H;
        F->tmapf_c = C;
    }
    FastHoloArgs h;
    h.data = reinterpret_cast<float2*>(a.data);
    h.H = P->H;
    h.W = P->W;
    h.frames = frames;
    h.beam = a.beam;
    h.tw_col = a.tw_col;
    h.q_row = a.q_row;
    h.q_col = a.q_col;
    h.scheme = a.scheme;
    h.idx = idx_out;
    h.binary = (P->scheme_kind == CGH_SCHEME_PHASE && P->nstates == 2 && P->offset == 0.0) ? 1 : 0;
    h.tile_ctr = static_cast<unsigned*>(F->ctr.p);
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_HOLO, true));
    cudaError_t e;
    switch (P->H) {
        case 512: e = holo_launch<512>(P, h, F->tmap_frames); break;
        case 1024: e = holo_launch<1024>(P, h, F->tmap_frames); break;
        case 2048: e = holo_launch<2048>(P, h, F->tmap_frames); break;
        case 4096: e = holo_launch<4096>(P, h, F->tmap_frames); break;
        default: return fail(CGH_ERR_UNSUPPORTED, "fast OSPR column pass H=%d", P->H);
    }
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_HOLO, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "fast OSPR column pass: %s", cudaGetErrorString(e));
    return CGH_OK;
}

// ---- OSPR K1 / K3 ----------------------------------------------------------
constexpr int kOsprTH = 256, kOsprMinB = 2;

template <int N>
static cudaError_t gen_launch(cgh_plan* P, const FastOsprArgs& o) {
    using S = FastShape<N, kOsprTH>;
    const size_t smem = size_t(S::LINES) * ((S::LW + 15) / 16 * 16) * sizeof(float2);
    auto k = fast_ospr_gen<N, kOsprTH, kOsprMinB>;
    if (cudaError_t e = ensure_smem_attr<fast_ospr_gen<N, kOsprTH, kOsprMinB>>(smem); e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(kOsprMinB * sm_count(P->dev), (o.frames * o.H + S::LINES - 1) / S::LINES));
    return launch_pdl(k, grid, kOsprTH, smem, P->st, o);
}

template <int N>
static cudaError_t acc_launch(cgh_plan* P, const FastOsprArgs& o) {
    using S = FastShape<N, kOsprTH>;
    const size_t smem = (size_t(TwTables<N, kOsprTH>::WORDS) + size_t(S::LINES) * 2 * ((S::LW + 15) / 16 * 16)) * sizeof(float2);
    auto k = fast_ospr_acc<N, kOsprTH, kOsprMinB>;
    if (cudaError_t e = ensure_smem_attr<fast_ospr_acc<N, kOsprTH, kOsprMinB>>(smem); e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(kOsprMinB * sm_count(P->dev), (o.H + S::LINES - 1) / S::LINES));
    return launch_pdl(k, grid, kOsprTH, smem, P->st, o);
}

static int fast_ospr_common(cgh_plan* P, const PassArgs<float>& a, FastOsprArgs& o) {
    FastState* F = static_cast<FastState*>(P->fast);
    if (!F) {
        F = new FastState();
        P->fast = F;
    }
    if (!F->ctr.p) {
        CGH_TRY(ensure(P, F->ctr, 64));
        CGH_CUDA(cudaMemsetAsync(F->ctr.p, 0, 64, P->st));
    }
    o.data = reinterpret_cast<float2*>(a.data);
    o.H = P->H;
    o.W = P->W;
    o.frames = a.frames;
    o.frame0 = a.frame0;
    o.nframes_total = a.nframes_total;
    o.tgt = a.tgt;
    o.tw_row = a.tw_row;
    o.scale = a.scale;
    o.intensity = a.intensity;
    o.load_intensity = a.load_intensity;
    o.store_intensity = a.store_intensity;
    o.tile_ctr = static_cast<unsigned*>(F->ctr.p);
    return CGH_OK;
}

// K1: line start states + random-phase rows + inverse row FFT
int fast_ospr_gen(cgh_plan* P, const PassArgs<float>& a) {
    FastOsprArgs o;
    CGH_TRY(fast_ospr_common(P, a, o));
    FastState* F = static_cast<FastState*>(P->fast);
    const int lines = a.frames * P->H;
    CGH_TRY(ensure(P, F->line_state, sizeof(Pcg64) * size_t(std::max(lines, 1))));
    ospr_line_states<<<(lines + 255) / 256, 256, 0, P->st>>>(a.frame_rng, a.frame0, a.frames, P->H, P->W,
                                                            static_cast<Pcg64*>(F->line_state.p));
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    o.line_state = static_cast<const Pcg64*>(F->line_state.p);
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_OSPR_GEN, true));
    cudaError_t e;
    switch (P->W) {
        case 512: e = gen_launch<512>(P, o); break;
        case 1024: e = gen_launch<1024>(P, o); break;
        case 2048: e = gen_launch<2048>(P, o); break;
        case 4096: e = gen_launch<4096>(P, o); break;
        default: return fail(CGH_ERR_UNSUPPORTED, "fast OSPR row pass W=%d", P->W);
    }
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_OSPR_GEN, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "fast OSPR generation: %s", cudaGetErrorString(e));
    return CGH_OK;
}

// K3: forward rows, intensity accumulation, per-line partials, fixed-order totals
int fast_ospr_acc(cgh_plan* P, const PassArgs<float>& a) {
    FastOsprArgs o;
    CGH_TRY(fast_ospr_common(P, a, o));
    FastState* F = static_cast<FastState*>(P->fast);
    const bool tail = (a.frame0 + a.frames == a.nframes_total);
    const size_t nq = size_t(3 * a.frames + 2);
    CGH_TRY(ensure(P, F->line_part, sizeof(double) * nq * P->H));
    o.line_part = static_cast<double*>(F->line_part.p);
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_OSPR_ACC, true));
    cudaError_t e;
    switch (P->W) {
        case 512: e = acc_launch<512>(P, o); break;
        case 1024: e = acc_launch<1024>(P, o); break;
        case 2048: e = acc_launch<2048>(P, o); break;
        case 4096: e = acc_launch<4096>(P, o); break;
        default: return fail(CGH_ERR_UNSUPPORTED, "fast OSPR accumulation W=%d", P->W);
    }
    if (e == cudaSuccess) {
        ospr_line_reduce<<<a.frames + (tail ? 1 : 0), 256, 0, P->st>>>(
            static_cast<const double*>(F->line_part.p), P->H, a.frames, a.frame0, tail ? 1 : 0, a.nframes_total,
            a.red.denom, a.red.rescale, a.red.out);
        e = cudaGetLastError();
    }
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_OSPR_ACC, false));
    P->launches += 2;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "fast OSPR accumulation: %s", cudaGetErrorString(e));
    return CGH_OK;
}

int fast_row(cgh_plan* P, const PassArgs<float>& a) {
    const FastArgs f = fast_args(P, a);
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_HOLO, true));
    cudaError_t e;
    switch (P->W) {
        case 512: e = row_launch<512>(P, f); break;
        case 1024: e = row_launch<1024>(P, f); break;
        case 2048: e = row_launch<2048>(P, f); break;
        case 4096: e = row_launch<4096>(P, f); break;
        default: return fail(CGH_ERR_UNSUPPORTED, "fast row pass W=%d", P->W);
    }
    if (P->profiling) CGH_TRY(prof_mark(P, ROW_HOLO, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "fast row pass: %s", cudaGetErrorString(e));
    return CGH_OK;
}

int fast_col(cgh_plan* P, const PassArgs<float>& a) {
    const FastArgs f = fast_args(P, a);
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_GS, true));
    cudaError_t e;
    switch (P->H) {
        case 256: e = col_launch<256>(P, f); break;
        case 512: e = col_launch<512>(P, f); break;
        case 1024: e = col_launch<1024>(P, f); break;
        case 2048: e = col_launch<2048>(P, f); break;
        case 4096: e = col_launch<4096>(P, f); break;
        default: return fail(CGH_ERR_UNSUPPORTED, "fast column pass H=%d", P->H);
    }
    if (P->profiling) CGH_TRY(prof_mark(P, 8 + COL_GS, false));
    P->launches += 1;
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "fast column pass: %s", cudaGetErrorString(e));
    return CGH_OK;
}

}  // namespace cgh
