// Host runtime + C-ABI for transforms, GS and OSPR (include/cghb200.h).
#include <algorithm>
#include <cmath>
#include <atomic>
#include <mutex>
#include <thread>

#include "runtime.cuh"
#include "host_pool.h"
#include <cstring>

namespace cgh {

// ================================================================= errors
static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

std::shared_mutex& device_gate(int dev) {
    static std::shared_mutex m[64];
    return m[dev & 63];
}

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// ================================================================= tables
// exp(-2 pi i k / n), k in [0, n), evaluated in long double.
void twiddle_table(int n, std::vector<double>& out) {
    out.resize(2 * size_t(n));
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < n; ++k) {
        long double a = -2.0L * pi * (long double)k / (long double)n;
        out[2 * k] = (double)cosl(a);
        out[2 * k + 1] = (double)sinl(a);
    }
}

// Separable Fresnel factor exp(i pi c^2 p^2 / (lambda z)), c = idx - n/2.
// Product of the row and column factors equals fresnel_prefactor
// (propagation.py:97-107) up to rounding of the reference's own fp64 argument.
void chirp_table(int n, double pitch, double wl, double dist, std::vector<double>& out) {
    out.resize(2 * size_t(n));
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < n; ++k) {
        long double c = (long double)k - (long double)n / 2.0L;
        long double a = pi * c * c * (long double)pitch * (long double)pitch / ((long double)wl * (long double)dist);
        out[2 * k] = (double)cosl(a);
        out[2 * k + 1] = (double)sinl(a);
    }
}

static int upload_table(cgh_plan* P, DevBuf& b, const std::vector<double>& v) {
    const size_t n = v.size() / 2;
    if (P->prec == CGH_FP64) {
        CGH_TRY(ensure(P, b, n * 16));
        CGH_CUDA(cudaMemcpyAsync(b.p, v.data(), n * 16, cudaMemcpyHostToDevice, P->st));
    } else {
        std::vector<float> f(v.begin(), v.end());
        CGH_TRY(ensure(P, b, n * 8));
        CGH_CUDA(cudaMemcpyAsync(b.p, f.data(), n * 8, cudaMemcpyHostToDevice, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));   // f is a temporary
    }
    return CGH_OK;
}

// ================================================================== plans
int ensure(cgh_plan* P, DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return CGH_OK;
    if (b.p) CGH_CUDA(cudaFreeAsync(b.p, P->st));
    b.p = nullptr;
    b.cap = 0;
    CGH_CUDA(cudaMallocAsync(&b.p, bytes, P->st));
    b.cap = bytes;
    return CGH_OK;
}

int ensure_res(cgh_plan* P, size_t n) {
    if (P->res_cap >= n) return CGH_OK;
    if (P->res_h) {
        CGH_CUDA(cudaStreamSynchronize(P->st));
        cudaFreeHost(P->res_h);
    }
    P->res_h = nullptr;
    P->res_cap = 0;
    n = std::max<size_t>(n, 1024);
    CGH_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&P->res_h), n * sizeof(double), cudaHostAllocMapped));
    CGH_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->res_d), P->res_h, 0));
    P->res_cap = n;
    return CGH_OK;
}

int ensure_events(cgh_plan* P, size_t n) {
    while (P->evpool.size() < n) {
        cudaEvent_t e;
        CGH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P->evpool.push_back(e);
    }
    return CGH_OK;
}

static std::once_flag g_pool_once[64];

int plan_init(cgh_plan* P, const cgh_problem* pb) {
    if (!pb) return fail(CGH_ERR_VALUE, "null problem");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    if (pb->device < 0 || pb->device >= ndev) return fail(CGH_ERR_VALUE, "device %d out of range (%d devices)", pb->device, ndev);
    if (pb->height < 1 || pb->width < 1) return fail(CGH_ERR_DIMENSION, "empty shape %dx%d", pb->height, pb->width);
    // power-of-two sides run the radix-16 passes; other sides Bluestein line DFTs (anysize.cu)
    if (pb->height < 2 || pb->width < 2 || pb->height > kMaxAnyLine || pb->width > kMaxAnyLine)
        return fail(CGH_ERR_UNSUPPORTED, "shape %dx%d: the CUDA path implements sides 2..%d",
                    pb->height, pb->width, kMaxAnyLine);
    if (pb->precision != CGH_FP32 && pb->precision != CGH_FP64) return fail(CGH_ERR_VALUE, "bad precision");
    if (pb->n_states < 2 || !pb->states) return fail(CGH_ERR_VALUE, "scheme needs >= 2 states");
    if (pb->prop_kind == CGH_FRESNEL) {
        if (!(pb->wavelength > 0) || !(pb->pitch_x > 0) || !(pb->pitch_y > 0))
            return fail(CGH_ERR_INVALID_SPEC, "fresnel needs positive wavelength and pitches");
        if (pb->distance == 0) return fail(CGH_ERR_INVALID_SPEC, "fresnel distance must be nonzero");
    } else if (pb->prop_kind != CGH_FOURIER) {
        return fail(CGH_ERR_INVALID_SPEC, "unknown propagation kind %d", pb->prop_kind);
    }
    CGH_CUDA(cudaSetDevice(pb->device));
    std::call_once(g_pool_once[pb->device & 63], [&] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, pb->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    P->dev = pb->device;
    P->H = pb->height;
    P->W = pb->width;
    P->prec = pb->precision;
    P->scheme_kind = pb->scheme_kind;
    P->nstates = pb->n_states;
    P->offset = pb->phase_offset;
    P->step = pb->scheme_kind == CGH_SCHEME_PHASE ? 2.0 * 3.141592653589793 / double(pb->n_states) : 0.0;
    P->prop_kind = pb->prop_kind;
    P->wl = pb->wavelength;
    P->dist = pb->distance;
    P->px = pb->pitch_x;
    P->py = pb->pitch_y;
    P->rescale = pb->rescale;
    P->idx_bytes = pb->n_states <= 256 ? 1 : 4;
    CGH_CUDA(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
    CGH_CUDA(cudaEventCreate(&P->ev0));
    CGH_CUDA(cudaEventCreate(&P->ev1));
    // states
    const size_t ns = size_t(pb->n_states);
    CGH_TRY(ensure(P, P->states64, ns * 16));
    CGH_CUDA(cudaMemcpyAsync(P->states64.p, pb->states, ns * 16, cudaMemcpyHostToDevice, P->st));
    std::vector<float> s32(2 * ns);
    for (size_t i = 0; i < 2 * ns; ++i) s32[i] = float(pb->states[i]);
    CGH_TRY(ensure(P, P->states32, ns * 8));
    CGH_CUDA(cudaMemcpyAsync(P->states32.p, s32.data(), ns * 8, cudaMemcpyHostToDevice, P->st));
    // tables
    std::vector<double> t;
    if (is_pow2(P->W)) {
        twiddle_table(P->W, t);
        CGH_TRY(upload_table(P, P->tw_row, t));
    } else {
        blue_pack_table(P->W, t);
        CGH_TRY(upload_table(P, P->tw_row, t));
        CGH_TRY(blue_finish_table(P->prec, P->W, P->tw_row.p, P->st));
    }
    if (is_pow2(P->H)) {
        twiddle_table(P->H, t);
        CGH_TRY(upload_table(P, P->tw_col, t));
    } else {
        blue_pack_table(P->H, t);
        CGH_TRY(upload_table(P, P->tw_col, t));
        CGH_TRY(blue_finish_table(P->prec, P->H, P->tw_col.p, P->st));
    }
    if (P->prop_kind == CGH_FRESNEL) {
        chirp_table(P->H, P->py, P->wl, P->dist, t);
        CGH_TRY(upload_table(P, P->q_row, t));
        chirp_table(P->W, P->px, P->wl, P->dist, t);
        CGH_TRY(upload_table(P, P->q_col, t));
    }
    CGH_TRY(ensure(P, P->counter, 64));
    CGH_CUDA(cudaMemsetAsync(P->counter.p, 0, 64, P->st));
    CGH_TRY(ensure(P, P->stats, 8 * sizeof(double)));
    CGH_CUDA(cudaStreamSynchronize(P->st));   // s32 is a temporary
    return CGH_OK;
}

void plan_free(cgh_plan* P) {
    if (!P) return;
    cudaSetDevice(P->dev);
    if (P->st) cudaStreamSynchronize(P->st);
    fast_free(P);
    wl_free(P);
    cgh::DevBuf* bufs[] = {&P->states64, &P->states32, &P->tw_row, &P->tw_col, &P->q_row, &P->q_col, &P->data,
                           &P->tgt, &P->beam, &P->idx, &P->field, &P->partials, &P->counter, &P->stats, &P->stage,
                           &P->mask, &P->frame_rng, &P->intensity, &P->sa_buf};
    for (auto* b : bufs)
        if (b->p) cudaFreeAsync(b->p, P->st);
    if (P->st) cudaStreamSynchronize(P->st);
    if (P->res_h) cudaFreeHost(P->res_h);
    for (void* h : P->pin) cudaFreeHost(h);
    if (P->pin_amp) cudaFreeHost(P->pin_amp);
    for (auto s : P->amp_st) cudaStreamDestroy(s);
    for (auto e : P->amp_ev) cudaEventDestroy(e);
    for (auto st : P->pin_st) cudaStreamDestroy(st);
    for (auto e : P->pin_ev) cudaEventDestroy(e);
    for (auto e : P->evpool) cudaEventDestroy(e);
    if (P->ev0) cudaEventDestroy(P->ev0);
    if (P->ev1) cudaEventDestroy(P->ev1);
    if (P->st) cudaStreamDestroy(P->st);
}

template <class T>
PassArgs<T> base_args(cgh_plan* P) {
    PassArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.data = static_cast<cx<T>*>(P->data.p);
    a.frame_stride = long(P->H) * P->W;
    a.H = P->H;
    a.W = P->W;
    a.tgt = static_cast<const T*>(P->tgt.p);
    a.beam = P->has_beam ? static_cast<const T*>(P->beam.p) : nullptr;
    a.tw_row = static_cast<const cx<T>*>(P->tw_row.p);
    a.tw_col = static_cast<const cx<T>*>(P->tw_col.p);
    a.q_row = P->prop_kind == CGH_FRESNEL ? static_cast<const cx<T>*>(P->q_row.p) : nullptr;
    a.q_col = P->prop_kind == CGH_FRESNEL ? static_cast<const cx<T>*>(P->q_col.p) : nullptr;
    a.scheme.kind = P->scheme_kind;
    a.scheme.n = P->nstates;
    a.scheme.offset = P->offset;
    a.scheme.step = P->step;
    a.scheme.states64 = static_cast<const double*>(P->states64.p);
    a.scheme.states32 = static_cast<const float*>(P->states32.p);
    a.gain = T(0);
    a.scale = T(1.0 / std::sqrt(double(P->H) * double(P->W)));
    a.idx_bytes = P->idx_bytes;
    a.red.partials = static_cast<double*>(P->partials.p);
    a.red.counter = static_cast<unsigned*>(P->counter.p);
    a.red.denom = static_cast<const double*>(P->stats.p) + 1;
    a.red.rescale = P->rescale;
    return a;
}
template PassArgs<float> base_args<float>(cgh_plan*);
template PassArgs<double> base_args<double>(cgh_plan*);

// Upload the target (complex128, centred), mask and illumination; build the
// shifted amplitude/mask plane and the beam amplitude; read back statistics.
template <class T>
static int prep_target(cgh_plan* P, const double* target, const uint8_t* mask, const double* illum) {
    const long n = long(P->H) * P->W;
    CGH_TRY(ensure(P, P->stage, size_t(n) * 16 * (illum ? 2 : 1)));
    CGH_TRY(ensure(P, P->mask, size_t(n)));
    CGH_TRY(ensure(P, P->tgt, size_t(n) * sizeof(T)));
    CGH_TRY(upload_staged(P, P->stage.p, target, size_t(n) * 16));
    CGH_CUDA(cudaMemcpyAsync(P->mask.p, mask, size_t(n), cudaMemcpyHostToDevice, P->st));
    double* ic = nullptr;
    if (illum) {
        ic = static_cast<double*>(P->stage.p) + 2 * n;
        CGH_TRY(ensure(P, P->beam, size_t(n) * sizeof(T)));
        CGH_TRY(upload_staged(P, ic, illum, size_t(n) * 16));
    }
    P->has_beam = illum != nullptr;
    P->stage_valid = true;
    const int grid = grid_for(n);
    CGH_TRY(ensure(P, P->partials, size_t(grid) * 5 * sizeof(double)));
    PrepStats ps;
    ps.partials = static_cast<double*>(P->partials.p);
    ps.counter = static_cast<unsigned*>(P->counter.p);
    ps.out = static_cast<double*>(P->stats.p);
    prep_kernel<T><<<grid, 256, 0, P->st>>>(static_cast<const double*>(P->stage.p), static_cast<const uint8_t*>(P->mask.p),
                                            ic, P->H, P->W, static_cast<T*>(P->tgt.p),
                                            illum ? static_cast<T*>(P->beam.p) : nullptr, nullptr, ps);
    P->launches += 1;
    CGH_CUDA(cudaGetLastError());
    double st[5];
    CGH_CUDA(cudaMemcpyAsync(st, P->stats.p, sizeof(st), cudaMemcpyDeviceToHost, P->st));
    CGH_CUDA(cudaStreamSynchronize(P->st));
    P->count_in = st[0];
    P->denom = st[1];
    P->nf_in = st[2];
    P->nf_all = st[3];
    P->nf_beam = st[4];
    P->target_ready = true;
    fast_invalidate_target(P);
    wl_invalidate_target(P);
    return CGH_OK;
}

constexpr int kStageThreads = 4;
constexpr size_t kStageChunk = size_t(4) << 20;   // bytes per pinned chunk (2 per thread)

int upload_staged(cgh_plan* P, void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(16) << 20)) {
        CGH_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, P->st));
        return CGH_OK;
    }
    if (P->pin.empty()) {
        for (int i = 0; i < 2 * kStageThreads; ++i) {
            void* h = nullptr;
            CGH_CUDA(cudaHostAlloc(&h, kStageChunk, cudaHostAllocDefault));
            P->pin.push_back(h);
            cudaEvent_t e;
            CGH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            P->pin_ev.push_back(e);
        }
        for (int t = 0; t < kStageThreads; ++t) {
            cudaStream_t st;
            CGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            P->pin_st.push_back(st);
        }
        cudaEvent_t e;   // start event (last slot)
        CGH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        P->pin_ev.push_back(e);
    }
    // pinned chunks still being read by an earlier upload's DMAs
    for (int i = 0; i < 2 * kStageThreads; ++i) CGH_CUDA(cudaEventSynchronize(P->pin_ev[i]));
    // the staging streams start after earlier work on P->st (dst may be in use)
    cudaEvent_t start = P->pin_ev[2 * kStageThreads];
    CGH_CUDA(cudaEventRecord(start, P->st));
    for (int t = 0; t < kStageThreads; ++t) CGH_CUDA(cudaStreamWaitEvent(P->pin_st[t], start, 0));
    const size_t slice = (bytes + kStageThreads - 1) / kStageThreads;
    std::atomic<int> err{0};
    auto worker = [&](int t) {
        cudaSetDevice(P->dev);
        const size_t lo = std::min(bytes, size_t(t) * slice), hi = std::min(bytes, lo + slice);
        int k = 0;
        for (size_t off = lo; off < hi; off += kStageChunk, ++k) {
            const int b = 2 * t + (k & 1);
            const size_t len = std::min(kStageChunk, hi - off);
            if (k >= 2 && cudaEventSynchronize(P->pin_ev[b]) != cudaSuccess) err = 1;   // chunk's previous DMA done
            memcpy(P->pin[b], static_cast<const char*>(src) + off, len);
            if (cudaMemcpyAsync(static_cast<char*>(dst) + off, P->pin[b], len, cudaMemcpyHostToDevice,
                                P->pin_st[t]) != cudaSuccess)
                err = 1;
            if (cudaEventRecord(P->pin_ev[b], P->pin_st[t]) != cudaSuccess) err = 1;
        }
    };
    HostPool::get().run(kStageThreads, worker);
    if (err) return fail(CGH_ERR_CUDA, "staged upload failed");
    for (int t = 0; t < kStageThreads; ++t) {
        CGH_CUDA(cudaEventRecord(P->pin_ev[2 * t], P->pin_st[t]));
        CGH_CUDA(cudaStreamWaitEvent(P->st, P->pin_ev[2 * t], 0));
    }
    // pinned chunks are reused by the next upload only after these DMAs: the
    // next call records `start` on P->st, which now waits for them
    return CGH_OK;
}

#if defined(__SSE2__)
// One contiguous run of L pixels of the amplitude preparation below, two
// complex128 values per SSE2 register pair, four pixels per step: out[i] =
// +-float(|t_i|) (sign bit set outside the mask), streamed; per-run count and
// sum of |t|^2 inside the mask (fixed order: two lanes, then lane 0 + lane 1).
// |t| = sqrt(re^2 + im^2) exactly as the scalar path; returns false if a
// pixel needs the scalar path's care (|t| >= 1e150, a nonzero |t| < 1e-150
// or squares that underflow to 0, NaN / Inf) or the run is not 4-aligned.
static bool amp_run_sse2(const double* t, const uint8_t* m, float* o, int L, double& cnt, double& den) {
    if ((L & 3) || (reinterpret_cast<uintptr_t>(o) & 15u)) return false;
    const __m128d big = _mm_set1_pd(1e150), small = _mm_set1_pd(1e-150), zd = _mm_setzero_pd();
    const __m128i zi = _mm_setzero_si128(), sign = _mm_set1_epi32(int(0x80000000u));
    __m128d dsum = zd;
    long in_count = 0;
    int bad = 0;
    for (int i = 0; i < L; i += 4) {
        const __m128d x0 = _mm_loadu_pd(t + 2 * i), x1 = _mm_loadu_pd(t + 2 * i + 2);
        const __m128d x2 = _mm_loadu_pd(t + 2 * i + 4), x3 = _mm_loadu_pd(t + 2 * i + 6);
        const __m128d s0 = _mm_mul_pd(x0, x0), s1 = _mm_mul_pd(x1, x1);
        const __m128d s2 = _mm_mul_pd(x2, x2), s3 = _mm_mul_pd(x3, x3);
        const __m128d a01 = _mm_sqrt_pd(_mm_add_pd(_mm_unpacklo_pd(s0, s1), _mm_unpackhi_pd(s0, s1)));
        const __m128d a23 = _mm_sqrt_pd(_mm_add_pd(_mm_unpacklo_pd(s2, s3), _mm_unpackhi_pd(s2, s3)));
        const __m128d q0 = _mm_cmpneq_pd(x0, zd), q1 = _mm_cmpneq_pd(x1, zd);
        const __m128d q2 = _mm_cmpneq_pd(x2, zd), q3 = _mm_cmpneq_pd(x3, zd);
        const __m128d nz01 = _mm_or_pd(_mm_unpacklo_pd(q0, q1), _mm_unpackhi_pd(q0, q1));
        const __m128d nz23 = _mm_or_pd(_mm_unpacklo_pd(q2, q3), _mm_unpackhi_pd(q2, q3));
        const __m128d f01 = _mm_or_pd(_mm_cmpnlt_pd(a01, big), _mm_and_pd(_mm_cmplt_pd(a01, small), nz01));
        const __m128d f23 = _mm_or_pd(_mm_cmpnlt_pd(a23, big), _mm_and_pd(_mm_cmplt_pd(a23, small), nz23));
        bad |= _mm_movemask_pd(_mm_or_pd(f01, f23));
        uint32_t mb;
        memcpy(&mb, m + i, 4);
        // 32-bit lane k all ones where mask byte k is 0 (outside the mask)
        const __m128i out32 = _mm_cmpeq_epi32(
            _mm_unpacklo_epi16(_mm_unpacklo_epi8(_mm_cvtsi32_si128(int(mb)), zi), zi), zi);
        const __m128 af = _mm_movelh_ps(_mm_cvtpd_ps(a01), _mm_cvtpd_ps(a23));
        _mm_stream_ps(o + i, _mm_xor_ps(af, _mm_castsi128_ps(_mm_and_si128(out32, sign))));
        const __m128d in01 = _mm_castsi128_pd(_mm_andnot_si128(_mm_unpacklo_epi32(out32, out32), _mm_set1_epi32(-1)));
        const __m128d in23 = _mm_castsi128_pd(_mm_andnot_si128(_mm_unpackhi_epi32(out32, out32), _mm_set1_epi32(-1)));
        dsum = _mm_add_pd(dsum, _mm_and_pd(_mm_mul_pd(a01, a01), in01));
        dsum = _mm_add_pd(dsum, _mm_and_pd(_mm_mul_pd(a23, a23), in23));
        in_count += 4 - __builtin_popcount(unsigned(_mm_movemask_ps(_mm_castsi128_ps(out32))));
    }
    if (bad) return false;
    double lanes[2];
    _mm_storeu_pd(lanes, dsum);
    cnt += double(in_count);
    den += lanes[0] + lanes[1];
    return true;
}
#endif

// fp32 plans whose runs never start from the backpropagated target: the
// shifted, mask-signed amplitude plane (prep_kernel's output) and the beam
// amplitude are built by host threads straight into pinned memory and copied
// in row chunks as they are produced: 4 B/px cross PCIe instead of the 16 B/px
// complex128 target plus the mask. Statistics in fp64, fixed order per thread
// and across threads.
static int prep_target_host_f32(cgh_plan* P, const double* target, const uint8_t* mask, const double* illum) {
    const int H = P->H, W = P->W;
    const long n = long(H) * W;
    const size_t plane = size_t(n) * sizeof(float);
    const size_t need = plane * (illum ? 2 : 1);
    const char* ntenv = getenv("CGHB200_PREP_THREADS");
    const int nt = ntenv ? std::max(1, std::min(64, atoi(ntenv)))
                         : std::max(1, std::min(16, int(std::thread::hardware_concurrency())));
    if (int(P->amp_st.size()) < nt) {
        while (int(P->amp_st.size()) < nt) {
            cudaStream_t st;
            CGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            P->amp_st.push_back(st);
            cudaEvent_t e;
            CGH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            P->amp_ev.push_back(e);
        }
    }
    for (auto st : P->amp_st) CGH_CUDA(cudaStreamSynchronize(st));   // earlier copies out of pin_amp done
    if (P->pin_amp_cap < need) {
        if (P->pin_amp) CGH_CUDA(cudaFreeHost(P->pin_amp));
        P->pin_amp = nullptr;
        P->pin_amp_cap = 0;
        CGH_CUDA(cudaHostAlloc(&P->pin_amp, need, cudaHostAllocDefault));
        P->pin_amp_cap = need;
    }
    CGH_TRY(ensure(P, P->tgt, plane));
    if (illum) CGH_TRY(ensure(P, P->beam, plane));
    P->has_beam = illum != nullptr;
    // the device buffers may still be read by earlier work on P->st
    cudaEvent_t start = P->amp_ev[0];
    CGH_CUDA(cudaEventRecord(start, P->st));
    for (int t = 0; t < nt; ++t) CGH_CUDA(cudaStreamWaitEvent(P->amp_st[t], start, 0));
    float* amp = static_cast<float*>(P->pin_amp);
    float* bamp = illum ? amp + n : nullptr;
    std::vector<double> st(size_t(nt) * 5, 0.0);
    std::atomic<int> err{0};
    auto mag = [](double re, double im) {
        const double t = std::sqrt(re * re + im * im);
        // overflow / underflow of the squares, non-finite input: as hypot
        if (!(t < 1e150) || t < 1e-150) return std::hypot(re, im);
        return t;
    };
    auto worker = [&](int t) {
        cudaSetDevice(P->dev);
        const int u0 = int(long(H) * t / nt), u1 = int(long(H) * (t + 1) / nt);
        const int rows_per_copy = std::max(1, int((size_t(256) << 10) / (size_t(W) * sizeof(float))));
        double cnt = 0, den = 0, nfm = 0, nfa = 0, nfb = 0;
        int flushed = u0;
        for (int u = u0; u < u1; ++u) {
            const int uc = u + H / 2 >= H ? u + H / 2 - H : u + H / 2;
            const double* trow = target + 2 * long(uc) * W;
            const uint8_t* mrow = mask + long(uc) * W;
            float* orow = amp + long(u) * W;
#if defined(__SSE2__)
            // vectorised row in its two contiguous runs (columns W/2.. then 0..)
            if (!(W & 1)) {
                double c = 0, d = 0;
                const int h = W / 2;
                if (amp_run_sse2(trow + 2 * long(h), mrow + h, orow, h, c, d) &&
                    amp_run_sse2(trow, mrow, orow + h, h, c, d)) {
                    cnt += c;
                    den += d;
                    goto beam_row;
                }
            }
#endif
            for (int v = 0; v < W; ++v) {
                const int vc = v + W / 2 >= W ? v + W / 2 - W : v + W / 2;
                const double re = trow[2 * vc], im = trow[2 * vc + 1];
                const double a = mag(re, im);
                const bool in = mrow[vc] != 0;
                const bool fin = std::isfinite(re) && std::isfinite(im);
                if (in) {
                    cnt += 1.0;
                    den += a * a;
                    if (!fin) nfm += 1.0;
                }
                if (!fin) nfa += 1.0;
                const float af = float(a);
                stream_store_f32(orow + v, in ? af : -af);   // -0.0 for dark pixels outside the mask
            }
        beam_row:
            if (bamp) {   // the beam is not shifted (hologram plane)
                const double* irow = illum + 2 * long(u) * W;
                float* brow = bamp + long(u) * W;
                for (int v = 0; v < W; ++v) {
                    const double br = irow[2 * v], bi = irow[2 * v + 1];
                    if (!(std::isfinite(br) && std::isfinite(bi))) nfb += 1.0;
                    stream_store_f32(brow + v, float(mag(br, bi)));
                }
            }
            if (u + 1 - flushed >= rows_per_copy || u + 1 == u1) {
                stream_fence();   // the streamed rows are in memory before the DMA reads them
                const size_t off = size_t(flushed) * W, len = size_t(u + 1 - flushed) * W * sizeof(float);
                if (cudaMemcpyAsync(static_cast<float*>(P->tgt.p) + off, amp + off, len, cudaMemcpyHostToDevice,
                                    P->amp_st[t]) != cudaSuccess)
                    err = 1;
                if (bamp && cudaMemcpyAsync(static_cast<float*>(P->beam.p) + off, bamp + off, len,
                                            cudaMemcpyHostToDevice, P->amp_st[t]) != cudaSuccess)
                    err = 1;
                flushed = u + 1;
            }
        }
        double* s = &st[size_t(t) * 5];
        s[0] = cnt;
        s[1] = den;
        s[2] = nfm;
        s[3] = nfa;
        s[4] = nfb;
    };
    HostPool::get().run(nt, worker);
    if (err) return fail(CGH_ERR_CUDA, "amplitude upload failed");
    for (int t = 0; t < nt; ++t) {
        CGH_CUDA(cudaEventRecord(P->amp_ev[t], P->amp_st[t]));
        CGH_CUDA(cudaStreamWaitEvent(P->st, P->amp_ev[t], 0));
    }
    double tot[5] = {0, 0, 0, 0, 0};
    for (int t = 0; t < nt; ++t)
        for (int q = 0; q < 5; ++q) tot[q] += st[size_t(t) * 5 + q];
    P->count_in = tot[0];
    P->denom = tot[1];
    P->nf_in = tot[2];
    P->nf_all = tot[3];
    P->nf_beam = tot[4];
    // the denominator is read on the device (ReduceArgs::denom -> stats[1])
    double dev_stats[5] = {tot[0], tot[1], tot[2], tot[3], tot[4]};
    // pageable source: the runtime stages it before returning (no stream sync
    // needed for the temporary), so the last amplitude DMAs overlap the
    // caller's next steps
    CGH_CUDA(cudaMemcpyAsync(P->stats.p, dev_stats, sizeof(dev_stats), cudaMemcpyHostToDevice, P->st));
    P->target_ready = true;
    P->stage_valid = false;
    fast_invalidate_target(P);
    wl_invalidate_target(P);
    return CGH_OK;
}

int plan_upload_target_ex(cgh_plan* P, const double* target, const uint8_t* mask, const double* illum, int flags) {
    if (!target || !mask) return fail(CGH_ERR_VALUE, "target and mask are required");
    CGH_CUDA(cudaSetDevice(P->dev));
    if ((flags & 1) && P->prec == CGH_FP32) return prep_target_host_f32(P, target, mask, illum);
    return P->prec == CGH_FP64 ? prep_target<double>(P, target, mask, illum) : prep_target<float>(P, target, mask, illum);
}

int plan_upload_target(cgh_plan* P, const double* target, const uint8_t* mask, const double* illum) {
    if (!target || !mask) return fail(CGH_ERR_VALUE, "target and mask are required");
    CGH_CUDA(cudaSetDevice(P->dev));
    return P->prec == CGH_FP64 ? prep_target<double>(P, target, mask, illum) : prep_target<float>(P, target, mask, illum);
}

int prof_mark(cgh_plan* P, int id, bool start) {
    cudaEvent_t e;
    CGH_CUDA(cudaEventCreate(&e));
    CGH_CUDA(cudaEventRecord(e, P->st));
    P->prof_ev.push_back(e);
    if (start) P->prof_id.push_back(id);
    return CGH_OK;
}

// ========================================================= progress queue
int ProgressQueue::init(cgh_plan* P_, const cgh_callbacks* cb_, size_t depth_, const double* values_, long stride_) {
    P = P_;
    cb = cb_;
    depth = std::min<size_t>(depth_, 63);
    values = values_;
    stride = stride_;
    ks.assign(64, 0);
    CGH_TRY(ensure_events(P, 64));
    evs.assign(P->evpool.begin(), P->evpool.begin() + 64);
    head = used = 0;
    return CGH_OK;
}

int ProgressQueue::push(long k) {
    const size_t slot = (head + used) % 64;
    ks[slot] = k;
    CGH_CUDA(cudaEventRecord(evs[slot], P->st));
    used += 1;
    if (used >= 64) return poll(true);
    return CGH_OK;
}

int ProgressQueue::poll(bool all) {
    while (used > 0) {
        cudaEvent_t e = evs[head];
        if (!all && used <= depth) {
            cudaError_t q = cudaEventQuery(e);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) CGH_CUDA(q);
        } else {
            CGH_CUDA(cudaEventSynchronize(e));
        }
        const long k = ks[head];
        if (cb && cb->progress) {
            volatile const double* v = values;
            cb->progress(cb->user, k + kbias, v[k * stride]);
        }
        head = (head + 1) % 64;
        used -= 1;
    }
    return CGH_OK;
}


// ============================================================= transforms
template <class T>
static int transform_exec(cgh_plan* P, const double* in, double* out, int op) {
    const long n = long(P->H) * P->W;
    const bool fres = P->prop_kind == CGH_FRESNEL && op >= 2;
    const bool fwd = (op == 0 || op == 2);
    CGH_TRY(ensure(P, P->stage, size_t(n) * 16));
    CGH_TRY(ensure(P, P->data, size_t(n) * sizeof(cx<T>)));
    CGH_TRY(ensure(P, P->counter, 64));
    CGH_CUDA(cudaMemcpyAsync(P->stage.p, in, size_t(n) * 16, cudaMemcpyHostToDevice, P->st));
    PassArgs<T> a = base_args<T>(P);
    const cx<T>* qr = fres ? a.q_row : nullptr;
    const cx<T>* qc = fres ? a.q_col : nullptr;
    unsigned* nf = static_cast<unsigned*>(P->counter.p) + 8;
    CGH_CUDA(cudaMemsetAsync(nf, 0, sizeof(unsigned), P->st));
    const int grid = grid_for(n);
    load_field_kernel<T><<<grid, 256, 0, P->st>>>(static_cast<const double*>(P->stage.p), a.data, P->H, P->W, fwd ? 0 : 1,
                                                  fwd ? qr : nullptr, fwd ? qc : nullptr, nf);
    CGH_CUDA(cudaGetLastError());
    unsigned nonfinite = 0;
    CGH_CUDA(cudaMemcpyAsync(&nonfinite, nf, sizeof(unsigned), cudaMemcpyDeviceToHost, P->st));
    CGH_CUDA(cudaStreamSynchronize(P->st));
    if (nonfinite) return fail(CGH_ERR_NONFINITE, "field contains NaN or Inf");
    a.scale = T(1);
    CGH_TRY(run_row<T>(P, fwd ? ROW_FWD : ROW_INV, a, 1));
    a.scale = T(1.0 / std::sqrt(double(P->H) * double(P->W)));
    CGH_TRY(run_col<T>(P, fwd ? COL_FWD : COL_INV, a, 1));
    store_field_kernel<T><<<grid, 256, 0, P->st>>>(a.data, static_cast<double*>(P->stage.p), P->H, P->W, fwd ? 1 : 0,
                                                   fwd ? nullptr : qr, fwd ? nullptr : qc);
    CGH_CUDA(cudaGetLastError());
    CGH_CUDA(cudaMemcpyAsync(out, P->stage.p, size_t(n) * 16, cudaMemcpyDeviceToHost, P->st));
    CGH_CUDA(cudaStreamSynchronize(P->st));
    return CGH_OK;
}

// ===================================================================== GS
// run_gs (algorithms.py:147-202) on a plan whose target is prepared.
template <class T>
static int gs_exec(cgh_plan* P, const cgh_gs_params* gp, int64_t* tk, double* tv, int64_t cap, cgh_report* rep,
                   const cgh_callbacks* cb, cx<T>* field_dev) {
    if (!P->target_ready) return fail(CGH_ERR_VALUE, "target not set");
    if (gp->init_mode != CGH_INIT_RANDOM_PHASE && gp->init_mode != CGH_INIT_BACKPROPAGATE)
        return fail(CGH_ERR_VALUE, "unknown init mode %d", gp->init_mode);
    // reference error order: init (backprop propagate_inverse) -> propagate(holo)
    // -> mse_error (empty mask, zero target) -> propagate_inverse(constrained)
    if (gp->init_mode == CGH_INIT_BACKPROPAGATE && P->nf_all > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf");
    if (P->nf_beam > 0) return fail(CGH_ERR_NONFINITE, "illumination contains NaN or Inf");
    if (P->count_in == 0) return fail(CGH_ERR_EMPTY_MASK, "metric mask has no true pixels");
    if (P->denom == 0) return fail(CGH_ERR_ZERO_TARGET, "target is zero inside the mask");
    if (P->nf_in > 0 && gp->iterations > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf inside the mask");
    const int iters = std::max(0, gp->iterations);
    const long n = long(P->H) * P->W;
    CGH_TRY(ensure(P, P->data, size_t(n) * sizeof(cx<T>)));
    CGH_TRY(ensure(P, P->idx, size_t(n) * P->idx_bytes));
    const int nb = std::max(row_grid_blocks<T>(P->W, P->H), col_grid_blocks<T>(P->H, P->W));
    CGH_TRY(ensure(P, P->partials, size_t(nb) * 8 * sizeof(double)));
    CGH_TRY(ensure_res(P, size_t(2 * (iters + 2))));
    P->idx_frames = 1;
    PassArgs<T> a = base_args<T>(P);
    a.rng = to_pcg(gp->rng);
    a.gain = T(gp->feedback_gain);
    const long launches0 = P->launches;
    CGH_CUDA(cudaEventRecord(P->ev0, P->st));

    auto run_init = [&](int quantize) -> int {
        PassArgs<T> b = a;
        b.quantize = quantize;
        b.idx_out = quantize ? P->idx.p : nullptr;
        b.field_out = quantize ? field_dev : nullptr;
        if (gp->init_mode == CGH_INIT_RANDOM_PHASE) return run_row<T>(P, ROW_INIT, b, 1);
        // backpropagate: ifftshift(T) -> inverse columns -> ROW_HOLO (rows + projection)
        if (!P->stage_valid)
            return fail(CGH_ERR_VALUE, "backpropagation start needs the complex target (cgh_plan_set_target)");
        load_field_kernel<T><<<grid_for(n), 256, 0, P->st>>>(static_cast<const double*>(P->stage.p), b.data, P->H, P->W, 1,
                                                             nullptr, nullptr, static_cast<unsigned*>(P->counter.p) + 8);
        P->launches += 1;
        CGH_CUDA(cudaGetLastError());
        CGH_TRY(run_col<T>(P, COL_INV, b, 1));
        return run_row<T>(P, ROW_HOLO, b, 1);
    };

    bool fast = false, wlp = false;
    if constexpr (sizeof(T) == 4) {
        fast = fast_eligible(P);
        if (fast) CGH_TRY(fast_prepare(P));
        // warp-line passes (2048^2): the plane stays column-tiled between the
        // relayouts; snapping row passes run on the row-major plane
        wlp = fast && !gp->quantize_each_iteration && wl_eligible(P);
        if (wlp) CGH_TRY(wl_prepare(P));
    }
    bool tiled = false;
    auto to_rowmajor = [&]() -> int {
        if (tiled) {
            CGH_TRY(wl_relayout(P, 0));
            tiled = false;
        }
        return CGH_OK;
    };
    CGH_TRY(run_init(iters == 0 ? 1 : 0));
    ProgressQueue pq;
    const bool has_cancel = cb && cb->cancel, has_progress = cb && cb->progress;
    CGH_TRY(pq.init(P, cb, has_cancel && has_progress ? 0 : (has_cancel ? 4 : 63), P->res_h, 2));
    long executed = 0;
    bool stop = false;
    long k_first = 0;
    if constexpr (sizeof(T) == 4) {
        // no per-iteration host hooks: iterations 0..iters-1 in one persistent
        // launch; only the last (snapping) hologram-plane pass is left below
        if (wlp && !has_cancel && !has_progress && iters >= 2 && !getenv("CGHB200_WL_NO_LOOP")) {
            CGH_TRY(wl_relayout(P, 1));
            tiled = true;
            CGH_TRY(wl_gs_loop(P, a, int(iters)));
            CGH_TRY(to_rowmajor());
            PassArgs<T> r = a;
            r.quantize = 1;
            r.idx_out = P->idx.p;
            r.field_out = field_dev;
            CGH_TRY(run_row<T>(P, ROW_HOLO, r, 1));
            executed = iters;
            k_first = iters;
        }
    }
    for (long k = k_first; k < iters; ++k) {
        if (cancelled(cb)) {
            stop = true;
            break;
        }
        PassArgs<T> c = a;
        c.red.out = P->res_d + 2 * k;
        if constexpr (sizeof(T) == 4) {
            if (wlp) {
                if (!tiled) {
                    CGH_TRY(wl_relayout(P, 1));
                    tiled = true;
                }
                CGH_TRY(wl_col(P, c));
            } else if (fast) {
                CGH_TRY(fast_col(P, c));
            } else {
                CGH_TRY(run_col<T>(P, COL_GS, c, 1));
            }
        } else {
            CGH_TRY(run_col<T>(P, COL_GS, c, 1));
        }
        if (has_progress || has_cancel) CGH_TRY(pq.push(k));
        const bool last = (k == iters - 1);
        PassArgs<T> r = a;
        r.quantize = (gp->quantize_each_iteration || last) ? 1 : 0;
        r.idx_out = last ? P->idx.p : nullptr;
        r.field_out = last ? field_dev : nullptr;
        bool done_fast = false;
        if constexpr (sizeof(T) == 4) {
            if (wlp && tiled && !r.quantize && !r.field_out) {
                CGH_TRY(wl_row(P, r));
                done_fast = true;
            } else if (fast && !r.quantize && !r.field_out) {
                CGH_TRY(to_rowmajor());
                CGH_TRY(fast_row(P, r));
                done_fast = true;
            }
        }
        if (!done_fast) {
            CGH_TRY(to_rowmajor());
            CGH_TRY(run_row<T>(P, ROW_HOLO, r, 1));
        }
        executed = k + 1;
        if (has_progress || has_cancel) CGH_TRY(pq.poll(false));
    }
    CGH_TRY(to_rowmajor());
    if (stop) {
        if (executed == 0) {
            CGH_TRY(run_init(1));
        } else {
            PassArgs<T> r = a;
            r.quantize = 1;
            r.idx_out = P->idx.p;
            r.field_out = field_dev;
            CGH_TRY(run_row<T>(P, ROW_HOLO, r, 1));
        }
    }
    {
        PassArgs<T> c = a;
        c.red.out = P->res_d + 2 * executed;
        CGH_TRY(run_col<T>(P, COL_FINAL, c, 1));
    }
    CGH_CUDA(cudaEventRecord(P->ev1, P->st));
    CGH_TRY(pq.poll(true));
    CGH_CUDA(cudaEventSynchronize(P->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, P->ev0, P->ev1);
    volatile const double* res = P->res_h;
    const double final_err = res[2 * executed];
    const double eff = res[2 * executed + 1];
    if (std::isnan(eff)) return fail(CGH_ERR_ZERO_FIELD, "replay field is zero");
    if (has_progress) cb->progress(cb->user, executed, final_err);
    const int64_t len = executed + 1;
    if (tk && tv) {
        if (cap < len) return fail(CGH_ERR_VALUE, "trace capacity %lld < %lld", (long long)cap, (long long)len);
        for (long k = 0; k < executed; ++k) {
            tk[k] = k;
            tv[k] = res[2 * k];
        }
        tk[executed] = executed;
        tv[executed] = final_err;
    }
    if (rep) {
        rep->final_error = final_err;
        rep->efficiency = eff;
        rep->iterations_executed = executed;
        rep->termination = stop ? CGH_CANCELLED : CGH_COMPLETED;
        rep->trace_len = len;
        rep->kernel_launches = P->launches - launches0;
        rep->device_ms = ms;
    }
    return CGH_OK;
}

// =================================================================== OSPR
// run_ospr (algorithms.py:473-530): batched K1/K2/K3 over frame groups.
template <class T>
static int ospr_exec(cgh_plan* P, const cgh_ospr_params* op, int64_t* tk, double* tv, int64_t cap, cgh_report* rep,
                     const cgh_callbacks* cb) {
    if (!P->target_ready) return fail(CGH_ERR_VALUE, "target not set");
    const int S = std::max(0, op->subframes);
    if (S > 0 && !op->frame_rng) return fail(CGH_ERR_VALUE, "frame streams missing");
    // reference order per frame: propagate_inverse(sub_target) -> ... -> mse_error
    if (P->nf_all > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf");
    if (P->nf_beam > 0) return fail(CGH_ERR_NONFINITE, "illumination contains NaN or Inf");
    if (P->count_in == 0) return fail(CGH_ERR_EMPTY_MASK, "metric mask has no true pixels");
    if (P->denom == 0) return fail(CGH_ERR_ZERO_TARGET, "target is zero inside the mask");
    const bool has_cancel = cb && cb->cancel, has_progress = cb && cb->progress;
    int gmax = 64;
    if (const char* e = getenv("CGHB200_OSPR_GROUP")) gmax = std::max(1, std::min(64, atoi(e)));
    const int G = (has_cancel || has_progress) ? 1 : std::min(S, gmax);
    const long n = long(P->H) * P->W;
    CGH_TRY(ensure(P, P->data, size_t(n) * sizeof(cx<T>) * std::max(G, 1)));
    CGH_TRY(ensure(P, P->idx, size_t(n) * P->idx_bytes * std::max(S, 1)));
    const bool carry = G < S;
    if (carry || has_cancel) CGH_TRY(ensure(P, P->intensity, size_t(n) * sizeof(T)));
    const int nb = std::max(row_grid_blocks<T>(P->W, P->H), col_grid_blocks<T>(P->H, P->W));
    CGH_TRY(ensure(P, P->partials, size_t(nb) * (3 * 64 + 2) * sizeof(double)));
    CGH_TRY(ensure_res(P, size_t(S + 2)));
    CGH_TRY(ensure(P, P->frame_rng, sizeof(Pcg64) * std::max(S, 1)));
    std::vector<Pcg64> fr(S);
    for (int i = 0; i < S; ++i) fr[i] = to_pcg(op->frame_rng[i]);
    if (S) CGH_CUDA(cudaMemcpyAsync(P->frame_rng.p, fr.data(), sizeof(Pcg64) * S, cudaMemcpyHostToDevice, P->st));
    PassArgs<T> a = base_args<T>(P);
    a.frame_rng = static_cast<const Pcg64*>(P->frame_rng.p);
    a.intensity = static_cast<T*>(P->intensity.p);
    a.red.out = P->res_d;
    a.nframes_total = S;
    const long launches0 = P->launches;
    CGH_CUDA(cudaEventRecord(P->ev0, P->st));
    ProgressQueue pq;
    CGH_TRY(pq.init(P, cb, has_cancel && has_progress ? 0 : 4, P->res_h, 1));
    pq.kbias = 1;   // progress(len(frames), err)
    int done = 0;
    bool stop = false;
    int g_start = 0;
    if constexpr (sizeof(T) == 4) {
        // 2048^2 fp32 without hooks: every subframe in one persistent launch
        if (S > 0 && !has_cancel && !has_progress && wl_ospr_eligible(P) && P->idx_bytes == 1) {
            CGH_TRY(wl_ospr_run(P, a, S));
            done = S;
            g_start = S;
        }
    }
    for (int g0 = g_start; g0 < S; g0 += G) {
        if (cancelled(cb)) {
            stop = true;
            break;
        }
        const int m = std::min(G, S - g0);
        PassArgs<T> b = a;
        b.frame0 = g0;
        b.frames = m;
        bool fast_ospr = false;
        if constexpr (sizeof(T) == 4) fast_ospr = fast_ospr_eligible(P);
        if constexpr (sizeof(T) == 4) {
            if (fast_ospr) CGH_TRY(fast_ospr_gen(P, b));
            else CGH_TRY(run_row<T>(P, ROW_OSPR_GEN, b, m));
        } else {
            CGH_TRY(run_row<T>(P, ROW_OSPR_GEN, b, m));
        }
        b.quantize = 1;
        b.idx_out = static_cast<uint8_t*>(P->idx.p) + size_t(g0) * n * P->idx_bytes;
        bool fast_done = false;
        if constexpr (sizeof(T) == 4) {
            if (fast_ospr_eligible(P)) {
                CGH_TRY(fast_ospr_holo(P, b, m, std::max(G, 1), static_cast<uint8_t*>(b.idx_out)));
                fast_done = true;
            }
        }
        if (!fast_done) CGH_TRY(run_col<T>(P, COL_HOLO, b, m));
        b.idx_out = nullptr;
        b.quantize = 0;
        b.load_intensity = g0 > 0 ? 1 : 0;
        b.store_intensity = (carry || has_cancel) ? 1 : 0;
        if constexpr (sizeof(T) == 4) {
            if (fast_ospr) CGH_TRY(fast_ospr_acc(P, b));
            else CGH_TRY(run_row<T>(P, ROW_OSPR_ACC, b, 1));
        } else {
            CGH_TRY(run_row<T>(P, ROW_OSPR_ACC, b, 1));
        }
        done = g0 + m;
        if (has_progress || has_cancel) {
            for (int f = g0; f < g0 + m; ++f) CGH_TRY(pq.push(f));
            CGH_TRY(pq.poll(false));
        }
    }
    if (stop && done > 0) {
        // efficiency of the frames produced so far
        PassArgs<T> b = a;
        b.frame0 = done;
        b.frames = 0;
        b.nframes_total = done;
        b.load_intensity = 1;
        CGH_TRY(run_row<T>(P, ROW_OSPR_ACC, b, 1));
    }
    CGH_CUDA(cudaEventRecord(P->ev1, P->st));
    CGH_TRY(pq.poll(true));
    CGH_CUDA(cudaEventSynchronize(P->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, P->ev0, P->ev1);
    P->idx_frames = done;
    volatile const double* res = P->res_h;
    double final_err, eff;
    int64_t len;
    if (done > 0) {
        final_err = res[done - 1];
        eff = res[done];
        if (std::isnan(eff)) return fail(CGH_ERR_ZERO_FIELD, "replay field is zero");
        len = done;
    } else {
        final_err = 1.0;   // zero replay scores sum(t^2)/sum(t^2) (algorithms.py:516-520)
        eff = 0.0;
        len = 1;
    }
    if (tk && tv) {
        if (cap < len) return fail(CGH_ERR_VALUE, "trace capacity %lld < %lld", (long long)cap, (long long)len);
        if (done > 0) {
            for (int f = 0; f < done; ++f) {
                tk[f] = f + 1;
                tv[f] = res[f];
            }
        } else {
            tk[0] = 0;
            tv[0] = final_err;
        }
    }
    if (rep) {
        rep->final_error = final_err;
        rep->efficiency = eff;
        rep->iterations_executed = done;
        rep->termination = stop ? CGH_CANCELLED : CGH_COMPLETED;
        rep->trace_len = len;
        rep->kernel_launches = P->launches - launches0;
        rep->device_ms = ms;
    }
    return CGH_OK;
}

// ====================================================== sharded OSPR part
// One rank's contiguous range [frame0, frame0 + m) of the S subframes of a
// run_ospr sharded across GPUs. Phase 1 generates the
// local subframes (K1, K2: index planes final) and accumulates their |R|^2
// from a zero base into the plan's intensity plane. The caller then sets the
// plane to the sum of the lower ranks' totals (cgh_plan_set_intensity) and
// phase 2 re-runs only K3 over the resident subframes with the global frame
// numbers, giving the reference's cumulative per-frame errors; the rank
// holding frame S-1 also gets the efficiency.
template <class T>
static int ospr_part_exec(cgh_plan* P, const cgh_ospr_params* op, int frame0, int nframes_total, int phase,
                          int64_t* tk, double* tv, int64_t cap, cgh_report* rep) {
    if (!P->target_ready) return fail(CGH_ERR_VALUE, "target not set");
    const int m = std::max(0, op->subframes);
    if (m < 1) return fail(CGH_ERR_VALUE, "a sharded OSPR part holds at least one subframe (got %d)", m);
    if (frame0 < 0 || frame0 + m > nframes_total) return fail(CGH_ERR_VALUE, "frames [%d, %d) outside %d", frame0, frame0 + m, nframes_total);
    if (phase != 1 && phase != 2) return fail(CGH_ERR_VALUE, "phase must be 1 or 2");
    if (P->nf_all > 0) return fail(CGH_ERR_NONFINITE, "target contains NaN or Inf");
    if (P->nf_beam > 0) return fail(CGH_ERR_NONFINITE, "illumination contains NaN or Inf");
    if (P->count_in == 0) return fail(CGH_ERR_EMPTY_MASK, "metric mask has no true pixels");
    if (P->denom == 0) return fail(CGH_ERR_ZERO_TARGET, "target is zero inside the mask");
    const long n = long(P->H) * P->W;
    const long launches0 = P->launches;
    CGH_TRY(ensure(P, P->intensity, size_t(n) * sizeof(T)));
    const int nb = std::max(row_grid_blocks<T>(P->W, P->H), col_grid_blocks<T>(P->H, P->W));
    CGH_TRY(ensure(P, P->partials, size_t(nb) * (3 * 64 + 2) * sizeof(double)));
    CGH_TRY(ensure_res(P, size_t(nframes_total + 2)));
    if (phase == 1) {   // buffers before base_args() captures their addresses
        if (!op->frame_rng) return fail(CGH_ERR_VALUE, "frame streams missing");
        CGH_TRY(ensure(P, P->data, size_t(n) * sizeof(cx<T>) * m));
        CGH_TRY(ensure(P, P->idx, size_t(n) * P->idx_bytes * m));
        CGH_TRY(ensure(P, P->frame_rng, sizeof(Pcg64) * m));
    } else if (P->data.cap < size_t(n) * sizeof(cx<T>) * m) {
        return fail(CGH_ERR_VALUE, "phase 2 needs the frames of phase 1 on this plan");
    }
    PassArgs<T> a = base_args<T>(P);
    a.intensity = static_cast<T*>(P->intensity.p);
    a.red.out = P->res_d;
    a.frames = m;
    CGH_CUDA(cudaEventRecord(P->ev0, P->st));
    if (phase == 1) {
        std::vector<Pcg64> fr(m);
        for (int i = 0; i < m; ++i) fr[i] = to_pcg(op->frame_rng[i]);
        CGH_CUDA(cudaMemcpyAsync(P->frame_rng.p, fr.data(), sizeof(Pcg64) * m, cudaMemcpyHostToDevice, P->st));
        CGH_CUDA(cudaStreamSynchronize(P->st));   // fr is a temporary
        a.frame_rng = static_cast<const Pcg64*>(P->frame_rng.p);
        // local numbering for the streams; errors of this phase are not used
        a.frame0 = 0;
        a.nframes_total = m;
        bool fast = false;
        if constexpr (sizeof(T) == 4) fast = fast_ospr_eligible(P);
        if constexpr (sizeof(T) == 4) {
            if (fast) CGH_TRY(fast_ospr_gen(P, a));
            else CGH_TRY(run_row<T>(P, ROW_OSPR_GEN, a, m));
        } else {
            CGH_TRY(run_row<T>(P, ROW_OSPR_GEN, a, m));
        }
        PassArgs<T> b = a;
        b.quantize = 1;
        b.idx_out = P->idx.p;
        bool fast_done = false;
        if constexpr (sizeof(T) == 4) {
            if (fast) {
                CGH_TRY(fast_ospr_holo(P, b, m, m, static_cast<uint8_t*>(b.idx_out)));
                fast_done = true;
            }
        }
        if (!fast_done) CGH_TRY(run_col<T>(P, COL_HOLO, b, m));
        P->idx_frames = m;
    }
    // K3: phase 1 from a zero base, phase 2 from the base the caller loaded;
    // groups of <= 64 resident subframes (the per-frame partial slots), the
    // intensity carried between groups as in ospr_exec
    bool fast = false;
    if constexpr (sizeof(T) == 4) fast = fast_ospr_eligible(P);
    for (int g0 = 0; g0 < m; g0 += 64) {
        PassArgs<T> c = a;
        c.data = a.data + size_t(g0) * n;
        c.frames = std::min(64, m - g0);
        c.frame0 = (phase == 1 ? 0 : frame0) + g0;
        c.nframes_total = phase == 1 ? m : nframes_total;
        c.load_intensity = (phase == 2 || g0 > 0) ? 1 : 0;
        c.store_intensity = 1;
        if constexpr (sizeof(T) == 4) {
            if (fast) CGH_TRY(fast_ospr_acc(P, c));
            else CGH_TRY(run_row<T>(P, ROW_OSPR_ACC, c, 1));
        } else {
            CGH_TRY(run_row<T>(P, ROW_OSPR_ACC, c, 1));
        }
    }
    CGH_CUDA(cudaEventRecord(P->ev1, P->st));
    CGH_CUDA(cudaEventSynchronize(P->ev1));
    float ms = 0;
    cudaEventElapsedTime(&ms, P->ev0, P->ev1);
    volatile const double* res = P->res_h;
    const bool tail = phase == 2 && frame0 + m == nframes_total;
    if (tk && tv) {
        if (cap < m) return fail(CGH_ERR_VALUE, "trace capacity %lld < %d", (long long)cap, m);
        for (int f = 0; f < m; ++f) {
            tk[f] = (phase == 2 ? frame0 : 0) + f + 1;
            tv[f] = res[(phase == 2 ? frame0 : 0) + f];
        }
    }
    if (rep) {
        rep->final_error = res[(phase == 2 ? frame0 : 0) + m - 1];
        rep->efficiency = tail ? res[nframes_total] : std::nan("");
        if (tail && std::isnan(rep->efficiency)) return fail(CGH_ERR_ZERO_FIELD, "replay field is zero");
        rep->iterations_executed = m;
        rep->termination = CGH_COMPLETED;
        rep->trace_len = m;
        rep->kernel_launches = P->launches - launches0;
        rep->device_ms = ms;
    }
    return CGH_OK;
}

template <class T>
__global__ void sum_planes_kernel(const T* const* __restrict__ planes, int count, long n, T* __restrict__ out) {
    for (long p = (long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        T s = T(0);
        for (int i = 0; i < count; ++i) s += planes[i][p];   // fixed order: planes 0, 1, ...
        out[p] = s;
    }
}

// ============================================================== quantize
__global__ void quantize_kernel(const double* __restrict__ v, long n, SchemeDev s, int32_t* __restrict__ out) {
    for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        out[i] = quantize_index<double>(s, mk<double>(v[2 * i], v[2 * i + 1]));
}

// Fixed-order fp64 masked sums (grid-stride ownership, block tree, last block).
__global__ void masked_sums_kernel(const double* __restrict__ rep, const double* __restrict__ tgt,
                                   const uint8_t* __restrict__ mask, long n, double scale, double* partials,
                                   unsigned* counter, double* out) {
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        const double r = hypot(rep[2 * i], rep[2 * i + 1]);
        const double t = hypot(tgt[2 * i], tgt[2 * i + 1]);
        acc[5] += r * r;
        if (mask[i]) {
            const double d = scale * r - t;
            acc[0] += 1.0;
            acc[1] += t * t;
            acc[2] += r * r;
            acc[3] += r * t;
            acc[4] += d * d;
        }
    }
    __shared__ double sh[32 * 6];
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_down_sync(0xffffffffu, acc[q], o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
        for (int q = 0; q < 6; ++q) sh[q * 32 + warp] = acc[q];
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 6; ++q) {
            double s = 0;
            for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
            partials[q * gridDim.x + blockIdx.x] = s;
        }
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {   // whole last block, fixed order (see prep_kernel)
        __threadfence();
        double tot[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            double s = 0;
            for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(&partials[q * gridDim.x + b]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
            tot[q] = s;
        }
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 6; ++q) sh[q * 32 + warp] = tot[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < 6; ++q) {
                double s = 0;
                for (int w = 0; w < nw; ++w) s += sh[q * 32 + w];
                out[q] = s;
            }
            *counter = 0u;
        }
    }
}

__global__ void random_doubles_kernel(Pcg64 g, long skip, long n, double* out) {
    for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
        Pcg64 h = g;
        pcg_advance(h, uint64_t(skip + i));
        out[i] = pcg_next_double(h);
    }
}

}  // namespace cgh

using namespace cgh;

// ================================================================== C ABI
extern "C" {

int cgh_version(void) { return 10000; }

const char* cgh_last_error(void) { return g_err.c_str(); }

int cgh_device_count(int32_t* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = (e == cudaSuccess) ? n : 0;
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(CGH_ERR_NO_DEVICE, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    return CGH_OK;
}

int cgh_plan_create(const cgh_problem* pb, cgh_plan** out) {
    if (!out) return fail(CGH_ERR_VALUE, "null output");
    *out = nullptr;
    cgh_plan* P = new (std::nothrow) cgh_plan();
    if (!P) return fail(CGH_ERR_MEMORY, "plan allocation");
    int s = plan_init(P, pb);
    if (s != CGH_OK) {
        plan_free(P);
        delete P;
        return s;
    }
    *out = P;
    return CGH_OK;
}

int cgh_plan_destroy(cgh_plan* plan) {
    if (plan) {
        plan_free(plan);
        delete plan;
    }
    return CGH_OK;
}

int cgh_plan_set_target(cgh_plan* plan, const double* target, const uint8_t* mask, const double* illumination) {
    if (!plan) return fail(CGH_ERR_VALUE, "null plan");
    return plan_upload_target(plan, target, mask, illumination);
}

int cgh_plan_set_target_ex(cgh_plan* plan, const double* target, const uint8_t* mask, const double* illumination,
                           int32_t flags) {
    if (!plan) return fail(CGH_ERR_VALUE, "null plan");
    return plan_upload_target_ex(plan, target, mask, illumination, flags);
}

int cgh_plan_gs(cgh_plan* plan, const cgh_gs_params* gp, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                cgh_report* rep, const cgh_callbacks* cb) {
    if (!plan || !gp) return fail(CGH_ERR_VALUE, "null argument");
    CGH_CUDA(cudaSetDevice(plan->dev));
    GateLock gate(plan->dev, wl_eligible(plan));   // the warp-line loop is a grid-barrier kernel
    return plan->prec == CGH_FP64 ? gs_exec<double>(plan, gp, trace_k, trace_v, trace_cap, rep, cb, nullptr)
                                  : gs_exec<float>(plan, gp, trace_k, trace_v, trace_cap, rep, cb, nullptr);
}

int cgh_plan_ospr(cgh_plan* plan, const cgh_ospr_params* op, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                  cgh_report* rep, const cgh_callbacks* cb) {
    if (!plan || !op) return fail(CGH_ERR_VALUE, "null argument");
    CGH_CUDA(cudaSetDevice(plan->dev));
    GateLock gate(plan->dev, wl_ospr_eligible(plan));
    return plan->prec == CGH_FP64 ? ospr_exec<double>(plan, op, trace_k, trace_v, trace_cap, rep, cb)
                                  : ospr_exec<float>(plan, op, trace_k, trace_v, trace_cap, rep, cb);
}

int cgh_plan_ospr_part(cgh_plan* plan, const cgh_ospr_params* op, int32_t frame0, int32_t nframes_total,
                       int32_t phase, int64_t* trace_k, double* trace_v, int64_t trace_cap, cgh_report* rep) {
    if (!plan || !op) return fail(CGH_ERR_VALUE, "null argument");
    CGH_CUDA(cudaSetDevice(plan->dev));
    GateLock gate(plan->dev, false);
    return plan->prec == CGH_FP64
               ? ospr_part_exec<double>(plan, op, frame0, nframes_total, phase, trace_k, trace_v, trace_cap, rep)
               : ospr_part_exec<float>(plan, op, frame0, nframes_total, phase, trace_k, trace_v, trace_cap, rep);
}

int cgh_plan_set_intensity(cgh_plan* plan, const void* const* planes, int32_t count) {
    if (!plan || count < 0 || (count > 0 && !planes)) return fail(CGH_ERR_VALUE, "bad arguments");
    CGH_CUDA(cudaSetDevice(plan->dev));
    const long n = long(plan->H) * plan->W;
    const size_t es = plan->prec == CGH_FP64 ? 8 : 4;
    CGH_TRY(ensure(plan, plan->intensity, size_t(n) * es));
    void* d_ptrs = nullptr;
    if (count > 0) {
        CGH_CUDA(cudaMallocAsync(&d_ptrs, sizeof(void*) * count, plan->st));
        CGH_CUDA(cudaMemcpyAsync(d_ptrs, planes, sizeof(void*) * count, cudaMemcpyHostToDevice, plan->st));
    }
    if (plan->prec == CGH_FP64)
        sum_planes_kernel<double><<<grid_for(n), 256, 0, plan->st>>>(static_cast<const double* const*>(d_ptrs), count, n,
                                                                     static_cast<double*>(plan->intensity.p));
    else
        sum_planes_kernel<float><<<grid_for(n), 256, 0, plan->st>>>(static_cast<const float* const*>(d_ptrs), count, n,
                                                                    static_cast<float*>(plan->intensity.p));
    plan->launches += 1;
    CGH_CUDA(cudaGetLastError());
    if (d_ptrs) CGH_CUDA(cudaFreeAsync(d_ptrs, plan->st));
    CGH_CUDA(cudaStreamSynchronize(plan->st));   // `planes` is a host temporary of the caller
    return CGH_OK;
}

int cgh_plan_copy_intensity(cgh_plan* plan, void* dst) {
    if (!plan || !dst || !plan->intensity.p) return fail(CGH_ERR_VALUE, "no intensity plane");
    CGH_CUDA(cudaSetDevice(plan->dev));
    const size_t bytes = size_t(plan->H) * plan->W * (plan->prec == CGH_FP64 ? 8 : 4);
    CGH_CUDA(cudaMemcpyAsync(dst, plan->intensity.p, bytes, cudaMemcpyDeviceToDevice, plan->st));
    CGH_CUDA(cudaStreamSynchronize(plan->st));
    return CGH_OK;
}

int cgh_plan_intensity(cgh_plan* plan, void** out_ptr, int64_t* out_bytes) {
    if (!plan || !out_ptr) return fail(CGH_ERR_VALUE, "bad arguments");
    *out_ptr = plan->intensity.p;
    if (out_bytes) *out_bytes = int64_t(plan->intensity.cap);
    return CGH_OK;
}

int cgh_plan_download_idx(cgh_plan* plan, void* out_idx, int64_t frames) {
    if (!plan || !out_idx) return fail(CGH_ERR_VALUE, "null argument");
    if (frames > plan->idx_frames) return fail(CGH_ERR_VALUE, "only %d index planes held", plan->idx_frames);
    CGH_CUDA(cudaSetDevice(plan->dev));
    const size_t bytes = size_t(frames) * plan->H * plan->W * plan->idx_bytes;
    if (bytes) CGH_CUDA(cudaMemcpyAsync(out_idx, plan->idx.p, bytes, cudaMemcpyDeviceToHost, plan->st));
    CGH_CUDA(cudaStreamSynchronize(plan->st));
    return CGH_OK;
}

int cgh_plan_profile(cgh_plan* plan, int32_t enable, double* ms, int64_t* counts, int32_t n) {
    if (!plan) return fail(CGH_ERR_VALUE, "null plan");
    CGH_CUDA(cudaSetDevice(plan->dev));
    if (ms && counts) {
        CGH_CUDA(cudaStreamSynchronize(plan->st));
        for (int i = 0; i < n; ++i) {
            ms[i] = 0;
            counts[i] = 0;
        }
        for (size_t k = 0; k < plan->prof_id.size() && 2 * k + 1 < plan->prof_ev.size(); ++k) {
            float t = 0;
            CGH_CUDA(cudaEventElapsedTime(&t, plan->prof_ev[2 * k], plan->prof_ev[2 * k + 1]));
            const int id = plan->prof_id[k];
            if (id >= 0 && id < n) {
                ms[id] += t;
                counts[id] += 1;
            }
        }
    }
    for (auto e : plan->prof_ev) cudaEventDestroy(e);
    plan->prof_ev.clear();
    plan->prof_id.clear();
    plan->profiling = enable != 0;
    return CGH_OK;
}

void* cgh_plan_stream(cgh_plan* plan) { return plan ? (void*)plan->st : nullptr; }

int cgh_plan_sync(cgh_plan* plan) {
    if (!plan) return fail(CGH_ERR_VALUE, "null plan");
    CGH_CUDA(cudaSetDevice(plan->dev));
    CGH_CUDA(cudaStreamSynchronize(plan->st));
    return CGH_OK;
}

struct PlanGuard {
    cgh_plan* p = nullptr;
    ~PlanGuard() { cgh_plan_destroy(p); }
};

int cgh_transform(const cgh_problem* pb, const double* in, double* out, int32_t op) {
    if (!in || !out || !pb) return fail(CGH_ERR_VALUE, "null buffer");
    if (op < 0 || op > 3) return fail(CGH_ERR_VALUE, "direction must be 'forward' or 'inverse'");
    if (pb->height >= 1 && pb->width >= 1 &&
        (!is_pow2(pb->height) || !is_pow2(pb->width) || pb->height > (1 << kMaxLog2) || pb->width > (1 << kMaxLog2))) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
        if (pb->device < 0 || pb->device >= ndev) return fail(CGH_ERR_VALUE, "device %d out of range", pb->device);
        return transform_any(pb, in, out, op);   // Bluestein line transforms (anysize.cu)
    }
    PlanGuard g;
    CGH_TRY(cgh_plan_create(pb, &g.p));
    return g.p->prec == CGH_FP64 ? transform_exec<double>(g.p, in, out, op) : transform_exec<float>(g.p, in, out, op);
}

int cgh_quantize(const cgh_problem* pb, const double* values, int64_t count, int32_t* out_idx) {
    if (count < 0 || (count > 0 && (!values || !out_idx))) return fail(CGH_ERR_VALUE, "bad buffers");
    if (count == 0) return CGH_OK;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    if (pb->n_states < 2 || !pb->states) return fail(CGH_ERR_VALUE, "scheme needs >= 2 states");
    CGH_CUDA(cudaSetDevice(pb->device));
    cudaStream_t st;
    CGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *dv = nullptr, *ds = nullptr;
    int32_t* di = nullptr;
    int rc = CGH_OK;
    const size_t ns = size_t(pb->n_states);
    auto cleanup = [&] {
        if (dv) cudaFreeAsync(dv, st);
        if (ds) cudaFreeAsync(ds, st);
        if (di) cudaFreeAsync(di, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    };
    do {
        if (cudaMallocAsync(&dv, size_t(count) * 16, st) != cudaSuccess || cudaMallocAsync(&ds, ns * 16, st) != cudaSuccess ||
            cudaMallocAsync(&di, size_t(count) * 4, st) != cudaSuccess) {
            rc = fail(CGH_ERR_MEMORY, "quantize buffers");
            break;
        }
        cudaMemcpyAsync(dv, values, size_t(count) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(ds, pb->states, ns * 16, cudaMemcpyHostToDevice, st);
        SchemeDev s;
        s.kind = pb->scheme_kind;
        s.n = pb->n_states;
        s.offset = pb->phase_offset;
        s.step = 2.0 * 3.141592653589793 / double(pb->n_states);
        s.states64 = ds;
        s.states32 = nullptr;
        quantize_kernel<<<grid_for(count), 256, 0, st>>>(dv, count, s, di);
        cudaMemcpyAsync(out_idx, di, size_t(count) * 4, cudaMemcpyDeviceToHost, st);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(CGH_ERR_CUDA, "quantize: %s", cudaGetErrorString(e));
    } while (0);
    cleanup();
    return rc;
}

int cgh_masked_sums(int32_t device, const double* replay, const double* target, const uint8_t* mask, int64_t count,
                    double scale, double* out) {
    if (count < 0 || !out || (count > 0 && (!replay || !target || !mask))) return fail(CGH_ERR_VALUE, "bad buffers");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    CGH_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    CGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const int grid = grid_for(std::max<int64_t>(count, 1));
    char* buf = nullptr;
    const size_t nb = size_t(std::max<int64_t>(count, 1));
    const size_t bytes = nb * 33 + size_t(grid) * 6 * 8 + 64 + 64;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&buf), bytes, st);
    if (e == cudaSuccess) {
        double* dr = reinterpret_cast<double*>(buf);
        double* dt = dr + 2 * nb;
        double* part = dt + 2 * nb;
        double* dout = part + size_t(grid) * 6;
        unsigned* ctr = reinterpret_cast<unsigned*>(dout + 8);
        uint8_t* dm = reinterpret_cast<uint8_t*>(ctr + 4);
        cudaMemcpyAsync(dr, replay, size_t(count) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dt, target, size_t(count) * 16, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dm, mask, size_t(count), cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(ctr, 0, 16, st);
        masked_sums_kernel<<<grid, 256, 0, st>>>(dr, dt, dm, count, scale, part, ctr, dout);
        cudaMemcpyAsync(out, dout, 6 * 8, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(buf, st);
        e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    cudaStreamDestroy(st);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "masked_sums: %s", cudaGetErrorString(e));
    return CGH_OK;
}

int cgh_gs_run(const cgh_problem* pb, const cgh_gs_params* gp, const double* target, const uint8_t* mask,
               const double* illumination, void* out_idx, double* out_field, int64_t* trace_k, double* trace_v,
               int64_t trace_cap, cgh_report* rep, const cgh_callbacks* cb) {
    if (!gp) return fail(CGH_ERR_VALUE, "null params");
    PlanGuard g;
    CGH_TRY(cgh_plan_create(pb, &g.p));
    cgh_plan* P = g.p;
    CGH_TRY(plan_upload_target(P, target, mask, illumination));
    const long n = long(P->H) * P->W;
    DevBuf& fb = P->field;
    if (out_field) CGH_TRY(ensure(P, fb, size_t(n) * (P->prec == CGH_FP64 ? 16 : 8)));
    GateLock gate(P->dev, wl_eligible(P));
    int s = P->prec == CGH_FP64
                ? gs_exec<double>(P, gp, trace_k, trace_v, trace_cap, rep, cb, out_field ? static_cast<cx<double>*>(fb.p) : nullptr)
                : gs_exec<float>(P, gp, trace_k, trace_v, trace_cap, rep, cb, out_field ? static_cast<cx<float>*>(fb.p) : nullptr);
    if (s != CGH_OK) return s;
    if (out_idx) CGH_TRY(cgh_plan_download_idx(P, out_idx, 1));
    if (out_field) {
        if (P->prec == CGH_FP64) {
            CGH_CUDA(cudaMemcpyAsync(out_field, fb.p, size_t(n) * 16, cudaMemcpyDeviceToHost, P->st));
            CGH_CUDA(cudaStreamSynchronize(P->st));
        } else {
            std::vector<float> tmp(2 * size_t(n));
            CGH_CUDA(cudaMemcpyAsync(tmp.data(), fb.p, size_t(n) * 8, cudaMemcpyDeviceToHost, P->st));
            CGH_CUDA(cudaStreamSynchronize(P->st));
            for (size_t i = 0; i < 2 * size_t(n); ++i) out_field[i] = tmp[i];
        }
    }
    return CGH_OK;
}

int cgh_ospr_run(const cgh_problem* pb, const cgh_ospr_params* op, const double* target, const uint8_t* mask,
                 const double* illumination, void* out_idx, int64_t* trace_k, double* trace_v, int64_t trace_cap,
                 cgh_report* rep, const cgh_callbacks* cb) {
    if (!op) return fail(CGH_ERR_VALUE, "null params");
    PlanGuard g;
    CGH_TRY(cgh_plan_create(pb, &g.p));
    cgh_plan* P = g.p;
    CGH_TRY(plan_upload_target(P, target, mask, illumination));
    cgh_report r{};
    CGH_TRY(cgh_plan_ospr(P, op, trace_k, trace_v, trace_cap, &r, cb));
    if (rep) *rep = r;
    if (out_idx && r.iterations_executed > 0) CGH_TRY(cgh_plan_download_idx(P, out_idx, r.iterations_executed));
    return CGH_OK;
}

int cgh_expand_states(const void* idx, int32_t idx_bytes, int64_t count, const double* states, int32_t n_states,
                      double* out, int32_t threads) {
    if (count < 0 || (count > 0 && (!idx || !states || !out)) || (idx_bytes != 1 && idx_bytes != 4))
        return fail(CGH_ERR_VALUE, "bad arguments");
    const int nt = std::max(1, std::min(threads > 0 ? threads : 8, 64));
    std::atomic<int> bad{0};
    // streaming 16-byte stores when the output is 16-byte aligned (numpy's
    // large arrays are): the complex128 plane is written once, never read here
#if defined(__SSE2__)
    const bool nt_ok = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
#else
    const bool nt_ok = false;
#endif
    auto work = [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            const int k = idx_bytes == 1 ? int(static_cast<const uint8_t*>(idx)[i]) : static_cast<const int32_t*>(idx)[i];
            if (k < 0 || k >= n_states) {
                bad = 1;
                continue;
            }
#if defined(__SSE2__)
            if (nt_ok) {
                _mm_stream_pd(out + 2 * i, _mm_set_pd(states[2 * k + 1], states[2 * k]));
                continue;
            }
#endif
            out[2 * i] = states[2 * k];
            out[2 * i + 1] = states[2 * k + 1];
        }
        stream_fence();
    };
    const int64_t chunk = (count + nt - 1) / nt;
    HostPool::get().run(nt, [&](int t) {
        const int64_t a = t * chunk, b = std::min(count, a + chunk);
        if (a < b) work(a, b);
    });
    if (bad) return fail(CGH_ERR_VALUE, "index outside the state table");
    return CGH_OK;
}

int cgh_prefault(void* p, int64_t bytes, int32_t threads) {
    if (bytes < 0 || (bytes > 0 && !p)) return fail(CGH_ERR_VALUE, "bad arguments");
    constexpr int64_t kPage = 4096;
    const int64_t pages = (bytes + kPage - 1) / kPage;
    const int nt = int(std::max<int64_t>(1, std::min<int64_t>({int64_t(threads > 0 ? threads : 4), 64, pages})));
    auto touch = [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) static_cast<volatile char*>(p)[i * kPage] = 0;
    };
    const int64_t chunk = (pages + nt - 1) / nt;
    HostPool::get().run(nt, [&](int t) {
        const int64_t a = t * chunk, b = std::min(pages, a + chunk);
        if (a < b) touch(a, b);
    });
    return CGH_OK;
}

int cgh_permutation(const cgh_pcg64* rng, int64_t n, int64_t* out) {
    if (!rng || (n > 0 && !out) || n < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    Pcg64 g = to_pcg(*rng);
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    for (int64_t i = n - 1; i > 0; --i) {
        const int64_t j = int64_t(pcg_interval(g, uint64_t(i)));
        std::swap(out[i], out[j]);
    }
    return CGH_OK;
}

int cgh_random_doubles(int32_t device, const cgh_pcg64* rng, int64_t skip, int64_t n, double* out) {
    if (!rng || n < 0 || (n > 0 && !out) || skip < 0) return fail(CGH_ERR_VALUE, "bad arguments");
    Pcg64 g = to_pcg(*rng);
    if (device < 0) {
        pcg_advance(g, uint64_t(skip));
        for (int64_t i = 0; i < n; ++i) out[i] = pcg_next_double(g);
        return CGH_OK;
    }
    CGH_CUDA(cudaSetDevice(device));
    double* d = nullptr;
    CGH_CUDA(cudaMalloc(&d, size_t(std::max<int64_t>(n, 1)) * 8));
    random_doubles_kernel<<<grid_for(n), 256>>>(g, skip, n, d);
    cudaError_t e = cudaMemcpy(out, d, size_t(n) * 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "random_doubles: %s", cudaGetErrorString(e));
    return CGH_OK;
}

}  // extern "C"
