// Host side + C ABI of the row-distributed GS slabs (slab_kernels.cuh,
// include/cghb200.h "row-distributed GS slabs"). The caller owns the slab
// buffers and the stream (torch tensors / NCCL in paper_2006_10509_b200/slab.py);
// this object owns the tables, the rank's target columns and beam rows, and
// the reduction scratch.
#include <algorithm>

#include "runtime.cuh"
#include "slab_kernels.cuh"

CGH_SLAB_EXTERN(float, 64)
CGH_SLAB_EXTERN(float, 128)
CGH_SLAB_EXTERN(float, 256)
CGH_SLAB_EXTERN(float, 512)
CGH_SLAB_EXTERN(float, 1024)
CGH_SLAB_EXTERN(float, 2048)
CGH_SLAB_EXTERN(float, 4096)
CGH_SLAB_EXTERN(float, 8192)
CGH_SLAB_EXTERN(float, 16384)
CGH_SLAB_EXTERN(double, 64)
CGH_SLAB_EXTERN(double, 128)
CGH_SLAB_EXTERN(double, 256)
CGH_SLAB_EXTERN(double, 512)
CGH_SLAB_EXTERN(double, 1024)
CGH_SLAB_EXTERN(double, 2048)
CGH_SLAB_EXTERN(double, 4096)
CGH_SLAB_EXTERN(double, 8192)

namespace cgh {

constexpr int kSlabMinN = 64;
constexpr int kSlabMaxN32 = 16384, kSlabMaxN64 = 8192;

template <class T>
static cudaError_t slab_dispatch(int N, const SlabArgs<T>& a, int mode, cudaStream_t st) {
    switch (N) {
        case 64: return slab_launch_n<T, 64>(a, mode, st);
        case 128: return slab_launch_n<T, 128>(a, mode, st);
        case 256: return slab_launch_n<T, 256>(a, mode, st);
        case 512: return slab_launch_n<T, 512>(a, mode, st);
        case 1024: return slab_launch_n<T, 1024>(a, mode, st);
        case 2048: return slab_launch_n<T, 2048>(a, mode, st);
        case 4096: return slab_launch_n<T, 4096>(a, mode, st);
        case 8192: return slab_launch_n<T, 8192>(a, mode, st);
        case 16384:
            if constexpr (sizeof(T) == 4) return slab_launch_n<T, 16384>(a, mode, st);
            else return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

template <class T>
static int slab_blocks_for(int N, int R) {
    switch (N) {
        case 64: return slab_blocks<T, 64>(R);
        case 128: return slab_blocks<T, 128>(R);
        case 256: return slab_blocks<T, 256>(R);
        case 512: return slab_blocks<T, 512>(R);
        case 1024: return slab_blocks<T, 1024>(R);
        case 2048: return slab_blocks<T, 2048>(R);
        case 4096: return slab_blocks<T, 4096>(R);
        case 8192: return slab_blocks<T, 8192>(R);
        default: return slab_blocks<T, 16384>(R);
    }
}

}  // namespace cgh

using namespace cgh;

struct cgh_slab {
    int dev = 0, N = 0, G = 1, rank = 0, R = 0, logS = 0, prec = CGH_FP32;
    cudaStream_t st = nullptr;
    int scheme_kind = 0, nstates = 0, idx_bytes = 1, prop_kind = CGH_FOURIER;
    double offset = 0, step = 0;
    void* states64 = nullptr;
    void* states32 = nullptr;
    void* tw = nullptr;
    void* q_row = nullptr;
    void* q_col = nullptr;
    void* tgt = nullptr;
    void* beam = nullptr;
    double* partials = nullptr;
    unsigned* counter = nullptr;
    bool ready = false;
};

namespace {

int slab_upload(cgh_slab* S, void** dst, const std::vector<double>& v) {
    const size_t n = v.size() / 2;
    if (S->prec == CGH_FP64) {
        CGH_CUDA(cudaMalloc(dst, n * 16));
        CGH_CUDA(cudaMemcpy(*dst, v.data(), n * 16, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> f(v.begin(), v.end());
        CGH_CUDA(cudaMalloc(dst, n * 8));
        CGH_CUDA(cudaMemcpy(*dst, f.data(), n * 8, cudaMemcpyHostToDevice));
    }
    return CGH_OK;
}

void slab_free(cgh_slab* S) {
    cudaSetDevice(S->dev);
    void* ps[] = {S->states64, S->states32, S->tw, S->q_row, S->q_col, S->tgt, S->beam, S->partials, S->counter};
    for (void* p : ps)
        if (p) cudaFree(p);
}

int slab_init(cgh_slab* S, const cgh_problem* pb, int world, int rank, void* stream) {
    if (!pb) return fail(CGH_ERR_VALUE, "null problem");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CGH_ERR_NO_DEVICE, "no CUDA device");
    if (pb->device < 0 || pb->device >= ndev) return fail(CGH_ERR_VALUE, "device %d out of range", pb->device);
    if (pb->height != pb->width) return fail(CGH_ERR_UNSUPPORTED, "slab runs need a square plane (got %dx%d)", pb->height, pb->width);
    const int N = pb->width;
    const int nmax = pb->precision == CGH_FP64 ? kSlabMaxN64 : kSlabMaxN32;
    if (!is_pow2(N) || N < kSlabMinN || N > nmax)
        return fail(CGH_ERR_UNSUPPORTED, "slab runs implement power-of-two N in %d..%d at this precision (got %d)", kSlabMinN,
                    nmax, N);
    if (world < 1 || !is_pow2(world == 1 ? 2 : world) || N % world || N / world < 1)
        return fail(CGH_ERR_VALUE, "world size %d must be a power of two dividing N = %d", world, N);
    if (rank < 0 || rank >= world) return fail(CGH_ERR_VALUE, "rank %d out of range (world %d)", rank, world);
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
    S->dev = pb->device;
    S->N = N;
    S->G = world;
    S->rank = rank;
    S->R = N / world;
    S->logS = 0;
    while ((1 << S->logS) < S->R) ++S->logS;
    S->prec = pb->precision;
    S->st = static_cast<cudaStream_t>(stream);
    S->scheme_kind = pb->scheme_kind;
    S->nstates = pb->n_states;
    S->offset = pb->phase_offset;
    S->step = pb->scheme_kind == CGH_SCHEME_PHASE ? 2.0 * 3.141592653589793 / double(pb->n_states) : 0.0;
    S->idx_bytes = pb->n_states <= 256 ? 1 : 4;
    S->prop_kind = pb->prop_kind;
    const size_t ns = size_t(pb->n_states);
    CGH_CUDA(cudaMalloc(&S->states64, ns * 16));
    CGH_CUDA(cudaMemcpy(S->states64, pb->states, ns * 16, cudaMemcpyHostToDevice));
    std::vector<float> s32(2 * ns);
    for (size_t i = 0; i < 2 * ns; ++i) s32[i] = float(pb->states[i]);
    CGH_CUDA(cudaMalloc(&S->states32, ns * 8));
    CGH_CUDA(cudaMemcpy(S->states32, s32.data(), ns * 8, cudaMemcpyHostToDevice));
    std::vector<double> t;
    twiddle_table(N, t);
    CGH_TRY(slab_upload(S, &S->tw, t));
    if (pb->prop_kind == CGH_FRESNEL) {
        chirp_table(N, pb->pitch_y, pb->wavelength, pb->distance, t);   // rows (global index)
        CGH_TRY(slab_upload(S, &S->q_row, t));
        chirp_table(N, pb->pitch_x, pb->wavelength, pb->distance, t);   // columns
        CGH_TRY(slab_upload(S, &S->q_col, t));
    }
    const int nb = std::max(slab_blocks_for<float>(N, S->R), slab_blocks_for<double>(N, S->R));
    CGH_CUDA(cudaMalloc(&S->partials, size_t(std::max(nb, 1)) * 4 * sizeof(double)));
    CGH_CUDA(cudaMalloc(&S->counter, 64));
    CGH_CUDA(cudaMemset(S->counter, 0, 64));
    return CGH_OK;
}

template <class T>
int slab_set_local(cgh_slab* S, const double* tgt, const double* beam) {
    const size_t n = size_t(S->R) * S->N;
    std::vector<T> buf(n);
    for (size_t i = 0; i < n; ++i) buf[i] = T(tgt[i]);   // keeps the sign bit of -0.0
    if (!S->tgt) CGH_CUDA(cudaMalloc(&S->tgt, n * sizeof(T)));
    CGH_CUDA(cudaMemcpy(S->tgt, buf.data(), n * sizeof(T), cudaMemcpyHostToDevice));
    if (beam) {
        for (size_t i = 0; i < n; ++i) buf[i] = T(beam[i]);
        if (!S->beam) CGH_CUDA(cudaMalloc(&S->beam, n * sizeof(T)));
        CGH_CUDA(cudaMemcpy(S->beam, buf.data(), n * sizeof(T), cudaMemcpyHostToDevice));
    } else if (S->beam) {
        CGH_CUDA(cudaFree(S->beam));
        S->beam = nullptr;
    }
    S->ready = true;
    return CGH_OK;
}

template <class T>
int slab_pass(cgh_slab* S, int mode, void* data, const cgh_gs_params* gp, int quantize, void* idx_out, double* sums) {
    if (mode < SLAB_INIT || mode > SLAB_FWD || mode == SLAB_HOLO_SNAP) return fail(CGH_ERR_VALUE, "bad slab pass mode %d", mode);
    if ((mode == SLAB_GS || mode == SLAB_FINAL) && (!S->ready || !sums))
        return fail(CGH_ERR_VALUE, "replay passes need the local target (cgh_slab_set_local) and a sums pointer");
    if (!data) return fail(CGH_ERR_VALUE, "null slab buffer");
    SlabArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.data = static_cast<cx<T>*>(data);
    a.R = S->R;
    a.logS = S->logS;
    a.line0 = S->rank * S->R;
    a.tgt = static_cast<const T*>(S->tgt);
    a.p.H = S->R;
    a.p.W = S->N;
    a.p.beam = static_cast<const T*>(S->beam);
    a.p.tw_row = static_cast<const cx<T>*>(S->tw);
    a.p.tw_col = a.p.tw_row;
    if (S->prop_kind == CGH_FRESNEL) {
        a.p.q_row = static_cast<const cx<T>*>(S->q_row) + a.line0;
        a.p.q_col = static_cast<const cx<T>*>(S->q_col);
    }
    a.p.scheme.kind = S->scheme_kind;
    a.p.scheme.n = S->nstates;
    a.p.scheme.offset = S->offset;
    a.p.scheme.step = S->step;
    a.p.scheme.states64 = static_cast<const double*>(S->states64);
    a.p.scheme.states32 = static_cast<const float*>(S->states32);
    a.p.quantize = quantize ? 1 : 0;
    a.p.idx_out = quantize ? idx_out : nullptr;
    a.p.idx_bytes = S->idx_bytes;
    a.gain = T(gp ? gp->feedback_gain : 0.0);
    a.scale = T(1.0 / double(S->N));   // 1/sqrt(N * N)
    if (gp) a.rng = to_pcg(gp->rng);
    a.red.partials = S->partials;
    a.red.counter = S->counter;
    a.red.out = sums;
    cudaError_t e = slab_dispatch<T>(S->N, a, mode, S->st);
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "slab pass (mode %d, N=%d): %s", mode, S->N, cudaGetErrorString(e));
    return CGH_OK;
}

}  // namespace

extern "C" {

int cgh_slab_create(const cgh_problem* pb, int32_t world, int32_t rank, void* stream, cgh_slab** out) {
    if (!out) return fail(CGH_ERR_VALUE, "null output handle");
    *out = nullptr;
    cgh_slab* S = new cgh_slab();
    int st = slab_init(S, pb, world, rank, stream);
    if (st != CGH_OK) {
        slab_free(S);
        delete S;
        return st;
    }
    *out = S;
    return CGH_OK;
}

int cgh_slab_destroy(cgh_slab* slab) {
    if (!slab) return CGH_OK;
    if (slab->st) cudaStreamSynchronize(slab->st);
    slab_free(slab);
    delete slab;
    return CGH_OK;
}

int cgh_slab_set_local(cgh_slab* slab, const double* tgt_local, const double* beam_local) {
    if (!slab || !tgt_local) return fail(CGH_ERR_VALUE, "null slab or target");
    CGH_CUDA(cudaSetDevice(slab->dev));
    return slab->prec == CGH_FP64 ? slab_set_local<double>(slab, tgt_local, beam_local)
                                  : slab_set_local<float>(slab, tgt_local, beam_local);
}

int cgh_slab_pass(cgh_slab* slab, int32_t mode, void* data, const cgh_gs_params* gp, int32_t quantize, void* idx_out,
                  double* sums) {
    if (!slab) return fail(CGH_ERR_VALUE, "null slab");
    CGH_CUDA(cudaSetDevice(slab->dev));
    return slab->prec == CGH_FP64 ? slab_pass<double>(slab, mode, data, gp, quantize, idx_out, sums)
                                  : slab_pass<float>(slab, mode, data, gp, quantize, idx_out, sums);
}

int cgh_slab_turn(cgh_slab* slab, const void* src, void* const* dst_blocks) {
    if (!slab || !src || !dst_blocks) return fail(CGH_ERR_VALUE, "null slab or buffer");
    if (slab->G > kMaxTurnBlocks) return fail(CGH_ERR_UNSUPPORTED, "at most %d ranks", kMaxTurnBlocks);
    CGH_CUDA(cudaSetDevice(slab->dev));
    const int S = slab->R;
    const int TL = slab->prec == CGH_FP64 ? turn_tile<double>() : turn_tile<float>();
    dim3 grid((S + TL - 1) / TL, (S + TL - 1) / TL, slab->G), block(32, 8);
    for (int g = 0; g < slab->G; ++g) {
        if (!dst_blocks[g]) return fail(CGH_ERR_VALUE, "null destination block %d", g);
        if (dst_blocks[g] == src) return fail(CGH_ERR_VALUE, "turn destination aliases the source");
    }
    if (slab->prec == CGH_FP64) {
        TurnTargets<double> t;
        for (int g = 0; g < slab->G; ++g) t.p[g] = static_cast<cx<double>*>(dst_blocks[g]);
        slab_turn_kernel<double><<<grid, block, 0, slab->st>>>(static_cast<const cx<double>*>(src), t, S);
    } else {
        TurnTargets<float> t;
        for (int g = 0; g < slab->G; ++g) t.p[g] = static_cast<cx<float>*>(dst_blocks[g]);
        slab_turn_kernel<float><<<grid, block, 0, slab->st>>>(static_cast<const cx<float>*>(src), t, S);
    }
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

int cgh_slab_transpose(cgh_slab* slab, const void* src, void* dst) {
    if (!slab || !src || !dst) return fail(CGH_ERR_VALUE, "null slab or buffer");
    if (src == dst) return fail(CGH_ERR_VALUE, "transpose needs distinct buffers");
    CGH_CUDA(cudaSetDevice(slab->dev));
    const int S = slab->R;
    dim3 grid((S + 31) / 32, (S + 31) / 32, slab->G), block(32, 8);
    if (slab->prec == CGH_FP64)
        slab_transpose_kernel<double><<<grid, block, 0, slab->st>>>(static_cast<const cx<double>*>(src),
                                                                    static_cast<cx<double>*>(dst), S);
    else
        slab_transpose_kernel<float><<<grid, block, 0, slab->st>>>(static_cast<const cx<float>*>(src),
                                                                   static_cast<cx<float>*>(dst), S);
    CGH_CUDA(cudaGetLastError());
    return CGH_OK;
}

}  // extern "C"
