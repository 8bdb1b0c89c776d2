// Centred unitary transforms of arbitrary H x W planes (propagation.py:81-123:
// fft2 forward/inverse, propagate, propagate_inverse) for the sides the
// power-of-two passes do not take. The reference accepts any SLM resolution
// 2..16384 (schema.py:51-63) and its tests transform 5 x 7 and 31 x 33 fields
// (tests/test_propagation.py:56-66).
//
// Each axis is a line DFT of length N computed with Bluestein's chirp-z
// identity nk = (n^2 + k^2 - (k - n)^2) / 2:
//     X_k = a_k * sum_n (x_n a_n) b_(k-n),   a_n = exp(-i pi n^2 / N), b = conj(a),
// a circular convolution of length M = pow2 >= 2N - 1 done with two M-point
// line FFTs (LineFft, the same Stockham code as the GS passes) and the
// M-point spectrum of b (computed once per call on the device). One CTA per
// line, line in registers, exchanges in shared memory; rows then columns
// (columns read with stride W). fp64 takes N <= 4096 (M <= 8192), fp32
// N <= 8192 (M <= 16384).
#include <cmath>
#include <vector>

#include "runtime.cuh"

namespace cgh {

template <class T>
struct BlueArgs {
    cx<T>* data;
    int N, lines;
    long line_stride, elem_stride;
    const cx<T>* chirp;   // [N] exp(-i pi n^2 / N)
    const cx<T>* filt;    // [M] FFT_M(b)
    const cx<T>* tw;      // [M] exp(-2 pi i k / M)
    int dir;              // -1 forward DFT, +1 inverse (unnormalised)
    T scale;
    int plain;            // plain forward M-point FFT of each line (builds filt)
};

template <class T, int M>
struct BlueShape {
    // 16384-point fp32 lines: 32 points per thread (as the slab passes)
    static constexpr int E = (sizeof(T) == 4 && M >= 16384) ? 32 : LineShape<T, M>::E;
    static constexpr int TF = M / E;
    static constexpr size_t SMEM = size_t(2) * line_words<T, M>() * sizeof(T);
};

template <class T, int M>
__global__ void __launch_bounds__(BlueShape<T, M>::TF) bluestein_kernel(BlueArgs<T> a) {
    using Sh = BlueShape<T, M>;
    constexpr int E = Sh::E, TF = Sh::TF;
    extern __shared__ __align__(16) unsigned char smem[];
    T* sre = reinterpret_cast<T*>(smem);
    T* sim = sre + line_words<T, M>();
    const int t = threadIdx.x;
    for (int line = blockIdx.x; line < a.lines; line += gridDim.x) {
        cx<T>* d = a.data + long(line) * a.line_stride;
        __syncthreads();
        cx<T> v[E];
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int j = t + r * TF;
            if (a.plain) {
                v[r] = d[long(j) * a.elem_stride];
            } else if (j < a.N) {
                const cx<T> c = a.chirp[j];
                v[r] = a.dir < 0 ? cmul(d[long(j) * a.elem_stride], c) : cmulc(d[long(j) * a.elem_stride], c);
            } else {
                v[r] = mk<T>(0, 0);
            }
        }
        LineFft<T, M, -1, E>::run(v, sre, sim, t, a.tw);
        if (a.plain) {
#pragma unroll
            for (int r = 0; r < E; ++r) d[long(t + r * TF) * a.elem_stride] = v[r];
            continue;
        }
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const cx<T> f = a.filt[t + r * TF];
            v[r] = a.dir < 0 ? cmul(v[r], f) : cmulc(v[r], f);
        }
        LineFft<T, M, +1, E>::run(v, sre, sim, t, a.tw);
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int j = t + r * TF;
            if (j < a.N) {
                const cx<T> c = a.chirp[j];
                const cx<T> y = a.dir < 0 ? cmul(v[r], c) : cmulc(v[r], c);
                d[long(j) * a.elem_stride] = y * a.scale;
            }
        }
    }
}

template <class T, int M>
static cudaError_t blue_launch_m(const BlueArgs<T>& a, int sms, cudaStream_t st) {
    using Sh = BlueShape<T, M>;
    if (Sh::SMEM > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(bluestein_kernel<T, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(Sh::SMEM));
        if (e != cudaSuccess) return e;
    }
    const int grid = std::max(1, std::min(a.lines, sms * 8));
    bluestein_kernel<T, M><<<grid, Sh::TF, Sh::SMEM, st>>>(a);
    return cudaGetLastError();
}

template <class T>
static int max_line_fft() { return sizeof(T) == 8 ? 8192 : 16384; }

template <class T>
static cudaError_t blue_launch(int M, const BlueArgs<T>& a, int sms, cudaStream_t st) {
    switch (M) {
        case 64: return blue_launch_m<T, 64>(a, sms, st);
        case 128: return blue_launch_m<T, 128>(a, sms, st);
        case 256: return blue_launch_m<T, 256>(a, sms, st);
        case 512: return blue_launch_m<T, 512>(a, sms, st);
        case 1024: return blue_launch_m<T, 1024>(a, sms, st);
        case 2048: return blue_launch_m<T, 2048>(a, sms, st);
        case 4096: return blue_launch_m<T, 4096>(a, sms, st);
        case 8192: return blue_launch_m<T, 8192>(a, sms, st);
        case 16384:
            if constexpr (sizeof(T) == 4) return blue_launch_m<T, 16384>(a, sms, st);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

static int blue_length(int n) {
    int m = 64;
    while (m < 2 * n - 1) m *= 2;
    return m;
}

namespace {

// Device buffers of one call, freed on every exit path.
struct CallBufs {
    cudaStream_t st = nullptr;
    std::vector<void*> ptrs;
    ~CallBufs() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
    void* alloc(size_t bytes) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) return nullptr;
        ptrs.push_back(p);
        return p;
    }
};

template <class T>
static cx<T>* upload_cx(CallBufs& B, const std::vector<double>& v) {
    const size_t n = v.size() / 2;
    cx<T>* d = static_cast<cx<T>*>(B.alloc(n * sizeof(cx<T>)));
    if (!d) return nullptr;
    std::vector<T> h(v.begin(), v.end());
    if (cudaMemcpyAsync(d, h.data(), n * sizeof(cx<T>), cudaMemcpyHostToDevice, B.st) != cudaSuccess) return nullptr;
    if (cudaStreamSynchronize(B.st) != cudaSuccess) return nullptr;   // h is a temporary
    return d;
}

// chirp exp(-i pi n^2 / N) (n^2 reduced mod 2N, long double) and the
// convolution kernel b = conj(chirp) wrapped to length M
static void chirp_tables(int N, int M, std::vector<double>& chirp, std::vector<double>& b) {
    const long double pi = 3.141592653589793238462643383279502884L;
    chirp.assign(2 * size_t(N), 0.0);
    b.assign(2 * size_t(M), 0.0);
    for (int n = 0; n < N; ++n) {
        const long long q = (long long)n * n % (2LL * N);
        const long double ang = -pi * (long double)q / (long double)N;
        chirp[2 * n] = (double)cosl(ang);
        chirp[2 * n + 1] = (double)sinl(ang);
        b[2 * n] = chirp[2 * n];
        b[2 * n + 1] = -chirp[2 * n + 1];
        if (n > 0) {
            b[2 * (M - n)] = b[2 * n];
            b[2 * (M - n) + 1] = b[2 * n + 1];
        }
    }
}

struct Axis {
    int N = 0, M = 0;
    const void* chirp = nullptr;
    const void* filt = nullptr;
    const void* tw = nullptr;
};

template <class T>
static int axis_setup(CallBufs& B, int N, int sms, Axis& ax) {
    ax.N = N;
    ax.M = blue_length(N);
    std::vector<double> chirp, b, tw;
    chirp_tables(N, ax.M, chirp, b);
    twiddle_table(ax.M, tw);
    cx<T>* dc = upload_cx<T>(B, chirp);
    cx<T>* df = upload_cx<T>(B, b);
    cx<T>* dt = upload_cx<T>(B, tw);
    if (!dc || !df || !dt) return fail(CGH_ERR_MEMORY, "transform tables");
    BlueArgs<T> a{};
    a.data = df;
    a.N = ax.M;
    a.lines = 1;
    a.line_stride = ax.M;
    a.elem_stride = 1;
    a.tw = dt;
    a.dir = -1;
    a.scale = T(1);
    a.plain = 1;
    CGH_CUDA(blue_launch<T>(ax.M, a, sms, B.st));
    ax.chirp = dc;
    ax.filt = df;
    ax.tw = dt;
    return CGH_OK;
}

}  // namespace

template <class T>
static int any_transform(const cgh_problem* pb, const double* in, double* out, int op) {
    const int H = pb->height, W = pb->width;
    if (H < 1 || W < 1) return fail(CGH_ERR_DIMENSION, "empty shape %dx%d", H, W);
    const int nmax = max_line_fft<T>() / 2;
    if (H > nmax || W > nmax)
        return fail(CGH_ERR_UNSUPPORTED, "shape %dx%d: non-power-of-two transforms take sides up to %d at this precision",
                    H, W, nmax);
    if (pb->prop_kind == CGH_FRESNEL) {   // as plan_init (propagation.py:49-55)
        if (!(pb->wavelength > 0) || !(pb->pitch_x > 0) || !(pb->pitch_y > 0))
            return fail(CGH_ERR_INVALID_SPEC, "fresnel needs positive wavelength and pitches");
        if (pb->distance == 0) return fail(CGH_ERR_INVALID_SPEC, "fresnel distance must be nonzero");
    } else if (pb->prop_kind != CGH_FOURIER) {
        return fail(CGH_ERR_INVALID_SPEC, "unknown propagation kind %d", pb->prop_kind);
    }
    const bool fres = pb->prop_kind == CGH_FRESNEL && op >= 2;
    const bool fwd = (op == 0 || op == 2);
    CGH_CUDA(cudaSetDevice(pb->device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, pb->device);
    CallBufs B;
    CGH_CUDA(cudaStreamCreateWithFlags(&B.st, cudaStreamNonBlocking));
    const long n = long(H) * W;
    double* stage = static_cast<double*>(B.alloc(size_t(n) * 16));
    cx<T>* data = static_cast<cx<T>*>(B.alloc(size_t(n) * sizeof(cx<T>)));
    unsigned* nf = static_cast<unsigned*>(B.alloc(sizeof(unsigned)));
    if (!stage || !data || !nf) return fail(CGH_ERR_MEMORY, "transform buffers");
    cx<T>* qr = nullptr;
    cx<T>* qc = nullptr;
    if (fres) {
        std::vector<double> r, c;
        chirp_table(H, pb->pitch_y, pb->wavelength, pb->distance, r);
        chirp_table(W, pb->pitch_x, pb->wavelength, pb->distance, c);
        qr = upload_cx<T>(B, r);
        qc = upload_cx<T>(B, c);
        if (!qr || !qc) return fail(CGH_ERR_MEMORY, "Fresnel tables");
    }
    Axis rows, cols;
    CGH_TRY(axis_setup<T>(B, W, sms, rows));
    CGH_TRY(axis_setup<T>(B, H, sms, cols));
    CGH_CUDA(cudaMemcpyAsync(stage, in, size_t(n) * 16, cudaMemcpyHostToDevice, B.st));
    CGH_CUDA(cudaMemsetAsync(nf, 0, sizeof(unsigned), B.st));
    const int grid = grid_for(n);
    load_field_kernel<T><<<grid, 256, 0, B.st>>>(stage, data, H, W, fwd ? 0 : 1, fwd ? qr : nullptr,
                                                 fwd ? qc : nullptr, nf);
    CGH_CUDA(cudaGetLastError());
    unsigned nonfinite = 0;
    CGH_CUDA(cudaMemcpyAsync(&nonfinite, nf, sizeof(unsigned), cudaMemcpyDeviceToHost, B.st));
    CGH_CUDA(cudaStreamSynchronize(B.st));
    if (nonfinite) return fail(CGH_ERR_NONFINITE, "field contains NaN or Inf");
    BlueArgs<T> a{};
    a.data = data;
    a.dir = fwd ? -1 : +1;
    a.plain = 0;
    // rows: H lines of W points
    a.N = W;
    a.lines = H;
    a.line_stride = W;
    a.elem_stride = 1;
    a.chirp = static_cast<const cx<T>*>(rows.chirp);
    a.filt = static_cast<const cx<T>*>(rows.filt);
    a.tw = static_cast<const cx<T>*>(rows.tw);
    a.scale = T(1.0 / double(rows.M));
    CGH_CUDA(blue_launch<T>(rows.M, a, sms, B.st));
    // columns: W lines of H points (stride W), unitary scale folded in
    a.N = H;
    a.lines = W;
    a.line_stride = 1;
    a.elem_stride = W;
    a.chirp = static_cast<const cx<T>*>(cols.chirp);
    a.filt = static_cast<const cx<T>*>(cols.filt);
    a.tw = static_cast<const cx<T>*>(cols.tw);
    a.scale = T(1.0 / (double(cols.M) * std::sqrt(double(H) * double(W))));
    CGH_CUDA(blue_launch<T>(cols.M, a, sms, B.st));
    store_field_kernel<T><<<grid, 256, 0, B.st>>>(data, stage, H, W, fwd ? 1 : 0, fwd ? nullptr : qr,
                                                  fwd ? nullptr : qc);
    CGH_CUDA(cudaGetLastError());
    CGH_CUDA(cudaMemcpyAsync(out, stage, size_t(n) * 16, cudaMemcpyDeviceToHost, B.st));
    CGH_CUDA(cudaStreamSynchronize(B.st));
    return CGH_OK;
}

int transform_any(const cgh_problem* pb, const double* in, double* out, int op) {
    return pb->precision == CGH_FP32 ? any_transform<float>(pb, in, out, op) : any_transform<double>(pb, in, out, op);
}

}  // namespace cgh
