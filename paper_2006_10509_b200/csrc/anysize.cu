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

int blue_length(int n) {
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

// ====================================================== GS passes, any N
// The row/column pass modes of pass_kernels.cuh for a line length N that is
// not a power of two: the line DFTs are Bluestein transforms on M-point line
// FFTs, the per-pixel work (random-phase start, hologram projection and
// snapping, replay projection, error sums) is the same code as the
// power-of-two passes. Element j of the line sits at v[r], j = t + r * TF
// (TF = M / E threads), entries j >= N are zero.

template <class T, int M, int E>
__device__ __forceinline__ void blue_dft(cx<T> (&v)[E], int dir, int N, T* sre, T* sim, int t, const cx<T>* tab) {
    constexpr int TF = M / E;
    const cx<T>* chirp = tab;
    const cx<T>* filt = tab + N;
    const cx<T>* twm = tab + N + M;
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int j = t + r * TF;
        v[r] = j < N ? (dir < 0 ? cmul(v[r], chirp[j]) : cmulc(v[r], chirp[j])) : mk<T>(0, 0);
    }
    LineFft<T, M, -1, E>::run(v, sre, sim, t, twm);
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = dir < 0 ? cmul(v[r], filt[t + r * TF]) : cmulc(v[r], filt[t + r * TF]);
    LineFft<T, M, +1, E>::run(v, sre, sim, t, twm);
    const T inv = T(1) / T(M);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int j = t + r * TF;
        v[r] = j < N ? (dir < 0 ? cmul(v[r], chirp[j]) : cmulc(v[r], chirp[j])) * inv : mk<T>(0, 0);
    }
}

template <class T, int M>
struct AnyShape {
    static constexpr int E = LineShape<T, M>::E;
    static constexpr int TF = M / E;
    static constexpr size_t FFT_BYTES = size_t(2) * line_words<T, M>() * sizeof(T);
    static constexpr size_t SMEM = ((FFT_BYTES + 15) & ~size_t(15)) + kRedWords * sizeof(double);
};

template <class T, int M, int MODE>
__global__ void __launch_bounds__(AnyShape<T, M>::TF) any_row_kernel(PassArgs<T> a) {
    using Sh = AnyShape<T, M>;
    constexpr int E = Sh::E, TF = Sh::TF;
    extern __shared__ __align__(16) unsigned char smem[];
    T* sre = reinterpret_cast<T*>(smem);
    T* sim = sre + line_words<T, M>();
    const int t = threadIdx.x, m = blockIdx.x, N = a.W;
    cx<T>* row = a.data + long(blockIdx.y) * a.frame_stride + long(m) * N;
    cx<T> v[E];
    if constexpr (MODE == ROW_INIT) {
        // contiguous chunks of the row-major draws per thread, staged in smem
        const int ch = (N + TF - 1) / TF, j0 = t * ch, j1 = min(N, j0 + ch);
        if (j0 < j1) {
            Pcg64 g = a.rng;
            pcg_advance(g, uint64_t(long(m) * N + j0));
            for (int j = j0; j < j1; ++j) {
                const cx<T> z = unit_phase<T>(g);
                const T amp = a.beam ? a.beam[long(m) * N + j] : T(1);
                const cx<T> h = beam_zero_signs(amp, mk(amp * z.x, amp * z.y));
                sre[padx<T>(j)] = h.x;
                sim[padx<T>(j)] = h.y;
            }
        }
        __syncthreads();
        const bool fres = a.q_row != nullptr;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int n = t + r * TF;
            if (n < N) {
                cx<T> h = mk(sre[padx<T>(n)], sim[padx<T>(n)]);
                if (a.field_out) a.field_out[long(m) * N + n] = h;
                if (a.quantize) {
                    const int k = quantize_index<T>(a.scheme, h);
                    if (a.idx_out) {
                        const long p = long(m) * N + n;
                        if (a.idx_bytes == 1) static_cast<uint8_t*>(a.idx_out)[p] = (uint8_t)k;
                        else static_cast<int32_t*>(a.idx_out)[p] = k;
                    }
                    h = state_value<T>(a.scheme, k);
                }
                if (fres) h = cmul(h, cmul(a.q_row[m], a.q_col[n]));
                v[r] = h;
            } else {
                v[r] = mk<T>(0, 0);
            }
        }
        blue_dft<T, M, E>(v, -1, N, sre, sim, t, a.tw_row);
    } else if constexpr (MODE == ROW_OSPR_GEN) {
        // OSPR K1 (algorithms.py:494-499): frame blockIdx.y's random-phase
        // sub-target |T| exp(i 2 pi u), u drawn row-major over the CENTRED
        // plane, ifftshifted into uncentred row m (centred row (m + H/2) % H,
        // centred column c lands on uncentred column (c + N - N/2) % N; odd
        // sides included), then the inverse row DFT.
        const int uc = (m + a.H / 2) % a.H;
        const int ch = (N + TF - 1) / TF, j0 = t * ch, j1 = min(N, j0 + ch);
        if (j0 < j1) {
            Pcg64 g = a.frame_rng[a.frame0 + blockIdx.y];
            pcg_advance(g, uint64_t(long(uc) * N + j0));
            int k = (j0 + N - N / 2) % N;
            for (int j = j0; j < j1; ++j) {
                const cx<T> z = unit_phase<T>(g);
                const T amp = fabs(a.tgt[long(m) * N + k]);
                sre[padx<T>(k)] = amp * z.x;
                sim[padx<T>(k)] = amp * z.y;
                k = k + 1 == N ? 0 : k + 1;
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int n = t + r * TF;
            v[r] = n < N ? mk(sre[padx<T>(n)], sim[padx<T>(n)]) : mk<T>(0, 0);
        }
        blue_dft<T, M, E>(v, +1, N, sre, sim, t, a.tw_row);
    } else if constexpr (MODE == ROW_OSPR_ACC) {
        // OSPR K3 (algorithms.py:502-512): row m of every frame in
        // [frame0, frame0 + frames): forward row DFT, |R|^2 accumulated,
        // per-frame masked error sums of sqrt(I / i); the frame after the
        // last adds the efficiency sums. Same per-pixel code and fixed-order
        // reduction as row_kernel's ROW_OSPR_ACC, one CTA per row.
        __shared__ double blk[3 * 64 + 2];
        double* rs = red_scratch<T>(smem, Sh::FFT_BYTES);
        const long pix0 = long(m) * N;
        T inten[E], tv[E];
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int n = t + r * TF;
            inten[r] = (n < N && a.load_intensity) ? a.intensity[pix0 + n] : T(0);
            tv[r] = n < N ? a.tgt[pix0 + n] : T(-0.0);
        }
        for (int f = 0; f < a.frames; ++f) {
            const cx<T>* fr = a.data + long(f) * a.frame_stride + pix0;
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = t + r * TF < N ? fr[t + r * TF] : mk<T>(0, 0);
            blue_dft<T, M, E>(v, -1, N, sre, sim, t, a.tw_row);
            const T inv_n = T(1) / T(a.frame0 + f + 1);
            T sdd = 0, spp = 0, spd = 0;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if (t + r * TF >= N) continue;
                const cx<T> R = v[r] * a.scale;
                inten[r] += R.x * R.x + R.y * R.y;
                if (!signbit(tv[r])) {
                    const T p = dev_sqrt<T>(inten[r] * inv_n);
                    const T d = p - tv[r];
                    sdd += d * d;
                    spp += p * p;
                    spd += p * d;
                }
            }
            double acc[3] = {double(sdd), double(spp), double(spd)};
            block_reduce<3>(acc, rs);
            if (t == 0) {
                blk[3 * f + 0] = acc[0];
                blk[3 * f + 1] = acc[1];
                blk[3 * f + 2] = acc[2];
            }
        }
        const bool tail = (a.frame0 + a.frames == a.nframes_total);
        int nq = 3 * a.frames;
        if (tail) {
            const T inv_n = T(1) / T(a.nframes_total);
            T sin_ = 0, sall = 0;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                if (t + r * TF >= N) continue;
                const T p = dev_sqrt<T>(inten[r] * inv_n);
                const T pp = p * p;
                sall += pp;
                if (!signbit(tv[r])) sin_ += pp;
            }
            double acc[2] = {double(sin_), double(sall)};
            block_reduce<2>(acc, rs);
            if (t == 0) {
                blk[nq + 0] = acc[0];
                blk[nq + 1] = acc[1];
            }
            nq += 2;
        }
        if (a.store_intensity) {
#pragma unroll
            for (int r = 0; r < E; ++r)
                if (t + r * TF < N) a.intensity[pix0 + t + r * TF] = inten[r];
        }
        const int nblocks = gridDim.x;
        __shared__ int last;
        __syncthreads();
        if (t == 0) {
            for (int q = 0; q < nq; ++q) a.red.partials[long(q) * nblocks + blockIdx.x] = blk[q];
            __threadfence();
            last = (atomicAdd(a.red.counter, 1u) == unsigned(nblocks - 1));
        }
        __syncthreads();
        if (last) {
            __threadfence();
            const double denom = *a.red.denom;
            for (int f = 0; f < a.frames; ++f) {
                const double sdd = sum_partials(a.red, 3 * f + 0, nblocks, rs);
                const double spp = sum_partials(a.red, 3 * f + 1, nblocks, rs);
                const double spd = sum_partials(a.red, 3 * f + 2, nblocks, rs);
                if (t == 0) a.red.out[a.frame0 + f] = error_from_sums(sdd, spp, spd, denom, a.red.rescale);
            }
            if (tail) {
                const double sin_ = sum_partials(a.red, 3 * a.frames + 0, nblocks, rs);
                const double sall = sum_partials(a.red, 3 * a.frames + 1, nblocks, rs);
                if (t == 0)
                    a.red.out[a.nframes_total] = sall == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : sin_ / sall;
            }
            if (t == 0) *a.red.counter = 0u;
        }
        return;
    } else {   // ROW_FWD, ROW_INV, ROW_HOLO
#pragma unroll
        for (int r = 0; r < E; ++r) v[r] = t + r * TF < N ? row[t + r * TF] : mk<T>(0, 0);
        blue_dft<T, M, E>(v, MODE == ROW_FWD ? -1 : +1, N, sre, sim, t, a.tw_row);
        if constexpr (MODE == ROW_HOLO) {
#pragma unroll
            for (int r = 0; r < E; ++r)
                if (t + r * TF < N) v[r] = holo_project<T>(a, v[r], m, t + r * TF, 0);
            blue_dft<T, M, E>(v, -1, N, sre, sim, t, a.tw_row);
        } else if (a.scale != T(1)) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
        }
    }
#pragma unroll
    for (int r = 0; r < E; ++r)
        if (t + r * TF < N) row[t + r * TF] = v[r];
}

template <class T, int M, int MODE>
__global__ void __launch_bounds__(AnyShape<T, M>::TF) any_col_kernel(PassArgs<T> a) {
    using Sh = AnyShape<T, M>;
    constexpr int E = Sh::E, TF = Sh::TF;
    extern __shared__ __align__(16) unsigned char smem[];
    T* sre = reinterpret_cast<T*>(smem);
    T* sim = sre + line_words<T, M>();
    double* rs = red_scratch<T>(smem, Sh::FFT_BYTES);
    const int t = threadIdx.x, n = blockIdx.x, N = a.H;
    const long W = a.W;
    cx<T>* col = a.data + long(blockIdx.y) * a.frame_stride + n;
    cx<T> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) v[r] = t + r * TF < N ? col[long(t + r * TF) * W] : mk<T>(0, 0);
    if constexpr (MODE == COL_FWD || MODE == COL_INV) {
        blue_dft<T, M, E>(v, MODE == COL_FWD ? -1 : +1, N, sre, sim, t, a.tw_col);
        if (a.scale != T(1)) {
#pragma unroll
            for (int r = 0; r < E; ++r) v[r] = v[r] * a.scale;
        }
    } else if constexpr (MODE == COL_HOLO) {
        // OSPR K2: inverse column DFT -> hologram projection (+ index plane of
        // frame blockIdx.y) -> forward column DFT
        const long foff = long(blockIdx.y) * a.frame_stride;
        blue_dft<T, M, E>(v, +1, N, sre, sim, t, a.tw_col);
#pragma unroll
        for (int r = 0; r < E; ++r)
            if (t + r * TF < N) v[r] = holo_project<T>(a, v[r], t + r * TF, n, foff);
        blue_dft<T, M, E>(v, -1, N, sre, sim, t, a.tw_col);
    } else {   // COL_GS, COL_FINAL (col_kernel's epilogue)
        blue_dft<T, M, E>(v, -1, N, sre, sim, t, a.tw_col);
        T sdd = 0, srr = 0, srd = 0, sall = 0;
        const T gain = a.gain;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int u = t + r * TF;
            if (u >= N) continue;
            const cx<T> R = v[r] * a.scale;
            const T r2 = R.x * R.x + R.y * R.y;
            const T rr = dev_sqrt<T>(r2);
            const T tt = a.tgt[long(u) * W + n];
            sall += r2;
            cx<T> out = R;
            if (!signbit(tt)) {
                const T d = rr - tt;
                sdd += d * d;
                srr += r2;
                srd += rr * d;
                if constexpr (MODE == COL_GS) {
                    T want = tt + gain * (tt - rr);
                    want = want > T(0) ? want : T(0);
                    if (rr > T(0)) {
                        const T s = want / rr;
                        out = mk(R.x * s, R.y * s);
                    } else {
                        out = mk(want, T(0));
                    }
                }
            }
            v[r] = out;
        }
        if constexpr (MODE == COL_GS) blue_dft<T, M, E>(v, +1, N, sre, sim, t, a.tw_col);
        double acc[4] = {double(sdd), double(srr), double(srd), double(sall)};
        block_reduce<4>(acc, rs);
        const int nblocks = gridDim.x;
        if (publish_partials<4>(a.red, acc, nblocks, blockIdx.x)) {
            const double s_dd = sum_partials(a.red, 0, nblocks, rs);
            const double s_rr = sum_partials(a.red, 1, nblocks, rs);
            const double s_rd = sum_partials(a.red, 2, nblocks, rs);
            const double s_all = sum_partials(a.red, 3, nblocks, rs);
            if (threadIdx.x == 0) {
                a.red.out[0] = error_from_sums(s_dd, s_rr, s_rd, *a.red.denom, a.red.rescale);
                a.red.out[1] = s_all == 0.0 ? __longlong_as_double(0x7ff8000000000000LL) : s_rr / s_all;
                *a.red.counter = 0u;
            }
        }
        if constexpr (MODE == COL_FINAL) return;
    }
#pragma unroll
    for (int r = 0; r < E; ++r)
        if (t + r * TF < N) col[long(t + r * TF) * W] = v[r];
}

template <class T, int M, class K>
static cudaError_t any_launch(K kernel, int lines, int frames, cudaStream_t st, const PassArgs<T>& a) {
    using Sh = AnyShape<T, M>;
    if (Sh::SMEM > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Sh::SMEM));
        if (e != cudaSuccess) return e;
    }
    kernel<<<dim3(lines, frames), Sh::TF, Sh::SMEM, st>>>(a);
    return cudaGetLastError();
}

template <class T, int M>
static cudaError_t any_row_m(int mode, const PassArgs<T>& a, int frames, cudaStream_t st) {
    switch (mode) {
        case ROW_FWD: return any_launch<T, M>(any_row_kernel<T, M, ROW_FWD>, a.H, frames, st, a);
        case ROW_INV: return any_launch<T, M>(any_row_kernel<T, M, ROW_INV>, a.H, frames, st, a);
        case ROW_HOLO: return any_launch<T, M>(any_row_kernel<T, M, ROW_HOLO>, a.H, frames, st, a);
        case ROW_INIT: return any_launch<T, M>(any_row_kernel<T, M, ROW_INIT>, a.H, frames, st, a);
        case ROW_OSPR_GEN: return any_launch<T, M>(any_row_kernel<T, M, ROW_OSPR_GEN>, a.H, frames, st, a);
        case ROW_OSPR_ACC: return any_launch<T, M>(any_row_kernel<T, M, ROW_OSPR_ACC>, a.H, 1, st, a);
        default: return cudaErrorNotSupported;
    }
}

template <class T, int M>
static cudaError_t any_col_m(int mode, const PassArgs<T>& a, int frames, cudaStream_t st) {
    switch (mode) {
        case COL_FWD: return any_launch<T, M>(any_col_kernel<T, M, COL_FWD>, a.W, frames, st, a);
        case COL_INV: return any_launch<T, M>(any_col_kernel<T, M, COL_INV>, a.W, frames, st, a);
        case COL_GS: return any_launch<T, M>(any_col_kernel<T, M, COL_GS>, a.W, frames, st, a);
        case COL_FINAL: return any_launch<T, M>(any_col_kernel<T, M, COL_FINAL>, a.W, frames, st, a);
        case COL_HOLO: return any_launch<T, M>(any_col_kernel<T, M, COL_HOLO>, a.W, frames, st, a);
        default: return cudaErrorNotSupported;
    }
}

#define CGH_ANY_SIZES(X) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

template <class T>
cudaError_t launch_row_any(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st) {
    if (N < 1 || N > kMaxAnyLine) return cudaErrorInvalidValue;
#define CGH_ANY_ROW(MM) case MM: return any_row_m<T, MM>(mode, a, frames, st);
    switch (blue_length(N)) {
        CGH_ANY_SIZES(CGH_ANY_ROW)
        default: return cudaErrorInvalidValue;
    }
#undef CGH_ANY_ROW
}

template <class T>
cudaError_t launch_col_any(int mode, int N, const PassArgs<T>& a, int frames, cudaStream_t st) {
    if (N < 1 || N > kMaxAnyLine) return cudaErrorInvalidValue;
#define CGH_ANY_COL(MM) case MM: return any_col_m<T, MM>(mode, a, frames, st);
    switch (blue_length(N)) {
        CGH_ANY_SIZES(CGH_ANY_COL)
        default: return cudaErrorInvalidValue;
    }
#undef CGH_ANY_COL
}

template cudaError_t launch_row_any<float>(int, int, const PassArgs<float>&, int, cudaStream_t);
template cudaError_t launch_row_any<double>(int, int, const PassArgs<double>&, int, cudaStream_t);
template cudaError_t launch_col_any<float>(int, int, const PassArgs<float>&, int, cudaStream_t);
template cudaError_t launch_col_any<double>(int, int, const PassArgs<double>&, int, cudaStream_t);

// Packed Bluestein table of a plan axis of length N (host part): chirp [N],
// convolution kernel b [M] (its spectrum is taken on the device by
// blue_finish_table), twiddles exp(-2 pi i k / M) [M].
void blue_pack_table(int N, std::vector<double>& out) {
    const int M = blue_length(N);
    std::vector<double> chirp, b, tw;
    chirp_tables(N, M, chirp, b);
    twiddle_table(M, tw);
    out.clear();
    out.insert(out.end(), chirp.begin(), chirp.end());
    out.insert(out.end(), b.begin(), b.end());
    out.insert(out.end(), tw.begin(), tw.end());
}

int blue_finish_table(int prec, int N, void* dev_table, cudaStream_t st) {
    const int M = blue_length(N);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e;
    if (prec == CGH_FP64) {
        cx<double>* t = static_cast<cx<double>*>(dev_table);
        BlueArgs<double> a{};
        a.data = t + N;
        a.N = M;
        a.lines = 1;
        a.line_stride = M;
        a.elem_stride = 1;
        a.tw = t + N + M;
        a.dir = -1;
        a.scale = 1.0;
        a.plain = 1;
        e = blue_launch<double>(M, a, sms, st);
    } else {
        cx<float>* t = static_cast<cx<float>*>(dev_table);
        BlueArgs<float> a{};
        a.data = t + N;
        a.N = M;
        a.lines = 1;
        a.line_stride = M;
        a.elem_stride = 1;
        a.tw = t + N + M;
        a.dir = -1;
        a.scale = 1.0f;
        a.plain = 1;
        e = blue_launch<float>(M, a, sms, st);
    }
    if (e != cudaSuccess) return fail(CGH_ERR_CUDA, "Bluestein table (N=%d): %s", N, cudaGetErrorString(e));
    return CGH_OK;
}

int transform_any(const cgh_problem* pb, const double* in, double* out, int op) {
    return pb->precision == CGH_FP32 ? any_transform<float>(pb, in, out, op) : any_transform<double>(pb, in, out, op);
}

}  // namespace cgh
