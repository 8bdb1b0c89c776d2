// Packed complex64 arithmetic for the warp-line passes (sm_100a f32x2).
//
// A complex value lives in one 64-bit register pair (real part in the low
// half) and every complex add / subtract is ONE packed instruction (FADD2)
// instead of two scalar ones. The SM issues one warp instruction per clock
// per sub-partition; a packed instruction occupies the FMA pipe for two
// clocks but only one issue slot, so an issue-bound FFT gets the second slot
// back for its shared-memory and address instructions
// (scripts/micro/f32x2_mix.cu: 16 FADD + 8 ALU = 27 clocks per iteration,
// 8 FADD2 + 8 ALU = 16.5). The products keep the scalar code's roundings:
// each component is one IEEE multiply, add or fused multiply-add.
//
// Swaps (re <-> im), broadcasts of one half, and sign flips by constant
// (+-1, -+1) pairs are operand modifiers of FADD2/FMUL2/FFMA2 (.LO_HI,
// .F32, .NP, -R): ptxas folds make(im(a), re(a)), make(s, s) and products
// with such constants into the consuming instruction.
#pragma once
#include "cx.cuh"

namespace cgh {
namespace pk {

typedef unsigned long long pc;

__device__ __forceinline__ pc make(float x, float y) {
    pc r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
    return r;
}
__device__ __forceinline__ float re(pc a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
    return x;
}
__device__ __forceinline__ float im(pc a) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a));
    return y;
}
__device__ __forceinline__ pc add(pc a, pc b) {
    pc r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ pc sub(pc a, pc b) {
    pc r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ pc mul(pc a, pc b) {
    pc r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// a * b + c per half, one rounding
__device__ __forceinline__ pc fma(pc a, pc b, pc c) {
    pc r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ pc bc(float s) { return make(s, s); }
__device__ __forceinline__ pc swap(pc a) { return make(im(a), re(a)); }
__device__ __forceinline__ pc neg(pc a) { return make(-re(a), -im(a)); }

__device__ __forceinline__ pc from(cx<float> a) { return make(a.x, a.y); }
__device__ __forceinline__ cx<float> to(pc a) { return mk(re(a), im(a)); }

// DIR * i * a as a constant-signed swap: DIR < 0: (a.y, -a.x); DIR > 0: (-a.y, a.x)
template <int DIR>
__device__ __forceinline__ pc rot_sign() {
    return DIR < 0 ? make(1.0f, -1.0f) : make(-1.0f, 1.0f);
}
// b + DIR * i * d and b - DIR * i * d (one FFMA2 each)
template <int DIR>
__device__ __forceinline__ pc add_rot(pc b, pc d) { return fma(swap(d), rot_sign<DIR>(), b); }
template <int DIR>
__device__ __forceinline__ pc sub_rot(pc b, pc d) { return fma(swap(d), rot_sign<-DIR>(), b); }
template <int DIR>
__device__ __forceinline__ pc rot90(pc a) { return mul(swap(a), rot_sign<DIR>()); }

// a * exp(DIR * 2 pi i M / R), compile-time root: c * a + s * (-a.y, a.x)
template <int DIR, long M, long R>
__device__ __forceinline__ pc mul_root(pc a) {
    constexpr long m = ((M % R) + R) % R;
    if constexpr (m == 0) {
        return a;
    } else if constexpr (4 * m == R) {
        return rot90<DIR>(a);
    } else if constexpr (2 * m == R) {
        return neg(a);
    } else if constexpr (4 * m == 3 * R) {
        return rot90<-DIR>(a);
    } else {
        constexpr float c = float(detail::rcos(m, R));
        constexpr float s = float(DIR * detail::rsin(m, R));
        return fma(swap(a), make(-s, s), mul(a, bc(c)));
    }
}

// a * w and a * conj(w) for a run-time twiddle w = (wx, wy) given as the
// broadcast wx and the pair wn = (-wy, wy)
__device__ __forceinline__ pc wn_of(pc w) { return mul(bc(im(w)), make(-1.0f, 1.0f)); }
__device__ __forceinline__ pc cmul_n(pc a, float wx, pc wn) { return fma(swap(a), wn, mul(a, bc(wx))); }
__device__ __forceinline__ pc cmulc_n(pc a, float wx, pc wn) { return fma(neg(swap(a)), wn, mul(a, bc(wx))); }
// a * w (D < 0) or a * conj(w) (D > 0)
template <int D>
__device__ __forceinline__ pc cmul_d(pc a, float wx, pc wn) {
    if constexpr (D < 0) return cmul_n(a, wx, wn);
    else return cmulc_n(a, wx, wn);
}
template <int D>
__device__ __forceinline__ pc cmul_d(pc a, pc w) {
    return cmul_d<D>(a, re(w), wn_of(w));
}

// ---- in-place DFTs of R points v[0], v[S], ..., natural order out (as
// fft_block.cuh's Dft, same factorisations)
template <int R, int DIR, int S>
struct Dft;

template <int DIR, int S>
struct Dft<2, DIR, S> {
    __device__ __forceinline__ static void run(pc* v) {
        const pc a = v[0], b = v[S];
        v[0] = add(a, b);
        v[S] = sub(a, b);
    }
};

template <int DIR, int S>
struct Dft<4, DIR, S> {
    __device__ __forceinline__ static void run(pc* v) {
        const pc a = add(v[0], v[2 * S]), b = sub(v[0], v[2 * S]);
        const pc c = add(v[S], v[3 * S]), d = sub(v[S], v[3 * S]);
        v[0] = add(a, c);
        v[2 * S] = sub(a, c);
        v[S] = add_rot<DIR>(b, d);
        v[3 * S] = sub_rot<DIR>(b, d);
    }
};

template <int R1, int R2, int DIR, int S>
struct DftSplit {
    template <int N2>
    __device__ __forceinline__ static void inner(pc* v) {
        if constexpr (N2 < R2) {
            Dft<R1, DIR, S * R2>::run(v + S * N2);
            twiddle<N2, 1>(v);
            inner<N2 + 1>(v);
        }
    }
    template <int N2, int K1>
    __device__ __forceinline__ static void twiddle(pc* v) {
        if constexpr (K1 < R1) {
            v[S * (N2 + R2 * K1)] = mul_root<DIR, long(N2) * K1, long(R1) * R2>(v[S * (N2 + R2 * K1)]);
            twiddle<N2, K1 + 1>(v);
        }
    }
    template <int K1>
    __device__ __forceinline__ static void outer(pc* v) {
        if constexpr (K1 < R1) {
            Dft<R2, DIR, S>::run(v + S * R2 * K1);
            outer<K1 + 1>(v);
        }
    }
    __device__ __forceinline__ static void run(pc* v) {
        inner<0>(v);
        outer<0>(v);
        pc tmp[R1 * R2];
#pragma unroll
        for (int i = 0; i < R1 * R2; ++i) tmp[i] = v[S * i];
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1)
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) v[S * (k1 + R1 * k2)] = tmp[R2 * k1 + k2];
    }
};

template <int DIR, int S>
struct Dft<8, DIR, S> {
    __device__ __forceinline__ static void run(pc* v) { DftSplit<2, 4, DIR, S>::run(v); }
};
template <int DIR, int S>
struct Dft<16, DIR, S> {
    __device__ __forceinline__ static void run(pc* v) { DftSplit<4, 4, DIR, S>::run(v); }
};

}  // namespace pk
}  // namespace cgh
