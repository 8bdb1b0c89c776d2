// Complex arithmetic and compile-time roots of unity for the FFT passes.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace cgh {

template <class T>
struct alignas(2 * sizeof(T)) cx {
    T x, y;
};

template <class T>
__host__ __device__ __forceinline__ cx<T> mk(T a, T b) {
    cx<T> r;
    r.x = a;
    r.y = b;
    return r;
}
template <class T>
__device__ __forceinline__ cx<T> operator+(cx<T> a, cx<T> b) { return mk(a.x + b.x, a.y + b.y); }
template <class T>
__device__ __forceinline__ cx<T> operator-(cx<T> a, cx<T> b) { return mk(a.x - b.x, a.y - b.y); }
template <class T>
__device__ __forceinline__ cx<T> operator*(cx<T> a, T s) { return mk(a.x * s, a.y * s); }
template <class T>
__device__ __forceinline__ cx<T> cmul(cx<T> a, cx<T> b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <class T>
__device__ __forceinline__ cx<T> cmulc(cx<T> a, cx<T> b) {
    return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <class T>
__device__ __forceinline__ cx<T> conj(cx<T> a) { return mk(a.x, -a.y); }

// ---- complex64 in packed f32x2 instructions (sm_100a FADD2 / FMUL2 /
// FFMA2): the value's two halves are one 64-bit register pair; a complex add
// is one instruction instead of two and a complex product two instead of
// four (see pcx.cuh). Same IEEE roundings per component as the scalar forms.
// Non-template overloads: preferred to the templates above for cx<float>.
namespace f2 {
__device__ __forceinline__ unsigned long long pack(cx<float> a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ cx<float> unpack(unsigned long long r) {
    cx<float> a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ unsigned long long mul(unsigned long long a, unsigned long long b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ unsigned long long fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
}  // namespace f2

__device__ __forceinline__ cx<float> operator+(cx<float> a, cx<float> b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2::pack(a)), "l"(f2::pack(b)));
    return f2::unpack(r);
}
__device__ __forceinline__ cx<float> operator-(cx<float> a, cx<float> b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2::pack(a)), "l"(f2::pack(b)));
    return f2::unpack(r);
}
__device__ __forceinline__ cx<float> operator*(cx<float> a, float s) {
    return f2::unpack(f2::mul(f2::pack(a), f2::pack(mk(s, s))));
}
// a * b = b.x * a + b.y * (-a.y, a.x)
__device__ __forceinline__ cx<float> cmul(cx<float> a, cx<float> b) {
    return f2::unpack(f2::fma(f2::pack(mk(a.y, a.x)), f2::pack(mk(-b.y, b.y)), f2::mul(f2::pack(a), f2::pack(mk(b.x, b.x)))));
}
// a * conj(b) = b.x * a + b.y * (a.y, -a.x)
__device__ __forceinline__ cx<float> cmulc(cx<float> a, cx<float> b) {
    return f2::unpack(f2::fma(f2::pack(mk(a.y, a.x)), f2::pack(mk(b.y, -b.y)), f2::mul(f2::pack(a), f2::pack(mk(b.x, b.x)))));
}

// Read-only cached load of a complex value.
__device__ __forceinline__ cx<float> ldg_cx(const cx<float>* p) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(p));
    return mk(v.x, v.y);
}
__device__ __forceinline__ cx<double> ldg_cx(const cx<double>* p) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(p));
    return mk(v.x, v.y);
}

// Multiply by DIR*i (DIR = -1 forward transform, +1 inverse).
template <int DIR, class T>
__device__ __forceinline__ cx<T> rot90(cx<T> a) {
    if constexpr (DIR < 0) return mk(a.y, -a.x);
    else return mk(-a.y, a.x);
}

// ---- compile-time cos/sin of 2*pi*m/R (octant reduced Taylor, ~1 ulp) -------
namespace detail {
constexpr double kPi = 3.14159265358979323846264338327950288;
__host__ __device__ constexpr double taylor_sin(double x) {
    double x2 = x * x, term = x, sum = x;
    for (int k = 1; k < 14; ++k) {
        term *= -x2 / ((2.0 * k) * (2.0 * k + 1.0));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double taylor_cos(double x) {
    double x2 = x * x, term = 1.0, sum = 1.0;
    for (int k = 1; k < 14; ++k) {
        term *= -x2 / ((2.0 * k - 1.0) * (2.0 * k));
        sum += term;
    }
    return sum;
}
// cos/sin(2 pi m / R) for integer m (any sign), exact at multiples of pi/2.
__host__ __device__ constexpr void root(long m, long R, double& c, double& s) {
    m %= R;
    if (m < 0) m += R;
    // angle = 2*pi*m/R ; reduce by octants: 8*m/R
    long q8 = (8 * m) / R;           // octant 0..7
    long rem_num = 8 * m - q8 * R;   // remainder numerator over (8R): angle = (q8 + rem_num/R) * pi/4
    double frac = double(rem_num) / double(R);   // in [0,1)
    double base_c = 0, base_s = 0;
    // angle within octant: a = frac * pi/4 ; total = q8*pi/4 + a
    double a = frac * (kPi / 4.0);
    double ca = taylor_cos(a), sa = taylor_sin(a);
    // rotate by q8 * pi/4
    const double h = 0.70710678118654752440084436210484903928;
    double rc[8] = {1, h, 0, -h, -1, -h, 0, h};
    double rs[8] = {0, h, 1, h, 0, -h, -1, -h};
    base_c = rc[q8];
    base_s = rs[q8];
    if (rem_num == 0) {
        c = base_c;
        s = base_s;
    } else if ((q8 & 1) == 0) {
        // even octant: base is axis-aligned, exact rotation
        c = base_c * ca - base_s * sa;
        s = base_s * ca + base_c * sa;
    } else {
        // odd octant: use the complementary angle from the next axis for accuracy
        double b = (1.0 - frac) * (kPi / 4.0);
        double cb = taylor_cos(b), sb = taylor_sin(b);
        long q = (q8 + 1) & 7;
        // angle = q*pi/4 - b
        c = rc[q] * cb + rs[q] * sb;
        s = rs[q] * cb - rc[q] * sb;
    }
}
__host__ __device__ constexpr double rcos(long m, long R) {
    double c = 0, s = 0;
    root(m, R, c, s);
    return c;
}
__host__ __device__ constexpr double rsin(long m, long R) {
    double c = 0, s = 0;
    root(m, R, c, s);
    return s;
}
}  // namespace detail

// W = exp(DIR * 2*pi*i * M / R) as compile-time constants.
template <class T, int DIR, long M, long R>
__device__ __forceinline__ cx<T> twc() {
    constexpr double c = detail::rcos(M, R);
    constexpr double s = detail::rsin(M, R);
    return mk<T>(T(c), T(DIR * s));
}

template <class T, int DIR, long M, long R>
__device__ __forceinline__ cx<T> mul_root(cx<T> a) {
    constexpr long m = ((M % R) + R) % R;
    if constexpr (m == 0) {
        return a;
    } else if constexpr (4 * m == R) {
        return rot90<DIR>(a);
    } else if constexpr (2 * m == R) {
        return mk(-a.x, -a.y);
    } else if constexpr (4 * m == 3 * R) {
        return rot90<-DIR>(a);
    } else if constexpr (std::is_same<T, float>::value) {
        // compile-time root c + i s: c * a + s * (-a.y, a.x), the constants as
        // immediate / uniform operands of one FMUL2 and one FFMA2
        constexpr float c = float(detail::rcos(m, R));
        constexpr float s = float(DIR * detail::rsin(m, R));
        return f2::unpack(f2::fma(f2::pack(mk(a.y, a.x)), f2::pack(mk(-s, s)), f2::mul(f2::pack(a), f2::pack(mk(c, c)))));
    } else {
        return cmul(a, twc<T, DIR, m, R>());
    }
}

}  // namespace cgh
