// Device/host emulation of numpy's PCG64 bit generator and the Generator
// methods the hot path draws from (semantics in oracle/pcg64_model.py,
// checked against numpy by tests/test_rng_model.py and, on the GPU, by
// tests/test_gpu_rng.py):
//   step:    s <- s * MULT + inc  (mod 2^128)
//   next64:  rotr64(hi ^ lo, hi >> 58) of the NEW state
//   double:  (next64 >> 11) * 2^-53                         (Generator.random)
//   next32:  low half of a fresh next64, high half buffered (has_uint32)
//   bounded: Lemire 32-bit rejection                        (Generator.integers)
//   advance: log-time jump of the affine LCG map
#pragma once
#include <cstdint>

namespace cgh {

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state;
    u128 inc;
    int has_uint32;
    uint32_t uinteger;
};

__host__ __device__ __forceinline__ u128 pcg_mult() {
    return (u128(0x2360ED051FC65DA4ULL) << 64) | u128(0x4385DF649FCCF645ULL);
}

__host__ __device__ __forceinline__ uint64_t pcg_next64(Pcg64& g) {
    g.state = g.state * pcg_mult() + g.inc;
    const uint64_t hi = uint64_t(g.state >> 64), lo = uint64_t(g.state);
    const uint64_t x = hi ^ lo;
    const unsigned rot = unsigned(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ __forceinline__ double pcg_next_double(Pcg64& g) {
    return double(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// float(x) for x = 2u, shifted to [-1, 1) (x - 2 when x > 1), u = next_double:
// the same value as float((2.0 * u > 1.0) ? 2.0 * u - 2.0 : 2.0 * u) computed in
// fp64 (u = x53 * 2^-53 exactly, the shift is exact, and rounding commutes with
// the power-of-two scale), without fp64 arithmetic.
__host__ __device__ __forceinline__ float pcg_next_halfturns(Pcg64& g) {
    const long long x53 = (long long)(pcg_next64(g) >> 11);
    const long long xi = x53 > (1LL << 52) ? x53 - (1LL << 53) : x53;
    return float(xi) * 2.220446049250313e-16f;   // 2^-52
}

__host__ __device__ __forceinline__ uint32_t pcg_next32(Pcg64& g) {
    if (g.has_uint32) {
        g.has_uint32 = 0;
        return g.uinteger;
    }
    const uint64_t v = pcg_next64(g);
    g.has_uint32 = 1;
    g.uinteger = uint32_t(v >> 32);
    return uint32_t(v & 0xFFFFFFFFULL);
}

// Generator.integers(high) for 1 <= high <= 2^32 (numpy: buffered Lemire).
__host__ __device__ __forceinline__ uint32_t pcg_integers(Pcg64& g, uint64_t high) {
    const uint64_t rng = high - 1;
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFULL) return pcg_next32(g);
    const uint32_t excl = uint32_t(rng + 1);
    uint64_t m = uint64_t(pcg_next32(g)) * excl;
    uint32_t left = uint32_t(m);
    if (left < excl) {
        const uint32_t thresh = uint32_t((0xFFFFFFFFULL - rng) % excl);
        while (left < thresh) {
            m = uint64_t(pcg_next32(g)) * excl;
            left = uint32_t(m);
        }
    }
    return uint32_t(m >> 32);
}

// numpy random_interval(max): masked rejection sampling.
__host__ __device__ __forceinline__ uint64_t pcg_interval(Pcg64& g, uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (mx <= 0xFFFFFFFFULL) {
        while ((v = (pcg_next32(g) & mask)) > mx) {
        }
    } else {
        while ((v = (pcg_next64(g) & mask)) > mx) {
        }
    }
    return v;
}

// Jump ahead by delta steps.
__host__ __device__ __forceinline__ void pcg_advance(Pcg64& g, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0;
    u128 cur_mult = pcg_mult(), cur_plus = g.inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    g.state = acc_mult * g.state + acc_plus;
}

}  // namespace cgh
