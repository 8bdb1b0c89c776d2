// Host check: pcg_next_halfturns == float(2u or 2u-2) computed in fp64, bit for bit.
// nvcc -O2 -std=c++17 --expt-relaxed-constexpr -o check_halfturns check_halfturns.cu && ./check_halfturns
#include <cstdio>
#include <cstring>
#include "../../paper_2006_10509_b200/csrc/pcg64.cuh"
using namespace cgh;
int main() {
    Pcg64 a, b;
    a.state = (u128(0x0123456789ABCDEFULL) << 64) | 0xFEDCBA9876543210ULL;
    a.inc = (u128(0x1111111111111111ULL) << 64) | 0x2222222222222223ULL;
    a.has_uint32 = 0;
    a.uinteger = 0;
    b = a;
    long bad = 0;
    const long n = 20000000;
    for (long i = 0; i < n; ++i) {
        double x = 2.0 * pcg_next_double(a);
        if (x > 1.0) x -= 2.0;
        const float f0 = float(x), f1 = pcg_next_halfturns(b);
        if (memcmp(&f0, &f1, 4) != 0) ++bad;
    }
    // edge values of x53: 0, 1, 2^52 - 1, 2^52, 2^52 + 1, 2^53 - 1
    const long long edges[] = {0, 1, (1LL << 52) - 1, 1LL << 52, (1LL << 52) + 1, (1LL << 53) - 1};
    for (long long x53 : edges) {
        double x = 2.0 * (double(x53) * (1.0 / 9007199254740992.0));
        if (x > 1.0) x -= 2.0;
        const long long xi = x53 > (1LL << 52) ? x53 - (1LL << 53) : x53;
        const float f0 = float(x), f1 = float(xi) * 2.220446049250313e-16f;
        if (memcmp(&f0, &f1, 4) != 0) ++bad;
    }
    printf("%ld draws + 6 edges: %ld mismatches\n", n, bad);
    return bad != 0;
}
