// Test helper: the host build of csrc/glibc_exp.cuh vs the system libm exp(), bit for bit.
// Prints "<checked> <mismatches>" and the first mismatches. Built by tests/test_glibc_exp.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "glibc_exp.cuh"

static const uint64_t kTab[] = SGB_GLIBC_EXP_TAB;

static uint64_t bits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}

int main() {
    uint64_t s = 0x1234567;
    auto next = [&] {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    auto uni = [&] { return static_cast<double>(next() >> 11) * 0x1.0p-53; };
    long long n = 0, bad = 0;
    auto check = [&](double x) {
        volatile double xv = x;
        const double want = ::exp(xv);
        const double got = sgb::gx::exp(xv, kTab);
        ++n;
        if (bits(want) != bits(got) && !(want != want && got != got)) {
            if (bad < 10) std::printf("x=%a libm=%a ours=%a\n", x, want, got);
            ++bad;
        }
    };
    const double specials[] = {0.0, -0.0, 1e-300, -1e-300, 0x1p-54, -0x1p-54, 0x1p-55, 1.0, -1.0, 709.7, 709.8,
                               -708.4, -708.5, -745.1, -745.2, -1000.0, -1024.0, -1e308, 1e308, INFINITY,
                               -INFINITY, NAN, 512.0, -512.0, 0x1.fffffffffffffp9, -0x1.fffffffffffffp9};
    for (double x : specials) check(x);
    for (int i = 0; i < (1 << 22); ++i) check(-40.0 * uni());           // sampling range (logit gaps / T)
    for (int i = 0; i < (1 << 21); ++i) check(-750.0 * uni());          // down to the subnormal edge
    for (int i = 0; i < (1 << 20); ++i) check(-1100.0 + 2200.0 * uni());  // both special paths
    for (int i = 0; i < (1 << 20); ++i) check((uni() - 0.5) * 0x1p-40);  // tiny arguments
    for (int i = 0; i < (1 << 22); ++i) {                                 // arbitrary bit patterns
        uint64_t u = next();
        double x;
        std::memcpy(&x, &u, 8);
        check(x);
    }
    // the CDF terms exactly as sample_token forms them: (double(float l) - max) / T
    for (int i = 0; i < (1 << 22); ++i) {
        const float l = static_cast<float>((uni() - 0.5) * 40.0);
        const double mx = static_cast<double>(static_cast<float>(20.0 * uni()));
        const double T = (i & 3) == 0 ? 1.0 : (i & 3) == 1 ? 0.7 : (i & 3) == 2 ? 1.5 : 0.3;
        volatile double x = (static_cast<double>(l) - mx) / T;
        check(x);
    }
    std::printf("%lld %lld\n", n, bad);
    return bad != 0;
}
