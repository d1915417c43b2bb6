// CPU check of the device "%.17g" formatter (paper_2509_06971_b200/csrc/g17.cuh,
// host build) against glibc's snprintf, which the reference's writers call
// (field_io.cpp:15-19).  Usage: test_g17 [random_count] [seed]; exit 0 = identical.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "g17.cuh"

static long fails = 0, checked = 0;

static void check(double v) {
    char want[64], got[64];
    std::snprintf(want, sizeof want, "%.17g", v);
    const int n = petto_b200::g17::format(v, got);
    got[n] = 0;
    ++checked;
    if (std::strcmp(want, got) != 0 && fails++ < 20) {
        unsigned long long b;
        std::memcpy(&b, &v, 8);
        std::printf("MISMATCH bits=%016llx want=%s got=%s\n", b, want, got);
    }
}

int main(int argc, char** argv) {
    const long count = argc > 1 ? std::atol(argv[1]) : 2000000;
    const unsigned seed = argc > 2 ? (unsigned)std::atol(argv[2]) : 12345u;
    // special values and edge cases
    const double sp[] = {0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 1e-4, 9.9999999999999995e-5, 1e-5, 1e16, 1e17,
                         99999999999999999.0, 1e308, 1.7976931348623157e308, 2.2250738585072014e-308,
                         4.9406564584124654e-324, 2.2250738585072009e-308, INFINITY, -INFINITY, NAN, -NAN,
                         123.456, 0.30000000000000004, 1.0 / 3.0, 2.0 / 3.0, 1e-300, 5e-324, 1e22, 1e23};
    for (double v : sp) check(v);
    // integers, powers of two and of ten, and their neighbours
    for (int e = -1074; e <= 1023; ++e) {
        const double v = std::ldexp(1.0, e);
        check(v);
        check(std::nextafter(v, 0.0));
        check(std::nextafter(v, INFINITY));
    }
    for (int k = -325; k <= 308; ++k) {
        const double v = std::pow(10.0, k);
        check(v);
        check(std::nextafter(v, 0.0));
        check(std::nextafter(v, INFINITY));
    }
    for (long i = 0; i < 200000; ++i) check((double)i), check(-(double)i * 7.0), check(i * 0.5), check(i * 0.125);
    // exact ties at the 18th significant digit: (2D+1) 5^e 2^(e-1) and m 2^-k
    for (long d = 1; d < 20000; ++d)
        for (int e = 5; e <= 12; ++e) check((double)(2 * (100000000000000ll + d * 7919) + 1) * std::pow(5.0, e) * std::ldexp(1.0, e - 1));
    std::mt19937_64 rng(seed);
    // random bit patterns (whole range), random values in typical field ranges
    for (long i = 0; i < count; ++i) {
        unsigned long long b = rng();
        double v;
        std::memcpy(&v, &b, 8);
        check(v);
        const double u = std::ldexp((double)(rng() >> 11), -53);
        check(u * 2.0 - 1.0);
        check((u - 0.5) * 1e-3);
        check(u * std::pow(10.0, (int)(rng() % 40) - 20));
    }
    std::printf("g17: %ld values checked, %ld mismatches\n", checked, fails);
    return fails ? 1 : 0;
}
