// tests/cpp/test_log.cpp — TEST INFRASTRUCTURE: the restated glibc log (csrc/log_glibc.h, used by the
// device tracer for the step draw, render.hpp:116) against the system libm log, bit for bit, over
// the tracer's whole input set shape: 1 - u for splitmix64 draws u (rng.hpp:54-63), the values next
// to 1 (k * 2^-53 steps), the smallest inputs, and every table subinterval boundary.
#include "log_glibc.h"

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static uint64_t bits(double x)
{
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}

int main(int argc, char** argv)
{
    const long n = argc > 1 ? std::atol(argv[1]) : 20000000;
    long bad = 0, tested = 0;
    auto check = [&](double w) {
        ++tested;
        if (bits(svdbgpu::glibc_log(w)) != bits(std::log(w))) {
            if (bad < 5)
                std::printf("mismatch at %a: %a vs libm %a\n", w, svdbgpu::glibc_log(w), std::log(w));
            ++bad;
        }
    };
    uint64_t s = 0x5EEDull;
    for (long j = 0; j < n; ++j) { // the draw distribution: w = 1 - u
        s += 0x9E3779B97F4A7C15ull;
        uint64_t x = s;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        x ^= x >> 31;
        const double w = 1.0 - double(x >> 11) * 0x1.0p-53;
        if (w > 0.0)
            check(w);
    }
    for (long k = 1; k <= 2000000; ++k) { // next to 1 and the smallest inputs
        check(1.0 - double(k) * 0x1.0p-53);
        check(double(k) * 0x1.0p-53);
    }
    for (int i = 0; i < 4096; ++i) { // around the subinterval and range boundaries
        const double z = std::ldexp(1.0, -(i % 60)) * (0.6875 + (i / 60) * (0.6875 / 68.0));
        for (int d = -3; d <= 3; ++d)
            check(std::nextafter(z, d < 0 ? 0.0 : 2.0) + 0.0 * d);
    }
    std::printf("glibc_log: %ld mismatches of %ld\n", bad, tested);
    return bad ? 1 : 0;
}
