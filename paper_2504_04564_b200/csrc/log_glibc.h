// log_glibc.h — the natural logarithm exactly as the reference's std::log computes it.
//
// The reference draws every free-flight step as t -= log(1 - u) * inv_maj (render.hpp:116) with
// glibc's log. glibc 2.39 (this image) implements it with the ARM optimized-routines algorithm and,
// on x86-64 CPUs with FMA (the dispatched __log_fma build), fuses the products shown below. This is
// that algorithm restated — table-driven reduction x = 2^k z, z ~ c (128 subintervals), log1p of
// r = z/c - 1 by a degree-5 polynomial, and a separate degree-11 polynomial within [1-2^-4, 1+0.0645)
// — with the constants generated from this image's libm (tools/gen_log_table.py -> log_table.inc).
// Every FP operation and fused multiply-add is explicit (TUs build with -fmad=false / -ffp-contract=off),
// so host and device give the same bits; tests/cpp/test_log.cpp checks it against the system log.
// Domain: positive normal doubles (the tracer calls it on 1 - u in [2^-53, 1]).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#include "log_table.inc"

#ifdef __CUDACC__
#define SVDB_HD __host__ __device__ __forceinline__
#else
#define SVDB_HD inline
#endif

namespace svdbgpu {

struct alignas(16) LogTabEntry {
    double invc, logc;
};

#ifdef __CUDACC__
static __device__ const LogTabEntry kLogTabDev[128] = {SVDB_LOG_TAB};
#endif
static const LogTabEntry kLogTabHost[128] = {SVDB_LOG_TAB};

SVDB_HD uint64_t log_asuint(double x)
{
#ifdef __CUDA_ARCH__
    return uint64_t(__double_as_longlong(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
#endif
}

SVDB_HD double log_asdouble(uint64_t u)
{
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    std::memcpy(&x, &u, 8);
    return x;
#endif
}

SVDB_HD double glibc_log(double x)
{
    using std::fma;
    const uint64_t ix = log_asuint(x);
    constexpr uint64_t kLo = 0x3FEE000000000000ull; // asuint64(1.0 - 0x1p-4)
    constexpr uint64_t kHi = 0x3FF1090000000000ull; // asuint64(1.0 + 0x1.09p-4)
    if (ix - kLo < kHi - kLo) {
        if (ix == 0x3FF0000000000000ull)
            return 0.0;
        const double r = x - 1.0, r2 = r * r, r3 = r * r2;
        const double i2 = fma(r3, SVDB_LOG_B10, fma(r2, SVDB_LOG_B9, fma(r, SVDB_LOG_B8, SVDB_LOG_B7)));
        const double i1 = fma(r3, i2, fma(r2, SVDB_LOG_B6, fma(r, SVDB_LOG_B5, SVDB_LOG_B4)));
        const double p = fma(r3, i1, fma(r2, SVDB_LOG_B3, fma(r, SVDB_LOG_B2, SVDB_LOG_B1)));
        double w = r * 0x1p27;
        const double rhi = r + w - w;
        const double rlo = r - rhi;
        const double rr = rhi * rhi; // exact: rhi has <= 26 significant bits
        const double hi = fma(rr, SVDB_LOG_B0, r);
        double lo = fma(rr, SVDB_LOG_B0, r - hi);
        lo = fma(SVDB_LOG_B0 * rlo, rhi + r, lo);
        return fma(r3, p, lo) + hi;
    }
    // x = 2^k z with z in [0x1.6p-1, 0x1.6p0) split into 128 subintervals around c = 1/invc
    constexpr uint64_t kOff = 0x3FE6000000000000ull;
    const uint64_t tmp = ix - kOff;
    const int i = int((tmp >> 45) & 127u);
    const int k = int(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & (0xFFFull << 52));
#ifdef __CUDA_ARCH__
    // one 16-B load; the 2 KB table is marked evict-last so the leaf data streaming through L1
    // does not push it out (a shared-memory copy measured 2% slower: one CTA less per SM)
    double invc, logc;
    asm("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];"
        : "=d"(invc), "=d"(logc)
        : "l"(reinterpret_cast<const double2*>(kLogTabDev) + i));
#else
    const double invc = kLogTabHost[i].invc, logc = kLogTabHost[i].logc;
#endif
    const double z = log_asdouble(iz);
    const double r = fma(z, invc, -1.0);
    const double kd = double(k);
    const double w = fma(kd, SVDB_LOG_LN2HI, logc);
    const double hi = w + r;
    const double lo = fma(kd, SVDB_LOG_LN2LO, w - hi + r);
    const double r2 = r * r;
    const double p = fma(r2, fma(r, SVDB_LOG_A4, SVDB_LOG_A3), fma(r, SVDB_LOG_A2, SVDB_LOG_A1));
    return fma(r * r2, p, fma(r2, SVDB_LOG_A0, lo)) + hi;
}

} // namespace svdbgpu
