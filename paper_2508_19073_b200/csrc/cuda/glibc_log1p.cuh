// log1p bit-identical to the host C library the reference links: glibc 2.39's
// x86-64 __log1p_fma (sysdeps/ieee754/dbl-64/s_log1p.c built with -mfma, the
// ifunc variant on FMA-capable CPUs) — the fdlibm algorithm with glibc's
// Estrin-style polynomial, every floating-point operation and every fused
// multiply-add exactly where that build has one. The reference's exponential
// arrival gaps go through it (rng.hpp:41-44: -mean * log1p(-u)), and a 1-ulp
// difference in one gap moves every later submit time, so device-generated
// traces need this function rather than CUDA's log1p.
//
// Pinned by carma_host_check_log1p (host build of the same code) against the
// C library's log1p on random, small and branch-boundary inputs
// (tests/test_host.py). Compiled without contraction (--fmad=false /
// -ffp-contract=off): the fused operations are the explicit fma() calls.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

namespace carma_b200 {

#if defined(__CUDACC__)
#define CARMA_HD __host__ __device__
#else
#define CARMA_HD
#endif

CARMA_HD inline uint32_t l1p_hi(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint32_t>(__double2hiint(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return static_cast<uint32_t>(u >> 32);
#endif
}

CARMA_HD inline double l1p_sethi(double x, uint32_t h) {
#if defined(__CUDA_ARCH__)
    return __hiloint2double(static_cast<int>(h), __double2loint(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    u = (u & 0xffffffffull) | (static_cast<uint64_t>(h) << 32);
    std::memcpy(&x, &u, 8);
    return x;
#endif
}

CARMA_HD inline double glibc_log1p(double x) {
    constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                     Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                     Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                     Lp7 = 1.479819860511658591e-01;
    double f = 0.0, c = 0.0, u;
    int32_t k = 1, hu = 0;
    const int32_t hx = static_cast<int32_t>(l1p_hi(x));
    const int32_t ax = hx & 0x7fffffff;
    if (hx < 0x3FDA827A) {  // x < 0.41422
        if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;  // x <= -1
        if (ax < 0x3e200000) {  // |x| < 2^-29
            if (ax < 0x3c900000) return x;
            return fma(-(x * x), 0.5, x);
        }
        if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec3u)) {  // -0.2929 < x < 0.41422
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return x + x;
    }
    if (k != 0) {
        if (hx < 0x43400000) {
            u = 1.0 + x;
            hu = static_cast<int32_t>(l1p_hi(u));
            k = (hu >> 20) - 1023;
            c = k > 0 ? 1.0 - (u - x) : x - (u - 1.0);
            c /= u;
        } else {
            u = x;
            hu = static_cast<int32_t>(l1p_hi(u));
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = l1p_sethi(u, static_cast<uint32_t>(hu | 0x3ff00000));
        } else {
            k += 1;
            u = l1p_sethi(u, static_cast<uint32_t>(hu | 0x3fe00000));
            hu = (0x00100000 - hu) >> 2;
        }
        f = u - 1.0;
    }
    const double hfsq = (0.5 * f) * f;
    const double dk = static_cast<double>(k);
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = fma(dk, ln2_lo, c);
            return fma(dk, ln2_hi, c);
        }
        const double R = hfsq * fma(-0.66666666666666666, f, 1.0);
        if (k == 0) return f - R;
        return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
    }
    const double s = f / (2.0 + f);
    const double z = s * s;
    const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
    const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
    const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, z2 * R2)));
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return fma(dk, ln2_hi, -((hfsq - (s * (hfsq + R) + fma(dk, ln2_lo, c))) - f));
}

}  // namespace carma_b200
