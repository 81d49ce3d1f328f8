// expf_glibc.cuh — glibc-exact expf on the device (shared by kernels.cu and train.cu).
#pragma once
#include <cstdint>

namespace smoe {

// expf as glibc computes it (sysdeps/ieee754/flt-32/e_expf.c, the table and
// constants of __exp2f_data, verified against this image's libm.so.6): the
// reference's estimator SiLU calls std::exp(float) (estimator.cpp:121), so the
// GPU reproduces glibc's algorithm bit for bit instead of CUDA's expf.
static __constant__ unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

__device__ inline float expf_glibc(float x) {
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {  // |x| >= 88 (top12(88.0f)) and specials
        if (ux == 0xff800000u) return 0.0f;  // -inf
        if (abstop >= 0x7f8) return x + x;   // inf / nan
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);  // overflow
        if (x < -0x1.9fe368p6f) return 0.0f;                        // underflow
    }
    const double InvLn2N = 0x1.71547652b82fep+5, Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13,
                 C2 = 0x1.62e42ff0c52d6p-6;
    const double xd = static_cast<double>(x);
    const double z = __dmul_rn(InvLn2N, xd);
    double kd = __dadd_rn(z, Shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, Shift);
    const double r = __dsub_rn(z, kd);
    const unsigned long long t = kExp2fTab[ki % 32] + (ki << 47);
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double zz = __dadd_rn(__dmul_rn(C0, r), C1);
    const double r2 = __dmul_rn(r, r);
    double y = __dadd_rn(__dmul_rn(C2, r), 1.0);
    y = __dadd_rn(__dmul_rn(zz, r2), y);
    y = __dmul_rn(y, s);
    return static_cast<float>(y);
}

}  // namespace smoe
