// glibc_exp.cuh -- bit-exact port of glibc 2.39's exp (x86_64) for the
// exponential ziggurat's wedge test.
//
// numpy's random_standard_exponential (distributions.c) accepts a wedge
// draw when (fe[i-1]-fe[i]) * u + fe[i] < exp(-x), with the host libm's exp.
// glibc >= 2.28 computes exp with sysdeps/ieee754/dbl-64/e_exp.c (N = 128
// table, degree-5 polynomial, data __exp_data) and resolves it by IFUNC:
// __exp_fma on CPUs with FMA+AVX2 (the a*b+c of the reduction and the
// polynomial fused), the SSE2/AVX builds otherwise (no fusion).  Both are
// restated here from the disassembly of the host libm (objdump of
// libm.so.6: the FMA variant's vfmadd sequence, the SSE2 variant's
// mulsd/addsd order); the constants and table are that libm's own bytes
// (glibc_exp_tables.cuh, tools/gen_glibc_exp_table.py).  The variant follows
// the host CPU exactly like log1p's (cs_host_log1p_variant: FMA && AVX2).
//
// Domain: the ziggurat calls exp(-x) for 0 <= x < r = 7.697...; the port
// covers |x| < 512 (the main path) and the tiny-argument path, which is all
// of that; other arguments fall back to the CUDA exp (never reached here).
// tests/test_exp_port.py compiles this file as host C++ and compares it
// with the host libm on every CPU test run.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "glibc_exp_tables.cuh"

#if defined(__CUDACC__)
#define CS_XHD __host__ __device__
#else
#define CS_XHD
#endif

namespace cs {

CS_XHD inline double ex_bits2d(uint64_t u) {
    double d;
#if defined(__CUDA_ARCH__)
    d = __longlong_as_double((long long)u);
#else
    memcpy(&d, &u, 8);
#endif
    return d;
}
CS_XHD inline uint64_t ex_d2bits(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}
#if defined(__CUDA_ARCH__)
#define EX_ADD(a, b) __dadd_rn((a), (b))
#define EX_SUB(a, b) __dsub_rn((a), (b))
#define EX_MUL(a, b) __dmul_rn((a), (b))
#define EX_FMA(a, b, c) __fma_rn((a), (b), (c))
#define EX_TAB CS_EXP_TAB
#else
#define EX_ADD(a, b) ((a) + (b))
#define EX_SUB(a, b) ((a) - (b))
#define EX_MUL(a, b) ((a) * (b))
#define EX_FMA(a, b, c) fma((a), (b), (c))
#define EX_TAB CS_EXP_TAB_H
#endif

// exp(x) as glibc computes it; fma = 1 for the FMA+AVX2 build.
CS_XHD inline double glibc_exp(double x, int fma_variant) {
    const uint64_t ux = ex_d2bits(x);
    const uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {  // |x| < 2^-54 or |x| >= 512 (or inf/nan)
        if (abstop < 0x3c9u) return EX_ADD(1.0, x);
        return exp(x);  // outside the ziggurat's domain
    }
    const double InvLn2N = ex_bits2d(CS_EXP_INVLN2N_BITS), Shift = ex_bits2d(CS_EXP_SHIFT_BITS);
    const double NegLn2hiN = ex_bits2d(CS_EXP_NEGLN2HIN_BITS), NegLn2loN = ex_bits2d(CS_EXP_NEGLN2LON_BITS);
    const double C2 = ex_bits2d(CS_EXP_C2_BITS), C3 = ex_bits2d(CS_EXP_C3_BITS);
    const double C4 = ex_bits2d(CS_EXP_C4_BITS), C5 = ex_bits2d(CS_EXP_C5_BITS);
    double kd, r, tmp;
    uint64_t ki;
    if (fma_variant) {
        kd = EX_FMA(x, InvLn2N, Shift);
        ki = ex_d2bits(kd);
        kd = EX_SUB(kd, Shift);
        r = EX_FMA(kd, NegLn2hiN, x);
        r = EX_FMA(kd, NegLn2loN, r);
    } else {
        kd = EX_ADD(EX_MUL(InvLn2N, x), Shift);
        ki = ex_d2bits(kd);
        kd = EX_SUB(kd, Shift);
        r = EX_ADD(EX_ADD(EX_MUL(NegLn2hiN, kd), x), EX_MUL(kd, NegLn2loN));
    }
    const uint64_t idx = 2 * (ki & 127);
    const uint64_t top = ki << 45;
    const double tail = ex_bits2d(EX_TAB[idx]);
    const uint64_t sbits = EX_TAB[idx + 1] + top;
    const double r2 = EX_MUL(r, r);
    if (fma_variant) {
        const double t1 = EX_FMA(r, C3, C2);
        const double t2 = EX_FMA(r, C5, C4);
        const double a = EX_FMA(t1, r2, EX_ADD(r, tail));
        tmp = EX_FMA(EX_MUL(r2, r2), t2, a);
        const double scale = ex_bits2d(sbits);
        return EX_FMA(scale, tmp, scale);
    }
    const double t1 = EX_ADD(EX_MUL(C3, r), C2);
    const double t2 = EX_ADD(EX_MUL(r, C5), C4);
    tmp = EX_ADD(EX_ADD(EX_MUL(t1, r2), EX_ADD(tail, r)), EX_MUL(t2, EX_MUL(r2, r2)));
    const double scale = ex_bits2d(sbits);
    return EX_ADD(EX_MUL(tmp, scale), scale);
}

#undef EX_ADD
#undef EX_SUB
#undef EX_MUL
#undef EX_FMA
#undef EX_TAB

}  // namespace cs
