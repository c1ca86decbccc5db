// glibc_log1p.cuh -- bit-exact device port of glibc 2.39's log1p (x86_64).
//
// numpy's ziggurat tail (distributions.c random_standard_exponential, idx==0)
// returns r - npy_log1p(-next_double) and npy_log1p is the host libm's log1p.
// glibc 2.39 resolves log1p through an IFUNC: on CPUs with FMA+AVX2 it runs
// __log1p_fma (the fdlibm s_log1p.c algorithm compiled with -mfma, so several
// a*b+c are fused), otherwise the SSE2 build (no fusion).  Both variants are
// ported; variant selection mirrors glibc's resolver and is done on the host
// (cs_host_log1p_variant()).  Verified bit-exact against both libm variants on
// 1e8 inputs; tests/test_log1p_port.py compiles THIS file as host C++ and
// compares it with the host libm on every CPU test run.
//
// Every arithmetic step is an explicit round-to-nearest intrinsic: the file
// must not depend on -fmad settings.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

// Host twin: the same source compiles as plain C++ (g++ -ffp-contract=off) so
// tests/test_log1p_port.py can compare it with the host libm without a GPU.
#if defined(__CUDACC__)
#define CS_HD __host__ __device__
#else
#define CS_HD
#endif
#if defined(__CUDA_ARCH__)
#define CS_ADD(a, b) __dadd_rn((a), (b))
#define CS_SUB(a, b) __dsub_rn((a), (b))
#define CS_MUL(a, b) __dmul_rn((a), (b))
#define CS_DIV(a, b) __ddiv_rn((a), (b))
#define CS_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define CS_ADD(a, b) ((a) + (b))
#define CS_SUB(a, b) ((a) - (b))
#define CS_MUL(a, b) ((a) * (b))
#define CS_DIV(a, b) ((a) / (b))
#define CS_FMA(a, b, c) fma((a), (b), (c))
#endif

namespace cs {

CS_HD inline int32_t hi_word(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    return (int32_t)(u >> 32);
}

CS_HD inline double set_hi_word(double x, int32_t h) {
    uint64_t u;
    memcpy(&u, &x, 8);
    u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32);
    double r;
    memcpy(&r, &u, 8);
    return r;
}

CS_HD inline double glibc_log1p(double x, int fma_variant) {
    const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
    const double two54 = 1.80143985094819840000e+16;
    const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                 Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                 Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                 Lp7 = 1.479819860511658591e-01;
    double hfsq, f = 0.0, c = 0.0, s, z, R, u;
    int32_t k, hx, hu = 0, ax;
    hx = hi_word(x);
    ax = hx & 0x7fffffff;
    k = 1;
    if (hx < 0x3FDA827A) {
        if (ax >= 0x3ff00000) {
            if (x == -1.0) return -two54 / 0.0;
            return (x - x) / (x - x);
        }
        if (ax < 0x3e200000) {
            if (CS_ADD(two54, x) > 0.0 && ax < 0x3c900000) return x;
            const double xx = CS_MUL(x, x);
            return fma_variant ? CS_FMA(-xx, 0.5, x) : CS_SUB(x, CS_MUL(xx, 0.5));
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return CS_ADD(x, x);
    }
    if (k != 0) {
        if (hx < 0x43400000) {
            u = CS_ADD(1.0, x);
            hu = hi_word(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? CS_SUB(1.0, CS_SUB(u, x)) : CS_SUB(x, CS_SUB(u, 1.0));
            c = CS_DIV(c, u);
        } else {
            u = x;
            hu = hi_word(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = set_hi_word(u, hu | 0x3ff00000);
        } else {
            k += 1;
            u = set_hi_word(u, hu | 0x3fe00000);
            hu = (0x00100000 - hu) >> 2;
        }
        f = CS_SUB(u, 1.0);
    }
    hfsq = CS_MUL(CS_MUL(0.5, f), f);
    const double dk = (double)k;
    if (hu == 0) {
        if (f == 0.0) {
            if (k == 0) return 0.0;
            if (fma_variant) return CS_FMA(dk, ln2_hi, CS_FMA(dk, ln2_lo, c));
            c = CS_ADD(c, CS_MUL(dk, ln2_lo));
            return CS_ADD(CS_MUL(dk, ln2_hi), c);
        }
        R = fma_variant ? CS_MUL(CS_FMA(-f, 0.66666666666666666, 1.0), hfsq)
                        : CS_MUL(hfsq, CS_SUB(1.0, CS_MUL(0.66666666666666666, f)));
        if (k == 0) return CS_SUB(f, R);
        if (fma_variant)
            return CS_FMA(dk, ln2_hi, -CS_SUB(CS_SUB(R, CS_FMA(dk, ln2_lo, c)), f));
        return CS_SUB(CS_MUL(dk, ln2_hi),
                         CS_SUB(CS_SUB(R, CS_ADD(CS_MUL(dk, ln2_lo), c)), f));
    }
    s = CS_DIV(f, CS_ADD(2.0, f));
    z = CS_MUL(s, s);
    if (fma_variant) {
        const double R2 = CS_FMA(z, Lp3, Lp2), R3 = CS_FMA(z, Lp5, Lp4), R4 = CS_FMA(z, Lp7, Lp6);
        const double z2 = CS_MUL(z, z), z4 = CS_MUL(z2, z2), z6 = CS_MUL(z4, z2);
        R = CS_FMA(z6, R4, CS_FMA(z4, R3, CS_FMA(z, Lp1, CS_MUL(z2, R2))));
    } else {
        const double R1 = CS_MUL(z, Lp1), z2 = CS_MUL(z, z);
        const double R2 = CS_ADD(Lp2, CS_MUL(z, Lp3)), z4 = CS_MUL(z2, z2);
        const double R3 = CS_ADD(Lp4, CS_MUL(z, Lp5)), z6 = CS_MUL(z4, z2);
        const double R4 = CS_ADD(Lp6, CS_MUL(z, Lp7));
        R = CS_ADD(CS_ADD(CS_ADD(R1, CS_MUL(z2, R2)), CS_MUL(z4, R3)), CS_MUL(z6, R4));
    }
    const double shr = CS_MUL(s, CS_ADD(hfsq, R));
    if (k == 0) return CS_SUB(f, CS_SUB(hfsq, shr));
    if (fma_variant)
        return CS_FMA(dk, ln2_hi, -CS_SUB(CS_SUB(hfsq, CS_ADD(shr, CS_FMA(dk, ln2_lo, c))), f));
    return CS_SUB(CS_MUL(dk, ln2_hi),
                     CS_SUB(CS_SUB(hfsq, CS_ADD(shr, CS_ADD(CS_MUL(dk, ln2_lo), c))), f));
}

}  // namespace cs
