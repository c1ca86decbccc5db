// cs_rng.cuh -- Philox4x64-10, numpy SeedSequence and the numpy exponential
// ziggurat, restated for sm_100a.  Bit-exact with numpy 2.3.5 / glibc 2.39.
//
// Reference call sites (/root/reference/pkg/src/chainserve):
//   sim.py:141-143  Generator(Philox(SeedSequence(entropy=seed, spawn_key=(rep,))))
//   sim.py:145      rng.exponential(1.0 / rate, n)   -> scale * standard_exponential
//   sim.py:159      rng.exponential(1.0, n)          (drawn after all n arrival draws)
// numpy semantics restated here:
//   * Philox key = SeedSequence.generate_state(2, uint64); counter starts at 0 and
//     is incremented BEFORE each block, so block b uses counter {b+1,0,0,0};
//     words are consumed in order 0..3 within a block (philox_next).
//   * next_double(u64) = (u64 >> 11) * 2^-53.
//   * random_standard_exponential: 256-layer ziggurat with tables
//     we/ke/fe (zig_tables.cuh, pinned against numpy's rodata), tail
//     r - log1p(-next_double), wedge (fe[i-1]-fe[i])*u + fe[i] < exp(-x);
//     log1p and exp are ports of the host glibc's (glibc_log1p.cuh,
//     glibc_exp.cuh), so every accept/reject decision is the host's.
#pragma once
#include <stdint.h>

#include "glibc_exp.cuh"
#include "glibc_log1p.cuh"
#include "zig_tables.cuh"

namespace cs {

constexpr uint64_t PH_M0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t PH_M1 = 0xCA5A826395121157ULL;
constexpr uint64_t PH_W0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t PH_W1 = 0xBB67AE8584CAA73BULL;

// Philox4x64-10 of counter {c0,0,0,0} (numpy counters never exceed 2^64 here).
__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                              uint64_t k0, uint64_t k1, uint64_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += PH_W0;
            k1 += PH_W1;
        }
        const uint64_t lo0 = PH_M0 * c0, hi0 = __umul64hi(PH_M0, c0);
        const uint64_t lo1 = PH_M1 * c2, hi1 = __umul64hi(PH_M1, c2);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// The 10 round keys of one stream, staged in shared memory by its warp
// (ks[r] = {k0 + r*W0, k1 + r*W1}): held in registers they took 40 of the
// stream kernels' 128, and the slow-attempt loop then spilled.
__device__ __forceinline__ void philox_key_schedule(ulonglong2* ks, int lane, uint64_t k0, uint64_t k1) {
    if (lane < 10) ks[lane] = make_ulonglong2(k0 + (uint64_t)lane * PH_W0, k1 + (uint64_t)lane * PH_W1);
    __syncwarp();
}

// Philox4x64-10 of counter {c0,0,0,0} with the round keys read from ks.
__device__ __forceinline__ void philox4x64_10_ks(uint64_t c0, const ulonglong2* ks, uint64_t out[4]) {
    uint64_t c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const ulonglong2 k = ks[r];
        const uint64_t lo0 = PH_M0 * c0, hi0 = __umul64hi(PH_M0, c0);
        const uint64_t lo1 = PH_M1 * c2, hi1 = __umul64hi(PH_M1, c2);
        const uint64_t n0 = hi1 ^ c1 ^ k.x, n2 = hi0 ^ c3 ^ k.y;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

// Ziggurat tables staged in shared memory (random per-lane layer index).
struct ZigSmem {
    double we[256];
    uint64_t ke[256];
    double fe[256];
};

__device__ __forceinline__ void zig_load(ZigSmem* z) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        z->we[i] = __longlong_as_double((long long)CS_ZIG_WE_BITS_D[i]);
        z->ke[i] = CS_ZIG_KE_D[i];
        z->fe[i] = __longlong_as_double((long long)CS_ZIG_FE_BITS_D[i]);
    }
}

__device__ __forceinline__ double u64_to_unit(uint64_t w) {
    // (w >> 11) * (1.0 / 9007199254740992.0): exact
    return __dmul_rn((double)(w >> 11), 1.1102230246251565e-16);
}

// Result of one ziggurat ATTEMPT that starts at word w (and may need word w2).
// adv = words consumed (1 or 2); has = attempt produced a value.
struct ZigAttempt {
    double v;
    int adv;
    bool has;
};

__device__ __forceinline__ bool zig_fast(const ZigSmem* z, uint64_t w, double* x) {
    const uint64_t ri = w >> 11;
    const int idx = (int)((w >> 3) & 0xFF);
    *x = __dmul_rn((double)ri, z->we[idx]);
    return ri < z->ke[idx];
}

__device__ __forceinline__ ZigAttempt zig_slow(const ZigSmem* z, uint64_t w, uint64_t w2,
                                            int log1p_fma) {
    const uint64_t ri = w >> 11;
    const int idx = (int)((w >> 3) & 0xFF);
    const double x = __dmul_rn((double)ri, z->we[idx]);
    const double u = u64_to_unit(w2);
    ZigAttempt a;
    a.adv = 2;
    if (idx == 0) {
        const double r = __longlong_as_double((long long)CS_ZIG_EXP_R_BITS);
        a.v = __dsub_rn(r, glibc_log1p(-u, log1p_fma));
        a.has = true;
    } else {
        // numpy: (fe[idx-1]-fe[idx]) * next_double + fe[idx] < exp(-x), no
        // contraction, exp = the host glibc's (same build variant as log1p)
        const double y = __dadd_rn(__dmul_rn(__dsub_rn(z->fe[idx - 1], z->fe[idx]), u), z->fe[idx]);
        a.v = x;
        a.has = y < glibc_exp(-x, log1p_fma);
    }
    return a;
}

}  // namespace cs
