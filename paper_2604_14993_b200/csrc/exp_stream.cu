// exp_stream.cu -- warp-parallel numpy-exact exponential streams.
//
// Replaces, bit for bit, Generator(Philox(key)).exponential(1.0, n) as used by
// the reference at sim.py:145,159 (the arrival gaps are scale * S[0:n] and the
// sizes are S[n:2n] of ONE stream S = standard_exponential(2n); the survey's
// common-random-number identity).
//
// Layout: one warp per stream.  A chunk is 32 NB consecutive Philox blocks
// (lane l owns blocks 32 NB c + NB l + b, b < NB, i.e. its NW = 4 NB words
// are the chunk's words NW l .. NW l + NW - 1).
// Every word is classified as the START of a ziggurat attempt (fast accept:
// 1 word, value x; slow: 2 words, value or reject).  Whether a word actually
// starts an attempt depends on all earlier words, but an attempt never spans
// more than 2 words, so each lane's NW words form a transfer function
// {entry offset 0|1} -> {exit offset 0|1, values emitted}.  A 5-step warp
// shuffle scan composes those functions, giving every lane its true entry
// offset and output position.  A slow attempt starting at the chunk's last
// word is carried into the next chunk (resolved by lane 0 with word 0).
#include <cuda_runtime.h>

#include "cs_rng.cuh"
#include "cs_internal.cuh"

namespace cs {

// The generator loop of one stream (one warp).  For every chunk, emit(i, v)
// is called by the lanes holding values (i = index within the chunk, in
// stream order) and then chunk_done(produced, tot) by every lane (produced =
// the stream's values before this chunk, tot = this chunk's count; emitted
// values may run past n_draws, the callbacks clip).
template <bool SCAN2, int NB, bool PIPE, typename Emit, typename Done>
__device__ __forceinline__ int64_t gen_stream(const ZigSmem* zs, int lane, const ulonglong2* ks,
                                              int64_t n_draws, int log1p_fma, Emit&& emit, Done&& chunk_done) {
    constexpr int NW = 4 * NB;  // words per lane per chunk (NB Philox blocks)
    int64_t produced = 0;
    int entry = 0;        // warp-uniform: offset of the first attempt in this chunk
    uint64_t pend_w = 0;  // word that started the carried slow attempt (entry == 1)
    uint64_t chunk = 0;
    // PIPE: software-pipelined, the next chunk's Philox blocks (a long
    // dependent multiply chain per lane) are computed while this chunk is
    // classified, scanned and emitted
    uint64_t wn[NW];
    if (PIPE) {
#pragma unroll
        for (int b = 0; b < NB; b++) philox4x64_10_ks(lane * NB + b + 1, ks, wn + 4 * b);
    }
    while (produced < n_draws) {
        uint64_t w[NW];
        if (PIPE) {
#pragma unroll
            for (int q = 0; q < NW; q++) w[q] = wn[q];
#pragma unroll
            for (int b = 0; b < NB; b++) philox4x64_10_ks((chunk + 1) * 32 * NB + lane * NB + b + 1, ks, wn + 4 * b);
        } else {
#pragma unroll
            for (int b = 0; b < NB; b++) philox4x64_10_ks(chunk * 32 * NB + lane * NB + b + 1, ks, w + 4 * b);
        }
        const uint64_t wnext = __shfl_down_sync(0xffffffffu, w[0], 1);

        // Per-word attempt results.
        double v[NW];
        int adv[NW];
        bool has[NW];
        // Fast accepts first; a lane's slow attempts (about one word in 90:
        // 3/4 of the chunks have one somewhere in the warp) then run in ONE
        // loop, so a chunk pays the divergent slow path about once instead
        // of once per word position.  Bit 16: the attempt carried from the
        // previous chunk (lane 0, entry 1), resolved with this chunk's word 0.
        unsigned slow = lane == 0 && entry == 1 ? 1u << 16 : 0u;
#pragma unroll
        for (int p = 0; p < NW; p++) {
            double x;
            const bool f = zig_fast(zs, w[p], &x);
            v[p] = f ? x : 0.0;  // a slow attempt at the chunk's last word is carried
            adv[p] = f ? 1 : 2;
            has[p] = f;
            if (!f && (p < NW - 1 || lane < 31)) slow |= 1u << p;
        }
        bool carry_has = false;
        double carry_v = 0.0;
        while (slow) {
            const int p = __ffs(slow) - 1;
            slow &= slow - 1;
            uint64_t a = pend_w, b = w[0];
#pragma unroll
            for (int q = 0; q < NW; q++)
                if (p == q) {
                    a = w[q];
                    b = q < NW - 1 ? w[q + 1 < NW ? q + 1 : q] : wnext;
                }
            const ZigAttempt r = zig_slow(zs, a, b, log1p_fma);
#pragma unroll
            for (int q = 0; q < NW; q++)
                if (p == q) {
                    v[q] = r.v;
                    has[q] = r.has;
                }
            if (p == 16) {
                carry_v = r.v;
                carry_has = r.has;
            }
        }

        // Transfer function of this lane: per entry offset e, E_e = exit
        // offset | values emitted << 1.
        int e0, e1;
        {
            int p = 0, c = 0;
#pragma unroll
            for (int q = 0; q < NW; q++)
                if (p == q) {
                    c += has[q];
                    p += adv[q];
                }
            e0 = (p - NW) | (c << 1);
            p = 1;
            c = carry_has ? 1 : 0;
#pragma unroll
            for (int q = 1; q < NW; q++)
                if (p == q) {
                    c += has[q];
                    p += adv[q];
                }
            e1 = (p - NW) | (c << 1);
        }
        // Inclusive Kogge-Stone scan of function composition (prefix then
        // self): the prefix's exit offset picks this lane's entry, counts add.
        // SCAN2: two shuffles a step on the packed words (fewer instructions,
        // for the issue-bound single-point kernel); else four on the split
        // fields (shorter dependent chain, for the latency-bound prefix
        // kernel: 1 block per SM on config 2).
        if (SCAN2) {
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int p0 = __shfl_up_sync(0xffffffffu, e0, d);
                const int p1 = __shfl_up_sync(0xffffffffu, e1, d);
                if (lane >= d) {
                    const int n0 = ((p0 & 1) ? e1 : e0) + (p0 & ~1);
                    const int n1 = ((p1 & 1) ? e1 : e0) + (p1 & ~1);
                    e0 = n0;
                    e1 = n1;
                }
            }
        } else {
            int x0 = e0 & 1, x1 = e1 & 1, c0 = e0 >> 1, c1 = e1 >> 1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int px0 = __shfl_up_sync(0xffffffffu, x0, d);
                const int px1 = __shfl_up_sync(0xffffffffu, x1, d);
                const int pc0 = __shfl_up_sync(0xffffffffu, c0, d);
                const int pc1 = __shfl_up_sync(0xffffffffu, c1, d);
                if (lane >= d) {
                    const int nx0 = px0 ? x1 : x0, nc0 = pc0 + (px0 ? c1 : c0);
                    const int nx1 = px1 ? x1 : x0, nc1 = pc1 + (px1 ? c1 : c0);
                    x0 = nx0;
                    c0 = nc0;
                    x1 = nx1;
                    c1 = nc1;
                }
            }
            e0 = x0 | (c0 << 1);
            e1 = x1 | (c1 << 1);
        }
        const int ex0 = __shfl_up_sync(0xffffffffu, e0, 1);
        const int ex1 = __shfl_up_sync(0xffffffffu, e1, 1);
        const int ex = entry ? ex1 : ex0;
        const int my_entry = lane == 0 ? entry : (ex & 1);
        int pos = lane == 0 ? 0 : (ex >> 1);

        // Emit this lane's values.
        if (carry_has) emit(pos++, carry_v);
        {
            int p = my_entry;
#pragma unroll
            for (int q = 0; q < NW; q++)
                if (p == q) {
                    if (has[q]) emit(pos++, v[q]);
                    p += adv[q];
                }
        }
        // Chunk totals from lane 31; detect a carried attempt at the last word.
        const int last = __shfl_sync(0xffffffffu, entry ? e1 : e0, 31);
        const int tot = last >> 1, nxt = last & 1;
        pend_w = __shfl_sync(0xffffffffu, w[NW - 1], 31);
        chunk_done(produced, tot);
        produced += tot;
        entry = nxt;
        chunk++;
    }
    return (int64_t)chunk;
}

// streams (warps) per block; each warp's chunk loop is latency-bound, so the
// block shape barely matters (4 per block measured 2% slower than 8), but two
// blocks must fit one SM: capped at 128 registers (unbounded, the IL4 variant
// took 134 -> one block per SM, config 5's 4096 streams in 4 waves instead of
// 2: 119 -> 83 ms per chunk)
constexpr int EXP_WARPS = 8;
// Two Philox blocks (8 words) per lane per chunk, both computed at the top
// of the chunk (two independent multiply chains): the per-chunk scan, slow
// loop and write setup serve 256 words instead of 128.  Measured against one
// block per lane with the next chunk's block software-pipelined: config 5
// stream chunk 70.8 -> 61.2 ms, config 2 fused streams 3.15 -> 2.91 ms; two
// blocks software-pipelined spill (64.1 ms), four spill heavily.
constexpr int EXP_NB = 2, PFX_NB = 2;
constexpr bool EXP_PIPE = false, PFX_PIPE = false;

// The simulator's interleaved stream layout (jffc_seg.cu il4_off): stream r's
// value i at (r / 32) * 32 * ld + (i / 4) * 128 + (r % 32) * 4 + i % 4.
__device__ __forceinline__ int64_t il4_pos(int64_t i) { return ((i >> 2) << 7) + (i & 3); }

// A chunk's values cv[0, tot) to stream positions produced.. of row o (IL4),
// clipped at n_draws (> produced); value i + 32 lies 32 / 4 * 128 further.
__device__ __forceinline__ void il4_write_chunk(double* __restrict__ o, const double* cv, int lane,
                                                int64_t produced, int tot, int64_t n_draws) {
    const int lim = n_draws - produced < tot ? (int)(n_draws - produced) : tot;
    double* __restrict__ p = o + il4_pos(produced + lane);
    for (int i = lane; i < lim; i += 32, p += 1024) *p = cv[i];
}

// IL4: the interleaved layout, each chunk written in order from a per-warp
// buffer (4 consecutive lanes fill one 32-byte sector).
template <bool IL4>
__global__ void __launch_bounds__(EXP_WARPS * 32, 2) exp_streams_kernel(const uint64_t* __restrict__ keys,
                                                                     int64_t n_streams, int64_t n_draws,
                                                                     double* __restrict__ out, int64_t ld,
                                                                     int log1p_fma) {
    __shared__ ZigSmem zs;
    __shared__ double sh_vals[IL4 ? EXP_WARPS : 1][128 * EXP_NB + 8];
    __shared__ ulonglong2 sh_ks[EXP_WARPS][10];
    zig_load(&zs);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t stream = (int64_t)blockIdx.x * EXP_WARPS + (threadIdx.x >> 5);
    if (stream >= n_streams) return;
    double* __restrict__ o = IL4 ? out + (stream >> 5) * 32 * ld + (stream & 31) * 4 : out + stream * ld;
    double* cv = sh_vals[IL4 ? (threadIdx.x >> 5) : 0];
    int64_t base = 0;
    ulonglong2* ks = sh_ks[threadIdx.x >> 5];
    philox_key_schedule(ks, lane, keys[2 * stream], keys[2 * stream + 1]);
    gen_stream<true, EXP_NB, EXP_PIPE>(
        &zs, lane, ks, n_draws, log1p_fma,
        [&](int i, double x) {
            if (IL4)
                cv[i] = x;
            else if (base + i < n_draws)
                o[base + i] = x;
        },
        [&](int64_t produced, int tot) {
            if (IL4) {
                __syncwarp();
                il4_write_chunk(o, cv, lane, produced, tot, n_draws);
                __syncwarp();
            }
            base = produced + tot;
        });
}

// The arrival-time prefix of single-point streams (P = 1, interleaved): one
// thread per stream runs the exact np.cumsum chain a_j = a_{j-1} + (1/lam) *
// S_j over its gaps and records a_j at the listed job indices.  Fused into
// the generating warp this chain (8 cycles per job on one lane, the loop
// issued by the whole warp) nearly doubled the config-5 stream kernel; alone
// it runs near the DADD latency: the gaps are staged through a per-thread
// cp.async ring in shared memory laid out [batch slot][gap pair][thread]
// (16-byte pieces: a warp's shared reads are conflict-free).
constexpr int PR_B = 32, PR_NBUF = 16, PR_THREADS = 32;
__global__ void __launch_bounds__(PR_THREADS) prefix_p1_kernel(const double* __restrict__ S, int64_t n_streams,
                                                               int64_t ld, const PrefixPlan pp) {
    extern __shared__ __align__(16) double2 pr_ring[];  // [PR_NBUF][PR_B / 2][PR_THREADS]
    const int lane = threadIdx.x;
    const int64_t r = (int64_t)blockIdx.x * PR_THREADS + lane;
    const bool valid = r < n_streams;
    const double* __restrict__ src = S + (valid ? (r >> 5) * 32 * ld + (r & 31) * 4 : 0);
    const double sc = __ddiv_rn(1.0, pp.pts[0].lam);
    const int64_t n = pp.n_cum;
    const int64_t nb = (n + PR_B - 1) / PR_B;
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(pr_ring);
    auto issue = [&](int64_t b) {
        if (valid && b < nb) {
            const uint32_t d = ring_s + (uint32_t)(((b % PR_NBUF) * (PR_B / 2) * PR_THREADS + lane) * 16);
#pragma unroll
            for (int k = 0; k < PR_B / 2; k++)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + k * PR_THREADS * 16),
                             "l"(src + il4_pos(b * PR_B + 2 * k))
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int b = 0; b < PR_NBUF - 1; b++) issue(b);
    double a = 0.0;
    int ev = 0;
    for (int64_t b = 0; b < nb; b++) {
        issue(b + PR_NBUF - 1);
        asm volatile("cp.async.wait_group %0;" ::"n"(PR_NBUF - 1) : "memory");
        const double2* x = pr_ring + (b % PR_NBUF) * (PR_B / 2) * PR_THREADS + lane;
        double v[PR_B];
#pragma unroll
        for (int k = 0; k < PR_B / 2; k++) {
            const double2 t = x[k * PR_THREADS];
            v[2 * k] = __dmul_rn(sc, t.x);
            v[2 * k + 1] = __dmul_rn(sc, t.y);
        }
        const int64_t j0 = b * PR_B;
        const bool evb = ev < pp.nev && pp.ev_idx[ev] < j0 + PR_B;
        if (!evb && j0 > 0 && j0 + PR_B <= n) {
#pragma unroll
            for (int k = 0; k < PR_B; k++) a = __dadd_rn(a, v[k]);
        } else {
#pragma unroll
            for (int k = 0; k < PR_B; k++) {
                const int64_t j = j0 + k;
                if (j < n) {
                    a = j == 0 ? v[k] : __dadd_rn(a, v[k]);
                    while (ev < pp.nev && pp.ev_idx[ev] == j) {
                        if (valid) pp.out[r * pp.ncol + pp.ev_col[ev]] = a;
                        ev++;
                    }
                }
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Streams plus the segmented simulator's arrival-time prefix (jffc_seg.cu):
// while the first n_cum draws of stream r are generated, lane p of its warp
// (p < P, the sweep points sharing the stream) runs the exact sequential
// cumsum a_j = a_{j-1} + (1/lam_p) * S_j of np.cumsum over each chunk's values
// (in shared memory) and records a_j at the listed job indices into
// out[(r * P + p) * ncol + col].
// (Measured against a split design -- producer warps handing chunks to
// separate prefix warps through a shared-memory ring -- which lost: the
// prefix lanes of one warp serve several streams in lockstep and stall the
// producers, 3.9 -> 5.9 ms on config 2, 56 -> 192 ms per 2048 config-5 streams.)
//
// IL4: the output in the interleaved layout, written from the chunk buffer in
// order.

// W streams per block.  W = 16 (whole_sm): a block fills one SM's register
// file, so the kernel occupies ceil(R / 16) whole SMs and leaves the others to
// the statistics of the previous sweep running beside it (engine.py's
// pipeline); alone on the GPU, 8-warp blocks spread over every SM are faster.
template <bool IL4, int W>
__global__ void __launch_bounds__(W * 32, W == 16 ? 1 : 2) exp_streams_prefix_kernel(
    const uint64_t* __restrict__ keys, int64_t n_streams, int64_t n_draws, double* __restrict__ out,
    int64_t ld, int log1p_fma, const PrefixPlan pp) {
    __shared__ ZigSmem zs;
    __shared__ double sh_vals[W][128 * PFX_NB + 8];  // a chunk's values (<= 128 NB + carry), per warp
    __shared__ ulonglong2 sh_ks[W][10];
    zig_load(&zs);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t stream = (int64_t)blockIdx.x * W + warp;
    if (stream >= n_streams) return;
    double* __restrict__ o = IL4 ? out + (stream >> 5) * 32 * ld + (stream & 31) * 4 : out + stream * ld;
    double* cv = sh_vals[warp];
    // lane p < P: point p's chain (P <= 32)
    const bool pl = lane < pp.P;
    const double sc = pl ? __ddiv_rn(1.0, pp.pts[lane].lam) : 0.0;
    double* rec = pl ? pp.out + (stream * pp.P + lane) * pp.ncol : nullptr;
    double a = 0.0;
    int ev = 0;  // next event of the (uniform) event list
    int64_t base = 0;
    ulonglong2* ks = sh_ks[threadIdx.x >> 5];
    philox_key_schedule(ks, lane, keys[2 * stream], keys[2 * stream + 1]);
    gen_stream<false, PFX_NB, PFX_PIPE>(
        &zs, lane, ks, n_draws, log1p_fma,
        [&](int i, double x) {
            cv[i] = x;
            if (!IL4 && base + i < n_draws) o[base + i] = x;
        },
        [&](int64_t produced, int tot) {
            __syncwarp();
            if (IL4) {  // the chunk's values in order: 4-value sectors of this row
                il4_write_chunk(o, cv, lane, produced, tot, n_draws);
            }
            if (produced < pp.n_cum) {
                const int cnt = (int)min((int64_t)tot, pp.n_cum - produced);
                const int32_t j0 = (int32_t)produced;
                if (pl) {
                    if (j0 > 0 && (ev >= pp.nev || pp.ev_idx[ev] >= j0 + cnt)) {  // no event in the chunk
                        int i = 0;
                        for (; i + 4 <= cnt; i += 4) {
                            a = __dadd_rn(a, __dmul_rn(sc, cv[i]));
                            a = __dadd_rn(a, __dmul_rn(sc, cv[i + 1]));
                            a = __dadd_rn(a, __dmul_rn(sc, cv[i + 2]));
                            a = __dadd_rn(a, __dmul_rn(sc, cv[i + 3]));
                        }
                        for (; i < cnt; i++) a = __dadd_rn(a, __dmul_rn(sc, cv[i]));
                    } else {
                        for (int i = 0; i < cnt; i++) {
                            const double x = __dmul_rn(sc, cv[i]);
                            const int32_t j = j0 + i;
                            a = j == 0 ? x : __dadd_rn(a, x);
                            while (ev < pp.nev && pp.ev_idx[ev] == j) {
                                rec[pp.ev_col[ev]] = a;
                                ev++;
                            }
                        }
                    }
                }
                ev = __shfl_sync(0xffffffffu, ev, 0);  // lanes >= P track the event list too
            }
            base = produced + tot;
            __syncwarp();  // cv is rewritten by the next chunk
        });
}

// Measurement kernel (no reference counterpart): Philox4x64-10 blocks as
// fast as the SMs generate them, XOR-folded per thread so nothing is
// optimised away and nothing is stored per block.  The simulator's RNG
// floor is reported against this rate (bench.py roofline.rng_floor).
__global__ void __launch_bounds__(256) philox_peak_kernel(int64_t blocks_per_thread, uint64_t k0, uint64_t k1,
                                                          uint64_t* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t acc = 0;
    for (int64_t i = 0; i < blocks_per_thread; i++) {
        uint64_t w[4];
        philox4x64_10(t + stride * (uint64_t)i + 1, 0, 0, 0, k0, k1, w);
        acc ^= w[0] ^ w[1] ^ w[2] ^ w[3];
    }
    out[t] = acc;
}

}  // namespace cs

extern "C" int cs_philox_peak_impl(int64_t blocks_per_thread, int32_t grid, uint64_t* d_out, void* stream) {
    cs::philox_peak_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(blocks_per_thread, 0x0123456789abcdefULL,
                                                                   0xfedcba9876543210ULL, d_out);
    return cs::check_launch("philox_peak_kernel");
}

extern "C" int cs_exp_streams_impl(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws,
                                   double* d_out, int64_t ld, int log1p_fma, void* stream) {
    if (n_streams <= 0 || n_draws <= 0) return 0;
    const int64_t blocks = (n_streams + cs::EXP_WARPS - 1) / cs::EXP_WARPS;
    cs::exp_streams_kernel<false><<<(unsigned)blocks, cs::EXP_WARPS * 32, 0, (cudaStream_t)stream>>>(
        d_keys, n_streams, n_draws, d_out, ld, log1p_fma);
    return cs::check_launch("exp_streams_kernel");
}

// Single-point interleaved streams: generation, then the prefix pass.
extern "C" int cs_exp_streams_il4_p1_impl(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws,
                                          double* d_out, int64_t ld, int log1p_fma, const cs::PrefixPlan* plan,
                                          void* stream) {
    if (n_streams <= 0 || n_draws <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t blocks = (n_streams + cs::EXP_WARPS - 1) / cs::EXP_WARPS;
    cs::exp_streams_kernel<true><<<(unsigned)blocks, cs::EXP_WARPS * 32, 0, st>>>(d_keys, n_streams, n_draws,
                                                                                  d_out, ld, log1p_fma);
    int rc = cs::check_launch("exp_streams_kernel<il4>");
    if (rc) return rc;
    const size_t smem = sizeof(double) * cs::PR_NBUF * cs::PR_B * cs::PR_THREADS;
    cudaFuncSetAttribute(cs::prefix_p1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cs::prefix_p1_kernel<<<(unsigned)((n_streams + cs::PR_THREADS - 1) / cs::PR_THREADS), cs::PR_THREADS, smem,
                           st>>>(d_out, n_streams, ld, *plan);
    return cs::check_launch("prefix_p1_kernel");
}

// Streams plus the segmented simulator's arrival-time prefix (jffc_seg.cu).
extern "C" int cs_exp_streams_prefix_impl(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws,
                                          double* d_out, int64_t ld, int log1p_fma,
                                          const cs::PrefixPlan* plan, int il4, int whole_sm, void* stream) {
    if (n_streams <= 0 || n_draws <= 0) return 0;
    const int w = whole_sm ? 16 : 8;
    const int64_t blocks = (n_streams + w - 1) / w;
    cudaStream_t st = (cudaStream_t)stream;
#define CS_PFX(IL, W) \
    cs::exp_streams_prefix_kernel<IL, W><<<(unsigned)blocks, W * 32, 0, st>>>(d_keys, n_streams, n_draws, d_out, ld, log1p_fma, *plan)
    if (il4 && whole_sm)
        CS_PFX(true, 16);
    else if (il4)
        CS_PFX(true, 8);
    else if (whole_sm)
        CS_PFX(false, 16);
    else
        CS_PFX(false, 8);
#undef CS_PFX
    return cs::check_launch("exp_streams_prefix_kernel");
}
