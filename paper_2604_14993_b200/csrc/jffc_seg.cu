// jffc_seg.cu -- time-parallel single-chain JFFC simulation (K = 1, C <= 16).
//
// The reference's replication (sim.py:255-296) is one serial event loop.
// With one chain of capacity C it is FCFS over C identical slots: job j
// starts at st_j = max(a_j, W[0]) where W is the sorted multiset of slot
// free times (Kiefer-Wolfowitz; the per-JOB recursion of jffc_sim.cu's k1
// kernel).  This file splits every replication into S job-index SEGMENTS
// [b_s, b_{s+1}) simulated concurrently (one thread per (segment, row)):
//
//  * segment s starts from an EMPTY system at job b_s (its arrival time
//    a_{b_s} comes from an exact sequential cumsum pre-pass, the very
//    operations np.cumsum performs).  Its W is a lower bound of the true W.
//  * the true trajectory and segment s's run COUPLE at the first step j
//    where the two W's are identical (finish times, job identities and the
//    emission count): from there on every start, finish and emission is the
//    same IEEE operation on the same operands, so segment s's results are
//    bit-exact from j on.  Segment 0 is exact from job 0.
//  * an exact segment runs past its range end ("phase 2") and compares its
//    W with the next segment's checkpoints (stored during that segment's own
//    run); on a match it hands over and stops.  If it passes a whole segment
//    without coupling, that segment is marked SKIPPED and the exact one keeps
//    going (worst case: one serial replication, e.g. for rho >= 1).
//  * responses are written in completion order at the position the exact
//    run would give them: a segment's emission counter starts at the number
//    of counted jobs before b_s, which equals the exact count at the coupling
//    step (both W's hold the same jobs).  Garbage written by a segment before
//    it was coupled into is overwritten by the exact predecessor's phase 2,
//    which first waits until that segment's phase 1 is DONE.
//  * per-job sums: wait/service (sim.py:238-240) and the time integrals of
//    the number in system and in service over the windows (area, busy,
//    sim.py:224-231) are accumulated PER JOB as clipped intervals
//    [max(a, w_start), min(f, T)) instead of per event; the owner chain of
//    segments is summed by the finalize kernel.  These sums are therefore
//    reassociated (agree to ~1e-13 relative, asserted <= 1e-12 in the tests);
//    responses, their order, counted, window, lambda_eff and end_queue are
//    bit-exact.  CS_SIM_EXACT=1 selects jffc_sim.cu's serial kernel, which
//    replays the reference's event order and is bit-exact in every field.
//
// All segments of a launch must be resident at once (phase-2 waits): the
// kernel is launched cooperatively and S is chosen from the occupancy.
//
// Responses are staged per lane in a shared-memory ring and flushed as whole
// 128-byte lines, 8 threads per line with 16-byte stores (4 lines per warp
// store instruction) instead of one scattered 8-byte store per lane per job.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "cs_internal.cuh"

namespace cs {
namespace seg {

constexpr int NAGG = 6;  // wait, service, area_mid, area_end, busy, end_queue
constexpr int AG_WAIT = 0, AG_SERV = 1, AG_AMID = 2, AG_AEND = 3, AG_BUSY = 4, AG_ENDQ = 5;
// job blocks: every per-job sum is accumulated per global block of BS jobs
// (sequentially inside the block) and the blocks are added in order by the
// finalize kernel -- one fixed association for a given n, whatever the
// segment count, the batch shape or the GPU count
constexpr int64_t BS = 256;
#ifndef CS_SEG_MAXQ
#define CS_SEG_MAXQ 28
#endif
constexpr int MAXQ = CS_SEG_MAXQ;
constexpr uint32_t DONE = 1u << 30;
constexpr int32_t ST_UNKNOWN = 0, ST_SKIPPED = 1;  // status >= 2: EXACT, coupled at job (status - 2)

// checkpoint offsets from a segment's first job, in blocks: dense first
// (typical coupling within 32-300 jobs), sparser for the rho -> 1 tails
__host__ __device__ inline int64_t ck_offset(int q) {
    // 1..8, 10..16 step 2, 20..32 step 4, 40..64 step 8, 80..192 step 16 blocks
    const int m = q <= 8 ? q : q <= 12 ? 2 * q - 8 : q <= 16 ? 4 * q - 32 : q <= 20 ? 8 * q - 96 : 16 * q - 256;
    return BS * m;
}

// Segment lengths may grow linearly with the segment index: segment s gets a
// share (1 + k (2s - S + 1) / (S - 1)) / S of the row, k = -CS_SEG_SKEW/1000.
// With single-warp blocks spread over all SMs the early segments ran ahead
// (older warps, launched first) and shorter early segments helped (kernel,
// config 2 / config-5 chunk of 2048 reps: skew 0 10.99 / 17.60 ms, -100
// 10.12 / 16.87, -150 10.35 / 16.53).  With whole-SM blocks (every scheduler
// holding 4 consecutive segments of one row group) equal segments are best:
// config 2 kernel / pipelined step, skew -100 10.36 / 15.51 ms, 0 10.15 /
// 15.32, +50 10.50 / 15.61, +100 10.33 / 15.52.  Results do not depend on it.
#ifndef CS_SEG_SKEW
#define CS_SEG_SKEW 0  // per mille
#endif
__host__ __device__ inline int64_t seg_begin(int s, int S, int64_t n) {
    if (s <= 0) return 0;
    if (s >= S) return n;
    const int64_t num = (int64_t)s * (S - 1) * 1000 + (int64_t)CS_SEG_SKEW * s * (S - s);
    return (n * num / ((int64_t)S * (S - 1) * 1000)) / BS * BS;
}

struct Args {
    const cs_sim_point* pts;
    const double* rates;
    const int32_t* caps;
    const double* S;  // streams [R][lds], or the interleaved layout (il4)
    int64_t lds;
    int32_t il4;      // streams in the 32-row sector-interleaved layout (see below)
    int32_t P, R, RT, rb;
    int64_t n, warm;
    double* resp;
    int64_t ldr;
    double* busy_out;
    int32_t ldb;
    cs_rep_summary* summ;
    // workspace
    double* prefix;    // [T][S + 3]: a_{b_s} (s < S), w_start, t_mid, t_end
    double* ckf;       // [S][G][Q][CMAX + 1][32]   fin[CMAX], n_resp (bits)
    uint32_t* ckk;     // [S][G][Q][CMAX][32]       keys
    double* blk;       // [NB][NAGG][T]             per-block sums
    int32_t* status;   // [S][T]
    int32_t* spec;     // [S][T] 1 once the row's speculative phase 2 has stopped (writes visible)
    uint32_t* progress;  // [S][G]
    int32_t nseg, G, Q, cmax;
    int64_t nblk;
    unsigned long long* trace;  // development: [blocks][4] globaltimer stamps or NULL
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin-wait polls are relaxed (L2, no L1 invalidation: an acquire load
// invalidates the SM's whole L1, i.e. the stream lines the other warps on
// the SM are reading); one acquire fence follows the successful poll.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int32_t* p, int32_t v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l1_if(const void* a, bool c) {
    asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; @p prefetch.global.L1 [%0];}" ::"l"(a), "r"((unsigned)c));
}
__device__ __forceinline__ void prefetch_l2_if(const void* a, bool c) {
    asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; @p prefetch.global.L2 [%0];}" ::"l"(a), "r"((unsigned)c));
}
__device__ __forceinline__ void st_v2(double* p, double x, double y) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ double dmax0(double x) { return x > 0.0 ? x : 0.0; }
// explicit shared-window accesses (32-bit addresses: no generic-to-shared
// conversion on the per-job path)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// ---------------------------------------------------------------------------
// Pre-pass: the exact arrival times at the segment starts and at the
// warm-up / mid / last arrivals (np.cumsum order: a_0 = x_0, a_i = a_{i-1} + x_i,
// x_i = (1/lam) * S_i, sim.py:147).  One thread per row, lanes of a warp share
// streams (the P points of a rep), so the stream loads are broadcasts.
// ---------------------------------------------------------------------------
constexpr int PF_U = 16;     // values per chunk (one 128-byte line of a row)
constexpr int PF_NBUF = 24;  // chunks in flight (cp.async ring): ~4000 cycles of DRAM latency

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(32) seg_prefix_kernel(Args A) {
    // the warp's distinct stream rows (lanes of a rep share one): chunk k
    // of local row q at ring[k % NBUF][q][0..16)
    extern __shared__ __align__(16) double pf_ring[];
    const int lane = threadIdx.x;
    const int64_t T = (int64_t)A.P * A.R;
    const int64_t tid0 = (int64_t)blockIdx.x * 32 + lane;
    const bool valid = tid0 < T;
    const int64_t tid = valid ? tid0 : (int64_t)blockIdx.x * 32;
    const int32_t r = (int32_t)(tid / A.P), p = (int32_t)(tid % A.P);
    const int32_t r_lo = (int32_t)(((int64_t)blockIdx.x * 32) / A.P);
    const int64_t t_last = min((int64_t)blockIdx.x * 32 + 31, T - 1);
    const int nr = (int)(t_last / A.P) - r_lo + 1;  // distinct rows, <= 32
    const int q_own = r - r_lo;
    const double scale = __ddiv_rn(1.0, A.pts[p].lam);
    const int32_t n = (int32_t)A.n, warm = (int32_t)A.warm, mid = warm + (n - warm) / 2;
    const int S = A.nseg;
    double* out = A.prefix + tid * (S + 3);
    // recorded job indices (uniform over the grid): segment starts, warm-up,
    // mid and last arrival
    int si = 1;
    bool got_w = false, got_m = false;
    auto next_ev = [&]() {  // smallest index not recorded yet
        int32_t ev = n - 1;
        if (si < S) ev = min(ev, (int32_t)seg_begin(si, S, n));
        if (!got_w) ev = min(ev, warm);
        if (!got_m) ev = min(ev, mid);
        return ev;
    };
    auto record = [&](int32_t j, double a) {
        while (si < S && seg_begin(si, S, n) == j) {
            if (valid) out[si] = a;
            si++;
        }
        if (!got_w && j == warm) {
            if (valid) out[S] = a;
            got_w = true;
        }
        if (!got_m && j == mid) {
            if (valid) out[S + 1] = a;
            got_m = true;
        }
        if (j == n - 1 && valid) out[S + 2] = a;
    };
    // one sequential cumsum (the DADD chain is the critical path); stream
    // lines staged NBUF-1 chunks ahead through cp.async, 8 lanes per line
    const int nchunks = (n + PF_U - 1) / PF_U;
    const int piece = lane & 7;
    auto issue = [&](int k) {
        if (k < nchunks) {
            for (int q0 = 0; q0 < nr; q0 += 4) {
                const int q = q0 + (lane >> 3);
                if (q < nr) {
                    const double* src = A.S + (int64_t)(r_lo + q) * A.lds + (int64_t)k * PF_U + 2 * piece;
                    cp_async16(pf_ring + ((size_t)(k % PF_NBUF) * nr + q) * PF_U + 2 * piece, src);
                }
            }
        }
        cp_async_commit();
    };
    for (int k = 0; k < PF_NBUF - 1; k++) issue(k);
    // x[] holds chunk k already scaled (the DMULs and shared loads of chunk
    // k+1 overlap the DADD chain of chunk k)
    double x[PF_U];
    cp_async_wait<PF_NBUF - 2>();
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PF_U; u++) x[u] = __dmul_rn(scale, pf_ring[(size_t)q_own * PF_U + u]);
    double a = x[0];
    if (valid) out[0] = a;
    int32_t ev = next_ev();
    for (int k = 0; k < nchunks; k++) {
        __syncwarp();  // every lane is done with the slot chunk k-1 used
        issue(k + PF_NBUF - 1);
        cp_async_wait<PF_NBUF - 2>();  // chunk k+1 landed
        __syncwarp();
        double y[PF_U];
        const double* c = pf_ring + ((size_t)((k + 1) % PF_NBUF) * nr + q_own) * PF_U;
#pragma unroll
        for (int u = 0; u < PF_U; u++) y[u] = c[u];
        const int32_t j0 = k * PF_U;
        if (j0 > 0 && ev >= j0 + PF_U) {  // no recorded index in this chunk: plain cumsum
#pragma unroll
            for (int u = 0; u < PF_U; u++) a = __dadd_rn(a, x[u]);
        } else {
#pragma unroll
            for (int u = 0; u < PF_U; u++) {
                const int32_t j = j0 + u;
                if (j > 0) a = __dadd_rn(a, x[u]);
                if (j == ev) {
                    record(j, a);
                    ev = j == n - 1 ? INT32_MAX : next_ev();
                }
            }
        }
#pragma unroll
        for (int u = 0; u < PF_U; u++) x[u] = __dmul_rn(scale, y[u]);
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// The segment kernel.  Block = one warp = 32 rows (lanes) of one segment.
// ---------------------------------------------------------------------------
enum { PH_A = 0, PH_B = 1, PH_C = 2 };  // before warm-up / first / second half of the window

// <= 128 registers: 16 warps per SM (measured against 20 and 24 warps with
// spills: 13.6 / 14.7 / 17.8 ms on config 2; without the bound ptxas took 144)
#ifndef CS_SEG_UNROLL
#define CS_SEG_UNROLL 4  // measured on config 2: 1 11.77, 2 11.83, 4 11.10 ms
#endif
constexpr int SEG_UNROLL = CS_SEG_UNROLL;  // jobs per trip of the step loops
// Stream layouts.  Row-major [R][lds] serves warps whose lanes share a few
// rows (P >= 16 points per stream: one L1 line per row feeds 16 jobs).  With
// few points per stream every lane reads its own row and 32 rows x 2 streams
// of live 128-byte lines per warp overflow L1 at 16 warps per SM; the
// interleaved layout (cs_sim_streams picks it) stores 32 consecutive rows as
// one group with each row's values in 4-value sectors side by side:
// element (r, i) at (r / 32) * 32 * lds + (i / 4) * 128 + (r % 32) * 4 + i % 4,
// so a warp's step reads 8 lines, each consumed within 4 steps.
__device__ __forceinline__ int64_t il4_off(int64_t i) { return ((i >> 2) << 7) + (i & 3); }

// One warp's shared memory (a block holds SEG_WPB of them).
template <int CMAX>
struct SegSmem {
    double ring[32 * 33];  // response ring: element (pos, lane) at [pos & 31][lane], row pitch 33 doubles
    double rbuf[CMAX * 32];  // response of the job holding slot id
    double* row[32];         // response row of each lane
    int4 meta[32];           // per-lane flush line: start, first, end, has
};

// Blocks of SEG_WPB warps (one block fills an SM's register file at 128
// registers): a launch of U units occupies ceil(U / 16) whole SMs, every
// scheduler holding 4 units -- 4 consecutive segments of one row group when
// S = 4 -- instead of U single-warp blocks spread 3 or 4 to a scheduler over
// all SMs (the kernel ends with the 4-warp schedulers either way; the SMs it
// does not need stay free for the next sweep's streams).
constexpr int SEG_WPB = 16;

template <int CMAX, bool IL4>
__global__ void __launch_bounds__(32 * SEG_WPB, 1) jffc_seg_kernel(Args A) {
    constexpr int ID_BITS = CMAX <= 8 ? 3 : 4;
    constexpr uint32_t DUMMY = 0x80000000u;  // an initially idle slot, not a job
    constexpr uint32_t J_MASK = (1u << (31 - ID_BITS)) - 1;
    constexpr uint32_t ID_MASK = (1u << ID_BITS) - 1;
    constexpr int FCK = CMAX + 1;
    constexpr unsigned FULL = 0xffffffffu;

    extern __shared__ __align__(16) unsigned char seg_smem[];
    const int wib = threadIdx.x >> 5;
    SegSmem<CMAX>& wsm = reinterpret_cast<SegSmem<CMAX>*>(seg_smem)[wib];
    double* const sh_ring = wsm.ring;
    double* const sh_rbuf = wsm.rbuf;
    double** const sh_row = wsm.row;
    int4* const sh_meta = wsm.meta;

    const int lane = threadIdx.x & 31;
    const int S = A.nseg, G = A.G, Q = A.Q;
    // scheduler z = 4 * block + (warp & 3) hosts units 4z .. 4z + 3 (unit = g * S + s)
    const int64_t uo = ((int64_t)blockIdx.x * 4 + (wib & 3)) * 4 + (wib >> 2);
    if (uo >= (int64_t)S * G) return;
    const int s = (int)(uo % S), g = (int)(uo / S);
    const int64_t T = (int64_t)A.P * A.R;
    const int64_t tid = (int64_t)g * 32 + lane;
    const bool valid = tid < T;
    const int64_t te = valid ? tid : 0;
    const int32_t r = (int32_t)(te / A.P), p = (int32_t)(te % A.P);
    const int64_t o = (int64_t)p * A.RT + A.rb + r;
    const int64_t n = A.n, warm = A.warm, mid = warm + (n - warm) / 2;
    const cs_sim_point pt = A.pts[p];
    const double inv_mu = __ddiv_rn(1.0, A.rates[pt.chain_base]);
    const int32_t cap = A.caps[pt.chain_base];
    const double scale = __ddiv_rn(1.0, pt.lam);
    const double* __restrict__ gap =
        IL4 ? A.S + (int64_t)(r >> 5) * 32 * A.lds + (r & 31) * 4 : A.S + (int64_t)r * A.lds;
    const double* __restrict__ szs = gap + n;  // row-major only
    const double* pre = A.prefix + te * (S + 3);
    const double Ws = pre[S], Tm = pre[S + 1], Te = pre[S + 2];
    sh_row[lane] = (A.resp && valid) ? A.resp + o * A.ldr : nullptr;
    const bool writes = A.resp != nullptr;
    double* blk = A.blk + te;

    const int64_t b = seg_begin(s, S, n), e = seg_begin(s + 1, S, n);
    const int unit = s * G + g;
    unsigned long long* tr = A.trace ? A.trace + (int64_t)unit * 4 : nullptr;
    if (tr && lane == 0) tr[0] = gtimer();

    // ---- lane state
    double fin[CMAX];
    uint32_t key[CMAX];
#pragma unroll
    for (int k = 0; k < CMAX; k++) {
        fin[k] = k < cap ? -INFINITY : INFINITY;
        key[k] = DUMMY | (uint32_t)k;
    }
    const uint32_t rbuf_a = smem_addr(sh_rbuf + lane);  // slot id k at + k * 256
    const uint32_t ring_a = smem_addr(sh_ring + lane);  // position p at + (p & 31) * 264
    // positions are < n - warm < 2^27: 32-bit
    int32_t n_resp = (int32_t)(b > warm ? b - warm : 0);  // counted jobs before b = the exact position at coupling
    int32_t fl_lo = n_resp;                               // first position not yet flushed
    double ag[NAGG];
#pragma unroll
    for (int k = 0; k < NAGG; k++) ag[k] = 0.0;
    bool act = valid;  // lane simulates / writes / accumulates

    int32_t j = (int32_t)b;
    const int32_t warm_key = (int32_t)warm << ID_BITS;
    double a = pre[s];  // a_b
    const double* __restrict__ gp = gap + b + 1;  // gap of job j+1 (row-major)
    const double* __restrict__ sp = szs + b;      // size of job j (row-major)
    double g1, g2, sz, sz1;
    if (IL4) {
        g1 = __ldg(gap + il4_off(b + 1));
        g2 = __ldg(gap + il4_off(b + 2));
        sz = __ldg(gap + il4_off(n + b));
        sz1 = __ldg(gap + il4_off(n + b + 1));
    } else {
        g1 = __ldg(gp), g2 = __ldg(gp + 1), sz = __ldg(sp), sz1 = __ldg(sp + 1);
    }
    __syncwarp();

    // ---- helpers (warp-uniform control flow) ---------------------------
    auto ring_put = [&](int32_t pos, double v) { sts_f64(ring_a + (uint32_t)(pos & 31) * 264u, v); };
    // flush complete lines (final: also the trailing partial line) of the
    // lanes in `who`; lines go out 4 per warp instruction, 8 threads x 16 B
    // each; the first and last line of a lane's range element by element.
    auto flush = [&](bool final, bool who) {
        for (;;) {
            const int32_t ls = fl_lo & ~15;
            const int32_t hi_full = ls + 16;
            const bool has = who && (final ? fl_lo < n_resp : hi_full <= n_resp);
            const int32_t hi = hi_full < n_resp ? hi_full : n_resp;
            const unsigned mask = __ballot_sync(FULL, has);
            if (!mask) break;
            if (writes) {
                sh_meta[lane] = make_int4(ls, fl_lo, hi, has ? 1 : 0);
                __syncwarp();
                const int grp = lane >> 3, c = lane & 7;
#pragma unroll 1
                for (int L0 = 0; L0 < 32; L0 += 4) {
                    if (((mask >> L0) & 15u) == 0) continue;
                    const int L = L0 + grp;
                    const int4 md = sh_meta[L];
                    if (md.w) {
                        const int32_t p0 = md.x + 2 * c;
                        const double2 v = make_double2(sh_ring[(p0 & 31) * 33 + L], sh_ring[((p0 + 1) & 31) * 33 + L]);
                        double* dst = sh_row[L] + p0;
                        if (p0 >= md.y && p0 + 1 < md.z) {
                            st_v2(dst, v.x, v.y);
                        } else {
                            if (p0 >= md.y && p0 < md.z) dst[0] = v.x;
                            if (p0 + 1 >= md.y && p0 + 1 < md.z) dst[1] = v.y;
                        }
                    }
                }
                __syncwarp();
            }
            if (has) fl_lo = hi;
        }
    };
    // the next stream lines into L1 and a few ahead into L2, once per 16 jobs
    auto prefetch = [&]() {
        if (IL4) {
            prefetch_l2_if(gap + il4_off(n + j + 80), true);
            prefetch_l2_if(gap + il4_off(j + 80), true);
        } else {
            prefetch_l1_if(sp + 16, true);
            prefetch_l1_if(gp + 16, true);
            prefetch_l2_if(sp + 80, true);
            prefetch_l2_if(gp + 80, true);
        }
    };

    // one job (step j) of the recursion; PH picks the sums' form, act_l
    // predicates emission and sums on the lane's active flag
    // (every lane steps; an inactive lane's results are never stored: its
    // flushes and block sums are gated on its active flag)
    auto step = [&](auto ph_tag) {
        constexpr int PH = decltype(ph_tag)::value;
        const double m = fin[0];
        const uint32_t k0 = key[0];
        const uint32_t ra = rbuf_a + (k0 & ID_MASK) * 256u;
        const double rv = lds_f64(ra);  // response of the slot's previous job
        const double aj = a;
        const double st = m <= aj ? aj : m;
        const double d = __dmul_rn(sz, inv_mu);
        const double f = __dadd_rn(st, d);
        const double rr = __dsub_rn(f, aj);
        // a real job (dummies are negative) of index >= warm: key >= warm << ID_BITS
        const bool counted = (int32_t)k0 >= warm_key;
        ring_put(n_resp, rv);  // slot n_resp is free (< 32 unflushed): kept only if counted
        n_resp += counted;
        sts_f64(ra, rr);
        // remove W[0], insert (f, j): equal finish goes after (larger job index)
        const uint32_t nk = ((uint32_t)j << ID_BITS) | (k0 & ID_MASK);
        bool lt[CMAX];
#pragma unroll
        for (int k = 0; k < CMAX - 1; k++) lt[k] = fin[k + 1] <= f;
        lt[CMAX - 1] = false;
#pragma unroll
        for (int k = 0; k < CMAX; k++) {
            const bool before = k == 0 ? true : lt[k - 1];
            const double nf = lt[k] ? fin[k + 1 < CMAX ? k + 1 : k] : (before ? f : fin[k]);
            const uint32_t nkk = lt[k] ? key[k + 1 < CMAX ? k + 1 : k] : (before ? nk : key[k]);
            fin[k] = nf;
            key[k] = nkk;
        }
        // next job's inputs (stream rows are padded: cursors may run past n)
        a = __dadd_rn(a, __dmul_rn(scale, g1));
        g1 = g2;
        sz = sz1;
        if (IL4) {
            g2 = __ldg(gap + il4_off(j + 3));
            sz1 = __ldg(gap + il4_off(n + j + 2));
        } else {
            gp++;
            sp++;
            g2 = __ldg(gp + 1);
            sz1 = __ldg(sp + 1);
        }
        j++;
        // per-job sums over the windows (interval [a, f) in system, [st, f)
        // in service, clipped to [w_start, T]); jobs that end past the
        // window's end (rare: in system at mid / at the last arrival) take
        // the clipped form, the rest the plain one
        if (PH == PH_A) {  // a <= w_start: clipped on both sides
            {
                const bool fe = f <= Te;
                const double he = fe ? f : Te;
                const double hm = f <= Tm ? f : Tm;
                const double lo = st >= Ws ? st : Ws;
                ag[AG_AEND] = __dadd_rn(ag[AG_AEND], dmax0(__dsub_rn(he, Ws)));
                ag[AG_AMID] = __dadd_rn(ag[AG_AMID], dmax0(__dsub_rn(hm, Ws)));
                ag[AG_BUSY] = __dadd_rn(ag[AG_BUSY], dmax0(__dsub_rn(he, lo)));
                ag[AG_ENDQ] += st > Te ? 1.0 : 0.0;
            }
        } else {
            const bool slow = f > (PH == PH_B ? Tm : Te);
            if (__any_sync(FULL, slow)) {
                {
                    const bool fe = f <= Te;
                    ag[AG_WAIT] = __dadd_rn(ag[AG_WAIT], __dsub_rn(st, aj));
                    ag[AG_SERV] = __dadd_rn(ag[AG_SERV], d);
                    ag[AG_AEND] = __dadd_rn(ag[AG_AEND], fe ? rr : __dsub_rn(Te, aj));
                    ag[AG_BUSY] = __dadd_rn(ag[AG_BUSY], fe ? __dsub_rn(f, st) : dmax0(__dsub_rn(Te, st)));
                    if (PH == PH_B) ag[AG_AMID] = __dadd_rn(ag[AG_AMID], f <= Tm ? rr : __dsub_rn(Tm, aj));
                    ag[AG_ENDQ] += st > Te ? 1.0 : 0.0;
                }
            } else {  // f <= T: the plain intervals
                ag[AG_WAIT] = __dadd_rn(ag[AG_WAIT], __dsub_rn(st, aj));
                ag[AG_SERV] = __dadd_rn(ag[AG_SERV], d);
                ag[AG_AEND] = __dadd_rn(ag[AG_AEND], rr);
                ag[AG_BUSY] = __dadd_rn(ag[AG_BUSY], __dsub_rn(f, st));
                if (PH == PH_B) ag[AG_AMID] = __dadd_rn(ag[AG_AMID], rr);
            }
        }
    };
    using TA = std::integral_constant<int, PH_A>;
    using TB = std::integral_constant<int, PH_B>;
    using TC = std::integral_constant<int, PH_C>;
    // up to 16 steps to jn (a multiple of 16 or the range end), split at the
    // warm-up and mid indices
    auto run_to = [&](int64_t jn) {
        while (j < jn) {
            if (j < warm) {
                const int cnt = (int)((warm < jn ? warm : jn) - j);
#pragma unroll SEG_UNROLL
                for (int k = 0; k < cnt; k++) step(TA());
            } else if (j < mid) {
                const int cnt = (int)((mid < jn ? mid : jn) - j);
#pragma unroll SEG_UNROLL
                for (int k = 0; k < cnt; k++) step(TB());
            } else {
                const int cnt = (int)(jn - j);
#pragma unroll SEG_UNROLL
                for (int k = 0; k < cnt; k++) step(TC());
            }
        }
    };
    auto drain = [&](bool act_l) {  // the remaining slots complete in sorted order
#pragma unroll
        for (int k = 0; k < CMAX; k++) {
            const uint32_t kk = key[k];
            const bool counted = act_l && !(kk & DUMMY) && fin[k] < INFINITY &&
                                 (int64_t)((kk >> ID_BITS) & J_MASK) >= warm;
            if (counted) ring_put(n_resp, lds_f64(rbuf_a + (kk & ID_MASK) * 256u));
            n_resp += counted;
        }
    };
    // the block that just ended (j a multiple of BS, or n)
    auto put_block = [&](bool act_l) {
        if (act_l) {
            double* bp = blk + (int64_t)((j - 1) / (int32_t)BS) * NAGG * T;
#pragma unroll
            for (int k = 0; k < NAGG; k++) bp[k * T] = ag[k];
        }
#pragma unroll
        for (int k = 0; k < NAGG; k++) ag[k] = 0.0;
    };

    // ---- phase 1: own range [b, e); checkpoints (state before job
    // b + ck_offset(q)) for the predecessor's coupling test
    double* ckf = A.ckf + (((int64_t)s * G + g) * Q) * FCK * 32 + lane;
    uint32_t* ckk = A.ckk + (((int64_t)s * G + g) * Q) * CMAX * 32 + lane;
    {
        int q = 1;
        int64_t next_ck = Q >= 1 ? b + ck_offset(1) : INT64_MAX;
        while (j < e) {
            const int64_t jn = (j + 16 < e) ? j + 16 : e;  // b is a multiple of BS
            prefetch();
            run_to(jn);
            flush(false, act);
            if (j % (int32_t)BS == 0 || j == n) put_block(act);
            if (j == next_ck) {
                double* cf = ckf + (int64_t)(q - 1) * FCK * 32;
                uint32_t* ck = ckk + (int64_t)(q - 1) * CMAX * 32;
#pragma unroll
                for (int k = 0; k < CMAX; k++) {
                    cf[k * 32] = fin[k];
                    ck[k * 32] = key[k];
                }
                cf[CMAX * 32] = __longlong_as_double((int64_t)n_resp);
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(A.progress + unit, (uint32_t)q);
                q++;
                next_ck = q <= Q ? b + ck_offset(q) : INT64_MAX;
            }
        }
    }
    if (tr && lane == 0) tr[1] = gtimer();
    if (e == n) {  // the last segment finishes the row
        drain(act);
        flush(true, act);
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(A.progress + unit, DONE | (uint32_t)Q);
        if (tr && lane == 0) tr[2] = tr[3] = gtimer();
        return;
    }
    flush(true, act);  // everything this segment emitted in its own range
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(A.progress + unit, DONE | (uint32_t)Q);

    // ---- phase 2, speculative: every lane runs on past its range at once,
    // as if this segment were exact, and polls its verdict every chunk (set
    // by the exact run that couples into this segment -- exact -- or that
    // passes through it -- SKIPPED).  If the verdict is exact, the run from
    // here on is exact too (this segment's trajectory has been the true one
    // since the coupling point).  If SKIPPED, the lane stops; everything it
    // wrote past its range is rewritten by the exact run, which enters the
    // next range only after this lane's spec flag (all its writes visible).
    // The decisions this lane takes about later segments (passed through:
    // SKIPPED; coupled into: exact) are released only once its own verdict is
    // exact.  Waits only run forward (frontier gating, spec flags of later
    // segments; the last segment has no phase 2): no deadlock.  Round 1's
    // form waited for the verdict first, which serialised the hand-overs of
    // a row into a chain (the kernel's last 1.5 ms on config 2).
    int32_t stv = !valid ? ST_SKIPPED : s == 0 ? 2 : ST_UNKNOWN;
    act = valid;
    int32_t skip_to = s + 1;           // segments [s + 1, skip_to) passed through (unreleased)
    int32_t hand_t = -1, hand_j = 0;   // coupled into hand_t at job hand_j (unreleased)
    bool flagged = false;              // spec flag set
    int32_t* const spec_s = A.spec + (int64_t)s * T + tid;
    auto release_pending = [&]() {     // this lane's verdict is exact
        for (int32_t u = s + 1; u < skip_to; u++) st_release(A.status + (int64_t)u * T + tid, ST_SKIPPED);
        skip_to = s + 1;
        if (hand_t >= 0) st_release(A.status + (int64_t)hand_t * T + tid, (int32_t)(2 + hand_j));
        hand_t = -1;
    };
    auto stop_lanes = [&](bool who) {  // warp-uniform call: the lanes in `who` stop
        __threadfence();
        if (who && valid && !flagged) {
            st_release(spec_s, 1);
            flagged = true;
        }
    };
    auto poll = [&]() {  // warp-uniform call
        bool now_skipped = false;
        if (act && stv == ST_UNKNOWN) {
            stv = ld_relaxed(A.status + (int64_t)s * T + tid);
            if (stv >= 2) {
                fence_acquire();
                release_pending();
            } else if (stv == ST_SKIPPED) {
                act = false;
                now_skipped = true;
            }
        }
        if (__any_sync(FULL, now_skipped)) stop_lanes(now_skipped);
    };
    if (tr && lane == 0) tr[2] = gtimer();
    int t = s + 1;
    while (__any_sync(FULL, act)) {
        // Entering segment t's range while t may still run its phase 1: every
        // write into its range must land after t's own write of the same
        // place.  t publishes at checkpoint q (release) its blocks up to job
        // bt + ck_offset(q) and, per row, its emission count there -- the
        // complete lines below it are flushed; DONE publishes everything.
        // So: run a chunk only up to t's latest published job (blocks and
        // checkpoints there exist), flush only lines below t's flushed
        // frontier, and hand over at a coupling only once t has flushed past
        // our emissions (t's still-unflushed pre-coupling values would
        // otherwise land after ours).  t never waits for us: no deadlock.
        const uint32_t* prog = A.progress + (int64_t)t * G + g;
        const int64_t bt = seg_begin(t, S, n), et = seg_begin(t + 1, S, n);
        const double* tcf = A.ckf + (((int64_t)t * G + g) * Q) * FCK * 32 + lane;
        const uint32_t* tck = A.ckk + (((int64_t)t * G + g) * Q) * CMAX * 32 + lane;
        uint32_t qt = 0;                 // t's latest checkpoint seen
        int64_t jt = bt;                 // t's blocks / checkpoints exist up to here
        int32_t ft = INT32_MIN;          // t's flushed frontier for this lane's row
        auto refresh = [&]() {
            const uint32_t pv = ld_relaxed(prog);
            if (pv & DONE) {
                if (jt != INT64_MAX) {
                    fence_acquire();
                    jt = INT64_MAX;
                    ft = INT32_MAX;
                }
            } else if (pv > qt) {
                fence_acquire();
                qt = pv;
                jt = bt + ck_offset((int)qt);
                ft = (int32_t)__double_as_longlong(__ldcg(tcf + (int64_t)(qt - 1) * FCK * 32 + CMAX * 32)) & ~15;
            }
        };
        auto wait_for = [&](auto ok) {  // warp-uniform: until every lane's condition holds
            if (__all_sync(FULL, ok())) return;
            refresh();
            while (!__all_sync(FULL, ok())) {
                __nanosleep(256);
                refresh();
            }
        };
        int q = 1;
        int64_t next_ck = Q >= 1 ? bt + ck_offset(1) : INT64_MAX;
        while (j < et && __any_sync(FULL, act)) {
            const int64_t jn = (j + 16 < et) ? j + 16 : et;
            wait_for([&] { return jn <= jt; });
            prefetch();
            run_to(jn);
            wait_for([&] { return !act || (n_resp & ~15) <= ft; });
            flush(false, act);
            if (j % (int32_t)BS == 0 || j == n) put_block(act);
            if (j == next_ck) {
                bool same = act;
                if (act) {
                    const double* cf = tcf + (int64_t)(q - 1) * FCK * 32;
                    const uint32_t* ck = tck + (int64_t)(q - 1) * CMAX * 32;
#pragma unroll
                    for (int k = 0; k < CMAX; k++)
                        same = same && __ldcg(cf + k * 32) == fin[k] &&
                               ((__ldcg(ck + k * 32) ^ key[k]) & ~ID_MASK) == 0;
                    same = same && __double_as_longlong(__ldcg(cf + CMAX * 32)) == (int64_t)n_resp;
                }
                if (__any_sync(FULL, same)) {
                    wait_for([&] { return !same || n_resp <= ft; });
                    flush(true, same);  // our emissions before the hand-over
                    if (same) {
                        if (stv >= 2) {
                            release_pending();
                            st_release(A.status + (int64_t)t * T + tid, (int32_t)(2 + j));
                        } else {
                            hand_t = t;
                            hand_j = (int32_t)j;
                        }
                        act = false;
                    }
                    stop_lanes(same);
                }
                q++;
                next_ck = q <= Q ? bt + ck_offset(q) : INT64_MAX;
            }
            poll();
        }
        if (j == et && __any_sync(FULL, act)) {
            wait_for([&] { return jt == INT64_MAX; });  // t's range entirely ours from here
            if (et == n) {  // ran through the last segment: these lanes finish the row
                drain(act);
                flush(true, act);
                const bool fin_now = act;
                act = false;
                stop_lanes(fin_now);
            } else {
                if (act) {
                    skip_to = t + 1;
                    if (stv >= 2) release_pending();
                }
                // t's own speculative writes past its range land before ours
                const int32_t* spec_t = A.spec + (int64_t)t * T + tid;
                while (!__all_sync(FULL, !act || ld_relaxed(spec_t) != 0)) {
                    __nanosleep(256);
                    poll();
                }
                fence_acquire();
                t++;
            }
        }
    }
    // this lane has stopped: flag it, then settle its decisions once its own
    // verdict is known (they only matter if it is exact)
    stop_lanes(true);
    while (__any_sync(FULL, valid && stv == ST_UNKNOWN && (hand_t >= 0 || skip_to > s + 1))) {
        if (valid && stv == ST_UNKNOWN) {
            stv = ld_relaxed(A.status + (int64_t)s * T + tid);
            if (stv >= 2) {
                fence_acquire();
                release_pending();
            }
        }
        __nanosleep(256);
    }
    if (tr && lane == 0) tr[3] = gtimer();
}

// ---------------------------------------------------------------------------
// Finalize: per row, add the block sums in block order (every block was
// written last by the exact run over it) and form the RepResult fields as
// sim.py:298-324 does.
// ---------------------------------------------------------------------------
__global__ void seg_finalize_kernel(Args A) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T = (int64_t)A.P * A.R;
    if (tid >= T) return;
    const int S = A.nseg;
    const int32_t r = (int32_t)(tid / A.P), p = (int32_t)(tid % A.P);
    const int64_t o = (int64_t)p * A.RT + A.rb + r;
    const int64_t n = A.n, warm = A.warm;
    const double* pre = A.prefix + tid * (S + 3);
    double ag[NAGG];
    for (int k = 0; k < NAGG; k++) ag[k] = 0.0;
    const double* bp = A.blk + tid;
    // the blocks in order; 8 blocks' loads issued ahead of their adds (the
    // add chains are sequential, the loads are not)
    constexpr int KB = 8;
    int64_t kb = 0;
    for (; kb + KB <= A.nblk; kb += KB) {
        double v[KB][NAGG];
#pragma unroll
        for (int u = 0; u < KB; u++)
#pragma unroll
            for (int k = 0; k < NAGG; k++) v[u][k] = __ldcs(bp + ((kb + u) * NAGG + k) * T);
#pragma unroll
        for (int u = 0; u < KB; u++)
#pragma unroll
            for (int k = 0; k < NAGG; k++) ag[k] = __dadd_rn(ag[k], v[u][k]);
    }
    for (; kb < A.nblk; kb++)
        for (int k = 0; k < NAGG; k++) ag[k] = __dadd_rn(ag[k], bp[(kb * NAGG + k) * T]);
    const double w_start = pre[S], t_mid = pre[S + 1], t_end = pre[S + 2];
    cs_rep_summary out;
    const double window = __dsub_rn(t_end, w_start);
    out.wait_sum = ag[AG_WAIT];
    out.service_sum = ag[AG_SERV];
    out.counted = n - warm;
    out.window_s = window;
    const double area_end = ag[AG_AEND], area_mid = ag[AG_AMID];
    if (window > 0.0) {
        out.mean_occupancy = __ddiv_rn(area_end, window);
        out.lambda_effective = __ddiv_rn((double)(n - warm), window);
    } else {
        out.mean_occupancy = NAN;
        out.lambda_effective = NAN;
    }
    out.occ_first_half = t_mid > w_start ? __ddiv_rn(area_mid, __dsub_rn(t_mid, w_start)) : NAN;
    out.occ_second_half =
        t_end > t_mid ? __ddiv_rn(__dsub_rn(area_end, area_mid), __dsub_rn(t_end, t_mid)) : NAN;
    out.end_queue_len = (int64_t)ag[AG_ENDQ];
    out.w_start = w_start;
    out.t_mid = t_mid;
    out.area_mid = area_mid;
    out.t_end = t_end;
    out.area_end = area_end;
    out.resp_sum = NAN;  // filled by the statistics pass (numpy pairwise order)
    out.resp_mean = NAN;
    A.summ[o] = out;
    A.busy_out[o * A.ldb] = ag[AG_BUSY];
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct Plan {
    int S, G, Q, cmax;
    int64_t T, nblk;
    size_t off_prefix, off_ckf, off_ckk, off_blk, off_status, off_spec, off_progress, bytes;
};

static int pick_cmax(int32_t max_cap) { return max_cap <= 4 ? 4 : max_cap <= 7 ? 7 : max_cap <= 8 ? 8 : 16; }

template <int CMAX, bool IL4>
static int max_resident_blocks() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (dev < 64 && cached[dev]) return cached[dev];
    int per_sm = 0, sms = 0;
    const int smem = (int)(sizeof(SegSmem<CMAX>) * SEG_WPB);
    if (cudaFuncSetAttribute(jffc_seg_kernel<CMAX, IL4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jffc_seg_kernel<CMAX, IL4>, 32 * SEG_WPB, smem) !=
            cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const int v = per_sm * SEG_WPB * sms;  // resident units (warps)
    if (dev < 64) cached[dev] = v;
    return v;
}

static int resident_blocks(int cmax) {
    switch (cmax) {
        case 4: return std::min(max_resident_blocks<4, false>(), max_resident_blocks<4, true>());
        case 7: return std::min(max_resident_blocks<7, false>(), max_resident_blocks<7, true>());
        case 8: return std::min(max_resident_blocks<8, false>(), max_resident_blocks<8, true>());
        default: return std::min(max_resident_blocks<16, false>(), max_resident_blocks<16, true>());
    }
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// S (segments per row): as many as keep every segment of the launch resident
// (phase-2 waits), segments of >= 8 blocks.  The results do not depend on S.
static Plan make_plan(int32_t P, int32_t R, int32_t max_cap, int64_t n) {
    Plan pl{};
    pl.cmax = pick_cmax(max_cap);
    pl.T = (int64_t)P * R;
    pl.G = (int)((pl.T + 31) / 32);
    pl.nblk = (n + BS - 1) / BS;
    const int cap_blocks = resident_blocks(pl.cmax);
    const int s_fit = pl.G > 0 && cap_blocks > 0 ? std::max(1, cap_blocks / pl.G) : 1;
    const int s_len = (int)std::max<int64_t>(1, std::min<int64_t>(64, n / (8 * BS)));
    int S = std::min(s_fit, s_len);
    if (const char* e = getenv("CS_SEG_S")) S = std::max(1, std::min(std::min(s_fit, s_len), atoi(e)));
    pl.S = S;
    int64_t lmin = n;
    for (int s = 0; s < S; s++) lmin = std::min(lmin, seg_begin(s + 1, S, n) - seg_begin(s, S, n));
    int Q = 0;
    while (Q < MAXQ && ck_offset(Q + 1) < lmin) Q++;
    pl.Q = Q;
    size_t off = 0;
    pl.off_prefix = off;
    off = align256(off + sizeof(double) * pl.T * (S + 3));
    pl.off_ckf = off;
    off = align256(off + sizeof(double) * (size_t)S * pl.G * std::max(Q, 1) * (pl.cmax + 1) * 32);
    pl.off_ckk = off;
    off = align256(off + sizeof(uint32_t) * (size_t)S * pl.G * std::max(Q, 1) * pl.cmax * 32);
    pl.off_blk = off;
    off = align256(off + sizeof(double) * (size_t)pl.nblk * NAGG * pl.T);
    pl.off_status = off;
    off = align256(off + sizeof(int32_t) * (size_t)S * pl.T);
    pl.off_spec = off;
    off = align256(off + sizeof(int32_t) * (size_t)S * pl.T);
    pl.off_progress = off;
    off = align256(off + sizeof(uint32_t) * (size_t)S * pl.G);
    pl.bytes = off;
    return pl;
}

template <int CMAX, bool IL4>
static int launch(const Plan& pl, Args A, cudaStream_t st) {
    const int units = pl.S * pl.G;
    const int blocks = (units + SEG_WPB - 1) / SEG_WPB;
    const size_t smem = sizeof(SegSmem<CMAX>) * SEG_WPB;
    cudaFuncSetAttribute(jffc_seg_kernel<CMAX, IL4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const bool trace = getenv("CS_SEG_TRACE") != nullptr;  // development timeline (stderr)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (trace) {
        cudaMalloc(&A.trace, sizeof(unsigned long long) * 4 * units);
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, st);
    }
    if (pl.S > 1) {  // phase-2 waits need every segment resident
        void* params[] = {&A};
        const cudaError_t e =
            cudaLaunchCooperativeKernel((const void*)jffc_seg_kernel<CMAX, IL4>, dim3(blocks), dim3(32 * SEG_WPB),
                                        params, smem, st);
        if (e != cudaSuccess) return check_cuda(e, "jffc_seg_kernel (cooperative launch)");
    } else {
        jffc_seg_kernel<CMAX, IL4><<<blocks, 32 * SEG_WPB, smem, st>>>(A);
    }
    int rc = check_launch("jffc_seg_kernel");
    if (rc) return rc;
    if (trace) {
        cudaEventRecord(ev1, st);
        cudaEventSynchronize(ev1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        fprintf(stderr, "jffc_seg_kernel %.3f ms\n", ms);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        std::vector<unsigned long long> h((size_t)4 * units);
        cudaMemcpyAsync(h.data(), A.trace, h.size() * 8, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        cudaFree(A.trace);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < units; b++) t0 = std::min(t0, h[4 * b]);
        for (int s = 0; s < pl.S; s++) {
            std::vector<double> v[4];
            for (int g = 0; g < pl.G; g++)
                for (int k = 0; k < 4; k++) v[k].push_back((h[4 * ((size_t)s * pl.G + g) + k] - t0) * 1e-6);
            fprintf(stderr, "seg %d:", s);
            for (int k = 0; k < 4; k++) {
                std::sort(v[k].begin(), v[k].end());
                fprintf(stderr, " [%s %.3f/%.3f/%.3f ms]", k == 0 ? "start" : k == 1 ? "ph1end" : k == 2 ? "ph2start" : "end",
                        v[k][0], v[k][v[k].size() / 2], v[k].back());
            }
            fprintf(stderr, "\n");
        }
    }
    seg_finalize_kernel<<<(int)((pl.T + 63) / 64), 64, 0, st>>>(A);  // >= 2 blocks per SM on config 2
    return check_launch("seg_finalize_kernel");
}

}  // namespace seg
}  // namespace cs

// Workspace bytes of the segmented path (0 when it does not apply).
extern "C" int64_t cs_seg_workspace_bytes_impl(int32_t P, int32_t R, int32_t max_chains, int32_t max_cap,
                                               int64_t n) {
    if (max_chains > 1 || max_cap > 16 || n >= (1ll << 27) || P <= 0 || R <= 0) return 0;
    return (int64_t)cs::seg::make_plan(P, R, max_cap, n).bytes;
}

// The arrival-time prefix plan for the fused stream kernel (exp_stream.cu):
// rows of the workspace's prefix table, recorded at the segment starts and
// the warm-up / mid / last arrivals.  Returns false when the fused path does
// not apply (more than 32 points per stream or more events than the plan holds).
extern "C" bool cs_seg_prefix_plan(int32_t P, int32_t R, int32_t max_cap, int64_t n, int64_t warm,
                                   const cs_sim_point* d_points, void* d_ws, cs::PrefixPlan* pp) {
    using namespace cs::seg;
    const Plan pl = make_plan(P, R, max_cap, n);
    if (P > 32 * cs::PrefixPlan::MAXP32 || pl.S + 3 > cs::PrefixPlan::MAXEV) return false;
    const int S = pl.S;
    const int64_t mid = warm + (n - warm) / 2;
    std::vector<std::pair<int64_t, int>> ev;
    for (int s = 0; s < S; s++) ev.push_back({seg_begin(s, S, n), s});
    ev.push_back({warm, S});
    ev.push_back({mid, S + 1});
    ev.push_back({n - 1, S + 2});
    std::stable_sort(ev.begin(), ev.end(), [](auto& a, auto& b) { return a.first < b.first; });
    pp->pts = d_points;
    pp->P = P;
    pp->nev = (int32_t)ev.size();
    pp->ncol = S + 3;
    pp->n_cum = n;
    for (size_t i = 0; i < ev.size(); i++) {
        pp->ev_idx[i] = (int32_t)ev[i].first;
        pp->ev_col[i] = ev[i].second;
    }
    pp->out = (double*)((char*)d_ws + pl.off_prefix);
    return true;
}

// The plan the segmented path would use: out[0..4) = segments per row,
// warps per segment, checkpoints per segment, slot capacity instance.
extern "C" int cs_seg_plan(int32_t P, int32_t R, int32_t max_cap, int64_t n, int32_t* out) {
    const cs::seg::Plan pl = cs::seg::make_plan(P, R, max_cap, n);
    out[0] = pl.S;
    out[1] = pl.G;
    out[2] = pl.Q;
    out[3] = pl.cmax;
    return CS_OK;
}

// Segmented single-chain simulation of P points x R replications (the chunk
// rb.. of RT); same outputs as cs_jffc_sim_impl's k1 path, except d_jobs
// (trace) which this path does not produce.
extern "C" int cs_seg_sim_impl(const cs_sim_point* d_points, int32_t P, const double* d_rates,
                               const int32_t* d_caps, int32_t max_cap, const double* d_streams,
                               int64_t lds, int32_t rb, int32_t R, int32_t RT, int64_t n, int64_t warm,
                               double* d_resp, int64_t ldr, double* d_busy, int32_t ldb,
                               cs_rep_summary* d_summ, void* d_ws, int64_t ws_bytes, int32_t flags,
                               void* stream) {
    using namespace cs;
    using namespace cs::seg;
    const Plan pl = make_plan(P, R, max_cap, n);
    if (pl.T == 0) return CS_OK;
    if (d_ws == nullptr || ws_bytes < (int64_t)pl.bytes) {
        set_error("cs_jffc_sim: segmented path needs %lld workspace bytes", (long long)pl.bytes);
        return CS_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)d_ws;
    const bool prefix_ready = flags & CS_SIM_PREFIX_READY;
    Args A{};
    A.il4 = (flags & CS_SIM_STREAMS_IL4) ? 1 : 0;
    A.pts = d_points;
    A.rates = d_rates;
    A.caps = d_caps;
    A.S = d_streams;
    A.lds = lds;
    A.P = P;
    A.R = R;
    A.RT = RT;
    A.rb = rb;
    A.n = n;
    A.warm = warm;
    A.resp = d_resp;
    A.ldr = ldr;
    A.busy_out = d_busy;
    A.ldb = ldb;
    A.summ = d_summ;
    A.prefix = (double*)(ws + pl.off_prefix);
    A.ckf = (double*)(ws + pl.off_ckf);
    A.ckk = (uint32_t*)(ws + pl.off_ckk);
    A.blk = (double*)(ws + pl.off_blk);
    A.status = (int32_t*)(ws + pl.off_status);
    A.spec = (int32_t*)(ws + pl.off_spec);
    A.progress = (uint32_t*)(ws + pl.off_progress);
    A.nblk = pl.nblk;
    A.nseg = pl.S;
    A.G = pl.G;
    A.Q = pl.Q;
    A.cmax = pl.cmax;
    // statuses (segment 0 exact) and progress words: fresh per launch
    int rc = check_cuda(cudaMemsetAsync(ws + pl.off_status, 0, pl.off_progress + sizeof(uint32_t) * pl.S * pl.G -
                                                                  pl.off_status, st),
                        "seg workspace reset");
    if (rc) return rc;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (!prefix_ready && getenv("CS_SEG_TRACE")) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, st);
    }
    if (!prefix_ready) {
        // ring of the prefix pass: PF_NBUF chunks x (distinct rows per warp) lines
        const int rows_per_warp = (int)std::min<int64_t>(32, (31 + P - 1) / P + 1);
        const size_t smem = sizeof(double) * PF_NBUF * rows_per_warp * PF_U;
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(seg_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        seg_prefix_kernel<<<(int)((pl.T + 31) / 32), 32, smem, st>>>(A);
        if ((rc = check_launch("seg_prefix_kernel"))) return rc;
    }
    if (ev0) {
        cudaEventRecord(ev1, st);
        cudaEventSynchronize(ev1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        fprintf(stderr, "seg_prefix_kernel %.3f ms (S=%d G=%d Q=%d)\n", ms, pl.S, pl.G, pl.Q);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    switch (pl.cmax) {
        case 4: return A.il4 ? launch<4, true>(pl, A, st) : launch<4, false>(pl, A, st);
        case 7: return A.il4 ? launch<7, true>(pl, A, st) : launch<7, false>(pl, A, st);
        case 8: return A.il4 ? launch<8, true>(pl, A, st) : launch<8, false>(pl, A, st);
        default: return A.il4 ? launch<16, true>(pl, A, st) : launch<16, false>(pl, A, st);
    }
}
