// stats.cu -- run_sim aggregation over the stored responses (sim.py:406-438).
//
// Per replication, responses.mean() (sim.py:407) is numpy's pairwise sum
// (loops_utils.h.src @TYPE@_pairwise_sum: blocks <= 128 summed with 8
// accumulators, larger ranges split at n/2 rounded down to a multiple of 8)
// over the completion-ordered responses, divided by the count.  The split
// tree depends only on the row length m; the host builds it once (leaves +
// post-order internal nodes) and the device evaluates it bit-exactly: 8 lanes
// per leaf (lane j = accumulator j), the exact ((r0+r1)+(r2+r3))+((r4+r5)+
// (r6+r7)) shuffle combine, then a per-row walk of the internal nodes.
//
// Quantiles need exact order statistics of each sweep point's merged
// responses (the values np.quantile interpolates between).  An exact
// sample-select whose only full read of the responses is the leaf-sum pass:
//   1. sample = 4 consecutive responses (one sector) of every 128 of each row
//      (1/32 of the bytes, spread over the whole run).  The sample order
//      statistics at ranks k|S|/N -+ 12 sigma bracket each target; they are
//      located on the device by two histogram levels (responses >= +0, so
//      bit order == value order): a 15-bit digit-0 histogram and a 12-bit
//      histogram of the next bits within the selected buckets (sb_* kernels).
//   2. the leaf-sum pass also counts the values below each bracket (whole
//      high-word ranges: the high 32 bits decide) and collects the values
//      inside it (staged per lane in shared memory by predicated stores,
//      handed over in batches with exact reservations).
//   3. if below <= k < below + |inside| (verified; else the bracket widens and
//      step 2 repeats), the k-th value is found by 12-bit digit rounds over
//      the few candidates, starting below the bracket's common bit prefix.
//   Groups of <= 2^20 responses take an exact selection over every value
//   (select_rows: digit-0 histogram, bucket compaction, digit rounds).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "cs_internal.cuh"

namespace cs {

constexpr int H0_BITS = 15;
constexpr int H0_BINS = 1 << H0_BITS;
constexpr int RD_BITS = 12;  // digit width of the selection rounds
constexpr int RD_BINS = 1 << RD_BITS;
constexpr int MAX_LISTS = 6;   // quantile brackets per group
constexpr int SEL_LISTS = 12;  // ranks per group of one exact selection (sample: both bracket ends)

__device__ __forceinline__ uint64_t dbits(double v) { return (uint64_t)__double_as_longlong(v); }

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Logical view of each row: logical index s -> physical (s / chunk) * stride + s % chunk.
struct RowView {
    int64_t len;     // logical values per row
    int32_t chunk_log2;   // 2^chunk_log2 consecutive values taken ...
    int32_t stride_log2;  // ... every 2^stride_log2 values (chunk == stride: contiguous)
    __host__ __device__ int64_t phys(int64_t s) const {
        return ((s >> chunk_log2) << stride_log2) | (s & ((1ll << chunk_log2) - 1));
    }
};

// Digit-0 (bits 62..48) histogram; a block takes a contiguous range of rows and
// flushes its shared histogram whenever the group changes.
__global__ void __launch_bounds__(1024) hist0_rows_kernel(const double* __restrict__ resp, int64_t n_rows,
                                                          RowView rv, int64_t ldr, int64_t rows_per_group,
                                                          uint32_t* __restrict__ hist0,
                                                          unsigned long long* __restrict__ n_bad) {
    extern __shared__ uint32_t sh[];
    const int64_t per_block = (n_rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = (int64_t)blockIdx.x * per_block;
    const int64_t r1 = min(n_rows, r0 + per_block);
    if (r0 >= r1) return;
    for (int64_t g = r0 / rows_per_group; g <= (r1 - 1) / rows_per_group; g++) {
        for (int b = threadIdx.x; b < H0_BINS; b += blockDim.x) sh[b] = 0;
        __syncthreads();
        const int64_t ga = max(r0, g * rows_per_group), gb = min(r1, (g + 1) * rows_per_group);
        constexpr int R = 4;  // rows in flight per thread (memory-level parallelism)
        for (int64_t row = ga; row < gb; row += R) {
            for (int64_t s = threadIdx.x; s < rv.len; s += blockDim.x) {
                const int64_t ps = rv.phys(s);
                uint64_t u[R];
#pragma unroll
                for (int r = 0; r < R; r++) u[r] = row + r < gb ? dbits(__ldg(resp + (row + r) * ldr + ps)) : 0ull;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    if (row + r >= gb) continue;
                    if (u[r] >> 63)
                        atomicAdd(n_bad, 1ull);
                    else
                        atomicAdd(&sh[u[r] >> 48], 1u);
                }
            }
        }
        __syncthreads();
        uint32_t* gh = hist0 + g * H0_BINS;
        for (int b = threadIdx.x; b < H0_BINS; b += blockDim.x)
            if (sh[b]) atomicAdd(&gh[b], sh[b]);
        __syncthreads();
    }
}

// Candidate appends without a returning atomic on the critical path: lane q
// owns list q's reservation of CAND_CHUNK slots (base, used) and the next
// reservation, requested a whole chunk ahead (next), so the atomic's latency
// is hidden behind the chunk's appends.  Reserved slots that stay unused hold
// the sentinel (all ones: above every response's bit pattern), which never
// changes a rank counted from below.
constexpr int CAND_CHUNK = 32;  // == warp size: sealing is one store per lane
struct CandChunks {
    unsigned long long base, next;
    int used;
    uint32_t in;  // values appended (owner lane)
};

__device__ __forceinline__ void cand_open(CandChunks& c, int lane, int nl, unsigned long long* __restrict__ fill_g) {
    c.base = c.next = 0;
    c.used = 0;
    c.in = 0;
    if (lane < nl) {
        c.base = atomicAdd(&fill_g[lane], (unsigned long long)CAND_CHUNK);
        c.next = atomicAdd(&fill_g[lane], (unsigned long long)CAND_CHUNK);
    }
}

// Append w to local list ql (every lane calls it; ql < 0: nothing) -- the
// part for list q; the caller loops q over the lists.  Only warp-uniform
// branches: a divergent branch makes the compiler wait for every load in
// flight (the row pass keeps the next leaf group's loads in flight across
// the appends).  cap_q / dst_q: list q's capacity and storage.
__device__ __forceinline__ void cand_push(CandChunks& c, int lane, int q, int ql, double w,
                                          unsigned long long* __restrict__ fill_g, unsigned long long cap_q,
                                          double* __restrict__ dst_q) {
    const unsigned msk = __ballot_sync(0xffffffffu, ql == q);
    if (msk == 0) return;
    const int cnt = __popc(msk);
    const int u = __shfl_sync(0xffffffffu, c.used, q);
    const unsigned long long b = __shfl_sync(0xffffffffu, c.base, q);
    const unsigned long long nb = __shfl_sync(0xffffffffu, c.next, q);
    const int pos = u + __popc(msk & ((1u << lane) - 1u));
    const bool cross = u + cnt > CAND_CHUNK;  // this append crosses into the next reservation
    const unsigned long long slot =
        pos >= CAND_CHUNK ? nb + (unsigned long long)(pos - CAND_CHUNK) : b + (unsigned long long)pos;
    const bool own = lane == q;
    c.used = own ? (cross ? u + cnt - CAND_CHUNK : u + cnt) : c.used;
    c.base = (own && cross) ? nb : c.base;
    c.in += own ? (uint32_t)cnt : 0u;
    if (own && cross) c.next = atomicAdd(&fill_g[q], (unsigned long long)CAND_CHUNK);
    if (ql == q && slot < cap_q) dst_q[slot] = w;  // overflow: host check
}

// Compaction of the values whose digit 0 is one of the group's selected
// buckets: a warp per row, chunked appends (the lists are pre-set to the
// sentinel, so no sealing).
__global__ void __launch_bounds__(256) compact_bucket_kernel(
    const double* __restrict__ resp, int64_t n_rows, RowView rv, int64_t ldr, int64_t rows_per_group,
    const int32_t* __restrict__ grp_nlist, const uint32_t* __restrict__ grp_bucket,
    const int64_t* __restrict__ off, const int64_t* __restrict__ cap, unsigned long long* __restrict__ fill,
    double* __restrict__ cand) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n_rows; row += warps) {
        const int64_t g = row / rows_per_group;
        const int nl = grp_nlist[g];
        const int64_t gl0 = g * SEL_LISTS;
        uint32_t bk[SEL_LISTS];
#pragma unroll
        for (int q = 0; q < SEL_LISTS; q++) bk[q] = q < nl ? grp_bucket[gl0 + q] : 0xffffffffu;
        CandChunks cc;
        cand_open(cc, lane, nl, fill + gl0);
        const double* __restrict__ a = resp + row * ldr;
        constexpr int U = 8;  // loads in flight per lane
        for (int64_t base = 0; base < rv.len; base += 32 * U) {
            double v[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int64_t s = base + 32 * k + lane;
                v[k] = s < rv.len ? __ldg(a + rv.phys(s)) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < U; k++) {
                int ql = -1;
                if (base + 32 * k + lane < rv.len) {
                    const uint32_t d0 = (uint32_t)(dbits(v[k]) >> 48);
#pragma unroll
                    for (int q = 0; q < SEL_LISTS; q++)
                        if (bk[q] == d0) ql = q;
                }
                // only the lists some lane appends to (usually one)
                for (unsigned m = __reduce_or_sync(0xffffffffu, ql >= 0 ? 1u << ql : 0u); m; m &= m - 1)
                {
                    const int q = __ffs(m) - 1;
                    cand_push(cc, lane, q, ql, v[k], fill + gl0, (unsigned long long)cap[gl0 + q], cand + off[gl0 + q]);
                }
            }
        }
    }
}

// bit if d[q] <= wid[q] for some q, else 0: one predicate chained through
// the compares (setp .or), one select
template <int NB>
__device__ __forceinline__ uint32_t near_bit(const uint32_t (&d)[NB], const uint32_t (&wid)[NB], uint32_t bit) {
    uint32_t r;
    if (NB == 3) {
        asm("{\n\t.reg .pred p;\n\t"
            "setp.le.u32 p, %1, %2;\n\t"
            "setp.le.or.u32 p, %3, %4, p;\n\t"
            "setp.le.or.u32 p, %5, %6, p;\n\t"
            "selp.b32 %0, %7, 0, p;\n\t}"
            : "=r"(r)
            : "r"(d[0]), "r"(wid[0]), "r"(d[1 % NB]), "r"(wid[1 % NB]), "r"(d[2 % NB]), "r"(wid[2 % NB]), "r"(bit));
    } else {
        bool nr = false;
#pragma unroll
        for (int q = 0; q < NB; q++) nr |= d[q] <= wid[q];
        r = nr ? bit : 0u;
    }
    return r;
}

// Bracket state of one row (registers only: fixed sizes, static indices).
template <int NB>
struct Brackets {
    uint64_t lo[NB], hi[NB];
    uint32_t lo_hw[NB], hi_hw[NB], wid_hw[NB];
    uint32_t cnt[NB];
};

// Classify one value: counts values below each bracket and returns the
// bracket list it falls in (or -1).  The high 32 bits decide unless they lie
// within a bracket's high-word range; then the exact 64-bit compare runs.
template <int NB>
__device__ __forceinline__ int classify_one(Brackets<NB>& br, uint64_t u, bool have) {
    const uint32_t hw = (uint32_t)(u >> 32);
    int slot = -1;
#pragma unroll
    for (int q = 0; q < NB; q++) {
        const bool below_hw = hw < br.lo_hw[q];
        const bool near = hw >= br.lo_hw[q] && hw <= br.hi_hw[q];
        bool below = below_hw;
        if (near) {  // rare: exact 64-bit compare
            below = u < br.lo[q];
            if (!below && u <= br.hi[q]) slot = q;
        }
        br.cnt[q] += (have && below) ? 1u : 0u;
    }
    return have ? slot : -1;
}

// The one full pass, one warp per replication row: numpy pairwise leaf sums
// (8 lanes per leaf, 4 leaves at a time; a leaf's values are loaded up front
// for memory-level parallelism) into a per-warp shared-memory array, the
// split tree combined height by height with the lanes in parallel, and the
// optional bracket counting/compaction.  The plan (leaf offsets, lengths,
// height-ordered nodes) sits in shared memory.
constexpr int LB_WARPS = 8;
// Per-lane staging of the values inside a bracket: appended with predicated
// shared-memory stores (no branch: a divergent branch or a warp collective
// inside a loop makes the compiler wait for the next leaf group's loads, which
// the pass keeps in flight), handed to the candidate lists when some lane
// could overflow in the next group, and at the row's end.

// T = value slots per lane and leaf: 8*T >= the plan's longest leaf (numpy
// leaves hold 64..128 values; 90000-value rows have 80/88-value leaves, so
// T = 12 there instead of 16 saves a quarter of the per-slot work)
template <int NB, int T>
__global__ void __launch_bounds__(LB_WARPS * 32, 2) row_stats_kernel(
    const double* __restrict__ resp, int64_t n_rows, int64_t rows_per_group, int64_t ldr, int64_t m,
    const int32_t* __restrict__ g_plan, int32_t L, cs_rep_summary* __restrict__ summ,
    double* __restrict__ row_sums, int do_bracket, const int32_t* __restrict__ grp_nlist,
    const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi, const int64_t* __restrict__ off,
    const int64_t* __restrict__ cap, unsigned long long* __restrict__ fill,
    unsigned long long* __restrict__ below, unsigned long long* __restrict__ inside,
    double* __restrict__ cand, int32_t n_heights, double* __restrict__ leaf_scratch, int32_t stg_slots,
    int32_t plan_in_smem) {
    // shared: per-warp leaf values [LB_WARPS][L] doubles, then the plan:
    // leaf offset[L], leaf length[L], height offsets[n_heights + 1] and the
    // internal nodes in height order as (a, b) pairs: v[a] = v[a] + v[b]
    // (a = the node's leftmost leaf, b = its right child's leftmost leaf)
    // leaf values: shared memory, or (long rows) a global scratch slice per warp
    extern __shared__ double row_sh[];
    const int STG = stg_slots;  // >= T + 3
    double* stage_sh = row_sh;  // [LB_WARPS][STG][32]
    double* leaf_sh = row_sh + (size_t)LB_WARPS * STG * 32;
    // the plan: in shared memory, or (long rows: 4 words per leaf) read
    // through L1 from global memory, which keeps two blocks per SM
    int32_t* plan_sh = reinterpret_cast<int32_t*>(leaf_scratch ? leaf_sh : leaf_sh + (size_t)LB_WARPS * L);
    const int plan_words = 2 * L + (n_heights + 1) + 2 * (L - 1);
    if (plan_in_smem)
        for (int q = threadIdx.x; q < plan_words; q += blockDim.x) plan_sh[q] = g_plan[q];
    const int32_t* plan = plan_in_smem ? plan_sh : g_plan;
    __syncthreads();
    const int32_t* leaf_off = plan;
    const int32_t* leaf_len = plan + L;
    const int32_t* h_off = plan + 2 * L;
    const int32_t* nodes = h_off + n_heights + 1;
    double* lv = leaf_scratch
                     ? leaf_scratch + ((size_t)blockIdx.x * LB_WARPS + (threadIdx.x >> 5)) * (size_t)L
                     : leaf_sh + (size_t)(threadIdx.x >> 5) * L;
    const int lane = threadIdx.x & 31, j = lane & 7, sub = lane >> 3, warp = threadIdx.x >> 5;
    double* const stg = stage_sh + (size_t)warp * STG * 32 + lane;  // slot i at stg[32 * i]
    for (int64_t row = (int64_t)blockIdx.x * LB_WARPS + warp; row < n_rows; row += (int64_t)gridDim.x * LB_WARPS) {
        const int64_t g = row / rows_per_group;
        const int nl = do_bracket ? grp_nlist[g] : 0;  // warp-uniform, <= NB (checked on the host)
        Brackets<NB> br;
#pragma unroll
        for (int q = 0; q < NB; q++) {
            br.lo[q] = q < nl ? lo[g * MAX_LISTS + q] : ~0ull;
            br.hi[q] = q < nl ? hi[g * MAX_LISTS + q] : 0ull;
            br.lo_hw[q] = (uint32_t)(br.lo[q] >> 32);
            br.hi_hw[q] = (uint32_t)(br.hi[q] >> 32);
            br.wid_hw[q] = q < nl ? br.hi_hw[q] - br.lo_hw[q] : 0u;
            br.cnt[q] = 0;
        }
        const double* __restrict__ rowp = resp + row * ldr;
        const int64_t gl0 = g * MAX_LISTS;
        unsigned long long capq[NB];
        double* dstq[NB];
#pragma unroll
        for (int q = 0; q < NB; q++) {
            capq[q] = q < nl ? (unsigned long long)cap[gl0 + q] : 0ull;
            dstq[q] = q < nl ? cand + off[gl0 + q] : cand;
        }
        auto list_of = [&](double w) {  // bracket list of an inside value
            const uint32_t hw = (uint32_t)(dbits(w) >> 32);
            int ql = 0;
#pragma unroll
            for (int q = 1; q < NB; q++) ql = hw - br.lo_hw[q] <= br.wid_hw[q] ? q : ql;
            return ql;
        };
        // Hand the staged values to the candidate lists: per list a warp scan
        // of the lanes' counts and one exact reservation (atomicAdd by lane
        // 31), then every lane stores its values at its offsets.
        uint32_t ns = 0;  // this lane's staged values
        auto drain_stage = [&]() {
            const int nmax = (int)__reduce_max_sync(0xffffffffu, ns);
            if (nmax == 0) return;
            uint32_t cq[NB];
#pragma unroll
            for (int q = 0; q < NB; q++) cq[q] = 0;
            for (int i = 0; i < nmax; i++) {
                const int ql = (uint32_t)i < ns ? list_of(stg[32 * i]) : -1;
#pragma unroll
                for (int q = 0; q < NB; q++) cq[q] += ql == q ? 1u : 0u;
            }
            unsigned long long pos[NB];
#pragma unroll
            for (int q = 0; q < NB; q++) {
                uint32_t inc = cq[q];
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += o;
                }
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
                unsigned long long base = 0;
                if (lane == 31 && tot) {
                    base = atomicAdd(&fill[gl0 + q], (unsigned long long)tot);
                    atomicAdd(&inside[gl0 + q], (unsigned long long)tot);
                }
                pos[q] = __shfl_sync(0xffffffffu, base, 31) + (inc - cq[q]);
            }
            for (int i = 0; i < nmax; i++) {
                if ((uint32_t)i < ns) {
                    const double w = stg[32 * i];
                    const int ql = list_of(w);
#pragma unroll
                    for (int q = 0; q < NB; q++)
                        if (ql == q) {
                            if (pos[q] < capq[q]) dstq[q][pos[q]] = w;  // overflow: host check
                            pos[q]++;
                        }
                }
            }
            ns = 0;
        };
        auto stage = [&](bool p, double w) {  // predicated, no branch
            if (p) {
                stg[32 * ns] = w;
                ns++;
            }
        };
        // Software pipeline: the next leaf group's loads are in flight while
        // this group is summed and classified.
        // Slots past a leaf's 8-aligned end hold +0.0, which leaves the lane
        // sums unchanged (all values are >= +0) and is counted "below" by the
        // fast path exactly when 0 < lo_hw; that is undone per lane at the end.
        uint32_t npad = 0;
        auto load_group = [&](int leaf0, double (&buf)[T]) {
            const int leaf = leaf0 + sub;
            const int len = leaf < L ? leaf_len[leaf] : 0;
            const double* __restrict__ a = rowp + (leaf < L ? leaf_off[leaf] : 0);
            const int main_end = len >= 8 ? len - len % 8 : 0;
#pragma unroll
            for (int t = 0; t < T; t++) buf[t] = (j + 8 * t < main_end) ? __ldg(a + j + 8 * t) : 0.0;
        };
        auto process_group = [&](int l0, const double (&v)[T]) {
            const int leaf = l0 + sub;
            const bool valid = leaf < L;
            const int len = valid ? leaf_len[leaf] : 0;
            const double* __restrict__ a = rowp + (valid ? leaf_off[leaf] : 0);
            const int main_end = len >= 8 ? len - len % 8 : 0;
            const int nvalid = main_end > j ? (main_end - j + 7) >> 3 : 0;  // slots t < nvalid hold data
            double acc = v[0];
#pragma unroll
            for (int t = 1; t < T; t++) acc = __dadd_rn(acc, v[t]);  // pads add +0.0
            if (do_bracket) {
                // brackets are whole high-word ranges (host side), so the high
                // word decides: d = hw - lo_hw, "below" is its sign (all high
                // words < 2^31) and "inside" is d <= wid
                npad += (uint32_t)(T - nvalid);
#pragma unroll
                for (int t = 0; t < T; t++) {
                    const uint32_t hw = (uint32_t)(dbits(v[t]) >> 32);
                    uint32_t d[NB];
#pragma unroll
                    for (int q = 0; q < NB; q++) {
                        d[q] = hw - br.lo_hw[q];
                        br.cnt[q] += d[q] >> 31;
                    }
                    // a pad (+0.0, slot >= nvalid) is inside a bracket starting at 0
                    stage(near_bit<NB>(d, br.wid_hw, 1u) && t < nvalid, v[t]);
                }
                if (__any_sync(0xffffffffu, ns > (uint32_t)(STG - T))) drain_stage();
            }
            // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) in numpy's order
            const double s1 = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, 1));
            const double s2 = __dadd_rn(s1, __shfl_down_sync(0xffffffffu, s1, 2));
            double res = __dadd_rn(s2, __shfl_down_sync(0xffffffffu, s2, 4));
            // remainder (last leaf of the row) / tiny leaf (< 8 values): lane j == 0
            const int rem_begin = len >= 8 ? main_end : 0;
            if (len < 8) res = 0.0;
            const int rem = __reduce_max_sync(0xffffffffu, len - rem_begin);
            for (int t = 0; t < rem; t++) {
                const int idx = rem_begin + t;
                const bool have = j == 0 && idx < len;
                const double w = have ? a[idx] : 0.0;
                if (have) res = __dadd_rn(res, w);
                if (do_bracket) {
                    stage(classify_one<NB>(br, dbits(w), have) >= 0, w);
                    if (__any_sync(0xffffffffu, ns >= (uint32_t)STG)) drain_stage();
                }
            }
            if (j == 0 && valid) lv[leaf] = res;  // leaves l0..l0+3 (lanes 0, 8, 16, 24)
        };
        double nv[T];
        load_group(0, nv);
        for (int l0 = 0; l0 < L; l0 += 4) {
            double v[T];
#pragma unroll
            for (int t = 0; t < T; t++) v[t] = nv[t];
            load_group(l0 + 4, nv);
            process_group(l0, v);
        }
        if (do_bracket) {
            drain_stage();
#pragma unroll
            for (int q = 0; q < NB; q++) br.cnt[q] -= ((0u - br.lo_hw[q]) >> 31) * npad;
        }
        // the split tree, one height at a time: nodes of equal height have
        // disjoint subtrees, so the lanes combine them in parallel
        __syncwarp();
        for (int h = 0; h < n_heights; h++) {
            for (int i = h_off[h] + lane; i < h_off[h + 1]; i += 32) {
                const int na = nodes[2 * i], nb = nodes[2 * i + 1];
                lv[na] = __dadd_rn(lv[na], lv[nb]);
            }
            __syncwarp();
        }
        if (lane == 0) {
            const double total = L > 0 ? lv[0] : 0.0;
            if (row_sums) row_sums[row] = total;
            if (summ) {
                summ[row].resp_sum = total;
                summ[row].resp_mean = m > 0 ? __ddiv_rn(total, (double)m) : NAN;
            }
        }
        if (do_bracket) {
#pragma unroll
            for (int q = 0; q < NB; q++) {
                uint32_t c = br.cnt[q];
                for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
                if (lane == 0 && q < nl && c) atomicAdd(&below[g * MAX_LISTS + q], (unsigned long long)c);
            }

        }
    }
}

// ---------------------------------------------------------------------------
// Sample brackets on the device (the sample only has to bracket each target;
// the full pass verifies): per group, the digit-0 histogram of the sample
// (hist0_rows_kernel) locates each sample rank's 15-bit bucket; a second
// histogram of the next 12 bits (bits 47..36) over the sample values in those
// buckets locates it to within 2^36 of its bit pattern (16 high-word units:
// a relative 2^-16 of its bucket, far inside the +-12 sigma margin).  3 MB of
// counters for 16 groups: cheap to all-reduce when sharded.  No compaction, no
// digit rounds, one small read-back.
constexpr int H1_BITS = 12, H1_BINS = 1 << H1_BITS;  // bits 47..36
constexpr int SB_SLOTS = 2 * MAX_LISTS;  // sample ranks per group (both bracket ends)

// The bucket of each sample rank (block per group: block scan of the 32K bins
// in shared memory, then a binary search per rank).  rep[i]: the first slot
// with the same bucket (its hist1 plane is shared).
__global__ void __launch_bounds__(1024) sb_select0_kernel(const uint32_t* __restrict__ hist0, int n_slots,
                                                          const int64_t* __restrict__ srank,
                                                          uint32_t* __restrict__ bucket, int64_t* __restrict__ resid,
                                                          int32_t* __restrict__ rep) {
    extern __shared__ uint32_t cum[];  // [H0_BINS] inclusive prefix
    __shared__ uint32_t part[1024];
    const uint32_t* h = hist0 + (size_t)blockIdx.x * H0_BINS;
    constexpr int PER = H0_BINS / 1024;
    uint32_t loc[PER], acc = 0;
#pragma unroll
    for (int k = 0; k < PER; k++) acc += (loc[k] = h[threadIdx.x * PER + k]);
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {  // inclusive scan of the partial sums
        const uint32_t v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
#pragma unroll
    for (int k = 0; k < PER; k++) cum[threadIdx.x * PER + k] = (run += loc[k]);
    __syncthreads();
    if (threadIdx.x < (unsigned)n_slots) {
        const int i = threadIdx.x;
        const int64_t r = srank[(size_t)blockIdx.x * n_slots + i];
        int lo = 0, hi = H0_BINS - 1;  // first bin with cum > r
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int64_t)cum[mid] > r) hi = mid;
            else lo = mid + 1;
        }
        bucket[(size_t)blockIdx.x * SB_SLOTS + i] = (uint32_t)lo;
        resid[(size_t)blockIdx.x * SB_SLOTS + i] = r - (lo ? (int64_t)cum[lo - 1] : 0);
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)n_slots) {
        const int i = threadIdx.x;
        const uint32_t b = bucket[(size_t)blockIdx.x * SB_SLOTS + i];
        int r0 = i;
        for (int j = 0; j < i; j++)
            if (bucket[(size_t)blockIdx.x * SB_SLOTS + j] == b) {
                r0 = j;
                break;
            }
        rep[(size_t)blockIdx.x * SB_SLOTS + i] = r0;
    }
}

// bits 47..36 of the sample values whose digit 0 is a selected bucket, into
// the plane of that bucket's first slot (global atomics: the values spread)
__global__ void __launch_bounds__(256) sb_hist1_kernel(const double* __restrict__ resp, int64_t n_rows, RowView rv,
                                                       int64_t ldr, int64_t rows_per_group, int n_slots,
                                                       const uint32_t* __restrict__ bucket,
                                                       const int32_t* __restrict__ rep,
                                                       uint32_t* __restrict__ hist1) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < n_rows; row += warps) {
        const int64_t g = row / rows_per_group;
        uint32_t bk[SB_SLOTS];
#pragma unroll
        for (int q = 0; q < SB_SLOTS; q++)
            bk[q] = q < n_slots && rep[g * SB_SLOTS + q] == q ? bucket[g * SB_SLOTS + q] : 0xffffffffu;
        const double* __restrict__ a = resp + row * ldr;
        uint32_t* hg = hist1 + (size_t)g * SB_SLOTS * H1_BINS;
        constexpr int U = 8;
        for (int64_t base = 0; base < rv.len; base += 32 * U) {
            uint64_t u[U];
#pragma unroll
            for (int k = 0; k < U; k++) {
                const int64_t s = base + 32 * k + lane;
                u[k] = s < rv.len ? dbits(__ldg(a + rv.phys(s))) : ~0ull;
            }
#pragma unroll
            for (int k = 0; k < U; k++) {
                const uint32_t d0 = (uint32_t)(u[k] >> 48);
                int ql = -1;
#pragma unroll
                for (int q = 0; q < SB_SLOTS; q++)
                    if (bk[q] == d0) ql = q;
                if (ql >= 0) atomicAdd(&hg[(size_t)ql * H1_BINS + ((u[k] >> 36) & (H1_BINS - 1))], 1u);
            }
        }
    }
}

// per (group, slot): the bit prefix (62..36) of the sample order statistic
__global__ void __launch_bounds__(1024) sb_select1_kernel(const uint32_t* __restrict__ hist1, int n_slots,
                                                          const uint32_t* __restrict__ bucket,
                                                          const int64_t* __restrict__ resid,
                                                          const int32_t* __restrict__ rep,
                                                          uint64_t* __restrict__ prefix) {
    extern __shared__ uint32_t cum[];  // [H1_BINS]
    __shared__ uint32_t part[1024];
    const int g = blockIdx.x / n_slots, i = blockIdx.x % n_slots;
    const size_t gi = (size_t)g * SB_SLOTS + i;
    const uint32_t* h = hist1 + ((size_t)g * SB_SLOTS + rep[gi]) * H1_BINS;
    constexpr int PER = H1_BINS / 1024;
    uint32_t loc[PER], acc = 0;
#pragma unroll
    for (int k = 0; k < PER; k++) acc += (loc[k] = h[threadIdx.x * PER + k]);
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        const uint32_t v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
#pragma unroll
    for (int k = 0; k < PER; k++) cum[threadIdx.x * PER + k] = (run += loc[k]);
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t r = resid[gi];
        int lo = 0, hi = H1_BINS - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int64_t)cum[mid] > r) hi = mid;
            else lo = mid + 1;
        }
        prefix[gi] = ((uint64_t)bucket[gi] << 48) | ((uint64_t)lo << 36);
    }
}

struct SelSlot {
    uint64_t prefix;   // fixed high bits (above the current digit)
    int64_t rank;      // remaining rank among the candidates sharing the prefix
    int64_t cand_off;  // candidate list
    int64_t cand_len;
    int32_t shift0;    // this slot's first digit (its candidates share every bit above it)
    int32_t compacted; // 1: cand_off/cand_len index the compacted candidates
};

// Histogram of the digit [shift, shift+12) over each slot's candidates that
// match its prefix; shared-memory privatised (candidates cluster in few bins).
__global__ void __launch_bounds__(512) round_hist_kernel(const double* __restrict__ cand,
                                                         const double* __restrict__ ccand,
                                                         const SelSlot* __restrict__ slots, int n_slots,
                                                         int shift, uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[RD_BINS];
    const int s = blockIdx.y;
    const SelSlot sl = slots[s];
    if (shift > sl.shift0) return;  // the digit is part of the slot's common prefix
    const double* __restrict__ src = sl.compacted ? ccand : cand;
    for (int b = threadIdx.x; b < RD_BINS; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    const uint64_t hi_mask = shift + RD_BITS >= 64 ? 0ull : ~((1ull << (shift + RD_BITS)) - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sl.cand_len;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = dbits(src[sl.cand_off + i]);
        if ((u & hi_mask) == sl.prefix) atomicAdd(&sh[(u >> shift) & (RD_BINS - 1)], 1u);
    }
    __syncthreads();
    uint32_t* h = hist + (int64_t)s * RD_BINS;
    for (int b = threadIdx.x; b < RD_BINS; b += blockDim.x)
        if (sh[b]) atomicAdd(&h[b], sh[b]);
}

__global__ void __launch_bounds__(1024) round_select_kernel(SelSlot* __restrict__ slots, int shift,
                                                            const uint32_t* __restrict__ hist) {
    const int s = blockIdx.x;
    if (shift > slots[s].shift0) return;
    __shared__ unsigned long long part[1024];
    const uint32_t* h = hist + (int64_t)s * RD_BINS;
    constexpr int PER = RD_BINS / 1024;
    unsigned long long acc = 0;
#pragma unroll
    for (int b = 0; b < PER; b++) acc += h[threadIdx.x * PER + b];
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {
        unsigned long long v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0ull;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    const long long rank = slots[s].rank;
    const unsigned long long before = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
    if ((long long)before <= rank && rank < (long long)part[threadIdx.x]) {
        unsigned long long c = before;
        for (int b = threadIdx.x * PER; b < (threadIdx.x + 1) * PER; b++) {
            if ((long long)(c + h[b]) > rank) {
                slots[s].prefix |= ((uint64_t)b << shift);
                slots[s].rank = rank - (long long)c;
                break;
            }
            c += h[b];
        }
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
// CS_TRACE_STATS=1: host timestamps at the statistics' phase boundaries
static void trace(const char* what, cudaStream_t st) {
    const bool on = getenv("CS_TRACE_STATS") != nullptr;
    if (!on) return;
    static double t0 = 0;
    cudaStreamSynchronize(st);
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    const double t = ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    if (!strcmp(what, "begin")) t0 = t;
    fprintf(stderr, "[stats] %-14s %8.3f ms\n", what, t - t0);
}

struct DBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaStream_t st = nullptr;
    ~DBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    int alloc(size_t bytes, cudaStream_t s) {
        st = s;
        n = bytes;
        return pool_alloc(&p, bytes, s);
    }
    template <class T>
    T* as() const {
        return (T*)p;
    }
};

// 12-bit digit rounds at shifts first_shift, first_shift-12, ..., 0 (first_shift
// a multiple of 12); slot prefixes must already hold the bits above first_shift+12.
// After every slot's first digit round the candidates still sharing its
// prefix are few: copy them out (per slot, into its own region) so the later
// rounds read only those.  A slot whose matches overflow its region keeps
// its list.
__global__ void __launch_bounds__(512) round_compact_kernel(const double* __restrict__ cand,
                                                            const SelSlot* __restrict__ slots, int shift,
                                                            double* __restrict__ out, int64_t region,
                                                            unsigned long long* __restrict__ cnt) {
    const int s = blockIdx.y, lane = threadIdx.x & 31;
    const SelSlot sl = slots[s];
    const uint64_t hi_mask = shift >= 64 ? 0ull : ~((1ull << shift) - 1);
    double* dst = out + (int64_t)s * region;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < sl.cand_len; i0 += stride) {
        const int64_t i = i0 + lane;
        const double v = i < sl.cand_len ? cand[sl.cand_off + i] : 0.0;
        const bool m = i < sl.cand_len && (dbits(v) & hi_mask) == sl.prefix;
        const unsigned bal = __ballot_sync(0xffffffffu, m);
        if (!bal) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&cnt[s], (unsigned long long)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const unsigned long long pos = base + __popc(bal & ((1u << lane) - 1u));
        if (m && pos < (unsigned long long)region) dst[pos] = v;
    }
}

__global__ void round_compact_fix_kernel(SelSlot* __restrict__ slots, int n_slots, int64_t region,
                                         const unsigned long long* __restrict__ cnt) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_slots || cnt[s] > (unsigned long long)region) return;
    slots[s].cand_off = (int64_t)s * region;
    slots[s].cand_len = (int64_t)cnt[s];
    slots[s].compacted = 1;
}

static int run_rounds(std::vector<SelSlot>& slots, const double* d_cand, int first_shift, bool dist,
                      cudaStream_t st) {
    const int n_slots = (int)slots.size();
    if (n_slots == 0) return CS_OK;
    DBuf b_slots, b_hist;
    int rc;
    if ((rc = b_slots.alloc(sizeof(SelSlot) * n_slots, st)) ||
        (rc = b_hist.alloc(sizeof(uint32_t) * RD_BINS * (size_t)n_slots, st)))
        return rc;
    cudaMemcpyAsync(b_slots.p, slots.data(), b_slots.n, cudaMemcpyHostToDevice, st);
    int64_t max_len = 1;
    for (auto& s : slots) max_len = std::max(max_len, s.cand_len);
    const int bx = (int)std::max<int64_t>(1, std::min<int64_t>((max_len + 4095) / 4096, 64));
    // after the round at the lowest first digit every slot has had its first
    // round: compact there if more rounds follow
    int min_shift0 = first_shift;
    for (auto& s : slots) min_shift0 = std::min(min_shift0, (int)s.shift0);
    const int64_t region = std::max<int64_t>(4096, max_len / 32);
    DBuf b_ccand, b_ccnt;
    for (int shift = first_shift; shift >= 0; shift -= RD_BITS) {
        cudaMemsetAsync(b_hist.p, 0, b_hist.n, st);
        round_hist_kernel<<<dim3(bx, n_slots), 512, 0, st>>>(d_cand, b_ccand.as<double>(), b_slots.as<SelSlot>(),
                                                              n_slots, shift, b_hist.as<uint32_t>());
        if ((rc = check_launch("round_hist_kernel"))) return rc;
        if (dist && (rc = allreduce_u32(b_hist.p, (size_t)RD_BINS * n_slots, st))) return rc;
        round_select_kernel<<<n_slots, 1024, 0, st>>>(b_slots.as<SelSlot>(), shift, b_hist.as<uint32_t>());
        if ((rc = check_launch("round_select_kernel"))) return rc;
        if (shift == min_shift0 && shift > 0 && max_len > 4 * region) {
            if ((rc = b_ccand.alloc(sizeof(double) * region * (size_t)n_slots, st)) ||
                (rc = b_ccnt.alloc(sizeof(unsigned long long) * n_slots, st)))
                return rc;
            cudaMemsetAsync(b_ccnt.p, 0, b_ccnt.n, st);
            round_compact_kernel<<<dim3(bx, n_slots), 512, 0, st>>>(d_cand, b_slots.as<SelSlot>(), shift,
                                                                     b_ccand.as<double>(), region,
                                                                     b_ccnt.as<unsigned long long>());
            if ((rc = check_launch("round_compact_kernel"))) return rc;
            round_compact_fix_kernel<<<(n_slots + 127) / 128, 128, 0, st>>>(b_slots.as<SelSlot>(), n_slots, region,
                                                                             b_ccnt.as<unsigned long long>());
            if ((rc = check_launch("round_compact_fix_kernel"))) return rc;
        }
    }
    cudaMemcpyAsync(slots.data(), b_slots.p, b_slots.n, cudaMemcpyDeviceToHost, st);
    return check_cuda(cudaStreamSynchronize(st), "rounds sync");
}

// Exact order statistics over the logical view of every row (groups of
// rows_per_group rows); ranks: n_groups x n_ranks, 0-based.
static int select_rows(const double* d_resp, int64_t n_groups, int64_t rows_per_group, RowView rv,
                       int64_t ldr, const std::vector<int64_t>& ranks, int n_ranks, std::vector<double>& out,
                       bool dist, cudaStream_t st) {
    const int64_t n_rows = n_groups * rows_per_group;
    int rc;
    DBuf b_h0, b_bad;
    if ((rc = b_h0.alloc(sizeof(uint32_t) * H0_BINS * (size_t)n_groups, st)) ||
        (rc = b_bad.alloc(sizeof(unsigned long long), st)))
        return rc;
    cudaMemsetAsync(b_h0.p, 0, b_h0.n, st);
    cudaMemsetAsync(b_bad.p, 0, b_bad.n, st);
    const size_t smem = sizeof(uint32_t) * H0_BINS;
    cudaFuncSetAttribute(hist0_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int blocks = (int)std::min<int64_t>(n_rows, 2 * sm_count());
    hist0_rows_kernel<<<blocks, 1024, smem, st>>>(d_resp, n_rows, rv, ldr, rows_per_group, b_h0.as<uint32_t>(),
                                                  b_bad.as<unsigned long long>());
    if ((rc = check_launch("hist0_rows_kernel"))) return rc;
    if (dist && ((rc = allreduce_u32(b_h0.p, (size_t)H0_BINS * n_groups, st)) ||
                 (rc = allreduce_u64(b_bad.p, 1, st))))
        return rc;
    // pinned read-back buffer (2 MB for 16 groups), kept across calls
    static thread_local uint32_t* h0 = nullptr;
    static thread_local size_t h0_cap = 0;
    const size_t h0_need = (size_t)H0_BINS * n_groups + 2;
    if (h0_cap < h0_need) {
        if (h0) cudaFreeHost(h0);
        if ((rc = check_cuda(cudaMallocHost(&h0, sizeof(uint32_t) * h0_need), "cudaMallocHost"))) {
            h0 = nullptr;
            h0_cap = 0;
            return rc;
        }
        h0_cap = h0_need;
    }
    unsigned long long& bad = *reinterpret_cast<unsigned long long*>(h0 + (size_t)H0_BINS * n_groups);
    cudaMemcpyAsync(h0, b_h0.p, b_h0.n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&bad, b_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st);
    if ((rc = check_cuda(cudaStreamSynchronize(st), "select hist sync"))) return rc;
    trace("  sel hist0", st);
    if (bad) {
        set_error("cs_rep_stats: %llu negative responses (impossible for valid input)", bad);
        return CS_INTERNAL;
    }
    std::vector<int32_t> nlist(n_groups, 0);
    std::vector<uint32_t> bucket((size_t)n_groups * SEL_LISTS, 0xffffffffu);
    std::vector<int64_t> off((size_t)n_groups * SEL_LISTS, 0), cap((size_t)n_groups * SEL_LISTS, 0);
    std::vector<SelSlot> slots((size_t)n_groups * n_ranks);
    int64_t total = 0;
    std::vector<int> order(n_ranks);
    std::vector<uint32_t> bin_of(n_ranks);
    std::vector<int64_t> below_of(n_ranks);
    for (int64_t g = 0; g < n_groups; g++) {
        const uint32_t* hg = h0 + (size_t)g * H0_BINS;
        // one walk over the bins for all of the group's ranks, in rank order
        for (int q = 0; q < n_ranks; q++) order[q] = q;
        std::sort(order.begin(), order.end(),
                  [&](int x, int y) { return ranks[g * n_ranks + x] < ranks[g * n_ranks + y]; });
        {
            int64_t c = 0;
            uint32_t b = 0;
            for (int i = 0; i < n_ranks; i++) {
                const int64_t rank = ranks[g * n_ranks + order[i]];
                for (; b < (uint32_t)H0_BINS; b++) {
                    if (c + (int64_t)hg[b] > rank) break;
                    c += hg[b];
                }
                bin_of[order[i]] = b;
                below_of[order[i]] = c;
            }
        }
        for (int q = 0; q < n_ranks; q++) {
            const int64_t rank = ranks[g * n_ranks + q];
            const int64_t c = below_of[q];
            const uint32_t b = bin_of[q];
            int list = -1;
            for (int l = 0; l < nlist[g]; l++)
                if (bucket[g * SEL_LISTS + l] == b) list = l;
            if (list < 0) {
                list = nlist[g]++;
                bucket[g * SEL_LISTS + list] = b;
                off[g * SEL_LISTS + list] = total;
                // + the reserved-but-unused slots: < 2 chunks per row
                cap[g * SEL_LISTS + list] = hg[b] + 2 * CAND_CHUNK * rows_per_group;
                total += cap[g * SEL_LISTS + list];
            }
            SelSlot& s = slots[g * n_ranks + q];
            s.prefix = (uint64_t)b << 48;
            s.shift0 = 36;  // bits 47..0 below the digit-0 bucket
            s.rank = rank - c;
            s.cand_off = off[g * SEL_LISTS + list];
            s.cand_len = cap[g * SEL_LISTS + list];
        }
    }
    trace("  sel buckets", st);
    DBuf b_nl, b_bk, b_off, b_cap, b_fill, b_cand;
    if ((rc = b_nl.alloc(sizeof(int32_t) * n_groups, st)) ||
        (rc = b_bk.alloc(sizeof(uint32_t) * SEL_LISTS * n_groups, st)) ||
        (rc = b_off.alloc(sizeof(int64_t) * SEL_LISTS * n_groups, st)) ||
        (rc = b_cap.alloc(sizeof(int64_t) * SEL_LISTS * n_groups, st)) ||
        (rc = b_fill.alloc(sizeof(unsigned long long) * SEL_LISTS * n_groups, st)) ||
        (rc = b_cand.alloc(sizeof(double) * std::max<int64_t>(total, 1), st)))
        return rc;
    cudaMemcpyAsync(b_nl.p, nlist.data(), b_nl.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_bk.p, bucket.data(), b_bk.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_off.p, off.data(), b_off.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_cap.p, cap.data(), b_cap.n, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(b_fill.p, 0, b_fill.n, st);
    cudaMemsetAsync(b_cand.p, 0xff, b_cand.n, st);  // CAND_SENTINEL
    compact_bucket_kernel<<<(unsigned)std::min<int64_t>((n_rows + 7) / 8, (int64_t)sm_count() * 16), 256, 0, st>>>(
        d_resp, n_rows, rv, ldr, rows_per_group, b_nl.as<int32_t>(), b_bk.as<uint32_t>(), b_off.as<int64_t>(),
        b_cap.as<int64_t>(), b_fill.as<unsigned long long>(), b_cand.as<double>());
    if ((rc = check_launch("compact_bucket_kernel"))) return rc;
    trace("  sel compact", st);
    if ((rc = run_rounds(slots, b_cand.as<double>(), 36, dist, st))) return rc;  // bits 47..0
    out.resize(slots.size());
    for (size_t i = 0; i < slots.size(); i++) memcpy(&out[i], &slots[i].prefix, 8);
    return CS_OK;
}

// Bit prefixes (62..36) of the sample order statistics at srank[g][i]
// (i < n_slots <= SB_SLOTS) over the logical view rv of every row.
static int sample_brackets(const double* d_resp, int64_t n_groups, int64_t rows_per_group, RowView rv,
                           int64_t ldr, const std::vector<int64_t>& srank, int n_slots,
                           std::vector<uint64_t>& out, bool dist, cudaStream_t st) {
    const int64_t n_rows = n_groups * rows_per_group;
    const size_t gs = (size_t)n_groups * SB_SLOTS;
    int rc;
    DBuf b_h0, b_bad, b_rank, b_bucket, b_resid, b_rep, b_h1, b_pref;
    if ((rc = b_h0.alloc(sizeof(uint32_t) * H0_BINS * (size_t)n_groups, st)) ||
        (rc = b_bad.alloc(sizeof(unsigned long long), st)) ||
        (rc = b_rank.alloc(sizeof(int64_t) * srank.size(), st)) ||
        (rc = b_bucket.alloc(sizeof(uint32_t) * gs, st)) || (rc = b_resid.alloc(sizeof(int64_t) * gs, st)) ||
        (rc = b_rep.alloc(sizeof(int32_t) * gs, st)) ||
        (rc = b_h1.alloc(sizeof(uint32_t) * H1_BINS * gs, st)) || (rc = b_pref.alloc(sizeof(uint64_t) * gs, st)))
        return rc;
    cudaMemsetAsync(b_h0.p, 0, b_h0.n, st);
    cudaMemsetAsync(b_bad.p, 0, b_bad.n, st);
    cudaMemsetAsync(b_h1.p, 0, b_h1.n, st);
    cudaMemcpyAsync(b_rank.p, srank.data(), b_rank.n, cudaMemcpyHostToDevice, st);
    cudaFuncSetAttribute(hist0_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * H0_BINS));
    hist0_rows_kernel<<<(int)std::min<int64_t>(n_rows, 2 * sm_count()), 1024, sizeof(uint32_t) * H0_BINS, st>>>(
        d_resp, n_rows, rv, ldr, rows_per_group, b_h0.as<uint32_t>(), b_bad.as<unsigned long long>());
    if ((rc = check_launch("hist0_rows_kernel"))) return rc;
    if (dist && ((rc = allreduce_u32(b_h0.p, (size_t)H0_BINS * n_groups, st)) ||
                 (rc = allreduce_u64(b_bad.p, 1, st))))
        return rc;
    cudaFuncSetAttribute(sb_select0_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * H0_BINS));
    sb_select0_kernel<<<(unsigned)n_groups, 1024, sizeof(uint32_t) * H0_BINS, st>>>(
        b_h0.as<uint32_t>(), n_slots, b_rank.as<int64_t>(), b_bucket.as<uint32_t>(), b_resid.as<int64_t>(),
        b_rep.as<int32_t>());
    if ((rc = check_launch("sb_select0_kernel"))) return rc;
    sb_hist1_kernel<<<(unsigned)std::min<int64_t>((n_rows + 7) / 8, (int64_t)sm_count() * 16), 256, 0, st>>>(
        d_resp, n_rows, rv, ldr, rows_per_group, n_slots, b_bucket.as<uint32_t>(), b_rep.as<int32_t>(),
        b_h1.as<uint32_t>());
    if ((rc = check_launch("sb_hist1_kernel"))) return rc;
    if (dist && (rc = allreduce_u32(b_h1.p, (size_t)H1_BINS * gs, st))) return rc;
    cudaFuncSetAttribute(sb_select1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * H1_BINS));
    sb_select1_kernel<<<(unsigned)(n_groups * n_slots), 1024, sizeof(uint32_t) * H1_BINS, st>>>(
        b_h1.as<uint32_t>(), n_slots, b_bucket.as<uint32_t>(), b_resid.as<int64_t>(), b_rep.as<int32_t>(),
        b_pref.as<uint64_t>());
    if ((rc = check_launch("sb_select1_kernel"))) return rc;
    std::vector<uint64_t> pref(gs);
    unsigned long long bad = 0;
    cudaMemcpyAsync(pref.data(), b_pref.p, b_pref.n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&bad, b_bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st);
    if ((rc = check_cuda(cudaStreamSynchronize(st), "sample brackets sync"))) return rc;
    if (bad) {
        set_error("cs_rep_stats: %llu negative responses (impossible for valid input)", bad);
        return CS_INTERNAL;
    }
    out.assign((size_t)n_groups * n_slots, 0);
    for (int64_t g = 0; g < n_groups; g++)
        for (int i = 0; i < n_slots; i++) out[g * n_slots + i] = pref[g * SB_SLOTS + i];
    return CS_OK;
}

// Split tree of numpy's pairwise sum for rows of m values (cached per m):
// leaves in order, and the internal nodes grouped by height (leaves 0): a
// node stores its value in its leftmost leaf's slot, so combining it is
// v[a] = v[a] + v[b] with a = its leftmost leaf, b = its right child's.
struct PairwisePlan {
    int64_t m = -1;
    std::vector<int32_t> leaf_off, leaf_len;
    std::vector<std::vector<int32_t>> by_height;  // (a, b) pairs per height - 1
};

// returns (height, leftmost leaf) of the subtree over [off, off + n)
static std::pair<int, int32_t> plan_build(PairwisePlan& pl, int64_t off, int64_t n) {
    if (n <= 128) {
        pl.leaf_off.push_back((int32_t)off);
        pl.leaf_len.push_back((int32_t)n);
        return {0, (int32_t)pl.leaf_off.size() - 1};
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const auto l = plan_build(pl, off, n2);
    const auto r = plan_build(pl, off + n2, n - n2);
    const int h = std::max(l.first, r.first) + 1;
    if ((int)pl.by_height.size() < h) pl.by_height.resize(h);
    pl.by_height[h - 1].push_back(l.second);
    pl.by_height[h - 1].push_back(r.second);
    return {h, l.second};
}

static const PairwisePlan& pairwise_plan(int64_t m) {
    static thread_local PairwisePlan pl;
    if (pl.m != m) {
        pl = PairwisePlan();
        pl.m = m;
        if (m > 0) plan_build(pl, 0, m);
    }
    return pl;
}

}  // namespace cs

using namespace cs;

extern "C" int cs_rep_stats_impl(const double* d_resp, int32_t n_groups, int64_t rows_per_group, int64_t m,
                                 int64_t ldr, cs_rep_summary* d_summ, const int64_t* ranks,
                                 int32_t n_ranks, double* out_values, double* d_row_sums, int32_t dist_flag,
                                 void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    // sharded: every rank holds rows_per_group rows of each group (equal shards);
    // ranks refer to the union over all ranks
    const bool dist = dist_flag && dist_active();
    const int64_t shards = dist ? dist_nranks() : 1;
    const int64_t n_rows = (int64_t)n_groups * rows_per_group;
    if (n_rows == 0 || m == 0) return CS_OK;
    if (ranks != nullptr && n_ranks > MAX_LISTS) {
        set_error("cs_rep_stats: at most %d ranks per group", MAX_LISTS);
        return CS_INVALID;
    }
    const bool want_ranks = ranks != nullptr && n_ranks > 0;
    const int64_t N = rows_per_group * m * shards;  // values per group (all shards)
    std::vector<int64_t> target(want_ranks ? (size_t)n_groups * n_ranks : 0);
    for (size_t i = 0; i < target.size(); i++) {
        int64_t k = ranks[i];
        if (k < 0) k += N;
        if (k < 0 || k >= N) {
            set_error("cs_rep_stats: rank out of range");
            return CS_INVALID;
        }
        target[i] = k;
    }
    int rc;
    // ---- pairwise plan (leaf offsets, lengths, height-ordered nodes) ----
    const PairwisePlan& pl = pairwise_plan(m);
    const int32_t L = (int32_t)pl.leaf_off.size();
    const int32_t n_heights = (int32_t)pl.by_height.size();
    const size_t plan_words = 2 * (size_t)L + n_heights + 1 + 2 * (size_t)std::max(L - 1, 0);
    const size_t plan_bytes = sizeof(int32_t) * plan_words;
    const int max_leaf = pl.leaf_len.empty() ? 0 : *std::max_element(pl.leaf_len.begin(), pl.leaf_len.end());
    const bool slots12 = max_leaf <= 96;  // 8 lanes x 12 slots cover every leaf's 8-aligned body
    const int t_slots = slots12 ? 12 : 16;
    // shared memory: the inside-value staging ring ([LB_WARPS][stg][32] doubles;
    // a deep ring keeps its hand-overs rare), the leaf sums when they fit
    // beside it with two blocks per SM (else a global scratch slice per
    // warp, L2-resident), the plan
    auto stage_bytes = [&](int stg) { return sizeof(double) * LB_WARPS * 32 * (size_t)stg; };
    const size_t lv_bytes = sizeof(double) * LB_WARPS * (size_t)L;
    const bool plan_in_smem = plan_bytes <= 32 * 1024;  // long rows (config 5: 160 KB): global, L1-cached
    const size_t plan_sm = plan_in_smem ? plan_bytes : 0;
    const bool leaves_in_smem = stage_bytes(t_slots + 28) + lv_bytes + plan_sm <= 110 * 1024;
    int stg = t_slots + 28;
    while (stg > t_slots + 3 && stage_bytes(stg) + (leaves_in_smem ? lv_bytes : 0) + plan_sm > 224 * 1024) stg--;
    const size_t smem = stage_bytes(stg) + (leaves_in_smem ? lv_bytes : 0) + plan_sm;
    if (smem > 224 * 1024) {
        set_error("cs_rep_stats: rows of %lld responses exceed the on-chip pairwise plan", (long long)m);
        return CS_UNSUPPORTED;
    }
    DBuf b_plan;
    if ((rc = b_plan.alloc(std::max<size_t>(sizeof(int32_t) * plan_words, 16), st))) return rc;
    {
        std::vector<int32_t> h;
        h.reserve(plan_words);
        h.insert(h.end(), pl.leaf_off.begin(), pl.leaf_off.end());
        h.insert(h.end(), pl.leaf_len.begin(), pl.leaf_len.end());
        int32_t acc = 0;
        for (int k = 0; k <= n_heights; k++) {
            h.push_back(acc);
            if (k < n_heights) acc += (int32_t)pl.by_height[k].size() / 2;
        }
        for (auto& v : pl.by_height) h.insert(h.end(), v.begin(), v.end());
        cudaMemcpyAsync(b_plan.p, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice, st);
        if ((rc = check_cuda(cudaStreamSynchronize(st), "plan upload"))) return rc;  // h dies here
    }
    for (auto k : {row_stats_kernel<3, 12>, row_stats_kernel<3, 16>, row_stats_kernel<MAX_LISTS, 12>,
                   row_stats_kernel<MAX_LISTS, 16>})
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 16));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n_rows + LB_WARPS - 1) / LB_WARPS,
                                                                   (int64_t)sm_count() * 8));
    DBuf b_leaf;  // long rows: leaf values in global scratch (one slice per resident warp)
    if (!leaves_in_smem && (rc = b_leaf.alloc(sizeof(double) * (size_t)blocks * LB_WARPS * (size_t)L, st)))
        return rc;
    double* leaf_scratch = leaves_in_smem ? nullptr : b_leaf.as<double>();
    int max_brackets = 0;  // set per bracket attempt; selects the kernel instance
    auto leaf_pass = [&](int do_bracket, const int32_t* nl, const uint64_t* lo, const uint64_t* hi,
                         const int64_t* off, const int64_t* cap, unsigned long long* fill,
                         unsigned long long* below, unsigned long long* inside, double* cand) {
        auto k = max_brackets <= 3 ? (slots12 ? row_stats_kernel<3, 12> : row_stats_kernel<3, 16>)
                                   : (slots12 ? row_stats_kernel<MAX_LISTS, 12> : row_stats_kernel<MAX_LISTS, 16>);
        k<<<blocks, LB_WARPS * 32, std::max<size_t>(smem, 16), st>>>(
            d_resp, n_rows, rows_per_group, ldr, m, b_plan.as<int32_t>(), L, d_summ, d_row_sums, do_bracket,
            nl, lo, hi, off, cap, fill, below, inside, cand, n_heights, leaf_scratch, stg, plan_in_smem ? 1 : 0);
        return check_launch("row_stats_kernel");
    };
    const RowView full{m, 40, 40};  // contiguous
    // one 32-byte sector (4 responses) of every 128: 1/32 of the bytes, and far
    // less autocorrelated (queueing makes consecutive responses similar) than
    // long chunks
    const int64_t n_chunks = m / 128, tail = std::min<int64_t>(4, m % 128);
    const RowView sample{n_chunks * 4 + tail, 2, 7};
    if (!want_ranks || N <= (1 << 20) || sample.len < 64) {
        if ((rc = leaf_pass(0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr)))
            return rc;
        if (!want_ranks) return CS_OK;
        std::vector<double> vals;  // small groups: exact selection over all values
        if ((rc = select_rows(d_resp, n_groups, rows_per_group, full, ldr, target, n_ranks, vals, dist, st)))
            return rc;
        for (size_t i = 0; i < vals.size(); i++) out_values[i] = vals[i];
        return CS_OK;
    }
    const int64_t NS = rows_per_group * sample.len * shards;  // sample size per group
    const size_t T = target.size();
    double widen = 1.0;
    for (int attempt = 0; attempt < 4; attempt++, widen *= 8.0) {
        // ---- 1. sample order statistics bracketing each target ----
        std::vector<int64_t> r_lo(T), r_hi(T);
        for (size_t i = 0; i < T; i++) {
            const double p = (double)target[i] / (double)N;
            const double ks = p * (double)NS;
            // 12 binomial sigmas: margin for the residual autocorrelation of the sample
            const double delta = widen * (12.0 * sqrt(ks * (1.0 - p) + 1.0) + 64.0);
            r_lo[i] = std::max<int64_t>(0, (int64_t)floor(ks - delta));
            r_hi[i] = std::min<int64_t>(NS - 1, (int64_t)ceil(ks + delta));
        }
        // both bracket ends of every target in ONE exact selection over the sample
        std::vector<int64_t> r_both((size_t)n_groups * 2 * n_ranks);
        for (int64_t g = 0; g < n_groups; g++)
            for (int q = 0; q < n_ranks; q++) {
                r_both[(g * 2 * n_ranks) + q] = r_lo[g * n_ranks + q];
                r_both[(g * 2 * n_ranks) + n_ranks + q] = r_hi[g * n_ranks + q];
            }
        std::vector<uint64_t> p_both, p_lo(T), p_hi(T);  // bit prefixes 62..36 of the sample statistics
        trace("begin", st);
        if ((rc = sample_brackets(d_resp, n_groups, rows_per_group, sample, ldr, r_both, 2 * n_ranks, p_both, dist,
                                  st)))
            return rc;
        trace("sample brackets", st);
        for (int64_t g = 0; g < n_groups; g++)
            for (int q = 0; q < n_ranks; q++) {
                p_lo[g * n_ranks + q] = p_both[g * 2 * n_ranks + q];
                p_hi[g * n_ranks + q] = p_both[g * 2 * n_ranks + n_ranks + q];
            }
        std::vector<int32_t> nlist(n_groups, 0);
        const size_t L6 = (size_t)n_groups * MAX_LISTS;
        std::vector<uint64_t> lo(L6, ~0ull), hi(L6, 0);
        std::vector<int> list_of(T);
        std::vector<int64_t> est(L6, 0);
        for (int64_t g = 0; g < n_groups; g++) {
            std::vector<int> idx(n_ranks);
            for (int q = 0; q < n_ranks; q++) idx[q] = q;
            // whole high-word ranges: the row pass classifies on the high 32 bits
            // alone (a sample statistic lies in [prefix, prefix + 2^36))
            auto a_of = [&](int q) { return r_lo[g * n_ranks + q] == 0 ? 0ull : p_lo[g * n_ranks + q] & ~0xffffffffull; };
            auto b_of = [&](int q) {
                return r_hi[g * n_ranks + q] == NS - 1 ? 0x7fffffffffffffffull : p_hi[g * n_ranks + q] | 0xfffffffffull;
            };
            std::sort(idx.begin(), idx.end(), [&](int x, int y) { return a_of(x) < a_of(y); });
            for (int q : idx) {
                const uint64_t a = a_of(q), b = b_of(q);
                int l = nlist[g] - 1;
                if (l >= 0 && a <= hi[g * MAX_LISTS + l]) {
                    hi[g * MAX_LISTS + l] = std::max(hi[g * MAX_LISTS + l], b);
                } else {
                    l = nlist[g]++;
                    lo[g * MAX_LISTS + l] = a;
                    hi[g * MAX_LISTS + l] = b;
                }
                list_of[g * n_ranks + q] = l;
                est[g * MAX_LISTS + l] += r_hi[g * n_ranks + q] - r_lo[g * n_ranks + q] + 1;
            }
        }
        std::vector<int64_t> off(L6, 0), cap(L6, 0);
        int64_t total = 0;
        int top_bit = 0;  // highest bit where some bracket's lo and hi differ
        for (int64_t g = 0; g < n_groups; g++)
            for (int l = 0; l < nlist[g]; l++) {
                const double scale = (double)N / (double)NS;
                // + the reserved-but-unused slots: < 2 chunks per row and list
                const int64_t c = std::min<int64_t>(N, (int64_t)(4.0 * est[g * MAX_LISTS + l] * scale) + 4096) +
                                  2 * CAND_CHUNK * rows_per_group;
                off[g * MAX_LISTS + l] = total;
                cap[g * MAX_LISTS + l] = c;
                total += c;
                const uint64_t d = lo[g * MAX_LISTS + l] ^ hi[g * MAX_LISTS + l];
                if (d) top_bit = std::max(top_bit, 63 - __builtin_clzll(d));
            }
        // ---- 2. the one full pass: leaf sums + bracket counts/compaction ----
        DBuf b_nl, b_lo, b_hi, b_off, b_cap, b_fill, b_below, b_inside, b_cand;
        if ((rc = b_nl.alloc(sizeof(int32_t) * n_groups, st)) || (rc = b_lo.alloc(8 * L6, st)) ||
            (rc = b_hi.alloc(8 * L6, st)) || (rc = b_off.alloc(8 * L6, st)) || (rc = b_cap.alloc(8 * L6, st)) ||
            (rc = b_fill.alloc(8 * L6, st)) || (rc = b_below.alloc(8 * L6, st)) || (rc = b_inside.alloc(8 * L6, st)) ||
            (rc = b_cand.alloc(sizeof(double) * std::max<int64_t>(total, 1), st)))
            return rc;
        cudaMemcpyAsync(b_nl.p, nlist.data(), b_nl.n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b_lo.p, lo.data(), b_lo.n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b_hi.p, hi.data(), b_hi.n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b_off.p, off.data(), b_off.n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b_cap.p, cap.data(), b_cap.n, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(b_fill.p, 0, b_fill.n, st);
        cudaMemsetAsync(b_below.p, 0, b_below.n, st);
        cudaMemsetAsync(b_inside.p, 0, b_inside.n, st);
        max_brackets = *std::max_element(nlist.begin(), nlist.end());
        trace("bracket setup", st);
        if ((rc = leaf_pass(1, b_nl.as<int32_t>(), b_lo.as<uint64_t>(), b_hi.as<uint64_t>(), b_off.as<int64_t>(),
                            b_cap.as<int64_t>(), b_fill.as<unsigned long long>(), b_below.as<unsigned long long>(), b_inside.as<unsigned long long>(),
                            b_cand.as<double>())))
            return rc;
        // fill = reserved slots (the candidate lists' lengths, sealed tails
        // included); inside = values actually inside the brackets
        std::vector<unsigned long long> fill(L6), below(L6), inside_all(L6), overflow(L6);
        cudaMemcpyAsync(fill.data(), b_fill.p, b_fill.n, cudaMemcpyDeviceToHost, st);
        if (!dist) {  // one read-back of all the counts
            cudaMemcpyAsync(inside_all.data(), b_inside.p, b_inside.n, cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(below.data(), b_below.p, b_below.n, cudaMemcpyDeviceToHost, st);
        }
        if ((rc = check_cuda(cudaStreamSynchronize(st), "bracket sync"))) return rc;
        for (size_t li = 0; li < L6; li++) overflow[li] = (int64_t)fill[li] > cap[li] ? 1 : 0;
        if (dist) {  // global below / inside counts and any-rank overflow: one all-reduce (sum)
            DBuf b_cnt3;
            if ((rc = b_cnt3.alloc(3 * 8 * L6, st))) return rc;
            char* c3 = (char*)b_cnt3.p;
            cudaMemcpyAsync(c3, b_below.p, 8 * L6, cudaMemcpyDeviceToDevice, st);
            cudaMemcpyAsync(c3 + 8 * L6, b_inside.p, 8 * L6, cudaMemcpyDeviceToDevice, st);
            cudaMemcpyAsync(c3 + 16 * L6, overflow.data(), 8 * L6, cudaMemcpyHostToDevice, st);
            if ((rc = allreduce_u64(c3, 3 * L6, st))) return rc;
            cudaMemcpyAsync(below.data(), c3, 8 * L6, cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(inside_all.data(), c3 + 8 * L6, 8 * L6, cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(overflow.data(), c3 + 16 * L6, 8 * L6, cudaMemcpyDeviceToHost, st);  // > 0: some rank
            if ((rc = check_cuda(cudaStreamSynchronize(st), "bracket sync 2"))) return rc;
        }
        trace("row pass+counts", st);
        // ---- 3. verify the brackets, exact rounds over the candidates ----
        const int first_shift = (top_bit / RD_BITS) * RD_BITS;  // digits cover bits <= top_bit
        const uint64_t keep = first_shift + RD_BITS >= 64 ? 0ull : ~((1ull << (first_shift + RD_BITS)) - 1);
        bool ok = true;
        std::vector<SelSlot> slots(T);
        for (size_t i = 0; i < T && ok; i++) {
            const int64_t g = (int64_t)i / n_ranks;
            const size_t li = g * MAX_LISTS + list_of[i];
            const int64_t k = target[i];
            if (overflow[li] || (int64_t)below[li] > k || k >= (int64_t)(below[li] + inside_all[li])) {
                if (getenv("CS_DEBUG_STATS"))
                    fprintf(stderr, "[cs_rep_stats] bracket miss: attempt %d slot %zu k=%lld below=%llu "
                            "fill=%llu local=%llu cap=%lld ovf=%llu lo=%016llx hi=%016llx dist=%d\n",
                            attempt, i, (long long)k, below[li], inside_all[li], fill[li], (long long)cap[li],
                            overflow[li], (unsigned long long)lo[li], (unsigned long long)hi[li], (int)dist);
                ok = false;
                break;
            }
            // the slot's own first digit: below its bracket's highest differing bit
            const uint64_t dlh = lo[li] ^ hi[li];
            const int tb = dlh ? 63 - __builtin_clzll(dlh) : 0;
            const int sh0 = std::min(first_shift, (tb / RD_BITS) * RD_BITS);
            const uint64_t keep_s = sh0 + RD_BITS >= 64 ? 0ull : ~((1ull << (sh0 + RD_BITS)) - 1);
            slots[i].shift0 = sh0;
            slots[i].prefix = lo[li] & keep_s;  // bits shared by every candidate of the bracket
            slots[i].rank = k - (int64_t)below[li];
            slots[i].cand_off = off[li];
            slots[i].cand_len = (int64_t)fill[li];  // this rank's candidates
        }
        if (!ok) continue;  // the sample missed a target (or overflowed): widen, retry
        if ((rc = run_rounds(slots, b_cand.as<double>(), first_shift, dist, st))) return rc;
        trace("cand rounds", st);
        for (size_t i = 0; i < T; i++) memcpy(&out_values[i], &slots[i].prefix, 8);
        return CS_OK;
    }
    std::vector<double> vals;  // last resort: exact selection over everything
    if ((rc = select_rows(d_resp, n_groups, rows_per_group, full, ldr, target, n_ranks, vals, dist, st))) return rc;
    for (size_t i = 0; i < vals.size(); i++) out_values[i] = vals[i];
    return CS_OK;
}
