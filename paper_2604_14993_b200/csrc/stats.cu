// stats.cu -- run_sim aggregation over the stored responses (sim.py:406-438).
//
//  * per-replication responses.mean() (sim.py:407) is numpy's pairwise sum
//    (numpy/_core/src/umath/loops_utils.h.src, @TYPE@_pairwise_sum: blocks of
//    <=128 summed with 8 accumulators, larger ranges split at n/2 rounded down
//    to a multiple of 8) divided by the count.  The split tree depends only on
//    the row length m, so the host builds it once (leaves + post-order
//    internal nodes) and the device evaluates it: bit-exact with numpy.
//  * exact order statistics of each sweep point's merged responses (the values
//    np.quantile interpolates between, sim.py:436-438) by MSB-radix select on
//    the IEEE bit patterns (responses are >= +0, so bit order == value order):
//    digit 0 = bits 62..48 (15 bits) histogrammed in the SAME pass as the leaf
//    sums; then the selected digit-0 buckets are compacted and three 16-bit
//    digit rounds run on the candidates only.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "cs_internal.cuh"

namespace cs {

constexpr int H0_BITS = 15;
constexpr int H0_BINS = 1 << H0_BITS;
constexpr int HR_BINS = 1 << 16;

__device__ __forceinline__ uint64_t dbits(double v) { return (uint64_t)__double_as_longlong(v); }

// Leaf sum exactly as numpy's pairwise_sum for n <= 128.
__device__ __forceinline__ double leaf_sum(const double* __restrict__ a, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
    int i = 8;
    const int stop = n - (n % 8);
    for (; i < stop; i += 8) {
        const double2 v0 = *reinterpret_cast<const double2*>(a + i);
        const double2 v1 = *reinterpret_cast<const double2*>(a + i + 2);
        const double2 v2 = *reinterpret_cast<const double2*>(a + i + 4);
        const double2 v3 = *reinterpret_cast<const double2*>(a + i + 6);
        r0 = __dadd_rn(r0, v0.x);
        r1 = __dadd_rn(r1, v0.y);
        r2 = __dadd_rn(r2, v1.x);
        r3 = __dadd_rn(r3, v1.y);
        r4 = __dadd_rn(r4, v2.x);
        r5 = __dadd_rn(r5, v2.y);
        r6 = __dadd_rn(r6, v3.x);
        r7 = __dadd_rn(r7, v3.y);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

// Pass A: leaf sums of every (row, leaf) + digit-0 histogram per group.
__global__ void __launch_bounds__(1024) leaf_hist_kernel(
    const double* __restrict__ resp, int64_t n_rows, int64_t ldr, int64_t rows_per_group,
    const int32_t* __restrict__ leaf_off, const int32_t* __restrict__ leaf_len, int32_t L,
    double* __restrict__ leaf_sums, uint32_t* __restrict__ hist0, int do_hist,
    unsigned long long* __restrict__ n_negative) {
    extern __shared__ uint32_t sh[];  // H0_BINS counters
    const int64_t total = n_rows * L;
    const int64_t per_block = (total + gridDim.x - 1) / gridDim.x;
    const int64_t beg = (int64_t)blockIdx.x * per_block;
    const int64_t end = min(total, beg + per_block);
    if (beg >= end) return;
    const int64_t g_first = (beg / L) / rows_per_group;
    const int64_t g_last = ((end - 1) / L) / rows_per_group;
    for (int64_t g = g_first; g <= g_last; g++) {
        const int64_t gb = max(beg, g * rows_per_group * L);
        const int64_t ge = min(end, (g + 1) * rows_per_group * L);
        if (do_hist) {
            for (int b = threadIdx.x; b < H0_BINS; b += blockDim.x) sh[b] = 0;
            __syncthreads();
        }
        for (int64_t w = gb + threadIdx.x; w < ge; w += blockDim.x) {
            const int64_t row = w / L;
            const int leaf = (int)(w % L);
            const double* a = resp + row * ldr + leaf_off[leaf];
            const int n = leaf_len[leaf];
            leaf_sums[w] = leaf_sum(a, n);
            if (do_hist) {
                for (int i = 0; i < n; i++) {
                    const uint64_t u = dbits(a[i]);
                    if (u >> 63) {
                        atomicAdd(n_negative, 1ull);
                    } else {
                        atomicAdd(&sh[u >> 48], 1u);
                    }
                }
            }
        }
        if (do_hist) {
            __syncthreads();
            uint32_t* gh = hist0 + g * H0_BINS;
            for (int b = threadIdx.x; b < H0_BINS; b += blockDim.x)
                if (sh[b]) atomicAdd(&gh[b], sh[b]);
            __syncthreads();
        }
    }
}

// Pass A': combine leaf sums along the split tree (post-order), one thread per row.
__global__ void tree_combine_kernel(const double* __restrict__ leaf_sums, int32_t L,
                                    const int32_t* __restrict__ node_l, const int32_t* __restrict__ node_r,
                                    int32_t n_nodes, double* __restrict__ scratch, int64_t n_rows,
                                    int64_t m, cs_rep_summary* __restrict__ summ,
                                    double* __restrict__ row_sums) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n_rows) return;
    const double* ls = leaf_sums + row * L;
    double* sc = scratch + row * (int64_t)(n_nodes > 0 ? n_nodes : 1);
    double last = L > 0 ? ls[0] : 0.0;
    for (int q = 0; q < n_nodes; q++) {
        const int a = node_l[q], b = node_r[q];
        const double va = a < L ? ls[a] : sc[a - L];
        const double vb = b < L ? ls[b] : sc[b - L];
        last = __dadd_rn(va, vb);
        sc[q] = last;
    }
    if (row_sums) row_sums[row] = last;
    if (summ) {
        summ[row].resp_sum = last;
        summ[row].resp_mean = m > 0 ? __ddiv_rn(last, (double)m) : NAN;
    }
}

// Per-slot selection state.
struct SelSlot {
    uint64_t prefix;   // selected high bits so far (already shifted into place)
    int64_t rank;      // remaining rank within the candidates with that prefix
    int64_t cand_off;  // candidate list offset / length
    int64_t cand_len;
    int32_t group;
    int32_t list;      // candidate list id
};

// Pass B: compact the values of each group whose digit 0 equals one of the
// group's selected buckets (lists are distinct per (group, bucket)).
__global__ void compact_kernel(const double* __restrict__ resp, int64_t n_rows, int64_t m,
                               int64_t ldr, int64_t rows_per_group,
                               const int32_t* __restrict__ grp_nlist,
                               const uint32_t* __restrict__ grp_bucket,  // [g][6]
                               const int64_t* __restrict__ grp_off,      // [g][6]
                               unsigned long long* __restrict__ fill,    // [g][6]
                               double* __restrict__ cand) {
    const int lane = threadIdx.x & 31;
    for (int64_t row = blockIdx.x; row < n_rows; row += gridDim.x) {
        const int64_t g = row / rows_per_group;
        const int nl = grp_nlist[g];
        uint32_t bk[6];
#pragma unroll
        for (int q = 0; q < 6; q++) bk[q] = q < nl ? grp_bucket[g * 6 + q] : 0xffffffffu;
        const double* __restrict__ a = resp + row * ldr;
        // blockDim is a multiple of 32, so every warp runs the same trip count
        for (int64_t base = 0; base < m; base += blockDim.x) {
            const int64_t q0 = base + threadIdx.x;
            int list = -1;
            double v = 0.0;
            if (q0 < m) {
                v = a[q0];
                const uint32_t d0 = (uint32_t)(dbits(v) >> 48);
#pragma unroll
                for (int q = 0; q < 6; q++)
                    if (bk[q] == d0) list = (int)(g * 6 + q);
            }
            const unsigned active = __ballot_sync(0xffffffffu, list >= 0);
            if (list >= 0) {
                const unsigned peers = __match_any_sync(active, list);
                const int leader = __ffs(peers) - 1;
                const int rank_in = __popc(peers & ((1u << lane) - 1));
                unsigned long long basei = 0;
                if (lane == leader) basei = atomicAdd(&fill[list], (unsigned long long)__popc(peers));
                basei = __shfl_sync(peers, basei, leader);
                cand[grp_off[list] + (int64_t)basei + rank_in] = v;
            }
        }
    }
}

// Rounds 1..3: histogram of the 16-bit digit at `shift` over candidates whose
// bits above the digit equal the slot prefix.
__global__ void round_hist_kernel(const double* __restrict__ cand, const SelSlot* __restrict__ slots,
                                  int n_slots, int shift, uint32_t* __restrict__ hist) {
    const int s = blockIdx.y;
    if (s >= n_slots) return;
    const SelSlot sl = slots[s];
    const uint64_t hi_mask = ~((1ull << (shift + 16)) - 1);
    uint32_t* h = hist + (int64_t)s * HR_BINS;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < sl.cand_len;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = dbits(cand[sl.cand_off + i]);
        if ((u & hi_mask) == sl.prefix) atomicAdd(&h[(u >> shift) & 0xFFFF], 1u);
    }
}

// Select the bucket holding `rank` in each slot's histogram; one block per slot.
__global__ void __launch_bounds__(1024) round_select_kernel(SelSlot* __restrict__ slots, int n_slots,
                                                            int shift, const uint32_t* __restrict__ hist) {
    const int s = blockIdx.x;
    if (s >= n_slots) return;
    __shared__ unsigned long long part[1024];
    const uint32_t* h = hist + (int64_t)s * HR_BINS;
    const int per = HR_BINS / blockDim.x;
    unsigned long long acc = 0;
    for (int b = threadIdx.x * per; b < (threadIdx.x + 1) * per; b++) acc += h[b];
    part[threadIdx.x] = acc;
    __syncthreads();
    // inclusive scan (Hillis-Steele) over partials
    for (int d = 1; d < (int)blockDim.x; d <<= 1) {
        unsigned long long v = threadIdx.x >= (unsigned)d ? part[threadIdx.x - d] : 0ull;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    const long long rank = slots[s].rank;
    const unsigned long long before = threadIdx.x ? part[threadIdx.x - 1] : 0ull;
    if ((long long)before <= rank && rank < (long long)part[threadIdx.x]) {
        unsigned long long c = before;
        for (int b = threadIdx.x * per; b < (threadIdx.x + 1) * per; b++) {
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
struct PairwisePlan {
    std::vector<int32_t> leaf_off, leaf_len, node_l, node_r;
};

static int32_t build_plan(PairwisePlan& pl, int64_t off, int64_t n) {
    if (n <= 128) {
        pl.leaf_off.push_back((int32_t)off);
        pl.leaf_len.push_back((int32_t)n);
        return (int32_t)(pl.leaf_off.size() - 1);
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const int32_t a = build_plan(pl, off, n2);
    const int32_t b = build_plan(pl, off + n2, n - n2);
    pl.node_l.push_back(a);
    pl.node_r.push_back(b);
    return -(int32_t)pl.node_l.size();  // internal: encoded below
}

// Node ids: leaves 0..L-1, internal node q -> L + q.  build_plan returns
// negative ids for internal nodes; fix them up after the leaf count is known.
static PairwisePlan make_plan(int64_t m) {
    PairwisePlan pl;
    std::vector<int32_t> dummy;
    if (m <= 0) return pl;
    build_plan(pl, 0, m);
    const int32_t L = (int32_t)pl.leaf_off.size();
    for (auto& x : pl.node_l)
        if (x < 0) x = L + (-x - 1);
    for (auto& x : pl.node_r)
        if (x < 0) x = L + (-x - 1);
    return pl;
}

struct Buf {
    void* p = nullptr;
    size_t n = 0;
};

static int dmalloc(Buf& b, size_t bytes, cudaStream_t st) {
    b.n = bytes;
    if (bytes == 0) return CS_OK;
    return check_cuda(cudaMallocAsync(&b.p, bytes, st), "cudaMallocAsync");
}
static void dfree(Buf& b, cudaStream_t st) {
    if (b.p) cudaFreeAsync(b.p, st);
    b.p = nullptr;
}

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

}  // namespace cs

using namespace cs;

// Per-row numpy pairwise sums -> summ[row].resp_mean (and row_sums if given);
// optionally the digit-0 histogram (for the rank selection).
static int row_stats(const double* d_resp, int64_t n_rows, int64_t m, int64_t ldr,
                     int64_t rows_per_group, cs_rep_summary* d_summ, double* d_row_sums,
                     uint32_t* d_hist0, unsigned long long* d_neg, cudaStream_t st) {
    const PairwisePlan pl = make_plan(m);
    const int32_t L = (int32_t)pl.leaf_off.size();
    const int32_t NN = (int32_t)pl.node_l.size();
    Buf b_lo, b_ll, b_nl, b_nr, b_ls, b_sc;
    int rc = CS_OK;
    if ((rc = dmalloc(b_lo, sizeof(int32_t) * L, st)) || (rc = dmalloc(b_ll, sizeof(int32_t) * L, st)) ||
        (rc = dmalloc(b_nl, sizeof(int32_t) * (NN + 1), st)) ||
        (rc = dmalloc(b_nr, sizeof(int32_t) * (NN + 1), st)) ||
        (rc = dmalloc(b_ls, sizeof(double) * (size_t)n_rows * L, st)) ||
        (rc = dmalloc(b_sc, sizeof(double) * (size_t)n_rows * (NN > 0 ? NN : 1), st)))
        return rc;
    cudaMemcpyAsync(b_lo.p, pl.leaf_off.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_ll.p, pl.leaf_len.data(), sizeof(int32_t) * L, cudaMemcpyHostToDevice, st);
    if (NN) {
        cudaMemcpyAsync(b_nl.p, pl.node_l.data(), sizeof(int32_t) * NN, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(b_nr.p, pl.node_r.data(), sizeof(int32_t) * NN, cudaMemcpyHostToDevice, st);
    }
    const size_t smem = d_hist0 ? sizeof(uint32_t) * H0_BINS : 0;
    if (smem) cudaFuncSetAttribute(leaf_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t work = n_rows * L;
    int blocks = sm_count();
    if (work < (int64_t)blocks * 256) blocks = (int)std::max<int64_t>(1, (work + 255) / 256);
    leaf_hist_kernel<<<blocks, 1024, smem, st>>>(d_resp, n_rows, ldr, rows_per_group,
                                                 (const int32_t*)b_lo.p, (const int32_t*)b_ll.p, L,
                                                 (double*)b_ls.p, d_hist0, d_hist0 != nullptr, d_neg);
    if ((rc = check_launch("leaf_hist_kernel"))) return rc;
    tree_combine_kernel<<<(unsigned)((n_rows + 127) / 128), 128, 0, st>>>(
        (const double*)b_ls.p, L, (const int32_t*)b_nl.p, (const int32_t*)b_nr.p, NN, (double*)b_sc.p,
        n_rows, m, d_summ, d_row_sums);
    if ((rc = check_launch("tree_combine_kernel"))) return rc;
    dfree(b_lo, st);
    dfree(b_ll, st);
    dfree(b_nl, st);
    dfree(b_nr, st);
    dfree(b_ls, st);
    dfree(b_sc, st);
    return CS_OK;
}

extern "C" int cs_rep_stats_impl(const double* d_resp, int32_t n_groups, int64_t rows_per_group,
                                 int64_t m, int64_t ldr, cs_rep_summary* d_summ,
                                 const int64_t* ranks, int32_t n_ranks, double* out_values,
                                 double* d_row_sums, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n_rows = (int64_t)n_groups * rows_per_group;
    if (n_rows == 0 || m == 0) return CS_OK;
    if (n_ranks > 6) {
        set_error("cs_rep_stats: at most 6 ranks per group");
        return CS_INVALID;
    }
    const bool select = ranks != nullptr && n_ranks > 0;
    Buf b_h0, b_neg;
    int rc = CS_OK;
    if (select) {
        if ((rc = dmalloc(b_h0, sizeof(uint32_t) * H0_BINS * (size_t)n_groups, st)) ||
            (rc = dmalloc(b_neg, sizeof(unsigned long long), st)))
            return rc;
        cudaMemsetAsync(b_h0.p, 0, b_h0.n, st);
        cudaMemsetAsync(b_neg.p, 0, b_neg.n, st);
    }
    rc = row_stats(d_resp, n_rows, m, ldr, rows_per_group, d_summ, d_row_sums,
                   (uint32_t*)b_h0.p, (unsigned long long*)b_neg.p, st);
    if (rc || !select) {
        dfree(b_h0, st);
        dfree(b_neg, st);
        return rc;
    }
    // ---- digit 0 selection on the host (2 MB for 16 groups) ----
    std::vector<uint32_t> h0((size_t)H0_BINS * n_groups);
    unsigned long long neg = 0;
    cudaMemcpyAsync(h0.data(), b_h0.p, b_h0.n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&neg, b_neg.p, sizeof(neg), cudaMemcpyDeviceToHost, st);
    if ((rc = check_cuda(cudaStreamSynchronize(st), "rep_stats sync"))) return rc;
    if (neg) {
        set_error("cs_rep_stats: %llu negative responses (impossible for valid input)", neg);
        return CS_INTERNAL;
    }
    const int64_t n_vals = rows_per_group * m;
    std::vector<SelSlot> slots((size_t)n_groups * n_ranks);
    std::vector<int32_t> g_nlist(n_groups, 0);
    std::vector<uint32_t> g_bucket((size_t)n_groups * 6, 0xffffffffu);
    std::vector<int64_t> g_off((size_t)n_groups * 6, 0), g_len((size_t)n_groups * 6, 0);
    int64_t total_cand = 0;
    for (int g = 0; g < n_groups; g++) {
        const uint32_t* hg = h0.data() + (size_t)g * H0_BINS;
        for (int q = 0; q < n_ranks; q++) {
            int64_t rank = ranks[(size_t)g * n_ranks + q];
            if (rank < 0) rank += n_vals;
            if (rank < 0 || rank >= n_vals) {
                set_error("cs_rep_stats: rank out of range");
                return CS_INVALID;
            }
            int64_t c = 0;
            uint32_t b = 0;
            for (; b < (uint32_t)H0_BINS; b++) {
                if (c + hg[b] > (uint64_t)rank) break;
                c += hg[b];
            }
            int list = -1;
            for (int l = 0; l < g_nlist[g]; l++)
                if (g_bucket[g * 6 + l] == b) list = l;
            if (list < 0) {
                list = g_nlist[g]++;
                g_bucket[g * 6 + list] = b;
                g_off[g * 6 + list] = total_cand;
                g_len[g * 6 + list] = hg[b];
                total_cand += hg[b];
            }
            SelSlot& s = slots[(size_t)g * n_ranks + q];
            s.prefix = (uint64_t)b << 48;
            s.rank = rank - c;
            s.cand_off = g_off[g * 6 + list];
            s.cand_len = g_len[g * 6 + list];
            s.group = g;
            s.list = g * 6 + list;
        }
    }
    Buf b_nl, b_bk, b_off, b_fill, b_cand, b_slots, b_hist;
    const int n_slots = (int)slots.size();
    if ((rc = dmalloc(b_nl, sizeof(int32_t) * n_groups, st)) ||
        (rc = dmalloc(b_bk, sizeof(uint32_t) * 6 * n_groups, st)) ||
        (rc = dmalloc(b_off, sizeof(int64_t) * 6 * n_groups, st)) ||
        (rc = dmalloc(b_fill, sizeof(unsigned long long) * 6 * n_groups, st)) ||
        (rc = dmalloc(b_cand, sizeof(double) * (size_t)std::max<int64_t>(total_cand, 1), st)) ||
        (rc = dmalloc(b_slots, sizeof(SelSlot) * n_slots, st)) ||
        (rc = dmalloc(b_hist, sizeof(uint32_t) * HR_BINS * (size_t)n_slots, st)))
        return rc;
    cudaMemcpyAsync(b_nl.p, g_nlist.data(), b_nl.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_bk.p, g_bucket.data(), b_bk.n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_off.p, g_off.data(), b_off.n, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(b_fill.p, 0, b_fill.n, st);
    cudaMemcpyAsync(b_slots.p, slots.data(), b_slots.n, cudaMemcpyHostToDevice, st);
    compact_kernel<<<(unsigned)std::min<int64_t>(n_rows, (int64_t)sm_count() * 16), 256, 0, st>>>(d_resp, n_rows, m, ldr, rows_per_group,
                                                   (const int32_t*)b_nl.p, (const uint32_t*)b_bk.p,
                                                   (const int64_t*)b_off.p,
                                                   (unsigned long long*)b_fill.p, (double*)b_cand.p);
    if ((rc = check_launch("compact_kernel"))) return rc;
    for (int round = 1; round <= 3; round++) {
        const int shift = 48 - 16 * round;
        cudaMemsetAsync(b_hist.p, 0, b_hist.n, st);
        dim3 grid(std::max(1, sm_count() * 4 / std::max(1, n_slots)), n_slots);
        round_hist_kernel<<<grid, 256, 0, st>>>((const double*)b_cand.p, (const SelSlot*)b_slots.p,
                                                n_slots, shift, (uint32_t*)b_hist.p);
        if ((rc = check_launch("round_hist_kernel"))) return rc;
        round_select_kernel<<<n_slots, 1024, 0, st>>>((SelSlot*)b_slots.p, n_slots, shift,
                                                      (const uint32_t*)b_hist.p);
        if ((rc = check_launch("round_select_kernel"))) return rc;
    }
    cudaMemcpyAsync(slots.data(), b_slots.p, b_slots.n, cudaMemcpyDeviceToHost, st);
    rc = check_cuda(cudaStreamSynchronize(st), "rep_stats select sync");
    for (int s = 0; s < n_slots && rc == CS_OK; s++) {
        uint64_t u = slots[s].prefix;
        double v;
        memcpy(&v, &u, 8);
        out_values[s] = v;
    }
    dfree(b_h0, st);
    dfree(b_neg, st);
    dfree(b_nl, st);
    dfree(b_bk, st);
    dfree(b_off, st);
    dfree(b_fill, st);
    dfree(b_cand, st);
    dfree(b_slots, st);
    dfree(b_hist, st);
    return rc;
}
