// compose.cu -- batched GBP-CR block placement and GCA chain composition.
//
// gbp_kernel: one CTA per composition point (placement.py:35-132).
//   m_j(c) = min(M_j // (s_m + s_c*c), L), t_j = tau_c + tau_p*m_j (mul, add);
//   block-wide bitonic sort of the m_j > 0 servers on (t_j / m_j, id rank)
//   (Python sorts by (float, str): the host passes the str order as a rank);
//   then the greedy chain scan (frontier arithmetic + sequential float sums)
//   by one thread, exactly as the reference's loop.
//
// gca_kernel: one CTA per placement (cache_alloc.py:65-135, model.py:130-231).
//   The routing graph is a DAG ordered by frontier f = a + m (an edge u->v
//   needs a_v <= f_u <= b_v < f_v).  Node labels are computed level by level in
//   increasing frontier: label(v) = min over live u of
//   (cost_u + w(u,v), path(u) ++ v) with Python tuple order; that equals the
//   reference's heap-Dijkstra keyed (cost, node-order tuple).
//   Live edge u->v  <=>  v == tail  or  resid_v >= b_v + 1 - f_u, i.e. the live
//   predecessors of v are the nodes whose frontier lies in
//   [max(a_v, b_v + 1 - resid_v), b_v]: contiguous frontier buckets.
//   Equal costs are broken by comparing the label paths through parent
//   pointers (first differing node order from the head).
//   Rounds after the first are incremental: a node's label is a function of
//   its live predecessor set and those predecessors' labels, so only nodes
//   whose live set shrank (the last chain's servers) or with a predecessor
//   whose label (cost, path) changed are recomputed; the others keep theirs.
//   Changed labels stamp their frontier bucket, and a node checks the stamps
//   of its predecessor buckets.  Same labels as the full DP, far fewer scans.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "cs_internal.cuh"

namespace cs {

// ---------------------------------------------------------------------------
// GBP-CR
// ---------------------------------------------------------------------------
struct SortKey {
    double amort;
    int32_t rank;
    int32_t idx;
};

__device__ __forceinline__ bool key_less(const SortKey& a, const SortKey& b) {
    return a.amort < b.amort || (a.amort == b.amort && a.rank < b.rank);
}

__global__ void __launch_bounds__(1024) gbp_kernel(
    const cs_compose_point* __restrict__ pts, const int64_t* __restrict__ mem,
    const double* __restrict__ tau_c, const double* __restrict__ tau_p,
    const int32_t* __restrict__ id_rank, int32_t* __restrict__ first, int32_t* __restrict__ count,
    int32_t* __restrict__ max_blocks, double* __restrict__ bound_time, int32_t* __restrict__ order,
    int32_t* __restrict__ chain_end, int32_t* __restrict__ n_chains, double* __restrict__ scaled_rate,
    int32_t* __restrict__ rate_satisfied, int32_t* __restrict__ status, int32_t sort_cap, int32_t mt_smem) {
    extern __shared__ SortKey keys[];  // sort_cap entries (power of two), then per server m_j, t_j
    int32_t* s_m = reinterpret_cast<int32_t*>(keys + sort_cap);
    double* s_t = reinterpret_cast<double*>(keys + sort_cap) + (sort_cap + 1) / 2;
    __shared__ int n_keys;
    const cs_compose_point pt = pts[blockIdx.x];
    const int J = pt.n_servers;
    const int64_t sb = pt.server_base;
    const int64_t L = pt.block_count;
    if (threadIdx.x == 0) n_keys = 0;
    __syncthreads();
    bool bad = pt.arrival_rate < 0.0 || !(0.0 < pt.load_target && pt.load_target < 1.0) ||
               pt.capacity < 1 || J > sort_cap;
    if (bad) {
        if (threadIdx.x == 0) {
            status[blockIdx.x] = CS_INVALID;
            n_chains[blockIdx.x] = 0;
        }
        return;
    }
    const int64_t per_block = pt.block_bytes + pt.cache_slot_bytes * pt.capacity;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        int64_t m = mem[sb + j] / per_block;
        if (m > L) m = L;
        const double t = __dadd_rn(tau_c[sb + j], __dmul_rn(tau_p[sb + j], (double)m));
        max_blocks[sb + j] = (int32_t)m;
        bound_time[sb + j] = t;
        if (mt_smem) {  // the greedy scan below reads them from shared memory
            s_m[j] = (int32_t)m;
            s_t[j] = t;
        }
        first[sb + j] = 0;
        count[sb + j] = 0;
        order[sb + j] = -1;
        chain_end[sb + j] = 0;
        if (m > 0) {
            const int q = atomicAdd(&n_keys, 1);
            keys[q].amort = __ddiv_rn(t, (double)m);
            keys[q].rank = id_rank[sb + j];
            keys[q].idx = j;
        }
    }
    __syncthreads();
    const int nk = n_keys;
    int P2 = 1;
    while (P2 < nk) P2 <<= 1;
    for (int q = nk + threadIdx.x; q < P2; q += blockDim.x) {
        keys[q].amort = INFINITY;
        keys[q].rank = 0x7fffffff;
        keys[q].idx = -1;
    }
    __syncthreads();
    // bitonic sort (ascending) of P2 keys; one key per thread (P2 == the
    // block): the exchanges with a partner in the same warp go through
    // shuffles (40 of a 1024-sort's 55 steps), the others through shared memory
    if (P2 == (int)blockDim.x) {
        const int i = threadIdx.x;
        SortKey my = keys[i];
        for (int k = 2; k <= P2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                SortKey o;
                if (j >= 32) {
                    __syncthreads();
                    keys[i] = my;
                    __syncthreads();
                    o = keys[i ^ j];
                } else {
                    o.amort = __shfl_xor_sync(0xffffffffu, my.amort, j);
                    o.rank = __shfl_xor_sync(0xffffffffu, my.rank, j);
                    o.idx = __shfl_xor_sync(0xffffffffu, my.idx, j);
                }
                const bool keep_min = ((i & k) == 0) == ((i & j) == 0);
                const bool o_less = key_less(o, my);
                if (keep_min == o_less) my = o;
            }
        }
        __syncthreads();
        keys[i] = my;
        __syncthreads();
    } else
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    SortKey a = keys[i], b = keys[ixj];
                    const bool swap = up ? key_less(b, a) : key_less(a, b);
                    if (swap) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x != 0) return;
    if (nk == 0) {
        status[blockIdx.x] = CS_INFEASIBLE;
        n_chains[blockIdx.x] = 0;
        scaled_rate[blockIdx.x] = 0.0;
        rate_satisfied[blockIdx.x] = 0;
        return;
    }
    const double target = __ddiv_rn(pt.arrival_rate, __dmul_rn(pt.load_target, (double)pt.capacity));
    int64_t frontier = 1;
    double chain_time = 0.0, rate = 0.0;
    int nch = 0, cur_begin = 0, q = 0;
    for (; q < nk; q++) {
        const int j = keys[q].idx;
        const int64_t m = mt_smem ? s_m[j] : max_blocks[sb + j];
        const int64_t a = frontier < L - m + 1 ? frontier : L - m + 1;
        first[sb + j] = (int32_t)a;
        count[sb + j] = (int32_t)m;
        order[sb + q] = j;
        chain_time = __dadd_rn(chain_time, mt_smem ? s_t[j] : bound_time[sb + j]);
        const int64_t fr = frontier + m - 1;
        frontier = (fr < L ? fr : L) + 1;
        if (frontier > L) {
            rate = __dadd_rn(rate, __ddiv_rn(1.0, chain_time));
            chain_end[sb + q] = 1;
            nch++;
            cur_begin = q + 1;
            if (rate >= target) {
                q++;
                break;
            }
            frontier = 1;
            chain_time = 0.0;
        }
    }
    for (int u = cur_begin; u < q; u++) {  // incomplete trailing chain is cleared
        const int j = keys[u].idx;
        first[sb + j] = 0;
        count[sb + j] = 0;
        order[sb + u] = -1;
    }
    n_chains[blockIdx.x] = nch;
    scaled_rate[blockIdx.x] = rate;
    rate_satisfied[blockIdx.x] = rate >= target;
    status[blockIdx.x] = CS_OK;
}

// ---------------------------------------------------------------------------
// GCA
// ---------------------------------------------------------------------------
struct GcaNode {
    int32_t fr, ra, rb;  // frontier, inclusive block range
    int32_t ord;         // node order for lexicographic ties (head 0 < ids < tail)
    int32_t srv;         // server index within the point (-1 for head/tail)
    int32_t parent;      // label parent (node index), -1 = none
    int32_t depth;       // label path length - 1
    int32_t pad;
    int64_t resid;
    double tc, tp;
    double cost;         // label cost, +inf = unreachable
};

// true iff path(u1) ++ v  <  path(u2) ++ v  (Python tuple order on node orders)
__device__ __forceinline__ bool lex_less(const GcaNode* __restrict__ nd, int u1, int u2, int v) {
    if (u1 == u2) return false;
    int a = u1, b = u2;
    int da = nd[a].depth, db = nd[b].depth;
    int a_below = -1, b_below = -1;  // node just below the current a/b on its path
    while (da > db) {
        a_below = a;
        a = nd[a].parent;
        da--;
    }
    while (db > da) {
        b_below = b;
        b = nd[b].parent;
        db--;
    }
    if (a == b) {
        // one path is a prefix of the other: the next element is compared with v
        if (a_below >= 0) return nd[a_below].ord < nd[v].ord;  // u2 is the prefix
        return nd[v].ord < nd[b_below].ord;                    // u1 is the prefix
    }
    while (nd[a].parent != nd[b].parent) {
        a = nd[a].parent;
        b = nd[b].parent;
    }
    return nd[a].ord < nd[b].ord;
}

// PySum (cs_internal.cuh): CPython >= 3.12 builtin sum() of floats.

#ifndef GCA_SPIN_NS
#define GCA_SPIN_NS 20  // back-off of a warp waiting for its predecessors' buckets
#endif

// Per-group scalars of the GCA body (a CTA, or one warp of a CTA).
struct GcaShared {
    int nodes, status;
    unsigned long long edges;
};

// One placement's GCA, run by a group: the whole CTA (WARP = false: large
// routing graphs, the warps share each round's nodes through per-bucket
// finish counters) or one warp (WARP = true: small graphs -- a moderate-rate
// placement uses ~90 of 1000 servers -- one instance per warp, many per CTA;
// the warp takes the nodes in bucket order itself, no waits).  Same labels,
// same chains either way.
template <bool WARP>
__device__ __forceinline__ void gca_body(
    const int p, unsigned char* __restrict__ smem, GcaShared* __restrict__ sh,
    const cs_compose_point* __restrict__ pts, const int64_t* __restrict__ mem,
    const double* __restrict__ tau_c, const double* __restrict__ tau_p,
    const int32_t* __restrict__ id_rank, const int32_t* __restrict__ first_all,
    const int32_t* __restrict__ count_all, const int64_t* __restrict__ residual, int32_t max_chains,
    int32_t max_hops, int32_t* __restrict__ chain_srv, int32_t* __restrict__ chain_len,
    int32_t* __restrict__ caps_out, double* __restrict__ times_out, int32_t* __restrict__ n_chains_out,
    int64_t* __restrict__ n_edges_out, int32_t* __restrict__ status_out, int32_t max_nodes,
    int32_t max_levels) {
    GcaNode* nd = reinterpret_cast<GcaNode*>(smem);
    int32_t* bucket = reinterpret_cast<int32_t*>(nd + max_nodes);  // nodes sorted by frontier
    int32_t* boff = bucket + max_nodes;                            // bucket offsets [0, L+3]
    int32_t* bcnt = boff + max_levels + 1;     // [max_levels] labels finished in a bucket, all rounds
    int32_t* dstamp = bcnt + max_levels;       // [max_levels] round in which a bucket had a label change
    int32_t* chstamp = dstamp + max_levels;    // [max_nodes] position -> round in which its label changed
    int32_t* rstamp = chstamp + max_nodes;     // [max_nodes] node -> round whose live predecessor set shrank
    int32_t* posn = rstamp + max_nodes;        // [max_nodes] node -> its position in `bucket`
    int32_t* pfr = posn + max_nodes;           // [max_nodes] position -> frontier of its node
    double* pcost = reinterpret_cast<double*>(((uintptr_t)(pfr + max_nodes) + 7) & ~(uintptr_t)7);  // position -> label cost
    const cs_compose_point pt = pts[p];
    const int J = pt.n_servers;
    const int64_t sb = pt.server_base;
    const int L = (int)pt.block_count;
    const int tid = WARP ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
    const int nthr = WARP ? 32 : (int)blockDim.x;
    const int lane = tid & 31, warp = WARP ? 0 : tid >> 5, nwarps = nthr >> 5;
    auto gsync = [&]() {
        if (WARP) __syncwarp();
        else __syncthreads();
    };

    if (tid == 0) {
        sh->status = CS_OK;
        sh->edges = 0;
        sh->nodes = 0;
    }
    gsync();
    // --- nodes: 0 = head, then used servers (server order), last = tail ---
    if (tid == 0) {
        int v = 1;
        for (int j = 0; j < J; j++) {
            if (count_all[sb + j] <= 0) continue;
            if (v >= max_nodes - 1) {
                sh->status = CS_INVALID;
                break;
            }
            GcaNode& n = nd[v];
            n.srv = j;
            n.ra = first_all[sb + j];
            n.rb = first_all[sb + j] + count_all[sb + j] - 1;
            n.fr = n.rb + 1;
            n.ord = id_rank[sb + j] + 1;
            n.tc = tau_c[sb + j];
            n.tp = tau_p[sb + j];
            const int64_t budget_bytes = mem[sb + j] - pt.block_bytes * (int64_t)count_all[sb + j];
            if (budget_bytes < 0) {
                sh->status = CS_INVALID;
                break;
            }
            const int64_t budget = budget_bytes / pt.cache_slot_bytes;
            if (residual) {
                const int64_t r = residual[sb + j];
                if (r < 0 || r > budget) {
                    sh->status = CS_INVALID;
                    break;
                }
                n.resid = r;
            } else {
                n.resid = budget;
            }
            v++;
        }
        GcaNode& h = nd[0];
        h.srv = -1;
        h.ra = 0;
        h.rb = 0;
        h.fr = 1;
        h.ord = 0;
        h.tc = h.tp = 0.0;
        h.resid = 0;
        GcaNode& t = nd[v];
        t.srv = -1;
        t.ra = L + 1;
        t.rb = L + 1;
        t.fr = L + 2;
        t.ord = 0x7fffffff;
        t.tc = t.tp = 0.0;
        t.resid = 0;
        sh->nodes = v + 1;
    }
    gsync();
    if (sh->status != CS_OK || L + 3 > max_levels) {
        if (tid == 0) {
            status_out[p] = CS_INVALID;
            n_chains_out[p] = 0;
            n_edges_out[p] = 0;
        }
        return;
    }
    const int V = sh->nodes, TAIL = V - 1;
    // --- bucket nodes by frontier (stable counting sort; V is small) ---
    if (tid == 0) {
        for (int f = 0; f <= L + 3; f++) boff[f] = 0;
        for (int v = 0; v < V; v++) boff[nd[v].fr]++;
        int acc = 0;
        for (int f = 0; f <= L + 3; f++) {
            const int c = boff[f];
            boff[f] = acc;
            acc += c;
        }
        for (int v = 0; v < V; v++) {
            const int e = boff[nd[v].fr]++;
            bucket[e] = v;
            posn[v] = e;
            pfr[e] = nd[v].fr;
        }
        for (int f = L + 3; f > 0; f--) boff[f] = boff[f - 1];
        boff[0] = 0;
    }
    gsync();
    // --- edge count (feasible_edges, model.py:179-187): sum_v |{u: a_v <= f_u <= b_v}| ---
    for (int v = 1 + tid; v < V; v += nthr) {
        const int lo = nd[v].ra, hi = nd[v].rb;
        atomicAdd(&sh->edges, (unsigned long long)(boff[hi + 1] - boff[lo]));
    }
    gsync();
    const int64_t E = (int64_t)sh->edges;
    for (int v = tid; v < V; v += nthr) {
        nd[v].cost = v == 0 ? 0.0 : INFINITY;
        nd[v].parent = -1;
        nd[v].depth = 0;
        chstamp[posn[v]] = -1;
        rstamp[v] = -1;
        pcost[posn[v]] = v == 0 ? 0.0 : INFINITY;
    }
    for (int f = tid; f < max_levels; f += nthr) {
        bcnt[f] = 0;
        dstamp[f] = -1;
    }
    gsync();
    int K = 0;
    int64_t it = 0;
    for (it = 0; it <= E; it++) {
        const int32_t its = (int32_t)it;
        // --- DP labels in frontier order, without block barriers: warp w takes
        //     the nodes at bucket positions boff[2] + w, + nwarps, ... in order
        //     and waits only for its live predecessors' labels of this round
        //     (lower positions: the lowest unfinished node can always go on):
        //     bucket f is final in round `it` once bcnt[f] = (it+1) x its size.
        //     Round 0 labels every node; later rounds recompute a node only if
        //     its live set shrank (the last chain's servers) or a predecessor's
        //     label changed (its bucket stamped), else it keeps its label. ---
        volatile int32_t* vcnt = bcnt;
        for (int e0 = boff[2] + warp; e0 < boff[L + 3]; e0 += nwarps) {
            const int v = bucket[e0];
            const GcaNode& nv = nd[v];
            int lo = nv.ra;
            if (v != TAIL) {
                const int64_t need = (int64_t)nv.rb + 1 - nv.resid;  // f_u >= need
                if (need > lo) lo = need > (int64_t)(L + 3) ? L + 3 : (int)need;
            }
            const int hi = nv.rb;
            const int p0 = lo <= hi ? boff[lo] : 0, p1 = lo <= hi ? boff[hi + 1] : 0;
            bool dirty = its == 0 || rstamp[v] == its;
            for (int fb = (lo > 2 ? lo : 2); fb <= hi; fb += 32) {  // bucket 1: the head, always final
                const int f = fb + lane;
                if (!WARP) {
                    const int need = f <= hi ? (its + 1) * (boff[f + 1] - boff[f]) : 0;
                    while (!__all_sync(0xffffffffu, f > hi || vcnt[f] >= need)) __nanosleep(GCA_SPIN_NS);
                    __threadfence_block();  // acquire: the predecessors' labels
                }
                dirty = dirty || __any_sync(0xffffffffu, f <= hi && dstamp[f] == its);
            }
            if (dirty) {
                // scan of the live predecessors by bucket position: their label
                // costs and frontiers sit in position order (no node lookup);
                // ties within a lane by path order (Python tuples)
                double best = INFINITY;
                int be = -1;  // best position
                for (int e = p0 + lane; e < p1; e += 32) {
                    const double cu = pcost[e];
                    if (!(cu < INFINITY)) continue;
                    const double w =
                        v == TAIL ? 0.0 : __dadd_rn(nv.tc, __dmul_rn(nv.tp, (double)(nv.rb + 1 - pfr[e])));
                    const double c = __dadd_rn(cu, w);
                    if (be < 0 || c < best || (c == best && lex_less(nd, bucket[e], bucket[be], v))) {
                        best = c;
                        be = e;
                    }
                }
                // warp argmin: costs are >= 0, so their bit patterns order as
                // the values; two 32-bit min-reductions, exact cost ties across
                // lanes (rare) by path order
                const uint64_t cb = be >= 0 ? (uint64_t)__double_as_longlong(best) : ~0ull;
                const uint32_t chi = (uint32_t)(cb >> 32);
                const uint32_t mhi = __reduce_min_sync(0xffffffffu, chi);
                const uint32_t mlo = __reduce_min_sync(0xffffffffu, chi == mhi ? (uint32_t)cb : 0xffffffffu);
                const unsigned wm = __ballot_sync(0xffffffffu, be >= 0 && chi == mhi && (uint32_t)cb == mlo);
                int bu = -1;
                if (wm) {
                    int bpos = __shfl_sync(0xffffffffu, be, __ffs(wm) - 1);
                    best = __shfl_sync(0xffffffffu, best, __ffs(wm) - 1);
                    for (unsigned m = wm & (wm - 1); m; m &= m - 1) {
                        const int cand = __shfl_sync(0xffffffffu, be, __ffs(m) - 1);
                        if (lex_less(nd, bucket[cand], bucket[bpos], v)) bpos = cand;
                    }
                    bu = bucket[bpos];
                }
                if (lane == 0) {
                    const int op = nd[v].parent;
                    const bool changed =
                        bu != op || (bu >= 0 && (best != nd[v].cost || chstamp[posn[bu]] == its));
                    if (changed) {
                        nd[v].cost = bu >= 0 ? best : INFINITY;
                        pcost[e0] = bu >= 0 ? best : INFINITY;
                        nd[v].parent = bu;
                        nd[v].depth = bu >= 0 ? nd[bu].depth + 1 : 0;
                        chstamp[e0] = its;
                        dstamp[nv.fr] = its;
                    }
                }
            }
            __syncwarp();
            if (!WARP && lane == 0) {
                __threadfence_block();  // release: the label before its count
                atomicAdd(&bcnt[nv.fr], 1);
            }
        }
        gsync();
        if (nd[TAIL].parent < 0) break;  // tail unreachable: allocation done
        // --- allocate the chain (one thread; cache_alloc.py:115-131) ---
        if (tid == 0) {
            const int len = nd[TAIL].depth - 1;  // real servers on the path
            if (K >= max_chains || len < 1 || len > max_hops) {
                sh->status = CS_INTERNAL;
            } else {
                int32_t* out = chain_srv + ((int64_t)p * max_chains + K) * max_hops;
                int v = nd[TAIL].parent;
                for (int h = len - 1; h >= 0; h--) {  // node indices, head->tail order
                    out[h] = v;
                    v = nd[v].parent;
                }
                int64_t cap = -1;
                int u = 0;
                for (int h = 0; h < len; h++) {
                    const int w = out[h];
                    const int64_t m = (int64_t)nd[w].rb + 1 - nd[u].fr;
                    const int64_t c = nd[w].resid / m;
                    if (cap < 0 || c < cap) cap = c;
                    u = w;
                }
                if (cap < 1) {
                    sh->status = CS_INTERNAL;  // "admissible hops must support at least one job"
                } else {
                    PySum T;
                    T.init();
                    u = 0;
                    for (int h = 0; h < len; h++) {
                        const int w = out[h];
                        const int64_t m = (int64_t)nd[w].rb + 1 - nd[u].fr;
                        T.add(__dadd_rn(nd[w].tc, __dmul_rn(nd[w].tp, (double)m)));
                        nd[w].resid -= m * cap;
                        rstamp[w] = (int32_t)(it + 1);  // live predecessor set shrinks next round
                        out[h] = nd[w].srv;
                        u = w;
                    }
                    T.add(0.0);  // hop into the tail costs 0.0
                    for (int h = len; h < max_hops; h++) out[h] = -1;
                    caps_out[(int64_t)p * max_chains + K] = (int32_t)cap;
                    times_out[(int64_t)p * max_chains + K] = T.result();
                    chain_len[(int64_t)p * max_chains + K] = len;
                }
            }
        }
        gsync();
        if (sh->status != CS_OK) break;
        K++;
    }
    if (tid == 0) {
        if (sh->status == CS_OK && it > E) sh->status = CS_INTERNAL;  // no termination
        status_out[p] = sh->status;
        n_chains_out[p] = K;
        n_edges_out[p] = E;
    }
}


__global__ void __launch_bounds__(512, 2) gca_kernel(
    const cs_compose_point* __restrict__ pts, const int64_t* __restrict__ mem,
    const double* __restrict__ tau_c, const double* __restrict__ tau_p,
    const int32_t* __restrict__ id_rank, const int32_t* __restrict__ first_all,
    const int32_t* __restrict__ count_all, const int64_t* __restrict__ residual, int32_t max_chains,
    int32_t max_hops, int32_t* __restrict__ chain_srv, int32_t* __restrict__ chain_len,
    int32_t* __restrict__ caps_out, double* __restrict__ times_out, int32_t* __restrict__ n_chains_out,
    int64_t* __restrict__ n_edges_out, int32_t* __restrict__ status_out, int32_t max_nodes,
    int32_t max_levels) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ GcaShared sh;
    gca_body<false>(blockIdx.x, smem, &sh, pts, mem, tau_c, tau_p, id_rank, first_all, count_all, residual,
                    max_chains, max_hops, chain_srv, chain_len, caps_out, times_out, n_chains_out, n_edges_out,
                    status_out, max_nodes, max_levels);
}

constexpr int GCA_GW = 8;  // instances (warps) per CTA of the warp form

__global__ void __launch_bounds__(32 * GCA_GW) gca_warp_kernel(
    int32_t n_points, size_t group_bytes, const cs_compose_point* __restrict__ pts,
    const int64_t* __restrict__ mem, const double* __restrict__ tau_c, const double* __restrict__ tau_p,
    const int32_t* __restrict__ id_rank, const int32_t* __restrict__ first_all,
    const int32_t* __restrict__ count_all, const int64_t* __restrict__ residual, int32_t max_chains,
    int32_t max_hops, int32_t* __restrict__ chain_srv, int32_t* __restrict__ chain_len,
    int32_t* __restrict__ caps_out, double* __restrict__ times_out, int32_t* __restrict__ n_chains_out,
    int64_t* __restrict__ n_edges_out, int32_t* __restrict__ status_out, int32_t max_nodes,
    int32_t max_levels) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ GcaShared sh[GCA_GW];
    const int w = threadIdx.x >> 5;
    const int p = blockIdx.x * GCA_GW + w;
    if (p >= n_points) return;  // whole warps: the body syncs only its own warp
    gca_body<true>(p, smem + (size_t)w * group_bytes, &sh[w], pts, mem, tau_c, tau_p, id_rank, first_all,
                   count_all, residual, max_chains, max_hops, chain_srv, chain_len, caps_out, times_out,
                   n_chains_out, n_edges_out, status_out, max_nodes, max_levels);
}

// Servers a placement uses (count > 0), max over the points: the routing
// graph's size, which picks the GCA form and sizes its shared memory.
__global__ void __launch_bounds__(256) used_servers_kernel(const cs_compose_point* __restrict__ pts,
                                                           const int32_t* __restrict__ count_all,
                                                           int32_t* __restrict__ max_used) {
    const cs_compose_point pt = pts[blockIdx.x];
    int c = 0;
    for (int j = threadIdx.x; j < pt.n_servers; j += blockDim.x) c += count_all[pt.server_base + j] > 0;
    for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
    __shared__ int part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += part[w];
        atomicMax(max_used, t);
    }
}

}  // namespace cs

using namespace cs;

extern "C" int cs_gbp_batch_impl(const cs_compose_point* d_points, int32_t n_points,
                                 int32_t max_servers, const int64_t* d_mem, const double* d_tau_c,
                                 const double* d_tau_p, const int32_t* d_id_rank, int32_t* d_first,
                                 int32_t* d_count, int32_t* d_max_blocks, double* d_bound_time,
                                 int32_t* d_order, int32_t* d_chain_end, int32_t* d_n_chains,
                                 double* d_scaled_rate, int32_t* d_rate_satisfied,
                                 int32_t* d_status, void* stream) {
    if (n_points <= 0) return CS_OK;
    int cap = 1;
    while (cap < max_servers) cap <<= 1;
    if (cap < 32) cap = 32;
    size_t smem = sizeof(SortKey) * cap + sizeof(double) * ((cap + 1) / 2 + cap);
    const int mt_smem = smem <= 200 * 1024;  // else the scan reads m_j, t_j from global memory
    if (!mt_smem) smem = sizeof(SortKey) * cap;
    if (smem > 200 * 1024) {
        set_error("cs_gbp_batch: %d servers per point exceeds the shared-memory sort (max 12800)",
                  max_servers);
        return CS_UNSUPPORTED;
    }
    cudaFuncSetAttribute(gbp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = cap >= 1024 ? 1024 : cap;
    gbp_kernel<<<n_points, threads, smem, (cudaStream_t)stream>>>(
        d_points, d_mem, d_tau_c, d_tau_p, d_id_rank, d_first, d_count, d_max_blocks, d_bound_time,
        d_order, d_chain_end, d_n_chains, d_scaled_rate, d_rate_satisfied, d_status, cap, mt_smem);
    return check_launch("gbp_kernel");
}

extern "C" int cs_gca_batch_impl(const cs_compose_point* d_points, int32_t n_points,
                                 int32_t max_servers, int32_t max_blocks_L, const int64_t* d_mem,
                                 const double* d_tau_c, const double* d_tau_p,
                                 const int32_t* d_id_rank, const int32_t* d_first,
                                 const int32_t* d_count, const int64_t* d_residual,
                                 int32_t max_chains, int32_t max_hops, int32_t* d_chain_srv,
                                 int32_t* d_chain_len, int32_t* d_caps, double* d_times,
                                 int32_t* d_n_chains, int64_t* d_n_edges, int32_t* d_status,
                                 void* stream) {
    if (n_points <= 0) return CS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int max_levels = max_blocks_L + 4;
    auto group_bytes = [&](int nodes) {  // the body's shared-memory layout for `nodes` nodes
        const size_t b = sizeof(GcaNode) * nodes + sizeof(int32_t) * (nodes + max_levels + 1) +
                         sizeof(int32_t) * (2 * (size_t)max_levels + 4 * (size_t)nodes) + sizeof(double) * nodes + 8;
        return (b + 15) & ~(size_t)15;
    };
    // nodes of the largest routing graph of the batch: used servers + head + tail
    int32_t used = max_servers;
    {
        int32_t* d_used = nullptr;
        if (cudaMallocAsync((void**)&d_used, sizeof(int32_t), st) == cudaSuccess) {
            cudaMemsetAsync(d_used, 0, sizeof(int32_t), st);
            used_servers_kernel<<<n_points, 256, 0, st>>>(d_points, d_count, d_used);
            cudaMemcpyAsync(&used, d_used, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
            cudaFreeAsync(d_used, st);
            if (cudaStreamSynchronize(st) != cudaSuccess) return check_launch("used_servers_kernel");
            used = std::min(used, max_servers);
        } else {
            cudaGetLastError();
        }
    }
    const size_t gw_bytes = group_bytes(used + 2);
    if (gw_bytes <= 24 * 1024) {  // small graphs: one instance per warp
        const size_t smem = gw_bytes * GCA_GW;
        cudaFuncSetAttribute(gca_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gca_warp_kernel<<<(n_points + GCA_GW - 1) / GCA_GW, 32 * GCA_GW, smem, st>>>(
            n_points, gw_bytes, d_points, d_mem, d_tau_c, d_tau_p, d_id_rank, d_first, d_count, d_residual,
            max_chains, max_hops, d_chain_srv, d_chain_len, d_caps, d_times, d_n_chains, d_n_edges, d_status,
            used + 2, max_levels);
        return check_launch("gca_warp_kernel");
    }
    // large graphs: one CTA per instance (sized by the fleet, as measured best:
    // fewer resident CTAs keep the waiting warps from crowding the SM)
    const int max_nodes = max_servers + 2;
    const size_t smem = group_bytes(max_nodes);
    if (smem > 220 * 1024) {
        set_error("cs_gca_batch: %d servers per point exceeds shared memory", max_servers);
        return CS_UNSUPPORTED;
    }
    cudaFuncSetAttribute(gca_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gca_kernel<<<n_points, 512, smem, st>>>(
        d_points, d_mem, d_tau_c, d_tau_p, d_id_rank, d_first, d_count, d_residual, max_chains,
        max_hops, d_chain_srv, d_chain_len, d_caps, d_times, d_n_chains, d_n_edges, d_status,
        max_nodes, max_levels);
    return check_launch("gca_kernel");
}
