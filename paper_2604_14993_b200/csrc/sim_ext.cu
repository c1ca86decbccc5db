// sim_ext.cu -- the rest of run_sim's signature on the GPU (SURVEY.md §8(f)
// rows 2-4): dedicated-queue baseline policies jsq / sa-jsq / jiq / sed
// (chainserve sim.py:104-117,279-286), sampled and trace-driven workloads
// (sim.py:161-178,199-203; workload.py:124-167) and the time-horizon Poisson
// mode (sim.py:146-158,187-190), all bit-exact with _simulate_once.
//
// Same execution model as jffc_sim_warp_kernel (one WARP per replication,
// in-service slots spread over the lanes in shared memory, warp argmin by
// REDUX.MIN on the finish time's bits, chain k owned by lane k % 32), with
// every size a runtime value and per-chain state in shared memory:
//  * dedicated policies: per-chain FIFO rings (job, arrival) in a global
//    workspace; the arrival decision is a lane-local best over owned chains
//    followed by REDUX.MIN (jsq: (z+q, k); jiq: first k with z+q < c, else
//    jsq; sed: ((z+q+1)/mu_k, k) compared on the double's bits, then k).
//  * time horizon: a pre-pass replays numpy's block generation (4096 gaps,
//    cumsum(block) + total) to find the block count (sizes start after the
//    last block), the arrivals <= t_end (at most n) and the warm-up index
//    (searchsorted(arrivals, cut, 'left')); the event loop then regenerates
//    the same arrival values with a block cursor.
//  * trace workloads: a job's duration on chain k is the reference's hop sum
//    sum_h [ tout*(rtt+ovh)/1000 + ((blk_ovh + pre*tin) + dec*(tout-1))/1000 * m_h ]
//    evaluated in hop order with the same IEEE operations.
//  * advance() keeps the reference's `dt > 0` guard (sampled / trace arrival
//    arrays are caller data).
#include <cuda_runtime.h>
#include <math.h>

#include "cs_internal.cuh"

extern "C" int cs_device_count(void);

namespace cs {

constexpr int EXT_WARPS = 4;
constexpr int64_t HBLK = 4096;  // numpy block size of the time-horizon mode (sim.py:151)

// arrival sequence of the Poisson modes: x_i = scale * S[i];
// POISSON: a_i = cumsum(x)_i; HORIZON: a_i = cumsum(block(i))_{i mod 4096} + total_{block(i)-1}
template <int WL>
struct ArrCursor {
    const double* g;
    double scale;
    int64_t idx;  // index of the next arrival
    double acc;   // running cumsum (within the current block for HORIZON)
    double base;  // HORIZON: total of the previous blocks (block[-1])
    __device__ void init(const double* gaps, double sc) {
        g = gaps;
        scale = sc;
        idx = 0;
        acc = 0.0;
        base = 0.0;
    }
    __device__ double next() {
        const double x = __dmul_rn(scale, __ldg(g + idx));
        if (WL == CS_WL_HORIZON) {
            if ((idx & (HBLK - 1)) == 0) {
                if (idx > 0) base = __dadd_rn(acc, base);
                acc = x;
            } else {
                acc = __dadd_rn(acc, x);
            }
            idx++;
            return __dadd_rn(acc, base);
        }
        acc = idx == 0 ? x : __dadd_rn(acc, x);
        idx++;
        return acc;
    }
};

struct ExtLayout {  // per-warp shared memory (doubles)
    int chains, spl;
    __device__ size_t words() const { return (size_t)chains * 5 + (size_t)spl * 96; }
};

template <int WL, bool DED, bool TRACE>
__global__ void __launch_bounds__(32 * EXT_WARPS) sim_ext_kernel(const cs_sim_ext_args a, int spl_max) {
    constexpr uint32_t FULL = 0xffffffffu;
    constexpr uint64_t JOB_MASK = (1ull << 40) - 1;
    extern __shared__ double xsm[];
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int32_t P = a.n_points;
    if (w >= (int64_t)P * a.n_reps) return;  // warp-uniform
    const int32_t r = (int32_t)(w / P);
    const int32_t p = (int32_t)(w % P);
    const int64_t o = (int64_t)p * a.n_reps_total + a.rep_begin + r;
    const int CH = a.max_chains;
    const ExtLayout L{CH, spl_max};
    double* base = xsm + (threadIdx.x >> 5) * L.words();
    double* inv_mu = base;
    double* busy = base + CH;
    double* rate = base + 2 * CH;
    int32_t* z = reinterpret_cast<int32_t*>(base + 3 * CH);
    int32_t* capk = z + CH;
    int32_t* qh = reinterpret_cast<int32_t*>(base + 4 * CH);
    int32_t* qt = qh + CH;
    double* sfin = base + 5 * CH + lane;
    uint64_t* skey = reinterpret_cast<uint64_t*>(sfin + spl_max * 32);
    double* srsp = sfin + spl_max * 64;

    const cs_sim_point pt = a.points[p];
    const int K = pt.n_chains;
    const int kpl = (K + 31) / 32;
    int c_lane = 0;
    for (int k = lane; k < K; k += 32) {
        rate[k] = a.rates[pt.chain_base + k];
        inv_mu[k] = __ddiv_rn(1.0, rate[k]);
        capk[k] = a.caps[pt.chain_base + k];
        busy[k] = 0.0;
        z[k] = 0;
        qh[k] = 0;
        qt[k] = 0;
        c_lane += capk[k];
    }
    const int spl = min(spl_max, (int)((__reduce_add_sync(FULL, (uint32_t)c_lane) + 31) / 32));
    const uint32_t occ_full = (1u << spl) - 1;
    for (int s = 0; s < spl; s++) sfin[s * 32] = INFINITY;
    uint32_t occ = 0;
    double lmf = INFINITY;
    int lms = 0;
    bool ltie = false;
    __syncwarp();

    // ---- the arrival sequence, n and warm-up of this replication
    const double scale = __ddiv_rn(1.0, pt.lam);
    const double* gaps = a.streams ? a.streams + (int64_t)r * a.lds : nullptr;
    int64_t n = a.n_jobs, warm = a.warm, size_off = a.n_jobs;
    if (WL == CS_WL_HORIZON) {  // sim.py:146-158,187-190
        ArrCursor<CS_WL_HORIZON> c;
        c.init(gaps, scale);
        const double t_end = a.horizon_time_s, cut = a.warmup_cut_s;
        double total = 0.0;
        int64_t count = 0, kept = 0, wc = 0;
        bool open = true;  // arrivals are nondecreasing: kept ones form a prefix
        while (total < t_end && count < a.n_jobs) {
            for (int64_t b = 0; b < HBLK; b++) {
                const double v = c.next();
                if (open && v <= t_end && kept < a.n_jobs) {
                    kept++;
                    wc += v < cut;
                } else {
                    open = false;
                }
            }
            total = __dadd_rn(c.acc, c.base);
            count += HBLK;
        }
        n = kept;
        warm = wc;
        size_off = count;  // sizes = exponential(1.0, n) after every block draw
        int status = CS_OK;
        if (n == 0)
            status = CS_REP_EMPTY_HORIZON;
        else if (warm >= n)
            status = CS_REP_WARMUP_ALL;
        if (lane == 0) {
            if (a.rep_jobs) a.rep_jobs[o] = n;
            a.rep_status[o] = status;
        }
        if (status != CS_OK) return;
    } else if (lane == 0) {
        if (a.rep_jobs) a.rep_jobs[o] = n;
        a.rep_status[o] = CS_OK;
    }
    const double* sizes = (WL == CS_WL_SAMPLED) ? a.sizes : (gaps ? gaps + size_off : nullptr);
    ArrCursor<WL == CS_WL_HORIZON ? CS_WL_HORIZON : CS_WL_POISSON> lead, lag;
    if (WL <= CS_WL_HORIZON) {
        lead.init(gaps, scale);
        lag.init(gaps, scale);
    }
    double* __restrict__ rp = a.responses ? a.responses + o * a.ldr : nullptr;
    double* __restrict__ jrow = TRACE ? a.jobs + o * a.n_jobs * 4 : nullptr;
    double2* ring = DED ? reinterpret_cast<double2*>(a.queue_workspace) +
                              (size_t)w * CH * (size_t)a.queue_capacity
                        : nullptr;
    const int32_t qmask = a.queue_capacity - 1;

    const int64_t nm1 = n - 1, mid = warm + (n - warm) / 2;
    int64_t i = 0, s_next = 0, n_resp = 0, n_sys = 0, end_queue = 0;
    int cnt = 0;
    bool started = false, overflow = false;
    double t_arr = (WL <= CS_WL_HORIZON) ? lead.next() : a.arrivals[0];
    double last_t = 0.0, area = 0.0, wait_sum = 0.0, service_sum = 0.0;
    double w_start = NAN, t_mid = NAN, area_mid = NAN, t_end = NAN, area_end = NAN;

    for (int64_t ev = 0; ev < 2 * n; ev++) {
        const uint64_t fb = (uint64_t)__double_as_longlong(lmf);
        const uint32_t fhi = (uint32_t)(fb >> 32), flo = (uint32_t)fb;
        const uint32_t mhi = __reduce_min_sync(FULL, fhi);
        const uint32_t mlo = __reduce_min_sync(FULL, fhi == mhi ? flo : FULL);
        const double F = __longlong_as_double((long long)(((uint64_t)mhi << 32) | mlo));
        const bool comp = cnt > 0 && F <= t_arr;  // sim.py:259
        const double t = comp ? F : t_arr;
        const double dt = __dsub_rn(t, last_t);
        if (dt > 0.0) {  // advance (sim.py:224-231)
            area = __dadd_rn(area, __dmul_rn((double)n_sys, dt));
            for (int m = 0; m < kpl; m++) {
                const int k = lane + 32 * m;
                if (k < K) busy[k] = __dadd_rn(busy[k], __dmul_rn((double)z[k], dt));
            }
            last_t = t;
        }
        bool start;
        int kk;
        int64_t jj;
        double a_j;
        if (comp) {
            const bool cand = fhi == mhi && flo == mlo;
            uint32_t tied = __ballot_sync(FULL, cand);
            if ((tied & (tied - 1)) || __any_sync(FULL, cand && ltie)) {
                uint64_t kmin = ~0ull;
                if (cand) {
                    for (int s = 0; s < spl; s++)
                        if (sfin[s * 32] == lmf && skey[s * 32] < kmin) {
                            kmin = skey[s * 32];
                            lms = s;
                        }
                }
                const uint32_t khi = __reduce_min_sync(FULL, (uint32_t)(kmin >> 32));
                const uint32_t klo =
                    __reduce_min_sync(FULL, (uint32_t)(kmin >> 32) == khi ? (uint32_t)kmin : FULL);
                tied = __ballot_sync(FULL, cand && kmin == (((uint64_t)khi << 32) | klo));
            }
            const int wl = __ffs(tied) - 1;
            uint32_t info = 0;
            if (lane == wl) {
                const uint64_t kw = skey[lms * 32];
                const double rv = srsp[lms * 32];
                sfin[lms * 32] = INFINITY;
                occ &= ~(1u << lms);
                const bool counted = (int64_t)(kw & JOB_MASK) >= warm;
                if (counted && rp) rp[n_resp] = rv;  // finish_job (sim.py:244-252)
                info = ((uint32_t)(kw >> 40) << 1) | (counted ? 1u : 0u);
                double mn = INFINITY;
                int mi = 0;
                bool tie = false;
                for (int s = 0; s < spl; s++) {
                    const double f = sfin[s * 32];
                    const bool lt = f < mn;
                    tie = lt ? false : (tie || f == mn);
                    mn = lt ? f : mn;
                    mi = lt ? s : mi;
                }
                lmf = mn;
                lms = mi;
                ltie = tie;
            }
            info = __shfl_sync(FULL, info, wl);
            const int kc = (int)(info >> 1);
            n_resp += info & 1;
            if ((kc & 31) == lane) z[kc]--;
            cnt--;
            n_sys--;
            kk = kc;
            if (DED) {  // head of chain kc's own queue (sim.py:262-265)
                int has = 0;
                double2 e = make_double2(0.0, 0.0);
                if ((kc & 31) == lane && qt[kc] > qh[kc]) {
                    e = ring[(size_t)kc * a.queue_capacity + (qh[kc] & qmask)];
                    qh[kc]++;
                    has = 1;
                }
                start = __shfl_sync(FULL, has, kc & 31) != 0;
                a_j = __shfl_sync(FULL, e.x, kc & 31);
                jj = (int64_t)__double_as_longlong(__shfl_sync(FULL, e.y, kc & 31));
            } else {  // head of the central queue (contiguous range [s_next, i))
                start = s_next < i;
                jj = s_next;
                if (start) {
                    if (WL <= CS_WL_HORIZON)
                        a_j = lag.next();
                    else
                        a_j = __ldg(a.arrivals + s_next);
                } else {
                    a_j = 0.0;
                }
            }
        } else {
            if (i == warm && !started) {  // sim.py:269-275
                started = true;
                w_start = t;
                last_t = t;
                area = 0.0;
                for (int m = 0; m < kpl; m++)
                    if (lane + 32 * m < K) busy[lane + 32 * m] = 0.0;
            }
            n_sys++;
            jj = i;
            a_j = t;
            if (!DED) {  // fastest free chain (sim.py:278)
                uint32_t cand = FULL;
                for (int m = kpl - 1; m >= 0; m--) {
                    const int k = lane + 32 * m;
                    if (k < K && z[k] < capk[k]) cand = (uint32_t)k;
                }
                const uint32_t kf = __reduce_min_sync(FULL, cand);
                start = kf != FULL;
                kk = (int)kf;
                if (start && WL <= CS_WL_HORIZON) lag = lead;  // job i starts now: lag catches up
            } else {     // policy_step (sim.py:104-117)
                uint32_t tbest = FULL, kbest = FULL, idle = FULL;
                double vbest = INFINITY;
                for (int m = 0; m < kpl; m++) {
                    const int k = lane + 32 * m;
                    if (k >= K) break;
                    const uint32_t tot = (uint32_t)(z[k] + (qt[k] - qh[k]));
                    if (a.policy == CS_POLICY_SED) {
                        const double v = __ddiv_rn((double)(tot + 1), rate[k]);
                        if (v < vbest) {  // k ascending: first of equals kept
                            vbest = v;
                            kbest = (uint32_t)k;
                        }
                    } else {
                        if (tot < tbest) {
                            tbest = tot;
                            kbest = (uint32_t)k;
                        }
                        if (idle == FULL && (int)tot < capk[k]) idle = (uint32_t)k;
                    }
                }
                uint32_t target;
                if (a.policy == CS_POLICY_SED) {
                    const uint64_t vb = (uint64_t)__double_as_longlong(vbest);
                    const uint32_t vh = __reduce_min_sync(FULL, (uint32_t)(vb >> 32));
                    const uint32_t vl = __reduce_min_sync(FULL, (uint32_t)(vb >> 32) == vh ? (uint32_t)vb : FULL);
                    target = __reduce_min_sync(FULL, vb == (((uint64_t)vh << 32) | vl) ? kbest : FULL);
                } else {
                    target = FULL;
                    if (a.policy == CS_POLICY_JIQ) target = __reduce_min_sync(FULL, idle);
                    if (target == FULL) {
                        const uint32_t tm = __reduce_min_sync(FULL, tbest);
                        target = __reduce_min_sync(FULL, tbest == tm ? kbest : FULL);
                    }
                }
                kk = (int)target;
                int can = 0;
                if ((kk & 31) == lane) {
                    can = z[kk] < capk[kk];
                    if (!can) {  // parked in its dedicated queue (sim.py:282-284)
                        if (qt[kk] - qh[kk] > qmask) {
                            overflow = true;
                        } else {
                            ring[(size_t)kk * a.queue_capacity + (qt[kk] & qmask)] =
                                make_double2(t, __longlong_as_double((long long)i));
                            qt[kk]++;
                        }
                    }
                }
                start = __shfl_sync(FULL, can, kk & 31) != 0;
            }
            if (i == mid) {  // sim.py:291-295
                t_mid = t;
                area_mid = area;
            }
            if (i == nm1) {
                t_end = t;
                area_end = area;
                for (int m = 0; m < kpl; m++) {
                    const int k = lane + 32 * m;
                    if (k < K) a.busy[o * a.ldb + k] = busy[k];
                }
                if (DED) {
                    int ql = 0;
                    for (int m = 0; m < kpl; m++) {
                        const int k = lane + 32 * m;
                        if (k < K) ql += qt[k] - qh[k];
                    }
                    end_queue = (int64_t)__reduce_add_sync(FULL, (uint32_t)ql);
                } else {
                    end_queue = start ? 0 : (i + 1 - s_next);
                }
            }
            i++;
            if (i < n)
                t_arr = (WL <= CS_WL_HORIZON) ? lead.next() : __ldg(a.arrivals + i);
            else
                t_arr = INFINITY;
        }
        if (start) {  // start_job(jj, kk, t) (sim.py:233-242)
            double d;
            if (WL == CS_WL_TRACE) {  // ServiceTimeModel.request_service_time (workload.py:150-164)
                const int c = pt.chain_base + kk;
                const double tin = (double)__ldg(a.tokens_in + jj);
                const int32_t to = __ldg(a.tokens_out + jj);
                const double tout = (double)to, tout1 = (double)(to - 1);
                d = 0.0;
                for (int h = __ldg(a.hop_begin + c); h < __ldg(a.hop_begin + c + 1); h++) {
                    const double* sp = a.server_param + 4 * (size_t)__ldg(a.hop_server + h);
                    const double tc = __ddiv_rn(__dmul_rn(tout, __ldg(sp)), 1000.0);
                    const double tms = __dadd_rn(__dadd_rn(__ldg(sp + 1), __dmul_rn(__ldg(sp + 2), tin)),
                                                 __dmul_rn(__ldg(sp + 3), tout1));
                    d = __dadd_rn(d, tc);
                    d = __dadd_rn(d, __dmul_rn(__ddiv_rn(tms, 1000.0), (double)__ldg(a.hop_blocks + h)));
                }
            } else {
                d = __dmul_rn(__ldg(sizes + jj), inv_mu[kk]);
            }
            if ((kk & 31) == lane) z[kk]++;
            if (jj >= warm) {
                wait_sum = __dadd_rn(wait_sum, __dsub_rn(t, a_j));
                service_sum = __dadd_rn(service_sum, d);
            }
            const double f = __dadd_rn(t, d);
            const int tl = __ffs(__ballot_sync(FULL, occ != occ_full)) - 1;
            if (lane == tl) {
                const int slot = __ffs(~occ) - 1;
                sfin[slot * 32] = f;
                skey[slot * 32] = ((uint64_t)kk << 40) | (uint64_t)jj;
                srsp[slot * 32] = __dsub_rn(f, a_j);
                occ |= 1u << slot;
                if (f < lmf) {
                    lmf = f;
                    lms = slot;
                    ltie = false;
                } else if (f == lmf) {
                    ltie = true;
                }
            }
            if (TRACE && lane < 4)
                jrow[jj * 4 + lane] = lane == 0 ? a_j : (lane == 1 ? t : (lane == 2 ? f : (double)kk));
            cnt++;
            if (!DED) s_next++;
        }
        __syncwarp();
    }

    if (DED && __any_sync(FULL, overflow)) {
        if (lane == 0) a.rep_status[o] = CS_REP_QUEUE_OVERFLOW;
    }
    if (lane != 0) return;
    cs_rep_summary out;
    const double window = __dsub_rn(t_end, w_start);
    out.wait_sum = wait_sum;
    out.service_sum = service_sum;
    out.counted = n_resp;
    out.window_s = window;
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
    out.end_queue_len = end_queue;
    out.w_start = w_start;
    out.t_mid = t_mid;
    out.area_mid = area_mid;
    out.t_end = t_end;
    out.area_end = area_end;
    out.resp_sum = NAN;
    out.resp_mean = NAN;
    a.summary[o] = out;
}

// numpy pairwise_sum (loops_utils.h.src) of a[0:n]: leaves of <= 128 values
// (8 accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the remainder;
// < 8 values: 0.0 + sequential), split at n/2 rounded down to a multiple of 8.
__device__ double np_leaf(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
    for (int q = 0; q < 8; q++) r[q] = a[q];
    int64_t i = 8;
    for (; i < n - n % 8; i += 8)
        for (int q = 0; q < 8; q++) r[q] = __dadd_rn(r[q], a[i + q]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

// the recursion unrolled onto explicit stacks (device recursion would need
// a dynamic call stack): tasks are "evaluate [off, off+n)" or "combine the
// two values on top"; depth <= 3 per level, <= 40 levels for n < 2^46
__device__ double np_pairwise(const double* a, int64_t n) {
    int64_t t_off[128], t_n[128];  // t_n < 0: combine task
    double vals[64];
    int ts = 0, vs = 0;
    t_off[ts] = 0;
    t_n[ts++] = n;
    while (ts > 0) {
        ts--;
        const int64_t off = t_off[ts], m = t_n[ts];
        if (m < 0) {
            const double b = vals[--vs];
            const double l = vals[--vs];
            vals[vs++] = __dadd_rn(l, b);
        } else if (m <= 128) {
            vals[vs++] = np_leaf(a + off, m);
        } else {
            int64_t m2 = m / 2;
            m2 -= m2 % 8;
            t_off[ts] = 0;
            t_n[ts++] = -1;  // combine after both halves
            t_off[ts] = off + m2;
            t_n[ts++] = m - m2;
            t_off[ts] = off;
            t_n[ts++] = m2;  // left half first
        }
    }
    return vals[0];
}

// Ragged response rows (time-horizon mode: each replication simulates its
// own number of jobs): per-row numpy pairwise sums, and +inf padding past
// each row's count so the uniform-row order-statistic pass sees the padding
// above every response.
__global__ void ragged_rows_kernel(double* __restrict__ resp, int32_t n_rows, int64_t ldr,
                                   const int64_t* __restrict__ counts, double* __restrict__ sums) {
    const int row = blockIdx.x;
    if (row >= n_rows) return;
    double* a = resp + (int64_t)row * ldr;
    const int64_t c = counts[row];
    if (threadIdx.x == 0) sums[row] = np_pairwise(a, c);
    for (int64_t i = c + threadIdx.x; i < ldr; i += blockDim.x) a[i] = INFINITY;
}

template <int WL, bool DED>
static int launch_ext(const cs_sim_ext_args& a, int spl_max, cudaStream_t st) {
    const int64_t total = (int64_t)a.n_points * a.n_reps;
    const int blocks = (int)((total + EXT_WARPS - 1) / EXT_WARPS);
    const size_t smem = (size_t)EXT_WARPS * ((size_t)a.max_chains * 5 + (size_t)spl_max * 96) * sizeof(double);
    auto kern = a.jobs ? sim_ext_kernel<WL, DED, true> : sim_ext_kernel<WL, DED, false>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        set_error("cs_sim_ext: %zu bytes of shared memory per block unavailable", smem);
        return CS_UNSUPPORTED;
    }
    kern<<<blocks, 32 * EXT_WARPS, smem, st>>>(a, spl_max);
    return check_launch("sim_ext_kernel");
}

}  // namespace cs

extern "C" int cs_sim_ext(const cs_sim_ext_args* args, void* stream) {
    using namespace cs;
    if (cs_device_count() == 0) {
        set_error("cs_sim_ext: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (!args) {
        set_error("cs_sim_ext: null arguments");
        return CS_INVALID;
    }
    const cs_sim_ext_args& a = *args;
    if (a.n_points < 0 || a.n_reps < 0 || a.n_jobs < 1 || a.max_chains < 1 || a.max_capacity < 1 ||
        !a.points || !a.rates || !a.caps || !a.summary || !a.busy || !a.rep_status ||
        a.policy < CS_POLICY_JFFC || a.policy > CS_POLICY_SED || a.workload < CS_WL_POISSON ||
        a.workload > CS_WL_TRACE) {
        set_error("cs_sim_ext: invalid arguments");
        return CS_INVALID;
    }
    if (a.max_chains > 256 || a.max_capacity > 512 || a.n_jobs >= (1ll << 40)) {
        set_error("cs_sim_ext: K <= 256 chains and C <= 512 slots supported (got K=%d, C=%d)",
                  a.max_chains, a.max_capacity);
        return CS_UNSUPPORTED;
    }
    const bool ded = a.policy != CS_POLICY_JFFC;
    if (ded && (!a.queue_workspace || a.queue_capacity < 1 ||
                (a.queue_capacity & (a.queue_capacity - 1)) != 0)) {
        set_error("cs_sim_ext: dedicated policies need a queue workspace (power-of-two capacity)");
        return CS_INVALID;
    }
    if ((a.workload <= CS_WL_HORIZON && !a.streams) ||
        (a.workload == CS_WL_SAMPLED && (!a.arrivals || !a.sizes)) ||
        (a.workload == CS_WL_TRACE && (!a.arrivals || !a.tokens_in || !a.tokens_out || !a.hop_begin ||
                                       !a.hop_server || !a.hop_blocks || !a.server_param))) {
        set_error("cs_sim_ext: workload inputs missing");
        return CS_INVALID;
    }
    if ((int64_t)a.n_points * a.n_reps == 0) return CS_OK;
    const int spl_max = (a.max_capacity + 31) / 32;
    cudaStream_t st = (cudaStream_t)stream;
#define CS_EXT(WL)                                                        \
    return ded ? launch_ext<WL, true>(a, spl_max, st) : launch_ext<WL, false>(a, spl_max, st)
    switch (a.workload) {
        case CS_WL_POISSON: CS_EXT(CS_WL_POISSON);
        case CS_WL_HORIZON: CS_EXT(CS_WL_HORIZON);
        case CS_WL_SAMPLED: CS_EXT(CS_WL_SAMPLED);
        default: CS_EXT(CS_WL_TRACE);
    }
#undef CS_EXT
}

extern "C" int cs_ragged_rows(double* d_resp, int32_t n_rows, int64_t ldr, const int64_t* d_counts,
                              double* d_sums, void* stream) {
    using namespace cs;
    if (cs_device_count() == 0) {
        set_error("cs_ragged_rows: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (n_rows < 0 || ldr < 0 || (n_rows > 0 && (!d_resp || !d_counts || !d_sums))) {
        set_error("cs_ragged_rows: invalid arguments");
        return CS_INVALID;
    }
    if (n_rows == 0) return CS_OK;
    ragged_rows_kernel<<<n_rows, 256, 0, (cudaStream_t)stream>>>(d_resp, n_rows, ldr, d_counts, d_sums);
    return check_launch("ragged_rows_kernel");
}
