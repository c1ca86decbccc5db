/*
 * cs_oracle.c -- CPU ORACLE (test infrastructure only; see cs_oracle.h).
 *
 * Plain-C restatement of the reference's hot path.  Compile with
 * -ffp-contract=off: Python never fuses a*b+c, so neither may we.
 * The ziggurat's rare branches call the host libm's log1p/exp exactly as
 * numpy's npy_log1p/exp do (numpy/random/src/distributions/distributions.c).
 */
#include "cs_oracle.h"
#include "zig_tables.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ======================================================================== */
/* SeedSequence  (numpy/random/bit_generator.pyx, DEFAULT_POOL_SIZE = 4)      */
/* ======================================================================== */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_POOL 4

static uint32_t ss_hashmix(uint32_t value, uint32_t* hc) {
    value ^= *hc;
    *hc *= SS_MULT_A;
    value *= *hc;
    value ^= value >> 16;
    return value;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

void orc_seedseq_key(const uint32_t* entropy, int n_entropy, const uint32_t* spawn,
                     int n_spawn, uint64_t key_out[2]) {
    /* get_assembled_entropy: run entropy zero-padded to the pool size when a
     * spawn key is present, then the spawn words. */
    uint32_t ent[64];
    int n = 0;
    for (int i = 0; i < n_entropy && n < 64; i++) ent[n++] = entropy[i];
    if (n_spawn > 0)
        while (n < SS_POOL) ent[n++] = 0u;
    for (int i = 0; i < n_spawn && n < 64; i++) ent[n++] = spawn[i];

    uint32_t pool[SS_POOL];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < SS_POOL; i++) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, &hc);
    for (int s = 0; s < SS_POOL; s++)
        for (int d = 0; d < SS_POOL; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = SS_POOL; s < n; s++)
        for (int d = 0; d < SS_POOL; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));

    /* generate_state(2, uint64) = 4 uint32 words viewed little-endian. */
    uint32_t w[4];
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < 4; i++) {
        uint32_t v = pool[i % SS_POOL];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    key_out[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    key_out[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

static int to_words(uint64_t v, uint32_t* out) {
    /* _int_to_uint32_array: little-endian 32-bit chunks, [0] for zero. */
    int n = 0;
    if (v == 0) out[n++] = 0;
    while (v > 0) {
        out[n++] = (uint32_t)(v & 0xffffffffu);
        v >>= 32;
    }
    return n;
}

void orc_philox_key(uint64_t seed, uint64_t rep, uint64_t key_out[2]) {
    uint32_t e[2], s[2];
    int ne = to_words(seed, e), ns = to_words(rep, s);
    orc_seedseq_key(e, ne, s, ns, key_out);
}

/* ======================================================================== */
/* Philox4x64-10 (Random123; numpy/random/src/philox/philox.h)                */
/* ======================================================================== */
#define PH_M0 0xD2E7470EE14C6C93ULL
#define PH_M1 0xCA5A826395121157ULL
#define PH_W0 0x9E3779B97F4A7C15ULL
#define PH_W1 0xBB67AE8584CAA73BULL

static inline uint64_t mulhilo(uint64_t a, uint64_t b, uint64_t* hi) {
    unsigned __int128 p = (unsigned __int128)a * b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
}

void orc_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += PH_W0;
            k1 += PH_W1;
        }
        uint64_t hi0, hi1;
        uint64_t lo0 = mulhilo(PH_M0, c0, &hi0);
        uint64_t lo1 = mulhilo(PH_M1, c2, &hi1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

typedef struct {
    uint64_t key[2];
    uint64_t ctr[4];
    uint64_t buf[4];
    int pos;
    int64_t words;
} ph_stream;

static void ph_init(ph_stream* s, const uint64_t key[2]) {
    s->key[0] = key[0];
    s->key[1] = key[1];
    s->ctr[0] = s->ctr[1] = s->ctr[2] = s->ctr[3] = 0;
    s->pos = 4;
    s->words = 0;
}

static inline uint64_t ph_next64(ph_stream* s) {
    s->words++;
    if (s->pos < 4) return s->buf[s->pos++];
    /* philox_next: increment the 256-bit counter, then generate. */
    if (++s->ctr[0] == 0)
        if (++s->ctr[1] == 0)
            if (++s->ctr[2] == 0) ++s->ctr[3];
    orc_philox4x64_10(s->ctr, s->key, s->buf);
    s->pos = 1;
    return s->buf[0];
}

static inline double ph_next_double(ph_stream* s) {
    return (double)(ph_next64(s) >> 11) * (1.0 / 9007199254740992.0);
}

void orc_philox_raw(const uint64_t key[2], int64_t n, uint64_t* out) {
    ph_stream s;
    ph_init(&s, key);
    for (int64_t i = 0; i < n; i++) out[i] = ph_next64(&s);
}

/* ======================================================================== */
/* Ziggurat standard exponential (numpy random_standard_exponential)          */
/* ======================================================================== */
static inline double bits2d(uint64_t b) {
    double d;
    memcpy(&d, &b, 8);
    return d;
}

static double zig_exp(ph_stream* s) {
    for (;;) {
        uint64_t ri = ph_next64(s);
        ri >>= 3;
        uint8_t idx = (uint8_t)(ri & 0xFF);
        ri >>= 8;
        double x = (double)ri * bits2d(CS_ZIG_WE_BITS[idx]);
        if (ri < CS_ZIG_KE[idx]) return x;
        if (idx == 0) return bits2d(CS_ZIG_EXP_R_BITS) - log1p(-ph_next_double(s));
        double fe0 = bits2d(CS_ZIG_FE_BITS[idx - 1]), fe1 = bits2d(CS_ZIG_FE_BITS[idx]);
        if ((fe0 - fe1) * ph_next_double(s) + fe1 < exp(-x)) return x;
    }
}

int64_t orc_standard_exponential(const uint64_t key[2], int64_t n, double* out) {
    ph_stream s;
    ph_init(&s, key);
    for (int64_t i = 0; i < n; i++) out[i] = zig_exp(&s);
    return s.words;
}

/* ======================================================================== */
/* JFFC discrete-event simulation (sim.py:_simulate_once, Poisson, jffc)      */
/* ======================================================================== */
typedef struct {
    double finish;
    int32_t k;
    int64_t j;
} ev;

static inline int ev_less(const ev* a, const ev* b) {
    if (a->finish != b->finish) return a->finish < b->finish;
    if (a->k != b->k) return a->k < b->k;
    return a->j < b->j;
}

static void heap_push(ev* h, int64_t* n, ev e) {
    int64_t i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!ev_less(&h[i], &h[p])) break;
        ev t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}

static ev heap_pop(ev* h, int64_t* n) {
    ev top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && ev_less(&h[l], &h[m])) m = l;
        if (r < *n && ev_less(&h[r], &h[m])) m = r;
        if (m == i) break;
        ev t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}

int orc_simulate_once(int K, const double* rates, const int32_t* caps, double lam, int64_t n,
                      double warmup_fraction, uint64_t seed, uint64_t rep, double* responses,
                      double* busy_out, double* jobs, orc_rep_summary* out) {
    if (K < 1 || n < 1 || !(lam > 0)) return ORC_INVALID;
    /* _materialize (sim.py:136-160): arrivals = cumsum(exponential(1/lam, n)),
     * sizes = exponential(1.0, n) drawn after all arrival draws. */
    double* arr = (double*)malloc(sizeof(double) * n);
    double* size = (double*)malloc(sizeof(double) * n);
    double* start_t = jobs ? (double*)malloc(sizeof(double) * n) : NULL;
    int32_t* z = (int32_t*)calloc(K, sizeof(int32_t));
    double* busy = (double*)calloc(K, sizeof(double));
    double* inv_mu = (double*)malloc(sizeof(double) * K);
    int64_t cap_total = 0;
    for (int k = 0; k < K; k++) cap_total += caps[k];
    ev* heap = (ev*)malloc(sizeof(ev) * (cap_total + 1));
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!arr || !size || !z || !busy || !inv_mu || !heap || !queue || (jobs && !start_t)) {
        free(arr); free(size); free(start_t); free(z); free(busy); free(inv_mu); free(heap); free(queue);
        return ORC_INTERNAL;
    }
    uint64_t key[2];
    orc_philox_key(seed, rep, key);
    ph_stream s;
    ph_init(&s, key);
    double scale = 1.0 / lam;
    double acc = 0.0;
    for (int64_t j = 0; j < n; j++) {
        double g = scale * zig_exp(&s);
        acc = (j == 0) ? g : acc + g;
        arr[j] = acc;
    }
    for (int64_t j = 0; j < n; j++) size[j] = 1.0 * zig_exp(&s);

    int64_t warm = (int64_t)(warmup_fraction * (double)n);
    int64_t mid = warm + (n - warm) / 2;
    for (int k = 0; k < K; k++) inv_mu[k] = 1.0 / rates[k];

    int64_t hn = 0, qh = 0, qt = 0;
    int64_t n_sys = 0, n_resp = 0, end_queue = 0;
    int started = 0;
    double last_t = 0.0, area = 0.0, w_start = NAN;
    double t_mid = NAN, area_mid = NAN, t_end = NAN, area_end = NAN;
    double wait_sum = 0.0, service_sum = 0.0;

#define ADVANCE(T)                                                   \
    do {                                                             \
        double dt_ = (T) - last_t;                                   \
        if (dt_ > 0.0) {                                             \
            area += (double)n_sys * dt_;                             \
            for (int k_ = 0; k_ < K; k_++) busy[k_] += (double)z[k_] * dt_; \
            last_t = (T);                                            \
        }                                                            \
    } while (0)

#define START_JOB(J, KK, T)                                          \
    do {                                                             \
        z[KK] += 1;                                                  \
        double d_ = size[J] * inv_mu[KK];                            \
        if (start_t) start_t[J] = (T);                               \
        if ((J) >= warm) {                                           \
            wait_sum += (T) - arr[J];                                \
            service_sum += d_;                                       \
        }                                                            \
        ev e_ = {(T) + d_, (KK), (J)};                               \
        heap_push(heap, &hn, e_);                                    \
    } while (0)

    int64_t i = 0;
    while (i < n || hn > 0) {
        double t_arr = i < n ? arr[i] : INFINITY;
        if (hn > 0 && heap[0].finish <= t_arr) {
            ev e = heap_pop(heap, &hn);
            double t = e.finish;
            ADVANCE(t);
            z[e.k] -= 1;
            n_sys -= 1;
            if (e.j >= warm) responses[n_resp++] = t - arr[e.j];
            if (jobs) {
                jobs[4 * e.j + 0] = arr[e.j];
                jobs[4 * e.j + 1] = start_t[e.j];
                jobs[4 * e.j + 2] = t;
                jobs[4 * e.j + 3] = (double)e.k;
            }
            if (qh < qt) {
                int64_t jj = queue[qh++];
                START_JOB(jj, e.k, t);
            }
            continue;
        }
        double t = t_arr;
        ADVANCE(t);
        if (i == warm && !started) {
            started = 1;
            w_start = t;
            last_t = t;
            area = 0.0;
            for (int k = 0; k < K; k++) busy[k] = 0.0;
        }
        n_sys += 1;
        int target = -1;
        for (int k = 0; k < K; k++)
            if (z[k] < caps[k]) {
                target = k;
                break;
            }
        if (target >= 0) {
            START_JOB(i, target, t);
        } else {
            queue[qt++] = i;
        }
        if (i == mid) {
            t_mid = t;
            area_mid = area;
        }
        if (i == n - 1) {
            t_end = t;
            area_end = area;
            for (int k = 0; k < K; k++) busy_out[k] = busy[k];
            end_queue = qt - qh;
        }
        i++;
    }
#undef ADVANCE
#undef START_JOB

    double window = t_end - w_start;
    out->wait_sum = wait_sum;
    out->service_sum = service_sum;
    out->counted = n_resp;
    out->window_s = window;
    if (window > 0) {
        out->mean_occupancy = area_end / window;
        out->lambda_effective = (double)(n - warm) / window;
    } else {
        out->mean_occupancy = NAN;
        out->lambda_effective = NAN;
    }
    out->occ_first_half = t_mid > w_start ? area_mid / (t_mid - w_start) : NAN;
    out->occ_second_half = t_end > t_mid ? (area_end - area_mid) / (t_end - t_mid) : NAN;
    out->end_queue_len = end_queue;
    out->w_start = w_start;
    out->t_mid = t_mid;
    out->area_mid = area_mid;
    out->t_end = t_end;
    out->area_end = area_end;

    free(arr); free(size); free(start_t); free(z); free(busy); free(inv_mu); free(heap); free(queue);
    return ORC_OK;
}

/* ======================================================================== */
/* _simulate_once with explicit inputs (sim.py:181-324, every policy):       */
/* arrivals[n] and per-(job, chain) durations come from the caller, who      */
/* restates _materialize / duration() (sim.py:136-178,199-203) in numpy.     */
/* dur: size-based when dur_kn == NULL (d = sizes[j] * (1.0/rates[k])), else */
/* dur_kn[j*K + k] (trace workloads).  policy: 0 jffc (central FIFO queue),  */
/* 1 jsq, 2 sa-jsq, 3 jiq, 4 sed (policy_step, sim.py:75-117; one FIFO per   */
/* chain).  Same outputs as orc_simulate_once.                               */
/* ======================================================================== */
static int policy_arrival(int policy, int K, const double* rates, const int32_t* caps,
                          const int32_t* z, const int64_t* qlen) {
    if (policy == 0) {
        for (int k = 0; k < K; k++)
            if (z[k] < caps[k]) return k;
        return -1;
    }
    int best = 0;
    if (policy == 4) { /* sed: min ((totals+1)/rates[k], k) */
        double bv = 0.0;
        for (int k = 0; k < K; k++) {
            double v = (double)(z[k] + qlen[k] + 1) / rates[k];
            if (k == 0 || v < bv) {
                bv = v;
                best = k;
            }
        }
        return best;
    }
    if (policy == 3) /* jiq: first idle (totals < caps), else jsq */
        for (int k = 0; k < K; k++)
            if (z[k] + qlen[k] < caps[k]) return k;
    int64_t bt = 0; /* jsq / sa-jsq: min (totals, k) */
    for (int k = 0; k < K; k++) {
        int64_t tot = z[k] + qlen[k];
        if (k == 0 || tot < bt) {
            bt = tot;
            best = k;
        }
    }
    return best;
}

int orc_simulate_ext(int K, const double* rates, const int32_t* caps, int policy, int64_t n,
                     int64_t warm, const double* arr, const double* sizes, const double* dur_kn,
                     double* responses, double* busy_out, double* jobs, orc_rep_summary* out) {
    if (K < 1 || n < 1 || warm < 0 || warm >= n || policy < 0 || policy > 4) return ORC_INVALID;
    double* start_t = (double*)malloc(sizeof(double) * n);
    int32_t* z = (int32_t*)calloc(K, sizeof(int32_t));
    double* busy = (double*)calloc(K, sizeof(double));
    double* inv_mu = (double*)malloc(sizeof(double) * K);
    int64_t cap_total = 0;
    for (int k = 0; k < K; k++) cap_total += caps[k];
    ev* heap = (ev*)malloc(sizeof(ev) * (cap_total + 1));
    /* queues: central (policy 0) or one per chain; each a FIFO of job ids,
     * stored as a chain-tagged array with per-chain linked order */
    int64_t* qnext = (int64_t*)malloc(sizeof(int64_t) * n);  /* next job of the same queue */
    int nq = policy == 0 ? 1 : K;
    int64_t* qhead = (int64_t*)malloc(sizeof(int64_t) * nq);
    int64_t* qtail = (int64_t*)malloc(sizeof(int64_t) * nq);
    int64_t* qlen = (int64_t*)calloc(K, sizeof(int64_t));
    if (!start_t || !z || !busy || !inv_mu || !heap || !qnext || !qhead || !qtail || !qlen) {
        free(start_t); free(z); free(busy); free(inv_mu); free(heap); free(qnext);
        free(qhead); free(qtail); free(qlen);
        return ORC_INTERNAL;
    }
    for (int q = 0; q < nq; q++) qhead[q] = qtail[q] = -1;
    for (int k = 0; k < K; k++) inv_mu[k] = 1.0 / rates[k];
    int64_t mid = warm + (n - warm) / 2;
    int64_t hn = 0, n_sys = 0, n_resp = 0, end_queue = 0, qtot = 0;
    int started = 0;
    double last_t = 0.0, area = 0.0, w_start = NAN;
    double t_mid = NAN, area_mid = NAN, t_end = NAN, area_end = NAN;
    double wait_sum = 0.0, service_sum = 0.0;

#define ADV(T)                                                                 \
    do {                                                                       \
        double dt_ = (T) - last_t;                                             \
        if (dt_ > 0.0) {                                                       \
            area += (double)n_sys * dt_;                                       \
            for (int k_ = 0; k_ < K; k_++) busy[k_] += (double)z[k_] * dt_;    \
            last_t = (T);                                                      \
        }                                                                      \
    } while (0)
#define START(J, KK, T)                                                        \
    do {                                                                       \
        z[KK] += 1;                                                            \
        double d_ = dur_kn ? dur_kn[(J) * K + (KK)] : sizes[J] * inv_mu[KK];   \
        start_t[J] = (T);                                                      \
        if ((J) >= warm) {                                                     \
            wait_sum += (T) - arr[J];                                          \
            service_sum += d_;                                                 \
        }                                                                      \
        ev e_ = {(T) + d_, (KK), (J)};                                         \
        heap_push(heap, &hn, e_);                                              \
    } while (0)

    int64_t i = 0;
    while (i < n || hn > 0) {
        double t_arr = i < n ? arr[i] : INFINITY;
        if (hn > 0 && heap[0].finish <= t_arr) {
            ev e = heap_pop(heap, &hn);
            double t = e.finish;
            ADV(t);
            z[e.k] -= 1;
            n_sys -= 1;
            if (e.j >= warm) responses[n_resp++] = t - arr[e.j];
            if (jobs) {
                jobs[4 * e.j + 0] = arr[e.j];
                jobs[4 * e.j + 1] = start_t[e.j];
                jobs[4 * e.j + 2] = t;
                jobs[4 * e.j + 3] = (double)e.k;
            }
            int q = policy == 0 ? 0 : e.k;
            if (qhead[q] >= 0) {
                int64_t jj = qhead[q];
                qhead[q] = qnext[jj];
                if (qhead[q] < 0) qtail[q] = -1;
                if (policy != 0) qlen[q]--;
                qtot--;
                START(jj, e.k, t);
            }
            continue;
        }
        double t = t_arr;
        ADV(t);
        if (i == warm && !started) {
            started = 1;
            w_start = t;
            last_t = t;
            area = 0.0;
            for (int k = 0; k < K; k++) busy[k] = 0.0;
        }
        n_sys += 1;
        int target = policy_arrival(policy, K, rates, caps, z, qlen);
        int q = -1;
        if (policy == 0) {
            if (target < 0) q = 0;
        } else if (z[target] >= caps[target]) {
            q = target;
        }
        if (q < 0) {
            START(i, target, t);
        } else {
            qnext[i] = -1;
            if (qtail[q] >= 0) qnext[qtail[q]] = i; else qhead[q] = i;
            qtail[q] = i;
            if (policy != 0) qlen[q]++;
            qtot++;
        }
        if (i == mid) {
            t_mid = t;
            area_mid = area;
        }
        if (i == n - 1) {
            t_end = t;
            area_end = area;
            for (int k = 0; k < K; k++) busy_out[k] = busy[k];
            end_queue = qtot;
        }
        i++;
    }
#undef ADV
#undef START
    double window = t_end - w_start;
    out->wait_sum = wait_sum;
    out->service_sum = service_sum;
    out->counted = n_resp;
    out->window_s = window;
    if (window > 0) {
        out->mean_occupancy = area_end / window;
        out->lambda_effective = (double)(n - warm) / window;
    } else {
        out->mean_occupancy = NAN;
        out->lambda_effective = NAN;
    }
    out->occ_first_half = t_mid > w_start ? area_mid / (t_mid - w_start) : NAN;
    out->occ_second_half = t_end > t_mid ? (area_end - area_mid) / (t_end - t_mid) : NAN;
    out->end_queue_len = end_queue;
    out->w_start = w_start;
    out->t_mid = t_mid;
    out->area_mid = area_mid;
    out->t_end = t_end;
    out->area_end = area_end;
    free(start_t); free(z); free(busy); free(inv_mu); free(heap); free(qnext);
    free(qhead); free(qtail); free(qlen);
    return ORC_OK;
}

typedef struct {
    int K;
    const double* rates;
    const int32_t* caps;
    double lam, wf;
    int64_t n, warm;
    uint64_t seed;
    int64_t rep_begin, rep_end, next;
    double *responses, *busy;
    orc_rep_summary* out;
    pthread_mutex_t mu;
    int status;
} reps_job;

static void* reps_worker(void* p) {
    reps_job* jb = (reps_job*)p;
    for (;;) {
        pthread_mutex_lock(&jb->mu);
        int64_t r = jb->next++;
        pthread_mutex_unlock(&jb->mu);
        if (r >= jb->rep_end) break;
        int64_t li = r - jb->rep_begin;
        int st = orc_simulate_once(jb->K, jb->rates, jb->caps, jb->lam, jb->n, jb->wf, jb->seed,
                                   (uint64_t)r, jb->responses + li * (jb->n - jb->warm),
                                   jb->busy + li * jb->K, NULL, jb->out + li);
        if (st != ORC_OK) jb->status = st;
    }
    return NULL;
}

int orc_simulate_reps(int K, const double* rates, const int32_t* caps, double lam, int64_t n,
                      double warmup_fraction, uint64_t seed, int64_t rep_begin, int64_t rep_end,
                      int n_threads, double* responses, double* busy, orc_rep_summary* out) {
    reps_job jb;
    jb.K = K;
    jb.rates = rates;
    jb.caps = caps;
    jb.lam = lam;
    jb.wf = warmup_fraction;
    jb.n = n;
    jb.warm = (int64_t)(warmup_fraction * (double)n);
    jb.seed = seed;
    jb.rep_begin = rep_begin;
    jb.rep_end = rep_end;
    jb.next = rep_begin;
    jb.responses = responses;
    jb.busy = busy;
    jb.out = out;
    jb.status = ORC_OK;
    pthread_mutex_init(&jb.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * n_threads);
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, reps_worker, &jb);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&jb.mu);
    return jb.status;
}

/* ======================================================================== */
/* GBP-CR: reservation_profile + greedy_block_placement (placement.py:35-132) */
/* ======================================================================== */
typedef struct {
    double amort;
    int32_t rank;
    int32_t idx;
} gbp_key;

static int gbp_cmp(const void* a, const void* b) {
    const gbp_key* x = (const gbp_key*)a;
    const gbp_key* y = (const gbp_key*)b;
    if (x->amort < y->amort) return -1;
    if (x->amort > y->amort) return 1;
    return (x->rank > y->rank) - (x->rank < y->rank);
}

int orc_gbp(int J, const int64_t* mem, const double* tau_c, const double* tau_p,
            const int32_t* id_rank, int64_t L, int64_t s_m, int64_t s_c, int64_t capacity,
            double arrival_rate, double load_target, int32_t* first, int32_t* count,
            int32_t* max_blocks, double* bound_time, int32_t* chain_members,
            int32_t* chain_offsets, int32_t* n_chains, double* scaled_rate,
            int32_t* rate_satisfied) {
    if (arrival_rate < 0) return ORC_INVALID;
    if (!(0 < load_target && load_target < 1)) return ORC_INVALID;
    if (capacity < 1) return ORC_INVALID;
    int64_t per_block = s_m + s_c * capacity;
    gbp_key* keys = (gbp_key*)malloc(sizeof(gbp_key) * (J > 0 ? J : 1));
    int nk = 0;
    for (int j = 0; j < J; j++) {
        int64_t m = mem[j] / per_block;
        if (m > L) m = L;
        max_blocks[j] = (int32_t)m;
        bound_time[j] = tau_c[j] + tau_p[j] * (double)m;
        first[j] = 0;
        count[j] = 0;
        if (m > 0) {
            keys[nk].amort = bound_time[j] / (double)m;
            keys[nk].rank = id_rank[j];
            keys[nk].idx = j;
            nk++;
        }
    }
    *n_chains = 0;
    chain_offsets[0] = 0;
    *scaled_rate = 0.0;
    *rate_satisfied = 0;
    if (nk == 0) {
        free(keys);
        return ORC_INFEASIBLE;
    }
    qsort(keys, nk, sizeof(gbp_key), gbp_cmp);
    double target = arrival_rate / (load_target * (double)capacity);
    int64_t frontier = 1;
    double chain_time = 0.0, rate = 0.0;
    int cur_begin = 0, n_members = 0;
    for (int q = 0; q < nk; q++) {
        int j = keys[q].idx;
        int64_t m = max_blocks[j];
        int64_t a = frontier < L - m + 1 ? frontier : L - m + 1;
        first[j] = (int32_t)a;
        count[j] = (int32_t)m;
        chain_members[n_members++] = j;
        chain_time += bound_time[j];
        int64_t fr = frontier + m - 1;
        frontier = (fr < L ? fr : L) + 1;
        if (frontier > L) {
            rate += 1.0 / chain_time;
            (*n_chains)++;
            chain_offsets[*n_chains] = n_members;
            cur_begin = n_members;
            if (rate >= target) break;
            frontier = 1;
            chain_time = 0.0;
        }
    }
    for (int q = cur_begin; q < n_members; q++) {
        first[chain_members[q]] = 0;
        count[chain_members[q]] = 0;
    }
    *scaled_rate = rate;
    *rate_satisfied = rate >= target;
    free(keys);
    return ORC_OK;
}

/* ======================================================================== */
/* GCA: greedy_cache_allocation with lexicographic Dijkstra (cache_alloc.py)  */
/* ======================================================================== */
typedef struct {
    double cost;
    int32_t node;
    int32_t len;
    int64_t parent; /* entry index, -1 for the head entry */
} dj_entry;

typedef struct {
    const dj_entry* ent;
    const int32_t* order;
    int32_t* pa;
    int32_t* pb;
} dj_ctx;

static void dj_path(const dj_ctx* c, int64_t e, int32_t* out) {
    int32_t len = c->ent[e].len;
    for (int32_t i = len - 1; i >= 0; i--) {
        out[i] = c->ent[e].node;
        e = c->ent[e].parent;
    }
}

/* Python tuple order on (cost, idx-tuple): cache_alloc.py:45-61 */
static int dj_less(const dj_ctx* c, int64_t a, int64_t b) {
    const dj_entry* x = &c->ent[a];
    const dj_entry* y = &c->ent[b];
    if (x->cost != y->cost) return x->cost < y->cost;
    dj_path(c, a, c->pa);
    dj_path(c, b, c->pb);
    int n = x->len < y->len ? x->len : y->len;
    for (int i = 0; i < n; i++) {
        int oa = c->order[c->pa[i]], ob = c->order[c->pb[i]];
        if (oa != ob) return oa < ob;
    }
    return x->len < y->len;
}

static void dj_push(const dj_ctx* c, int64_t* h, int64_t* n, int64_t e) {
    int64_t i = (*n)++;
    h[i] = e;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!dj_less(c, h[i], h[p])) break;
        int64_t t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}

static int64_t dj_pop(const dj_ctx* c, int64_t* h, int64_t* n) {
    int64_t top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && dj_less(c, h[l], h[m])) m = l;
        if (r < *n && dj_less(c, h[r], h[m])) m = r;
        if (m == i) break;
        int64_t t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}

int orc_gca(int J, const int64_t* mem, const double* tau_c, const double* tau_p,
            const int32_t* id_rank, int64_t L, int64_t s_m, int64_t s_c, const int32_t* first,
            const int32_t* count, const int64_t* residual, int32_t max_chains,
            int32_t max_members, int32_t* chain_members, int32_t* chain_offsets, int32_t* caps,
            double* times, int32_t* n_chains, int64_t* n_edges) {
    /* nodes: 0 = head, 1..U = used servers in server order, U+1 = tail */
    int U = 0;
    for (int j = 0; j < J; j++) U += count[j] > 0;
    int V = U + 2, TAIL = U + 1;
    int32_t* srv = (int32_t*)malloc(sizeof(int32_t) * V);      /* node -> server idx */
    int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * V);       /* frontier */
    int64_t* ra = (int64_t*)malloc(sizeof(int64_t) * V);       /* range a */
    int64_t* rb = (int64_t*)malloc(sizeof(int64_t) * V);       /* range b */
    int64_t* resid = (int64_t*)malloc(sizeof(int64_t) * V);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * V);
    int v = 1;
    srv[0] = -1;
    fr[0] = 1;
    ra[0] = 0;
    rb[0] = 0;
    for (int j = 0; j < J; j++) {
        if (count[j] <= 0) continue;
        srv[v] = j;
        ra[v] = first[j];
        rb[v] = first[j] + count[j] - 1;
        fr[v] = first[j] + count[j];
        int64_t budget_bytes = mem[j] - s_m * (int64_t)count[j];
        if (budget_bytes < 0) goto invalid;
        int64_t budget = budget_bytes / s_c;
        if (residual) {
            if (residual[j] < 0 || residual[j] > budget) goto invalid;
            resid[v] = residual[j];
        } else {
            resid[v] = budget;
        }
        v++;
    }
    srv[TAIL] = -1;
    fr[TAIL] = L + 2;
    ra[TAIL] = L + 1;
    rb[TAIL] = L + 1;
    /* _node_order: head 0, used servers sorted by id string, tail last */
    order[0] = 0;
    order[TAIL] = U + 1;
    for (int a = 1; a <= U; a++) {
        int o = 1;
        for (int b = 1; b <= U; b++)
            if (id_rank[srv[b]] < id_rank[srv[a]]) o++;
        order[a] = o;
    }
    /* feasible_edges over the extended node set (model.py:163-187) */
    int64_t E = 0;
    for (int s = 0; s < V; s++)
        for (int d = 0; d < V; d++)
            if (s != d && d != 0 && s != TAIL && ra[d] <= fr[s] && fr[s] <= rb[d]) E++;
    *n_edges = E;
    int32_t* esrc = (int32_t*)malloc(sizeof(int32_t) * (E + 1));
    int32_t* edst = (int32_t*)malloc(sizeof(int32_t) * (E + 1));
    int64_t* em = (int64_t*)malloc(sizeof(int64_t) * (E + 1));
    double* ecost = (double*)malloc(sizeof(double) * (E + 1));
    unsigned char* live = (unsigned char*)malloc(E + 1);
    int64_t e = 0;
    for (int s = 0; s < V; s++)
        for (int d = 0; d < V; d++)
            if (s != d && d != 0 && s != TAIL && ra[d] <= fr[s] && fr[s] <= rb[d]) {
                esrc[e] = s;
                edst[e] = d;
                em[e] = rb[d] + 1 - fr[s];
                ecost[e] = d == TAIL ? 0.0 : tau_c[srv[d]] + tau_p[srv[d]] * (double)em[e];
                e++;
            }
    for (e = 0; e < E; e++) live[e] = edst[e] == TAIL || resid[edst[e]] >= em[e];

    /* adjacency (CSR by source) over the static edge list */
    int64_t* adj_off = (int64_t*)calloc(V + 1, sizeof(int64_t));
    for (e = 0; e < E; e++) adj_off[esrc[e] + 1]++;
    for (int s = 0; s < V; s++) adj_off[s + 1] += adj_off[s];
    int64_t* adj = (int64_t*)malloc(sizeof(int64_t) * (E + 1));
    {
        int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * V);
        for (int s = 0; s < V; s++) fill[s] = adj_off[s];
        for (e = 0; e < E; e++) adj[fill[esrc[e]]++] = e;
        free(fill);
    }
    int64_t ent_cap = E + 2;
    dj_entry* ent = (dj_entry*)malloc(sizeof(dj_entry) * ent_cap);
    int64_t* heap = (int64_t*)malloc(sizeof(int64_t) * ent_cap);
    int32_t* pa = (int32_t*)malloc(sizeof(int32_t) * V);
    int32_t* pb = (int32_t*)malloc(sizeof(int32_t) * V);
    dj_ctx ctx = {ent, order, pa, pb};
    unsigned char* settled = (unsigned char*)malloc(V);
    int32_t* path = (int32_t*)malloc(sizeof(int32_t) * V);
    int K = 0, members = 0;
    chain_offsets[0] = 0;
    int status = ORC_OK;
    int64_t it;
    for (it = 0; it < E + 1; it++) {
        /* _shortest_path (cache_alloc.py:40-62) */
        memset(settled, 0, V);
        int64_t hn = 0, n_ent = 0;
        ent[0].cost = 0.0;
        ent[0].node = 0;
        ent[0].len = 1;
        ent[0].parent = -1;
        n_ent = 1;
        dj_push(&ctx, heap, &hn, 0);
        int found = 0, plen = 0;
        while (hn > 0) {
            int64_t top = dj_pop(&ctx, heap, &hn);
            int node = ent[top].node;
            if (settled[node]) continue;
            settled[node] = 1;
            if (node == TAIL) {
                found = 1;
                plen = ent[top].len;
                dj_path(&ctx, top, path);
                break;
            }
            for (int64_t q = adj_off[node]; q < adj_off[node + 1]; q++) {
                int64_t ed = adj[q];
                if (!live[ed] || settled[edst[ed]]) continue;
                if (n_ent >= ent_cap) { status = ORC_INTERNAL; goto done; }
                ent[n_ent].cost = ent[top].cost + ecost[ed];
                ent[n_ent].node = edst[ed];
                ent[n_ent].len = ent[top].len + 1;
                ent[n_ent].parent = top;
                dj_push(&ctx, heap, &hn, n_ent);
                n_ent++;
            }
        }
        if (!found) break;
        /* cap = min(resid // m) over real hops; resid update; re-filter */
        int64_t cap = -1;
        for (int p = 1; p < plen; p++) {
            int d = path[p];
            if (d == TAIL) continue;
            int64_t m = rb[d] + 1 - fr[path[p - 1]];
            int64_t c = resid[d] / m;
            if (cap < 0 || c < cap) cap = c;
        }
        if (cap < 1) { status = ORC_INTERNAL; goto done; }
        for (int p = 1; p < plen; p++) {
            int d = path[p];
            if (d == TAIL) continue;
            resid[d] -= (rb[d] + 1 - fr[path[p - 1]]) * cap;
        }
        for (e = 0; e < E; e++)
            if (live[e] && edst[e] != TAIL && resid[edst[e]] < em[e]) live[e] = 0;
        /* build_chain -> chain_service_time (model.py:229-231) is Python's
         * builtin sum() starting from int 0; CPython >= 3.12 sums floats with
         * Neumaier compensation (bltinmodule.c builtin_sum_impl). */
        double T = 0.0, comp = 0.0;
        for (int p = 1; p < plen; p++) {
            int d = path[p];
            double c = d == TAIL ? 0.0
                                 : tau_c[srv[d]] + tau_p[srv[d]] * (double)(rb[d] + 1 - fr[path[p - 1]]);
            if (p == 1) {
                T = c;
            } else {
                double t = T + c;
                if (fabs(T) >= fabs(c)) comp += (T - t) + c;
                else comp += (c - t) + T;
                T = t;
            }
        }
        if (comp != 0.0 && isfinite(comp)) T += comp;
        if (K >= max_chains || members + plen - 2 > max_members) { status = ORC_INTERNAL; goto done; }
        for (int p = 1; p < plen - 1; p++) chain_members[members++] = srv[path[p]];
        caps[K] = (int32_t)cap;
        times[K] = T;
        K++;
        chain_offsets[K] = members;
    }
    if (it == E + 1) status = ORC_INTERNAL; /* failed to terminate */
done:
    *n_chains = K;
    free(heap); free(ent); free(pa); free(pb); free(settled); free(path); free(adj); free(adj_off);
    free(esrc); free(edst); free(em); free(ecost); free(live);
    free(srv); free(fr); free(ra); free(rb); free(resid); free(order);
    return status;
invalid:
    free(srv); free(fr); free(ra); free(rb); free(resid); free(order);
    *n_chains = 0;
    *n_edges = 0;
    return ORC_INVALID;
}
