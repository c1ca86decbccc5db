// capi.cu -- extern "C" entry points of libchainserve_b200 (include/chainserve_b200.h).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "cs_internal.cuh"

// implemented in the kernel translation units
extern "C" int cs_exp_streams_impl(const uint64_t*, int64_t, int64_t, double*, int64_t, int, void*);
extern "C" int cs_jffc_sim_impl(const cs_sim_point*, int32_t, const double*, const int32_t*, int32_t,
                                int32_t, const double*, int64_t, int32_t, int32_t, int32_t, int64_t,
                                int64_t, double*, int64_t, double*, int32_t, cs_rep_summary*, double*,
                                void*, int64_t, int32_t, void*);
extern "C" int cs_exp_streams_prefix_impl(const uint64_t*, int64_t, int64_t, double*, int64_t, int,
                                          const cs::PrefixPlan*, int, int, void*);
extern "C" int cs_exp_streams_il4_p1_impl(const uint64_t*, int64_t, int64_t, double*, int64_t, int,
                                          const cs::PrefixPlan*, void*);
extern "C" bool cs_seg_prefix_plan(int32_t, int32_t, int32_t, int64_t, int64_t, const cs_sim_point*, void*,
                                   cs::PrefixPlan*);
namespace cs {
bool use_seg(int32_t max_chains, int32_t max_cap, int64_t n);
}
extern "C" int64_t cs_jffc_sim_workspace_bytes_impl(int32_t, int32_t, int32_t, int32_t, int64_t);
extern "C" int cs_philox_peak_impl(int64_t, int32_t, uint64_t*, void*);
extern "C" int cs_rep_stats_impl(const double*, int32_t, int64_t, int64_t, int64_t, cs_rep_summary*,
                                 const int64_t*, int32_t, double*, double*, int32_t, void*);
extern "C" int cs_gbp_batch_impl(const cs_compose_point*, int32_t, int32_t, const int64_t*,
                                 const double*, const double*, const int32_t*, int32_t*, int32_t*,
                                 int32_t*, double*, int32_t*, int32_t*, int32_t*, double*, int32_t*,
                                 int32_t*, void*);
extern "C" int cs_gca_batch_impl(const cs_compose_point*, int32_t, int32_t, int32_t, const int64_t*,
                                 const double*, const double*, const int32_t*, const int32_t*,
                                 const int32_t*, const int64_t*, int32_t, int32_t, int32_t*, int32_t*,
                                 int32_t*, double*, int32_t*, int64_t*, int32_t*, void*);

namespace cs {
static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// The engine's own stream-ordered pool per device (not the device's default
// pool, which other libraries share).  Freed scratch stays reserved: with a
// release threshold the driver trims the pool at every synchronisation and
// the next allocation re-maps it (measured 18-40 ms per multi-GB buffer, more
// than a whole config-2 sweep); cs_release_memory() trims on request.
static cudaMemPool_t g_pools[64] = {};

void ensure_mem_pool() { (void)engine_pool(); }

cudaMemPool_t engine_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&g_pools[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            g_pools[dev] = nullptr;
            return nullptr;
        }
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return g_pools[dev];
}

int pool_alloc(void** p, size_t n, cudaStream_t st) {
    cudaMemPool_t pool = engine_pool();
    const cudaError_t e = pool ? cudaMallocFromPoolAsync(p, n ? n : 16, pool, st) : cudaMallocAsync(p, n ? n : 16, st);
    return check_cuda(e, "cudaMallocFromPoolAsync");
}

// ---- numpy SeedSequence (bit_generator.pyx), restated for the product ----
static uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}
static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    r ^= r >> 16;
    return r;
}
static void seedseq_key(const uint32_t* ent_in, int n_ent, const uint32_t* spawn, int n_spawn,
                        uint64_t key[2]) {
    std::vector<uint32_t> ent(ent_in, ent_in + n_ent);
    if (n_spawn > 0)
        while (ent.size() < 4) ent.push_back(0u);  // pad run entropy to the pool size
    ent.insert(ent.end(), spawn, spawn + n_spawn);
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
    for (int i = 0; i < 4; i++) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (size_t s = 4; s < ent.size(); s++)
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(ent[s], hc));
    uint32_t w[4];
    uint32_t hb = 0x8b51f9ddu;
    for (int i = 0; i < 4; i++) {
        uint32_t v = pool[i];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    key[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    key[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}
}  // namespace cs

using namespace cs;

extern "C" {

const char* cs_version(void) { return "chainserve_b200 0.1.0 (sm_100a)"; }
int64_t cs_launch_count(void) { return g_launches.load(); }
const char* cs_last_error(void) { return g_err; }

int cs_host_log1p_variant(void) {
#if defined(__x86_64__)
    __builtin_cpu_init();
    return (__builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2")) ? 1 : 0;
#else
    return 0;
#endif
}

int cs_release_memory(void) {
    cudaMemPool_t pool = engine_pool();
    if (!pool) return CS_OK;
    int rc = check_cuda(cudaDeviceSynchronize(), "cs_release_memory sync");
    if (rc) return rc;
    return check_cuda(cudaMemPoolTrimTo(pool, 0), "cudaMemPoolTrimTo");
}

int cs_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int cs_philox_keys(const uint32_t* entropy, int32_t n_entropy, const uint64_t* reps, int64_t n_reps,
                   uint64_t* keys) {
    if (n_entropy < 1 || n_entropy > 60) {
        set_error("cs_philox_keys: entropy must have 1..60 uint32 words");
        return CS_INVALID;
    }
    for (int64_t i = 0; i < n_reps; i++) {
        uint32_t sp[2];
        int ns = 0;
        uint64_t r = reps[i];
        if (r == 0) sp[ns++] = 0;
        while (r > 0) {
            sp[ns++] = (uint32_t)(r & 0xffffffffu);
            r >>= 32;
        }
        seedseq_key(entropy, n_entropy, sp, ns, keys + 2 * i);
    }
    return CS_OK;
}

int cs_exp_streams(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out,
                   int64_t ld, int32_t log1p_variant, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_exp_streams: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (ld < n_draws) {
        set_error("cs_exp_streams: ld < n_draws");
        return CS_INVALID;
    }
    const int v = log1p_variant < 0 ? cs_host_log1p_variant() : log1p_variant;
    return cs_exp_streams_impl(d_keys, n_streams, n_draws, d_out, ld, v, stream);
}

int cs_philox_peak(int64_t blocks_per_thread, int32_t grid, uint64_t* d_out, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_philox_peak: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (blocks_per_thread < 1 || grid < 1) {
        set_error("cs_philox_peak: invalid sizes");
        return CS_INVALID;
    }
    return cs_philox_peak_impl(blocks_per_thread, grid, d_out, stream);
}

int64_t cs_jffc_sim_workspace_bytes(int32_t n_points, int32_t n_reps, int32_t max_chains,
                                    int32_t max_capacity, int64_t n_jobs) {
    return cs_jffc_sim_workspace_bytes_impl(n_points, n_reps, max_chains, max_capacity, n_jobs);
}

int cs_jffc_sim_ex(const cs_sim_point* d_points, int32_t n_points, const double* d_rates,
                   const int32_t* d_caps, int32_t max_chains, int32_t max_capacity,
                   const double* d_streams, int64_t lds, int32_t rep_begin, int32_t n_reps,
                   int32_t n_reps_total, int64_t n_jobs, int64_t warm, double* d_responses, int64_t ldr,
                   double* d_busy, int32_t ldb, cs_rep_summary* d_summary, double* d_jobs,
                   void* d_workspace, int64_t workspace_bytes, int32_t flags, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_jffc_sim: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (n_jobs < 1 || warm < 0 || warm >= n_jobs || max_chains < 1 || max_capacity < 1 ||
        ldb < max_chains || lds < 2 * n_jobs || rep_begin < 0 || rep_begin + n_reps > n_reps_total ||
        (ldr & 1)) {
        set_error("cs_jffc_sim: invalid sizes");
        return CS_INVALID;
    }
    if ((flags & CS_SIM_STREAMS_IL4) && (d_jobs != nullptr || (flags & CS_SIM_FORCE_EVENT_LOOP) ||
                                         !cs::use_seg(max_chains, max_capacity, n_jobs))) {
        set_error("cs_jffc_sim: interleaved streams are read by the segmented path only");
        return CS_INVALID;
    }
    return cs_jffc_sim_impl(d_points, n_points, d_rates, d_caps, max_chains, max_capacity, d_streams,
                            lds, rep_begin, n_reps, n_reps_total, n_jobs, warm, d_responses, ldr,
                            d_busy, ldb, d_summary, d_jobs, d_workspace, workspace_bytes, flags, stream);
}

int cs_jffc_sim(const cs_sim_point* d_points, int32_t n_points, const double* d_rates,
                const int32_t* d_caps, int32_t max_chains, int32_t max_capacity,
                const double* d_streams, int64_t lds, int32_t rep_begin, int32_t n_reps,
                int32_t n_reps_total, int64_t n_jobs, int64_t warm, double* d_responses, int64_t ldr,
                double* d_busy, int32_t ldb, cs_rep_summary* d_summary, double* d_jobs,
                void* d_workspace, int64_t workspace_bytes, void* stream) {
    return cs_jffc_sim_ex(d_points, n_points, d_rates, d_caps, max_chains, max_capacity, d_streams, lds,
                          rep_begin, n_reps, n_reps_total, n_jobs, warm, d_responses, ldr, d_busy, ldb,
                          d_summary, d_jobs, d_workspace, workspace_bytes, 0, stream);
}

int cs_sim_streams(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out, int64_t ld,
                   int32_t log1p_variant, const cs_sim_point* d_points, int32_t n_points,
                   int32_t max_chains, int32_t max_capacity, int64_t n_jobs, int64_t warm,
                   void* d_workspace, int64_t workspace_bytes, int32_t* sim_flags, void* stream) {
    return cs_sim_streams_ex(d_keys, n_streams, n_draws, d_out, ld, log1p_variant, d_points, n_points, max_chains,
                             max_capacity, n_jobs, warm, d_workspace, workspace_bytes, 0, sim_flags, stream);
}

int cs_sim_streams_ex(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out, int64_t ld,
                      int32_t log1p_variant, const cs_sim_point* d_points, int32_t n_points,
                      int32_t max_chains, int32_t max_capacity, int64_t n_jobs, int64_t warm,
                      void* d_workspace, int64_t workspace_bytes, int32_t opts, int32_t* sim_flags,
                      void* stream) {
    if (sim_flags) *sim_flags = 0;
    if (cs_device_count() == 0) {
        set_error("cs_sim_streams: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (ld < n_draws || n_jobs < 1 || warm < 0 || warm >= n_jobs || n_draws < 2 * n_jobs) {
        set_error("cs_sim_streams: invalid sizes");
        return CS_INVALID;
    }
    const int v = log1p_variant < 0 ? cs_host_log1p_variant() : log1p_variant;
    cs::PrefixPlan pp;
    const int64_t need = cs_jffc_sim_workspace_bytes_impl(n_points, (int32_t)n_streams, max_chains,
                                                          max_capacity, n_jobs);
    if (sim_flags && d_workspace && workspace_bytes >= need && cs::use_seg(max_chains, max_capacity, n_jobs) &&
        cs_seg_prefix_plan(n_points, (int32_t)n_streams, max_capacity, n_jobs, warm, d_points, d_workspace, &pp)) {
        // few points per stream: every simulator lane reads its own row
        const bool il4 = n_points < 16 && n_streams % 32 == 0 && ld % 4 == 0;
        // one point per stream: the prefix chain in its own pass (one thread
        // per stream) instead of one lane of each generating warp
        const int rc = (il4 && n_points == 1)
                           ? cs_exp_streams_il4_p1_impl(d_keys, n_streams, n_draws, d_out, ld, v, &pp, stream)
                           : cs_exp_streams_prefix_impl(d_keys, n_streams, n_draws, d_out, ld, v, &pp, il4,
                                                        (opts & CS_STREAMS_WHOLE_SM) ? 1 : 0, stream);
        if (rc == CS_OK) *sim_flags = CS_SIM_PREFIX_READY | (il4 ? CS_SIM_STREAMS_IL4 : 0);
        return rc;
    }
    return cs_exp_streams_impl(d_keys, n_streams, n_draws, d_out, ld, v, stream);
}

int cs_rep_stats(const double* d_resp, int32_t n_groups, int64_t rows_per_group, int64_t m,
                 int64_t ldr, cs_rep_summary* d_summary, const int64_t* ranks, int32_t n_ranks,
                 double* out_values, double* d_row_sums, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_rep_stats: no CUDA device");
        return CS_ERR_CUDA;
    }
    ensure_mem_pool();
    return cs_rep_stats_impl(d_resp, n_groups, rows_per_group, m, ldr, d_summary, ranks, n_ranks,
                             out_values, d_row_sums, 0, stream);
}

int cs_rep_stats_dist(const double* d_resp, int32_t n_groups, int64_t rows_per_group, int64_t m,
                      int64_t ldr, cs_rep_summary* d_summary, const int64_t* ranks, int32_t n_ranks,
                      double* out_values, double* d_row_sums, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_rep_stats_dist: no CUDA device");
        return CS_ERR_CUDA;
    }
    ensure_mem_pool();
    return cs_rep_stats_impl(d_resp, n_groups, rows_per_group, m, ldr, d_summary, ranks, n_ranks,
                             out_values, d_row_sums, 1, stream);
}

int cs_gbp_batch(const cs_compose_point* d_points, int32_t n_points, int32_t max_servers,
                 const int64_t* d_mem, const double* d_tau_c, const double* d_tau_p,
                 const int32_t* d_id_rank, int32_t* d_first, int32_t* d_count, int32_t* d_max_blocks,
                 double* d_bound_time, int32_t* d_order, int32_t* d_chain_end, int32_t* d_n_chains,
                 double* d_scaled_rate, int32_t* d_rate_satisfied, int32_t* d_status, void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_gbp_batch: no CUDA device");
        return CS_ERR_CUDA;
    }
    return cs_gbp_batch_impl(d_points, n_points, max_servers, d_mem, d_tau_c, d_tau_p, d_id_rank,
                             d_first, d_count, d_max_blocks, d_bound_time, d_order, d_chain_end,
                             d_n_chains, d_scaled_rate, d_rate_satisfied, d_status, stream);
}

int cs_gca_batch(const cs_compose_point* d_points, int32_t n_points, int32_t max_servers,
                 int32_t max_block_count, const int64_t* d_mem, const double* d_tau_c,
                 const double* d_tau_p, const int32_t* d_id_rank, const int32_t* d_first,
                 const int32_t* d_count, const int64_t* d_residual, int32_t max_chains,
                 int32_t max_hops, int32_t* d_chain_srv, int32_t* d_chain_len, int32_t* d_caps,
                 double* d_times, int32_t* d_n_chains, int64_t* d_n_edges, int32_t* d_status,
                 void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_gca_batch: no CUDA device");
        return CS_ERR_CUDA;
    }
    return cs_gca_batch_impl(d_points, n_points, max_servers, max_block_count, d_mem, d_tau_c,
                             d_tau_p, d_id_rank, d_first, d_count, d_residual, max_chains, max_hops,
                             d_chain_srv, d_chain_len, d_caps, d_times, d_n_chains, d_n_edges,
                             d_status, stream);
}

// ---------------------------------------------------------------------------
// End-to-end sweep from HOST buffers (the reference-facing call for C/FFI
// users; the Python run_sim/run_sim_batch use it too).  Everything between
// the H2D copy of the configuration and the D2H copy of the results runs on
// the device.  Replications [rep_begin, rep_begin + n_reps) of seed
// `entropy` are simulated for every point (a shard when rep_begin > 0).
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    int alloc(size_t n, cudaStream_t s) {
        st = s;
        if (n == 0) n = 16;
        return pool_alloc(&p, n, s);
    }
};

int cs_run_sim_host(const cs_sim_point* points, int32_t n_points, const double* rates,
                    const int32_t* caps, int32_t n_chain_entries, const uint32_t* entropy,
                    int32_t n_entropy, int32_t rep_begin, int32_t n_reps, int64_t n_jobs,
                    int64_t warm, const int64_t* ranks, int32_t n_ranks, int32_t log1p_variant,
                    int64_t max_stream_bytes, cs_rep_summary* out_summary, double* out_busy,
                    int32_t ldb, double* out_rank_values, double* out_responses, double* out_jobs,
                    void* stream) {
    if (cs_device_count() == 0) {
        set_error("cs_run_sim_host: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (n_jobs < 1 || warm < 0 || warm >= n_jobs || n_reps < 0 || n_points < 0 || rep_begin < 0) {
        set_error("cs_run_sim_host: invalid sizes (need n_jobs >= 1, 0 <= warm < n_jobs)");
        return CS_INVALID;
    }
    if (n_reps == 0 || n_points == 0) return CS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    ensure_mem_pool();
    int rc = CS_OK;
    int32_t max_chains = 1, max_cap = 1;
    for (int p = 0; p < n_points; p++) {
        max_chains = std::max(max_chains, points[p].n_chains);
        int c = 0;
        for (int k = 0; k < points[p].n_chains; k++) c += caps[points[p].chain_base + k];
        max_cap = std::max(max_cap, c);
    }
    if (ldb < max_chains) {
        set_error("cs_run_sim_host: ldb < max chains");
        return CS_INVALID;
    }
    const int64_t m = n_jobs - warm;
    const int64_t ldr = (m + 15) & ~15ll;  // rows start on 128-byte lines
    const int64_t lds = 2 * n_jobs;
    const int64_t rows = (int64_t)n_points * n_reps;
    // replications per stream chunk (bounded stream scratch)
    int64_t chunk = n_reps;
    if (max_stream_bytes > 0) {
        const int64_t cmax = std::max<int64_t>(1, std::min<int64_t>(n_reps, max_stream_bytes / (lds * 8)));
        // equal chunks, multiples of 32 where possible (the simulator's
        // interleaved stream layout needs whole 32-row groups)
        const int64_t nch = (n_reps + cmax - 1) / cmax;
        chunk = (n_reps + nch - 1) / nch;
        if (nch > 1 && cmax >= 32) chunk = std::min(cmax / 32 * 32, (chunk + 31) / 32 * 32);
    }
    DevBuf b_pts, b_rates, b_caps, b_keys, b_S, b_resp, b_busy, b_summ, b_jobs, b_ws;
    if ((rc = b_pts.alloc(sizeof(cs_sim_point) * n_points, st)) ||
        (rc = b_rates.alloc(sizeof(double) * n_chain_entries, st)) ||
        (rc = b_caps.alloc(sizeof(int32_t) * n_chain_entries, st)) ||
        (rc = b_keys.alloc(sizeof(uint64_t) * 2 * chunk, st)) ||
        (rc = b_S.alloc(sizeof(double) * (lds * chunk + CS_STREAM_PAD), st)) ||
        (rc = b_resp.alloc(sizeof(double) * ldr * rows, st)) ||
        (rc = b_busy.alloc(sizeof(double) * ldb * rows, st)) ||
        (rc = b_summ.alloc(sizeof(cs_rep_summary) * rows, st)))
        return rc;
    if (out_jobs && (rc = b_jobs.alloc(sizeof(double) * 4 * n_jobs * rows, st))) return rc;
    const int64_t wsb = cs_jffc_sim_workspace_bytes_impl(n_points, (int32_t)chunk, max_chains, max_cap, n_jobs);
    if (wsb > 0 && (rc = b_ws.alloc(wsb, st))) return rc;
    cudaMemcpyAsync(b_pts.p, points, sizeof(cs_sim_point) * n_points, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_rates.p, rates, sizeof(double) * n_chain_entries, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(b_caps.p, caps, sizeof(int32_t) * n_chain_entries, cudaMemcpyHostToDevice, st);
    std::vector<uint64_t> reps(chunk), keys(2 * chunk);
    for (int64_t c0 = 0; c0 < n_reps; c0 += chunk) {
        const int64_t cn = std::min<int64_t>(chunk, n_reps - c0);
        for (int64_t i = 0; i < cn; i++) reps[i] = (uint64_t)(rep_begin + c0 + i);
        if ((rc = cs_philox_keys(entropy, n_entropy, reps.data(), cn, keys.data()))) return rc;
        // the host vector is reused next chunk: order the copy before it
        cudaMemcpyAsync(b_keys.p, keys.data(), sizeof(uint64_t) * 2 * cn, cudaMemcpyHostToDevice, st);
        int32_t sim_flags = 0;
        if ((rc = cs_sim_streams((const uint64_t*)b_keys.p, cn, lds, (double*)b_S.p, lds, log1p_variant,
                                 (const cs_sim_point*)b_pts.p, n_points, max_chains, max_cap, n_jobs, warm,
                                 out_jobs ? nullptr : b_ws.p, wsb, &sim_flags, st)))
            return rc;
        if ((rc = cs_jffc_sim_impl((const cs_sim_point*)b_pts.p, n_points, (const double*)b_rates.p,
                                   (const int32_t*)b_caps.p, max_chains, max_cap, (const double*)b_S.p,
                                   lds, (int32_t)c0, (int32_t)cn, n_reps, n_jobs, warm,
                                   (double*)b_resp.p, ldr, (double*)b_busy.p, ldb,
                                   (cs_rep_summary*)b_summ.p, (double*)b_jobs.p, b_ws.p, wsb,
                                   sim_flags, st)))
            return rc;
        // the serial single-chain kernel (exact mode / job records) flags rows
        // whose merge feed backed up on exact finish-time ties (counted = -1):
        // such a chunk is simulated again with the per-event kernel
        if (max_chains <= 1 && max_cap <= 16 && (out_jobs || !use_seg(max_chains, max_cap, n_jobs))) {
            std::vector<cs_rep_summary> hs((size_t)n_points * n_reps);
            cudaMemcpyAsync(hs.data(), b_summ.p, sizeof(cs_rep_summary) * hs.size(), cudaMemcpyDeviceToHost, st);
            if ((rc = check_cuda(cudaStreamSynchronize(st), "chunk summaries"))) return rc;
            bool redo = false;
            for (int32_t p = 0; p < n_points && !redo; p++)
                for (int64_t i = 0; i < cn; i++)
                    if (hs[(size_t)p * n_reps + c0 + i].counted < 0) redo = true;
            if (redo &&
                (rc = cs_jffc_sim_impl((const cs_sim_point*)b_pts.p, n_points, (const double*)b_rates.p,
                                       (const int32_t*)b_caps.p, max_chains, max_cap, (const double*)b_S.p,
                                       lds, (int32_t)c0, (int32_t)cn, n_reps, n_jobs, warm, (double*)b_resp.p,
                                       ldr, (double*)b_busy.p, ldb, (cs_rep_summary*)b_summ.p,
                                       (double*)b_jobs.p, b_ws.p, wsb, CS_SIM_FORCE_EVENT_LOOP, st)))
                return rc;
        }
        if (c0 + chunk < n_reps && (rc = check_cuda(cudaStreamSynchronize(st), "chunk sync"))) return rc;
    }
    rc = cs_rep_stats_impl((const double*)b_resp.p, n_points, n_reps, m, ldr, (cs_rep_summary*)b_summ.p,
                           ranks, n_ranks, out_rank_values, nullptr, 0, st);
    if (rc) return rc;
    cudaMemcpyAsync(out_summary, b_summ.p, sizeof(cs_rep_summary) * rows, cudaMemcpyDeviceToHost, st);
    if (out_busy) cudaMemcpyAsync(out_busy, b_busy.p, sizeof(double) * ldb * rows, cudaMemcpyDeviceToHost, st);
    if (out_responses)  // rows of m values (host rows are dense, device rows padded to ldr)
        cudaMemcpy2DAsync(out_responses, sizeof(double) * m, b_resp.p, sizeof(double) * ldr,
                          sizeof(double) * m, rows, cudaMemcpyDeviceToHost, st);
    if (out_jobs)
        cudaMemcpyAsync(out_jobs, b_jobs.p, sizeof(double) * 4 * n_jobs * rows, cudaMemcpyDeviceToHost, st);
    return check_cuda(cudaStreamSynchronize(st), "cs_run_sim_host sync");
}

}  // extern "C"
