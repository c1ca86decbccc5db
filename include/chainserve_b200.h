/*
 * chainserve_b200.h -- C-ABI of the B200 engine for the chainserve hot path.
 *
 * The reference (arXiv 2604.14993, /root/reference/pkg) is pure Python and has
 * no FFI: its drop-in surface is the Python API re-exported by
 * pkg/src/chainserve/__init__.py:3-65.  Each entry point below replaces the
 * reference function named in its comment (file:line relative to
 * /root/reference/pkg/src/chainserve).  The Python package
 * paper_2604_14993_b200 binds these symbols with ctypes and keeps the
 * reference's signatures, dataclasses and exceptions; INTEGRATION.md shows the
 * binding.
 *
 * Conventions
 *   * plain pointers + sizes; "d_" pointers are CUDA device pointers, all
 *     others host pointers; `stream` is a cudaStream_t passed as void*.
 *   * every call returns a status (CS_OK ...); cs_last_error() gives a
 *     thread-local message for the last non-OK status.
 *   * no global mutable state except per-device scratch caches; calls are
 *     reentrant per stream.  Device calls are asynchronous on `stream`.
 *   * there is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns CS_ERR_CUDA.
 */
#ifndef CHAINSERVE_B200_H
#define CHAINSERVE_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference's exceptions by the shim) ---- */
#define CS_OK 0
#define CS_INFEASIBLE 1   /* InfeasibleError (placement.py:91-94)          */
#define CS_INVALID 2      /* ValueError (model.py, sim.py:47-68, ...)      */
#define CS_INTERNAL 3     /* AssertionError (cache_alloc.py:119,133)       */
#define CS_ERR_CUDA 4     /* CUDA runtime failure / no device              */
#define CS_UNSUPPORTED 5  /* NotImplementedError (mode outside the path)   */
#define CS_UNSTABLE 6     /* UnstableError (analysis.py:96-97,132-133)     */

const char* cs_version(void);
const char* cs_last_error(void);
/* 1 if this host's glibc resolves log1p to its FMA variant (CPU has FMA and
 * AVX2), else 0 -- numpy's ziggurat tail calls that libm (see glibc_log1p.cuh). */
int cs_host_log1p_variant(void);
/* number of visible CUDA devices (0 when none) */
int cs_device_count(void);
/* kernels launched by this library since load (all threads) */
int64_t cs_launch_count(void);
/* The host-level calls (cs_run_sim_host, cs_rep_stats*) take their device
 * scratch from a private stream-ordered pool that keeps freed memory reserved
 * for the next call (re-mapping tens of GB per call costs more than the
 * simulation).  This returns the current device's unused reserve to the
 * driver; it blocks until the device is idle. */
int cs_release_memory(void);

/* ------------------------------------------------------------------------ */
/* RNG                                                                        */
/* ------------------------------------------------------------------------ */
/* Philox keys of np.random.SeedSequence(entropy=<entropy words>,
 * spawn_key=(reps[i],)).generate_state(2, np.uint64)  -- replaces sim.py:141-143.
 * entropy: the seed as little-endian uint32 words (numpy's
 * _coerce_to_uint32_array).  keys: 2*n_reps uint64 (host). */
int cs_philox_keys(const uint32_t* entropy, int32_t n_entropy, const uint64_t* reps,
                   int64_t n_reps, uint64_t* keys);

/* For each of n_streams keys, n_draws values of
 * Generator(Philox(key)).exponential(1.0, n_draws) (numpy ziggurat) into
 * d_out[s*ld + i].  Replaces rng.exponential at sim.py:145,159.
 * log1p_variant: 1 = glibc FMA build, 0 = SSE2 build, -1 = this host's. */
int cs_exp_streams(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out,
                   int64_t ld, int32_t log1p_variant, void* stream);

/* ------------------------------------------------------------------------ */
/* JFFC simulation                                                            */
/* ------------------------------------------------------------------------ */
#define CS_STREAM_PAD 512 /* doubles of readable tail padding after the stream buffer */

/* One sweep point: a composed system (chains chain_base..chain_base+K-1 of the
 * rates/caps arrays, rates descending) under Poisson arrivals of rate lam. */
typedef struct {
    int32_t n_chains;
    int32_t chain_base;
    double lam;
} cs_sim_point;

/* Per-replication result: the RepResult fields of sim.py:120-133 computed
 * exactly as sim.py:298-324 does, plus the raw snapshots they derive from. */
typedef struct {
    double wait_sum;
    double service_sum;
    int64_t counted;
    double window_s;
    double mean_occupancy;
    double occ_first_half;
    double occ_second_half;
    double lambda_effective;
    int64_t end_queue_len;
    double w_start, t_mid, area_mid, t_end, area_end;
    double resp_sum;     /* numpy pairwise sum of the responses             */
    double resp_mean;    /* responses.mean() = resp_sum / counted (sim.py:407) */
} cs_rep_summary;

/* _simulate_once (sim.py:181-324; Poisson workload, policy "jffc",
 * horizon_time_s None) for every (point p, replication r) of a chunk of
 * n_reps replications starting at rep_begin (of n_reps_total).  Chunk row r
 * reads stream row r of d_streams (2*n_jobs draws, row stride lds):
 * arrivals = cumsum((1/lam) * S[0:n]), sizes = S[n:2n].
 * The stream buffer must stay readable CS_STREAM_PAD doubles past the last
 * row (the simulator's cursors and prefetches run ahead without clamping).
 * Outputs are point-major, o = p*n_reps_total + rep_begin + r:
 *   d_responses[o*ldr + q]  q < n-warm, completion order (NULL: not stored;
 *                           ldr even: the single-chain path writes whole
 *                           lines with 16-byte stores; a multiple of 16
 *                           keeps every line 128-byte aligned)
 *   d_busy[o*ldb + k]       busy_time_s (ldb >= max_chains)
 *   d_summary[o]
 *   d_jobs[(o*n + j)*4 ..]  (arrival, start, finish, chain) or NULL.
 * Single-chain compositions (K = 1, C <= 16) without d_jobs take the
 * segmented time-parallel kernel (csrc/jffc_seg.cu): responses, counted,
 * window, lambda_effective and end_queue bit-exact; wait/service sums,
 * occupancy areas and busy time summed per job in fixed job blocks
 * (reassociated, ~1e-13 relative).  Environment CS_SIM_EXACT=1 selects the
 * serial kernel that is bit-exact in every field.  That path and the
 * generic kernel (K > 512 or C > 1024) need cs_jffc_sim_workspace_bytes()
 * of d_workspace.
 * warm = int(warmup_fraction * n) computed by the caller as Python does. */
int cs_jffc_sim(const cs_sim_point* d_points, int32_t n_points, const double* d_rates,
                const int32_t* d_caps, int32_t max_chains, int32_t max_capacity,
                const double* d_streams, int64_t lds, int32_t rep_begin, int32_t n_reps,
                int32_t n_reps_total, int64_t n_jobs, int64_t warm, double* d_responses,
                int64_t ldr, double* d_busy, int32_t ldb, cs_rep_summary* d_summary,
                double* d_jobs, void* d_workspace, int64_t workspace_bytes, void* stream);

int64_t cs_jffc_sim_workspace_bytes(int32_t n_points, int32_t n_reps, int32_t max_chains,
                                    int32_t max_capacity, int64_t n_jobs);

/* cs_exp_streams for a following cs_jffc_sim_ex of the same shape: when the
 * segmented single-chain path applies (and n_points <= 32), the stream kernel
 * also runs the exact arrival-time cumsum of every (replication, point) row
 * and records the simulator's per-segment start times into d_workspace
 * (sized by cs_jffc_sim_workspace_bytes).  *sim_flags receives the flags the
 * simulation call must take: CS_SIM_PREFIX_READY (it skips its own pre-pass)
 * and, with fewer than 16 points per stream (n_streams a multiple of 32, ld of
 * 4), CS_SIM_STREAMS_IL4: d_out then holds the streams in the simulator's
 * 32-row interleaved layout (stream r's value i at (r/32)*32*ld + (i/4)*128 +
 * (r%32)*4 + i%4), readable by the segmented simulator only. */
#define CS_SIM_PREFIX_READY 1
#define CS_SIM_STREAMS_IL4 4
/* cs_jffc_sim_ex: take the per-event register kernel for single-chain
 * compositions instead of the serial recursion kernel (its fallback when
 * exact finish-time ties back up the recursion's merge feed: counted = -1) */
#define CS_SIM_FORCE_EVENT_LOOP 2
int cs_sim_streams(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out, int64_t ld,
                   int32_t log1p_variant, const cs_sim_point* d_points, int32_t n_points,
                   int32_t max_chains, int32_t max_capacity, int64_t n_jobs, int64_t warm,
                   void* d_workspace, int64_t workspace_bytes, int32_t* sim_flags, void* stream);

/* cs_sim_streams with options.  CS_STREAMS_WHOLE_SM: the fused kernel runs
 * 16 streams per block, each block filling one SM (ceil(n_streams / 16) SMs),
 * for a caller that runs other work on the remaining SMs at the same time
 * (the pipelined engine: the statistics of the previous sweep); alone on the
 * GPU the default 8-stream blocks over every SM are faster. */
#define CS_STREAMS_WHOLE_SM 1
int cs_sim_streams_ex(const uint64_t* d_keys, int64_t n_streams, int64_t n_draws, double* d_out, int64_t ld,
                      int32_t log1p_variant, const cs_sim_point* d_points, int32_t n_points,
                      int32_t max_chains, int32_t max_capacity, int64_t n_jobs, int64_t warm,
                      void* d_workspace, int64_t workspace_bytes, int32_t opts, int32_t* sim_flags,
                      void* stream);

/* cs_jffc_sim with flags (CS_SIM_PREFIX_READY: d_workspace holds the prefix
 * cs_sim_streams wrote for exactly these streams and shape; CS_SIM_STREAMS_IL4:
 * d_streams is in the interleaved layout; pass cs_sim_streams' *sim_flags). */
int cs_jffc_sim_ex(const cs_sim_point* d_points, int32_t n_points, const double* d_rates,
                   const int32_t* d_caps, int32_t max_chains, int32_t max_capacity,
                   const double* d_streams, int64_t lds, int32_t rep_begin, int32_t n_reps,
                   int32_t n_reps_total, int64_t n_jobs, int64_t warm, double* d_responses,
                   int64_t ldr, double* d_busy, int32_t ldb, cs_rep_summary* d_summary,
                   double* d_jobs, void* d_workspace, int64_t workspace_bytes, int32_t flags,
                   void* stream);

/* Measurement helper (no reference counterpart): generate
 * grid*256*blocks_per_thread Philox4x64-10 blocks, XOR-folded into
 * d_out[grid*256]; timed by bench.py as the RNG peak the simulator's
 * RNG-floor fraction is quoted against. */
int cs_philox_peak(int64_t blocks_per_thread, int32_t grid, uint64_t* d_out, void* stream);

/* Engine-side introspection (no reference counterpart): the launch plan of
 * the segmented single-chain path for this shape on the current device --
 * out[0] segments per replication, out[1] warps per segment, out[2]
 * checkpoints per segment, out[3] the slot-count instance (4/7/8/16). */
int cs_seg_plan(int32_t n_points, int32_t n_reps, int32_t max_capacity, int64_t n_jobs, int32_t* out);

/* ---- the rest of run_sim's signature ---------- */
/* _simulate_once for the dedicated-queue baseline policies (sim.py:104-117,
 * 279-286), the sampled and trace workloads (sim.py:161-178,199-203,
 * workload.py:124-167) and the time-horizon Poisson mode (sim.py:146-158,
 * 187-190).  One warp per (point, replication); K <= 256, C <= 512. */
#define CS_POLICY_JFFC 0
#define CS_POLICY_JSQ 1
#define CS_POLICY_SA_JSQ 2
#define CS_POLICY_JIQ 3
#define CS_POLICY_SED 4

#define CS_WL_POISSON 0  /* streams: gaps S[0:n], sizes S[n:2n]            */
#define CS_WL_HORIZON 1  /* streams: 4096-gap blocks cumsum(block)+total, then
                            sizes; arrivals <= t_end, at most n_jobs        */
#define CS_WL_SAMPLED 2  /* arrivals[n], sizes[n] shared by all replications */
#define CS_WL_TRACE 3    /* arrivals[n], tokens_in/out[n]; per-chain hops   */

/* per-replication status (d_rep_status) */
#define CS_REP_QUEUE_OVERFLOW 16  /* a dedicated queue exceeded queue_capacity */
#define CS_REP_EMPTY_HORIZON 17   /* no arrival inside the time horizon          */
#define CS_REP_WARMUP_ALL 18      /* warm-up consumed every arrival              */

typedef struct {
    const cs_sim_point* points;   /* lam used by CS_WL_POISSON / CS_WL_HORIZON */
    int32_t n_points;
    int32_t policy;               /* CS_POLICY_*                              */
    int32_t workload;             /* CS_WL_*                                  */
    int32_t max_chains, max_capacity;
    const double* rates;          /* chains at points[p].chain_base           */
    const int32_t* caps;
    const double* streams;        /* CS_WL_POISSON / CS_WL_HORIZON            */
    int64_t lds;
    double horizon_time_s;        /* CS_WL_HORIZON: t_end                     */
    double warmup_cut_s;          /* CS_WL_HORIZON: warmup_fraction * t_end   */
    const double* arrivals;       /* CS_WL_SAMPLED / CS_WL_TRACE              */
    const double* sizes;          /* CS_WL_SAMPLED                            */
    const int32_t* tokens_in;     /* CS_WL_TRACE                              */
    const int32_t* tokens_out;
    const int32_t* hop_begin;     /* CS_WL_TRACE: hops of global chain c are  */
    const int32_t* hop_server;    /*  hop_begin[c] .. hop_begin[c+1]-1        */
    const int32_t* hop_blocks;    /*  (server index, blocks_at_dst)           */
    const double* server_param;   /*  4 per server: rtt+overhead ms, block
                                      overhead ms, prefill ms, decode ms      */
    int32_t rep_begin, n_reps, n_reps_total;
    int64_t n_jobs;               /* n (HORIZON: the horizon_jobs cap)        */
    int64_t warm;                 /* int(warmup_fraction*n); HORIZON: per rep */
    double* responses;            /* as cs_jffc_sim (row o, completion order) */
    int64_t ldr;
    double* busy;
    int32_t ldb;
    cs_rep_summary* summary;
    double* jobs;                 /* NULL or [o][n][4] job records            */
    int64_t* rep_jobs;            /* NULL or per row o: jobs simulated (HORIZON) */
    int32_t* rep_status;          /* per row o: CS_OK or CS_REP_*             */
    void* queue_workspace;        /* dedicated policies: n_points*n_reps*
                                     max_chains*queue_capacity*16 bytes      */
    int32_t queue_capacity;       /* per chain, power of two                  */
} cs_sim_ext_args;

int cs_sim_ext(const cs_sim_ext_args* args, void* stream);

/* Ragged response rows (time-horizon mode, counts[row] responses each):
 * sums[row] = numpy pairwise sum of the row (responses.mean() numerator,
 * sim.py:407), and entries counts[row]..ldr-1 set to +inf so cs_rep_stats
 * can select the merged order statistics over uniform rows. */
int cs_ragged_rows(double* d_resp, int32_t n_rows, int64_t ldr, const int64_t* d_counts,
                   double* d_sums, void* stream);

/* ------------------------------------------------------------------------ */
/* Statistics over stored responses (run_sim aggregation, sim.py:406-438)     */
/* ------------------------------------------------------------------------ */
/* n_groups groups (sweep points) of rows_per_group consecutive response rows
 * of m values (row stride ldr, even).
 *  * d_summary[row].resp_mean = responses.mean() of the row, bit-exact with
 *    numpy's pairwise summation (sim.py:407); d_row_sums (optional) gets the
 *    row sums.
 *  * if ranks != NULL: exact order statistics.  ranks[g*n_ranks + i]
 *    (0-based, np.sort order of group g's merged responses; negative = from
 *    the end) -> out_values[g*n_ranks + i] (host).  Replaces
 *    np.sort(np.concatenate(...)) + the order statistics np.quantile
 *    interpolates (sim.py:406,436-438).  n_ranks <= 6.
 * Synchronises `stream`. */
int cs_rep_stats(const double* d_resp, int32_t n_groups, int64_t rows_per_group, int64_t m,
                 int64_t ldr, cs_rep_summary* d_summary, const int64_t* ranks, int32_t n_ranks,
                 double* out_values, double* d_row_sums, void* stream);

/* Sharded variant (one process per GPU, after cs_comm_init): every rank holds
 * rows_per_group rows of each group (equal shards); ranks index the union of
 * all ranks' responses; the histograms and bracket counts are all-reduced
 * over NCCL so every rank returns the same exact global order statistics. */
int cs_rep_stats_dist(const double* d_resp, int32_t n_groups, int64_t rows_per_group, int64_t m,
                      int64_t ldr, cs_rep_summary* d_summary, const int64_t* ranks, int32_t n_ranks,
                      double* out_values, double* d_row_sums, void* stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU: the engine's NCCL communicator (one process per GPU)            */
/* ------------------------------------------------------------------------ */
/* Replications shard across GPUs with no data-path exchange (sim.py:400-404
 * replications are independent); the only collectives are the final
 * statistics (cs_rep_stats_dist).  Rank 0 creates the id, the driver
 * broadcasts it (torch.distributed), every rank calls cs_comm_init. */
int cs_nccl_unique_id(void* out128);
int cs_comm_init(const void* unique_id128, int32_t nranks, int32_t rank);
int cs_comm_destroy(void);

/* ------------------------------------------------------------------------ */
/* End to end from HOST buffers                                               */
/* ------------------------------------------------------------------------ */
/* run_sim (sim.py:397-456) for n_points sweep points sharing seed `entropy`
 * (uint32 words) and replications [rep_begin, rep_begin+n_reps): keys ->
 * streams -> simulation -> per-rep means + order statistics, all on the
 * device.  points/rates/caps/ranks are host arrays; outputs are host arrays:
 * out_summary[o], out_busy[o*ldb + k], out_rank_values[g*n_ranks + i],
 * out_responses (NULL or rows*(n-warm), completion order), out_jobs (NULL or
 * rows*n*4).  max_stream_bytes bounds the stream scratch
 * (replications are processed in chunks; 0 = unbounded). */
int cs_run_sim_host(const cs_sim_point* points, int32_t n_points, const double* rates,
                    const int32_t* caps, int32_t n_chain_entries, const uint32_t* entropy,
                    int32_t n_entropy, int32_t rep_begin, int32_t n_reps, int64_t n_jobs,
                    int64_t warm, const int64_t* ranks, int32_t n_ranks, int32_t log1p_variant,
                    int64_t max_stream_bytes, cs_rep_summary* out_summary, double* out_busy,
                    int32_t ldb, double* out_rank_values, double* out_responses, double* out_jobs,
                    void* stream);

/* ------------------------------------------------------------------------ */
/* Composition: GBP-CR placement and GCA chain composition                   */
/* ------------------------------------------------------------------------ */
/* One composition point: servers server_base..server_base+J-1 of the fleet
 * SoA arrays, service (L, s_m, s_c), design parameter c, lambda, rho_bar. */
typedef struct {
    int32_t n_servers;
    int32_t server_base;
    int64_t block_count;
    int64_t block_bytes;
    int64_t cache_slot_bytes;
    int64_t capacity;
    double arrival_rate;
    double load_target;
} cs_compose_point;

/* greedy_block_placement for every point (placement.py:35-132).
 * Per point p (offsets server_base): first/count/max_blocks/bound_time[J];
 * order[J] = GBP visit order (-1 padded); chain_end[J] = 1 where a chain
 * closes in `order`; n_chains[p]; scaled_rate[p]; rate_satisfied[p];
 * status[p] in {CS_OK, CS_INFEASIBLE, CS_INVALID}.  All device pointers. */
int cs_gbp_batch(const cs_compose_point* d_points, int32_t n_points, int32_t max_servers,
                 const int64_t* d_mem,
                 const double* d_tau_c, const double* d_tau_p, const int32_t* d_id_rank,
                 int32_t* d_first, int32_t* d_count, int32_t* d_max_blocks, double* d_bound_time,
                 int32_t* d_order, int32_t* d_chain_end, int32_t* d_n_chains,
                 double* d_scaled_rate, int32_t* d_rate_satisfied, int32_t* d_status,
                 void* stream);

/* greedy_cache_allocation for every point's placement (cache_alloc.py:65-135,
 * model.py:130-231).  d_residual: per-server residual slots or NULL for the
 * full budget.  Outputs per point p, capacity max_chains chains of at most
 * max_hops servers: chain_srv[(p*max_chains + k)*max_hops + h] (server index
 * within the point, -1 padded), chain_len, caps, times (service_time_s),
 * n_chains[p], n_edges[p], status[p]. */
int cs_gca_batch(const cs_compose_point* d_points, int32_t n_points, int32_t max_servers,
                 int32_t max_block_count, const int64_t* d_mem,
                 const double* d_tau_c, const double* d_tau_p, const int32_t* d_id_rank,
                 const int32_t* d_first, const int32_t* d_count, const int64_t* d_residual,
                 int32_t max_chains, int32_t max_hops, int32_t* d_chain_srv,
                 int32_t* d_chain_len, int32_t* d_caps, double* d_times, int32_t* d_n_chains,
                 int64_t* d_n_edges, int32_t* d_status, void* stream);

/* ---- occupancy bounds (analysis.py:67-147): the capacity-sweep caller ---- */

/* One composed system: chains chain_base..+n_chains-1 of d_rates/d_caps
 * (rates descending, as ChainRates), arrival rate lam. */
typedef struct {
    int32_t n_chains;
    int32_t chain_base;
    double lam;
} cs_bound_point;

typedef struct {
    double lower_occupancy;   /* birth-death with death_rate_bounds()[0]  */
    double upper_occupancy;   /* birth-death with death_rate_bounds()[1]  */
    double lower_response_s;  /* lower_occupancy / lam (Little)           */
    double upper_response_s;
    double total_rate;        /* sum(r*c), CPython float sum (analysis.py:60) */
    int32_t total_capacity;
    int32_t status;           /* CS_OK, or CS_UNSTABLE when lam >= total_rate */
} cs_bounds_out;

/* occupancy_bounds() for every point (replaces analysis.py:121-147 per
 * call; bound_curve analysis.py:270-297 batches the capacity sweep through
 * it).  d_workspace: n_points * 2 * (max_capacity + 1) doubles. */
int cs_occupancy_bounds(const cs_bound_point* d_points, int32_t n_points, const double* d_rates,
                        const int32_t* d_caps, int32_t max_capacity, double* d_workspace,
                        cs_bounds_out* d_out, void* stream);

/* birth_death_mean_occupancy() (analysis.py:84-109) with explicit death
 * rates d_death[base .. base+n_states-1] and total_rate; lam < total_rate
 * and all death rates > 0 are the caller's checks (ValueError/UnstableError
 * raised before the call).  d_workspace: n_points * (max_states + 1)
 * doubles. */
typedef struct {
    int32_t n_states;
    int32_t base;
    double lam;
    double total_rate;
} cs_bd_point;

int cs_birth_death_occupancy(const cs_bd_point* d_points, int32_t n_points,
                             const double* d_death, int32_t max_states, double* d_workspace,
                             double* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CHAINSERVE_B200_H */
