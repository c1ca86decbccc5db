// cs_internal.cuh -- shared helpers of the libchainserve_b200 sources.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/chainserve_b200.h"

namespace cs {

// Thread-local last-error message (cs_last_error()).
void set_error(const char* fmt, ...);

// Every kernel launch of the library is followed by check_launch(), which
// also counts it (cs_launch_count(): evidence of the GPU path in benchmarks).
void count_launch();

inline int check_launch(const char* what) {
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

inline int check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

// The engine's private stream-ordered pool (capi.cu): scratch of the
// host-level calls comes from it; pool_alloc = cudaMallocFromPoolAsync.
void ensure_mem_pool();
cudaMemPool_t engine_pool();
int pool_alloc(void** p, size_t n, cudaStream_t st);

// NCCL all-reduces of the sharded statistics (dist.cu); no-ops without a
// multi-rank communicator.
bool dist_active();
int dist_nranks();
int allreduce_u32(void* buf, size_t count, cudaStream_t st);
int allreduce_u64(void* buf, size_t count, cudaStream_t st);
int allreduce_max_u64(void* buf, size_t count, cudaStream_t st);

// Arrival-time prefix of the segmented single-chain simulator, computed
// while the exponential streams are generated (exp_stream.cu, jffc_seg.cu).
struct PrefixPlan {
    static constexpr int MAXEV = 72;   // job indices recorded per row
    static constexpr int MAXP32 = 1;   // points per stream: up to 32 (more: the standalone pre-pass)
    const cs_sim_point* pts;           // lam of every point
    int32_t P;                         // points sharing each stream
    int32_t nev, ncol;
    int64_t n_cum;                     // the first n_cum draws are the gaps
    int32_t ev_idx[MAXEV];             // ascending job indices
    int32_t ev_col[MAXEV];             // output column of each
    double* out;                       // [stream * P + p][ncol]
};

// Python-semantics helpers (no contraction; explicit IEEE round-to-nearest).
__device__ __forceinline__ double py_div(double a, double b) { return __ddiv_rn(a, b); }

// CPython 3.12 sum() of floats: Neumaier compensated summation starting from
// int 0 (Python/bltinmodule.c builtin_sum_impl), used for chain service
// times (model.py:204) and total rates (analysis.py:60).
struct PySum {
    double f, c;
    bool started;
    __device__ void init() {
        f = 0.0;
        c = 0.0;
        started = false;
    }
    __device__ void add(double x) {
        if (!started) {
            f = x;  // int 0 + x
            started = true;
            return;
        }
        const double t = __dadd_rn(f, x);
        if (fabs(f) >= fabs(x))
            c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else
            c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        f = t;
    }
    __device__ double result() const { return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f; }
};

}  // namespace cs
