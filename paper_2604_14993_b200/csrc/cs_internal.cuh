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

// Keep freed stream-ordered allocations in the device pool instead of
// returning them to the OS at every synchronisation (default threshold 0).
void ensure_mem_pool();

// NCCL all-reduces of the sharded statistics (dist.cu); no-ops without a
// multi-rank communicator.
bool dist_active();
int dist_nranks();
int allreduce_u32(void* buf, size_t count, cudaStream_t st);
int allreduce_u64(void* buf, size_t count, cudaStream_t st);
int allreduce_max_u64(void* buf, size_t count, cudaStream_t st);

// Python-semantics helpers (no contraction; explicit IEEE round-to-nearest).
__device__ __forceinline__ double py_div(double a, double b) { return __ddiv_rn(a, b); }

}  // namespace cs
