// dist.cu -- the single cross-GPU exchange of a sharded sweep, over NCCL.
//
// Replications are independent (sim.py:400-404), so a sweep shards by
// replication block with no data-path communication.  What crosses GPUs is
// only the final aggregation: the per-replication summaries (all-gathered by
// the Python driver) and, for the exact global quantiles, the radix-select
// histograms and bracket counts of stats.cu (all-reduced here, a few hundred
// KB per round over NVLink/NVSwitch).  One communicator per process (one
// process per GPU); bootstrapped by the driver broadcasting the unique id.
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

#include "cs_internal.cuh"

namespace cs {

static ncclComm_t g_comm = nullptr;
static int g_rank = 0, g_nranks = 1;

bool dist_active() { return g_comm != nullptr && g_nranks > 1; }
int dist_nranks() { return dist_active() ? g_nranks : 1; }

static int nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        set_error("%s: %s", what, ncclGetErrorString(r));
        return CS_ERR_CUDA;
    }
    return CS_OK;
}

int allreduce_u32(void* buf, size_t count, cudaStream_t st) {
    if (!dist_active()) return CS_OK;
    return nccl_check(ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, g_comm, st), "ncclAllReduce(u32)");
}

int allreduce_u64(void* buf, size_t count, cudaStream_t st) {
    if (!dist_active()) return CS_OK;
    return nccl_check(ncclAllReduce(buf, buf, count, ncclUint64, ncclSum, g_comm, st), "ncclAllReduce(u64)");
}

int allreduce_max_u64(void* buf, size_t count, cudaStream_t st) {
    if (!dist_active()) return CS_OK;
    return nccl_check(ncclAllReduce(buf, buf, count, ncclUint64, ncclMax, g_comm, st), "ncclAllReduce(max)");
}

}  // namespace cs

using namespace cs;

extern "C" int cs_nccl_unique_id(void* out128) {
    ncclUniqueId id;
    int rc = nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
    if (rc == CS_OK) memcpy(out128, &id, sizeof(id));
    return rc;
}

extern "C" int cs_comm_init(const void* uid128, int32_t nranks, int32_t rank) {
    if (g_comm) {
        ncclCommDestroy(g_comm);
        g_comm = nullptr;
    }
    ncclUniqueId id;
    memcpy(&id, uid128, sizeof(id));
    const int rc = nccl_check(ncclCommInitRank(&g_comm, nranks, id, rank), "ncclCommInitRank");
    if (rc == CS_OK) {
        g_rank = rank;
        g_nranks = nranks;
    }
    return rc;
}

extern "C" int cs_comm_destroy(void) {
    if (g_comm) ncclCommDestroy(g_comm);
    g_comm = nullptr;
    g_nranks = 1;
    g_rank = 0;
    return CS_OK;
}
