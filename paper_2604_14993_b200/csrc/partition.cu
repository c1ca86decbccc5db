// partition.cu -- SM partitions for the pipelined sweep engine (green contexts).
//
// A sweep's simulator blocks stay resident for the whole simulation (one
// serial job chain per thread), so its length is set by the most loaded SM.
// Run beside it on shared SMs, the previous sweep's statistics and the next
// sweep's streams either pile the simulator's blocks onto a few SMs or steal
// issue slots from the most loaded ones (measured 40-59 ms per sweep,
// bimodal).  Splitting the device's SMs into two green contexts gives the
// simulator a fixed set of SMs (its blocks spread evenly, nothing else runs
// there) and everything else the remainder.  Kernels are launched through the
// runtime API on the partitions' streams; memory and events stay those of the
// primary context.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "chainserve_b200.h"
#include "cs_internal.cuh"

namespace {

struct Partition {
    bool made = false;
    int rc = CS_OK;
    int sim_sms = 0, aux_sms = 0, sim_sms_actual = 0;
    CUgreenCtx g_sim = nullptr, g_aux = nullptr;
    CUstream s_sim = nullptr, s_aux[2] = {nullptr, nullptr};
};

constexpr int MAX_PARTS = 8;  // per device, keyed by the simulator's SM count
Partition g_part[64][MAX_PARTS];
std::mutex g_part_mu;

// driver entry points through the runtime (no link-time libcuda dependency:
// the library must load on hosts without a driver)
struct Drv {
    CUresult (*DeviceGet)(CUdevice*, int);
    CUresult (*DeviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType);
    CUresult (*DevSmResourceSplitByCount)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*,
                                          unsigned, unsigned);
    CUresult (*DevResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned);
    CUresult (*GreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
    CUresult (*GreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned, int);
    CUresult (*GetErrorString)(CUresult, const char**);
};

int load_drv(Drv& d) {
    struct {
        const char* name;
        void** fn;
    } tab[] = {{"cuDeviceGet", (void**)&d.DeviceGet},
               {"cuDeviceGetDevResource", (void**)&d.DeviceGetDevResource},
               {"cuDevSmResourceSplitByCount", (void**)&d.DevSmResourceSplitByCount},
               {"cuDevResourceGenerateDesc", (void**)&d.DevResourceGenerateDesc},
               {"cuGreenCtxCreate", (void**)&d.GreenCtxCreate},
               {"cuGreenCtxStreamCreate", (void**)&d.GreenCtxStreamCreate},
               {"cuGetErrorString", (void**)&d.GetErrorString}};
    for (auto& t : tab) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint(t.name, t.fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || *t.fn == nullptr) {
            cs::set_error("cs_sm_partition: driver entry point %s unavailable", t.name);
            return CS_ERR_CUDA;
        }
    }
    return CS_OK;
}

Drv g_drv;

int drv(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return CS_OK;
    const char* e = nullptr;
    if (g_drv.GetErrorString) g_drv.GetErrorString(r, &e);
    cs::set_error("cs_sm_partition: %s: %s", what, e ? e : "?");
    return CS_ERR_CUDA;
}

}  // namespace

extern "C" int cs_sm_partition(int32_t sim_sms, void** sim_stream, void** aux_streams,
                               int32_t* out_sim_sms, int32_t* out_aux_sms) {
    if (cs_device_count() == 0) {
        cs::set_error("cs_sm_partition: no CUDA device");
        return CS_ERR_CUDA;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_part_mu);
    Partition* slot = nullptr;
    for (auto& q : g_part[dev & 63])
        if (q.made && q.sim_sms == sim_sms) slot = &q;
    if (!slot)
        for (auto& q : g_part[dev & 63])
            if (!q.made && !slot) slot = &q;
    if (!slot) {
        cs::set_error("cs_sm_partition: too many partition shapes on one device");
        return CS_INVALID;
    }
    Partition& P = *slot;
    if (!P.made) {
        P.made = true;
        P.sim_sms = sim_sms;
        int rc;
        CUdevice cd;
        CUdevResource all, grp[1], rest;
        unsigned n = 1;
        CUdevResourceDesc d_sim, d_aux;
        cudaFree(nullptr);  // the runtime's primary context exists
        const Drv& D = g_drv;
        if ((!D.DeviceGet && (rc = load_drv(g_drv))) || (rc = drv(D.DeviceGet(&cd, dev), "cuDeviceGet")) ||
            (rc = drv(D.DeviceGetDevResource(cd, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource")) ||
            (rc = drv(D.DevSmResourceSplitByCount(grp, &n, &all, &rest, 0, (unsigned)sim_sms),
                      "cuDevSmResourceSplitByCount")) ||
            (rc = drv(D.DevResourceGenerateDesc(&d_sim, grp, 1), "cuDevResourceGenerateDesc")) ||
            (rc = drv(D.DevResourceGenerateDesc(&d_aux, &rest, 1), "cuDevResourceGenerateDesc")) ||
            (rc = drv(D.GreenCtxCreate(&P.g_sim, d_sim, cd, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate")) ||
            (rc = drv(D.GreenCtxCreate(&P.g_aux, d_aux, cd, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate")) ||
            (rc = drv(D.GreenCtxStreamCreate(&P.s_sim, P.g_sim, CU_STREAM_NON_BLOCKING, 0),
                      "cuGreenCtxStreamCreate")) ||
            (rc = drv(D.GreenCtxStreamCreate(&P.s_aux[0], P.g_aux, CU_STREAM_NON_BLOCKING, 0),
                      "cuGreenCtxStreamCreate")) ||
            (rc = drv(D.GreenCtxStreamCreate(&P.s_aux[1], P.g_aux, CU_STREAM_NON_BLOCKING, 0),
                      "cuGreenCtxStreamCreate"))) {
            P.rc = rc;
            return rc;
        }
        if (n != 1 || rest.sm.smCount == 0) {
            cs::set_error("cs_sm_partition: cannot split %u SMs at %d", all.sm.smCount, sim_sms);
            P.rc = CS_INVALID;
            return CS_INVALID;
        }
        P.sim_sms = sim_sms;
        P.rc = CS_OK;
        P.aux_sms = (int)rest.sm.smCount;
        P.sim_sms_actual = (int)grp[0].sm.smCount;
    }
    if (P.rc != CS_OK) return P.rc;
    *sim_stream = (void*)P.s_sim;
    aux_streams[0] = (void*)P.s_aux[0];
    aux_streams[1] = (void*)P.s_aux[1];
    if (out_sim_sms) *out_sim_sms = P.sim_sms_actual;
    if (out_aux_sms) *out_aux_sms = P.aux_sms;
    return CS_OK;
}
