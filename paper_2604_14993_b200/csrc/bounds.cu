// bounds.cu -- steady-state occupancy bounds of fastest-free dispatch,
// batched over composed systems (chainserve analysis.py:67-147), the
// per-capacity evaluation inside bound_curve / tune_capacity_bound
// (analysis.py:270-336).
//
// One CTA per (system, bound): blockIdx.y = 0 packs jobs onto the fastest
// chains (death_rate_bounds()[0] -> lower occupancy), 1 onto the slowest
// (death_rate_bounds()[1] -> upper occupancy).  Per state n = 1..C a thread
// evaluates the death rate with the reference's sequential per-chain sum
// (bit-exact), then log(lam) - log(d_n); the log-weight cumsum runs in state
// order on one thread (np.cumsum order); logsumexp (scipy 1.18 form: the
// maximal terms are split out, log1p(s/m) + log(m) + max) and the weighted
// head sum are block reductions.  log/exp are CUDA's (<= 1 ulp from numpy's),
// so results carry a stated tolerance, not bit-exactness.
#include <cuda_runtime.h>
#include <math.h>

#include "cs_internal.cuh"

extern "C" int cs_device_count(void);

namespace cs {

constexpr int BD_THREADS = 256;

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < BD_THREADS / 32; i++) t = __dadd_rn(t, red[i]);
        red[BD_THREADS / 32] = t;
    }
    __syncthreads();
    return red[BD_THREADS / 32];
}

__device__ double block_max(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = -INFINITY;
        for (int i = 0; i < BD_THREADS / 32; i++) t = fmax(t, red[i]);
        red[BD_THREADS / 32] = t;
    }
    __syncthreads();
    return red[BD_THREADS / 32];
}

// birth_death_mean_occupancy (analysis.py:84-109).  On entry w[n], n=1..C,
// holds log(lam) - log(d_n); w[0] is set here.  Returns the mean occupancy.
__device__ double bd_occupancy(double* w, int C, double lam, double nu, double* red) {
    if (threadIdx.x == 0) {  // log_w = [0] ++ cumsum(...)   (analysis.py:101)
        w[0] = 0.0;
        double acc = w[1];
        for (int n = 2; n <= C; n++) {
            acc = __dadd_rn(acc, w[n]);
            w[n] = acc;
        }
    }
    __syncthreads();
    const double wC = w[C];
    const double tail = __dsub_rn(__dadd_rn(wC, log(nu)), log(__dsub_rn(nu, lam)));  // :102
    // logsumexp(log_w[:C] ++ [tail])   (:103)
    double mx = threadIdx.x == 0 ? tail : -INFINITY;
    for (int n = threadIdx.x; n < C; n += BD_THREADS) mx = fmax(mx, w[n]);
    const double amax = block_max(mx, red);
    double cnt = 0.0, s = 0.0;
    for (int n = threadIdx.x; n <= C; n += BD_THREADS) {
        const double a = n < C ? w[n] : tail;
        if (a == amax)
            cnt = __dadd_rn(cnt, 1.0);
        else
            s = __dadd_rn(s, exp(__dsub_rn(a, amax)));
    }
    const double m = block_sum(cnt, red);
    s = block_sum(s, red);
    if (s != 0.0) s = __ddiv_rn(s, m);
    const double log_z = __dadd_rn(__dadd_rn(log1p(s), log(m)), amax);
    // head = sum(n * exp(log_w[1:C] - log_z))   (:104-105)
    double h = 0.0;
    for (int n = 1 + threadIdx.x; n < C; n += BD_THREADS)
        h = __dadd_rn(h, __dmul_rn((double)n, exp(__dsub_rn(w[n], log_z))));
    const double head = block_sum(h, red);
    const double rho = __ddiv_rn(lam, nu);
    const double one_m = __dsub_rn(1.0, rho);
    const double fac = __dadd_rn(__ddiv_rn(rho, __dmul_rn(one_m, one_m)), __ddiv_rn((double)C, one_m));
    const double queued = __dmul_rn(exp(__dsub_rn(wC, log_z)), fac);  // :106
    return __dadd_rn(head, queued);
}

__global__ void __launch_bounds__(BD_THREADS) occupancy_bounds_kernel(
    const cs_bound_point* __restrict__ pts, const double* __restrict__ rates,
    const int32_t* __restrict__ caps, int32_t max_cap, double* __restrict__ ws,
    cs_bounds_out* __restrict__ out) {
    __shared__ double red[BD_THREADS / 32 + 1];
    __shared__ double s_nu;
    __shared__ int s_C;
    const int p = blockIdx.x, y = blockIdx.y;
    const cs_bound_point pt = pts[p];
    const int K = pt.n_chains;
    const double* __restrict__ mu = rates + pt.chain_base;
    const int32_t* __restrict__ cp = caps + pt.chain_base;
    if (threadIdx.x == 0) {  // ChainRates.total_rate / total_capacity (analysis.py:58-64)
        PySum nu;
        nu.init();
        int C = 0;
        for (int k = 0; k < K; k++) {
            nu.add(__dmul_rn(mu[k], (double)cp[k]));
            C += cp[k];
        }
        s_nu = nu.result();
        s_C = C;
    }
    __syncthreads();
    const double nu = s_nu, lam = pt.lam;
    const int C = s_C;
    if (!(lam < nu) || C > max_cap) {
        if (threadIdx.x == 0 && y == 0) {
            out[p].total_rate = nu;
            out[p].total_capacity = C;
            out[p].status = C > max_cap ? CS_INVALID : CS_UNSTABLE;
        }
        return;
    }
    double* w = ws + ((size_t)p * 2 + y) * (size_t)(max_cap + 1);
    const double llam = log(lam);
    // death_rate_bounds(rates, n) (analysis.py:67-81), n = 1..C
    for (int n = 1 + threadIdx.x; n <= C; n += BD_THREADS) {
        double d = 0.0;
        if (y == 0) {
            int ahead = 0;
            for (int k = 0; k < K; k++) {
                d = __dadd_rn(d, __dmul_rn(mu[k], (double)min(cp[k], max(n - ahead, 0))));
                ahead += cp[k];
            }
        } else {
            int behind = C;
            for (int k = 0; k < K; k++) {
                behind -= cp[k];
                d = __dadd_rn(d, __dmul_rn(mu[k], (double)min(cp[k], max(n - behind, 0))));
            }
        }
        w[n] = __dsub_rn(llam, log(d));
    }
    __syncthreads();
    const double occ = bd_occupancy(w, C, lam, nu, red);
    if (threadIdx.x == 0) {
        const double resp = __ddiv_rn(occ, lam);
        if (y == 0) {
            out[p].lower_occupancy = occ;
            out[p].lower_response_s = resp;
            out[p].total_rate = nu;
            out[p].total_capacity = C;
            out[p].status = CS_OK;
        } else {
            out[p].upper_occupancy = occ;
            out[p].upper_response_s = resp;
        }
    }
}

__global__ void __launch_bounds__(BD_THREADS) birth_death_kernel(
    const cs_bd_point* __restrict__ pts, const double* __restrict__ death, int32_t max_states,
    double* __restrict__ ws, double* __restrict__ out) {
    __shared__ double red[BD_THREADS / 32 + 1];
    const int p = blockIdx.x;
    const cs_bd_point pt = pts[p];
    const int C = pt.n_states;
    double* w = ws + (size_t)p * (size_t)(max_states + 1);
    const double llam = log(pt.lam);
    for (int n = 1 + threadIdx.x; n <= C; n += BD_THREADS)
        w[n] = __dsub_rn(llam, log(death[pt.base + n - 1]));
    __syncthreads();
    const double occ = bd_occupancy(w, C, pt.lam, pt.total_rate, red);
    if (threadIdx.x == 0) out[p] = occ;
}

}  // namespace cs

extern "C" int cs_occupancy_bounds(const cs_bound_point* d_points, int32_t n_points,
                                   const double* d_rates, const int32_t* d_caps,
                                   int32_t max_capacity, double* d_workspace, cs_bounds_out* d_out,
                                   void* stream) {
    using namespace cs;
    if (cs_device_count() == 0) {
        set_error("cs_occupancy_bounds: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (n_points < 0 || max_capacity < 1 || !d_points || !d_rates || !d_caps || !d_workspace || !d_out) {
        set_error("cs_occupancy_bounds: invalid arguments");
        return CS_INVALID;
    }
    if (n_points == 0) return CS_OK;
    occupancy_bounds_kernel<<<dim3(n_points, 2), BD_THREADS, 0, (cudaStream_t)stream>>>(
        d_points, d_rates, d_caps, max_capacity, d_workspace, d_out);
    return check_launch("occupancy_bounds_kernel");
}

extern "C" int cs_birth_death_occupancy(const cs_bd_point* d_points, int32_t n_points,
                                        const double* d_death, int32_t max_states,
                                        double* d_workspace, double* d_out, void* stream) {
    using namespace cs;
    if (cs_device_count() == 0) {
        set_error("cs_birth_death_occupancy: no CUDA device");
        return CS_ERR_CUDA;
    }
    if (n_points < 0 || max_states < 1 || !d_points || !d_death || !d_workspace || !d_out) {
        set_error("cs_birth_death_occupancy: invalid arguments");
        return CS_INVALID;
    }
    if (n_points == 0) return CS_OK;
    birth_death_kernel<<<n_points, BD_THREADS, 0, (cudaStream_t)stream>>>(d_points, d_death,
                                                                          max_states, d_workspace,
                                                                          d_out);
    return check_launch("birth_death_kernel");
}
