// Latency / throughput of a few FP64 operations on this GPU (development
// probe for the simulator's per-job critical path).  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double x0, double y, int n) {
    double x = x0;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) x = __dadd_rn(x, y);
    long long t1 = clock64();
    double z = x;
    for (int i = 0; i < n; i++) z = __dmul_rn(z, y);
    long long t2 = clock64();
    double w = z;
    for (int i = 0; i < n; i++) w = (w <= y) ? y : w + 1e-300;  // DSETP + FSEL + DADD
    long long t3 = clock64();
    float f = (float)w;
    for (int i = 0; i < n; i++) f = f * 1.0000001f + 1e-7f;
    long long t4 = clock64();
    out[0] = x + z + w + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

// 8 independent DADD chains per thread: throughput-bound with enough warps
__global__ void thr(double* out, double y, int n) {
    double x[8];
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x + k;
    for (int i = 0; i < n; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = __dadd_rn(x[k], y);
    double s = 0;
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 32);
    const int n = 4096;
    lat<<<1, 32>>>(d, c, 1.0, 1e-3, n);
    lat<<<1, 32>>>(d, c, 1.0, 1e-3, n);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: dadd %.2f dmul %.2f dsetp+fsel+dadd %.2f ffma %.2f\n",
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int m = 20000;
        thr<<<sms, 32 * warps>>>(d, 1e-3, m);
        cudaEventRecord(a);
        thr<<<sms, 32 * warps>>>(d, 1e-3, m);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double dadds = (double)sms * warps * 32 * 8 * m;
        printf("warps/SM %2d: %.3f ms, %.1f DADD lanes/clk/SM at 1.965 GHz (%.2f TFLOP/s)\n", warps, ms,
               dadds / (ms * 1e-3) / sms / 1.965e9, dadds / (ms * 1e-3) / 1e12);
    }
    return 0;
}
