// Whole-GPU rate of the non-fused fp64 operations the fp64 plans are made of
// (tools only; VERDICT r1 "FP64 non-tensor throughput was never measured").
// DADD.rn and DMUL.rn with 8 independent accumulators per thread, 1024 threads
// per SM x 4 waves, timed with CUDA events; prints G op/s and op/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(256) k_rate(double *out, int iters, double b) {
    double a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.5 + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = OP == 0 ? __dadd_rn(a[i], b) : __dmul_rn(a[i], b);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.678) out[0] = s;  // never true: keeps the loop
}
template <int OP>
static void run(const char *name, int sms, double mhz, double *d) {
    const int iters = 1 << 14, grid = sms * 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_rate<OP><<<grid, 256>>>(d, iters, OP == 0 ? 1.0 : 1.0000001);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_rate<OP><<<grid, 256>>>(d, iters, OP == 0 ? 1.0 : 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * 256 * 8 * iters;
    double gops = ops / (ms * 1e-3) / 1e9;
    printf("{\"op\": \"%s\", \"ms\": %.4f, \"gops\": %.1f, \"op_per_clk_per_sm\": %.2f, \"sm_mhz_assumed\": %.0f}\n", name, ms,
           gops, gops * 1e9 / (sms * mhz * 1e6), mhz);
}
int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    double *d;
    cudaMalloc(&d, 64);
    printf("{\"device\": \"%s\", \"sms\": %d, \"max_sm_mhz\": %.0f}\n", p.name, p.multiProcessorCount, khz / 1e3);
    run<0>("dadd.rn.f64", p.multiProcessorCount, khz / 1e3, d);
    run<1>("dmul.rn.f64", p.multiProcessorCount, khz / 1e3, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("cuda error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
