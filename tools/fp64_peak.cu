// fp64_peak.cu — measured DFMA throughput of this B200 (roofline denominator check).
// Each thread runs 8 independent DFMA chains; grid = SMs x 8 blocks x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}
int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1024 * sizeof(double));
    const int iters = 1 << 16, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"sms\": %d, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"dfma_per_clk_per_sm_at_1965MHz\": %.2f}\n",
           sms, fmas / (best * 1e-3), 2 * fmas / (best * 1e-3) / 1e12, fmas / (best * 1e-3) / sms / 1.965e9);
    return 0;
}
