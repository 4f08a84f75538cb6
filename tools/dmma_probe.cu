// dmma_probe.cu — does B200's fp64 MMA (mma.sync m8n8k4 f64) run beside the DFMA pipe?
// Kernels: DFMA only, DMMA only, both interleaved; prints fp64 flop rates.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int KIND>
__global__ void __launch_bounds__(128) probe(double *out, int iters) {
    double x[8], acc[8][2];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x * 1e-3 + i; acc[i][0] = acc[i][1] = 0.0; }
    const double a = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (KIND == 0 || KIND == 2) x[i] = fma(x[i], a, b);
            if (KIND == 1 || KIND == 2) dmma(acc[i], a + i, b);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i] + acc[i][0] + acc[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int KIND>
void run(const char *name, int sms, double *out) {
    const int iters = 1 << 12, blocks = sms * 8, threads = 128;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<KIND><<<blocks, threads>>>(out, 16);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        probe<KIND><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warps = (double)blocks * threads / 32;
    const double dfma_flops = (KIND == 0 || KIND == 2) ? (double)blocks * threads * iters * 8 * 2 : 0;
    const double dmma_flops = (KIND == 1 || KIND == 2) ? warps * iters * 8 * (8 * 8 * 4 * 2) : 0;
    printf("{\"kind\": \"%s\", \"ms\": %.3f, \"dfma_tflops\": %.2f, \"dmma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
           name, best, dfma_flops / best / 1e9, dmma_flops / best / 1e9, (dfma_flops + dmma_flops) / best / 1e9);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1024 * sizeof(double));
    run<0>("dfma", sms, out);
    run<1>("dmma", sms, out);
    run<2>("dfma+dmma", sms, out);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
