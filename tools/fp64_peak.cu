// fp64_peak.cu — attainable fp64-pipe throughput of this B200 (roofline denominator check).
// Variants: DFMA with uniform operands, DFMA with per-thread operands, DMUL, and a mix close
// to the pole kernel's (fp64 : LDS : MUFU.RCP64H ~ 142 : 9 : 2). All: grid = SMs x 16 blocks
// x 128 threads, 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(128) loop_kernel(double *out, int iters, double a, double b) {
    __shared__ double sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 1e-3 * i;
    __syncthreads();
    double x[8], y[8], z[8];
    for (int i = 0; i < 8; ++i) {
        x[i] = threadIdx.x * 1e-3 + i;
        y[i] = a + 1e-9 * (threadIdx.x + i);
        z[i] = b - 1e-9 * i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (KIND == 0) x[i] = fma(x[i], a, b);
                if (KIND == 1) x[i] = fma(x[i], y[i], z[(i + u) & 7]);
                if (KIND == 2) x[i] = x[i] * y[i];
            }
            if (KIND == 3) {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y[i], z[(i + u) & 7]);
                // ~ 8 fp64 : 0.5 LDS : 0.125 MUFU
                if (u & 1) x[u] += sh[(it + u) & 255];
                if (u == 3) {
                    double r;
                    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[2] + 3.0));
                    x[1] = fma(x[1], r, 1e-30);
                }
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int KIND>
void run(const char *name, int sms, double *out) {
    const int iters = 1 << 13, blocks = sms * 16, threads = 128;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    loop_kernel<KIND><<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        loop_kernel<KIND><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double ops = (double)blocks * threads * iters * 64 * (KIND == 3 ? 1.0 : 1.0);
    printf("{\"kind\": \"%s\", \"fp64_ops_per_s\": %.4e, \"per_clk_per_sm_at_1965MHz\": %.2f, \"ms\": %.3f}\n",
           name, ops / (best * 1e-3), ops / (best * 1e-3) / sms / 1.965e9, best);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, 1024 * sizeof(double));
    run<0>("dfma_uniform_operands", sms, out);
    run<1>("dfma_register_operands", sms, out);
    run<2>("dmul", sms, out);
    run<3>("dfma_with_lds_mufu_mix", sms, out);
    return 0;
}
