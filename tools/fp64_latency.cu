// fp64_latency.cu — DFMA dependent-chain latency and the parallelism needed to fill the fp64
// pipe of one SM: one block of W warps, C independent DFMA chains per thread; reports
// DFMA per clock per SM (clock64 over the loop). Run: ./tools/fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chain(double *out, long long *cyc, int iters, double a, double b) {
    double x[C];
#pragma unroll
    for (int i = 0; i < C; ++i) x[i] = threadIdx.x * 1e-3 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += x[i];
    if (s == 1234.5) out[threadIdx.x] = s;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(double *out, long long *dcyc) {
    const int iters = 256;
    for (int W : {1, 2, 4, 8, 12, 16, 24, 32}) {
        chain<C><<<1, 32 * W>>>(out, dcyc, iters, 0.999999, 1e-7);
        cudaDeviceSynchronize();
        long long cyc;
        cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
        double fmas = 32.0 * W * iters * 16 * C;
        printf("{\"chains_per_thread\": %d, \"warps\": %d, \"dfma_per_clk_sm\": %.2f, \"cycles_per_dep_dfma\": %.2f}\n",
               C, W, fmas / cyc, (double)cyc / (iters * 16));
    }
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    run<1>(out, cyc);
    run<2>(out, cyc);
    run<4>(out, cyc);
    run<8>(out, cyc);
    return 0;
}
