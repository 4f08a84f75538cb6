// diag.cu — measurement entry point: the attainable fp64-pipe rate of this GPU, the roofline
// denominator of the pole kernel (the fp64 peak is not in MEASURED_PEAKS.json; bench.py
// measures it in the same run as the step, DESIGN.md §6.1 "Roofline").
//
// Kernel: every thread runs 8 independent DFMA chains x[i] = fma(x[i], y[i], z[j]) with
// per-thread register operands (the pole kernel's operand pattern: its DFMAs read register
// and shared-memory-broadcast operands); grid = SMs x 16 blocks of 128 threads, so every
// scheduler holds 16 warps x 8 chains — far more than the 4 independent DFMAs per SMSP that
// hide the 8-cycle latency (profiles/r01_fp64_latency.jsonl). Counted: 1 fp64-pipe op per DFMA.
#include <cuda_runtime.h>

#include "launch.h"
#include "../../include/rexi.h"

namespace {

__global__ void __launch_bounds__(128) dfma_peak_kernel(double *out, int iters, double a, double b) {
    double x[8], y[8], z[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = threadIdx.x * 1e-3 + i;
        y[i] = a + 1e-9 * (threadIdx.x + i);
        z[i] = b - 1e-9 * i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y[i], z[(i + u) & 7]);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;   // never true; keeps the chains live
}

}  // namespace

extern "C" rexi_status_t rexi_fp64_peak(int device, int reps, double *ops_per_s, double *best_ms) {
    if (!ops_per_s || reps < 1) {
        rexi::set_last_error("rexi_fp64_peak: null output or reps < 1");
        return REXI_EINVAL;
    }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    double *out = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int sms = 0;
    float best = 1e30f;
    const int iters = 1 << 12, threads = 128;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 16;
    if (e == cudaSuccess) e = cudaMalloc(&out, threads * sizeof(double));
    if (e == cudaSuccess) e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    if (e == cudaSuccess) {
        dfma_peak_kernel<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);   // warm-up
        e = cudaGetLastError();
    }
    for (int r = 0; r < reps && e == cudaSuccess; ++r) {
        cudaEventRecord(e0);
        dfma_peak_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        e = cudaEventSynchronize(e1);
        float ms = 0;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
        if (e == cudaSuccess && ms < best) best = ms;
    }
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (out) cudaFree(out);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        rexi::set_last_error(cudaGetErrorString(e));
        return REXI_ECUDA;
    }
    const double ops = (double)blocks * threads * iters * 64.0;
    *ops_per_s = ops / (best * 1e-3);
    if (best_ms) *best_ms = best;
    return REXI_OK;
}
