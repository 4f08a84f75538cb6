// Cycle cost of the fused step's warp FFT (small2_ffts) and of the Stockham fft_in_smem on the
// same shared-memory slabs, one CTA of 256 threads, 6 transforms of 64 points (the C1 shape).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -o tools/fft_probe tools/fft_probe.cu
#include "../paper_2008_11607_b200/csrc/kernels.cu"
#include <cstdio>

using namespace rexi;

__global__ void fft_probe_kernel(long long *out, const cd *tw_g, int mode) {
    constexpr int LOGD = 6, D = 64, PL = padded_len(D);
    __shared__ cd slab[6 * (PL + 1)];
    __shared__ cd tws[D];
    for (int i = threadIdx.x; i < 6 * (PL + 1); i += blockDim.x) slab[i] = mk(i * 1e-3, 0.5);
    for (int i = threadIdx.x; i < D; i += blockDim.x) tws[i] = tw_g[i];
    __syncthreads();
    long long t[6];
    for (int r = 0; r < 6; ++r) {
        t[r] = clock64();
        if (mode == 0) {
            small2_ffts<LOGD>(slab, PL + 1, 6, 6, tws, r & 1);   // (the warp-shuffle variant when measured)
        } else {
            const int tf = 8, col = threadIdx.x / tf, tt = threadIdx.x - col * tf;
            if (r & 1) fft_in_smem<true, true>(slab + col * (PL + 1), D, LOGD, tt, tf, tws, col < 6);
            else fft_in_smem<false, true>(slab + col * (PL + 1), D, LOGD, tt, tf, tws, col < 6);
        }
    }
    const long long t6 = clock64();
    if (threadIdx.x == 0)
        for (int r = 0; r < 6; ++r) out[r] = (r < 5 ? t[r + 1] : t6) - t[r];
    if (threadIdx.x == 1) out[8] = (long long)(slab[3].x * 1e6);
}

int main() {
    cd h[64];
    for (int j = 0; j < 64; ++j) h[j] = cd{cos(-2 * M_PI * j / 64), sin(-2 * M_PI * j / 64)};
    cd *tw;
    long long *d;
    cudaMalloc(&tw, sizeof h);
    cudaMalloc(&d, 16 * sizeof(long long));
    cudaMemcpy(tw, h, sizeof h, cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            fft_probe_kernel<<<1, 256>>>(d, tw, mode);
            cudaDeviceSynchronize();
        }
        long long o[16];
        cudaMemcpy(o, d, sizeof o, cudaMemcpyDeviceToHost);
        printf("{\"probe\": \"fft64x6\", \"kind\": \"%s\", \"cycles_per_call\": [%lld, %lld, %lld, %lld, %lld, %lld], \"err\": \"%s\"}\n",
               mode == 0 ? "warp_shuffle_radix2" : "stockham_radix8_smem", o[0], o[1], o[2], o[3], o[4], o[5],
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
