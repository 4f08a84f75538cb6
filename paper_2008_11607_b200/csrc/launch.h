// launch.h — host-side launchers of the device kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace rexi {

cudaError_t fft_setup_attributes();
cudaError_t launch_fft_rows(const void *const in[3], void *const out[3], bool real_in, bool real_out,
                            const cd *tw, int D, int inverse, double scale, cudaStream_t st);
cudaError_t launch_fft_cols(const void *const in[3], void *const out[3], const cd *tw, int D,
                            int inverse, double scale, cudaStream_t st);
int pole_modes_per_block(int mpt);
bool pole_config_supported(int variant, int mpt, int pu, int minb);
cudaError_t pole_occupancy(int variant, int mpt, int pu, int minb, int *blocks_per_sm);
cudaError_t launch_poles(const PoleArgs &a, int variant, int mpt, int pu, int minb, cudaStream_t st);
cudaError_t launch_finish(const FinishArgs &a, cudaStream_t st);
cudaError_t launch_fixup_k0(const FixupArgs &a, cudaStream_t st);
cudaError_t launch_hermitian(const cd *in, cd *out, long n_modes, int D, cudaStream_t st);

// Algorithmic work of the pole kernel per (pole, Fourier mode), counted from its source:
// flops (FMA = 2, MUL/ADD = 1) and fp64-pipe instructions (FMA/MUL/ADD = 1 each).
// The denominator 1/(kappa + K2) costs 7 ops / 11 flops; with MPT = 4 (K2 quads) it is shared
// by four modes. DESIGN.md "Pole kernel" lists the count line by line.
constexpr double kFlopsDZ = 131.0, kOpsDZ = 71.0;
constexpr double kFlopsUV = 183.0, kOpsUV = 101.0;
constexpr double kDenFlops = 11.0, kDenOps = 7.0;
// REXI (kind 2): solve 1 (num 6/12, den 7/11, eta1 4/6, delta1 4/8, zeta1 6/10) + 3 MACs 12/24.
constexpr double kFlopsREXI = 71.0, kOpsREXI = 39.0;
inline double pole_flops(int kind, int mpt) {
    const double f = kind == 0 ? kFlopsDZ : kind == 1 ? kFlopsUV : kFlopsREXI;
    return mpt == 4 ? f - kDenFlops * 0.75 : f;
}
inline double pole_ops(int kind, int mpt) {
    const double f = kind == 0 ? kOpsDZ : kind == 1 ? kOpsUV : kOpsREXI;
    return mpt == 4 ? f - kDenOps * 0.75 : f;
}

}  // namespace rexi
