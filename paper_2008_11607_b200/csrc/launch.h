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

// Algorithmic work of the pole kernel per (pole, Fourier mode), counted from its source:
// flops (FMA = 2, MUL/ADD = 1) and fp64-pipe instructions (FMA/MUL/ADD = 1 each).
// DESIGN.md "Pole kernel" lists the count line by line.
constexpr double kFlopsDZ = 131.0, kOpsDZ = 71.0;
constexpr double kFlopsUV = 183.0, kOpsUV = 101.0;

}  // namespace rexi
