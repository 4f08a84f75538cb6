// launch.h — host-side launchers of the device kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace rexi {

// thread-local text returned by rexi_last_error() (capi.cu); scalar.cu sets it on its failures
void set_last_error(const char *msg);

cudaError_t fft_setup_attributes();
// S1: real fields -> full spectrum (x scale); half = D x D complex scratch per field.
// half_out: only rows l <= D/2 of the spectrum are written (the R2C pole kernels' inputs)
cudaError_t launch_fft_forward(const double *const in[3], cd *const half[3], cd *const out[3],
                               const cd *tw, int D, double scale, cudaStream_t st, bool half_out = false);
// S5: Re(IDFT(in)) -> real fields; hermitian: in is known Hermitian (skip symmetrisation).
cudaError_t launch_fft_inverse(const cd *const in[3], cd *const half[3], double *const out[3],
                               bool hermitian, const cd *tw, int D, cudaStream_t st);
int pole_modes_per_block(int mpt);
bool pole_config_supported(int variant, int mpt, int pu, int minb);
cudaError_t pole_occupancy(int variant, int mpt, int pu, int minb, int *blocks_per_sm);
cudaError_t launch_poles(const PoleArgs &a, int variant, int mpt, int pu, int minb, cudaStream_t st);
cudaError_t launch_finish(const FinishArgs &a, cudaStream_t st);
bool pole_r2c_supported(int mpt, int pu, int minb);
long pole_r2c_blocks(int D, int mpt);
cudaError_t pole_r2c_occupancy(int mpt, int pu, int minb, int *blocks_per_sm);
cudaError_t launch_poles_r2c(const PoleArgs &a, int mpt, int pu, int minb, cudaStream_t st);
// explicit-solve R2C kernel (PFHX, kind 7; octet items, modes_per_thread 8)
bool pole_r2x_supported(int mpt, int pu, int minb);
cudaError_t pole_r2x_occupancy(int pu, int minb, int *blocks_per_sm);
long pole_r2x_blocks(int D, int minb);   // grid.x of the PFHX kernel (block size by min blocks)
cudaError_t launch_poles_r2x(const PoleArgs &a, int pu, int minb, cudaStream_t st);
// stream-K R2C (octet items, modes_per_thread 8): persistent grid of `ctas` blocks
cudaError_t launch_poles_r2c_sk(const PoleArgs &a, int pu, int ctas, cudaStream_t st);
cudaError_t pole_r2c_sk_occupancy(int pu, int *blocks_per_sm);
long pole_r2c_sk_tiles(int D);
long sk_slots_bound(long tiles, long poles, long ctas);
cudaError_t launch_finish_r2c_sk(const FinishArgs &a, cudaStream_t st);
cudaError_t launch_fixup_k0(const FixupArgs &a, cudaStream_t st, bool beside_pole_kernel);
cudaError_t launch_hermitian(const cd *in, cd *out, long n_modes, int D, cudaStream_t st);
// fused small-grid step (step_small2_kernel): octet work items; cluster size (16 where the
// device allows it, else 8; 0: cluster launch unavailable) and the number of resident clusters
// of that size; launch of a.n_clusters clusters
long small_step_items(int D);
constexpr int kSmallThreadsHost = 256;
int small2_cluster(int *resident);
cudaError_t launch_step_small2(const SmallArgs &a, int cs, cudaStream_t st);
// NEXT-3 1-D transforms: power-of-two n <= 2048 by Stockham passes (twiddle table of n entries
// from launch_twiddles), other n by a direct DFT; out = scale * DFT(in) (inverse: e^{+})
bool dft1d_uses_fft(long n);
cudaError_t launch_twiddles(cd *tw, int n, cudaStream_t st);
cudaError_t launch_dft1d(const cd *in, cd *out, long n, bool inverse, double scale, const cd *tw, cudaStream_t st);
// rows D/2+1 .. D-1 of a Hermitian spectrum from rows 1 .. D/2-1 (in place)
cudaError_t launch_mirror_rows(cd *acc, long n_modes, int D, cudaStream_t st);

// Algorithmic work of the pole kernel per (pole, Fourier mode), counted from its source:
// flops (FMA = 2, MUL/ADD = 1) and fp64-pipe instructions (FMA/MUL/ADD = 1 each), by kind.
//   kind 3 (DZ3, all three accumulated): 71 ops / 131 flops (DESIGN.md 6.1 table)
//   kind 0 (DZ): kind 3 without zeta2 (4/6) and the two zeta MACs (8/16): 59 / 109
//   kind 1 (UV, paper-literal): 101 / 183
//   kind 2 (REXI): solve 1 without zeta1 (num 6/12, den 7/11, eta1 4/6, delta1 4/8) + 2 MACs 8/16
//   kind 4 (PF): two solves of f0 (num 6/12 and numt 6/12, eta 4/6 each, delta 4/8 each),
//                shared den 7/11, 4 MACs 16/32: 51 / 95
//   kind 5 (PFH): PF without the two delta back-substitutions (4/8 each): 43 / 79
//   kind 6 (R2C pairs, real input): per K2 value, den 7/11, the delta0 weight sums sigma, tau'
//     (four real FMAs each from the planner's coefficients) 8/16 and the two fused weights
//     X1 q, Y1 q 8/12; per pair (two modes) num1 + num_t 2/4, the non-delta0 part w of
//     num1 - num_t 4/6 and 8 real-times-complex MACs 8/16 = 14/26.
//     A quad (4 modes, own K2) = 51 / 91; an octet (8 modes, shared K2) = 79 / 143, i.e.
//     12.75 / 22.75 resp. 9.875 / 17.875 per mode; modes_per_thread 8 uses octets for the
//     (H-1)(H-2)/2 interior quad pairs (a, b), (b, a) and half-discarded octets for the other
//     3(H-1) quads.
//   kind 7 (PFHX, explicit solves on R2C pairs, real input; the default): per K2 value and pole
//     den 7/11 and the per-pole delta0 coefficients sigma_n, tau'_n (2 MUL + 2 FMA each) 8/12;
//     per pair and pole the two right-hand sides num1 = Z + Q, num_t = Z - Q with
//     Z = h mu eta0 - sr m0 (2 FMA) and Q = delta0 + i (hn eta0 - si m0) (4 FMA), 4 ADD: 10/16,
//     the two solutions eta1 = q num1, eta_t = conj(q) num_t (2 MUL + 2 FMA each) 8/12, their
//     sum and difference (4 ADD) 4/4 and the Hermitian accumulation of eta and delta' (16 FMA)
//     16/32 = 38/64. An octet (8 modes, shared K2) = 167 / 279, i.e. 20.875 / 34.875 per mode
//     (+ the discarded halves of the 3(H-1) single-quad items, as for kind 6). (Before the
//     shared Z, Q: 12 FMA for num1, num_t, 175 / 311 per octet.)
// The denominator 1/(kappa + K2) costs 7 ops / 11 flops; with MPT = 4 (K2 quads) it is shared
// by four modes.
constexpr double kDenFlops = 11.0, kDenOps = 7.0;
inline double r2c_per_mode(int mpt, int D, double quad, double octet) {
    if (mpt != 8) return quad / 4.0;
    // every octet item (incl. the 3 (H-1) single quads run as half-discarded octets) costs
    // `octet`; the work per useful mode counts the discarded half
    const double H = D / 2, n_oct = H >= 3 ? (H - 1) * (H - 2) / 2 : 0, n_single = 3 * (H - 1);
    return (n_oct + n_single) * octet / (8 * n_oct + 4 * n_single);
}
inline double pole_flops(int kind, int mpt, int D) {
    if (kind == 6) return r2c_per_mode(mpt, D, 91.0, 143.0);
    if (kind == 7) return r2c_per_mode(8, D, 0.0, 279.0);
    const double f[6] = {109.0, 183.0, 53.0, 131.0, 95.0, 79.0};
    return mpt == 4 ? f[kind] - kDenFlops * 0.75 : f[kind];
}
inline double pole_ops(int kind, int mpt, int D) {
    if (kind == 6) return r2c_per_mode(mpt, D, 51.0, 79.0);
    if (kind == 7) return r2c_per_mode(8, D, 0.0, 167.0);
    const double f[6] = {59.0, 101.0, 29.0, 71.0, 51.0, 43.0};
    return mpt == 4 ? f[kind] - kDenOps * 0.75 : f[kind];
}

}  // namespace rexi
