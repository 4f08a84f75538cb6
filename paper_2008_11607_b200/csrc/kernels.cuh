// kernels.cuh — device code of librexi (sm_100a): batched fp64 FFT passes, the fused
// REXII pole kernel, the chunk reduction / velocity recovery and the K = 0 fix-up.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "planner.h"

#ifndef REXI_RCP_F32_SEED
#define REXI_RCP_F32_SEED 0
#endif

// REXI_CHECKED builds (librexi_checked.so, paper_2008_11607_b200/build.py --checked): device-side
// bounds checks on every global / shared-memory index of the default path, a trap on failure
// (the replacement for compute-sanitizer memcheck, which this pool does not allow). Compiled out
// otherwise.
#ifdef REXI_CHECKED
#include <cstdio>
#define RX_ASSERT(cond)                                                                            \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("REXI_CHECKED: (%s) failed at %s:%d block (%d,%d) thread %d\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                  \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define RX_ASSERT(cond) \
    do {                \
    } while (0)
#endif

namespace rexi {

// bytes of dynamic shared memory of the running block (%dynamic_smem_size)
__device__ __forceinline__ unsigned dyn_smem_bytes() {
    unsigned r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
// a complex index into the block's dynamic shared memory is in range
#define RX_SMEM(i) RX_ASSERT((long)(i) >= 0 && ((long)(i) + 1) * 16 <= (long)dyn_smem_bytes())

// ----------------------------------------------------------------------------- complex fp64
struct __align__(16) cd {
    double x, y;
};

__device__ __forceinline__ cd mk(double x, double y) { return cd{x, y}; }
// a*b
__device__ __forceinline__ cd cmul(cd a, cd b) {
    return mk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ cd cfma(cd a, cd b, cd c) {
    return mk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// c - a*b
__device__ __forceinline__ cd cfms(cd a, cd b, cd c) {
    return mk(fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y)));
}
// conj(a)*b + c
__device__ __forceinline__ cd cjfma(cd a, cd b, cd c) {
    return mk(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
// c - conj(a)*b
__device__ __forceinline__ cd cjfms(cd a, cd b, cd c) {
    return mk(fma(-a.x, b.x, fma(-a.y, b.y, c.x)), fma(-a.x, b.y, fma(a.y, b.x, c.y)));
}

// 1/d for d > 0 (normal range): MUFU.RCP64H seed + one cubic Newton step
// (relative error ~ e0^3 with e0 ~ 2^-20 seed error). Not correctly rounded; <= 1 ulp.
__device__ __forceinline__ double rcp_pos(double d) {
    double r;
#if REXI_RCP_F32_SEED
    // seed from the fp32 MUFU (XU pipe) instead of MUFU.RCP64H; |d| in fp32 range
    float rf;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"(__double2float_rn(d)));
    r = (double)rf;
#else
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
#endif
    double e = fma(-d, r, 1.0);
    e = fma(e, e, e);
    return fma(e, r, r);
}

// ----------------------------------------------------------------------------- pole kernel
struct PoleArgs {
    const cd *fhat;        // [3][D*D]
    cd *partial;           // [n_chunks][3][D*D]
    const PoleConst *poles;
    const R2CPole *rpoles; // the same poles, R2C kernel layout
    const R2XPole *xpoles; // the same poles, explicit-solve R2C kernel layout
    const double *ksym;    // [D]
    long pole_begin, pole_end;
    long n_modes;          // D*D
    int n_chunks;
    int D, log2D;
    double tau;            // c (tau-scaled Coriolis)
    double hmu;            // Re(alpha_n) = h mu (same for every pole)
    long sk_tiles;         // R2C stream-K: tiles of 128 octet items (0: chunked launch)
    int sk_slots;          // R2C stream-K: partial slots per tile
    long partial_cap;      // complex values in `partial` (REXI_CHECKED bounds checks)
    long n_poles;          // entries of the pole tables (REXI_CHECKED)
};

struct FinishArgs {
    const cd *partial;     // [n_chunks][3][D*D]
    cd *acc;               // [3][D*D]
    const cd *fhat;        // [3][D*D] (kinds 0, 2: for m0 = zeta0 - c eta0)
    const double *ksym;
    long n_modes;
    int n_chunks;
    int D, log2D;
    int kind;              // pole-kernel kind (0 DZ, 1 UV, 2 REXI, 3 DZ3)
    double tau;
    cd S;                  // zeta rebuild: sum over the pole range of w1/alpha + w2/|alpha|^2
    cd Sd;                 // kind 5: sum over the pole range of w1
    long sk_tiles;         // R2C stream-K (see PoleArgs); 0: chunked partials
    int sk_slots, sk_ctas;
    long sk_poles;         // pole-range length
    long partial_cap;      // complex values in `partial` (REXI_CHECKED)
    int half_out;          // R2C kinds: write only the modes with k <= D/2 (what the inverse
                           // transform of a Hermitian spectrum reads), not both modes of a pair
};

struct FixupArgs {
    int method;            // 0: REXII, 1: REXI
    int write_eta;         // R2C kind: also write eta = S e0 at the corners
    cd S;
    const cd *fhat;
    cd *acc;
    const PoleConst *poles;
    long pole_begin, pole_end;
    long n_modes;
    int D;
};

// ----------------------------------------------------------------------------- fused small-grid step
// The whole physical step S1..S5 for small grids as one launch of thread-block clusters
// (kernels.cu step_small2_kernel): forward FFT, PFHX pole loop with the K = 0 corners, R2C
// finish and inverse FFT, the stages exchanging data through distributed shared memory; the pole
// range split over n_clusters clusters whose partial spectra the last one to finish sums.
constexpr int kSmallMaxClusters = 9;   // 16-CTA clusters on 148 SMs
struct SmallArgs {
    const double *in[3];
    double *out[3];
    PoleArgs pole;         // xpoles, ksym, pole range, D, log2D, tau, hmu (r2x_setup_ld / r2x_tile)
    const PoleConst *poles;   // generic pole table (K = 0 corners)
    int method;            // 0: REXII, 1: REXI (corners: one solve per term)
    const cd *tw;
    double scale;          // D^-2
    long n_items;          // octet work items (r2c_items(D, 2, true))
    int stop_after;        // measurement only (REXI_SMALL_STOP): return after stage 0..4
    int steps;             // steps of a spectral-resident run (> 1 with one cluster only)
    int n_clusters;
    cd Sg[kSmallMaxClusters], Sdg[kSmallMaxClusters];   // per-cluster range sums (finish S, Sd)
    cd *cl_acc;            // [n_clusters][3][D][D/2 + 1] (n_clusters > 1)
    unsigned *counter;     // clusters arrived; 0 between launches (n_clusters > 1)
    long long *trace;      // measurement only (REXI_SMALL_TRACE): clock64 per CTA at stage marks
};

// ----------------------------------------------------------------------------- FFT passes
struct FftArgs {
    const void *in[3];
    void *out[3];
    const cd *twiddle;     // D/2 entries e^{-2 pi i j/D}
    int D, log2D;
    int per_block;         // rows (row pass) or columns (column pass) per block
    int inverse;           // 0: e^{-}, 1: e^{+}
    double scale;
    int half_out;          // forward columns: write only rows l <= D/2 of the spectrum (every
                           // representative of a {K, -K} pair; the R2C consumers read no other)
};

}  // namespace rexi
