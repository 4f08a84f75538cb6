// kernels.cu — device kernels of librexi (sm_100a, fp64).
//
//  * fft_{rows,cols}_{fwd,inv}{,16}_kernel : real 2-D FFT by batched radix-8 / radix-16 Stockham
//    passes in shared memory (S1 forward transform, S5 inverse transform + Re). PAPER.md:497 "all
//    computations ... in Fourier space"; Alg. 1 lines 1 and last.
//  * fft_cols_cl_kernel               : the column passes at 2048^2 and 4096^2 as 8-CTA clusters
//    (four-step, exchange through distributed shared memory, 128-byte row segments).
//  * pole_kernel_r2x_bulk (default, PFHX) : S2 + S3 for real fields on {K, -K} mode pairs grouped
//    in K2 octets: both Helmholtz-reduced solves of every pole for every pair, fused with the
//    weighted accumulation in registers (eq:lswEta); the pole table streamed
//    into shared memory by bulk copies (cp.async.bulk + mbarrier, double-buffered).
//    pole_kernel_r2x: the same with a register-staged table copy (the other tunings, and
//    REXI_R2X_BULK=0). pole_kernel_r2c (PFHR, collapsed, comparison only) and its stream-K
//    schedule pole_kernel_r2c_sk.
//  * pole_kernel<VARIANT>             : the same for the other variants (UV, DZ, DZ3, PF, PFH)
//    and for complex spectra (rexi_poles). No per-pole solution ever reaches HBM.
//  * finish_kernel (+ finish_r2c_sk)  : fixed-order sum of the per-chunk partial sums, zeta
//    rebuilt from the potential vorticity, (u, v) recovered from (delta, zeta).
//  * fixup_k0_kernel                  : the K = 0 modes (velocities decouple from delta, zeta
//    there): pure Coriolis 2x2 solves per pole.
//  * step_small2_kernel               : the whole step S1..S5 for small grids as one launch of
//    thread-block clusters, stage data exchanged through distributed shared memory.
//  * hermitian_kernel                 : the spectral form of Re(.) between rexi_run steps.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.h"

namespace rexi {

// ============================================================================= FFT
// Batched complex FFT of length D (power of two) in shared memory: Stockham autosort passes of
// radix 8 (then one radix-4 or radix-2 pass), each thread holding 8 values in registers per
// pass, twiddles e^{-2 pi i j / D} from a host table (long double, rounded). A block owns `nb`
// transforms (rows, or a strip of adjacent columns so global accesses stay coalesced); its
// threads = nb * max(1, D/8). Forward: e^{-}; inverse: e^{+} (conjugated twiddles/butterflies).

template <bool INV>
__device__ __forceinline__ cd mul_mi(cd a) {  // a * (-i) forward, a * (+i) inverse
    return INV ? mk(-a.y, a.x) : mk(a.y, -a.x);
}
__device__ __forceinline__ cd cadd(cd a, cd b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd csub(cd a, cd b) { return mk(a.x - b.x, a.y - b.y); }

template <bool INV>
__device__ __forceinline__ void dft2(cd *v) {
    const cd a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(cd *v) {
    // DIF: (v0 + v2, v1 + v3) -> X0, X2 ; (v0 - v2, -i (v1 - v3)) -> X1, X3
    const cd c0 = cadd(v[0], v[2]), c1 = cadd(v[1], v[3]);
    const cd c2 = csub(v[0], v[2]), c3 = mul_mi<INV>(csub(v[1], v[3]));
    v[0] = cadd(c0, c1);
    v[2] = csub(c0, c1);
    v[1] = cadd(c2, c3);
    v[3] = csub(c2, c3);
}

template <bool INV>
__device__ __forceinline__ void dft8(cd *v) {
    const double h = 0.70710678118654752440;  // cos(pi/4)
    cd b[8];
    for (int n = 0; n < 4; ++n) {
        b[n] = cadd(v[n], v[n + 4]);
        b[n + 4] = csub(v[n], v[n + 4]);
    }
    // odd half twiddles w8^n, n = 1, 2, 3 (forward w8 = e^{-i pi/4})
    {
        const cd x = b[5];
        b[5] = INV ? mk(h * (x.x - x.y), h * (x.x + x.y)) : mk(h * (x.x + x.y), h * (x.y - x.x));
        b[6] = mul_mi<INV>(b[6]);
        const cd y = b[7];
        b[7] = INV ? mk(-h * (y.x + y.y), h * (y.x - y.y)) : mk(h * (y.y - y.x), -h * (y.x + y.y));
    }
    dft4<INV>(b);       // -> X0, X2, X4, X6 in b[0], b[1], b[2], b[3]
    dft4<INV>(b + 4);   // -> X1, X3, X5, X7 in b[4..7]
    v[0] = b[0]; v[2] = b[1]; v[4] = b[2]; v[6] = b[3];
    v[1] = b[4]; v[3] = b[5]; v[5] = b[6]; v[7] = b[7];
}

// DFT of length 16 in registers, natural order in and out: n = 4 n1 + n2, k = k1 + 4 k2,
// X[k1 + 4 k2] = sum_n2 w4^(n2 k2) [w16^(n2 k1) sum_n1 w4^(n1 k1) x[4 n1 + n2]].
template <bool INV>
__device__ __forceinline__ void dft16(cd *v) {
    // cos / sin of 2 pi m / 16, m = 0..9 (products n2 k1 <= 9)
    constexpr double C[10] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613,
                              -1.0, -0.92387953251128675613};
    constexpr double S[10] = {0.0, 0.38268343236508977173, 0.70710678118654752440, 0.92387953251128675613,
                              1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173,
                              0.0, -0.38268343236508977173};
    cd y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        cd g[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
        dft4<INV>(g);
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            const int m = n2 * k1;
            // w16^m = cos(2 pi m/16) -+ i sin(2 pi m/16) (forward: e^{-})
            const double c = C[m], sn = INV ? S[m] : -S[m];
            y[n2][k1] = m == 0 ? g[k1] : mk(g[k1].x * c - g[k1].y * sn, g[k1].x * sn + g[k1].y * c);
        }
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        cd g[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
        dft4<INV>(g);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = g[k2];
    }
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(cd *v) {
    if (R == 16) dft16<INV>(v);
    else if (R == 8) dft8<INV>(v);
    else if (R == 4) dft4<INV>(v);
    else dft2<INV>(v);
}

// Padded shared-memory index: one pad slot per 8 values, so the stride-8 writes of the first
// Stockham pass (and the stride-N/8 reads) spread over the banks.
__device__ __forceinline__ int pidx(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int padded_len(int N) { return N + (N >> 3); }

// Twiddles w_r = e^{-+2 pi i r step / N}, r = 1..R-1, of one butterfly: w_1, w_2, w_4 from the
// table (e^{-2 pi i j / N}, j < N), the others as products of two or three of them (<= 3 ulp;
// the table loads through L1 were the FFT's limiter with one load per r).
// TWS: the table is in shared memory (fused small-grid step), read with generic loads.
template <bool TWS>
__device__ __forceinline__ double2 ld_tw(const double2 *p) {
    if (TWS) return *p;
    return __ldg(p);
}
template <int R, bool INV, bool TWS = false>
__device__ __forceinline__ void pass_twiddles(const cd *__restrict__ tw, int step, cd *w) {
    const double2 *t = reinterpret_cast<const double2 *>(tw);
    const double2 a = ld_tw<TWS>(t + step);
    w[1] = mk(a.x, INV ? -a.y : a.y);
    if (R >= 4) {
        const double2 b = ld_tw<TWS>(t + 2 * step);
        w[2] = mk(b.x, INV ? -b.y : b.y);
        w[3] = cmul(w[1], w[2]);
    }
    if (R >= 8) {
        const double2 c4 = ld_tw<TWS>(t + 4 * step);
        w[4] = mk(c4.x, INV ? -c4.y : c4.y);
        w[5] = cmul(w[1], w[4]);
        w[6] = cmul(w[2], w[4]);
        w[7] = cmul(w[3], w[4]);
    }
    if (R == 16) {
        const double2 c8 = ld_tw<TWS>(t + 8 * step);
        w[8] = mk(c8.x, INV ? -c8.y : c8.y);
#pragma unroll
        for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
    }
}

// The block's dynamic shared memory (all FFT kernels keep their transforms there).
__device__ __forceinline__ cd *rx_smem_base() {
    extern __shared__ cd rx_dyn_smem[];
    return rx_dyn_smem;
}

// REXI_CHECKED: fill the block's dynamic shared memory with NaN first, so a read of a slot the
// kernel never wrote propagates into the result (compared with the oracle by the checked tests).
__device__ __forceinline__ void rx_poison_smem() {
#ifdef REXI_CHECKED
    cd *b = rx_smem_base();
    const int n = (int)(dyn_smem_bytes() / sizeof(cd));
    for (int i = threadIdx.x; i < n; i += blockDim.x) b[i] = mk(__longlong_as_double(-1LL), __longlong_as_double(-1LL));
    __syncthreads();
#endif
}

// Element i of a transform held in shared memory at s[ix(i)]: PidxIx for a padded contiguous
// transform (pidx), other accessors for strided ones (columns of the fused small-grid step).
struct PidxIx {
    __device__ __forceinline__ int operator()(int i) const { return pidx(i); }
};

// One Stockham pass of radix R on the transform at s (length N, current span Ns); thread t of
// tf threads per transform handles butterflies j = t, t + tf, ... < N/R.
// V values per thread (8, or 16 for the radix-16 passes): V / R butterflies per thread.
template <int R, bool INV, class IX, bool TWS = false, int V = 8>
__device__ __forceinline__ void stockham_pass_ix(cd *s, IX ix, int N, int Ns, int t, int tf,
                                                 const cd *__restrict__ tw, bool act) {
    constexpr int PERMAX = V / R;
    const int nbf = N / R;
    cd v[V];
#pragma unroll
    for (int b = 0; b < PERMAX; ++b) {
        const int j = t + b * tf;
        if (act && b * tf < nbf && j < nbf) {
            const int k = j & (Ns - 1);
            const int step = k * (N / (Ns * R));  // twiddle index step: r * k * N / (Ns R)
            cd w[R];
            if (Ns > 1) pass_twiddles<R, INV, TWS>(tw, step, w);
            RX_ASSERT(Ns == 1 || R * step < N);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                RX_SMEM((s - rx_smem_base()) + ix(j + r * nbf));
                cd x = s[ix(j + r * nbf)];
                if (r > 0 && Ns > 1) x = cmul(x, w[r]);
                v[b * R + r] = x;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < PERMAX; ++b) {
        const int j = t + b * tf;
        if (act && b * tf < nbf && j < nbf) {
            dftR<R, INV>(v + b * R);
            const int k = j & (Ns - 1);
            const int d = (j - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                RX_SMEM((s - rx_smem_base()) + ix(d + r * Ns));
                s[ix(d + r * Ns)] = v[b * R + r];
            }
        }
    }
    __syncthreads();
}

template <int R, bool INV>
__device__ __forceinline__ void stockham_pass(cd *s, int N, int logN, int Ns, int t, int tf,
                                              const cd *__restrict__ tw, bool act = true) {
    (void)logN;
    stockham_pass_ix<R, INV>(s, PidxIx{}, N, Ns, t, tf, tw, act);
}

// act = false: the thread only joins the block barriers (blocks with more threads than
// transforms x tf, e.g. the fused small-grid step)
template <bool INV, class IX, bool TWS = false, int V = 8>
__device__ __forceinline__ void fft_in_smem_ix(cd *s, IX ix, int N, int logN, int t, int tf, const cd *tw,
                                               bool act) {
    int Ns = 1, rem = logN;
    while (rem >= 3) {
        stockham_pass_ix<8, INV, IX, TWS, V>(s, ix, N, Ns, t, tf, tw, act);
        Ns <<= 3;
        rem -= 3;
    }
    if (rem == 2) stockham_pass_ix<4, INV, IX, TWS, V>(s, ix, N, Ns, t, tf, tw, act);
    else if (rem == 1) stockham_pass_ix<2, INV, IX, TWS, V>(s, ix, N, Ns, t, tf, tw, act);
}

template <bool INV, bool TWS = false>
__device__ __forceinline__ void fft_in_smem(cd *s, int N, int logN, int t, int tf, const cd *tw,
                                            bool act = true) {
    fft_in_smem_ix<INV, PidxIx, TWS>(s, PidxIx{}, N, logN, t, tf, tw, act);
}

// ----------------------------------------------------------------------------- real 2-D FFT
// The physical fields are real, so both 2-D transforms use the two Hermitian symmetries
// (half the butterflies and half the shared-memory traffic of a complex 2-D FFT):
//  * rows: two real rows x1, x2 are transformed as one complex row z = x1 + i x2;
//    X1[k] = (Z[k] + conj Z[N-k]) / 2, X2[k] = (Z[k] - conj Z[N-k]) / (2i).
//  * half spectrum: a row's X[k] for k in [1, N/2) plus the two real values X[0], X[N/2]
//    packed into slot 0 as (X[0], X[N/2]) — N/2 complex slots per row.
//  * columns: only the N/2 columns of the half spectrum are transformed; slot 0 holds two real
//    columns packed as one complex column and is separated with the same rule along l.
// Shared memory: one transform per padded slab (pidx); column slabs are padded so that the 8
// lanes of a 128-bit shared-memory wavefront (C columns x 8/C rows) hit distinct bank groups.

__host__ __device__ __forceinline__ int col_stride(int N, int C) { return padded_len(N) + (C < 8 ? 8 / C : 1); }

// Forward rows: real fields -> half spectra. Block = nb row pairs of one field, tf = N/8 threads
// per pair.
__global__ void __launch_bounds__(1024) fft_rows_fwd_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, nb = a.per_block;
    const int tf = D >= 8 ? D / 8 : 1;
    const int H = D >> 1;
    const size_t pair0 = (size_t)blockIdx.x * nb;
    const int n = nb * D;   // complex values in the block
    const double *inp = static_cast<const double *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *outp = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    const int PL = padded_len(D);
    rx_poison_smem();
    cd tmp[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            const int pr = i >> log2D, x = i & (D - 1);
            const size_t g = (2 * (pair0 + pr)) * D + x;
            RX_ASSERT(g + D < (size_t)D * D);
            tmp[q] = mk(__ldg(inp + g), __ldg(inp + g + D));
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            RX_SMEM((i >> log2D) * PL + pidx(i & (D - 1)));
            smem[(i >> log2D) * PL + pidx(i & (D - 1))] = tmp[q];
        }
    }
    __syncthreads();
    const int row = threadIdx.x / tf, t = threadIdx.x - row * tf;
    fft_in_smem<false>(smem + row * PL, D, log2D, t, tf, a.twiddle);
    const double hs = 0.5 * a.scale;
    // half-spectrum outputs: nb pairs x H slots x 2 rows
    const int m = nb * H;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int pr = i / H, k = i - pr * H;
        const cd *Z = smem + pr * PL;
        cd X1, X2;
        if (k == 0) {
            const cd z0 = Z[pidx(0)], zh = Z[pidx(H)];
            X1 = mk(2.0 * hs * z0.x, 2.0 * hs * zh.x);
            X2 = mk(2.0 * hs * z0.y, 2.0 * hs * zh.y);
        } else {
            const cd zk = Z[pidx(k)], zm = Z[pidx(D - k)];
            X1 = mk(hs * (zk.x + zm.x), hs * (zk.y - zm.y));
            X2 = mk(hs * (zk.y + zm.y), hs * (zm.x - zk.x));
        }
        const size_t g = (2 * (pair0 + pr)) * D + k;
        RX_ASSERT(g + D < (size_t)D * D && k < H);
        outp[g] = X1;
        outp[g + D] = X2;
    }
}

// ----------------------------------------------------------------------------- radix-16 row passes
// Row passes for 512 <= D <= 8192 with 16 values per thread (T = D/16 threads per transform) and
// radix-16 Stockham passes: the first pass reads its 16 inputs straight from global memory into
// registers (x[j + r T], coalesced over j) and the inverse's last pass writes straight to global
// memory (x[j + r D/R]), so a 4096-point row makes 3 shared-memory round trips instead of 5 —
// the radix-8 row kernels were bound by the shared-memory pipe (ncu l1tex 80 % at 4096^2).
// NB row pairs per block keep >= 128 threads. Same arithmetic as the radix-8 path otherwise
// (separation of the two real rows, packing of X[0], X[N/2] into slot 0).
template <int LOGD>
struct Row16 {
    static constexpr int D = 1 << LOGD, H = D / 2, T = D / 16;
    static constexpr int NB = T >= 128 ? 1 : 128 / T;
    static constexpr int PL = padded_len(D);
};

// radix-16 passes Ns = 16, 256, ... while 4 or more bits remain, then one radix-2/4/8 pass;
// the caller did the first (Ns = 1) pass. Every thread of the block joins the barriers.
template <bool INV, int LOGD>
__device__ __forceinline__ void row16_rest(cd *s, int j, const cd *tw) {
    constexpr int D = 1 << LOGD, T = D / 16;
    int Ns = 16, rem = LOGD - 4;
#pragma unroll
    for (int it = 0; it < 3; ++it) {
        if (rem >= 4) {
            stockham_pass_ix<16, INV, PidxIx, false, 16>(s, PidxIx{}, D, Ns, j, T, tw, true);
            Ns <<= 4;
            rem -= 4;
        }
    }
    if (rem == 3) stockham_pass_ix<8, INV, PidxIx, false, 16>(s, PidxIx{}, D, Ns, j, T, tw, true);
    else if (rem == 2) stockham_pass_ix<4, INV, PidxIx, false, 16>(s, PidxIx{}, D, Ns, j, T, tw, true);
    else if (rem == 1) stockham_pass_ix<2, INV, PidxIx, false, 16>(s, PidxIx{}, D, Ns, j, T, tw, true);
}

template <int LOGD>
__global__ void __launch_bounds__(512) fft_rows_fwd16_kernel(FftArgs a) {
    using L = Row16<LOGD>;
    constexpr int D = L::D, H = L::H, T = L::T, NB = L::NB, PL = L::PL;
    extern __shared__ cd smem[];
    rx_poison_smem();
    const int f = blockIdx.y;
    const int pr = threadIdx.x / T, j = threadIdx.x - pr * T;
    const size_t pair = (size_t)blockIdx.x * NB + pr;
    const double *inp = static_cast<const double *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *outp = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    cd *s = smem + pr * PL;
    {
        cd v[16];
        const double *r1 = inp + (2 * pair) * D;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_ASSERT((2 * pair + 1) * D + j + r * T < (size_t)D * D);
            v[r] = mk(__ldg(r1 + j + r * T), __ldg(r1 + D + j + r * T));
        }
        dft16<false>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_SMEM(pr * PL + pidx(16 * j + r));
            s[pidx(16 * j + r)] = v[r];   // Stockham output of the Ns = 1 pass: 16 j + r
        }
    }
    __syncthreads();
    row16_rest<false, LOGD>(s, j, a.twiddle);
    const double hs = 0.5 * a.scale;
    for (int k = j; k < H; k += T) {
        cd X1, X2;
        if (k == 0) {
            const cd z0 = s[pidx(0)], zh = s[pidx(H)];
            X1 = mk(2.0 * hs * z0.x, 2.0 * hs * zh.x);
            X2 = mk(2.0 * hs * z0.y, 2.0 * hs * zh.y);
        } else {
            const cd zk = s[pidx(k)], zm = s[pidx(D - k)];
            X1 = mk(hs * (zk.x + zm.x), hs * (zk.y - zm.y));
            X2 = mk(hs * (zk.y + zm.y), hs * (zm.x - zk.x));
        }
        const size_t g = (2 * pair) * D + k;
        outp[g] = X1;
        outp[g + D] = X2;
    }
}

template <int LOGD>
__global__ void __launch_bounds__(512) fft_rows_inv16_kernel(FftArgs a) {
    using L = Row16<LOGD>;
    constexpr int D = L::D, H = L::H, T = L::T, NB = L::NB, PL = L::PL;
    extern __shared__ cd smem[];
    rx_poison_smem();
    const int f = blockIdx.y;
    const int pr = threadIdx.x / T, j = threadIdx.x - pr * T;
    const size_t pair = (size_t)blockIdx.x * NB + pr;
    const cd *inp = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    double *outp = static_cast<double *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    cd *s = smem + pr * PL;
    {
        // Z[p] = g1[p] + i g2[p] over the full circle from the two half-spectrum rows
        // (g[D - p] = conj g[p]; slot 0 packs the real values at p = 0 and p = H)
        const cd *g1r = inp + (2 * pair) * D, *g2r = g1r + D;
        cd v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int p = j + r * T;
            cd z;
            if (p == 0) {
                const cd g1 = g1r[0], g2 = g2r[0];
                z = mk(g1.x, g2.x);
            } else if (p == H) {
                const cd g1 = g1r[0], g2 = g2r[0];
                z = mk(g1.y, g2.y);
            } else if (p < H) {
                const cd g1 = g1r[p], g2 = g2r[p];
                z = mk(g1.x - g2.y, g1.y + g2.x);        // g1 + i g2
            } else {
                const cd g1 = g1r[D - p], g2 = g2r[D - p];
                z = mk(g1.x + g2.y, g2.x - g1.y);        // conj g1 + i conj g2
            }
            v[r] = z;
        }
        dft16<true>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_SMEM(pr * PL + pidx(16 * j + r));
            s[pidx(16 * j + r)] = v[r];
        }
    }
    __syncthreads();
    row16_rest<true, LOGD>(s, j, a.twiddle);
    const double sc = a.scale;
    double *o1 = outp + (2 * pair) * D;
#pragma unroll 4
    for (int x = j; x < D; x += T) {
        const cd v = s[pidx(x)];
        o1[x] = v.x * sc;
        o1[x + D] = v.y * sc;
    }
}

// ----------------------------------------------------------------------------- radix-16 column passes
// Column passes for 512 <= D <= 8192: C half-spectrum columns per block, T = D/16 threads per
// column (thread (c, j), c fastest, so a warp's loads cover C adjacent columns of a row), the
// first pass straight from global memory into registers, radix-16 Stockham passes in the
// column slabs, output as in the radix-8 column kernels.
template <int LOGD>
struct Col16 {
    static constexpr int D = 1 << LOGD, H = D / 2, T = D / 16;
    // 512 threads per block: C = 8 / 4 / 2 / 1 columns at D = 1024 / 2048 / 4096 / 8192 (the widest
    // row segment per load; measured best or equal against C = 1, 4, 8: profiles/r02o_fft16c.log)
    static constexpr int C = 512 / T >= 1 ? 512 / T : 1;
    static constexpr int STRIDE = padded_len(D) + 1;
};

template <int LOGD>
__global__ void __launch_bounds__(512) fft_cols_fwd16_kernel(FftArgs a) {
    using L = Col16<LOGD>;
    constexpr int D = L::D, H = L::H, T = L::T, C = L::C, STRIDE = L::STRIDE;
    extern __shared__ cd smem[];
    rx_poison_smem();
    const int f = blockIdx.y;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const int col0 = blockIdx.x * C;
    const cd *in = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *out = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    cd *s = smem + c * STRIDE;
    {
        cd v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_ASSERT(col0 + c < H);
            v[r] = in[(size_t)(j + r * T) * D + col0 + c];
        }
        dft16<false>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_SMEM(c * STRIDE + pidx(16 * j + r));
            s[pidx(16 * j + r)] = v[r];
        }
    }
    __syncthreads();
    row16_rest<false, LOGD>(s, j, a.twiddle);
    const double sc = a.scale;
    for (int i = threadIdx.x; i < C * D; i += blockDim.x) {
        const int l = i / C, cc = i % C;
        const int k = col0 + cc;
        const int lm = (D - l) & (D - 1);
        const cd v = smem[cc * STRIDE + pidx(l)];
        const bool lo = !a.half_out || l <= H, mlo = !a.half_out || lm <= H;
        if (k == 0) {
            // G = DFT(P), P = X0 + i XH (both real columns): F0 = (G + conj G(-l)) / 2,
            // FH = (G - conj G(-l)) / (2i)
            if (lo) {
                const cd w = smem[cc * STRIDE + pidx(lm)];
                const double hs = 0.5 * sc;
                out[(size_t)l * D] = mk(hs * (v.x + w.x), hs * (v.y - w.y));
                out[(size_t)l * D + H] = mk(hs * (v.y + w.y), hs * (w.x - v.x));
            }
        } else {
            if (lo) out[(size_t)l * D + k] = mk(v.x * sc, v.y * sc);
            if (mlo) out[(size_t)lm * D + (D - k)] = mk(v.x * sc, -v.y * sc);   // F(-K) = conj F(K)
        }
    }
}

template <int LOGD, bool SYM>
__global__ void __launch_bounds__(512) fft_cols_inv16_kernel(FftArgs a) {
    using L = Col16<LOGD>;
    constexpr int D = L::D, H = L::H, T = L::T, C = L::C, STRIDE = L::STRIDE;
    extern __shared__ cd smem[];
    rx_poison_smem();
    const int f = blockIdx.y;
    const int c = threadIdx.x % C, j = threadIdx.x / C;
    const int col0 = blockIdx.x * C;
    const int k = col0 + c;
    const cd *in = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *out = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    cd *s = smem + c * STRIDE;
    {
        cd v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const int l = j + r * T;
            const int lm = (D - l) & (D - 1);
            RX_ASSERT(k < H && l < D);
            if (k == 0) {
                cd t0 = in[(size_t)l * D], th = in[(size_t)l * D + H];
                if (SYM) {
                    const cd m0 = in[(size_t)lm * D], mh = in[(size_t)lm * D + H];
                    t0 = mk(0.5 * (t0.x + m0.x), 0.5 * (t0.y - m0.y));
                    th = mk(0.5 * (th.x + mh.x), 0.5 * (th.y - mh.y));
                }
                v[r] = mk(t0.x - th.y, t0.y + th.x);   // T0 + i TH
            } else {
                cd t = in[(size_t)l * D + k];
                if (SYM) {
                    const cd m = in[(size_t)lm * D + (D - k)];
                    t = mk(0.5 * (t.x + m.x), 0.5 * (t.y - m.y));
                }
                v[r] = t;
            }
        }
        dft16<true>(v);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            RX_SMEM(c * STRIDE + pidx(16 * j + r));
            s[pidx(16 * j + r)] = v[r];
        }
    }
    __syncthreads();
    row16_rest<true, LOGD>(s, j, a.twiddle);
    const double sc = a.scale;
    for (int i = threadIdx.x; i < C * D; i += blockDim.x) {
        const int r = i / C, cc = i % C;
        const cd v = smem[cc * STRIDE + pidx(r)];
        out[(size_t)r * D + col0 + cc] = mk(v.x * sc, v.y * sc);
    }
}

namespace cgx = cooperative_groups;

// cluster-wide barrier: barrier.cluster.arrive (.release) + wait (.acquire) — orders the shared::
// cluster and global-memory accesses of one stage before those of the next across the cluster
__device__ __forceinline__ void cluster_barrier() { cgx::this_cluster().sync(); }

// barrier.cluster split phases: arrive (relaxed: orders nothing) at kernel start, wait before
// the first DSMEM access (every CTA of the cluster has started); and the full barrier with
// release / acquire semantics between stages (orders shared::cluster and global accesses)
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// ----------------------------------------------------------------------------- cluster column passes
// Column passes with N1 x 16-byte row segments on every global load and store (N1 = 8 or 16):
// a cluster of N1 CTAs transforms N1 adjacent half-spectrum columns, four-step with D = N1 N2,
// n = N2 n1 + n2, k = k1 + N1 k2:
//   X[k1 + N1 k2] = sum_{n2} W_{N2}^{n2 k2} [ W_D^{n2 k1} sum_{n1} W_N1^{n1 k1} x[N2 n1 + n2] ].
// Stage 1, CTA c (rank in the cluster): thread (n2, col), n2 in [c N2/N1, (c+1) N2/N1), loads its
// N1 values x[N2 n1 + n2] straight from global memory, DFT-N1 in registers, twiddles W_D^{n2 k1},
// and stores result k1 into the shared memory of CTA k1 of the cluster (distributed shared
// memory, [n2][col]). Stage 2, after a cluster barrier: CTA k1 runs the N2-point Stockham passes
// on its N1 columns and writes rows k1 + N1 k2. The single-CTA column
// kernels above hold whole columns in one CTA, so at 4096^2 a load covers 2 columns = 32 bytes
// of a row (0.32 of HBM, profiles/r02q_aux_c4.md). Output handling (scale, the packed k = 0 pair,
// mirrors, half_out, the inverse's symmetrisation) as in fft_cols_fwd16 / fft_cols_inv16; the
// k = 0 separation reads the mirror row from the CTA that holds it (the one cluster with col0 = 0).
// MODE 0: forward; 1: inverse of a Hermitian spectrum; 2: inverse, symmetrising.
template <int LOGD, int N1, int IPT>
struct ColCl {
    // N1 = cluster size = columns per group (N1 x 16-byte row segments); D = N1 N2; IPT (n2,
    // column) items per thread in stage 1
    static constexpr int D = 1 << LOGD, H = D / 2, N2 = D / N1, LOGN1 = N1 == 16 ? 4 : 3;
    static constexpr int LOGN2 = LOGD - LOGN1;
    static constexpr int T = (N2 / N1) * N1 / IPT;   // threads per CTA
    static constexpr int V = N1 * N2 / T;            // values per thread in the stage-2 passes
    static constexpr size_t SMEM = (size_t)(N1 * N2 + N2) * sizeof(cd);   // [n2][N1 columns] + N2 twiddles
};

template <int N1>
struct ColIx {
    int col;
    __device__ __forceinline__ int operator()(int i) const { return i * N1 + col; }
};

template <int N1, bool INV>
__device__ __forceinline__ void dft_n1(cd *v) {
    if (N1 == 16) dft16<INV>(v);
    else dft8<INV>(v);
}

template <int LOGD, int MODE, int N1, int IPT>
// (IPT = 1: 2 CTAs per SM, <= 64 registers; IPT = 2: half the threads, 3 CTAs per SM)
__global__ void __launch_bounds__(ColCl<LOGD, N1, IPT>::T, IPT == 1 ? 2 : 3) fft_cols_cl_kernel(FftArgs a) {
    using L = ColCl<LOGD, N1, IPT>;
    constexpr int D = L::D, H = L::H, N2 = L::N2, T = L::T;
    constexpr bool INV = MODE != 0;
    extern __shared__ cd smem[];
    cd *buf = smem;                 // [n2][N1]
    cd *tw2 = smem + N1 * N2;       // W_{N2}^j = W_D^{N1 j}
    rx_poison_smem();
    cgx::cluster_group cl = cgx::this_cluster();
    const int c = (int)cl.block_rank();
    const int f = blockIdx.y;
    const int col0 = (int)(blockIdx.x / N1) * N1;
    const int tid = threadIdx.x;
    const cd *in = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *out = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    const double2 *twg = reinterpret_cast<const double2 *>(a.twiddle);
    for (int i = tid; i < N2; i += T) {
        const double2 w = __ldg(twg + N1 * i);
        tw2[i] = mk(w.x, w.y);
    }
    // DSMEM stores may only target CTAs that have started (and, in checked builds, finished
    // poisoning their shared memory): arrive now, wait just before the first remote store
    cluster_arrive_relaxed();
    // ---- stage 1 (all IPT x N1 loads of the thread issued before the first DFT)
    {
        const int col = tid % N1, k = col0 + col;
        cd v[IPT][N1];
#pragma unroll
        for (int it = 0; it < IPT; ++it) {
            const int n2 = c * (N2 / N1) + tid / N1 + it * (T / N1);
            RX_ASSERT(k < H && n2 < N2);
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                const int l = N2 * n1 + n2;
                if (MODE == 0) {
                    v[it][n1] = in[(size_t)l * D + k];
                } else {
                    const int lm = (D - l) & (D - 1);
                    if (k == 0) {
                        cd t0 = in[(size_t)l * D], th = in[(size_t)l * D + H];
                        if (MODE == 2) {
                            const cd m0 = in[(size_t)lm * D], mh = in[(size_t)lm * D + H];
                            t0 = mk(0.5 * (t0.x + m0.x), 0.5 * (t0.y - m0.y));
                            th = mk(0.5 * (th.x + mh.x), 0.5 * (th.y - mh.y));
                        }
                        v[it][n1] = mk(t0.x - th.y, t0.y + th.x);   // T0 + i TH
                    } else {
                        cd t = in[(size_t)l * D + k];
                        if (MODE == 2) {
                            const cd m = in[(size_t)lm * D + (D - k)];
                            t = mk(0.5 * (t.x + m.x), 0.5 * (t.y - m.y));
                        }
                        v[it][n1] = t;
                    }
                }
            }
        }
#pragma unroll
        for (int it = 0; it < IPT; ++it) {
            const int n2 = c * (N2 / N1) + tid / N1 + it * (T / N1);
            dft_n1<N1, INV>(v[it]);
            if (it == 0) cluster_wait();
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) {
                cd y = v[it][k1];
                if (k1 > 0) {
                    const double2 w = __ldg(twg + n2 * k1);   // W_D^{n2 k1}, n2 k1 < D
                    y = INV ? mk(fma(y.x, w.x, y.y * w.y), fma(y.y, w.x, -y.x * w.y))
                            : mk(fma(y.x, w.x, -y.y * w.y), fma(y.y, w.x, y.x * w.y));
                }
                cl.map_shared_rank(buf, k1)[n2 * N1 + col] = y;
            }
        }
    }
    cluster_barrier();
    // ---- stage 2: N2-point transforms of the N1 columns (k1 = c)
    {
        const int col = tid % N1, j = tid / N1;
        fft_in_smem_ix<INV, ColIx<N1>, true, L::V>(buf, ColIx<N1>{col}, N2, L::LOGN2, j, T / N1, tw2, true);
    }
    const double sc = a.scale;
    if (MODE != 0) {
        for (int i = tid; i < N1 * N2; i += T) {
            const int k2 = i / N1, col = i % N1;
            const cd v = buf[i];
            out[(size_t)(c + N1 * k2) * D + col0 + col] = mk(v.x * sc, v.y * sc);
        }
        return;
    }
    const bool zero = col0 == 0;   // uniform over the cluster
    if (zero) cluster_barrier();   // every CTA's stage 2 done: the k = 0 mirror rows are readable
    for (int i = tid; i < N1 * N2; i += T) {
        const int k2 = i / N1, col = i % N1;
        const int l = c + N1 * k2, k = col0 + col;
        const int lm = (D - l) & (D - 1);
        const cd v = buf[i];
        const bool lo = !a.half_out || l <= H, mlo = !a.half_out || lm <= H;
        if (k == 0) {
            // G = DFT(P), P = X0 + i XH (both real columns): F0 = (G + conj G(-l)) / 2,
            // FH = (G - conj G(-l)) / (2i); G(-l) is row lm = (lm mod N1) + N1 (lm / N1)
            if (lo) {
                const cd w = cl.map_shared_rank(buf, lm % N1)[(lm / N1) * N1];
                const double hs = 0.5 * sc;
                out[(size_t)l * D] = mk(hs * (v.x + w.x), hs * (v.y - w.y));
                out[(size_t)l * D + H] = mk(hs * (v.y + w.y), hs * (w.x - v.x));
            }
        } else {
            if (lo) out[(size_t)l * D + k] = mk(v.x * sc, v.y * sc);
            if (mlo) out[(size_t)lm * D + (D - k)] = mk(v.x * sc, -v.y * sc);   // F(-K) = conj F(K)
        }
    }
    if (zero) cluster_barrier();   // no CTA leaves while another reads its shared memory
}

// Forward columns: half spectra -> full spectrum (scaled). Block = C adjacent slots of one
// field; slot 0 is the packed (X[.][0], X[.][N/2]) pair of real columns.
__global__ void __launch_bounds__(1024) fft_cols_fwd_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, C = a.per_block;
    const int logC = __ffs(C) - 1;
    const int tf = D >= 8 ? D / 8 : 1;
    const int stride = col_stride(D, C);
    const int col0 = blockIdx.x * C;
    const cd *in = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *out = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    const int n = C << log2D;
    rx_poison_smem();
    cd tmp[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            RX_ASSERT(col0 + (i & (C - 1)) < (D >> 1) && (i >> logC) < D);
            tmp[q] = in[(size_t)(i >> logC) * D + col0 + (i & (C - 1))];
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            RX_SMEM((i & (C - 1)) * stride + pidx(i >> logC));
            smem[(i & (C - 1)) * stride + pidx(i >> logC)] = tmp[q];
        }
    }
    __syncthreads();
    const int col = threadIdx.x / tf, t = threadIdx.x - col * tf;
    fft_in_smem<false>(smem + col * stride, D, log2D, t, tf, a.twiddle);
    const double sc = a.scale;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int l = i >> logC, c = i & (C - 1);
        const int k = col0 + c;
        const int lm = (D - l) & (D - 1);
        RX_ASSERT(l < D && k < (D >> 1));
        const cd v = smem[c * stride + pidx(l)];
        const bool lo = !a.half_out || l <= (D >> 1), mlo = !a.half_out || lm <= (D >> 1);
        if (k == 0) {
            // G = DFT(P), P = X0 + i XH (both real columns): F0 = (G + conj G(-l)) / 2,
            // FH = (G - conj G(-l)) / (2i)
            if (lo) {
                const cd w = smem[c * stride + pidx(lm)];
                const double hs = 0.5 * sc;
                out[(size_t)l * D] = mk(hs * (v.x + w.x), hs * (v.y - w.y));
                out[(size_t)l * D + (D >> 1)] = mk(hs * (v.y + w.y), hs * (w.x - v.x));
            }
        } else {
            if (lo) out[(size_t)l * D + k] = mk(v.x * sc, v.y * sc);
            if (mlo) out[(size_t)lm * D + (D - k)] = mk(v.x * sc, -v.y * sc);   // F(-K) = conj F(K)
        }
    }
}

// Inverse columns: spectrum -> half-spectrum rows of Re(IDFT). SYM: symmetrise on load,
// T(K) = (S(K) + conj S(-K)) / 2, so Re(IDFT S) = IDFT T for any complex S; without SYM the
// input must already be Hermitian (the R2C finish writes the Hermitian part). Slot 0 carries
// the two self-mirror columns k = 0 and k = N/2 packed: IDFT(T0 + i TH) = x0 + i xH.
template <bool SYM>
__global__ void __launch_bounds__(1024) fft_cols_inv_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, C = a.per_block;
    const int logC = __ffs(C) - 1;
    const int tf = D >= 8 ? D / 8 : 1;
    const int stride = col_stride(D, C);
    const int col0 = blockIdx.x * C;
    const cd *in = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    cd *out = static_cast<cd *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    const int n = C << log2D;
    const int H = D >> 1;
    rx_poison_smem();
    cd tmp[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            const int l = i >> logC, k = col0 + (i & (C - 1));
            const int lm = (D - l) & (D - 1);
            RX_ASSERT(l < D && k < H);
            if (k == 0) {
                cd t0 = in[(size_t)l * D], th = in[(size_t)l * D + H];
                if (SYM) {
                    const cd m0 = in[(size_t)lm * D], mh = in[(size_t)lm * D + H];
                    t0 = mk(0.5 * (t0.x + m0.x), 0.5 * (t0.y - m0.y));
                    th = mk(0.5 * (th.x + mh.x), 0.5 * (th.y - mh.y));
                }
                tmp[q] = mk(t0.x - th.y, t0.y + th.x);   // T0 + i TH
            } else {
                cd t = in[(size_t)l * D + k];
                if (SYM) {
                    const cd m = in[(size_t)lm * D + (D - k)];
                    t = mk(0.5 * (t.x + m.x), 0.5 * (t.y - m.y));
                }
                tmp[q] = t;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            RX_SMEM((i & (C - 1)) * stride + pidx(i >> logC));
            smem[(i & (C - 1)) * stride + pidx(i >> logC)] = tmp[q];
        }
    }
    __syncthreads();
    const int col = threadIdx.x / tf, t = threadIdx.x - col * tf;
    fft_in_smem<true>(smem + col * stride, D, log2D, t, tf, a.twiddle);
    const double sc = a.scale;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            const int r = i >> logC, c = i & (C - 1);
            const cd v = smem[c * stride + pidx(r)];
            out[(size_t)r * D + col0 + c] = mk(v.x * sc, v.y * sc);
        }
    }
}

// Inverse rows: half-spectrum rows -> real fields, two rows per complex transform:
// Z[k] = g1[k] + i g2[k] over the full circle (g[N-k] = conj g[k]), IDFT(Z) = x1 + i x2.
__global__ void __launch_bounds__(1024) fft_rows_inv_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, nb = a.per_block;
    const int tf = D >= 8 ? D / 8 : 1;
    const int H = D >> 1;
    const size_t pair0 = (size_t)blockIdx.x * nb;
    const cd *inp = static_cast<const cd *>(f == 0 ? a.in[0] : f == 1 ? a.in[1] : a.in[2]);
    double *outp = static_cast<double *>(f == 0 ? a.out[0] : f == 1 ? a.out[1] : a.out[2]);
    const int PL = padded_len(D);
    rx_poison_smem();
    const int m = nb * H;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int pr = i / H, k = i - pr * H;
        const size_t g = (2 * (pair0 + pr)) * D + k;
        RX_ASSERT(g + D < (size_t)D * D);
        RX_SMEM(pr * PL + pidx(D - 1));
        const cd g1 = inp[g], g2 = inp[g + D];
        cd *Z = smem + pr * PL;
        if (k == 0) {
            Z[pidx(0)] = mk(g1.x, g2.x);
            Z[pidx(H)] = mk(g1.y, g2.y);
        } else {
            Z[pidx(k)] = mk(g1.x - g2.y, g1.y + g2.x);        // g1 + i g2
            Z[pidx(D - k)] = mk(g1.x + g2.y, g2.x - g1.y);    // conj g1 + i conj g2
        }
    }
    __syncthreads();
    const int row = threadIdx.x / tf, t = threadIdx.x - row * tf;
    fft_in_smem<true>(smem + row * PL, D, log2D, t, tf, a.twiddle);
    const double sc = a.scale;
    const int n = nb * D;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int i = threadIdx.x + q * blockDim.x;
        if (i < n) {
            const int pr = i >> log2D, x = i & (D - 1);
            const cd v = smem[pr * PL + pidx(x)];
            const size_t g = (2 * (pair0 + pr)) * D + x;
            RX_ASSERT(g + D < (size_t)D * D);
            outp[g] = v.x * sc;
            outp[g + D] = v.y * sc;
        }
    }
}

// ============================================================================= pole kernel
// Per mode (k, l): Kx = 2 pi k tau, Ky = 2 pi l tau (Nyquist zeroed), K2 = Kx^2 + Ky^2,
// c = tau. Input f0 = (e0, a, b) = (eta0^, u0^, v0^).
//   delta0 = i(Kx a + Ky b), zeta0 = i(Kx b - Ky a)        (tau-scaled)
//   m0 = zeta0 - c e0,  B0 = h mu e0 + delta0              (per mode, pole-independent)
// Solve 1, (alpha I + tau A) g1 = f0 — Helmholtz reduction (eq:lswEta):
//   eta1 (kappa + K2) = kappa/alpha e0 + delta0 - c/alpha zeta0 = alpha e0 + delta0 - (c/alpha) m0
//                     = B0 + i h n e0 - (c/alpha) m0          (alpha = h mu + i h n)
//   q = 1/(kappa + K2) = (dr - i ki)/(dr^2 + ki^2), dr = Re(kappa) + K2, ki = Im(kappa)
// Solve 2, (conj(alpha) I - tau A) g2 = g1: same with (alpha, Kx, Ky, c) -> (conj alpha, -Kx,
//   -Ky, -c); its denominator is conj(kappa + K2): eta2 = num2 * conj(q) (one reciprocal).
// DZ variant (default): back-substitution in (delta, zeta) = divergence/vorticity of g:
//   delta1 = alpha eta1 - e0,  zeta1 = m0/alpha + c eta1
//   num2 = conj(kappa/alpha) eta1 - delta1 - (c/conj(alpha)) zeta1,  eta2 = num2 conj(q)
//   delta2 = eta1 - conj(alpha) eta2,  zeta2 = (zeta1 - c delta2)/conj(alpha) = |1/alpha|^2 m0 + c eta2
//   acc(eta, delta, zeta) += w1 g1 + w2 g2;  (u, v) recovered per mode in finish_kernel.
// UV variant (paper-literal eq:lswVelocities): (u1,v1) = kappa^-1 [[alpha,-c],[c,alpha]] (p,q),
//   p = a + i Kx eta1, q = b + i Ky eta1; delta1, zeta1 from (u1, v1); likewise for g2.
// fp64-pipe instructions per (pole, mode): DZ 71, UV 101 (launch.h).
constexpr int kPoleBlock = 128;
#ifndef REXI_POLE_TILE
#define REXI_POLE_TILE 32
#endif
constexpr int kPoleTile = REXI_POLE_TILE;
// the R2C kernels run 2 blocks per SM, so they can afford a 4x larger pole tile in shared
// memory (36 KB): fewer block barriers per pole (measured ~1 % faster than 32)
constexpr int kR2CTile = 128;

struct ModeState {
    cd e0, B0, m0, ua, vb;   // f0 = (e0, ua, vb); B0 = h mu e0 + delta0; m0 = zeta0 - c e0
    cd Bt0;                  // h mu e0 - delta0 (PF kind)
    double K2, Kx, Ky;
    cd A0, A1, A2;           // accumulators: (eta, delta, zeta) [DZ] or (eta, u, v) [UV]
};

template <int VARIANT>
__device__ __forceinline__ void pole_solves_in(const PoleConst &P, ModeState &s, const cd e0in,
                                               const cd B0in, const cd m0in, const cd qd,
                                               const double c);

// 1/(kappa_n + K2) for one pole and one value of K2 (shared by every mode with that K2).
template <class PC>
__device__ __forceinline__ cd pole_den(const PC &P, const double K2) {
    const double dr = P.kr + K2;
    const double r = rcp_pos(fma(dr, dr, P.ki2));
    return mk(dr * r, -P.ki * r);
}

// One pole, one mode, given q = 1/(kappa + K2): both shifted solves and the weighted
// accumulation.
template <int VARIANT>
__device__ __forceinline__ void pole_solves(const PoleConst &P, ModeState &s, const cd qd,
                                            const double c) {
    pole_solves_in<VARIANT>(P, s, s.e0, s.B0, s.m0, qd, c);
}

template <int VARIANT>
__device__ __forceinline__ void pole_solves_in(const PoleConst &P, ModeState &s, const cd e0in,
                                               const cd B0in, const cd m0in, const cd qd,
                                               const double c) {
    const cd al = mk(P.ar, P.ai), s2 = mk(P.s2r, P.s2i), s1c = mk(P.s1cr, P.s1ci);
    const cd w1 = mk(P.w1r, P.w1i), w2 = mk(P.w2r, P.w2i);
    const double hn = P.ai;
    // ---- solve 1: Helmholtz for eta1 (eq:lswEta)
    const cd t = mk(fma(-hn, e0in.y, B0in.x), fma(hn, e0in.x, B0in.y));
    const cd num = cfms(s2, m0in, t);
    const cd eta1 = cmul(num, qd);
    if (VARIANT == 5) {
        // PFH: as PF, with the delta back-substitution folded into the weights:
        //   W1 delta1 + W2 delta_t = (W1 alpha) eta1 - (W2 conj(alpha)) eta_t - w1 e0,
        // the -w1 e0 term summed over the pole range in finish_kernel.
        const cd tt = mk(fma(hn, e0in.y, s.Bt0.x), fma(-hn, e0in.x, s.Bt0.y));   // Bt0 - i hn e0
        const cd numt = cjfms(s2, m0in, tt);
        const cd etat = cjfma(qd, numt, mk(0, 0));
        const cd W1 = mk(P.W1r, P.W1i), W2 = mk(P.W2r, P.W2i);
        const cd P1 = mk(P.P1r, P.P1i), P2 = mk(P.P2r, P.P2i);
        s.A0 = cfma(W2, etat, cfma(W1, eta1, s.A0));
        s.A1 = cfma(P2, etat, cfma(P1, eta1, s.A1));
    } else if (VARIANT == 4) {
        // Partial fractions (SURVEY.md 8(d) "allowed algebraic equivalents"):
        //   (conj(alpha) - B)^{-1} (alpha + B)^{-1} = [(alpha + B)^{-1} + (conj(alpha) - B)^{-1}] / (2 h mu)
        // so w1 g1 + w2 g2 = W1 g1 + W2 gt with gt = (conj(alpha) I - tau A)^{-1} f0: two independent
        // Helmholtz solves of the same right-hand side. For gt (same reduction, alpha -> conj(alpha),
        // B -> -B): eta_t (conj(kappa) + K2) = conj(alpha) e0 - delta0 - (c/conj(alpha)) m0,
        // delta_t = e0 - conj(alpha) eta_t; zeta rebuilt from eta in finish_kernel (as kind 0).
        const cd tt = mk(fma(hn, e0in.y, s.Bt0.x), fma(-hn, e0in.x, s.Bt0.y));   // Bt0 - i hn e0
        const cd numt = cjfms(s2, m0in, tt);                                      // - conj(c/alpha) m0
        const cd etat = cjfma(qd, numt, mk(0, 0));                                // conj(q) numt
        const cd del1 = cfma(al, eta1, mk(-e0in.x, -e0in.y));
        const cd delt = cjfms(al, etat, e0in);                                    // e0 - conj(alpha) eta_t
        const cd W1 = mk(P.W1r, P.W1i), W2 = mk(P.W2r, P.W2i);
        s.A0 = cfma(W2, etat, cfma(W1, eta1, s.A0));
        s.A1 = cfma(W2, delt, cfma(W1, del1, s.A1));
    } else if (VARIANT == 2) {
        // original REXI (eq:originalREXImatrix): one solve per term, acc += Gamma beta^Re g1.
        // zeta1 = m0/alpha + c eta1 is affine in eta1 (potential vorticity, see finish_kernel):
        // its pole sum is rebuilt there, so only (eta, delta) are accumulated.
        const cd del1 = cfma(al, eta1, mk(-e0in.x, -e0in.y));
        s.A0 = cfma(w1, eta1, s.A0);
        s.A1 = cfma(w1, del1, s.A1);
    } else if (VARIANT == 0 || VARIANT == 3) {
        const cd ia = mk(P.iar, P.iai);
        const cd del1 = cfma(al, eta1, mk(-e0in.x, -e0in.y));
        const cd zet1 = cfma(ia, m0in, mk(c * eta1.x, c * eta1.y));
        // ---- solve 2
        cd num2 = cfma(s1c, eta1, mk(-del1.x, -del1.y));
        num2 = cjfms(s2, zet1, num2);                            // - conj(c/alpha) zeta1
        const cd eta2 = cjfma(qd, num2, mk(0, 0));               // num2 * conj(q)
        const cd del2 = cjfms(al, eta2, eta1);                   // eta1 - conj(alpha) eta2
        // ---- accumulate w1 g1 + w2 g2
        s.A0 = cfma(w2, eta2, cfma(w1, eta1, s.A0));
        s.A1 = cfma(w2, del2, cfma(w1, del1, s.A1));
        if (VARIANT == 3) {
            // zeta2 = (zeta1 - c delta2)/conj(alpha) = |1/alpha|^2 m0 + c eta2; DZ (kind 0)
            // rebuilds the zeta pole sum from the eta pole sum instead (finish_kernel)
            const cd zet2 = mk(fma(P.ia2, m0in.x, c * eta2.x), fma(P.ia2, m0in.y, c * eta2.y));
            s.A2 = cfma(w2, zet2, cfma(w1, zet1, s.A2));
        }
    } else {
        const cd s3 = mk(P.s3r, P.s3i), s4 = mk(P.s4r, P.s4i);
        const double kx = s.Kx, ky = s.Ky;
        // eq:lswVelocities: (u1, v1) = (s3 p - s4 q, s4 p + s3 q)
        const cd p = mk(fma(-kx, eta1.y, s.ua.x), fma(kx, eta1.x, s.ua.y));
        const cd qq = mk(fma(-ky, eta1.y, s.vb.x), fma(ky, eta1.x, s.vb.y));
        const cd u1 = cfms(s4, qq, cmul(s3, p));
        const cd v1 = cfma(s3, qq, cmul(s4, p));
        // delta1 = i(kx u1 + ky v1), zeta1 = i(kx v1 - ky u1)
        const cd sd = mk(fma(kx, u1.x, ky * v1.x), fma(kx, u1.y, ky * v1.y));
        const cd sz = mk(fma(kx, v1.x, -ky * u1.x), fma(kx, v1.y, -ky * u1.y));
        const cd del1 = mk(-sd.y, sd.x), zet1 = mk(-sz.y, sz.x);
        // ---- solve 2
        cd num2 = cfma(s1c, eta1, mk(-del1.x, -del1.y));
        num2 = cjfms(s2, zet1, num2);
        const cd eta2 = cjfma(qd, num2, mk(0, 0));
        // p' = u1 - i kx eta2, q' = v1 - i ky eta2
        const cd p2 = mk(fma(kx, eta2.y, u1.x), fma(-kx, eta2.x, u1.y));
        const cd q2 = mk(fma(ky, eta2.y, v1.x), fma(-ky, eta2.x, v1.y));
        // (u2, v2) = (conj(s3) p' + conj(s4) q', -conj(s4) p' + conj(s3) q')
        const cd u2 = cjfma(s4, q2, cjfma(s3, p2, mk(0, 0)));
        const cd v2 = cjfms(s4, p2, cjfma(s3, q2, mk(0, 0)));
        s.A0 = cfma(w2, eta2, cfma(w1, eta1, s.A0));
        s.A1 = cfma(w2, u2, cfma(w1, u1, s.A1));
        s.A2 = cfma(w2, v2, cfma(w1, v1, s.A2));
    }
}

// Modes of "K2 quad" q of a D x D grid (D/2 x D/2 quads, q = a * D/2 + b): four modes with the
// same K2 = Kx^2 + Ky^2 (exactly, the symbols being odd in k and zero at 0 and Nyquist):
//   a, b > 0:  (a, b) (a, D-b) (D-a, b) (D-a, D-b)          [row l, column k]
//   a = 0 < b: (0, b) (0, D-b) (b, 0) (D-b, 0)              [axes]
//   b = 0 < a: (H, a) (H, D-a) (a, H) (D-a, H), H = D/2     [Nyquist lines]
//   a = b = 0: (0, 0) (0, H) (H, 0) (H, H)                  [K2 = 0]
// The quads partition all D^2 modes.
__device__ __forceinline__ void quad_modes(long q, int D, int log2D, long m[4]) {
    const int H = D >> 1;
    const int a = (int)(q >> (log2D - 1)), b = (int)(q & (H - 1));
    int l[4], k[4];
    if (a > 0 && b > 0) {
        l[0] = a; k[0] = b; l[1] = a; k[1] = D - b; l[2] = D - a; k[2] = b; l[3] = D - a; k[3] = D - b;
    } else if (b > 0) {
        l[0] = 0; k[0] = b; l[1] = 0; k[1] = D - b; l[2] = b; k[2] = 0; l[3] = D - b; k[3] = 0;
    } else if (a > 0) {
        l[0] = H; k[0] = a; l[1] = H; k[1] = D - a; l[2] = a; k[2] = H; l[3] = D - a; k[3] = H;
    } else {
        l[0] = 0; k[0] = 0; l[1] = 0; k[1] = H; l[2] = H; k[2] = 0; l[3] = H; k[3] = H;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) m[j] = ((long)l[j] << log2D) + k[j];
}

// ----------------------------------------------------------------------------- R2C pairs
// Real physical input => Hermitian spectrum, f0(-K) = conj(f0(K)) (symbols odd in K, G2). For
// the pair {K, -K} with representative K (the smaller linear index) and the PFH weights, the
// solves at -K follow from those at K (B0 = Bt0 + 2 d0, d0 = delta0):
//   eta1(-K)  = conj(eta_t(K) + conj(q) 2 d0),   eta_t(-K) = conj(eta1(K) - q 2 d0),
// so the Hermitian part that survives the final Re(IDFT(.)),
//   H(A)(K) = (A(K) + conj(A(-K))) / 2 = [Re sum_{n=-N}^{N} over the pair, "R2C" of SURVEY 8(d)],
// is accumulated directly per pole:
//   H_eta   += X1 eta1 + X2 eta_t + (conj(W1 q) - conj(W2) q) d0
//   H_delta' += Y1 eta1 + Y2 eta_t + (conj(P1 q) - conj(P2) q) d0
// (X, Y: half-weights from the planner; X2 = conj X1, Y2 = conj Y1). With eta1 = q num1 and
// eta_t = conj(q) num_t (the two Helmholtz solves, num = their right-hand sides) this is
//   H_eta += Re(X1 q) (num1 + num_t) + i Im(X1 q) (num1 - num_t) + sigma d0,
//   num1 + num_t = 2 h mu eta0 - 2 Re(c/alpha) m0,  num1 - num_t = 2 d0 + i (2 h n eta0 - 2 Im(c/alpha) m0),
// which r2c_tile evaluates for every pole and pair; the d0 coefficients
// sigma, tau' depend on the pole and K2 only and are summed per K2 value, applied after the
// pole loop. A thread owns one quad (mpt 4) or one octet item (mpt 8, two quads sharing K2);
// the corner quad (four self-mirror K = 0 modes) is left to fixup_k0_kernel.
struct PairState {
    cd e0, E2, D2, m0;       // data of the representative mode: eta0, 2 h mu eta0, 2 delta0, m0
    cd H0, H1;               // Hermitian accumulators: eta, delta' (before the e0 term)
};

// Per-pair state from the mode's spectrum (e = eta0^, d = delta0, z = zeta0).
__device__ __forceinline__ void pair_setup(PairState &s, cd e, cd d, cd z, double hmu, double c) {
    s.e0 = e;
    s.E2 = mk(2.0 * hmu * e.x, 2.0 * hmu * e.y);
    s.D2 = mk(2.0 * d.x, 2.0 * d.y);
    s.m0 = mk(fma(-c, e.x, z.x), fma(-c, e.y, z.y));
    s.H0 = mk(0, 0);
    s.H1 = mk(0, 0);
}

// Work items of the R2C kernel (four pairs = eight modes per thread):
//  * OCT: "octets" — the interior quads (a, b) and (b, a), 1 <= a < b < H, share K2 (square
//    grid, the same symbol in x and y), so one denominator and one (sigma, tau') sum per pole
//    serve eight modes; items n_oct.. hold one of the remaining 3 (H - 1) quads each (diagonal
//    a = b, axes, Nyquist lines), computed as a half-discarded octet.
//  * !OCT: NQ quads per thread in linear quad order.
// Quad 0 (the four K = 0 corners) is left to the fix-up kernel.
__host__ __device__ constexpr long r2c_n_oct(int D) {
    const long H = D >> 1;
    return H >= 3 ? (H - 1) * (H - 2) / 2 : 0;
}
__host__ __device__ constexpr long r2c_items(int D, int nq, bool oct) {
    const long H = D >> 1;
    if (oct) return r2c_n_oct(D) + 3 * (H - 1);
    return ((long)D * D / 4 + nq - 1) / nq;
}
// the s-th of the 3 (H - 1) non-octet quads (s < 3 (H - 1)) as a quad index a * H + b
__device__ __forceinline__ long r2c_single_quad(long s, int H) {
    long qa, qb;
    if (s < H - 1) { qa = s + 1; qb = s + 1; }
    else if (s < 2 * (H - 1)) { qa = 0; qb = s - (H - 1) + 1; }
    else { qa = s - 2 * (H - 1) + 1; qb = 0; }
    return qa * H + qb;
}

// Octet work item -> its two quads (quad index a * H + b), validity, shared K2.
__device__ __forceinline__ void r2c_octet_item(long item, int D, long quad[2], bool ok[2], bool &shared_k2) {
    const int H = D >> 1;
    const long n_oct = r2c_n_oct(D);
    if (item < n_oct) {
        // triangular decode: item = b'(b'-1)/2 + a', 0 <= a' < b' <= H - 2; (a, b) = (a'+1, b'+1)
        long bp = (long)((1.0 + sqrt(1.0 + 8.0 * (double)item)) * 0.5);
        while (bp * (bp - 1) / 2 > item) --bp;
        while ((bp + 1) * bp / 2 <= item) ++bp;
        const long ap = item - bp * (bp - 1) / 2;
        quad[0] = (ap + 1) * H + (bp + 1);
        quad[1] = (bp + 1) * H + (ap + 1);
        ok[0] = ok[1] = true;
        shared_k2 = true;
    } else {
        // one of the other 3 (H - 1) quads, as an octet whose second quad is a discarded copy
        // of the first: every item then costs the same (one denominator, four pairs per pole),
        // which keeps warps convergent and the stream-K split balanced (1.2 % extra work)
        const long sidx = item - n_oct;
        ok[0] = sidx < 3L * (H - 1);
        ok[1] = false;
        quad[0] = quad[1] = ok[0] ? r2c_single_quad(sidx, H) : 1;
        shared_k2 = true;
    }
}

// Representative mode of pair j (0, 1) of a quad: interior quads pair modes (0,3) and (1,2) of
// quad_modes, axis / Nyquist quads (0,1) and (2,3); the representative is the smaller index.
__device__ __forceinline__ long r2c_rep(long quad, int j, int D, int log2D) {
    long mq[4];
    quad_modes(quad, D, log2D, mq);
    const int H = D >> 1;
    const int qa = (int)(quad >> (log2D - 1)), qb = (int)(quad & (H - 1));
    return j == 0 ? mq[0] : ((qa > 0 && qb > 0) ? mq[1] : mq[2]);
}

// Stream-K partition of the (tile, pole) iteration space over the persistent CTAs: CTA i owns
// [W i / P, W (i + 1) / P), W = tiles x poles; sk_cta_of(x) is the CTA owning iteration x.
__host__ __device__ __forceinline__ long sk_cta_of(long x, long W, long P) {
    long i = (long)((double)x * (double)P / (double)W);
    if (i >= P) i = P - 1;
    if (i < 0) i = 0;
    while (i + 1 < P && W * (i + 1) / P <= x) ++i;
    while (i > 0 && W * i / P > x) --i;
    return i;
}

// One tile of poles for the thread's four pairs. SHARED: both quads have the same K2 (octet).
// Pole sums of the delta0 weights sigma = sum conj(W1 q) - conj(W2) q and tau' (P1, P2), as
// four real FMAs per pole each from the planner's real coefficients (planner.h).
// The sum/difference evaluation below also sends the delta0 part of (num1 - num_t) = 2 delta0 +
// i w to these sums: i Im(X1 q) 2 delta0 is a delta0 term with a pole-and-K2 coefficient; the
// planner folds its 2 Im(X1 q) (and 2 Im(Y1 q) for tau') into the coefficients (planner.h).
struct DSums {
    cd sg, ta;
    __device__ __forceinline__ cd sigma() const { return sg; }
    __device__ __forceinline__ cd tau() const { return ta; }
};
__device__ __forceinline__ DSums dsums_zero() { return DSums{mk(0, 0), mk(0, 0)}; }

template <int PU, int NQ, bool SHARED>
__device__ __forceinline__ void r2c_tile(const R2CPole *sp, int cnt, const double (&K2)[NQ],
                                         PairState (&st)[2 * NQ], DSums (&ds)[NQ]) {
    constexpr int NG = SHARED ? 1 : NQ;
#pragma unroll PU
    for (int qq = 0; qq < cnt; ++qq) {
        const R2CPole &P = sp[qq];
        const cd X1 = mk(P.X1r, P.X1i), Y1 = mk(P.Y1r, P.Y1i);
        // the solve's division by the Helmholtz symbol, eta1 = q num1 and eta_t = conj(q) num_t,
        // fused with the accumulation weights: X1 eta1 = (X1 q) num1, X2 eta_t = conj(X1 q) num_t
        // (X2 = conj(X1), Y2 = conj(Y1) by construction, planner.cpp), per pole and K2
        cd Aq[NG], Cq[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const cd q = pole_den(P, K2[g]);
            ds[g].sg = mk(fma(P.sgx1, q.x, fma(P.sgx2, q.y, ds[g].sg.x)), fma(P.sgy1, q.x, fma(P.sgy2, q.y, ds[g].sg.y)));
            ds[g].ta = mk(fma(P.tax1, q.x, fma(P.tax2, q.y, ds[g].ta.x)), fma(P.tay1, q.x, fma(P.tay2, q.y, ds[g].ta.y)));
            Aq[g] = cmul(X1, q);
            Cq[g] = cmul(Y1, q);
        }
        // The two Helmholtz right-hand sides of the pair, num1 = B0 + i hn eta0 - (c/alpha) m0
        // and num_t = Bt0 - i hn eta0 - conj(c/alpha) m0 (B0, Bt0 = h mu eta0 +- delta0), carry
        // conjugate weights (X1 q and its conjugate), so X1 q num1 + conj(X1 q) num_t
        // = Re(X1 q) (num1 + num_t) + i Im(X1 q) (num1 - num_t), with
        //   num1 + num_t = 2 h mu eta0 - 2 Re(c/alpha) m0,
        //   num1 - num_t = 2 delta0 + i (2 h n eta0 - 2 Im(c/alpha) m0)
        // (every pair still forms its right-hand sides for every pole, in this sum/difference basis)
        const double r2 = P.sr2, k2 = P.si2, g2 = P.hn2;
#pragma unroll
        for (int j = 0; j < 2 * NQ; ++j) {
            const int g = SHARED ? 0 : j >> 1;
            PairState &s = st[j];
            const cd S = mk(fma(-r2, s.m0.x, s.E2.x), fma(-r2, s.m0.y, s.E2.y));       // num1 + num_t
            const cd w = mk(fma(-k2, s.m0.x, g2 * s.e0.x), fma(-k2, s.m0.y, g2 * s.e0.y));
            // num1 - num_t = 2 delta0 + i w: i Im(A) (2 delta0 + i w) = i Im(A) 2 delta0 - Im(A) w,
            // the delta0 part going to the sums (DSums)
            s.H0 = mk(fma(Aq[g].x, S.x, fma(-Aq[g].y, w.x, s.H0.x)), fma(Aq[g].x, S.y, fma(-Aq[g].y, w.y, s.H0.y)));
            s.H1 = mk(fma(Cq[g].x, S.x, fma(-Cq[g].y, w.x, s.H1.x)), fma(Cq[g].x, S.y, fma(-Cq[g].y, w.y, s.H1.y)));
        }
    }
}

template <int PU, int MINB, int NQ, bool OCT>
__global__ void __launch_bounds__(kPoleBlock, MINB) pole_kernel_r2c(PoleArgs a) {
    __shared__ R2CPole sp[kR2CTile];
    const long n_modes = a.n_modes;
    const int chunk = blockIdx.y;
    const long len = a.pole_end - a.pole_begin;
    const long p0 = a.pole_begin + len * chunk / a.n_chunks;
    const long p1 = a.pole_begin + len * (chunk + 1) / a.n_chunks;
    const double c = a.tau;
    const double hmu = a.hmu;
    const int H = a.D >> 1;
    const long item = (long)blockIdx.x * kPoleBlock + threadIdx.x;
    long quad[NQ];
    bool ok[NQ];
    bool shared_k2 = false;
    if constexpr (OCT) {
        static_assert(!OCT || NQ == 2, "octet items hold two quads");
        r2c_octet_item(item, a.D, quad, ok, shared_k2);
    } else {
#pragma unroll
        for (int g = 0; g < NQ; ++g) {
            const long q = (long)blockIdx.x * (kPoleBlock * NQ) + g * kPoleBlock + threadIdx.x;
            ok[g] = q > 0 && q < (n_modes >> 2);
            quad[g] = ok[g] ? q : 1;
        }
    }
    long rep[2 * NQ];
    double K2[NQ];
    PairState st[2 * NQ];
#pragma unroll
    for (int g = 0; g < NQ; ++g) {
        const long qs = quad[g];
        long mq[4];
        quad_modes(qs, a.D, a.log2D, mq);
        // representatives: interior quads pair (0,3) and (1,2); axis / Nyquist quads (0,1), (2,3)
        const int qa = (int)(qs >> (a.log2D - 1)), qb = (int)(qs & (H - 1));
        rep[2 * g] = mq[0];
        rep[2 * g + 1] = (qa > 0 && qb > 0) ? mq[1] : mq[2];
        K2[g] = 0.0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const long mm = rep[2 * g + j];
            const int l = (int)(mm >> a.log2D), k = (int)(mm & (a.D - 1));
            const double kx = __ldg(&a.ksym[k]), ky = __ldg(&a.ksym[l]);
            const cd e = a.fhat[mm], uu = a.fhat[n_modes + mm], vv = a.fhat[2 * n_modes + mm];
            const cd d = mk(-fma(kx, uu.y, ky * vv.y), fma(kx, uu.x, ky * vv.x));
            const cd z = mk(-fma(kx, vv.y, -ky * uu.y), fma(kx, vv.x, -ky * uu.x));
            pair_setup(st[2 * g + j], e, d, z, hmu, c);
            K2[g] = fma(kx, kx, ky * ky);
        }
    }
    // the d0 terms of H_eta and H_delta' have pole-sum coefficients that depend on K2 only
    // (sigma, tau'): summed once per K2, applied to d0 after the pole loop
    DSums ds[NQ];
#pragma unroll
    for (int g = 0; g < NQ; ++g) ds[g] = dsums_zero();

    for (long pt = p0; pt < p1; pt += kR2CTile) {
        const int cnt = (int)min((long)kR2CTile, p1 - pt);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(a.rpoles + pt);
            double2 *dst = reinterpret_cast<double2 *>(sp);
            constexpr int kPer = (int)(sizeof(R2CPole) / sizeof(double2));
            for (int i = threadIdx.x; i < cnt * kPer; i += kPoleBlock) dst[i] = src[i];
        }
        __syncthreads();
        // octet items always share K2 (single quads run as half-discarded octets)
        if constexpr (OCT) r2c_tile<PU, NQ, true>(sp, cnt, K2, st, ds);
        else r2c_tile<PU, NQ, false>(sp, cnt, K2, st, ds);
    }
    if (OCT) {
#pragma unroll
        for (int g = 1; g < NQ; ++g) {
            ds[g] = ds[0];
        }
    }
    cd *out = a.partial + (size_t)chunk * 3 * n_modes;
#pragma unroll
    for (int g = 0; g < NQ; ++g) {
        if (ok[g]) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const PairState &s = st[2 * g + j];
                const cd d0 = mk(0.5 * s.D2.x, 0.5 * s.D2.y);
                out[rep[2 * g + j]] = cfma(ds[g].sigma(), d0, s.H0);
                out[n_modes + rep[2 * g + j]] = cfma(ds[g].tau(), d0, s.H1);
            }
        }
    }
}

// Stream-K R2C pole kernel (octet items): a persistent grid of P CTAs splits the W = tiles x
// poles iteration space evenly (every CTA runs the same number of pole iterations, so no wave
// tail); a CTA walks its range tile segment by tile segment and writes one partial per segment
// to slot (tile, segment): partial[((tile * slots + s) * 8 + 2 pair + {0: H_eta, 1: H_delta'})
// * 128 + tid]. finish_r2c_sk_kernel sums the segments of each tile in a fixed order.
// One 256-thread CTA per SM (8 warps, 2 per scheduler): two independent 128-thread CTAs on one
// SM do not share the fp64 pipe evenly (the older one is favoured), so with a static split the
// younger one would finish alone at half the issue rate; warps of one CTA stay within a pole
// tile of each other (block barrier per tile).
constexpr int kSkBlock = 256;

template <int PU>
__global__ void __launch_bounds__(kSkBlock, 1) pole_kernel_r2c_sk(PoleArgs a) {
    __shared__ R2CPole sp[kR2CTile];
    const long n_modes = a.n_modes;
    const long Nr = a.pole_end - a.pole_begin;
    const long T = a.sk_tiles, P = gridDim.x;
    const long W = T * Nr;
    const long g1 = W * (blockIdx.x + 1) / P;
    const double c = a.tau;
    const double hmu = a.hmu;
    for (long g = W * blockIdx.x / P; g < g1;) {
        const long t = g / Nr;
        const long plo = g - t * Nr;
        const long phi = min(Nr, plo + (g1 - g));
        const int seg = (int)(blockIdx.x - sk_cta_of(t * Nr, W, P));
        long quad[2];
        bool ok[2], shared_k2;
        r2c_octet_item(t * kSkBlock + threadIdx.x, a.D, quad, ok, shared_k2);
        double K2[2];
        PairState st[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long mm = r2c_rep(quad[j >> 1], j & 1, a.D, a.log2D);
            const int l = (int)(mm >> a.log2D), k = (int)(mm & (a.D - 1));
            const double kx = __ldg(&a.ksym[k]), ky = __ldg(&a.ksym[l]);
            const cd e = a.fhat[mm], uu = a.fhat[n_modes + mm], vv = a.fhat[2 * n_modes + mm];
            const cd d = mk(-fma(kx, uu.y, ky * vv.y), fma(kx, uu.x, ky * vv.x));
            const cd z = mk(-fma(kx, vv.y, -ky * uu.y), fma(kx, vv.x, -ky * uu.x));
            pair_setup(st[j], e, d, z, hmu, c);
            K2[j >> 1] = fma(kx, kx, ky * ky);
        }
        DSums ds[2] = {dsums_zero(), dsums_zero()};
        for (long pt = a.pole_begin + plo; pt < a.pole_begin + phi; pt += kR2CTile) {
            const int cnt = (int)min((long)kR2CTile, a.pole_begin + phi - pt);
            __syncthreads();
            {
                const double2 *src = reinterpret_cast<const double2 *>(a.rpoles + pt);
                double2 *dst = reinterpret_cast<double2 *>(sp);
                constexpr int kPer = (int)(sizeof(R2CPole) / sizeof(double2));
                for (int i = threadIdx.x; i < cnt * kPer; i += kSkBlock) dst[i] = src[i];
            }
            __syncthreads();
            r2c_tile<PU, 2, true>(sp, cnt, K2, st, ds);   // octet items share K2
        }
        {
            ds[1] = ds[0];
        }
        cd *out = a.partial + (((size_t)t * a.sk_slots + seg) * 8) * kSkBlock + threadIdx.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const cd d0 = mk(0.5 * st[j].D2.x, 0.5 * st[j].D2.y);
            out[(2 * j) * kSkBlock] = cfma(ds[j >> 1].sigma(), d0, st[j].H0);
            out[(2 * j + 1) * kSkBlock] = cfma(ds[j >> 1].tau(), d0, st[j].H1);
        }
        g += phi - plo;
    }
}

// ----------------------------------------------------------------------------- PFHX (default)
// Explicit-solve R2C pairs. For every pole n and every {K, -K} pair the kernel forms the two
// Helmholtz solutions of the pair's representative mode from that mode's own right-hand sides
// (eq:lswEta, tau-scaled; partial fractions of the two resolvents, SURVEY.md
// 8(d) allowed equivalent):
//   num1  = B0  + i hn eta0 - (c/alpha) m0          eta1  = q num1         (alpha_n I + tau A)
//   num_t = Bt0 - i hn eta0 - conj(c/alpha) m0      eta_t = conj(q) num_t  (conj(alpha_n) I - tau A)
// with q = 1/(kappa_n + K2), one reciprocal per pole and K2 value (shared by the octet's eight
// modes; the second system's denominator is its conjugate). The solves at -K follow from the
// Hermitian data (R2C pairs above): conj(eta1(-K)) = eta_t + 2 conj(q) delta0 and
// conj(eta_t(-K)) = eta1 - 2 q delta0, so the Hermitian part of the pair's weighted sum takes,
// for every pole,
//   H_eta    += X1 eta1 + conj(X1) eta_t + sigma_n delta0,   sigma_n = conj(W1 q) - conj(W2) q
//   H_delta' += Y1 eta1 + conj(Y1) eta_t + tau'_n delta0     (P1, P2 for tau'_n)
// where X1 eta1 + conj(X1) eta_t = Re(X1)(eta1 + eta_t) + i Im(X1)(eta1 - eta_t). The delta
// back-substitution of each solve (delta = alpha eta - eta0, first row) is folded into the
// weights (PFH); zeta and (u, v) follow once per mode in finish_kernel. The two right-hand
// sides share their parts (B0, Bt0 = h mu eta0 +- delta0, c/alpha = sr + i si):
//   num1 = Z + Q,  num_t = Z - Q,  Z = h mu eta0 - sr m0,  Q = delta0 + i (hn eta0 - si m0),
// 10 instead of 12 fp64 instructions per pair. fp64 work per pole: 7 (denominator) + 8
// (sigma_n, tau'_n) per K2 value, 38 per pair (launch.h).
struct XPair {
    cd e0, E, m0, d0;         // eta0, h mu eta0, zeta0 - c eta0, delta0
    cd H0, H1;                // Hermitian accumulators: eta, delta' (before the -Re(sum w1) eta0 term)
};

// One pole of the explicit-solve R2C kernel, given q = 1/(kappa_n + K2): both Helmholtz
// solutions of the item's four pairs and their weighted accumulation.
__device__ __forceinline__ void r2x_pole(const R2XPole &P, const cd q, XPair (&st)[4]) {
    const cd sg = mk(fma(P.sgx1, q.x, P.sgx2 * q.y), fma(P.sgy1, q.x, P.sgy2 * q.y));
    const cd ta = mk(fma(P.tax1, q.x, P.tax2 * q.y), fma(P.tay1, q.x, P.tay2 * q.y));
    const double hn = P.hn, sr = P.s2r, si = P.s2i;
    const double xr = P.X1r, xi = P.X1i, yr = P.Y1r, yi = P.Y1i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        XPair &s = st[j];
        // right-hand sides of the two shifted systems after the Helmholtz reduction
        const cd Z = mk(fma(-sr, s.m0.x, s.E.x), fma(-sr, s.m0.y, s.E.y));
        const cd Q = mk(fma(-hn, s.e0.y, fma(si, s.m0.y, s.d0.x)), fma(hn, s.e0.x, fma(-si, s.m0.x, s.d0.y)));
        const cd n1 = mk(Z.x + Q.x, Z.y + Q.y);   // num1  = B0  + i hn eta0 - (c/alpha) m0
        const cd nt = mk(Z.x - Q.x, Z.y - Q.y);   // num_t = Bt0 - i hn eta0 - conj(c/alpha) m0
        // the two Helmholtz solutions of this pole and mode
        const cd eta1 = cmul(q, n1);
        const cd etat = mk(fma(q.x, nt.x, q.y * nt.y), fma(q.x, nt.y, -q.y * nt.x));   // conj(q) nt
        // weighted accumulation of the Hermitian part
        const cd S = mk(eta1.x + etat.x, eta1.y + etat.y);
        const cd Df = mk(eta1.x - etat.x, eta1.y - etat.y);
        s.H0.x = fma(xr, S.x, fma(-xi, Df.y, fma(sg.x, s.d0.x, fma(-sg.y, s.d0.y, s.H0.x))));
        s.H0.y = fma(xr, S.y, fma(xi, Df.x, fma(sg.x, s.d0.y, fma(sg.y, s.d0.x, s.H0.y))));
        s.H1.x = fma(yr, S.x, fma(-yi, Df.y, fma(ta.x, s.d0.x, fma(-ta.y, s.d0.y, s.H1.x))));
        s.H1.y = fma(yr, S.y, fma(yi, Df.x, fma(ta.x, s.d0.y, fma(ta.y, s.d0.x, s.H1.y))));
    }
}

template <int PU>
__device__ __forceinline__ void r2x_tile(const R2XPole *sp, int cnt, const double K2, XPair (&st)[4]) {
#pragma unroll PU
    for (int qq = 0; qq < cnt; ++qq) r2x_pole(sp[qq], pole_den(sp[qq], K2), st);
}

// Spectrum load; CG: through L2 only (ld.global.cg), for data another CTA of the same launch
// wrote (the fused small-grid step), which must not be served from a stale L1 line.
template <bool CG>
__device__ __forceinline__ cd ld_spec(const cd *p) {
    if (CG) {
        const double2 v = __ldcg(reinterpret_cast<const double2 *>(p));
        return mk(v.x, v.y);
    }
    return *p;
}

// Per-item setup of the explicit-solve R2C kernel: the four {K, -K} pairs of octet item `item`
// (r2c_octet_item), their representative modes rep[], validity ok[] and the shared K2; the
// pair state from the representative's spectrum (pole-independent, kept in registers).
// ld(f, m, j) returns field f of the spectrum at mode m, the representative of the item's pair j;
// ks(i) the symbol of index i (global or L2-only loads, or the fused step's staged copy).
template <class LD, class KS>
__device__ __forceinline__ void r2x_setup_ld(const PoleArgs &a, long item, XPair (&st)[4], long (&rep)[4],
                                             bool (&ok)[2], double &K2, LD ld, KS ks) {
    const double c = a.tau;
    const double hmu = a.hmu;
    const int H = a.D >> 1;
    long quad[2];
    bool shared_k2 = false;
    r2c_octet_item(item, a.D, quad, ok, shared_k2);
    K2 = 0.0;
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        const long qs = quad[g];
        long mq[4];
        quad_modes(qs, a.D, a.log2D, mq);
        const int qa = (int)(qs >> (a.log2D - 1)), qb = (int)(qs & (H - 1));
        rep[2 * g] = mq[0];
        rep[2 * g + 1] = (qa > 0 && qb > 0) ? mq[1] : mq[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const long mm = rep[2 * g + j];
            RX_ASSERT(mm >= 0 && mm < a.n_modes);
            const int l = (int)(mm >> a.log2D), k = (int)(mm & (a.D - 1));
            const double kx = ks(k), ky = ks(l);
            const cd e = ld(0, mm, 2 * g + j), uu = ld(1, mm, 2 * g + j), vv = ld(2, mm, 2 * g + j);
            // delta0 = i (kx u + ky v), zeta0 = i (kx v - ky u)   (tau-scaled)
            const cd d = mk(-fma(kx, uu.y, ky * vv.y), fma(kx, uu.x, ky * vv.x));
            const cd z = mk(-fma(kx, vv.y, -ky * uu.y), fma(kx, vv.x, -ky * uu.x));
            XPair &s = st[2 * g + j];
            s.e0 = e;
            s.d0 = d;
            s.E = mk(hmu * e.x, hmu * e.y);
            s.m0 = mk(fma(-c, e.x, z.x), fma(-c, e.y, z.y));
            s.H0 = mk(0, 0);
            s.H1 = mk(0, 0);
            K2 = fma(kx, kx, ky * ky);   // the same for all four pairs of an octet item
        }
    }
}

// r2x_setup_ld from the global spectrum a.fhat; CG: through L2 only (the fused small-grid step,
// whose ksym is then the CTA's shared-memory copy, read with generic loads).
template <bool CG>
__device__ __forceinline__ void r2x_setup(const PoleArgs &a, long item, XPair (&st)[4], long (&rep)[4],
                                          bool (&ok)[2], double &K2) {
    const long n_modes = a.n_modes;
    r2x_setup_ld(
        a, item, st, rep, ok, K2, [&](int f, long m, int) { return ld_spec<CG>(a.fhat + f * n_modes + m); },
        [&](int i) { return CG ? a.ksym[i] : __ldg(&a.ksym[i]); });
}

// The item's Hermitian accumulators (eta, delta') at the representative modes of chunk `chunk`.
__device__ __forceinline__ void r2x_store(const PoleArgs &a, int chunk, const XPair (&st)[4],
                                          const long (&rep)[4], const bool (&ok)[2]) {
    const long n_modes = a.n_modes;
    cd *out = a.partial + (size_t)chunk * 3 * n_modes;
    RX_ASSERT(chunk >= 0 && chunk < a.n_chunks && ((long)chunk * 3 + 2) * n_modes <= a.partial_cap);
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        if (ok[g]) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                out[rep[2 * g + j]] = st[2 * g + j].H0;
                out[n_modes + rep[2 * g + j]] = st[2 * g + j].H1;
            }
        }
    }
}

// grid = (octet-item tiles of BS, pole chunks); a thread owns one octet item (four {K, -K}
// pairs with one K2, r2c_octet_item) and runs every pole of its chunk.
template <int PU, int MINB, int BS = kPoleBlock>
__global__ void __launch_bounds__(BS, MINB) pole_kernel_r2x(PoleArgs a) {
    __shared__ R2XPole sp[kR2CTile];
    const int chunk = blockIdx.y;
    const long len = a.pole_end - a.pole_begin;
    const long p0 = a.pole_begin + len * chunk / a.n_chunks;
    const long p1 = a.pole_begin + len * (chunk + 1) / a.n_chunks;
    const long item = (long)blockIdx.x * BS + threadIdx.x;
    RX_ASSERT(p0 >= 0 && p0 <= p1 && p1 <= a.n_poles);
    long rep[4];
    bool ok[2];
    double K2;
    XPair st[4];
    r2x_setup<false>(a, item, st, rep, ok, K2);
    for (long pt = p0; pt < p1; pt += kR2CTile) {
        const int cnt = (int)min((long)kR2CTile, p1 - pt);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(a.xpoles + pt);
            double2 *dst = reinterpret_cast<double2 *>(sp);
            constexpr int kPer = (int)(sizeof(R2XPole) / sizeof(double2));
            for (int i = threadIdx.x; i < cnt * kPer; i += BS) dst[i] = src[i];
        }
        __syncthreads();
        r2x_tile<PU>(sp, cnt, K2, st);
    }
    r2x_store(a, chunk, st, rep, ok);
}

// ---- bulk-copy (TMA engine) staging of the pole table: mbarrier + cp.async.bulk helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arm the barrier for `bytes` of transaction count and issue one 1-D bulk copy global -> shared
// that completes them (a single elected thread)
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "RX_MBAR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra RX_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// pole_kernel_r2x with the pole table double-buffered in shared memory: thread 0 streams tile
// t + 1 (cnt x 144 contiguous bytes) by one bulk copy on the TMA engine while the block computes
// tile t, and the first tile's copy overlaps the item setup's spectrum loads. One block barrier
// per tile (the buffer about to be refilled was read during tile t - 1) instead of two around a
// copy every thread waits for.
template <int PU, int MINB, int BS = kPoleBlock>
__global__ void __launch_bounds__(BS, MINB) pole_kernel_r2x_bulk(PoleArgs a) {
    __shared__ __align__(128) R2XPole sp[2][kR2CTile];
    __shared__ __align__(8) unsigned long long bar[2];
    const int chunk = blockIdx.y;
    const long len = a.pole_end - a.pole_begin;
    const long p0 = a.pole_begin + len * chunk / a.n_chunks;
    const long p1 = a.pole_begin + len * (chunk + 1) / a.n_chunks;
    const long item = (long)blockIdx.x * BS + threadIdx.x;
    RX_ASSERT(p0 >= 0 && p0 <= p1 && p1 <= a.n_poles);
    const int ntiles = (int)((p1 - p0 + kR2CTile - 1) / kR2CTile);
    auto tile_cnt = [&](int t) { return (int)min((long)kR2CTile, p1 - p0 - (long)t * kR2CTile); };
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init_fence();
    }
    __syncthreads();
    if (threadIdx.x == 0 && ntiles > 0)
        bulk_load(sp[0], a.xpoles + p0, (unsigned)(tile_cnt(0) * sizeof(R2XPole)), &bar[0]);
    long rep[4];
    bool ok[2];
    double K2;
    XPair st[4];
    r2x_setup<false>(a, item, st, rep, ok, K2);
    for (int t = 0; t < ntiles; ++t) {
        if (t + 1 < ntiles) {
            __syncthreads();   // every thread is done with tile t - 1, whose buffer is refilled
            if (threadIdx.x == 0)
                bulk_load(sp[(t + 1) & 1], a.xpoles + p0 + (long)(t + 1) * kR2CTile,
                          (unsigned)(tile_cnt(t + 1) * sizeof(R2XPole)), &bar[(t + 1) & 1]);
        }
        mbar_wait(&bar[t & 1], (unsigned)((t >> 1) & 1));
        r2x_tile<PU>(sp[t & 1], tile_cnt(t), K2, st);
    }
    r2x_store(a, chunk, st, rep, ok);
}

// grid = (tiles, pole chunks). MPT < 4: a thread owns MPT modes m = tile0 + j * 128 + tid.
// MPT = 4: a thread owns one K2 quad (quad_modes) and computes the pole denominator
// 1/(kappa_n + K2) once for its four modes. Every thread runs all poles of its chunk, PU poles
// per loop trip. MINB = resident blocks per SM asked of ptxas (register budget).
template <int VARIANT, int MPT, int PU, int MINB>
__global__ void __launch_bounds__(kPoleBlock, MINB)
pole_kernel(PoleArgs a) {
    constexpr bool QUAD = (MPT == 4);
    __shared__ PoleConst sp[kPoleTile];
    const long n_modes = a.n_modes;
    const int chunk = blockIdx.y;
    const long len = a.pole_end - a.pole_begin;
    const long p0 = a.pole_begin + len * chunk / a.n_chunks;
    const long p1 = a.pole_begin + len * (chunk + 1) / a.n_chunks;
    const double c = a.tau;
    const double hmu = a.hmu;

    long mode[MPT];
    bool valid[MPT];
    if (QUAD) {
        const long q = (long)blockIdx.x * kPoleBlock + threadIdx.x;
        const bool ok = q < (n_modes >> 2);
        long mq[4];
        quad_modes(ok ? q : 0, a.D, a.log2D, mq);
#pragma unroll
        for (int j = 0; j < MPT; ++j) {
            mode[j] = mq[j & 3];
            valid[j] = ok;
        }
    } else {
        const long tile0 = (long)blockIdx.x * (kPoleBlock * MPT);
#pragma unroll
        for (int j = 0; j < MPT; ++j) {
            const long m = tile0 + j * kPoleBlock + threadIdx.x;
            valid[j] = m < n_modes;
            mode[j] = valid[j] ? m : 0;
        }
    }

    ModeState st[MPT];
#pragma unroll
    for (int j = 0; j < MPT; ++j) {
        const long mm = mode[j];
        const int l = (int)(mm >> a.log2D), k = (int)(mm & (a.D - 1));
        const double kx = __ldg(&a.ksym[k]), ky = __ldg(&a.ksym[l]);
        const cd e = a.fhat[mm], uu = a.fhat[n_modes + mm], vv = a.fhat[2 * n_modes + mm];
        ModeState &s = st[j];
        s.e0 = e;
        s.ua = uu;
        s.vb = vv;
        s.Kx = kx;
        s.Ky = ky;
        // delta0 = i (kx u + ky v) ; zeta0 = i (kx v - ky u)
        const cd d = mk(-fma(kx, uu.y, ky * vv.y), fma(kx, uu.x, ky * vv.x));
        const cd z = mk(-fma(kx, vv.y, -ky * uu.y), fma(kx, vv.x, -ky * uu.x));
        s.B0 = mk(fma(hmu, e.x, d.x), fma(hmu, e.y, d.y));
        s.Bt0 = mk(fma(hmu, e.x, -d.x), fma(hmu, e.y, -d.y));
        s.m0 = mk(fma(-c, e.x, z.x), fma(-c, e.y, z.y));
        s.K2 = fma(kx, kx, ky * ky);
        s.A0 = mk(0, 0);
        s.A1 = mk(0, 0);
        s.A2 = mk(0, 0);
    }

    for (long pt = p0; pt < p1; pt += kPoleTile) {
        const int cnt = (int)min((long)kPoleTile, p1 - pt);
        __syncthreads();
        {
            const double2 *src = reinterpret_cast<const double2 *>(a.poles + pt);
            double2 *dst = reinterpret_cast<double2 *>(sp);
            constexpr int kPer = (int)(sizeof(PoleConst) / sizeof(double2));
            for (int i = threadIdx.x; i < cnt * kPer; i += kPoleBlock) dst[i] = src[i];
        }
        __syncthreads();
        int q = 0;
#pragma unroll 1
        for (; q + PU <= cnt; q += PU) {
#pragma unroll
            for (int u = 0; u < PU; ++u) {
                const PoleConst &P = sp[q + u];
                if (QUAD) {
                    const cd qd = pole_den(P, st[0].K2);
#pragma unroll
                    for (int j = 0; j < MPT; ++j) pole_solves<VARIANT>(P, st[j], qd, c);
                } else {
#pragma unroll
                    for (int j = 0; j < MPT; ++j) pole_solves<VARIANT>(P, st[j], pole_den(P, st[j].K2), c);
                }
            }
        }
        if (PU > 1) {
#pragma unroll 1
            for (; q < cnt; ++q) {
                const PoleConst &P = sp[q];
#pragma unroll
                for (int j = 0; j < MPT; ++j) pole_solves<VARIANT>(P, st[j], pole_den(P, st[j].K2), c);
            }
        }
    }
    cd *out = a.partial + (size_t)chunk * 3 * n_modes;
#pragma unroll
    for (int j = 0; j < MPT; ++j) {
        if (valid[j]) {
            const long m = mode[j];
            out[m] = st[j].A0;
            out[n_modes + m] = st[j].A1;
            if (VARIANT == 1 || VARIANT == 3) out[2 * n_modes + m] = st[j].A2;   // else rebuilt
        }
    }
}

// R2C finish of mode m (kinds 6, 7): if m represents a {K, -K} pair (the smaller linear index),
// sum the chunk partials in a fixed order, rebuild delta and zeta, recover (u, v) and write the
// Hermitian spectrum at both modes. CG: partial / fhat loads through L2 only (fused step).
template <bool CG>
__device__ __forceinline__ void finish_r2c_mode(const FinishArgs &a, long m) {
    const long n = a.n_modes;
    const int l = (int)(m >> a.log2D), k = (int)(m & (a.D - 1));
    const long mm = ((long)((a.D - l) & (a.D - 1)) << a.log2D) + ((a.D - k) & (a.D - 1));
    if (mm <= m) return;   // self-mirror K = 0 corner (fixup_k0_kernel), or the mirror of a pair
    RX_ASSERT(m >= 0 && mm < n && ((long)(a.n_chunks - 1) * 3 + 2) * n <= a.partial_cap);
    // m is the representative of {K, -K} (the smaller linear index): finish both modes
    cd h0 = mk(0, 0), h1 = mk(0, 0);
    for (int c = 0; c < a.n_chunks; ++c) {
        const cd *p = a.partial + (size_t)c * 3 * n;
        const cd x0 = ld_spec<CG>(p + m), x1 = ld_spec<CG>(p + n + m);
        h0 = mk(h0.x + x0.x, h0.y + x0.y);
        h1 = mk(h1.x + x1.x, h1.y + x1.y);
    }
    const double kx = a.ksym[k], ky = a.ksym[l];
    const cd e = ld_spec<CG>(a.fhat + m), uu = ld_spec<CG>(a.fhat + n + m), vv = ld_spec<CG>(a.fhat + 2 * n + m);
    const double c = a.tau;
    // H(delta) = H(delta') - Re(sum w1) e0 ; H(zeta) = Re(S) m0 + c H(eta)
    h1 = mk(fma(-a.Sd.x, e.x, h1.x), fma(-a.Sd.x, e.y, h1.y));
    const cd m0 = mk(fma(-c, e.x, -fma(kx, vv.y, -ky * uu.y)), fma(-c, e.y, fma(kx, vv.x, -ky * uu.x)));
    const cd h2 = mk(fma(a.S.x, m0.x, c * h0.x), fma(a.S.x, m0.y, c * h0.y));
    const double inv = 1.0 / fma(kx, kx, ky * ky);   // K2 > 0: only the corners have K2 = 0
    const cd t = mk(fma(kx, h1.x, -ky * h2.x), fma(kx, h1.y, -ky * h2.y));
    const cd w = mk(fma(ky, h1.x, kx * h2.x), fma(ky, h1.y, kx * h2.y));
    const cd U = mk(t.y * inv, -t.x * inv), V = mk(w.y * inv, -w.x * inv);
    const int H = a.D >> 1, km = (a.D - k) & (a.D - 1);
    if (!a.half_out || k <= H) {
        a.acc[m] = h0;
        a.acc[n + m] = U;
        a.acc[2 * n + m] = V;
    }
    if (!a.half_out || km <= H) {
        a.acc[mm] = mk(h0.x, -h0.y);   // the Hermitian spectrum at -K is the conjugate
        a.acc[n + mm] = mk(U.x, -U.y);
        a.acc[2 * n + mm] = mk(V.x, -V.y);
    }
}

// ============================================================================= finish
// Sums the chunk partials in a fixed order. Kinds 0 and 2 accumulate only (eta, delta): the
// zeta component of every solve is affine in its eta component (the third equation,
// -c delta + alpha zeta = zeta0 with delta = alpha eta - eta0: zeta = (zeta0 - c eta0)/alpha + c eta,
// i.e. potential vorticity zeta - c eta is carried by m0 = zeta0 - c eta0), so
//   A_zeta = S m0 + c A_eta,  S = sum_n (w1_n / alpha_n + w2_n / |alpha_n|^2)   (exact),
// with S summed on the host in extended precision for the pole range. Then, for the DZ kinds,
// (u, v) are recovered from (delta, zeta).
__global__ void __launch_bounds__(256) finish_kernel(FinishArgs a) {
    const long m = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long n = a.n_modes;
    if (m >= n) return;
    if (a.kind == 6 || a.kind == 7) {   // R2C pairs: Hermitian accumulators at the representative mode
        finish_r2c_mode<false>(a, m);
        return;
    }
    const bool pv = (a.kind == 0 || a.kind == 2 || a.kind == 4 || a.kind == 5);
    cd s0 = mk(0, 0), s1 = mk(0, 0), s2 = mk(0, 0);
    for (int c = 0; c < a.n_chunks; ++c) {  // fixed order: deterministic
        const cd *p = a.partial + (size_t)c * 3 * n;
        const cd x0 = p[m], x1 = p[n + m];
        s0 = mk(s0.x + x0.x, s0.y + x0.y);
        s1 = mk(s1.x + x1.x, s1.y + x1.y);
        if (!pv) {
            const cd x2 = p[2 * n + m];
            s2 = mk(s2.x + x2.x, s2.y + x2.y);
        }
    }
    if (a.kind != 1) {   // DZ accumulators: (delta, zeta) -> (u, v)
        const int l = (int)(m >> a.log2D), k = (int)(m & (a.D - 1));
        const double kx = a.ksym[k], ky = a.ksym[l];
        if (pv) {
            const cd e = a.fhat[m], uu = a.fhat[n + m], vv = a.fhat[2 * n + m];
            if (a.kind == 5) s1 = cfms(a.Sd, e, s1);   // delta sum: + sum(W2 - W1) e0 = - sum(w1) e0
            const double c = a.tau;
            // m0 = zeta0 - c eta0, zeta0 = i (kx v - ky u)
            const cd m0 = mk(fma(-c, e.x, -fma(kx, vv.y, -ky * uu.y)), fma(-c, e.y, fma(kx, vv.x, -ky * uu.x)));
            s2 = cfma(a.S, m0, mk(c * s0.x, c * s0.y));
        }
        const double K2 = fma(kx, kx, ky * ky);
        if (K2 > 0.0) {
            // delta = i(kx u + ky v), zeta = i(kx v - ky u)
            //  => u = -i (kx delta - ky zeta)/K2,  v = -i (ky delta + kx zeta)/K2
            const double inv = 1.0 / K2;
            const cd t = mk(fma(kx, s1.x, -ky * s2.x), fma(kx, s1.y, -ky * s2.y));
            const cd w = mk(fma(ky, s1.x, kx * s2.x), fma(ky, s1.y, kx * s2.y));
            s1 = mk(t.y * inv, -t.x * inv);
            s2 = mk(w.y * inv, -w.x * inv);
        }
    }
    a.acc[m] = s0;
    a.acc[n + m] = s1;
    a.acc[2 * n + m] = s2;
}

// Finish of the stream-K R2C kernel: one thread per (tile, pair, item lane); sums the tile's
// segment partials in segment order and rebuilds (u, v) from the Hermitian (eta, delta, zeta)
// sums (as finish_kernel, kind 6) at the representative K and, conjugated, at -K.
__global__ void __launch_bounds__(256) finish_r2c_sk_kernel(FinishArgs a) {
    const long gid = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int tid = (int)(gid & (kSkBlock - 1)), pair = (int)((gid >> 8) & 3);
    const long t = gid >> 10;
    if (t >= a.sk_tiles) return;
    long quad[2];
    bool ok[2], shared_k2;
    r2c_octet_item(t * kSkBlock + tid, a.D, quad, ok, shared_k2);
    if (!ok[pair >> 1]) return;
    const long n = a.n_modes;
    const long r = r2c_rep(quad[pair >> 1], pair & 1, a.D, a.log2D);
    const int rl = (int)(r >> a.log2D), rk = (int)(r & (a.D - 1));
    const long mm = ((long)((a.D - rl) & (a.D - 1)) << a.log2D) + ((a.D - rk) & (a.D - 1));
    const long Nr = a.sk_poles, P = a.sk_ctas, W = a.sk_tiles * Nr;
    const long i0 = sk_cta_of(t * Nr, W, P), i1 = sk_cta_of((t + 1) * Nr - 1, W, P);
    cd h0 = mk(0, 0), h1 = mk(0, 0);
    const cd *p = a.partial + ((size_t)t * a.sk_slots * 8 + 2 * pair) * kSkBlock + tid;
    for (long s = 0; s <= i1 - i0; ++s) {
        const cd x0 = p[s * 8 * kSkBlock], x1 = p[(s * 8 + 1) * kSkBlock];
        h0 = mk(h0.x + x0.x, h0.y + x0.y);
        h1 = mk(h1.x + x1.x, h1.y + x1.y);
    }
    const double kx = a.ksym[rk], ky = a.ksym[rl];
    const cd e = a.fhat[r], uu = a.fhat[n + r], vv = a.fhat[2 * n + r];
    const double c = a.tau;
    // H(delta) = H(delta') - Re(sum w1) e0 ; H(zeta) = Re(S) m0 + c H(eta)
    h1 = mk(fma(-a.Sd.x, e.x, h1.x), fma(-a.Sd.x, e.y, h1.y));
    const cd m0 = mk(fma(-c, e.x, -fma(kx, vv.y, -ky * uu.y)), fma(-c, e.y, fma(kx, vv.x, -ky * uu.x)));
    const cd h2 = mk(fma(a.S.x, m0.x, c * h0.x), fma(a.S.x, m0.y, c * h0.y));
    const double inv = 1.0 / fma(kx, kx, ky * ky);   // K2 > 0 off the corners
    const cd tt = mk(fma(kx, h1.x, -ky * h2.x), fma(kx, h1.y, -ky * h2.y));
    const cd w = mk(fma(ky, h1.x, kx * h2.x), fma(ky, h1.y, kx * h2.y));
    const cd U = mk(tt.y * inv, -tt.x * inv), V = mk(w.y * inv, -w.x * inv);
    a.acc[r] = h0;
    a.acc[n + r] = U;
    a.acc[2 * n + r] = V;
    a.acc[mm] = mk(h0.x, -h0.y);      // the Hermitian spectrum at -K is the conjugate
    a.acc[n + mm] = mk(U.x, -U.y);
    a.acc[2 * n + mm] = mk(V.x, -V.y);
}

// ============================================================================= K = 0 modes (DZ)
// Modes with Kx = Ky = 0: (0,0), (0,D/2), (D/2,0), (D/2,D/2). There tau A only couples u, v
// through Coriolis: (u1,v1) = kappa^-1 [[alpha,-c],[c,alpha]] (a,b) (eq:lswVelocities with
// grad eta = 0) and (u2,v2) = conj(kappa)^-1 [[conj alpha, c],[-c, conj alpha]] (u1,v1).
// BS = 1024 when the fix-up runs alone; 128 when it runs beside the pole kernel (R2C): a
// 1024-thread block needs a whole SM's register file and would hold back that SM's pole blocks
// for its duration, a 128-thread one fits next to two resident pole blocks.
template <int kFixBlock>
__global__ void __launch_bounds__(kFixBlock) fixup_k0_kernel(FixupArgs a) {
    __shared__ cd red[2][kFixBlock];
    const int D = a.D, H = D / 2;
    const int ls[4] = {0, 0, H, H}, ks[4] = {0, H, 0, H};
    const long m = (long)ls[blockIdx.x] * D + ks[blockIdx.x];
    const long n = a.n_modes;
    const cd ua = a.fhat[n + m], vb = a.fhat[2 * n + m];
    cd Au = mk(0, 0), Av = mk(0, 0);
    for (long p = a.pole_begin + threadIdx.x; p < a.pole_end; p += kFixBlock) {
        const PoleConst *P = a.poles + p;
        const cd s3 = mk(__ldg(&P->s3r), __ldg(&P->s3i)), s4 = mk(__ldg(&P->s4r), __ldg(&P->s4i));
        const cd w1 = mk(__ldg(&P->w1r), __ldg(&P->w1i)), w2 = mk(__ldg(&P->w2r), __ldg(&P->w2i));
        const cd u1 = cfms(s4, vb, cmul(s3, ua));
        const cd v1 = cfma(s3, vb, cmul(s4, ua));
        if (a.method == 1) {   // REXI: one solve per term
            Au = cfma(w1, u1, Au);
            Av = cfma(w1, v1, Av);
            continue;
        }
        const cd u2 = cjfma(s4, v1, cjfma(s3, u1, mk(0, 0)));
        const cd v2 = cjfms(s4, u1, cjfma(s3, v1, mk(0, 0)));
        Au = cfma(w2, u2, cfma(w1, u1, Au));
        Av = cfma(w2, v2, cfma(w1, v1, Av));
    }
    red[0][threadIdx.x] = Au;
    red[1][threadIdx.x] = Av;
    __syncthreads();
    for (int s = kFixBlock / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const cd x = red[0][threadIdx.x + s], y = red[1][threadIdx.x + s];
            red[0][threadIdx.x] = mk(red[0][threadIdx.x].x + x.x, red[0][threadIdx.x].y + x.y);
            red[1][threadIdx.x] = mk(red[1][threadIdx.x].x + y.x, red[1][threadIdx.x].y + y.y);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (a.write_eta) {
            // R2C kind: the pole kernel skips the corners; at K = 0, eta1 = e0/alpha and
            // eta2 = eta1/conj(alpha), so sum(w1 eta1 + w2 eta2) = S e0 with the finish-kernel S.
            // The R2C accumulator is the Hermitian part H(A), which at a self-mirror mode is Re A.
            a.acc[m] = mk(cmul(a.S, a.fhat[m]).x, 0.0);
            a.acc[n + m] = mk(red[0][0].x, 0.0);
            a.acc[2 * n + m] = mk(red[1][0].x, 0.0);
        } else {
            a.acc[n + m] = red[0][0];
            a.acc[2 * n + m] = red[1][0];
        }
    }
}

// ============================================================================= Re projection
// Spectral form of "take the real part in physical space": for a spectrum X of
// a complex field, Re(IDFT(X)) = IDFT(H X) with (H X)(k, l) = (X(k, l) + conj(X(-k, -l))) / 2
// (indices mod D; the Nyquist index is its own mirror). Used between the steps of a
// spectral-resident multi-step run (S6) instead of an inverse + forward FFT round trip.
__global__ void __launch_bounds__(256) hermitian_kernel(const cd *__restrict__ in, cd *__restrict__ out,
                                                        long n_modes, int D, int log2D) {
    const long m = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= n_modes) return;
    const int l = (int)(m >> log2D), k = (int)(m & (D - 1));
    const long mm = ((long)((D - l) & (D - 1)) << log2D) + ((D - k) & (D - 1));
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        const cd x = in[f * n_modes + m], y = in[f * n_modes + mm];
        out[f * n_modes + m] = mk(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
    }
}

// ============================================================================= launchers
// ============================================================================= fused small-grid step
constexpr int kSmallThreads = 256;


// Pole records cached in shared memory when the cluster's range fits (loaded before stage A).
constexpr int kSmallPoleCache = 256;

// For small grids the seven launches of a step (4 FFT passes, pole kernel, finish, K = 0 fix-up)
// cost more in launch gaps than in work (C1: 64^2, 47 poles). step_small2_kernel runs the whole
// step S1..S5 as ONE launch of thread-block clusters (16 CTAs where the device allows the
// non-portable size, else 8), every exchange between stages through distributed shared memory
// (DSMEM), the pole range optionally split over several clusters. Per cluster:
//   A  forward rows (own row pairs, local slabs) -> X1, X2 stored into the column owners' slabs
//   B  forward half-spectrum columns -> the spectrum rows l <= D/2, distributed by row over the
//      cluster (row l in CTA l mod CS)
//   C  PFHX pole loop over the cluster's pole range: a CTA owns a contiguous set of octet items,
//      its threads split them into (item, pole chunk) units; the spectrum at the items'
//      representative modes is read from the owning CTAs' shared memory; chunk partials meet
//      in local shared memory; the four K = 0 corners on the last warp of the last CTA
//   D  R2C finish of every pair by its chunk-0 thread -> the Hermitian spectrum at the modes
//      k <= D/2, stored into the inverse column owners' slabs (one cluster) or into the
//      cluster's slice of cl_acc (several clusters; the last cluster to arrive sums the slices
//      in cluster order and goes on alone)
//   E  inverse half-spectrum columns -> Z = g1 + i g2 stored into the row-pair owners' slabs
//   F  inverse rows -> the three real fields
// Four cluster barriers (A|B, B|C, D|E, E|F) and one block barrier (C|D); no intermediate array
// in global memory with one cluster. Shared memory (cd units, small2_layout): column slabs,
// one auxiliary slab (the k = D/2 values of the CTA's k = 0 column), a region that holds the row
// slabs in A and F and the spectrum rows + chunk partials in between, the pole cache, twiddles
// and symbols. Same arithmetic as the multi-launch path (r2x_setup_ld, r2x_tile, the
// finish_r2c_mode formulas), except the K = 0 pole sums, reduced in a different order.
struct Small2Layout {
    int nu_max;   // row pairs / columns per CTA
    int ni_max;   // octet items per CTA
    int cslab, aux, rreg, stg, corner, part, pcache, tw, ks, total;   // offsets / size in cd
};
// Octet items of CTA c: [small2_items_begin(c), small2_items_begin(c + 1)), split in proportion to
// the CTA's pole workers (256, the last CTA 224: its last warp runs the K = 0 corners).
// (32-bit arithmetic: items <= 2142 for D <= 128, so items * 256 * CS < 2^31)
__host__ __device__ __forceinline__ int small2_items_begin(int items, int c, int CS) {
    return c >= CS ? items : items * (256 * c) / (256 * CS - 32);
}
__host__ __device__ __forceinline__ int small2_item_owner(int item, int items, int CS) {
    const int c = ((item + 1) * (256 * CS - 32) - 1) / (items * 256);
    return c < CS - 1 ? c : CS - 1;
}
__host__ __device__ constexpr Small2Layout small2_layout(int D, int CS) {
    Small2Layout L{};
    const int H = D / 2, PL = padded_len(D);
    L.nu_max = (3 * H + CS - 1) / CS;
    const long items = r2c_items(D, 2, true), capb = 256L * CS - 32;
    L.ni_max = (int)((items * 256 + capb - 1) / capb + 1);
    L.cslab = 0;
    L.aux = L.cslab + L.nu_max * (PL + 1);
    L.rreg = L.aux + PL;
    // between A and F the row-slab region holds the staged spectrum of the CTA's items
    // [pair][field][item], the four corners [corner][field] and the chunk partials
    // [chunk][pair][eta, delta'][item] (ni * ch <= max(256, ni) units)
    L.stg = L.rreg;
    L.corner = L.stg + L.ni_max * 12;
    L.part = L.corner + 12;
    const int mid = L.ni_max * 12 + 12 + 8 * (L.ni_max > 256 ? L.ni_max : 256);
    const int rsize = L.nu_max * PL > mid ? L.nu_max * PL : mid;
    L.pcache = L.rreg + rsize;
    L.tw = L.pcache + kSmallPoleCache * (int)(sizeof(R2XPole) / sizeof(cd));
    L.ks = L.tw + D;
    L.total = L.ks + (D + 1) / 2;
    return L;
}

// Where stage B stores spectrum value (l, k), l <= D/2, for the pole stage: the CTA owning the
// item whose pair it represents and the staging index there (field f at idx + f * fstride;
// layout [pair][field][item], consecutive items in consecutive slots), or the corner slot of the
// last CTA (K = 0 modes); false if (l, k) represents no pair (a mirror).
// The inverse of r2c_octet_item / quad_modes / the representative choice of r2x_setup_ld.
__device__ __forceinline__ bool small2_stage_slot(int l, int k, int D, int items, int CS, const Small2Layout &L,
                                                  int &cta, int &idx, int &fstride) {
    const int H = D >> 1;
    const bool lb = (l == 0 || l == H), kb = (k == 0 || k == H);
    if (l > H) return false;
    if (lb && kb) {   // corner q = (l == H) * 2 + (k == H)
        cta = CS - 1;
        idx = L.corner + ((l == H ? 2 : 0) + (k == H ? 1 : 0)) * 3;
        fstride = 1;
        return true;
    }
    int a, b, j;
    if (lb) {
        if (k > H) return false;      // mirror of (l, D - k)
        if (l == 0) { a = 0; b = k; } else { a = k; b = 0; }
        j = 0;
    } else if (k == 0) {
        a = 0; b = l; j = 1;          // axis quad (0, l): pair {(l, 0), (D - l, 0)}
    } else if (k == H) {
        a = l; b = 0; j = 1;          // Nyquist quad (l, 0): pair {(l, H), (D - l, H)}
    } else {
        a = l; b = k < H ? k : D - k; j = k < H ? 0 : 1;   // interior quad (l, |k|)
    }
    const int n_oct = (int)r2c_n_oct(D);
    int item;
    int gq = 0;
    if (a > 0 && b > 0 && a != b) {
        const int ap = (a < b ? a : b) - 1, bp = (a < b ? b : a) - 1;
        item = bp * (bp - 1) / 2 + ap;
        gq = a < b ? 0 : 1;
    } else if (a == b) {
        item = n_oct + (a - 1);
    } else if (a == 0) {
        item = n_oct + (H - 1) + (b - 1);
    } else {
        item = n_oct + 2 * (H - 1) + (a - 1);
    }
    cta = small2_item_owner(item, items, CS);
    idx = L.stg + (2 * gq + j) * 3 * L.ni_max + (item - small2_items_begin(items, cta, CS));
    fstride = L.ni_max;
    return true;
}


// owner CTA of index u of P units split as [P c / CS, P (c + 1) / CS)
__device__ __forceinline__ int small2_owner(int u, int P, int CS) { return ((u + 1) * CS - 1) / P; }

// Representative mode of pair j (0..3) of octet item `item` (as r2x_setup_ld orders them);
// false for the discarded half of a single-quad item.
__device__ __forceinline__ bool r2x_pair_rep(long item, int D, int log2D, int j, long &rep) {
    const int H = D >> 1;
    long quad[2];
    bool ok[2], shared_k2;
    r2c_octet_item(item, D, quad, ok, shared_k2);
    const bool g1 = (j >> 1) != 0;   // selects, not a runtime array index (no local memory)
    if (!(g1 ? ok[1] : ok[0])) return false;
    const long qs = g1 ? quad[1] : quad[0];
    long mq[4];
    quad_modes(qs, D, log2D, mq);
    const int qa = (int)(qs >> (log2D - 1)), qb = (int)(qs & (H - 1));
    rep = (j & 1) == 0 ? mq[0] : ((qa > 0 && qb > 0) ? mq[1] : mq[2]);
    return true;
}

// The n (<= nmax) length-D transforms at s + j * ld (j < n) in shared memory (natural order at
// pidx(i), in place), X[k] = sum_i x[i] e^{-+2 pi i ik/D}, by the Stockham passes of the
// multi-launch kernels (tf = D/8 threads per transform), in rounds of blockDim / tf transforms
// (uniform round count: the passes hold block barriers). Not inlined: the step runs its code
// once, cold, so one copy for the four stages (A, B, E, F) costs less instruction fetch than
// four. (A warp-synchronous radix-2 variant with shfl.xor stages measured 1420 cycles against
// 1230 for these passes on the C1 shape: tools/fft_probe.cu.)
template <int LOGD>
__device__ __noinline__ void small2_ffts(cd *s, int ld, int n, int nmax, const cd *tws, bool inv) {
    constexpr int D = 1 << LOGD, tf = D >= 8 ? D / 8 : 1;
    const int per = (int)blockDim.x / tf, j0 = (int)threadIdx.x / tf, t = (int)threadIdx.x - j0 * tf;
    for (int base = 0; base < nmax; base += per) {
        const int j = base + j0;
        if (inv) fft_in_smem<true, true>(s + j * ld, D, LOGD, t, tf, tws, j < n);
        else fft_in_smem<false, true>(s + j * ld, D, LOGD, t, tf, tws, j < n);
    }
}

template <int LOGD, int CS>
__global__ void __launch_bounds__(kSmallThreads, 1) step_small2_kernel(SmallArgs a) {
    constexpr int D = 1 << LOGD, H = D >> 1, LOGH = LOGD - 1;
    constexpr int PL = padded_len(D);
    constexpr int stride = PL + 1;   // column slabs
    constexpr int P3 = 3 * H;        // row pairs (A, F) = half-spectrum columns (B, E), all fields
    extern __shared__ cd smem[];
    __shared__ int s_last;
    cgx::cluster_group cl = cgx::this_cluster();
    const int cta = (int)cl.block_rank();
    const int g = (int)(blockIdx.x / (unsigned)CS);   // cluster index
    const int NC = a.n_clusters;
    const int tid = threadIdx.x;
    constexpr int NT = kSmallThreads;
    // every offset a compile-time constant (CS is a template parameter): fewer live registers
    constexpr Small2Layout L = small2_layout(D, CS);
    const int u0 = (P3 * cta) / CS, u1 = (P3 * (cta + 1)) / CS;
    const int nu = u1 - u0;
    if (a.stop_after < -1) return;   // stage-timing measurements only
#define SMALL2_MARK(k)                                                             \
    do {                                                                           \
        if (a.trace && (tid == 0 || tid == kSmallThreads - 1))                     \
            a.trace[((long)blockIdx.x * 2 + (tid != 0)) * 16 + (k)] = clock64();   \
    } while (0)
    SMALL2_MARK(0);
    rx_poison_smem();          // (checked builds) before the arrival: no remote store is lost to it
    cluster_arrive_relaxed();
    RX_ASSERT(nu <= L.nu_max && (long)L.total * 16 <= (long)dyn_smem_bytes() && g < NC && a.steps >= 1 &&
              (a.steps == 1 || NC == 1));
    cd *cs_ = smem + L.cslab;          // column slabs
    cd *rr = smem + L.rreg;            // row slabs (A, F) | spectrum rows + partials (B..D)
    R2XPole *pc = reinterpret_cast<R2XPole *>(smem + L.pcache);
    cd *tws = smem + L.tw;
    double *ksm = reinterpret_cast<double *>(smem + L.ks);
    // this cluster's pole range
    const long pb_all = a.pole.pole_begin, np_all = a.pole.pole_end - a.pole.pole_begin;
    // (32-bit: a fused step has fewer than 2^31 / kSmallMaxClusters poles, checked on the host)
    const long pb = pb_all + (int)np_all * g / NC;
    const int npl = (int)(pb_all + (int)np_all * (g + 1) / NC - pb);
    const bool cached = npl <= kSmallPoleCache;
    if (cta == CS - 1 && tid >= kSmallThreads - 32) {
        // the corner warp's pole records (generic table, read in stage C): into L2 now
#pragma unroll 1
        for (long p = pb + (tid & 31); p < pb + npl; p += 32) {
            const char *q = reinterpret_cast<const char *>(a.poles + p);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(q + sizeof(PoleConst) - 1));
        }
    }
    // Preload (pole records, twiddles, symbols) and the A inputs: every global load of this
    // thread is issued before the first shared-memory store (one memory latency, not one per
    // loop trip; the inputs were flushed from L2 between steps)
    {
        constexpr int kPer = (int)(sizeof(R2XPole) / sizeof(double2));
        constexpr int RP = (kSmallPoleCache * kPer + kSmallThreads - 1) / kSmallThreads;
        constexpr int RI = (((3 * H + 7) / 8) * D + kSmallThreads - 1) / kSmallThreads;   // CS >= 8
        RX_ASSERT(NT == kSmallThreads && nu * D <= RI * NT);
        const double2 *psrc = reinterpret_cast<const double2 *>(a.pole.xpoles + pb);
        double2 *pdst = reinterpret_cast<double2 *>(pc);
        const int n2 = cached ? (int)npl * kPer : 0;
        double2 pv[RP], iv[RI];
#pragma unroll
        for (int r = 0; r < RP; ++r)
            if (tid + r * NT < n2) pv[r] = __ldg(psrc + tid + r * NT);
#pragma unroll
        for (int r = 0; r < RI; ++r) {
            const int i = tid + r * NT;
            if (i < nu * D) {
                const int pr = i >> LOGD, x = i & (D - 1);
                const int gp = u0 + pr, f = gp >> LOGH, pair = gp & (H - 1);
                const double *in = a.in[f] + (size_t)(2 * pair) * D + x;
                iv[r] = make_double2(__ldg(in), __ldg(in + D));
            }
        }
        cd tw0;
        double ks0 = 0.0;
        if (tid < D) {
            tw0 = a.tw[tid];
            ks0 = __ldg(a.pole.ksym + tid);
        }
#pragma unroll
        for (int r = 0; r < RP; ++r)
            if (tid + r * NT < n2) pdst[tid + r * NT] = pv[r];
        // ---- A: forward rows (local): two real rows per complex transform
#pragma unroll
        for (int r = 0; r < RI; ++r) {
            const int i = tid + r * NT;
            if (i < nu * D) rr[(i >> LOGD) * PL + pidx(i & (D - 1))] = mk(iv[r].x, iv[r].y);
        }
        if (tid < D) {
            tws[tid] = tw0;
            ksm[tid] = ks0;
        }
    }
    SMALL2_MARK(1);
    __syncthreads();
    if (a.stop_after < 0) {   // stage-timing measurements only
        cluster_wait();
        return;
    }
    small2_ffts<LOGD>(rr, PL, nu, L.nu_max, tws, false);
    SMALL2_MARK(2);
    cluster_wait();   // every CTA of the cluster runs: DSMEM stores may start
    for (int i = tid; i < nu * H; i += NT) {
        const int pr = i >> LOGH, k = i & (H - 1);
        const int gp = u0 + pr, f = gp >> LOGH, pair = gp & (H - 1);
        const cd *Z = rr + pr * PL;
        cd X1, X2;
        if (k == 0) {
            const cd z0 = Z[pidx(0)], zh = Z[pidx(H)];
            X1 = mk(z0.x, zh.x);
            X2 = mk(z0.y, zh.y);
        } else {
            const cd zk = Z[pidx(k)], zm = Z[pidx(D - k)];
            X1 = mk(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
            X2 = mk(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
        }
        const int gc = f * H + k, oc = small2_owner(gc, P3, CS);
        cd *col = cl.map_shared_rank(cs_, oc) + (gc - (P3 * oc) / CS) * stride;
        RX_ASSERT((gc - (P3 * oc) / CS) < L.nu_max);
        col[pidx(2 * pair)] = X1;
        col[pidx(2 * pair + 1)] = X2;
    }
    cluster_barrier();

    SMALL2_MARK(3);
    if (a.stop_after <= 0) return;   // stage-timing measurements only
    // ---- B: forward columns (local) -> the spectrum at every pair representative, D^-2, staged
    // in the shared memory of the CTA that owns the pair's octet item (and the K = 0 corners)
    small2_ffts<LOGD>(cs_, stride, nu, L.nu_max, tws, false);
    SMALL2_MARK(13);
    {
        const double sc = a.scale;
        const int items = (int)a.n_items;
        auto put_spec = [&](int f, int l, int k, cd v) {
            int oc, idx, fs;
            if (small2_stage_slot(l, k, D, items, CS, L, oc, idx, fs)) {
                RX_ASSERT(idx + f * fs < L.part);
                cl.map_shared_rank(smem, oc)[idx + f * fs] = v;
            }
        };
        for (int i = tid; i < nu * D; i += NT) {
            const int c = i >> LOGD, l = i & (D - 1);
            const int gc = u0 + c, f = gc >> LOGH, k = gc & (H - 1);
            const int lm = (D - l) & (D - 1);
            const cd v = cs_[c * stride + pidx(l)];
            if (k == 0) {
                if (l <= H) {
                    const cd w = cs_[c * stride + pidx(lm)];
                    const double hs = 0.5 * sc;
                    put_spec(f, l, 0, mk(hs * (v.x + w.x), hs * (v.y - w.y)));
                    put_spec(f, l, H, mk(hs * (v.y + w.y), hs * (w.x - v.x)));
                }
            } else {
                if (l <= H) put_spec(f, l, k, mk(v.x * sc, v.y * sc));
                if (lm <= H) put_spec(f, lm, D - k, mk(v.x * sc, -v.y * sc));
            }
        }
    }
    SMALL2_MARK(14);
    cluster_barrier();

    SMALL2_MARK(4);
    if (a.stop_after <= 1) return;   // stage-timing measurements only
    // ---- C + D: pole loop over (item, chunk) units, chunk partials in shared memory, finish
    const double c_tau = a.pole.tau;
    const cd Sg = a.Sg[g], Sdg = a.Sdg[g];
    // the Hermitian spectrum value v of field f at (l, k), k <= H: into the inverse column
    // owner's slab (T0 at k = 0, TH of the k = 0 column at k = H: the auxiliary slab), or into
    // this cluster's slice of cl_acc
    auto put_acc = [&](int f, int l, int k, cd v) {
        if (NC > 1) {
            a.cl_acc[(((size_t)g * 3 + f) * D + l) * (H + 1) + k] = v;
            return;
        }
        const int gc = f * H + (k == H ? 0 : k), oc = small2_owner(gc, P3, CS);
        cd *base = cl.map_shared_rank(smem, oc);
        if (k == H) base[L.aux + pidx(l)] = v;
        else base[L.cslab + (gc - (P3 * oc) / CS) * stride + pidx(l)] = v;
    };
    cd *stg = smem + L.stg;   // [pair][field][item]
    // Multi-step runs (a.steps > 1, one cluster): steps 1..K-1 finish into the staged spectrum
    // of the same CTA's items (the state stays in shared memory, Fourier space, Hermitian by
    // construction: PAPER.md:434's Re is the R2C pair sum), and only the last step goes on to
    // the inverse transform — no exchange between the steps of a run.
    for (int step = 0; step < a.steps; ++step) {
    const bool last = step == a.steps - 1;
    {
        const int items = (int)a.n_items;
        // item split weighted by the workers per CTA (the last CTA's last warp takes the corners)
        const int i0 = small2_items_begin(items, cta, CS), i1 = small2_items_begin(items, cta + 1, CS);
        const int ni = i1 - i0;
        const int W = cta == CS - 1 ? kSmallThreads - 32 : kSmallThreads;
        const int ch = ni > 0 ? max(1, min(npl, W / ni)) : 1;
        RX_ASSERT((long)ni * ch * 8 <= L.pcache - L.part);
        cd *part = smem + L.part;   // [chunk][item][pair][eta, delta']
        // one instance of the pole tile: the cached records or the global table, generic loads
        const R2XPole *src = cached ? pc : a.pole.xpoles + pb;
        for (int u = tid; u < ni * ch && tid < W; u += W) {
            const int il = u % ni, chunk = u / ni;
            XPair st[4];
            long rep[4];
            bool ok[2];
            double K2;
            r2x_setup_ld(
                a.pole, i0 + il, st, rep, ok, K2, [&](int f, long, int j) { return stg[(j * 3 + f) * L.ni_max + il]; },
                [&](int i) { return ksm[i]; });
            if (u == tid) SMALL2_MARK(5);
            const int p0 = npl * chunk / ch, p1 = a.stop_after == 2 ? p0 : npl * (chunk + 1) / ch;
            r2x_tile<1>(src + p0, p1 - p0, K2, st);   // one pole per trip: half the code of PU = 2
            if (u == tid) SMALL2_MARK(6);
            cd *p = part + (size_t)chunk * 8 * ni + il;   // [chunk][pair][eta, delta'][item]
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                p[(2 * j) * ni] = st[j].H0;
                p[(2 * j + 1) * ni] = st[j].H1;
            }
        }
        if (cta == CS - 1 && tid >= kSmallThreads - 32) {
            // the four K = 0 corners (fixup_k0_kernel): lanes stride the poles, every lane runs
            // the four corners of its poles (one pole record load serves four corners)
            const int lane = tid & 31;
            cd e0[4], ua[4], vb[4];
            double Au[4], Av[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {   // (0,0) (0,H) (H,0) (H,H)
                e0[q] = smem[L.corner + q * 3];
                ua[q] = smem[L.corner + q * 3 + 1];
                vb[q] = smem[L.corner + q * 3 + 2];
                Au[q] = 0.0;
                Av[q] = 0.0;
            }
            for (long p = pb + lane; p < pb + npl && a.stop_after != 2; p += 32) {
                const PoleConst *P = a.poles + p;
                const cd s3 = mk(__ldg(&P->s3r), __ldg(&P->s3i)), s4 = mk(__ldg(&P->s4r), __ldg(&P->s4i));
                const cd w1 = mk(__ldg(&P->w1r), __ldg(&P->w1i)), w2 = mk(__ldg(&P->w2r), __ldg(&P->w2i));
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const cd u1 = cfms(s4, vb[q], cmul(s3, ua[q]));
                    const cd v1 = cfma(s3, vb[q], cmul(s4, ua[q]));
                    // Re(w1 u1 + w2 u2): the self-mirror modes keep the real part (Hermitian part)
                    double ru = fma(w1.x, u1.x, -w1.y * u1.y), rv = fma(w1.x, v1.x, -w1.y * v1.y);
                    if (a.method != 1) {   // REXII: the second solve (REXI: one solve per term)
                        const cd u2 = cjfma(s4, v1, cjfma(s3, u1, mk(0, 0)));
                        const cd v2 = cjfms(s4, u1, cjfma(s3, v1, mk(0, 0)));
                        ru = fma(w2.x, u2.x, fma(-w2.y, u2.y, ru));
                        rv = fma(w2.x, v2.x, fma(-w2.y, v2.y, rv));
                    }
                    Au[q] += ru;
                    Av[q] += rv;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    Au[q] += __shfl_xor_sync(0xffffffffu, Au[q], o);
                    Av[q] += __shfl_xor_sync(0xffffffffu, Av[q], o);
                }
            }
            if (lane < 4) {
                // self-mirror modes: the Hermitian part is Re; eta = S e0 there
                const int q = lane, l = (q >> 1) * H, k = (q & 1) * H;
                double au = Au[0], av = Av[0];
                cd e = e0[0];
#pragma unroll
                for (int r = 1; r < 4; ++r) {
                    if (q == r) {
                        au = Au[r];
                        av = Av[r];
                        e = e0[r];
                    }
                }
                if (last) {
                    put_acc(0, l, k, mk(cmul(Sg, e).x, 0.0));
                    put_acc(1, l, k, mk(au, 0.0));
                    put_acc(2, l, k, mk(av, 0.0));
                } else {   // the next step's corner state (only this warp reads it)
                    smem[L.corner + q * 3] = mk(cmul(Sg, e).x, 0.0);
                    smem[L.corner + q * 3 + 1] = mk(au, 0.0);
                    smem[L.corner + q * 3 + 2] = mk(av, 0.0);
                }
            }
        }
        SMALL2_MARK(7);
        __syncthreads();
        SMALL2_MARK(8);
        // D: finish every pair of the CTA's items (all threads): chunk partials in a fixed
        // order, then the formulas of finish_r2c_mode from the pair's spectrum
        for (int t = tid; t < ni * 4; t += NT) {
            const int j = t / ni, il = t - j * ni;
            long m;
            if (!r2x_pair_rep(i0 + il, D, LOGD, j, m)) continue;
            cd h0 = mk(0, 0), h1 = mk(0, 0);
            for (int cc = 0; cc < ch; ++cc) {
                const cd *p = part + ((size_t)cc * 8 + 2 * j) * ni + il;
                h0 = mk(h0.x + p[0].x, h0.y + p[0].y);
                h1 = mk(h1.x + p[ni].x, h1.y + p[ni].y);
            }
            const int l = (int)(m >> LOGD), k = (int)(m & (D - 1));
            const double kx = ksm[k], ky = ksm[l];
            const cd *sp = stg + j * 3 * L.ni_max + il;
            const cd e = sp[0], uu = sp[L.ni_max], vv = sp[2 * L.ni_max];
            // H(delta) = H(delta') - Re(sum w1) e0 ; H(zeta) = Re(S) m0 + c H(eta)
            h1 = mk(fma(-Sdg.x, e.x, h1.x), fma(-Sdg.x, e.y, h1.y));
            const cd m0 = mk(fma(-c_tau, e.x, -fma(kx, vv.y, -ky * uu.y)), fma(-c_tau, e.y, fma(kx, vv.x, -ky * uu.x)));
            const cd h2 = mk(fma(Sg.x, m0.x, c_tau * h0.x), fma(Sg.x, m0.y, c_tau * h0.y));
            const double inv = 1.0 / fma(kx, kx, ky * ky);   // K2 > 0 off the corners
            const cd tt = mk(fma(kx, h1.x, -ky * h2.x), fma(kx, h1.y, -ky * h2.y));
            const cd w = mk(fma(ky, h1.x, kx * h2.x), fma(ky, h1.y, kx * h2.y));
            const cd U = mk(tt.y * inv, -tt.x * inv), V = mk(w.y * inv, -w.x * inv);
            if (!last) {   // the next step's state at the representative (read after the barrier)
                stg[j * 3 * L.ni_max + il] = h0;
                stg[(j * 3 + 1) * L.ni_max + il] = U;
                stg[(j * 3 + 2) * L.ni_max + il] = V;
                continue;
            }
            const int lm = (D - l) & (D - 1), km = (D - k) & (D - 1);
            const cd hv[3] = {h0, U, V};
            // the pair's two modes (the -K one conjugated) wherever k <= H; one copy of the stores
#pragma unroll 1
            for (int q = 0; q < 6; ++q) {
                const int fq = q % 3;
                const bool mir = q >= 3;
                if (mir ? km <= H : k <= H) {
                    const cd x = fq == 0 ? hv[0] : fq == 1 ? hv[1] : hv[2];   // (no local-memory array)
                    put_acc(fq, mir ? lm : l, mir ? km : k, mir ? mk(x.x, -x.y) : x);
                }
            }
        }
    }
    if (!last) __syncthreads();   // this step's state written before the next step's setup reads it
    }   // steps
    SMALL2_MARK(9);
    if (NC > 1) {
        // hand-off: the last cluster to arrive sums the clusters' spectra (fixed order) alone.
        // The cluster barrier orders every thread's cl_acc stores before thread 0's gpu-scope
        // fence (cumulative), which precedes its arrival on the counter
        cluster_barrier();
        if (cta == 0 && tid == 0) {
            __threadfence();
            const unsigned old = atomicAdd(a.counter, 1u);
            const int last = old == (unsigned)(NC - 1);
            if (last) *a.counter = 0u;   // every cluster has arrived: reset for the next launch
            __threadfence();
            for (int r = 0; r < CS; ++r) *cl.map_shared_rank(&s_last, r) = last;
        }
        cluster_barrier();
        if (!s_last) return;
        for (int i = tid; i < nu * D; i += NT) {
            const int c = i >> LOGD, l = i & (D - 1);
            const int gc = u0 + c, f = gc >> LOGH, k = gc & (H - 1);
            cd v = mk(0, 0), vh = mk(0, 0);
            for (int q = 0; q < NC; ++q) {
                const cd *src = a.cl_acc + (((size_t)q * 3 + f) * D + l) * (H + 1);
                const cd x = ld_spec<true>(src + k);
                v = mk(v.x + x.x, v.y + x.y);
                if (k == 0) {
                    const cd y = ld_spec<true>(src + H);
                    vh = mk(vh.x + y.x, vh.y + y.y);
                }
            }
            if (k == 0) v = mk(v.x - vh.y, v.y + vh.x);   // T0 + i TH
            cs_[c * stride + pidx(l)] = v;
        }
        __syncthreads();
    } else {
        cluster_barrier();
        // the k = 0 column packs T0 + i TH (TH arrived in the auxiliary slab)
        for (int i = tid; i < nu * D; i += NT) {
            const int c = i >> LOGD, l = i & (D - 1);
            if (((u0 + c) & (H - 1)) != 0) continue;
            const cd t0 = cs_[c * stride + pidx(l)], th = smem[L.aux + pidx(l)];
            cs_[c * stride + pidx(l)] = mk(t0.x - th.y, t0.y + th.x);
        }
        __syncthreads();
    }

    SMALL2_MARK(10);
    if (a.stop_after <= 3) return;   // stage-timing measurements only
    // ---- E: inverse columns (Hermitian input) -> Z rows into the row-pair owners
    small2_ffts<LOGD>(cs_, stride, nu, L.nu_max, tws, true);
    SMALL2_MARK(15);
    for (int i = tid; i < nu * H; i += NT) {
        const int c = i >> LOGH, p = i & (H - 1);
        const int gc = u0 + c, f = gc >> LOGH, k = gc & (H - 1);
        const cd g1 = cs_[c * stride + pidx(2 * p)], g2 = cs_[c * stride + pidx(2 * p + 1)];
        const int gp = f * H + p, oc = small2_owner(gp, P3, CS);
        cd *Z = cl.map_shared_rank(rr, oc) + (gp - (P3 * oc) / CS) * PL;
        if (k == 0) {
            Z[pidx(0)] = mk(g1.x, g2.x);
            Z[pidx(H)] = mk(g1.y, g2.y);
        } else {
            Z[pidx(k)] = mk(g1.x - g2.y, g1.y + g2.x);        // g1 + i g2
            Z[pidx(D - k)] = mk(g1.x + g2.y, g2.x - g1.y);    // conj g1 + i conj g2
        }
    }
    cluster_barrier();

    SMALL2_MARK(11);
    if (a.stop_after <= 4) return;   // stage-timing measurements only
    // ---- F: inverse rows (local) -> the three real fields
    small2_ffts<LOGD>(rr, PL, nu, L.nu_max, tws, true);
    for (int i = tid; i < nu * D; i += NT) {
        const int pr = i >> LOGD, x = i & (D - 1);
        const int gp = u0 + pr, f = gp >> LOGH, pair = gp & (H - 1);
        const cd v = rr[pr * PL + pidx(x)];
        const size_t gi = (size_t)(2 * pair) * D + x;
        a.out[f][gi] = v.x;
        a.out[f][gi + D] = v.y;
    }
    SMALL2_MARK(12);
#undef SMALL2_MARK
}

static int ilog2(int x) {
    int r = 0;
    while ((1 << r) < x) ++r;
    return r;
}

// FFT launch shapes: threads per transform tf = max(1, D/8); a row block holds nb row pairs
// (nb * tf <= 64 threads unless one pair needs more, nb <= D/2); a column block a strip of
// C <= 4 half-spectrum slots (C * tf <= 512, C <= D/2).
// REXI_FFT_ROWS / REXI_FFT_COLS (environment, read once): override the row pairs / columns per
// block of the FFT passes — a tuning knob for measurements (tools/time_fft.py), not a setting.
static int fft_env(const char *name) {
    const char *v = getenv(name);
    return v ? atoi(v) : 0;
}
static int fft_rows_per_block(int D) {
    static const int force = fft_env("REXI_FFT_ROWS");
    const int tf = D >= 8 ? D / 8 : 1;
    int nb = force > 0 ? force : 64 / tf;   // small blocks: latency-bound passes, more blocks in flight
    if (nb < 1) nb = 1;
    if (nb * tf > 1024) nb = 1024 / tf;
    if (nb > D / 2) nb = D / 2;
    return nb;
}
static int fft_cols_per_block(int D) {
    static const int force = fft_env("REXI_FFT_COLS");
    const int tf = D >= 8 ? D / 8 : 1;
    // measured (tools/time_fft.py, profiles/r02l_fft_tune.log): 4-column slabs beat 8 at 512^2
    // and 1024^2; at 4096^2 two columns per 1024-thread block (32-byte sectors per row instead
    // of 16 bytes) beat one: forward 1058 -> 887 us, inverse 901 -> 871 us
    int C = std::max(2, 512 / tf);
    if (C > 4) C = 4;
    if (force > 0) C = force;
    if (C * tf > 1024) C = 1024 / tf;
    if (C < 1) C = 1;
    if (C > D / 2) C = D / 2;
    return C;
}

cudaError_t fft_setup_attributes() {
    cudaError_t e;
    const int maxsm = 200 * 1024;
#define SETA(K) if ((e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    SETA(fft_rows_fwd_kernel)
    SETA(fft_cols_fwd_kernel)
    SETA(fft_cols_inv_kernel<true>)
    SETA(fft_cols_inv_kernel<false>)
    SETA(fft_rows_inv_kernel)
    SETA(fft_rows_fwd16_kernel<9>) SETA(fft_rows_fwd16_kernel<10>) SETA(fft_rows_fwd16_kernel<11>)
    SETA(fft_rows_fwd16_kernel<12>) SETA(fft_rows_fwd16_kernel<13>)
    SETA(fft_rows_inv16_kernel<9>) SETA(fft_rows_inv16_kernel<10>) SETA(fft_rows_inv16_kernel<11>)
    SETA(fft_rows_inv16_kernel<12>) SETA(fft_rows_inv16_kernel<13>)
    SETA(fft_cols_fwd16_kernel<9>) SETA(fft_cols_fwd16_kernel<10>) SETA(fft_cols_fwd16_kernel<11>)
    SETA(fft_cols_fwd16_kernel<12>) SETA(fft_cols_fwd16_kernel<13>)
#define SETB(L) SETA((fft_cols_inv16_kernel<L, false>)) SETA((fft_cols_inv16_kernel<L, true>))
    SETB(9) SETB(10) SETB(11) SETB(12) SETB(13)
#undef SETB
#undef SETA
    return cudaSuccess;
}

static FftArgs fft_args(const void *const in[3], void *const out[3], const cd *tw, int D, int per_block,
                        int inverse, double scale) {
    FftArgs a;
    for (int f = 0; f < 3; ++f) { a.in[f] = in[f]; a.out[f] = out[f]; }
    a.twiddle = tw;
    a.D = D;
    a.log2D = ilog2(D);
    a.per_block = per_block;
    a.inverse = inverse;
    a.half_out = 0;
    a.scale = scale;
    return a;
}

// radix-16 row kernels for 512 <= D <= 8192 (REXI_FFT_R16=0 in the environment selects the
// radix-8 row kernels instead: a measurement knob)
static bool fft16_rows(int lg) {
    static const int off = [] { const char *v = getenv("REXI_FFT_R16"); return v && atoi(v) == 0; }();
    return !off && lg >= 9 && lg <= 13;
}

// radix-16 column kernels for 512 <= D <= 8192 (REXI_FFT_C16=0 selects the radix-8 ones)
static bool fft16_cols(int lg) {
    static const int off = [] { const char *v = getenv("REXI_FFT_C16"); return v && atoi(v) == 0; }();
    // measured (profiles/r02n_fft16.log): radix-16 columns lose at 512^2 (19.5 vs 17.9 us
    // forward), win from 1024^2 on (-14 % at 1024^2, -22 % at 4096^2 with the radix-16 rows)
    return !off && lg >= 10 && lg <= 13;
}

// cluster column kernels (fft_cols_cl_kernel) for D = 2048, 4096 (REXI_FFT_CL=0 selects the
// single-CTA radix-16 ones; measured tools/time_fft.py, profiles/r02w_fft_cl.log: 4096^2 forward
// 388 -> 288 us, inverse 358 -> 303 us on the apply path, 2048^2 -7 %; at 1024^2 the L2-resident
// passes are latency-bound and gain nothing, at 8192^2 a cluster's 128 KB per CTA leaves one CTA
// per SM); false also if this device cannot launch them
// cluster width 8, one (n2, column) item per thread. Measured slower (ncu, 4096^2,
// profiles/r02z_fft_cl_width.md): 16-wide clusters with 256-byte segments (forward 338 vs 286 us,
// inverse 322 vs 283 us) and two items per thread at three CTAs per SM (313 / 299 us).
constexpr int kColClWidth = 8, kColClItems = 1;
static bool fft_cl_cols(int lg) {
    static const int off = [] { const char *v = getenv("REXI_FFT_CL"); return v && atoi(v) == 0; }();
    static int ok = -1;
    if (ok < 0) {
        ok = 1;
#define SETCL(L, N, I)                                                                                   \
    for (cudaError_t e :                                                                                 \
         {cudaFuncSetAttribute(fft_cols_cl_kernel<L, 0, N, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)ColCl<L, N, I>::SMEM),                                               \
          cudaFuncSetAttribute(fft_cols_cl_kernel<L, 1, N, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)ColCl<L, N, I>::SMEM),                                               \
          cudaFuncSetAttribute(fft_cols_cl_kernel<L, 2, N, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                               (int)ColCl<L, N, I>::SMEM)})                                              \
        if (e != cudaSuccess) ok = 0;
        SETCL(11, kColClWidth, kColClItems) SETCL(12, kColClWidth, kColClItems)
#undef SETCL
        cudaGetLastError();
    }
    return !off && ok && lg >= 11 && lg <= 12;
}

static cudaError_t launch_cols_cl(int mode, const void *const i3[3], void *const o3[3], const cd *tw, int D,
                                  double scale, cudaStream_t st, bool half_out) {
    constexpr int n1 = kColClWidth;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D / 2, 3);   // (H / n1 column groups) x n1 CTAs, fields
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = n1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FftArgs a = fft_args(i3, o3, tw, D, n1, mode ? 1 : 0, scale);
    a.half_out = half_out ? 1 : 0;
#define COLCL(L, N, I)                                                                                   \
    if (D == (1 << L) && ipt == I) {                                                                     \
        cfg.blockDim = dim3(ColCl<L, N, I>::T);                                                          \
        cfg.dynamicSmemBytes = ColCl<L, N, I>::SMEM;                                                     \
        if (mode == 0) return cudaLaunchKernelEx(&cfg, fft_cols_cl_kernel<L, 0, N, I>, a);               \
        if (mode == 1) return cudaLaunchKernelEx(&cfg, fft_cols_cl_kernel<L, 1, N, I>, a);               \
        return cudaLaunchKernelEx(&cfg, fft_cols_cl_kernel<L, 2, N, I>, a);                              \
    }
    constexpr int ipt = kColClItems;
    COLCL(11, kColClWidth, kColClItems) COLCL(12, kColClWidth, kColClItems)
#undef COLCL
    return cudaErrorInvalidValue;
}

// mode 0: forward; 1: inverse of a Hermitian spectrum; 2: inverse, symmetrising
static cudaError_t launch_cols16(int mode, const void *const i3[3], void *const o3[3], const cd *tw, int D,
                                 double scale, cudaStream_t st, bool half_out = false) {
#define COLS16(L)                                                                                        \
    if (D == (1 << L)) {                                                                                 \
        using CL = Col16<L>;                                                                             \
        FftArgs a = fft_args(i3, o3, tw, D, CL::C, mode ? 1 : 0, scale);                                \
        a.half_out = half_out ? 1 : 0;                                                                   \
        const dim3 grid((D / 2) / CL::C, 3);                                                             \
        const size_t sm = (size_t)CL::C * CL::STRIDE * sizeof(cd);                                      \
        if (mode == 0) fft_cols_fwd16_kernel<L><<<grid, CL::C * CL::T, sm, st>>>(a);                     \
        else if (mode == 1) fft_cols_inv16_kernel<L, false><<<grid, CL::C * CL::T, sm, st>>>(a);         \
        else fft_cols_inv16_kernel<L, true><<<grid, CL::C * CL::T, sm, st>>>(a);                         \
        return cudaGetLastError();                                                                       \
    }
    COLS16(9) COLS16(10) COLS16(11) COLS16(12) COLS16(13)
#undef COLS16
    return cudaErrorInvalidValue;
}

static cudaError_t launch_rows16(bool fwd, const void *const i3[3], void *const o3[3], const cd *tw, int D,
                                 cudaStream_t st) {
#define ROWS16(L)                                                                                        \
    if (D == (1 << L)) {                                                                                 \
        using RL = Row16<L>;                                                                             \
        const FftArgs a = fft_args(i3, o3, tw, D, RL::NB, fwd ? 0 : 1, 1.0);                            \
        const dim3 grid((D / 2) / RL::NB, 3);                                                            \
        const size_t sm = (size_t)RL::NB * RL::PL * sizeof(cd);                                         \
        if (fwd) fft_rows_fwd16_kernel<L><<<grid, RL::NB * RL::T, sm, st>>>(a);                          \
        else fft_rows_inv16_kernel<L><<<grid, RL::NB * RL::T, sm, st>>>(a);                              \
        return cudaGetLastError();                                                                       \
    }
    ROWS16(9) ROWS16(10) ROWS16(11) ROWS16(12) ROWS16(13)
#undef ROWS16
    return cudaErrorInvalidValue;
}

cudaError_t launch_fft_forward(const double *const in[3], cd *const half[3], cd *const out[3],
                               const cd *tw, int D, double scale, cudaStream_t st, bool half_out) {
    const int tf = D >= 8 ? D / 8 : 1;
    {
        const void *i3[3] = {in[0], in[1], in[2]};
        void *o3[3] = {half[0], half[1], half[2]};
        const int lg = ilog2(D);
        if (fft16_rows(lg)) {
            cudaError_t e = launch_rows16(true, i3, o3, tw, D, st);
            if (e != cudaSuccess) return e;
        } else {
            const FftArgs a = fft_args(i3, o3, tw, D, fft_rows_per_block(D), 0, 1.0);
            const dim3 grid((D / 2) / a.per_block, 3);
            const size_t sm = (size_t)a.per_block * padded_len(D) * sizeof(cd);
            fft_rows_fwd_kernel<<<grid, a.per_block * tf, sm, st>>>(a);
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
        }
    }
    const void *i3[3] = {half[0], half[1], half[2]};
    void *o3[3] = {out[0], out[1], out[2]};
    if (fft_cl_cols(ilog2(D))) return launch_cols_cl(0, i3, o3, tw, D, scale, st, half_out);
    if (fft16_cols(ilog2(D))) return launch_cols16(0, i3, o3, tw, D, scale, st, half_out);
    FftArgs a = fft_args(i3, o3, tw, D, fft_cols_per_block(D), 0, scale);
    a.half_out = half_out ? 1 : 0;
    const dim3 grid((D / 2) / a.per_block, 3);
    const size_t sm = (size_t)a.per_block * col_stride(D, a.per_block) * sizeof(cd);
    fft_cols_fwd_kernel<<<grid, a.per_block * tf, sm, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fft_inverse(const cd *const in[3], cd *const half[3], double *const out[3],
                               bool hermitian, const cd *tw, int D, cudaStream_t st) {
    const int tf = D >= 8 ? D / 8 : 1;
    if (fft_cl_cols(ilog2(D)) || fft16_cols(ilog2(D))) {
        const void *i3[3] = {in[0], in[1], in[2]};
        void *o3[3] = {half[0], half[1], half[2]};
        cudaError_t e = fft_cl_cols(ilog2(D)) ? launch_cols_cl(hermitian ? 1 : 2, i3, o3, tw, D, 1.0, st, false)
                                              : launch_cols16(hermitian ? 1 : 2, i3, o3, tw, D, 1.0, st);
        if (e != cudaSuccess) return e;
    } else {
        const void *i3[3] = {in[0], in[1], in[2]};
        void *o3[3] = {half[0], half[1], half[2]};
        const FftArgs a = fft_args(i3, o3, tw, D, fft_cols_per_block(D), 1, 1.0);
        const dim3 grid((D / 2) / a.per_block, 3);
        const size_t sm = (size_t)a.per_block * col_stride(D, a.per_block) * sizeof(cd);
        if (hermitian) fft_cols_inv_kernel<false><<<grid, a.per_block * tf, sm, st>>>(a);
        else fft_cols_inv_kernel<true><<<grid, a.per_block * tf, sm, st>>>(a);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const void *i3[3] = {half[0], half[1], half[2]};
    void *o3[3] = {out[0], out[1], out[2]};
    if (fft16_rows(ilog2(D))) return launch_rows16(false, i3, o3, tw, D, st);
    const FftArgs a = fft_args(i3, o3, tw, D, fft_rows_per_block(D), 1, 1.0);
    const dim3 grid((D / 2) / a.per_block, 3);
    const size_t sm = (size_t)a.per_block * padded_len(D) * sizeof(cd);
    fft_rows_inv_kernel<<<grid, a.per_block * tf, sm, st>>>(a);
    return cudaGetLastError();
}

// Supported (variant, modes per thread, poles per loop trip, min blocks per SM) instantiations.
// Kernel kinds: 0 = REXII DZ (eta, delta accumulated; zeta rebuilt), 1 = REXII UV,
// 2 = REXI (DZ back-substitution, zeta rebuilt), 3 = REXII DZ3 (all three accumulated),
// 4 = REXII PF (partial fractions: two independent solves of f0; zeta rebuilt),
// 5 = REXII PFH (PF with the delta back-substitution folded into the weights).
#define REXI_POLE_CONFIGS(X)                                                             \
    X(0, 1, 1, 8) X(0, 2, 1, 4) X(0, 2, 1, 5) X(0, 3, 1, 4) X(0, 4, 1, 3) X(0, 4, 1, 4)  \
    X(1, 1, 1, 6) X(1, 2, 1, 3) X(1, 2, 1, 4) X(1, 3, 1, 3) X(1, 4, 1, 2) X(1, 4, 1, 3)  \
    X(2, 1, 1, 8) X(2, 2, 1, 4) X(2, 4, 1, 4) X(2, 4, 1, 5)                               \
    X(3, 1, 1, 8) X(3, 2, 1, 4) X(3, 3, 1, 4) X(3, 4, 1, 2) X(3, 4, 1, 4)                 \
    X(4, 1, 1, 8) X(4, 2, 1, 3) X(4, 2, 1, 4) X(4, 3, 1, 4) X(4, 4, 1, 3) X(4, 4, 1, 4)  \
    X(5, 1, 1, 8) X(5, 2, 1, 3) X(5, 2, 1, 4) X(5, 3, 1, 4) X(5, 4, 1, 3) X(5, 4, 1, 4)  \
    X(5, 1, 2, 6) X(5, 2, 2, 3) X(5, 2, 2, 4) X(5, 4, 2, 2)

int pole_modes_per_block(int mpt) { return kPoleBlock * mpt; }

bool pole_config_supported(int variant, int mpt, int pu, int minb) {
#define X(V, M, U, B) if (variant == V && mpt == M && pu == U && minb == B) return true;
    REXI_POLE_CONFIGS(X)
#undef X
    return false;
}

cudaError_t pole_occupancy(int variant, int mpt, int pu, int minb, int *blocks_per_sm) {
#define X(V, M, U, B)                                                                       \
    if (variant == V && mpt == M && pu == U && minb == B)                                   \
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm,                  \
                                                             pole_kernel<V, M, U, B>,        \
                                                             kPoleBlock, 0);
    REXI_POLE_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t launch_poles(const PoleArgs &a, int variant, int mpt, int pu, int minb, cudaStream_t st) {
    const long mpb = kPoleBlock * mpt;
    const long tiles = (a.n_modes + mpb - 1) / mpb;   // MPT = 4: D^2/4 quads / 128 per block
    dim3 grid((unsigned)tiles, (unsigned)a.n_chunks);
#define X(V, M, U, B)                                                   \
    if (variant == V && mpt == M && pu == U && minb == B) {             \
        pole_kernel<V, M, U, B><<<grid, kPoleBlock, 0, st>>>(a);        \
        return cudaGetLastError();                                      \
    }
    REXI_POLE_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

// R2C pair kernel instantiations: (modes per thread M, poles per loop trip PU, min blocks).
// M = 4: one quad per thread; M = 8: octet items (shared K2, default); M = 16: two quads per
// thread in linear order (eight modes, no K2 sharing; kept for comparison).
#define REXI_R2C_CONFIGS(X) \
    X(4, 1, 4) X(4, 1, 5) X(4, 1, 6) X(4, 2, 3) X(4, 2, 4) X(4, 4, 3) \
    X(8, 1, 2) X(8, 1, 3) X(8, 2, 2) X(8, 3, 2) X(8, 4, 2) X(8, 8, 2) X(8, 2, 3) X(8, 4, 3) X(8, 8, 3) X(16, 2, 2)
#define R2C_KERNEL(M, U, B) pole_kernel_r2c<U, B, ((M) == 4 ? 1 : 2), ((M) == 8)>

bool pole_r2c_supported(int mpt, int pu, int minb) {
#define X(M, U, B) if (mpt == M && pu == U && minb == B) return true;
    REXI_R2C_CONFIGS(X)
#undef X
    return false;
}

long pole_r2c_blocks(int D, int mpt) {
    const long items = r2c_items(D, mpt == 4 ? 1 : 2, mpt == 8);
    return (items + kPoleBlock - 1) / kPoleBlock;
}

cudaError_t pole_r2c_occupancy(int mpt, int pu, int minb, int *blocks_per_sm) {
#define X(M, U, B) if (mpt == M && pu == U && minb == B) \
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, R2C_KERNEL(M, U, B), kPoleBlock, 0);
    REXI_R2C_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t launch_poles_r2c(const PoleArgs &a, int mpt, int pu, int minb, cudaStream_t st) {
    dim3 grid((unsigned)pole_r2c_blocks(a.D, mpt), (unsigned)a.n_chunks);
#define X(M, U, B) if (mpt == M && pu == U && minb == B) { \
    R2C_KERNEL(M, U, B)<<<grid, kPoleBlock, 0, st>>>(a); return cudaGetLastError(); }
    REXI_R2C_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

// Explicit-solve R2C kernel (PFHX, default) instantiations: (poles per loop trip, min blocks);
// octet items only (modes_per_thread 8). min blocks 2, 3: 128-thread blocks; 5, 6: 64-thread
// blocks (10 / 12 warps per SM at <= 200 / <= 168 registers).
#define REXI_R2X_CONFIGS(X) X(1, 2) X(2, 2) X(4, 2) X(8, 2) X(1, 3) X(2, 3) X(4, 3) X(8, 3) \
    X(4, 5) X(8, 5) X(4, 6) X(8, 6)

int r2x_block_size(int minb) { return minb >= 5 ? 64 : kPoleBlock; }
long pole_r2x_blocks(int D, int minb) {
    const int bs = r2x_block_size(minb);
    return (r2c_items(D, 2, true) + bs - 1) / bs;
}

bool pole_r2x_supported(int mpt, int pu, int minb) {
    if (mpt != 8) return false;
#define X(U, B) if (pu == U && minb == B) return true;
    REXI_R2X_CONFIGS(X)
#undef X
    return false;
}

#define R2X_KERNEL(U, B) pole_kernel_r2x<U, B, (B >= 5 ? 64 : kPoleBlock)>

cudaError_t pole_r2x_occupancy(int pu, int minb, int *blocks_per_sm) {
#define X(U, B) if (pu == U && minb == B) \
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, R2X_KERNEL(U, B), r2x_block_size(B), 0);
    REXI_R2X_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

// REXI_R2X_BULK=0 selects the register-staged pole-table copy instead of the bulk-copy kernel
// (measurement only)
static bool r2x_bulk_enabled() {
    static const bool on = [] {
        const char *e = getenv("REXI_R2X_BULK");
        return !(e && e[0] == '0');
    }();
    return on;
}


cudaError_t launch_poles_r2x(const PoleArgs &a, int pu, int minb, cudaStream_t st) {
    dim3 grid((unsigned)pole_r2x_blocks(a.D, minb), (unsigned)a.n_chunks);
    if (pu == 8 && minb == 2 && r2x_bulk_enabled()) {
        pole_kernel_r2x_bulk<8, 2, kPoleBlock><<<grid, kPoleBlock, 0, st>>>(a);
        return cudaGetLastError();
    }
#define X(U, B) if (pu == U && minb == B) { \
    R2X_KERNEL(U, B)<<<grid, r2x_block_size(B), 0, st>>>(a); return cudaGetLastError(); }
    REXI_R2X_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

#define REXI_R2C_SK_CONFIGS(X) X(1) X(2) X(3) X(4) X(8)

cudaError_t launch_poles_r2c_sk(const PoleArgs &a, int pu, int ctas, cudaStream_t st) {
#define X(U) if (pu == U) { pole_kernel_r2c_sk<U><<<ctas, kSkBlock, 0, st>>>(a); return cudaGetLastError(); }
    REXI_R2C_SK_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

cudaError_t pole_r2c_sk_occupancy(int pu, int *blocks_per_sm) {
#define X(U) if (pu == U) \
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, pole_kernel_r2c_sk<U>, kSkBlock, 0);
    REXI_R2C_SK_CONFIGS(X)
#undef X
    return cudaErrorInvalidValue;
}

long pole_r2c_sk_tiles(int D) { return (r2c_items(D, 2, true) + kSkBlock - 1) / kSkBlock; }

long sk_slots_bound(long tiles, long poles, long ctas) {
    // segments of one tile <= ceil(poles / floor(W / P)) + 1
    const long per = tiles * poles / ctas;
    return per > 0 ? (poles + per - 1) / per + 1 : -1;
}

cudaError_t launch_finish_r2c_sk(const FinishArgs &a, cudaStream_t st) {
    const long threads = a.sk_tiles * 4 * kSkBlock;
    finish_r2c_sk_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_finish(const FinishArgs &a, cudaStream_t st) {
    const long blocks = (a.n_modes + 255) / 256;
    finish_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Rows l = D/2 + 1 .. D - 1 of a Hermitian spectrum from rows 1 .. D/2 - 1: F(l, k) =
// conj F(D - l, (D - k) mod D). One thread per (field, mirrored mode); rows 0 and D/2 are
// self-mirror rows and are left as they are.
__global__ void __launch_bounds__(256) mirror_rows_kernel(cd *__restrict__ acc, long n_modes, int D, int log2D) {
    const long per = (long)(D / 2 - 1) << log2D;   // mirrored modes per field
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 3 * per) return;
    const int f = (int)(t / per);
    const long r = t - (long)f * per;
    const int l = D / 2 + 1 + (int)(r >> log2D), k = (int)(r & (D - 1));
    const long src = ((long)(D - l) << log2D) + ((D - k) & (D - 1));
    const cd x = acc[f * n_modes + src];
    acc[f * n_modes + ((long)l << log2D) + k] = mk(x.x, -x.y);
}

cudaError_t launch_mirror_rows(cd *acc, long n_modes, int D, cudaStream_t st) {
    const long work = 3L * (D / 2 - 1) * D;
    if (work <= 0) return cudaSuccess;
    mirror_rows_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(acc, n_modes, D, ilog2(D));
    return cudaGetLastError();
}

cudaError_t launch_hermitian(const cd *in, cd *out, long n_modes, int D, cudaStream_t st) {
    hermitian_kernel<<<(unsigned)((n_modes + 255) / 256), 256, 0, st>>>(in, out, n_modes, D, ilog2(D));
    return cudaGetLastError();
}

cudaError_t launch_fixup_k0(const FixupArgs &a, cudaStream_t st, bool beside_pole_kernel) {
    if (beside_pole_kernel) fixup_k0_kernel<128><<<4, 128, 0, st>>>(a);
    else fixup_k0_kernel<1024><<<4, 1024, 0, st>>>(a);
    return cudaGetLastError();
}

// ----------------------------------------------------------------------------- fused small-grid step
#define REXI_SMALL_LOGD(X) X(2) X(3) X(4) X(5) X(6) X(7)

long small_step_items(int D) { return r2c_items(D, 2, true); }

// DSMEM step (step_small2_kernel): shared memory per CTA for cluster size cs; the cluster size
// (16 where the device allows the non-portable size, else 8; 0: no cluster launch) and how many
// such clusters can be resident at once. Cached per process.
size_t small2_smem(int D, int cs) { return (size_t)small2_layout(D, cs).total * sizeof(cd); }

static int g_small2_cs = -1, g_small2_resident = 0;
int small2_cluster(int *resident) {
    if (g_small2_cs < 0) {
        g_small2_cs = 0;
        bool ok = true;
#define X(L)                                                                                                  \
    cudaFuncSetAttribute(step_small2_kernel<L, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);        \
    if (cudaFuncSetAttribute(step_small2_kernel<L, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,           \
                             (int)small2_smem(1 << L, 16)) != cudaSuccess ||                                   \
        cudaFuncSetAttribute(step_small2_kernel<L, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,            \
                             (int)small2_smem(1 << L, 8)) != cudaSuccess)                                      \
        ok = false;
        REXI_SMALL_LOGD(X)
#undef X
        cudaGetLastError();
        for (int want : {16, 8}) {
            if (!ok) break;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(want);
            cfg.blockDim = dim3(kSmallThreads);
            cfg.dynamicSmemBytes = small2_smem(128, want);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = want;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            const cudaError_t e = want == 16 ? cudaOccupancyMaxActiveClusters(&nclusters, step_small2_kernel<7, 16>, &cfg)
                                             : cudaOccupancyMaxActiveClusters(&nclusters, step_small2_kernel<7, 8>, &cfg);
            if (e == cudaSuccess && nclusters >= 1) {
                g_small2_cs = want;
                g_small2_resident = nclusters;
                break;
            }
            cudaGetLastError();
        }
    }
    if (resident) *resident = g_small2_resident;
    return g_small2_cs;
}

cudaError_t launch_step_small2(const SmallArgs &a, int cs, cudaStream_t st) {
    if (a.n_clusters < 1 || a.n_clusters > kSmallMaxClusters || (cs != 16 && cs != 8)) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * a.n_clusters);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = small2_smem(a.pole.D, cs);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
#define X(L)                                                                                         \
    if (a.pole.log2D == L)                                                                           \
        return cs == 16 ? cudaLaunchKernelEx(&cfg, step_small2_kernel<L, 16>, a)                     \
                        : cudaLaunchKernelEx(&cfg, step_small2_kernel<L, 8>, a);
    REXI_SMALL_LOGD(X)
#undef X
    return cudaErrorInvalidValue;
}

// ----------------------------------------------------------------------------- 1-D transforms (NEXT-3)
// The length-n DFT of one complex vector, out[j] = scale * sum_k in[k] e^{-+2 pi i j k / n}, for
// the circulant test matrices of Sec. 3.2 (rexi_circulant_apply): power-of-two n <= 2048 through
// the radix-8 Stockham passes of the 2-D transforms (one block, twiddles from a table made by
// sincospi), any other n by a direct DFT (one thread per output, index j k reduced mod n exactly).
__global__ void twiddle_table_kernel(cd *tw, int n) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double sn, cs;
    sincospi(-2.0 * (double)j / (double)n, &sn, &cs);
    tw[j] = mk(cs, sn);
}

template <bool INV>
__global__ void __launch_bounds__(256) fft1d_kernel(const cd *__restrict__ in, cd *__restrict__ out, int n,
                                                    int logn, double scale, const cd *__restrict__ tw) {
    extern __shared__ cd smem[];
    rx_poison_smem();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        RX_SMEM(pidx(i));
        smem[pidx(i)] = in[i];
    }
    __syncthreads();
    const int tf = n >= 8 ? n / 8 : 1;
    fft_in_smem<INV>(smem, n, logn, (int)threadIdx.x, tf, tw, (int)threadIdx.x < tf);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const cd v = smem[pidx(i)];
        out[i] = mk(v.x * scale, v.y * scale);
    }
}

__global__ void __launch_bounds__(256) dft1d_direct_kernel(const cd *__restrict__ in, cd *__restrict__ out, long n,
                                                           int sign, double scale) {
    const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double ar = 0.0, ai = 0.0;
    long idx = 0;   // (j * k) mod n, advanced by j each step (exact integers)
    for (long k = 0; k < n; ++k) {
        double sn, cs;
        sincospi((double)sign * 2.0 * (double)idx / (double)n, &sn, &cs);
        const cd x = in[k];
        ar = fma(x.x, cs, fma(-x.y, sn, ar));
        ai = fma(x.x, sn, fma(x.y, cs, ai));
        idx += j;
        if (idx >= n) idx -= n;
    }
    out[j] = mk(ar * scale, ai * scale);
}

bool dft1d_uses_fft(long n) { return n >= 2 && n <= 2048 && (n & (n - 1)) == 0; }

cudaError_t launch_twiddles(cd *tw, int n, cudaStream_t st) {
    twiddle_table_kernel<<<(n + 255) / 256, 256, 0, st>>>(tw, n);
    return cudaGetLastError();
}

// in != out required; tw: table of n entries (launch_twiddles) when dft1d_uses_fft(n)
cudaError_t launch_dft1d(const cd *in, cd *out, long n, bool inverse, double scale, const cd *tw, cudaStream_t st) {
    if (dft1d_uses_fft(n)) {
        const int nn = (int)n;
        const int threads = std::max(32, std::min(256, nn / 8));
        const size_t sm = (size_t)padded_len(nn) * sizeof(cd);
        if (inverse) fft1d_kernel<true><<<1, threads, sm, st>>>(in, out, nn, ilog2(nn), scale, tw);
        else fft1d_kernel<false><<<1, threads, sm, st>>>(in, out, nn, ilog2(nn), scale, tw);
        return cudaGetLastError();
    }
    dft1d_direct_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, n, inverse ? 1 : -1, scale);
    return cudaGetLastError();
}

}  // namespace rexi
