// kernels.cu — device kernels of librexi (sm_100a, fp64).
//
//  * fft_rows_kernel / fft_cols_kernel : batched radix-2 FFT passes in shared memory
//    (S1 forward transform, S5 inverse transform + Re). PAPER.md:497 "all computations
//    ... in Fourier space"; Alg. 1 lines 1 and last.
//  * pole_kernel<VARIANT>             : S2 + S3, the fused per-mode two-solve REXII pole
//    loop with the weighted accumulation in registers (eq:lswEta,
//    eq:lswVelocities). No per-pole solution ever reaches HBM.
//  * finish_kernel                    : fixed-order sum of the per-chunk partial sums and,
//    for the DZ variant, recovery of (u, v) from the accumulated (delta, zeta).
//  * fixup_k0_kernel                  : the K = 0 modes for the DZ variant (velocities
//    decouple from delta, zeta there): pure Coriolis 2x2 solves per pole.
#include "kernels.cuh"
#include "launch.h"

namespace rexi {

// ============================================================================= FFT
__device__ __forceinline__ int bitrev(int x, int log2n) {
    return (int)(__brev((unsigned)x) >> (32 - log2n));
}

// In-place iterative radix-2 DIT on `nfft` arrays of length D stored at s + f*stride,
// input already in bit-reversed order. Twiddle w_len^pos = tw[pos * D/len].
__device__ __forceinline__ void fft_stages(cd *s, int stride, int D, int log2D, int nfft,
                                           const cd *__restrict__ tw, int inverse) {
    const int halfD = D >> 1;
    const int nb = nfft * halfD;
    for (int lh = 1; lh <= log2D; ++lh) {
        const int half = 1 << (lh - 1);
        const int tstride = D >> lh;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int f = b >> (log2D - 1);
            const int bb = b & (halfD - 1);
            const int grp = bb >> (lh - 1);
            const int pos = bb & (half - 1);
            const int i0 = f * stride + (grp << lh) + pos;
            const int i1 = i0 + half;
            const double2 tw2 = __ldg(reinterpret_cast<const double2 *>(tw) + pos * tstride);
            cd w = mk(tw2.x, tw2.y);
            if (inverse) w.y = -w.y;
            const cd u = s[i0];
            const cd t = cmul(s[i1], w);
            s[i0] = mk(u.x + t.x, u.y + t.y);
            s[i1] = mk(u.x - t.x, u.y - t.y);
        }
        __syncthreads();
    }
}

// One block = `per_block` consecutive rows of one field. grid = (D/per_block, 3).
template <bool REAL_IN, bool REAL_OUT>
__global__ void __launch_bounds__(256) fft_rows_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, R = a.per_block;
    const size_t row0 = (size_t)blockIdx.x * R;
    const int n = R << log2D;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i >> log2D, x = i & (D - 1);
        const size_t g = (row0 + r) * (size_t)D + x;
        cd v;
        if (REAL_IN) v = mk(static_cast<const double *>(a.in[f])[g], 0.0);
        else v = static_cast<const cd *>(a.in[f])[g];
        smem[(r << log2D) + bitrev(x, log2D)] = v;
    }
    __syncthreads();
    fft_stages(smem, D, D, log2D, R, a.twiddle, a.inverse);
    const double sc = a.scale;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i >> log2D, k = i & (D - 1);
        const size_t g = (row0 + r) * (size_t)D + k;
        const cd v = smem[i];
        if (REAL_OUT) static_cast<double *>(a.out[f])[g] = v.x * sc;
        else static_cast<cd *>(a.out[f])[g] = mk(v.x * sc, v.y * sc);
    }
}

// One block = `per_block` (power of two) consecutive columns of one field; smem rows
// padded to D+1 to spread the transposed accesses over the banks.
__global__ void __launch_bounds__(256) fft_cols_kernel(FftArgs a) {
    extern __shared__ cd smem[];
    const int f = blockIdx.y;
    const int D = a.D, log2D = a.log2D, C = a.per_block;
    const int logC = __ffs(C) - 1;
    const int stride = D + 1;
    const size_t col0 = (size_t)blockIdx.x * C;
    const cd *in = static_cast<const cd *>(a.in[f]);
    cd *out = static_cast<cd *>(a.out[f]);
    const int n = C << log2D;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i >> logC, cc = i & (C - 1);
        smem[cc * stride + bitrev(r, log2D)] = in[(size_t)r * D + col0 + cc];
    }
    __syncthreads();
    fft_stages(smem, stride, D, log2D, C, a.twiddle, a.inverse);
    const double sc = a.scale;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int r = i >> logC, cc = i & (C - 1);
        const cd v = smem[cc * stride + r];
        out[(size_t)r * D + col0 + cc] = mk(v.x * sc, v.y * sc);
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
#ifndef REXI_POLE_BLOCK
#define REXI_POLE_BLOCK 128
#endif
constexpr int kPoleBlock = REXI_POLE_BLOCK;
constexpr int kPoleTile = 32;

struct ModeState {
    cd e0, B0, m0, ua, vb;   // f0 = (e0, ua, vb); B0 = h mu e0 + delta0; m0 = zeta0 - c e0
    double K2, Kx, Ky;
    cd A0, A1, A2;           // accumulators: (eta, delta, zeta) [DZ] or (eta, u, v) [UV]
};

// One pole, one mode: both shifted solves and the weighted accumulation.
template <int VARIANT>
__device__ __forceinline__ void pole_body(const PoleConst &P, ModeState &s, const double c) {
    const cd al = mk(P.ar, P.ai), s2 = mk(P.s2r, P.s2i), s1c = mk(P.s1cr, P.s1ci);
    const cd w1 = mk(P.w1r, P.w1i), w2 = mk(P.w2r, P.w2i);
    const double hn = P.ai;
    // ---- solve 1: Helmholtz for eta1 (eq:lswEta)
    const cd t = mk(fma(-hn, s.e0.y, s.B0.x), fma(hn, s.e0.x, s.B0.y));
    const cd num = cfms(s2, s.m0, t);
    const double dr = P.kr + s.K2;
    const double r = rcp_pos(fma(dr, dr, P.ki2));
    const cd qd = mk(dr * r, -P.ki * r);                        // 1/(kappa + K2)
    const cd eta1 = cmul(num, qd);
    if (VARIANT == 0) {
        const cd ia = mk(P.iar, P.iai);
        const cd del1 = cfma(al, eta1, mk(-s.e0.x, -s.e0.y));
        const cd zet1 = cfma(ia, s.m0, mk(c * eta1.x, c * eta1.y));
        // ---- solve 2
        cd num2 = cfma(s1c, eta1, mk(-del1.x, -del1.y));
        num2 = cjfms(s2, zet1, num2);                            // - conj(c/alpha) zeta1
        const cd eta2 = cjfma(qd, num2, mk(0, 0));               // num2 * conj(q)
        const cd del2 = cjfms(al, eta2, eta1);                   // eta1 - conj(alpha) eta2
        const cd zet2 = mk(fma(P.ia2, s.m0.x, c * eta2.x), fma(P.ia2, s.m0.y, c * eta2.y));
        // ---- accumulate w1 g1 + w2 g2
        s.A0 = cfma(w2, eta2, cfma(w1, eta1, s.A0));
        s.A1 = cfma(w2, del2, cfma(w1, del1, s.A1));
        s.A2 = cfma(w2, zet2, cfma(w1, zet1, s.A2));
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

// grid = (mode tiles of kPoleBlock * MPT modes, pole chunks). Each thread owns MPT modes and
// runs every pole of its chunk, PU poles per loop trip. MINB = resident blocks per SM asked
// of ptxas (register budget 65536 / (kPoleBlock * MINB) per thread).
template <int VARIANT, int MPT, int PU, int MINB>
__global__ void __launch_bounds__(kPoleBlock, MINB)
pole_kernel(PoleArgs a) {
    __shared__ PoleConst sp[kPoleTile];
    const long n_modes = a.n_modes;
    const long tile0 = (long)blockIdx.x * (kPoleBlock * MPT);
    const int chunk = blockIdx.y;
    const long len = a.pole_end - a.pole_begin;
    const long p0 = a.pole_begin + len * chunk / a.n_chunks;
    const long p1 = a.pole_begin + len * (chunk + 1) / a.n_chunks;
    double c = a.tau;
#if REXI_C_IN_REG
    asm volatile("mov.b64 %0, %0;" : "+d"(c));   // keep c in a per-thread register
#endif
    const double hmu = a.hmu;

    ModeState st[MPT];
#pragma unroll
    for (int j = 0; j < MPT; ++j) {
        const long m = tile0 + j * kPoleBlock + threadIdx.x;
        const long mm = m < n_modes ? m : 0;
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
            for (int i = threadIdx.x; i < cnt * 10; i += kPoleBlock) dst[i] = src[i];
        }
        __syncthreads();
        int q = 0;
#pragma unroll 1
        for (; q + PU <= cnt; q += PU) {
#if REXI_ABLATE_LDS
            // timing ablation only (wrong results): constants stay in registers
            const PoleConst Pr = sp[0];
#pragma unroll
            for (int u = 0; u < PU; ++u)
#pragma unroll
                for (int j = 0; j < MPT; ++j) pole_body<VARIANT>(Pr, st[j], c);
#else
#pragma unroll
            for (int u = 0; u < PU; ++u)
#pragma unroll
                for (int j = 0; j < MPT; ++j) pole_body<VARIANT>(sp[q + u], st[j], c);
#endif
        }
        if (PU > 1) {
#pragma unroll 1
            for (; q < cnt; ++q)
#pragma unroll
                for (int j = 0; j < MPT; ++j) pole_body<VARIANT>(sp[q], st[j], c);
        }
    }
    cd *out = a.partial + (size_t)chunk * 3 * n_modes;
#pragma unroll
    for (int j = 0; j < MPT; ++j) {
        const long m = tile0 + j * kPoleBlock + threadIdx.x;
        if (m < n_modes) {
            out[m] = st[j].A0;
            out[n_modes + m] = st[j].A1;
            out[2 * n_modes + m] = st[j].A2;
        }
    }
}

// ============================================================================= finish
__global__ void __launch_bounds__(256) finish_kernel(FinishArgs a) {
    const long m = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long n = a.n_modes;
    if (m >= n) return;
    cd s0 = mk(0, 0), s1 = mk(0, 0), s2 = mk(0, 0);
    for (int c = 0; c < a.n_chunks; ++c) {  // fixed order: deterministic
        const cd *p = a.partial + (size_t)c * 3 * n;
        const cd x0 = p[m], x1 = p[n + m], x2 = p[2 * n + m];
        s0 = mk(s0.x + x0.x, s0.y + x0.y);
        s1 = mk(s1.x + x1.x, s1.y + x1.y);
        s2 = mk(s2.x + x2.x, s2.y + x2.y);
    }
    if (a.variant == 0) {
        const int l = (int)(m >> a.log2D), k = (int)(m & (a.D - 1));
        const double kx = a.ksym[k], ky = a.ksym[l];
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

// ============================================================================= K = 0 modes (DZ)
// Modes with Kx = Ky = 0: (0,0), (0,D/2), (D/2,0), (D/2,D/2). There tau A only couples u, v
// through Coriolis: (u1,v1) = kappa^-1 [[alpha,-c],[c,alpha]] (a,b) (eq:lswVelocities with
// grad eta = 0) and (u2,v2) = conj(kappa)^-1 [[conj alpha, c],[-c, conj alpha]] (u1,v1).
constexpr int kFixBlock = 256;
__global__ void __launch_bounds__(kFixBlock) fixup_k0_kernel(FixupArgs a) {
    __shared__ cd red[2][kFixBlock];
    const int D = a.D, H = D / 2;
    const int ls[4] = {0, 0, H, H}, ks[4] = {0, H, 0, H};
    const long m = (long)ls[blockIdx.x] * D + ks[blockIdx.x];
    const long n = a.n_modes;
    const cd ua = a.fhat[n + m], vb = a.fhat[2 * n + m];
    cd Au = mk(0, 0), Av = mk(0, 0);
    for (long p = a.pole_begin + threadIdx.x; p < a.pole_end; p += kFixBlock) {
        const PoleConst P = a.poles[p];
        const cd s3 = mk(P.s3r, P.s3i), s4 = mk(P.s4r, P.s4i);
        const cd w1 = mk(P.w1r, P.w1i), w2 = mk(P.w2r, P.w2i);
        const cd u1 = cfms(s4, vb, cmul(s3, ua));
        const cd v1 = cfma(s3, vb, cmul(s4, ua));
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
        a.acc[n + m] = red[0][0];
        a.acc[2 * n + m] = red[1][0];
    }
}

// ============================================================================= launchers
static int ilog2(int x) {
    int r = 0;
    while ((1 << r) < x) ++r;
    return r;
}

static const int kFftElems = 4096;   // complex elements per FFT block (64 KB of smem)

cudaError_t fft_setup_attributes() {
    cudaError_t e;
    const int maxsm = 200 * 1024;
    if ((e = cudaFuncSetAttribute(fft_rows_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(fft_rows_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(fft_rows_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    if ((e = cudaFuncSetAttribute(fft_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
    return cudaSuccess;
}

cudaError_t launch_fft_rows(const void *const in[3], void *const out[3], bool real_in, bool real_out,
                            const cd *tw, int D, int inverse, double scale, cudaStream_t st) {
    FftArgs a;
    for (int f = 0; f < 3; ++f) { a.in[f] = in[f]; a.out[f] = out[f]; }
    a.twiddle = tw;
    a.D = D;
    a.log2D = ilog2(D);
    a.per_block = D >= kFftElems ? 1 : kFftElems / D;
    if (a.per_block > D) a.per_block = D;
    a.inverse = inverse;
    a.scale = scale;
    dim3 grid(D / a.per_block, 3);
    size_t sm = (size_t)a.per_block * D * sizeof(cd);
    if (real_in && !real_out) fft_rows_kernel<true, false><<<grid, 256, sm, st>>>(a);
    else if (!real_in && real_out) fft_rows_kernel<false, true><<<grid, 256, sm, st>>>(a);
    else fft_rows_kernel<false, false><<<grid, 256, sm, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fft_cols(const void *const in[3], void *const out[3], const cd *tw, int D,
                            int inverse, double scale, cudaStream_t st) {
    FftArgs a;
    for (int f = 0; f < 3; ++f) { a.in[f] = in[f]; a.out[f] = out[f]; }
    a.twiddle = tw;
    a.D = D;
    a.log2D = ilog2(D);
    int C = D >= kFftElems ? 1 : kFftElems / D;
    if (C > 16) C = 16;
    if (C > D) C = D;
    a.per_block = C;
    a.inverse = inverse;
    a.scale = scale;
    dim3 grid(D / C, 3);
    size_t sm = (size_t)C * (D + 1) * sizeof(cd);
    fft_cols_kernel<<<grid, 256, sm, st>>>(a);
    return cudaGetLastError();
}

// Supported (variant, modes per thread, poles per loop trip, min blocks per SM) instantiations.
#define REXI_POLE_CONFIGS(X)                                                             \
    X(0, 1, 1, 8) X(0, 2, 1, 4) X(0, 2, 1, 5) X(0, 2, 2, 3) X(0, 3, 1, 3) X(0, 3, 1, 4)  \
    X(0, 4, 1, 2) X(0, 4, 1, 3) X(0, 4, 1, 4)                                             \
    X(1, 1, 1, 6) X(1, 2, 1, 3) X(1, 2, 1, 4) X(1, 3, 1, 3) X(1, 4, 1, 2) X(1, 4, 1, 3)

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
    const long tiles = (a.n_modes + mpb - 1) / mpb;
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

cudaError_t launch_finish(const FinishArgs &a, cudaStream_t st) {
    const long blocks = (a.n_modes + 255) / 256;
    finish_kernel<<<(unsigned)blocks, 256, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_fixup_k0(const FixupArgs &a, cudaStream_t st) {
    fixup_k0_kernel<<<4, kFixBlock, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace rexi
