// scalar.cu — NEXT-3: the rational approximations applied to a diagonalised operator.
//
// For A = V E V^{-1} with purely imaginary eigenvalues (eq:AisVEV..eq:REXI_VEV_DECOMP,
// PAPER.md:232-259) every scalar form is evaluated per eigenvalue i x_j and multiplied into
// the eigen-coordinates in_j of the vector: out_j = phase * r(i x_j) * in_j, with
//   REXII  (eq:modifiedRexi):
//       r = sum_{n=-N}^{N} (c_{1,n} h mu + c_{2,n}(x + h n)) / ((alpha_{-n} - i x)(alpha_n + i x)),
//   REXI   (eq:originalRexi; REXIE, eq:REXIE, when V is real):
//       r = sum_n Re(beta^Re_n / (i x + alpha_n)) + i Re(beta^Im_n / (i x + alpha_n)),
//   REXI-M (the per-eigenvalue sum of eq:originalREXImatrix for a real A, before its Re):
//       r = sum_n beta^Re_n / (i x + alpha_n)  (the caller takes Re of the vector afterwards).
// A spectral shift (Remark 1) is the caller's x_j - nu and phase e^{tau nu}.
// One block per eigenvalue, threads stride over the 2N+1 terms (each a complex shifted
// "solve" 1/(alpha + i x)), fixed-order tree reduction.
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <new>
#include <string>
#include <vector>

#include "../../include/rexi.h"
#include "kernels.cuh"
#include "launch.h"
#include "planner.h"

using rexi::cd;
using rexi::cmul;
using rexi::mk;

namespace {

constexpr int kScalarBlock = 256;

template <int METHOD>
__global__ void __launch_bounds__(kScalarBlock) scalar_kernel(const rexi::ScalarTerm *__restrict__ t,
                                                              long nt, const double *__restrict__ x,
                                                              const cd *__restrict__ in, cd *out,
                                                              cd phase) {
    __shared__ cd red[kScalarBlock];
    const long j = blockIdx.x;
    const double xj = x[j];
    cd acc = mk(0, 0);
    for (long i = threadIdx.x; i < nt; i += kScalarBlock) {
        const rexi::ScalarTerm T = t[i];
        // d = alpha_n + i x ; 1/d = conj(d)/|d|^2
        const cd d = mk(T.ar, T.ai + xj);
        const double r = 1.0 / fma(d.x, d.x, d.y * d.y);
        const cd q = mk(d.x * r, -d.y * r);
        if (METHOD == REXI_SCALAR_REXII) {
            // (alpha_{-n} - i x)(alpha_n + i x) = |alpha_n + i x|^2 for real x
            const cd num = mk(fma(T.c2r, xj, T.C1r), fma(T.c2i, xj, T.C1i));
            acc = mk(fma(num.x, r, acc.x), fma(num.y, r, acc.y));
        } else if (METHOD == REXI_SCALAR_REXI) {
            const cd a = cmul(mk(T.bRr, T.bRi), q), b = cmul(mk(T.bIr, T.bIi), q);
            acc = mk(acc.x + a.x, acc.y + b.x);
        } else {
            const cd a = cmul(mk(T.bRr, T.bRi), q);
            acc = mk(acc.x + a.x, acc.y + a.y);
        }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kScalarBlock / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            red[threadIdx.x] = mk(red[threadIdx.x].x + red[threadIdx.x + s].x,
                                  red[threadIdx.x].y + red[threadIdx.x + s].y);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = cmul(phase, cmul(red[0], in[j]));
}

// i x_j = tau (lambda_j - nu): x_j = Im(tau (lambda_j - nu)) for real tau (the eigenvalues of
// the circulant are purely imaginary up to rounding; their real part is dropped).
__global__ void eig_to_x_kernel(const cd *__restrict__ lam, double *__restrict__ x, long n, double tau,
                                double nu_im) {
    const long j = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) x[j] = tau * (lam[j].y - nu_im);
}

}  // namespace

struct rexi_scalar_plan_s {
    int device = 0;
    double h = 0;
    long M = 0, N = 0;
    rexi::ScalarTerm *d_terms = nullptr;
    ~rexi_scalar_plan_s() {
        if (d_terms) cudaFree(d_terms);
    }
};

static rexi_status_t sfail(rexi_status_t s, const char *msg) {
    rexi::set_last_error(msg);
    return s;
}

extern "C" {

rexi_status_t rexi_scalar_plan_create(rexi_scalar_plan_t *out, double h, long M, int device) {
    if (!out) return sfail(REXI_EINVAL, "out is NULL");
    *out = nullptr;
    std::vector<rexi::ScalarTerm> terms;
    std::vector<char> err;
    int st;
    try {
        st = rexi::make_scalar_terms(terms, h, M, err);
    } catch (...) {
        return sfail(REXI_ENOMEM, "scalar term table allocation failed");
    }
    if (st != REXI_OK) return sfail((rexi_status_t)st, err.empty() ? "invalid h or M" : err.data());
    rexi_scalar_plan_s *p = new (std::nothrow) rexi_scalar_plan_s();
    if (!p) return sfail(REXI_ENOMEM, "host allocation failed");
    p->device = device;
    p->h = h;
    p->M = M;
    p->N = (long)(terms.size() - 1) / 2;
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) {
        delete p;
        cudaGetLastError();
        return sfail(REXI_ECUDA, "cudaSetDevice failed");
    }
    cudaError_t e = cudaMalloc((void **)&p->d_terms, sizeof(rexi::ScalarTerm) * terms.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_terms, terms.data(), sizeof(rexi::ScalarTerm) * terms.size(),
                       cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        delete p;
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? sfail(REXI_ENOMEM, "cudaMalloc (scalar terms) failed")
                                              : sfail(REXI_ECUDA, cudaGetErrorString(e));
    }
    *out = p;
    return REXI_OK;
}

rexi_status_t rexi_scalar_plan_destroy(rexi_scalar_plan_t p) {
    if (!p) return sfail(REXI_EINVAL, "null scalar plan");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    delete p;
    cudaSetDevice(prev);
    return REXI_OK;
}

long rexi_scalar_plan_terms(rexi_scalar_plan_t p) { return p ? 2 * p->N + 1 : -1; }

rexi_status_t rexi_scalar_apply(rexi_scalar_plan_t p, int method, long n, const double *x,
                                const double *in, double *out, double phase_re, double phase_im,
                                void *stream) {
    if (!p || n < 0 || (n > 0 && (!x || !in || !out))) return sfail(REXI_EINVAL, "null plan/pointer or n < 0");
    if (method != REXI_SCALAR_REXII && method != REXI_SCALAR_REXI && method != REXI_SCALAR_REXI_M)
        return sfail(REXI_EINVAL, "unknown scalar method");
    if (n == 0) return REXI_OK;
    if (n > 0x7fffffffL) return sfail(REXI_EINVAL, "n exceeds the grid limit (2^31 - 1)");
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(p->device) != cudaSuccess) {
        cudaGetLastError();
        return sfail(REXI_ECUDA, "cudaSetDevice failed");
    }
    const long nt = 2 * p->N + 1;
    const cd ph = cd{phase_re, phase_im};
    const cd *cin = reinterpret_cast<const cd *>(in);
    cd *cout = reinterpret_cast<cd *>(out);
    cudaStream_t st = (cudaStream_t)stream;
    if (method == REXI_SCALAR_REXII)
        scalar_kernel<REXI_SCALAR_REXII><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, cin, cout, ph);
    else if (method == REXI_SCALAR_REXI)
        scalar_kernel<REXI_SCALAR_REXI><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, cin, cout, ph);
    else
        scalar_kernel<REXI_SCALAR_REXI_M><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, cin, cout, ph);
    cudaError_t e = cudaGetLastError();
    cudaSetDevice(prev);
    return e == cudaSuccess ? REXI_OK : sfail(REXI_ECUDA, cudaGetErrorString(e));
}

rexi_status_t rexi_circulant_apply(rexi_scalar_plan_t p, int method, long n, const double *col,
                                   const double *f, double *out, double tau, double nu_re,
                                   double nu_im, void *stream) {
    if (!p || n < 1 || !col || !f || !out) return sfail(REXI_EINVAL, "null plan/pointer or n < 1");
    if (method != REXI_SCALAR_REXII && method != REXI_SCALAR_REXI && method != REXI_SCALAR_REXI_M)
        return sfail(REXI_EINVAL, "unknown scalar method");
    if (n > (1L << 20)) return sfail(REXI_EINVAL, "n > 2^20");
    if (!std::isfinite(tau) || !std::isfinite(nu_re) || !std::isfinite(nu_im))
        return sfail(REXI_EINVAL, "tau and nu must be finite");
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(p->device) != cudaSuccess) {
        cudaGetLastError();
        return sfail(REXI_ECUDA, "cudaSetDevice failed");
    }
    cudaStream_t st = (cudaStream_t)stream;
    // stream-ordered scratch: lambda, fh, out-hat (n complex each), x (n doubles), twiddles (n)
    void *work = nullptr;
    const size_t bytes = sizeof(cd) * (size_t)n * 4 + sizeof(double) * (size_t)n;
    cudaError_t e = cudaMallocAsync(&work, bytes, st);
    if (e == cudaSuccess) {
        cd *lam = static_cast<cd *>(work), *fh = lam + n, *oh = fh + n, *tw = oh + n;
        double *x = reinterpret_cast<double *>(tw + n);
        const bool fft = rexi::dft1d_uses_fft(n);
        // e^{tau nu}: the phase of Remark 1's shift
        const std::complex<double> ph = std::exp(tau * std::complex<double>(nu_re, nu_im));
        if (fft) e = rexi::launch_twiddles(tw, (int)n, st);
        if (e == cudaSuccess) e = rexi::launch_dft1d(reinterpret_cast<const cd *>(col), lam, n, false, 1.0, tw, st);
        if (e == cudaSuccess) e = rexi::launch_dft1d(reinterpret_cast<const cd *>(f), fh, n, false, 1.0, tw, st);
        if (e == cudaSuccess) {
            eig_to_x_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lam, x, n, tau, nu_im);
            e = cudaGetLastError();
        }
        const long nt = 2 * p->N + 1;
        const cd phc = cd{ph.real(), ph.imag()};
        if (e == cudaSuccess) {
            if (method == REXI_SCALAR_REXII)
                scalar_kernel<REXI_SCALAR_REXII><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, fh, oh, phc);
            else if (method == REXI_SCALAR_REXI)
                scalar_kernel<REXI_SCALAR_REXI><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, fh, oh, phc);
            else
                scalar_kernel<REXI_SCALAR_REXI_M><<<(unsigned)n, kScalarBlock, 0, st>>>(p->d_terms, nt, x, fh, oh, phc);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess)
            e = rexi::launch_dft1d(oh, reinterpret_cast<cd *>(out), n, true, 1.0 / (double)n, tw, st);
        cudaError_t ef = cudaFreeAsync(work, st);
        if (e == cudaSuccess) e = ef;
    }
    cudaSetDevice(prev);
    return e == cudaSuccess ? REXI_OK : sfail(REXI_ECUDA, cudaGetErrorString(e));
}

}  // extern "C"
