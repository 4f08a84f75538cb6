/*
 * rexi_oracle.c — ORACLE, test infrastructure only.
 *
 * A plain, slow, obviously-correct CPU evaluation of one REXII step of the
 * linearised rotating shallow-water equations (arXiv:2008.11607, Sec. 4).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. It shares no code, header,
 * table or constant with the CUDA product path (paper_2008_11607_b200/csrc).
 *
 *  - oracle_dft2_forward / oracle_dft2_inverse_real: the 2-D DFT by its
 *    definition, separable, O(D^3), twiddles cos/sin(2 pi (k x mod D)/D).
 *      Xhat(k,l) = D^-2 sum_{y,x} X[y][x] e^{-2 pi i (k x + l y)/D}
 *    "all computations will be conducted in Fourier space".
 *  - oracle_rexii_pole_sum: for every listed Fourier mode and every pole
 *    n = 0..N of eq:modifiedRexiMatrixReducedSum, the two
 *    shifted systems of PAPER.md:429-435
 *        (A + alpha_n I) g1 = f0 ,   (alpha_{-n} I - A) g2 = g1 ,
 *        g3 = Gamma_n C2_n (g1 + (C1_n/C2_n - alpha_{-n}) g2)
 *    are solved as DENSE 3x3 complex systems by Gaussian elimination with
 *    partial pivoting (deliberately NOT the Helmholtz algebra of eq:lswEta),
 *    and acc += g3, in ascending n. g3 is formed division-free (reading G4):
 *        g3 = Gamma_n ( C2_n g1 + (C1_n - C2_n alpha_{-n}) g2 ).
 *  - oracle_rexi_pole_sum: the original REXI, eq:originalREXImatrix
 *    (PAPER.md:326-330): acc += beta^Re_n (tau A + alpha_n I)^{-1} f0,
 *    n = -N..N, one dense solve per term.
 *
 * Per-mode symbol (Fourier-transformed, tau-scaled per
 * reading G3, Nyquist symbol zeroed per reading G2):
 *     tau*Ahat = [[0, -i Kx, -i Ky], [-i Kx, 0, tau], [-i Ky, -tau, 0]],
 *     Kx = 2 pi k tau, Ky = 2 pi l tau, k = wavenumber of column index.
 *
 * Spectral layout: field-major, then row l (y-wavenumber index), then
 * column k (x-wavenumber index); complex interleaved (re, im) doubles.
 * Physical layout: X[y][x], x fastest.
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static const double TWO_PI = 6.283185307179586476925286766559;

int oracle_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* e^{sign 2 pi i j / D} for j = 0..D-1 */
static cplx *twiddles(int D, double sign)
{
    cplx *w = (cplx *)malloc(sizeof(cplx) * (size_t)D);
    for (int j = 0; j < D; ++j) {
        double th = TWO_PI * (double)j / (double)D;
        w[j] = cos(th) + sign * I * sin(th);
    }
    return w;
}

/* Forward 2-D DFT of one real D x D field: X (real) -> Xhat (complex, scaled by D^-2). */
void oracle_dft2_forward(int D, const double *X, double *Xhat_ri)
{
    cplx *w = twiddles(D, -1.0);
    cplx *tmp = (cplx *)malloc(sizeof(cplx) * (size_t)D * D); /* tmp[y][k] */
    /* pass 1: along x for every row y */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < D; ++y)
        for (int k = 0; k < D; ++k) {
            cplx s = 0;
            for (int x = 0; x < D; ++x)
                s += X[(size_t)y * D + x] * w[((long)k * x) % D];
            tmp[(size_t)y * D + k] = s;
        }
    /* pass 2: along y for every column k */
    const double scale = 1.0 / ((double)D * (double)D);
#pragma omp parallel for schedule(static)
    for (int l = 0; l < D; ++l)
        for (int k = 0; k < D; ++k) {
            cplx s = 0;
            for (int y = 0; y < D; ++y)
                s += tmp[(size_t)y * D + k] * w[((long)l * y) % D];
            s *= scale;
            Xhat_ri[2 * ((size_t)l * D + k)] = creal(s);
            Xhat_ri[2 * ((size_t)l * D + k) + 1] = cimag(s);
        }
    free(tmp);
    free(w);
}

/* Inverse 2-D DFT followed by the real part: X[y][x] = Re sum_{l,k} Xhat(l,k) e^{+2 pi i (k x + l y)/D}. */
void oracle_dft2_inverse_real(int D, const double *Xhat_ri, double *X)
{
    cplx *w = twiddles(D, +1.0);
    cplx *tmp = (cplx *)malloc(sizeof(cplx) * (size_t)D * D); /* tmp[y][k] */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < D; ++y)
        for (int k = 0; k < D; ++k) {
            cplx s = 0;
            for (int l = 0; l < D; ++l) {
                size_t i = (size_t)l * D + k;
                s += (Xhat_ri[2 * i] + I * Xhat_ri[2 * i + 1]) * w[((long)l * y) % D];
            }
            tmp[(size_t)y * D + k] = s;
        }
#pragma omp parallel for schedule(static)
    for (int y = 0; y < D; ++y)
        for (int x = 0; x < D; ++x) {
            cplx s = 0;
            for (int k = 0; k < D; ++k)
                s += tmp[(size_t)y * D + k] * w[((long)k * x) % D];
            X[(size_t)y * D + x] = creal(s);
        }
    free(tmp);
    free(w);
}

/* Scaled wavenumber symbol for index j (0..D-1): 2 pi k tau, k = j or j - D; Nyquist -> 0 (G2). */
static double symbol(int j, int D, double tau, int nyquist_zero)
{
    int k = (j < D / 2) ? j : j - D;
    if (nyquist_zero && j == D / 2) return 0.0;
    return TWO_PI * (double)k * tau;
}

/* tau*Ahat for one mode. */
static void lrsw_symbol(double Kx, double Ky, double tau, cplx A[3][3])
{
    A[0][0] = 0;         A[0][1] = -I * Kx; A[0][2] = -I * Ky;
    A[1][0] = -I * Kx;   A[1][1] = 0;       A[1][2] = tau;
    A[2][0] = -I * Ky;   A[2][1] = -tau;    A[2][2] = 0;
}

/* Solve M x = b (3x3 complex) by Gaussian elimination with partial pivoting. */
static void gauss3(cplx M_in[3][3], const cplx b_in[3], cplx x[3])
{
    cplx M[3][3], b[3];
    memcpy(M, M_in, sizeof(M));
    memcpy(b, b_in, sizeof(b));
    for (int c = 0; c < 3; ++c) {
        int p = c;
        for (int r = c + 1; r < 3; ++r)
            if (cabs(M[r][c]) > cabs(M[p][c])) p = r;
        if (p != c) {
            for (int j = 0; j < 3; ++j) { cplx t = M[c][j]; M[c][j] = M[p][j]; M[p][j] = t; }
            cplx t = b[c]; b[c] = b[p]; b[p] = t;
        }
        for (int r = c + 1; r < 3; ++r) {
            cplx f = M[r][c] / M[c][c];
            for (int j = c; j < 3; ++j) M[r][j] -= f * M[c][j];
            b[r] -= f * b[c];
        }
    }
    for (int r = 2; r >= 0; --r) {
        cplx s = b[r];
        for (int j = r + 1; j < 3; ++j) s -= M[r][j] * x[j];
        x[r] = s / M[r][r];
    }
}

/*
 * REXII half-sum over poles n = 0..n_poles-1 for a list of modes.
 *   alpha_ri, C1_ri, C2_ri : 2*n_poles doubles (re, im) ; gamma: n_poles
 *   mode_l, mode_k         : row / column index of each listed mode
 *   fhat_ri                : n_modes x 3 complex (eta, u, v) inputs
 *   acc_ri                 : n_modes x 3 complex outputs (overwritten)
 */
void oracle_rexii_pole_sum(int D, double tau, int nyquist_zero, int n_poles,
                           const double *alpha_ri, const double *C1_ri, const double *C2_ri,
                           const double *gamma, long n_modes, const int *mode_l, const int *mode_k,
                           const double *fhat_ri, double *acc_ri)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (long m = 0; m < n_modes; ++m) {
        double Kx = symbol(mode_k[m], D, tau, nyquist_zero);
        double Ky = symbol(mode_l[m], D, tau, nyquist_zero);
        cplx A[3][3];
        lrsw_symbol(Kx, Ky, tau, A);
        cplx f0[3], acc[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c) f0[c] = fhat_ri[6 * m + 2 * c] + I * fhat_ri[6 * m + 2 * c + 1];
        for (int n = 0; n < n_poles; ++n) {
            cplx alpha = alpha_ri[2 * n] + I * alpha_ri[2 * n + 1];
            cplx alpha_m = conj(alpha);                 /* alpha_{-n} = h(mu - i n) */
            cplx C1 = C1_ri[2 * n] + I * C1_ri[2 * n + 1];
            cplx C2 = C2_ri[2 * n] + I * C2_ri[2 * n + 1];
            cplx M1[3][3], M2[3][3], g1[3], g2[3];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) {
                    M1[r][c] = A[r][c] + (r == c ? alpha : 0);     /* A + alpha_n I        */
                    M2[r][c] = -A[r][c] + (r == c ? alpha_m : 0);  /* alpha_{-n} I - A     */
                }
            gauss3(M1, f0, g1);
            gauss3(M2, g1, g2);
            for (int c = 0; c < 3; ++c)
                acc[c] += gamma[n] * (C2 * g1[c] + (C1 - C2 * alpha_m) * g2[c]);
        }
        for (int c = 0; c < 3; ++c) {
            acc_ri[6 * m + 2 * c] = creal(acc[c]);
            acc_ri[6 * m + 2 * c + 1] = cimag(acc[c]);
        }
    }
}

/*
 * Original REXI (eq:originalREXImatrix): acc = sum_n beta_n (tau A + alpha_n I)^{-1} f0
 * over the listed terms (full sum n = -N..N); the caller takes Re in physical space.
 */
void oracle_rexi_pole_sum(int D, double tau, int nyquist_zero, int n_terms,
                          const double *alpha_ri, const double *beta_ri,
                          long n_modes, const int *mode_l, const int *mode_k,
                          const double *fhat_ri, double *acc_ri)
{
#pragma omp parallel for schedule(dynamic, 16)
    for (long m = 0; m < n_modes; ++m) {
        double Kx = symbol(mode_k[m], D, tau, nyquist_zero);
        double Ky = symbol(mode_l[m], D, tau, nyquist_zero);
        cplx A[3][3];
        lrsw_symbol(Kx, Ky, tau, A);
        cplx f0[3], acc[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c) f0[c] = fhat_ri[6 * m + 2 * c] + I * fhat_ri[6 * m + 2 * c + 1];
        for (int n = 0; n < n_terms; ++n) {
            cplx alpha = alpha_ri[2 * n] + I * alpha_ri[2 * n + 1];
            cplx beta = beta_ri[2 * n] + I * beta_ri[2 * n + 1];
            cplx M1[3][3], g[3];
            for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c) M1[r][c] = A[r][c] + (r == c ? alpha : 0);
            gauss3(M1, f0, g);
            for (int c = 0; c < 3; ++c) acc[c] += beta * g[c];
        }
        for (int c = 0; c < 3; ++c) {
            acc_ri[6 * m + 2 * c] = creal(acc[c]);
            acc_ri[6 * m + 2 * c + 1] = cimag(acc[c]);
        }
    }
}
