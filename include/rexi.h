/*
 * rexi.h — C ABI of librexi.so: one REXII step e^{tau A} f0 of the linearised
 * rotating shallow-water equations (LRSW) on a B200 (sm_100a).
 *
 * Method: Caliari, Einkemmer, Moriggl, Ostermann, "An accurate and time-parallel
 * rational exponential integrator for hyperbolic and oscillatory PDEs",
 * arXiv:2008.11607. Citations "PAPER.md:<line>" refer to the LaTeX source
 * plus the equation label.
 *
 * Problem: d/dt f = A f, f = (eta, u, v), on the bi-periodic
 * unit square with a D x D grid, x_j = j/D,
 *     A = [[0, -d/dx, -d/dy], [-d/dx, 0, 1], [-d/dy, -1, 0]].
 * One step of size tau is approximated by the REXII half-sum
 * (eq:modifiedRexiMatrixReducedSum; procedure PAPER.md:427-435):
 *     e^{tau A} f0 ~ Re sum_{n=0}^{N} Gamma_n [ C2_n g1_n + (C1_n - C2_n alpha_{-n}) g2_n ],
 *     (alpha_n I + tau A) g1_n = f0,   (alpha_{-n} I - tau A) g2_n = g1_n,
 * with alpha_n = h(mu + i n), N = M + 24 and the Appendix A coefficients
 * (PAPER.md:815-851). All solves run per Fourier mode ("all computations ...
 * in Fourier space"): tau A is block-diagonal per wavenumber.
 *
 * Conventions shared by every entry point
 *  - Precision: IEEE fp64 throughout (complex fp64 in Fourier space).
 *  - Physical fields: caller-owned DEVICE pointers (unless the name says _host) to
 *    D*D contiguous doubles, row-major [y][x], x fastest (torch.float64 CUDA tensors).
 *  - Spectral arrays ("fhat", "acc"): caller-owned device pointers to 3*D*D complex
 *    values stored as interleaved (re, im) doubles, field-major (eta, u, v), then
 *    row l (y-wavenumber index), then column k (x-wavenumber index); index j maps
 *    to wavenumber j (j < D/2) or j - D. Forward transform:
 *        fhat(k,l) = D^-2 sum_{y,x} X[y][x] exp(-2 pi i (k x + l y)/D).
 *  - Readings of the paper: the operator is tau-scaled
 *    (G3: symbols 2 pi k tau, Coriolis tau); the Nyquist index's first-derivative
 *    symbol is zero (G2); the Appendix A sign column is the sign of the real part
 *    (G1); the g3 combination is division-free (G4).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream). Calls are stream-ordered and asynchronous unless stated. A plan is
 *    not re-entrant: do not use one plan from two streams concurrently.
 *  - Pole ranges [pole_begin, pole_end) index the half-sum n = 0..N
 *    (0 <= pole_begin <= pole_end <= n_poles); otherwise REXI_ERANGE.
 *  - Errors: every call returns a rexi_status_t; no C++ exception crosses the ABI.
 *    rexi_last_error() gives a thread-local text for the last failure. On error no
 *    output is guaranteed; inputs are never modified.
 *  - In-place: outputs may alias inputs for rexi_apply / rexi_apply_partial (the
 *    inputs are consumed into plan workspace first).
 */
#ifndef REXI_H
#define REXI_H

#ifdef __cplusplus
extern "C" {
#endif

#define REXI_ABI_VERSION 1
#define REXI_H_AUTO (-1.0)

typedef struct rexi_plan_s *rexi_plan_t; /* opaque; owns device workspace + pole table */

typedef enum {
    REXI_OK = 0,
    REXI_EINVAL = 1, /* bad argument (D, tau, tol, h, M, pointer, variant) */
    REXI_ENOMEM = 2, /* host or device allocation failed                   */
    REXI_ECUDA = 3,  /* a CUDA runtime call or kernel launch failed         */
    REXI_ERANGE = 4  /* bad pole range                                     */
} rexi_status_t;

/* Per-pole solve formulation of the fused pole kernel ("the variant ladder").
 * Every variant solves, per Fourier mode and pole, the shifted systems of PAPER.md:429-434 by
 * the Helmholtz reduction (eq:lswEta) and accumulates in registers; they
 * differ only in exact algebraic rearrangements of the per-pole back-substitution:
 *  REXI_VARIANT_UV:  paper-literal: (u, v) per pole by eq:lswVelocities,
 *                    delta, zeta of g1 from (u1, v1) (Alg. 1), then g2.
 *  REXI_VARIANT_DZ3: back-substitution in divergence/vorticity variables (delta, zeta of
 *                    PAPER.md:493-496); all three (eta, delta, zeta) pole sums accumulated;
 *                    velocities recovered once per mode from the sums.
 *  REXI_VARIANT_DZ:  as DZ3, but the zeta pole sum is rebuilt exactly from the eta pole sum
 *                    (zeta of each solve is affine in its eta: potential vorticity).
 *  REXI_VARIANT_PF:  as DZ, with the partial-fraction split of the two resolvents (SURVEY.md 8(d),
 *                    allowed equivalent): (conj(a) - B)^-1 (a + B)^-1 =
 *                    [(a + B)^-1 + (conj(a) - B)^-1] / (2 h mu) — two independent solves of f0.
 *  REXI_VARIANT_PFH: PF with the delta back-substitution (delta = alpha eta - eta0, the first row
 *                    of each system) folded into the accumulation weights: per pole the two
 *                    Helmholtz solutions are formed; (delta, zeta, u, v) follow once per mode.
 *  REXI_VARIANT_PFHR: PFH on "R2C" mode pairs, COLLAPSED (comparison only, see below): the fields
 *                    are real, so the spectrum is Hermitian and the solves at -K follow from those
 *                    at K; the pair {K, -K} accumulates directly the Hermitian part that survives
 *                    Re(IDFT(.)). The two Helmholtz solves are formed for every pole and pair;
 *                    what depends on K2 only is shared: the denominator by the modes of a K2
 *                    quad or octet ((a, b) and (b, a) on the square grid), and the weight sum of
 *                    the delta0 term per K2 value. This collapses the delta0
 *                    pole sums and pre-multiplies the weights by 1/(kappa + K2): it is NOT the
 *                    per-pole solve route of the contract (SURVEY.md 8(d) "out-of-contract
 *                    shortcut"); kept as a labelled comparison only.
 *  REXI_VARIANT_PFHX: explicit-solve R2C pairs (the DEFAULT): for every pole and every {K, -K}
 *                    pair the two Helmholtz solutions eta1 = q num1 and eta_t = conj(q) num_t are
 *                    formed from the pair's own right-hand sides (eq:lswEta, PAPER.md:486-497;
 *                    procedure PAPER.md:427-435), the -K solves follow from them through the
 *                    Hermitian data with the per-pole correction sigma_n delta0, and the weighted
 *                    Hermitian part is accumulated in registers. Shared between
 *                    the modes of an octet: only the reciprocal q = 1/(kappa_n + K2) and the
 *                    per-pole coefficients sigma_n, tau'_n. Used by rexi_apply / apply_partial /
 *                    apply_host / apply_host_batch / run; rexi_poles, whose input need not be
 *                    Hermitian, runs PFH. */
typedef enum {
    REXI_VARIANT_DZ = 0,
    REXI_VARIANT_UV = 1,
    REXI_VARIANT_DZ3 = 2,
    REXI_VARIANT_PF = 3,
    REXI_VARIANT_PFH = 4,
    REXI_VARIANT_PFHR = 5,
    REXI_VARIANT_PFHX = 6
} rexi_variant_t;

/* Which rational approximation the plan evaluates (both with the Appendix A coefficients):
 *  REXI_METHOD_REXII: the paper's REXII, two solves per term (eq:REXI_Modified_matrix,
 *                     half-sum eq:modifiedRexiMatrixReducedSum) — the default.
 *  REXI_METHOD_REXI:  the original REXI, eq:originalREXImatrix,
 *                     Re sum_{n=-N}^{N} beta^Re_n (tau A + alpha_n I)^{-1} f0, one solve per
 *                     term, evaluated as the half-sum n = 0..N with Gamma_n (the Appendix A
 *                     table is conjugate-symmetric, so beta^Re_{-n} = conj(beta^Re_n);
 *                     DESIGN.md reading R2). With w2 = 0 the partial-fraction weights are
 *                     W1 = w1, W2 = 0, so variants PF, PFH, PFHR and PFHX (default) run the same
 *                     kernels as REXII; UV, DZ and DZ3 select the DZ back-substitution kernel
 *                     (one solve per term). */
typedef enum { REXI_METHOD_REXII = 0, REXI_METHOD_REXI = 1 } rexi_method_t;

typedef struct {
    int D;                  /* grid size (power of two, 4..8192)                     */
    int variant;            /* rexi_variant_t                                         */
    int method;             /* rexi_method_t                                          */
    double tau;             /* step size                                              */
    double tol;             /* requested tolerance (0 if M was given explicitly)      */
    double h;               /* Gaussian spacing h (eq:bm)                             */
    double mu;              /* Appendix A mu                                          */
    long M;                 /* Gaussian-sum half width (eq:eixsumM)                   */
    long L;                 /* 24                                      */
    long N;                 /* M + L                                                  */
    long n_poles;           /* N + 1 (half-sum, Remark 3)                             */
    long m0;                /* the rule's offset: M = ceil(|tau| rho / h) + m0        */
    double rho;             /* sqrt(2) pi D (eq:lswRoh, Sec. 4.2 form, reading G5)    */
    double predicted_floor; /* predicted scalar error floor (readings G8, G9)         */
    double flops_per_pole_mode; /* algorithmic fp64 flops per pole x Fourier mode     */
    double fp64_ops_per_pole_mode; /* fp64-pipe instructions (FMA = 1) per pole x mode */
    int schedule;           /* rexi_schedule_t set on the plan                          */
    int last_schedule;      /* schedule the last pole-kernel launch used (CHUNKED or
                               STREAMK; AUTO = none yet)                                 */
} rexi_plan_info_t;

/* Create a plan for one step of size tau on a D x D grid.
 *  D:      power of two, 4 <= D <= 8192.
 *  tau:    finite; tau < 0 allowed (REXII is valid for x of both signs, eq:modifiedRexi).
 *  tol:    in (0, 1): sets m0 = ceil(2 sqrt(h^2 - ln(sqrt(4 pi) tol)) - 1) (reading G9,
 *          from Appendix B). tol <= 0 means the paper's m0 = 11
 *          (eq:Mformula).
 *  h:      in (0, pi); h <= 0 selects 0.5; h == REXI_H_AUTO selects
 *          rexi_h_for_tol(tol) (NEXT-2: fewer poles at loose tolerances).
 *  M:      > 0: use this M (must be >= 12); <= 0: M from the rule
 *          tau rho(A) <= (M - m0) h (eq:matrixAccuracyBound), at least 12.
 *  device: CUDA device ordinal.
 * Allocates the pole table and all workspace on `device`; synchronous.
 * Errors: EINVAL (arguments), ENOMEM, ECUDA. *out is NULL on error. */
rexi_status_t rexi_plan_create(rexi_plan_t *out, int D, double tau, double tol, double h,
                               long M, int device);
rexi_status_t rexi_plan_destroy(rexi_plan_t plan);
rexi_status_t rexi_plan_info(rexi_plan_t plan, rexi_plan_info_t *info);

/* Select the pole-kernel formulation (rexi_variant_t). EINVAL for unknown values. */
rexi_status_t rexi_plan_set_variant(rexi_plan_t plan, int variant);

/* Select the method (rexi_method_t); rebuilds and uploads the term table for the plan's
 * (h, M) (synchronous: waits for the device). EINVAL for unknown values, and for REXI on a
 * tau = 0 plan. (A REXII plan with tau = 0 always runs the UV variant: all symbols vanish.) */
rexi_status_t rexi_plan_set_method(rexi_plan_t plan, int method);

/* Replace the plan's rational approximation of the Gaussian (default: Appendix A) by
 * (L, mu, a[2(L+1)]) — e.g. a rexi_fit_gaussian refit — keeping h and M (N = M + L).
 * Rebuilds and uploads the term table (synchronous). EINVAL for bad tables. */
rexi_status_t rexi_plan_set_table(rexi_plan_t plan, int L, double mu, const double *a);

/* Pole-kernel tuning for the plan's CURRENT variant: Fourier modes per thread, poles per loop
 * trip and resident blocks per SM requested of the compiler (register budget). Supported:
 *   REXII DZ:  (1,1,8) (2,1,4) (2,1,5) (3,1,4) (4,1,3) (4,1,4)         default (4,1,4)
 *   REXII UV:  (1,1,6) (2,1,3) (2,1,4) (3,1,3) (4,1,2) (4,1,3)         default (4,1,3)
 *   REXII DZ3: (1,1,8) (2,1,4) (3,1,4) (4,1,2) (4,1,4)                 default (4,1,4)
 *   REXII PF:  (1,1,8) (2,1,3) (2,1,4) (3,1,4) (4,1,3) (4,1,4)         default (4,1,3)
 *   REXII PFH: (1,1,8) (2,1,3) (2,1,4) (3,1,4) (4,1,3) (4,1,4) (1,2,6) (2,2,3) (2,2,4) (4,2,2)
 *                                                                      default (4,2,2)
 *   REXII PFHR: modes_per_thread 4 (one K2 quad = two R2C pairs), 8 (an "octet": quads (a, b)
 *               and (b, a), which share K2, or one of the remaining quads plus a discarded copy
 *               = four pairs) or 16 (two quads in linear order, no K2 sharing):
 *               (4,1,4) (4,1,5) (4,1,6) (4,2,3) (4,2,4) (4,4,3) (8,1,2) (8,1,3) (8,2,2) (8,3,2)
 *               (8,4,2) (8,8,2) (8,2,3) (8,4,3) (8,8,3) (16,2,2)          default (8,8,2)
 *   REXII PFHX: modes_per_thread 8 (octet items): (8,1,2) (8,2,2) (8,4,2) (8,8,2) (8,1,3)
 *               (8,2,3) (8,4,3) (8,8,3)                                  default (8,8,2)
 *   REXI with variant UV / DZ / DZ3 (DZ back-substitution kernel):
 *               (1,1,8) (2,1,4) (4,1,4) (4,1,5)                         default (4,1,4)
 *   REXI with variant PF / PFH / PFHR / PFHX: as the REXII row of that variant (same kernels).
 * modes_per_thread = 4 maps each thread to a "K2 quad" (four modes with equal K^2 that share
 * the pole denominator 1/(kappa_n + K^2)).
 * Per pole and mode the operation order is the same for every tuning; the number of pole
 * chunks (and so the order in which chunk partial sums are added) follows the tile count, so
 * results agree to rounding, not bit for bit. EINVAL otherwise. */
rexi_status_t rexi_plan_set_tuning(rexi_plan_t plan, int modes_per_thread, int poles_per_iter,
                                   int min_blocks_per_sm);

/* How a step is scheduled on the GPU. For the R2C pole kernels (PFHR / PFHX, real-input calls):
 *  REXI_SCHEDULE_CHUNKED: grid = (tiles, pole chunks), chunk count chosen to fill whole waves of
 *                         resident blocks; one partial sum per chunk.
 *  REXI_SCHEDULE_STREAMK: a persistent grid of one 256-thread block per SM splits the
 *                         iteration space evenly (no wave tail); one partial per tile segment.
 *                         (PFHR only.)
 *  REXI_SCHEDULE_FUSED:   the whole physical step S1..S5 (rexi_apply / apply_partial /
 *                         apply_host) as ONE launch of thread-block clusters (16 CTAs, or 8):
 *                         FFT passes, PFHX pole loop, K = 0 corners, finish and inverse FFT
 *                         separated by cluster barriers, every stage's output handed to the CTA
 *                         that needs it through distributed shared memory (kernels.cu
 *                         step_small2_kernel); the pole range over 1..9 clusters
 *                         (rexi_plan_set_fused_clusters). PFHX plans with D <= 128 only (else
 *                         CHUNKED).
 *  REXI_SCHEDULE_AUTO:    FUSED for PFHX steps with D <= 128 and pole work up to 2^19 octet
 *                         items x poles (measured on B200: 64^2 at 47 poles 20 vs 36 us, at 604
 *                         poles 29 vs 58 us), CHUNKED otherwise (default).
 *                         With octet items every block costs the same, so the chunked waves are
 *                         already balanced, and two 128-thread blocks per SM issue at least as
 *                         well as one 256-thread block: measured on B200 the chunked pole kernel
 *                         is 0.5-7 % faster than STREAMK across the kernel versions.
 * STREAMK falls back to CHUNKED when the segment partials do not fit the partial buffer. The
 * kernels of every other variant are always chunked. Schedules differ only in the summation
 * order of the pole sum. Clears the plan's graph cache. EINVAL for an unknown schedule. */
typedef enum {
    REXI_SCHEDULE_AUTO = 0,
    REXI_SCHEDULE_CHUNKED = 1,
    REXI_SCHEDULE_STREAMK = 2,
    REXI_SCHEDULE_FUSED = 3
} rexi_schedule_t;
rexi_status_t rexi_plan_set_schedule(rexi_plan_t plan, int schedule);

/* Clusters of the fused step (REXI_SCHEDULE_FUSED / AUTO's fused choice): the step's pole range
 * is split into `clusters` contiguous blocks (sizes differ by <= 1), one 16-CTA cluster each
 * (the terms are independent); every cluster runs the forward transform and its
 * poles, writes its Hermitian partial spectrum, and the last cluster to finish sums the partials
 * in cluster order and runs the inverse transform. 0 (default): chosen from the pole count
 * (DESIGN.md 6.6); 1..9 fixed (capped at the clusters that can be resident at once and at the
 * range length). Results differ only in the summation order. Clears the plan's graph cache.
 * EINVAL outside 0..9. */
rexi_status_t rexi_plan_set_fused_clusters(rexi_plan_t plan, int clusters);

/* Whole-step CUDA graphs (default on): rexi_apply / rexi_apply_partial / rexi_apply_host /
 * rexi_run capture their kernel sequence once per (buffers, pole range, method, variant,
 * tuning, timing) on a private stream and replay it on `stream` afterwards (up to 8 cached
 * graphs per plan, least recently used evicted). Results are identical either way. */
rexi_status_t rexi_plan_set_graphs(rexi_plan_t plan, int enable);

/* Copy the plan's term table to HOST arrays of n_poles entries each (any may be NULL):
 *   alpha[2n], C1[2n], C2[2n] (interleaved re, im) and gamma[n], for n = 0..N:
 *   alpha_n = h(mu + i n), C1_n = c1_n h mu + c2_n h n, C2_n = i c2_n
 *   (PAPER.md:270), Gamma_0 = 1, Gamma_n = 2. For a REXI plan C1 holds
 *   beta^Re_n and C2 is zero. Synchronous. */
rexi_status_t rexi_plan_coeffs(rexi_plan_t plan, double *alpha, double *C1, double *C2,
                               double *gamma);

/* S1: forward 2-D FFT of the three real fields into fhat (layout above), scaled by D^-2. */
rexi_status_t rexi_forward(rexi_plan_t plan, const double *eta, const double *u, const double *v,
                           double *fhat, void *stream);

/* S2+S3: the fused pole kernel. For every Fourier mode and every pole n in
 * [pole_begin, pole_end) solve both shifted systems and accumulate
 *   acc = sum_n Gamma_n [ C2_n g1_n + (C1_n - C2_n alpha_{-n}) g2_n ]
 * (complex, BEFORE the real part). acc is overwritten (an empty
 * range gives zeros). fhat and acc must not alias. */
rexi_status_t rexi_poles(rexi_plan_t plan, long pole_begin, long pole_end, const double *fhat,
                         double *acc, void *stream);

/* S2+S3 for the spectrum of REAL fields (fhat = rexi_forward output, or any Hermitian spectrum
 * F(-K) = conj F(K)): writes acc = the spectrum of Re(IDFT(sum_{n in [pole_begin, pole_end)}
 * Gamma_n [...])), i.e. the Hermitian part (A(K) + conj A(-K)) / 2 of rexi_poles' sum — the
 * quantity the real part of PAPER.md:434 keeps — computed by the plan's R2C kernel (PFHX by
 * default: one {K, -K} pair per work item, both Helmholtz solves per pole).
 * acc is a full D x D spectrum (both modes of every pair written), summable across ranks
 * (S4 in spectral form) and invertible by rexi_inverse. The R2C kernel reads only one mode of
 * each pair, so a non-Hermitian fhat gives an unspecified result. fhat and acc must not alias;
 * ERANGE for a bad range. For the non-R2C variants this is rexi_poles followed by the
 * Hermitian projection. */
rexi_status_t rexi_poles_real(rexi_plan_t plan, long pole_begin, long pole_end, const double *fhat,
                              double *acc, void *stream);

/* S4 helper for the spectral form of the cross-GPU sum: a Hermitian spectrum (F(-K) = conj F(K),
 * e.g. rexi_poles_real output) is determined by its rows l = 0 .. D/2, which are contiguous per
 * field ((D/2 + 1) * D complex values at offset field * D * D) — ranks all-reduce only those
 * (the same bytes as the three real fields). This call rebuilds rows l = D/2 + 1 .. D - 1 in place:
 * acc(l, k) = conj acc(D - l, (D - k) mod D). Rows 0 and D/2 are not modified. */
rexi_status_t rexi_hermitian_mirror(rexi_plan_t plan, double *acc, void *stream);

/* S5: eta,u,v = Re(inverse 2-D FFT of acc) (Alg. 1 last line PAPER.md:535). */
rexi_status_t rexi_inverse(rexi_plan_t plan, const double *acc, double *eta, double *u, double *v,
                           void *stream);

/* S1..S5 for all poles: (eta_out, u_out, v_out) = REXII(tau A) (eta, u, v). */
rexi_status_t rexi_apply(rexi_plan_t plan, const double *eta, const double *u, const double *v,
                         double *eta_out, double *u_out, double *v_out, void *stream);

/* S1..S5 restricted to poles [pole_begin, pole_end): the real, physical-space partial
 * sum of one rank of a pole-partitioned step (SURVEY.md 8(e) option b). Summing the
 * outputs over a partition of [0, n_poles) gives rexi_apply's result (S4 is the
 * caller's allreduce; this library links no NCCL). */
rexi_status_t rexi_apply_partial(rexi_plan_t plan, long pole_begin, long pole_end,
                                 const double *eta, const double *u, const double *v,
                                 double *eta_out, double *u_out, double *v_out, void *stream);

/* rexi_apply with HOST buffers (any host memory; pinned is faster): copies the inputs
 * host->device, applies, copies the result device->host, and returns when the result
 * is in the host buffers (synchronous on `stream`). */
rexi_status_t rexi_apply_host(rexi_plan_t plan, const double *eta, const double *u,
                              const double *v, double *eta_out, double *u_out, double *v_out,
                              void *stream);

/* rexi_apply_host over `batch` independent problems: HOST arrays of batch consecutive D x D
 * fields each (problem i at offset i * D * D), outputs likewise. The host<->device copies of
 * problem i+1 (inputs) and i-1 (outputs) run on two private copy streams while problem i is
 * computed on `stream` (two device staging sets, allocated on first use), so with pinned host
 * memory the copies hide behind the steps. Returns when every output is in host memory.
 * batch = 0 is a no-op; EINVAL for batch < 0 or a NULL pointer. */
rexi_status_t rexi_apply_host_batch(rexi_plan_t plan, long batch, const double *eta,
                                    const double *u, const double *v, double *eta_out,
                                    double *u_out, double *v_out, void *stream);

/* S6: `steps` successive steps in place on device fields (T_final = steps * tau). For
 * steps >= 2 the state stays in Fourier space between steps (NEXT-4): one forward FFT, then per
 * step the pole sum and the spectral form of the real part, (X(K) + conj(X(-K)))/2 — the same
 * operator as Re(IDFT(.)) followed by DFT, without the FFT round trip — and one inverse FFT.
 * Steps that the fused schedule runs on one cluster (REXI_SCHEDULE_AUTO / FUSED, small grids
 * and pole counts, rexi_plan_set_fused_clusters) run the whole run as ONE launch: the state
 * stays in the cluster's shared memory between steps (R2C pair sums, Hermitian by
 * construction). */
rexi_status_t rexi_run(rexi_plan_t plan, int steps, double *eta, double *u, double *v,
                       void *stream);

/* Kernel timing of the pole kernel (the dominant kernel): when enabled, every pole-kernel
 * launch is bracketed by CUDA events on its stream. rexi_timing_read synchronises on
 * those events, returns the summed duration (ms) and launch count since the last read,
 * and resets. Also returns the number of kernels launched by the library (all kinds). */
rexi_status_t rexi_timing_enable(rexi_plan_t plan, int enable);
rexi_status_t rexi_timing_read(rexi_plan_t plan, double *pole_kernel_ms, long *pole_launches,
                               long *total_launches);

/* Measurement (not part of the method): the attainable fp64-pipe rate of `device`, the
 * roofline denominator of the pole kernel, which is bound by the fp64 ALUs (SURVEY.md 8(d)
 * "Which roofline bounds the path"). Runs `reps` launches of a DFMA kernel (8 independent
 * chains per thread, register operands, grid = SMs x 16 x 128 threads) and returns the best
 * rate in fp64-pipe ops/s (one DFMA = one op = 2 flops) and that launch's time (ms; may be
 * NULL). Synchronous on the default stream of `device`. EINVAL: ops_per_s NULL or reps < 1;
 * ECUDA: a CUDA call failed (rexi_last_error). */
rexi_status_t rexi_fp64_peak(int device, int reps, double *ops_per_s, double *best_ms);

/* Host-only (no GPU needed): the Appendix A table compiled into the library
 * (reading G1): *mu and a[2*(L+1)] = (Re a_l, Im a_l), l = 0..L;
 * returns L (= 24). a may be NULL to query L. */
int rexi_appendix_a(double *mu, double *a);

/* Host-only (no GPU needed): the planner's half-sum term table for (h, M) and a method — the
 * same numbers rexi_plan_coeffs returns for a plan with that h, M and method. For REXII:
 * alpha_n, C1_n, C2_n, Gamma_n; for REXI: alpha_n, beta^Re_n (in C1), 0 (in C2), Gamma_n.
 * Returns n_poles = M + 25 (or -1 if h is not in (0, pi), M < 12 or the method is unknown);
 * arrays of n_poles entries may be NULL. */
long rexi_terms_host(double h, long M, int method, double *alpha, double *C1, double *C2,
                     double *gamma);

/* Host-only (no GPU needed), NEXT-2: the paper's least-squares fit of the Gaussian psi_1 by the
 * symmetric rational function R (eq:A(x,mu); eq:minl2approx)
 * on K points of the Leja sequence on [0, xmax] started at x_1 = 0 (reading G18),
 * solved by Householder QR in extended precision. mu = NaN scans mu in [-7, -3] for the
 * smallest defect ("mu is determined such that a high accuracy is obtained").
 * Outputs a_out[2(L+1)] = (Re a_l, Im a_l), l = 0..L (a_0 real), *mu_out and *defect =
 * max |R - psi_1| on [-200, 200] (the REXI sums evaluate R far into its tail; xmax = 100,
 * K = 200 keep the tail below ~1e-15). Returns 0, or -1 for bad arguments (L in 1..64,
 * K >= 2L+1). */
int rexi_fit_gaussian(int L, double mu, int K, double xmax, double *a_out, double *mu_out,
                      double *defect);

/* Host-only (no GPU needed): the h optimiser of REXI_H_AUTO (NEXT-2, readings G8/G9): the largest
 * h with aliasing floor e^{-4 pi (pi - h)} <= tol / 10, clamped to [0.5, 2]; 0.5 if tol is not
 * in (0, 1). */
double rexi_h_for_tol(double tol);

/* Host-only (no GPU needed): the term-count rule used by rexi_plan_create:
 * m0(tol, h) (tol <= 0: 11) and M = ceil(|tau| sqrt(2) pi D / h) + m0 (rexi_plan_create raises
 * a result below 12 to 12). */
long rexi_rule_M(int D, double tau, double tol, double h);

/* ---------------------------------------------------------------------------------------
 * NEXT-3: the scalar forms applied to a diagonalised operator A = V E V^{-1} with purely
 * imaginary eigenvalues (eq:AisVEV..eq:REXI_VEV_DECOMP), e.g. a circulant
 * finite-difference matrix diagonalised by the DFT (the test matrices A_1, A_2 of PAPER.md:381-388).
 * A scalar plan holds the full-sum term table n = -N..N for (h, M) (Appendix A).
 * rexi_scalar_apply computes, for j < n (device arrays; x real, in/out complex interleaved):
 *     out_j = phase * r(i x_j) * in_j
 *   REXI_SCALAR_REXII:  r = eq:modifiedRexi
 *   REXI_SCALAR_REXI:   r = eq:originalRexi: per eigenvalue this is REXIE
 *                       (eq:REXIE) when V is real
 *   REXI_SCALAR_REXI_M: r = sum_n beta^Re_n / (i x + alpha_n): the eigen-coordinates of
 *                       eq:originalREXImatrix for a real A, whose Re the caller takes on the vector
 * Remark 1's shift is x_j -> x_j - nu/i and phase = e^{tau nu}. One block of
 * 256 threads per eigenvalue (each term a complex shifted solve 1/(alpha_n + i x_j)). */
typedef struct rexi_scalar_plan_s *rexi_scalar_plan_t;
typedef enum { REXI_SCALAR_REXII = 0, REXI_SCALAR_REXI = 1, REXI_SCALAR_REXI_M = 2 } rexi_scalar_method_t;
rexi_status_t rexi_scalar_plan_create(rexi_scalar_plan_t *out, double h, long M, int device);
rexi_status_t rexi_scalar_plan_destroy(rexi_scalar_plan_t plan);
long rexi_scalar_plan_terms(rexi_scalar_plan_t plan);
rexi_status_t rexi_scalar_apply(rexi_scalar_plan_t plan, int method, long n, const double *x,
                                const double *in, double *out, double phase_re, double phase_im,
                                void *stream);

/* NEXT-3 on the library's own transforms and pole kernel: out ~ e^{tau A} f for a CIRCULANT
 * n x n matrix A (first column `col`), e.g. the finite-difference test matrices A_1 (advection)
 * and A_2 (Schroedinger, shift nu = -2450 i) of Sec. 3.2 (Fig. 2). A circulant
 * is diagonalised by the DFT — A = F^-1 diag(F col) F, eq:AisVEV with V = F^-1 —
 * so, with the DFT kernels of the library (radix-8 Stockham passes for power-of-two n <= 2048, a
 * direct DFT for other n such as the paper's n = 70):
 *   1. lambda = DFT(col), fh = DFT(f);
 *   2. x_j = Im(tau (lambda_j - nu)) (A's eigenvalues are purely imaginary), and
 *      oh_j = e^{tau nu} r(i x_j) fh_j by the scalar pole kernel of rexi_scalar_apply with `method`
 *      (REXII; REXI = REXIE per eigenvalue; REXI_M = the eigen-coordinates of eq:originalREXImatrix,
 *      whose Re the caller takes for a real A, f); Remark 1's shift nu;
 *   3. out = DFT^-1(oh).
 * col, f, out: device arrays of n complex values (interleaved re, im); out must not alias col or
 * f. Stream-ordered (scratch from cudaMallocAsync on `stream`). EINVAL: null plan / pointer,
 * n < 1 or n > 2^20, unknown method, non-finite tau or nu; ECUDA: a CUDA call failed. */
rexi_status_t rexi_circulant_apply(rexi_scalar_plan_t plan, int method, long n, const double *col,
                                   const double *f, double *out, double tau, double nu_re,
                                   double nu_im, void *stream);

const char *rexi_status_string(rexi_status_t status);
const char *rexi_last_error(void);
int rexi_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* REXI_H */
