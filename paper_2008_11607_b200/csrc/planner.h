// planner.h — host planner of librexi (internal header; not part of the C ABI).
//
// Produces, in x87 extended precision rounded to fp64, the REXII term table of
// arXiv:2008.11607 and the per-pole constants consumed by the fused pole kernel.
#pragma once

#include <complex>
#include <vector>

namespace rexi {

// The rational approximation R(x) of psi_1 (eq:ratapproxgaus): mu and a_0..a_L
// (a_{-l} = conj(a_l)); Appendix A by default, or a NEXT-2 refit.
struct GaussTable {
    int L = 24;
    long double mu = 0;
    std::vector<std::complex<long double>> a;   // a_0..a_L
};
GaussTable appendix_a_table();

// Per-pole constants of the pole kernels (device layout, 28 doubles = 224 B).
// c = tau (tau-scaled Coriolis, reading G3); kappa = alpha^2 + c^2 (PAPER.md:476 with
// the tau scaling); w1 = Gamma C2, w2 = Gamma (C1 - C2 conj(alpha)) (reading G4).
struct alignas(16) PoleConst {
    double ar, ai;      // alpha_n = h(mu + i n)
    double s2r, s2i;    // c / alpha
    double iar, iai;    // 1 / alpha
    double s1cr, s1ci;  // conj(kappa / alpha) = conj(kappa)/conj(alpha)
    double kr, ki;      // kappa
    double ki2;         // Im(kappa)^2
    double w1r, w1i;    // Gamma_n C2_n
    double w2r, w2i;    // Gamma_n (C1_n - C2_n alpha_{-n})
    double s3r, s3i;    // alpha / kappa   (eq:lswVelocities, UV variant)
    double s4r, s4i;    // c / kappa
    double ia2;         // |1/alpha|^2
    double W1r, W1i;    // partial-fraction weights (PF kinds): w1 + w2 / (2 h mu)
    double W2r, W2i;    //                                       w2 / (2 h mu)
    double P1r, P1i;    // PFH: W1 alpha          (delta1 = alpha eta1 - e0 folded into the weights)
    double P2r, P2i;    // PFH: -W2 conj(alpha)   (delta_t = e0 - conj(alpha) eta_t)
};
static_assert(sizeof(PoleConst) == 224, "PoleConst layout");

// The constants the R2C pole kernel reads per pole, packed for nine 16-byte shared-memory loads
// (DESIGN.md 6.1): kappa; 2 h n; the R2C half-weights X1 = (W1 + conj W2)/2,
// Y1 = (P1 + conj P2)/2 (their partners are the conjugates); 2 Re(c/alpha), 2 Im(c/alpha); the
// delta0 weights as real coefficients of q = qr + i qi (W1 = a + ib, W2 = c + id):
// sigma = conj(W1) conj(q) - conj(W2) q + 2 i Im(X1 q)
//       = [(a-c) qr - (b+d) qi] + i [(d-b+2 Im X1) qr + (2 Re X1 - a - c) qi],
// tau' likewise with P1, P2, Y1 (the 2 i Im(X1 q) term: the delta0 part of the kernel's
// num1 - num_t, kernels.cu).
struct alignas(16) R2CPole {
    double kr, ki;
    double ki2, hn2;
    double X1r, X1i;
    double Y1r, Y1i;
    double sr2, si2;
    double sgx1, sgx2, sgy1, sgy2;
    double tax1, tax2, tay1, tay2;
};
static_assert(sizeof(R2CPole) == 144, "R2CPole layout");

// The constants the explicit-solve R2C kernel (PFHX, the default) reads per pole, nine 16-byte
// shared-memory loads: kappa, Im(kappa)^2, h n and c/alpha build the two Helmholtz solves of a
// mode pair, eta1 = q num1 and eta_t = conj(q) num_t (q = 1/(kappa + K2)); X1 = (W1 + conj W2)/2,
// Y1 = (P1 + conj P2)/2 weight them (partners conj X1, conj Y1); the per-pole coefficient of the
// -K correction 2 conj(q) delta0 resp. 2 q delta0 (kernels.cu, "R2C pairs") as real
// coefficients of q = qr + i qi (W1 = a + ib, W2 = c + id):
//   sigma_n = conj(W1 q) - conj(W2) q = [(a-c) qr - (b+d) qi] + i [(d-b) qr - (a+c) qi],
// tau'_n likewise with P1, P2. sigma_n and tau'_n are formed per pole and applied to each pair's
// delta0 per pole (no pole sum is formed before it meets a mode's data).
struct alignas(16) R2XPole {
    double kr, ki;
    double ki2, hn;
    double s2r, s2i;
    double X1r, X1i;
    double Y1r, Y1i;
    double sgx1, sgx2, sgy1, sgy2;
    double tax1, tax2, tay1, tay2;
};
static_assert(sizeof(R2XPole) == 144, "R2XPole layout");

struct Plan {
    GaussTable table;
    int D = 0;
    int method = 0;                  // 0: REXII (eq:REXI_Modified_matrix), 1: REXI (eq:originalREXImatrix)
    double tau = 0, tol = 0, h = 0, mu = 0;
    long M = 0, L = 24, N = 0, n_poles = 0, m0 = 11;
    double rho = 0, predicted_floor = 0;
    // term table, n = 0..N (interleaved re/im for complex entries)
    std::vector<double> alpha, C1, C2, gamma;   // REXI plans: C1 = beta^Re_n, C2 = 0
    std::vector<PoleConst> poles;
    std::vector<R2CPole> r2c;        // the same poles for the R2C kernel
    std::vector<R2XPole> r2x;        // the same poles for the explicit-solve R2C kernel
    // prefix sums (extended precision) of w1_n / alpha_n + w2_n / |alpha_n|^2, n = 0..N:
    // S(b, e) = pre[e] - pre[b] rebuilds the zeta pole sum from the eta pole sum (finish_kernel)
    std::vector<long double> spre_re, spre_im;
    // prefix sums of w1_n: the e0 term of the delta pole sum in the PFH kind
    std::vector<long double> wpre_re, wpre_im;
    std::vector<double> ksym;        // D tau-scaled derivative symbols, Nyquist zeroed (G2)
    std::vector<double> twiddle;     // D complex e^{-2 pi i j / D}
};

// Validates the arguments (see rexi.h) and fills `p`. Returns 0 or a rexi_status_t code;
// `err` receives a message.
int make_plan(Plan &p, int D, double tau, double tol, double h, long M, std::vector<char> &err,
              int method = 0, const GaussTable *table = nullptr);

// Full-sum term table n = -N..N for the scalar forms (NEXT-3): eq:modifiedRexi and
// eq:originalRexi.
struct ScalarTerm {
    double ar, ai;      // alpha_n = h(mu + i n)
    double C1r, C1i;    // c_{1,n} h mu + c_{2,n} h n
    double c2r, c2i;    // c_{2,n}
    double bRr, bRi;    // beta^Re_n
    double bIr, bIi;    // beta^Im_n
};
int make_scalar_terms(std::vector<ScalarTerm> &out, double h, long M, std::vector<char> &err,
                      const GaussTable *table = nullptr);

long m0_for_tol(double tol, double h);
double h_for_tol(double tol);

}  // namespace rexi
