// planner.cpp — host planner (S0 of SURVEY.md 8(a)): term count, b_m, c_{1,n}, c_{2,n},
// C_{1,n}, C_{2,n}, Gamma_n and the per-pole constants of the fused pole kernel.
// Extended precision (long double) throughout, rounded to fp64 once at the end.
#include "planner.h"

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>

#include "../../include/rexi.h"

namespace rexi {

using ld = long double;
using cld = std::complex<long double>;
using cd_pv_t = cld;

// Appendix A, PAPER.md:815-851 (tab:coef_al), L = 24. Reading G1: the printed sign
// column is the sign of the real part. a_{-l} = conj(a_l).
static const char *const kMu = "-5.133333333333333";
static const char *const kA[25][2] = {
    {"-6.520430828919864e+01", "0"},
    {"4.261818064131437e+01", "2.761406741120911e+01"},
    {"-9.801650304425239e+00", "-2.189295463610722e+01"},
    {"-1.054225194693395e+00", "6.791786454153551e+00"},
    {"7.950505668209775e-01", "-8.904997258367445e-01"},
    {"-1.218558380859130e-01", "3.321241563407446e-02"},
    {"7.365401806949337e-03", "2.212802103193251e-03"},
    {"-2.801087265991056e-04", "-5.566945197754387e-04"},
    {"1.254835436432561e-04", "-2.467200513365371e-04"},
    {"2.295472292491263e-04", "-8.494118951459107e-05"},
    {"1.858484460459430e-04", "9.242889460185034e-05"},
    {"4.068056518449676e-05", "1.653479957565515e-04"},
    {"-8.341508001647741e-05", "1.045331460447588e-04"},
    {"-9.970528169841103e-05", "-5.856228484297677e-06"},
    {"-3.499639858693093e-05", "-6.129059473910835e-05"},
    {"2.295021920298455e-05", "-4.099832469456381e-05"},
    {"2.931048772724314e-05", "1.708815129697846e-07"},
    {"7.502088478301169e-06", "1.525082051744077e-05"},
    {"-5.815291167450100e-06", "6.919604247338349e-06"},
    {"-4.069948458364005e-06", "-1.440010113050771e-06"},
    {"7.932524475429588e-08", "-1.794169428574330e-06"},
    {"6.120984882186265e-07", "-1.131894636585849e-07"},
    {"5.531365159161319e-08", "1.585749903175946e-07"},
    {"-2.867805871375946e-08", "1.239499740327838e-08"},
    {"-1.143081277095316e-09", "-2.763239274253499e-09"},
};
static const int kL = 24;
static const long double kPiL = 3.141592653589793238462643383279502884L;

static ld parse(const char *s) { return std::strtold(s, nullptr); }

GaussTable appendix_a_table() {
    GaussTable t;
    t.L = kL;
    t.mu = parse(kMu);
    t.a.resize((size_t)kL + 1);
    for (int l = 0; l <= kL; ++l) t.a[(size_t)l] = cld(parse(kA[l][0]), parse(kA[l][1]));
    return t;
}

// a_l for l = -L..L (conjugate-symmetric extension)
static cld a_coeff(const GaussTable &t, int l) {
    const int al = l < 0 ? -l : l;
    const cld a = t.a[(size_t)al];
    return l < 0 ? std::conj(a) : a;
}

long m0_for_tol(double tol, double h) {
    // Reading G9: Appendix B applied to the shifted-Gaussian tail
    // e^{h^2} psi_h((j+1) h) <= tol  =>  m0 = ceil(2 sqrt(h^2 - ln(sqrt(4 pi) tol)) - 1).
    if (!(tol > 0.0)) return 11;  // eq:Mformula
    double v = 2.0 * std::sqrt(h * h - std::log(std::sqrt(4.0 * M_PI) * tol)) - 1.0;
    return (long)std::ceil(v);
}

// NEXT-2 h optimiser (reading G9): the largest h whose aliasing floor
// e^{-4 pi (pi - h)} (reading G8) stays a factor 10 below tol, clamped to [0.5, 2]:
// fewer poles (M ~ tau rho / h) at the same tolerance.
double h_for_tol(double tol) {
    if (!(tol > 0.0 && tol < 1.0)) return 0.5;
    double h = M_PI - std::log(10.0 / tol) / (4.0 * M_PI);
    if (h < 0.5) h = 0.5;
    if (h > 2.0) h = 2.0;
    return h;
}

static void set_err(std::vector<char> &err, const char *msg) {
    err.assign(msg, msg + std::strlen(msg) + 1);
}

int make_plan(Plan &p, int D, double tau, double tol, double h, long M, std::vector<char> &err,
              int method, const GaussTable *table) {
    p.table = table ? *table : appendix_a_table();
    const GaussTable &T = p.table;
    const int kLt = T.L;
    if (kLt < 1 || (int)T.a.size() != kLt + 1) {
        set_err(err, "bad coefficient table");
        return REXI_EINVAL;
    }
    if (method != 0 && method != 1) {
        set_err(err, "method must be REXI_METHOD_REXII or REXI_METHOD_REXI");
        return REXI_EINVAL;
    }
    p.method = method;
    if (D < 4 || D > 8192 || (D & (D - 1)) != 0) {
        set_err(err, "D must be a power of two in [4, 8192]");
        return REXI_EINVAL;
    }
    if (!std::isfinite(tau)) { set_err(err, "tau must be finite"); return REXI_EINVAL; }
    if (h == REXI_H_AUTO) h = h_for_tol(tol);
    if (!(h > 0.0)) h = 0.5;
    if (!(h < M_PI)) { set_err(err, "h must lie in (0, pi) (PAPER.md:98)"); return REXI_EINVAL; }
    if (!(tol < 1.0) || std::isnan(tol)) { set_err(err, "tol must lie in (0, 1) (or <= 0 for m0 = 11)"); return REXI_EINVAL; }
    p.D = D;
    p.tau = tau;
    p.tol = tol > 0.0 ? tol : 0.0;
    p.h = h;
    p.m0 = m0_for_tol(tol, h);
    // eq:lswRoh in the sqrt(2) pi D form of the Sec. 4.2 display, reading G5.
    p.rho = std::sqrt(2.0) * M_PI * D;
    if (M <= 0) {
        double x = std::fabs(tau) * p.rho;                 // eq:matrixAccuracyBound
        M = (long)std::ceil(x / h) + p.m0;
        if (M < 12) M = 12;   // tiny |tau| rho: at least M - 11 >= 1 (eq:Mformula)
    }
    if (M < 12) { set_err(err, "M must be >= 12 (eq:Mformula needs M - 11 >= 1)"); return REXI_EINVAL; }
    if (M > 50000000L) { set_err(err, "M too large"); return REXI_EINVAL; }
    p.M = M;
    p.L = kLt;
    p.N = M + kLt;
    p.n_poles = p.N + 1;
    const ld hh = (ld)h;
    const ld mu = T.mu;
    p.mu = (double)mu;
    {
        ld alias = std::exp(-4.0L * kPiL * (kPiL - hh));                 // reading G8
        ld j1 = (ld)(p.m0 + 1) * hh;
        ld tail = std::exp(hh * hh) * std::exp(-j1 * j1 / (4.0L * hh * hh)) / std::sqrt(4.0L * kPiL);
        p.predicted_floor = (double)(alias + tail);
    }

    // eq:bm: b_m = e^{-i m h} e^{h^2}, m = -M..M (phase m*h in long double, G12).
    std::vector<cld> b((size_t)(2 * M + 1));
    const ld eh2 = std::exp(hh * hh);
    for (long m = -M; m <= M; ++m) {
        ld ph = (ld)m * hh;
        b[(size_t)(m + M)] = cld(eh2 * std::cos(ph), -eh2 * std::sin(ph));
    }
    const long N = p.N;
    p.alpha.assign(2 * (size_t)p.n_poles, 0.0);
    p.C1.assign(2 * (size_t)p.n_poles, 0.0);
    p.C2.assign(2 * (size_t)p.n_poles, 0.0);
    p.gamma.assign((size_t)p.n_poles, 0.0);
    p.poles.assign((size_t)p.n_poles, PoleConst{});
    p.r2c.assign((size_t)p.n_poles, R2CPole{});
    p.r2x.assign((size_t)p.n_poles, R2XPole{});
    p.spre_re.assign((size_t)p.n_poles + 1, 0.0L);
    p.spre_im.assign((size_t)p.n_poles + 1, 0.0L);
    p.wpre_re.assign((size_t)p.n_poles + 1, 0.0L);
    p.wpre_im.assign((size_t)p.n_poles + 1, 0.0L);
    const ld c = (ld)tau;  // tau-scaled Coriolis coefficient (reading G3)
    for (long n = 0; n <= N; ++n) {
        // c_{1,n} = h sum_{k=L1}^{L2} Re(a_k) b_{n-k},  c_{2,n} = h sum Im(a_k) b_{n-k}
        // L1(n) = max(-L, n - M), L2(n) = min(L, n + M)
        long L1 = std::max<long>(-kLt, n - M), L2 = std::min<long>(kLt, n + M);
        cld c1(0, 0), c2(0, 0), beta(0, 0);
        for (long k = L1; k <= L2; ++k) {
            cld ak = a_coeff(T, (int)k);
            const cld &bnk = b[(size_t)(n - k + M)];
            c1 += ak.real() * bnk;
            c2 += ak.imag() * bnk;
            beta += ak * bnk.real();   // beta^Re_n = h sum a_k Re(b_{n-k})
        }
        c1 *= hh;
        c2 *= hh;
        beta *= hh;
        // C_{1,n} = c_{1,n} h mu + c_{2,n} h n ; C_{2,n} = i c_{2,n}
        cld C1 = c1 * hh * mu + c2 * hh * (ld)n;
        cld C2 = cld(0, 1) * c2;
        if (method == 1) {   // REXI: the table carries beta^Re_n in C1 and zero in C2
            C1 = beta;
            C2 = cld(0, 0);
        }
        cld alpha(hh * mu, hh * (ld)n);                   // alpha_n = h(mu + i n)
        ld gam = (n == 0) ? 1.0L : 2.0L;                  // Gamma_n
        p.alpha[2 * n] = (double)alpha.real();  p.alpha[2 * n + 1] = (double)alpha.imag();
        p.C1[2 * n] = (double)C1.real();        p.C1[2 * n + 1] = (double)C1.imag();
        p.C2[2 * n] = (double)C2.real();        p.C2[2 * n + 1] = (double)C2.imag();
        p.gamma[n] = (double)gam;

        // Per-pole constants of the fused kernel.
        cld kappa = alpha * alpha + c * c;                // kappa_n (tau-scaled)
        cld w1 = gam * C2;                                // reading G4 (division-free g3)
        cld w2 = gam * (C1 - C2 * std::conj(alpha));
        if (method == 1) {
            // REXI half-sum: Re sum_{n=-N}^{N} beta_n (tau A + alpha_n)^{-1} f0
            //              = Re sum_{n=0}^{N} Gamma_n beta_n (...) f0 for real A, f0, since
            // beta^Re_{-n} = conj(beta^Re_n) with the symmetric Appendix A table (reading R2).
            w1 = gam * beta;
            w2 = cld(0, 0);
        }
        cld s2 = c / alpha, ia = 1.0L / alpha, s1c = std::conj(kappa / alpha);
        cld s3 = alpha / kappa, s4 = c / kappa;
        {
            const cd_pv_t sv = w1 * ia + w2 * std::norm(ia);
            p.spre_re[(size_t)n + 1] = p.spre_re[(size_t)n] + sv.real();
            p.spre_im[(size_t)n + 1] = p.spre_im[(size_t)n] + sv.imag();
            p.wpre_re[(size_t)n + 1] = p.wpre_re[(size_t)n] + w1.real();
            p.wpre_im[(size_t)n + 1] = p.wpre_im[(size_t)n] + w1.imag();
        }
        PoleConst &q = p.poles[(size_t)n];
        q.ar = (double)alpha.real();  q.ai = (double)alpha.imag();
        q.s2r = (double)s2.real();    q.s2i = (double)s2.imag();
        q.iar = (double)ia.real();    q.iai = (double)ia.imag();
        q.s1cr = (double)s1c.real();  q.s1ci = (double)s1c.imag();
        q.kr = (double)kappa.real();  q.ki = (double)kappa.imag();
        q.ki2 = (double)(kappa.imag() * kappa.imag());
        q.w1r = (double)w1.real();    q.w1i = (double)w1.imag();
        q.w2r = (double)w2.real();    q.w2i = (double)w2.imag();
        q.s3r = (double)s3.real();    q.s3i = (double)s3.imag();
        q.s4r = (double)s4.real();    q.s4i = (double)s4.imag();
        {
            // (conj(alpha) - B)^{-1} (alpha + B)^{-1} = [(alpha + B)^{-1} + (conj(alpha) - B)^{-1}]
            // / (alpha + conj(alpha)), alpha + conj(alpha) = 2 h mu (partial fractions)
            const cld W2 = w2 / (2.0L * alpha.real());
            const cld W1 = w1 + W2;
            q.W1r = (double)W1.real();  q.W1i = (double)W1.imag();
            q.W2r = (double)W2.real();  q.W2i = (double)W2.imag();
            const cld P1 = W1 * alpha, P2 = -W2 * std::conj(alpha);
            q.P1r = (double)P1.real();  q.P1i = (double)P1.imag();
            q.P2r = (double)P2.real();  q.P2i = (double)P2.imag();
            // R2C half-weights; the partner weights (W2 + conj W1)/2 and (P2 + conj P1)/2 are the
            // conjugates of these, which the kernel uses directly
            const cld X1 = (W1 + std::conj(W2)) * 0.5L;
            const cld Y1 = (P1 + std::conj(P2)) * 0.5L;
            R2CPole &rq = p.r2c[(size_t)n];
            rq.kr = q.kr;                 rq.ki = q.ki;
            rq.ki2 = q.ki2;               rq.hn2 = 2.0 * q.ai;        // exact (power-of-two scaling)
            rq.X1r = (double)X1.real();  rq.X1i = (double)X1.imag();
            rq.Y1r = (double)Y1.real();  rq.Y1i = (double)Y1.imag();
            rq.sr2 = 2.0 * q.s2r;        rq.si2 = 2.0 * q.s2i;
            // sigma also carries the delta0 part 2 i Im(X1 q) of the sum/difference evaluation
            // (kernels.cu): 2 Im(X1 q) = 2 X1i qr + 2 X1r qi joins the imaginary coefficients
            rq.sgx1 = (double)(W1.real() - W2.real());   rq.sgx2 = (double)(-(W1.imag() + W2.imag()));
            rq.sgy1 = (double)(W2.imag() - W1.imag() + 2.0L * X1.imag());
            rq.sgy2 = (double)(-(W1.real() + W2.real()) + 2.0L * X1.real());
            rq.tax1 = (double)(P1.real() - P2.real());   rq.tax2 = (double)(-(P1.imag() + P2.imag()));
            rq.tay1 = (double)(P2.imag() - P1.imag() + 2.0L * Y1.imag());
            rq.tay2 = (double)(-(P1.real() + P2.real()) + 2.0L * Y1.real());
            R2XPole &rx = p.r2x[(size_t)n];
            rx.kr = q.kr;                 rx.ki = q.ki;
            rx.ki2 = q.ki2;               rx.hn = q.ai;
            rx.s2r = q.s2r;               rx.s2i = q.s2i;
            rx.X1r = rq.X1r;              rx.X1i = rq.X1i;
            rx.Y1r = rq.Y1r;              rx.Y1i = rq.Y1i;
            rx.sgx1 = rq.sgx1;            rx.sgx2 = rq.sgx2;
            rx.sgy1 = (double)(W2.imag() - W1.imag());
            rx.sgy2 = (double)(-(W1.real() + W2.real()));
            rx.tax1 = rq.tax1;            rx.tax2 = rq.tax2;
            rx.tay1 = (double)(P2.imag() - P1.imag());
            rx.tay2 = (double)(-(P1.real() + P2.real()));
        }
        q.ia2 = (double)std::norm(ia);
    }

    // Fourier symbols: index j -> wavenumber k = j (j < D/2) else j - D; 2 pi k tau;
    // Nyquist index D/2 -> 0 (reading G2).
    p.ksym.assign((size_t)D, 0.0);
    for (int j = 0; j < D; ++j) {
        long k = (j < D / 2) ? j : (long)j - D;
        p.ksym[(size_t)j] = (j == D / 2) ? 0.0 : (double)(2.0L * kPiL * (ld)k * (ld)tau);
    }
    // FFT twiddles e^{-2 pi i j / D}, j = 0..D-1 (full circle, long double, rounded once).
    p.twiddle.assign(2 * (size_t)D, 0.0);
    for (int j = 0; j < D; ++j) {
        ld th = 2.0L * kPiL * (ld)j / (ld)D;
        p.twiddle[2 * (size_t)j] = (double)std::cos(th);
        p.twiddle[2 * (size_t)j + 1] = (double)(-std::sin(th));
    }
    return REXI_OK;
}

int make_scalar_terms(std::vector<ScalarTerm> &out, double h, long M, std::vector<char> &err,
                      const GaussTable *table) {
    if (!(h > 0.0 && h < M_PI)) { set_err(err, "h must lie in (0, pi) (PAPER.md:98)"); return REXI_EINVAL; }
    if (M < 12 || M > 50000000L) { set_err(err, "M must be in [12, 5e7]"); return REXI_EINVAL; }
    const GaussTable T = table ? *table : appendix_a_table();
    const int L = T.L;
    const long N = M + L;
    const ld hh = (ld)h, mu = T.mu, eh2 = std::exp(hh * hh);
    std::vector<cld> b((size_t)(2 * M + 1));
    for (long m = -M; m <= M; ++m) {
        const ld ph = (ld)m * hh;
        b[(size_t)(m + M)] = cld(eh2 * std::cos(ph), -eh2 * std::sin(ph));   // eq:bm
    }
    out.assign((size_t)(2 * N + 1), ScalarTerm{});
    for (long n = -N; n <= N; ++n) {
        const long L1 = std::max<long>(-L, n - M), L2 = std::min<long>(L, n + M);
        cld c1(0, 0), c2(0, 0), bR(0, 0), bI(0, 0);
        for (long k = L1; k <= L2; ++k) {
            const cld ak = a_coeff(T, (int)k), bnk = b[(size_t)(n - k + M)];
            c1 += ak.real() * bnk;
            c2 += ak.imag() * bnk;
            bR += ak * bnk.real();
            bI += ak * bnk.imag();
        }
        c1 *= hh; c2 *= hh; bR *= hh; bI *= hh;
        const cld C1 = c1 * hh * mu + c2 * hh * (ld)n;
        ScalarTerm &t = out[(size_t)(n + N)];
        t.ar = (double)(hh * mu);   t.ai = (double)(hh * (ld)n);
        t.C1r = (double)C1.real();  t.C1i = (double)C1.imag();
        t.c2r = (double)c2.real();  t.c2i = (double)c2.imag();
        t.bRr = (double)bR.real();  t.bRi = (double)bR.imag();
        t.bIr = (double)bI.real();  t.bIi = (double)bI.imag();
    }
    return REXI_OK;
}

}  // namespace rexi

extern "C" int rexi_appendix_a(double *mu, double *a) {
    if (mu) *mu = (double)rexi::parse(rexi::kMu);
    if (a)
        for (int l = 0; l <= rexi::kL; ++l) {
            a[2 * l] = (double)rexi::parse(rexi::kA[l][0]);
            a[2 * l + 1] = (double)rexi::parse(rexi::kA[l][1]);
        }
    return rexi::kL;
}

extern "C" long rexi_rule_M(int D, double tau, double tol, double h) {
    if (!(h > 0.0)) h = 0.5;
    double x = std::fabs(tau) * (std::sqrt(2.0) * M_PI * D);
    return (long)std::ceil(x / h) + rexi::m0_for_tol(tol, h);
}

extern "C" long rexi_terms_host(double h, long M, int method, double *alpha, double *C1, double *C2,
                                double *gamma) {
    if (!(h > 0.0 && h < M_PI) || M < 12) return -1;
    rexi::Plan p;
    std::vector<char> err;
    try {
        // D and tau do not enter the term table; D = 4, tau = 0 keep the rest cheap.
        if (rexi::make_plan(p, 4, 0.0, 0.0, h, M, err, method) != REXI_OK) return -1;
    } catch (...) {
        return -1;
    }
    const size_t n = (size_t)p.n_poles;
    if (alpha) std::memcpy(alpha, p.alpha.data(), 2 * n * sizeof(double));
    if (C1) std::memcpy(C1, p.C1.data(), 2 * n * sizeof(double));
    if (C2) std::memcpy(C2, p.C2.data(), 2 * n * sizeof(double));
    if (gamma) std::memcpy(gamma, p.gamma.data(), n * sizeof(double));
    return p.n_poles;
}

extern "C" double rexi_h_for_tol(double tol) { return rexi::h_for_tol(tol); }
