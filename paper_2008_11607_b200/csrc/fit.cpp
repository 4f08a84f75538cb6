// fit.cpp — NEXT-2: the paper's least-squares rational fit of the Gaussian (host, long double).
//
// eq:A(x,mu): R(x) = a0 mu/(x^2+mu^2) + sum_{l=1}^{L} [2 mu Re(a_l)(mu^2+l^2+x^2)
//   + 2 l Im(a_l)(mu^2+l^2-x^2)] / [x^4 + 2(mu^2-l^2)x^2 + (mu^2+l^2)^2], linear in
//   y = [a0, Re a_1..Re a_L, Im a_1..Im a_L];
// eq:minl2approx: minimise sum_k (psi_1(x_k) - R(x_k))^2 over K points;
// the points: "calculated iteratively. We start with x_1 = 0 and for selecting
// the next point x_{k+1} we use the same strategy that is used for minimizing the error in
// interpolation with Leja points" — reading G18: the Leja sequence on [0, xmax]
// (R and psi_1 are even), x_{k+1} = argmax over a uniform candidate grid of prod_j |x - x_j|,
// with xmax = 100 and K = 200 by default: the REXI sums use R(x/h + m) for |x/h + m| far
// beyond the Gaussian's support, so the fit must also keep the tail of R small (a fit on
// [0, 30] reaches 4e-15 there but leaves |R| ~ 1e-9 beyond 35).
#include <cmath>
#include <cstring>
#include <vector>

namespace {

using ld = long double;
const ld kPiL = 3.141592653589793238462643383279502884L;

ld psi1(ld x) { return std::exp(-x * x / 4.0L) / std::sqrt(4.0L * kPiL); }

// row of the design matrix G(x, mu, L) (2L+1 entries)
void design_row(ld x, ld mu, int L, ld *row) {
    const ld x2 = x * x;
    row[0] = mu / (x2 + mu * mu);
    for (int l = 1; l <= L; ++l) {
        const ld ll = (ld)l * l;
        const ld den = x2 * x2 + 2.0L * (mu * mu - ll) * x2 + (mu * mu + ll) * (mu * mu + ll);
        row[l] = 2.0L * mu * (mu * mu + ll + x2) / den;
        row[L + l] = 2.0L * (ld)l * (mu * mu + ll - x2) / den;
    }
}

// Leja sequence on [0, xmax] starting at 0, from `ncand` uniform candidates.
std::vector<ld> leja_points(int K, ld xmax, int ncand) {
    std::vector<ld> cand((size_t)ncand), logp((size_t)ncand, 0.0L);
    for (int i = 0; i < ncand; ++i) cand[(size_t)i] = xmax * (ld)i / (ld)(ncand - 1);
    std::vector<ld> pts;
    pts.push_back(0.0L);
    std::vector<char> used((size_t)ncand, 0);
    used[0] = 1;
    for (int i = 0; i < ncand; ++i) logp[(size_t)i] = std::log(std::fabs(cand[(size_t)i]) + 1e-300L);
    for (int k = 1; k < K; ++k) {
        int best = -1;
        for (int i = 0; i < ncand; ++i)
            if (!used[(size_t)i] && (best < 0 || logp[(size_t)i] > logp[(size_t)best])) best = i;
        if (best < 0) break;
        used[(size_t)best] = 1;
        const ld xb = cand[(size_t)best];
        pts.push_back(xb);
        for (int i = 0; i < ncand; ++i) logp[(size_t)i] += std::log(std::fabs(cand[(size_t)i] - xb) + 1e-300L);
    }
    return pts;
}

// min ||A y - b||_2 by Householder QR (A: m x n, m >= n, row-major), long double.
bool lstsq(std::vector<ld> A, std::vector<ld> b, int m, int n, std::vector<ld> &y) {
    for (int j = 0; j < n; ++j) {
        ld norm = 0;
        for (int i = j; i < m; ++i) norm += A[(size_t)i * n + j] * A[(size_t)i * n + j];
        norm = std::sqrt(norm);
        if (norm == 0) return false;
        const ld a0 = A[(size_t)j * n + j];
        const ld alpha = a0 > 0 ? -norm : norm;
        std::vector<ld> v((size_t)(m - j));
        v[0] = a0 - alpha;
        for (int i = j + 1; i < m; ++i) v[(size_t)(i - j)] = A[(size_t)i * n + j];
        ld vv = 0;
        for (ld t : v) vv += t * t;
        if (vv == 0) continue;
        for (int c = j; c < n; ++c) {
            ld s = 0;
            for (int i = j; i < m; ++i) s += v[(size_t)(i - j)] * A[(size_t)i * n + c];
            s = 2.0L * s / vv;
            for (int i = j; i < m; ++i) A[(size_t)i * n + c] -= s * v[(size_t)(i - j)];
        }
        ld s = 0;
        for (int i = j; i < m; ++i) s += v[(size_t)(i - j)] * b[(size_t)i];
        s = 2.0L * s / vv;
        for (int i = j; i < m; ++i) b[(size_t)i] -= s * v[(size_t)(i - j)];
    }
    y.assign((size_t)n, 0.0L);
    for (int j = n - 1; j >= 0; --j) {
        ld s = b[(size_t)j];
        for (int c = j + 1; c < n; ++c) s -= A[(size_t)j * n + c] * y[(size_t)c];
        if (A[(size_t)j * n + j] == 0) return false;
        y[(size_t)j] = s / A[(size_t)j * n + j];
    }
    return true;
}

ld fit_once(int L, ld mu, int K, ld xmax, std::vector<ld> &y) {
    const int n = 2 * L + 1;
    std::vector<ld> pts = leja_points(K, xmax, 30001);
    const int m = (int)pts.size();
    std::vector<ld> A((size_t)m * n), b((size_t)m);
    for (int i = 0; i < m; ++i) {
        design_row(pts[(size_t)i], mu, L, &A[(size_t)i * n]);
        b[(size_t)i] = psi1(pts[(size_t)i]);
    }
    if (!lstsq(A, b, m, n, y)) return -1;
    // defect max |R - psi_1| on [-200, 200] (even: [0, 200]): the REXI sums evaluate R at
    // x/h + m far outside the Gaussian's support, so the tail counts as much as the core
    ld worst = 0;
    std::vector<ld> row((size_t)n);
    for (int i = 0; i <= 40000; ++i) {
        const ld x = 200.0L * (ld)i / 40000.0L;
        design_row(x, mu, L, row.data());
        ld r = 0;
        for (int c = 0; c < n; ++c) r += row[(size_t)c] * y[(size_t)c];
        worst = std::max(worst, std::fabs(r - psi1(x)));
    }
    return worst;
}

}  // namespace

// See include/rexi.h.
extern "C" int rexi_fit_gaussian(int L, double mu, int K, double xmax, double *a_out, double *mu_out,
                                 double *defect) {
    if (L < 1 || L > 64 || K < 2 * L + 1 || !(xmax > 0)) return -1;
    std::vector<ld> y;
    ld best_mu = mu, best = -1;
    if (std::isnan(mu)) {   // scan mu in [-7, -3] ("mu is determined such that a
                            // high accuracy is obtained")
        for (int i = 0; i <= 80; ++i) {
            const ld m = -7.0L + 4.0L * (ld)i / 80.0L;
            std::vector<ld> yy;
            const ld d = fit_once(L, m, K, xmax, yy);
            if (d >= 0 && (best < 0 || d < best)) {
                best = d;
                best_mu = m;
            }
        }
    }
    const ld d = fit_once(L, best_mu, K, xmax, y);
    if (d < 0) return -1;
    if (a_out) {
        a_out[0] = (double)y[0];
        a_out[1] = 0.0;
        for (int l = 1; l <= L; ++l) {
            a_out[2 * l] = (double)y[(size_t)l];
            a_out[2 * l + 1] = (double)y[(size_t)(L + l)];
        }
    }
    if (mu_out) *mu_out = (double)best_mu;
    if (defect) *defect = (double)d;
    return 0;
}
