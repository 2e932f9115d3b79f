// quadrature.hpp -- collapsed (conical-product) Gauss-Jacobi rule on the
// reference simplex, host C++ (CUDA path's own implementation).
//
// PAPER.md P:89-107 and P:694 (FEniCS uses the collapsed rule of Karniadakis &
// Sherwin at high order); the paper does not fix the rule of the DoGIP weights,
// reading L10 fixes n = p + 3 points per direction.  Collapsed coordinates:
//   2D  x1 = s1, x2 = s2 (1 - s1)
//   3D  x1 = s1, x2 = s2 (1 - s1), x3 = s3 (1 - s1)(1 - s2)
// s_i Gauss-Jacobi with weight (1 - s)^(d - i) on [0, 1]; points ordered with
// s1 slowest.  Roots of P_n^(a,0) by simultaneous Newton (Aberth) iteration in
// long double, weights from the Christoffel formula.
#pragma once
#include <algorithm>
#include <cmath>
#include <vector>

namespace dogip {

// P_n^(a,0)(x) and P_{n-1}^(a,0)(x) by the three-term recurrence.
inline void jacobi_eval(int n, long double a, long double x, long double& pn, long double& pn1) {
    const long double b = 0.0L;
    long double p0 = 1.0L, p1 = (a - b) / 2 + (a + b + 2) / 2 * x;
    if (n == 0) { pn = p0; pn1 = 0; return; }
    for (int k = 2; k <= n; ++k) {
        long double c = 2 * k + a + b;
        long double a1 = 2 * k * (k + a + b) * (c - 2);
        long double a2 = (c - 1) * (a * a - b * b);
        long double a3 = (c - 2) * (c - 1) * c;
        long double a4 = 2 * (k + a - 1) * (k + b - 1) * c;
        long double p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
        p0 = p1; p1 = p2;
    }
    pn = p1; pn1 = p0;
}

// derivative from (2n+a+b)(1-x^2) P_n' = n[(a-b) - (2n+a+b) x] P_n + 2(n+a)(n+b) P_{n-1}
inline long double jacobi_deriv(int n, long double a, long double x, long double pn, long double pn1) {
    const long double b = 0.0L, c = 2 * n + a + b;
    return (n * ((a - b) - c * x) * pn + 2 * (n + a) * (n + b) * pn1) / (c * (1 - x * x));
}

// n-point rule for int_0^1 (1-s)^a g(s) ds; nodes ascending.
inline void gauss_jacobi_01(int n, int a, std::vector<double>& s, std::vector<double>& w) {
    std::vector<long double> x(n);
    for (int i = 0; i < n; ++i) x[i] = -std::cos((long double)M_PI * (i + 0.75L) / (n + 0.5L));
    for (int it = 0; it < 200; ++it) {
        long double maxd = 0;
        for (int i = 0; i < n; ++i) {
            long double pn, pn1;
            jacobi_eval(n, a, x[i], pn, pn1);
            long double dp = jacobi_deriv(n, a, x[i], pn, pn1);
            long double ratio = pn / dp, sum = 0;
            for (int j = 0; j < n; ++j)
                if (j != i) sum += 1.0L / (x[i] - x[j]);
            long double dx = ratio / (1 - ratio * sum);     // Aberth correction
            x[i] -= dx;
            maxd = std::max(maxd, std::fabs(dx));
        }
        if (maxd < 1e-19L) break;
    }
    std::sort(x.begin(), x.end());
    // Christoffel weights for P_n^(a,0) on [-1,1]:
    //   w_i = Gamma(n+a+1) Gamma(n+1) / (Gamma(n+a+1) n!) 2^(a+1) / ((1-x^2) P_n'(x)^2)
    //       = 2^(a+1) / ((1 - x^2) P_n'(x)^2)          (b = 0 makes the Gamma ratio 1)
    s.resize(n); w.resize(n);
    for (int i = 0; i < n; ++i) {
        long double pn, pn1;
        jacobi_eval(n, a, x[i], pn, pn1);
        long double dp = jacobi_deriv(n, a, x[i], pn, pn1);
        long double wi = std::pow(2.0L, a + 1) / ((1 - x[i] * x[i]) * dp * dp);
        s[i] = (double)((1 + x[i]) / 2);
        w[i] = (double)(wi / std::pow(2.0L, a + 1));      // map to [0,1] with (1-s)^a
    }
}

// The simplex rule: pts (n^d x d), wts (n^d); sum(wts) = 1/d!.
inline void simplex_rule(int d, int n, std::vector<double>& pts, std::vector<double>& wts) {
    std::vector<double> s1, w1, s2, w2, s3, w3;
    pts.clear(); wts.clear();
    if (d == 2) {
        gauss_jacobi_01(n, 1, s1, w1);
        gauss_jacobi_01(n, 0, s2, w2);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                pts.push_back(s1[i]);
                pts.push_back(s2[j] * (1.0 - s1[i]));
                wts.push_back(w1[i] * w2[j]);
            }
    } else {
        gauss_jacobi_01(n, 2, s1, w1);
        gauss_jacobi_01(n, 1, s2, w2);
        gauss_jacobi_01(n, 0, s3, w3);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                for (int k = 0; k < n; ++k) {
                    pts.push_back(s1[i]);
                    pts.push_back(s2[j] * (1.0 - s1[i]));
                    pts.push_back(s3[k] * (1.0 - s1[i]) * (1.0 - s2[j]));
                    wts.push_back(w1[i] * w2[j] * w3[k]);
                }
    }
}

}  // namespace dogip
