// tables.hpp -- exact reference-element tables for the CUDA path (host C++17).
//
// Lagrange P_k on the unit right simplex with equispaced barycentric lattice
// nodes (readings L1, L2, L5), built
// in exact rational arithmetic and rounded to fp64 once:
//   WP   Bhat_jl  = phi^l_V(xhat^j_W),           V = P_p, W = P_2p
//   EL   Bhat_rjl = d phi^l_V / d xhat_r (xhat^j_W), W = P_{2p-2}
// The basis is the barycentric product formula
//   phi_alpha(lambda) = prod_i prod_{m<alpha_i} (k lambda_i - m)/(m+1).
// Used by the code generator (gen/gen_bhat.cpp) and by the library's
// introspection entry points.  Shares no code with oracle/.
#pragma once
#include <array>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <vector>

namespace dogip {

// ---------------------------------------------------------------- rationals
struct Rat {
    int64_t n = 0, d = 1;
    Rat() = default;
    Rat(int64_t a) : n(a), d(1) {}
    Rat(int64_t a, int64_t b) { set((__int128)a, (__int128)b); }
    static __int128 gcd128(__int128 a, __int128 b) {
        if (a < 0) a = -a;
        if (b < 0) b = -b;
        while (b) { __int128 t = a % b; a = b; b = t; }
        return a;
    }
    void set(__int128 a, __int128 b) {
        if (b == 0) throw std::runtime_error("Rat: zero denominator");
        if (b < 0) { a = -a; b = -b; }
        __int128 g = gcd128(a, b);
        if (g > 1) { a /= g; b /= g; }
        const __int128 lim = (__int128)1 << 62;
        if (a >= lim || a <= -lim || b >= lim) throw std::runtime_error("Rat: overflow");
        n = (int64_t)a; d = (int64_t)b;
    }
    friend Rat operator+(Rat a, Rat b) { Rat r; r.set((__int128)a.n * b.d + (__int128)b.n * a.d, (__int128)a.d * b.d); return r; }
    friend Rat operator-(Rat a, Rat b) { Rat r; r.set((__int128)a.n * b.d - (__int128)b.n * a.d, (__int128)a.d * b.d); return r; }
    friend Rat operator*(Rat a, Rat b) { Rat r; r.set((__int128)a.n * b.n, (__int128)a.d * b.d); return r; }
    friend Rat operator/(Rat a, Rat b) { Rat r; r.set((__int128)a.n * b.d, (__int128)a.d * b.n); return r; }
    bool operator==(const Rat& o) const { return n == o.n && d == o.d; }
    bool operator!=(const Rat& o) const { return !(*this == o); }
    bool is_zero() const { return n == 0; }
    bool is_pm1() const { return d == 1 && (n == 1 || n == -1); }
    // correctly rounded (round-half-even) conversion of the exact quotient
    double to_double() const {
        if (n == 0) return 0.0;
        const bool neg = n < 0;
        unsigned __int128 a = neg ? (unsigned __int128)(-(__int128)n) : (unsigned __int128)n;
        unsigned __int128 b = (unsigned __int128)d;
        auto bitlen = [](unsigned __int128 x) { int l = 0; while (x) { ++l; x >>= 1; } return l; };
        int s = 54 - bitlen(a) + bitlen(b);          // a 2^s / b in (2^53, 2^55)
        unsigned __int128 num = a, den = b;
        if (s >= 0) num <<= s; else den <<= -s;
        unsigned __int128 q = num / den;
        bool sticky = (num % den) != 0;
        while (q >= ((unsigned __int128)1 << 54)) { sticky |= (bool)(q & 1); q >>= 1; s -= 1; }
        const bool guard = (bool)(q & 1);
        uint64_t mant = (uint64_t)(q >> 1);            // 53 bits
        if (guard && (sticky || (mant & 1))) ++mant;
        const double v = __builtin_ldexp((double)mant, 1 - s);
        return neg ? -v : v;
    }
};

inline int binom(int n, int k) {
    if (k < 0 || k > n) return 0;
    int64_t r = 1;
    for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return (int)r;
}
inline int dim_P(int d, int k) { return binom(k + d, d); }

// Barycentric multi-indices (alpha_0..alpha_d), |alpha| = k, alpha_1 fastest,
// alpha_d slowest (reading L5).
inline std::vector<std::array<int, 4>> multi_indices(int d, int k) {
    std::vector<std::array<int, 4>> out;
    if (d == 2) {
        for (int a2 = 0; a2 <= k; ++a2)
            for (int a1 = 0; a1 + a2 <= k; ++a1) out.push_back({k - a1 - a2, a1, a2, 0});
    } else {
        for (int a3 = 0; a3 <= k; ++a3)
            for (int a2 = 0; a2 + a3 <= k; ++a2)
                for (int a1 = 0; a1 + a2 + a3 <= k; ++a1)
                    out.push_back({k - a1 - a2 - a3, a1, a2, a3});
    }
    return out;
}

// Nodes of P_k as barycentric coordinates (exact); k = 0: the barycentre.
inline std::vector<std::array<Rat, 4>> nodes_bary(int d, int k) {
    std::vector<std::array<Rat, 4>> out;
    if (k == 0) {
        std::array<Rat, 4> b{};
        for (int i = 0; i <= d; ++i) b[i] = Rat(1, d + 1);
        out.push_back(b);
        return out;
    }
    for (auto& a : multi_indices(d, k)) {
        std::array<Rat, 4> b{};
        for (int i = 0; i <= d; ++i) b[i] = Rat(a[i], k);
        out.push_back(b);
    }
    return out;
}

// one factor f_a(lam) = prod_{m<a} (k lam - m)/(m+1) and its derivative
inline Rat factor(int a, int k, Rat lam) {
    Rat v(1);
    for (int m = 0; m < a; ++m) v = v * (Rat(k) * lam - Rat(m)) / Rat(m + 1);
    return v;
}
inline Rat dfactor(int a, int k, Rat lam) {
    Rat s(0);
    for (int m = 0; m < a; ++m) {
        Rat t = Rat(k, m + 1);
        for (int j = 0; j < a; ++j)
            if (j != m) t = t * (Rat(k) * lam - Rat(j)) / Rat(j + 1);
        s = s + t;
    }
    return s;
}

inline Rat phi_exact(const std::array<int, 4>& al, int d, int k, const std::array<Rat, 4>& lam) {
    Rat v(1);
    for (int i = 0; i <= d; ++i) v = v * factor(al[i], k, lam[i]);
    return v;
}

// d phi / d xhat_r = d/d lambda_r - d/d lambda_0  (xhat_r = lambda_r, reading L2)
inline Rat dphi_exact(const std::array<int, 4>& al, int d, int k, const std::array<Rat, 4>& lam, int r) {
    auto dlam = [&](int i) {
        Rat v = dfactor(al[i], k, lam[i]);
        for (int m = 0; m <= d; ++m)
            if (m != i) v = v * factor(al[m], k, lam[m]);
        return v;
    };
    return dlam(r) - dlam(0);
}

// Table: nblk x rows x cols; WP nblk = 1 (W_T x V_T), EL nblk = d.
struct Table {
    int nblk = 0, rows = 0, cols = 0;
    std::vector<Rat> v;
    Rat at(int b, int r, int c) const { return v[((size_t)b * rows + r) * cols + c]; }
};

inline Table bhat_table(int d, int p, int form) {
    Table t;
    auto A = multi_indices(d, p);
    auto W = nodes_bary(d, form == 0 ? 2 * p : 2 * p - 2);
    t.nblk = form == 0 ? 1 : d;
    t.rows = (int)W.size();
    t.cols = (int)A.size();
    t.v.resize((size_t)t.nblk * t.rows * t.cols);
    for (int b = 0; b < t.nblk; ++b)
        for (int j = 0; j < t.rows; ++j)
            for (int l = 0; l < t.cols; ++l)
                t.v[((size_t)b * t.rows + j) * t.cols + l] =
                    form == 0 ? phi_exact(A[l], d, p, W[j]) : dphi_exact(A[l], d, p, W[j], b + 1);
    return t;
}

// Barycentric partial derivatives D_i[j][l] = d phi^l_V / d lambda_i (xhat^j_W), i = 0..d,
// at the EL double-grid nodes (2p-2 lattice); Bhat_EL block r = D_{r+1} - D_0 (reading
// L2).  Each D_i is sparser than the difference (one lambda factor differentiated),
// so the generated EL body interpolates through them.
inline Table bary_deriv_table(int d, int p) {
    Table t;
    auto A = multi_indices(d, p);
    auto W = nodes_bary(d, 2 * p - 2);
    t.nblk = d + 1;
    t.rows = (int)W.size();
    t.cols = (int)A.size();
    t.v.resize((size_t)t.nblk * t.rows * t.cols);
    for (int i = 0; i <= d; ++i)
        for (int j = 0; j < t.rows; ++j)
            for (int l = 0; l < t.cols; ++l) {
                Rat v = dfactor(A[l][i], p, W[j][i]);
                for (int m = 0; m <= d; ++m)
                    if (m != i) v = v * factor(A[l][m], p, W[j][m]);
                t.v[((size_t)i * t.rows + j) * t.cols + l] = v;
            }
    return t;
}

// ------------------------------------------------- float evaluation (points)
// Basis of P_k at reference points (long double product formula).
inline void eval_basis_ld(int d, int k, const double* pts, int npts, double* out /* npts x dim */) {
    auto A = multi_indices(d, k);
    const int nb = (int)A.size();
    for (int q = 0; q < npts; ++q) {
        long double lam[4];
        long double s = 0;
        for (int r = 0; r < d; ++r) { lam[r + 1] = pts[q * d + r]; s += lam[r + 1]; }
        lam[0] = 1.0L - s;
        for (int c = 0; c < nb; ++c) {
            long double v = 1.0L;
            for (int i = 0; i <= d; ++i)
                for (int m = 0; m < A[c][i]; ++m) v *= ((long double)k * lam[i] - m) / (m + 1);
            out[(size_t)q * nb + c] = (double)v;
        }
    }
}

// Reference gradients d phi_c / d xhat_r = d/d lambda_r - d/d lambda_0 of P_k at points
// (long double product rule), out[(q * d + r) * dim + c].
inline void eval_grad_ld(int d, int k, const double* pts, int npts, double* out) {
    auto A = multi_indices(d, k);
    const int nb = (int)A.size();
    for (int q = 0; q < npts; ++q) {
        long double lam[4];
        long double s = 0;
        for (int r = 0; r < d; ++r) { lam[r + 1] = pts[q * d + r]; s += lam[r + 1]; }
        lam[0] = 1.0L - s;
        for (int c = 0; c < nb; ++c) {
            long double f[4], df[4];   // factor of coordinate i and its derivative in lambda_i
            for (int i = 0; i <= d; ++i) {
                long double v = 1.0L, dv = 0.0L;
                for (int m = 0; m < A[c][i]; ++m) {
                    const long double t = ((long double)k * lam[i] - m) / (m + 1);
                    dv = dv * t + v * (long double)k / (m + 1);
                    v *= t;
                }
                f[i] = v;
                df[i] = dv;
            }
            auto dlam = [&](int i) {
                long double v = df[i];
                for (int j = 0; j <= d; ++j)
                    if (j != i) v *= f[j];
                return v;
            };
            for (int r = 0; r < d; ++r) out[((size_t)q * d + r) * nb + c] = (double)(dlam(r + 1) - dlam(0));
        }
    }
}

// Simplex vertex offsets ({0,1}^d) of the d! simplices of one cell (reading L3).
inline std::vector<std::array<std::array<int, 3>, 4>> cell_simplices(int d) {
    std::vector<std::array<std::array<int, 3>, 4>> out;
    if (d == 2) {
        out.push_back({{{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 0, 0}}});
        out.push_back({{{0, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 0}}});
        return out;
    }
    const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (auto& pm : perms) {
        std::array<std::array<int, 3>, 4> s{};
        std::array<int, 3> o{0, 0, 0};
        s[0] = o;
        for (int i = 0; i < 3; ++i) { o[pm[i]] += 1; s[i + 1] = o; }
        out.push_back(s);
    }
    return out;
}

}  // namespace dogip
