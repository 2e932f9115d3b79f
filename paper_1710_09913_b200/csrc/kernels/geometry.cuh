// geometry.cuh -- per-element affine geometry and coefficient models, shared by the
// DoGIP weights kernels (weights.cu) and the quadrature-point matrix-free comparator
// (qp.cu).  F_T(xhat) = v_0 + R_T xhat, R_T = [v_1 - v_0, ..., v_d - v_0] (reading L6).
#pragma once
#include <cmath>
#include <cstdint>

#include "../../../include/dogip.h"
#include "common.cuh"

namespace dogip {
namespace {

struct Geo {
    double R[3][3], Rinv[3][3], S[3], det;
    int64_t cell;     // global cell index
    bool valid;
};

// Simplex vertex offsets of one cell (reading L3): 2D right split, 3D Kuhn (vertex v
// = sum of the first v axes of permutation s, permutations in lexicographic order).
// Compile-time D and register arithmetic only (no dynamically indexed local arrays).
template <int D>
__device__ __forceinline__ void simplex_offset(int s, int v, int o[3]) {
    o[0] = o[1] = o[2] = 0;
    if (v == 0) return;
    if constexpr (D == 2) {
        if (s == 0) { o[0] = 1; o[1] = (v == 2); }
        else { o[1] = 1; o[0] = (v == 1); }
    } else {
        // axes of permutation s packed 2 bits each, 6 bits per permutation:
        // {0,1,2},{0,2,1},{1,0,2},{1,2,0},{2,0,1},{2,1,0}
        constexpr unsigned long long PACK = (0ull | 1ull << 2 | 2ull << 4) | (0ull | 2ull << 2 | 1ull << 4) << 6 |
                                            (1ull | 0ull << 2 | 2ull << 4) << 12 | (1ull | 2ull << 2 | 0ull << 4) << 18 |
                                            (2ull | 0ull << 2 | 1ull << 4) << 24 | (2ull | 1ull << 2 | 0ull << 4) << 30;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int ax = (int)((PACK >> (6 * s + 2 * i)) & 3ull);
            const int add = i < v ? 1 : 0;
            o[0] += ax == 0 ? add : 0;
            o[1] += ax == 1 ? add : 0;
            o[2] += ax == 2 ? add : 0;
        }
    }
}

template <int D>
__device__ __forceinline__ Geo element_geo(const SlabGeo& g, const double* verts, int64_t eK, int* bad) {
    Geo G;
    const int64_t tile = eK / TILE;
    const int lane = (int)(eK % TILE);
    const TileCoord tc = tile_coord(g, tile);
    const int ci = tc.ci0 + lane;
    G.valid = ci < g.Nx;
    int64_t c[3] = {ci, tc.cj, tc.ck};
    if (D == 2) c[1] += g.zoff; else c[2] += g.zoff;
    if (!G.valid) c[0] = 0;
    G.cell = D == 2 ? c[0] + (int64_t)g.N * c[1] : c[0] + (int64_t)g.N * (c[1] + (int64_t)g.N * c[2]);
    const int64_t M = g.N + 1;
    double X[D + 1][D];
    int lat[D + 1][D];
#pragma unroll
    for (int v = 0; v <= D; ++v) {
        int o[3];
        simplex_offset<D>(tc.s, v, o);
        int64_t vid = 0, mul = 1;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            lat[v][a] = o[a];
            vid += (c[a] + o[a]) * mul;
            mul *= M;
        }
#pragma unroll
        for (int a = 0; a < D; ++a)
            X[v][a] = verts ? verts[vid * D + a] : (double)(c[a] + o[a]) / (double)g.N;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        G.S[a] = 0.0;
#pragma unroll
        for (int b = 0; b < 3; ++b) { G.R[a][b] = (a == b) ? 1.0 : 0.0; G.Rinv[a][b] = (a == b) ? 1.0 : 0.0; }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        G.S[a] = X[0][a];
#pragma unroll
        for (int b = 0; b < D; ++b) G.R[a][b] = X[b + 1][a] - X[0][a];   // columns v_b - v_0
    }
    int Rl[3][3];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Rl[a][b] = lat[b + 1][a] - lat[0][a];
    int detl;
    if constexpr (D == 2) {
        G.det = G.R[0][0] * G.R[1][1] - G.R[0][1] * G.R[1][0];
        detl = Rl[0][0] * Rl[1][1] - Rl[0][1] * Rl[1][0];
        const double id = 1.0 / G.det;
        G.Rinv[0][0] = G.R[1][1] * id;  G.Rinv[0][1] = -G.R[0][1] * id;
        G.Rinv[1][0] = -G.R[1][0] * id; G.Rinv[1][1] = G.R[0][0] * id;
    } else {
        const double (*R)[3] = G.R;
        const double c00 = R[1][1] * R[2][2] - R[1][2] * R[2][1];
        const double c01 = R[1][2] * R[2][0] - R[1][0] * R[2][2];
        const double c02 = R[1][0] * R[2][1] - R[1][1] * R[2][0];
        G.det = R[0][0] * c00 + R[0][1] * c01 + R[0][2] * c02;
        detl = Rl[0][0] * (Rl[1][1] * Rl[2][2] - Rl[1][2] * Rl[2][1]) -
               Rl[0][1] * (Rl[1][0] * Rl[2][2] - Rl[1][2] * Rl[2][0]) +
               Rl[0][2] * (Rl[1][0] * Rl[2][1] - Rl[1][1] * Rl[2][0]);
        const double id = 1.0 / G.det;
        G.Rinv[0][0] = c00 * id;
        G.Rinv[1][0] = c01 * id;
        G.Rinv[2][0] = c02 * id;
        G.Rinv[0][1] = (R[0][2] * R[2][1] - R[0][1] * R[2][2]) * id;
        G.Rinv[1][1] = (R[0][0] * R[2][2] - R[0][2] * R[2][0]) * id;
        G.Rinv[2][1] = (R[0][1] * R[2][0] - R[0][0] * R[2][1]) * id;
        G.Rinv[0][2] = (R[0][1] * R[1][2] - R[0][2] * R[1][1]) * id;
        G.Rinv[1][2] = (R[0][2] * R[1][0] - R[0][0] * R[1][2]) * id;
        G.Rinv[2][2] = (R[0][0] * R[1][1] - R[0][1] * R[1][0]) * id;
    }
    if (bad && G.valid && !(G.det * (double)detl > 0.0)) atomicOr(bad, 1);   // E_DEGENERATE_ELEMENT
    return G;
}

// coefficient components at physical point x: isotropic -> out[0] = m;
// tensor -> upper triangle row-major (2D: 3, 3D: 6 values)
template <int D>
__device__ __forceinline__ void coef_eval(int kind, const double* P, const double* per_cell, int64_t cell,
                                          const double* x, double* out) {
    constexpr int d = D;
    switch (kind) {
        case DOGIP_COEF_CONST: out[0] = P[0]; return;
        case DOGIP_COEF_PER_CELL: out[0] = per_cell[cell]; return;
        case DOGIP_COEF_SINCOS2D:
            out[0] = P[0] + P[1] * sin(2.0 * M_PI * x[0]) * cos(2.0 * M_PI * x[1]);
            return;
        case DOGIP_COEF_TANH_RADIAL: {
            double r2 = 0.0;
#pragma unroll
            for (int a = 0; a < d; ++a) { const double t = x[a] - P[4 + a]; r2 += t * t; }
            out[0] = P[0] + P[1] * tanh(P[2] * (sqrt(r2) - P[3]));
            return;
        }
        case DOGIP_COEF_ANISO_FOURIER: {
            const int n = (int)P[3];
            const double* kap = P + 4;
            const double* cc = P + 4 + 6 * n;
            double w[3] = {0.0, 0.0, 0.0};
            for (int m = 0; m < n; ++m) {
                // cos(arg + phi_i) = cos(arg) cos(phi_i) - sin(arg) sin(phi_i): one sincos per
                // mode instead of three cos (the phases are per-parameter constants)
                const double arg = 2.0 * M_PI * (x[0] * kap[3 * m] + x[1] * kap[3 * m + 1] + x[2] * kap[3 * m + 2]);
                double sa, ca;
                sincos(arg, &sa, &ca);
                const double* cphi = P + 4 + 9 * n;      // cos / sin of the phases (appended by
                const double* sphi = cphi + 3 * n;       // the host, abi.cu device_params)
#pragma unroll
                for (int i = 0; i < 3; ++i) w[i] += cc[3 * m + i] * (ca * cphi[3 * m + i] - sa * sphi[3 * m + i]);
            }
            double R[3][3];
            const double t = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
            if (t < 1e-12) {
                R[0][0] = 1; R[0][1] = -w[2]; R[0][2] = w[1];
                R[1][0] = w[2]; R[1][1] = 1; R[1][2] = -w[0];
                R[2][0] = -w[1]; R[2][1] = w[0]; R[2][2] = 1;
            } else {
                const double k0 = w[0] / t, k1 = w[1] / t, k2 = w[2] / t;
                const double K[3][3] = {{0, -k2, k1}, {k2, 0, -k0}, {-k1, k0, 0}};
                const double st = sin(t), ct1 = 1.0 - cos(t);
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) {
                        double k2ab = 0.0;
                        for (int c = 0; c < 3; ++c) k2ab += K[a][c] * K[c][b];
                        R[a][b] = (a == b ? 1.0 : 0.0) + st * K[a][b] + ct1 * k2ab;
                    }
            }
            int o = 0;
            for (int a = 0; a < 3; ++a)
                for (int b = a; b < 3; ++b) {
                    double s = 0.0;
                    for (int c = 0; c < 3; ++c) s += R[a][c] * P[c] * R[b][c];
                    out[o++] = s;
                }
            return;
        }
        case DOGIP_COEF_CONST_TENSOR: {
            int o = 0;
#pragma unroll
            for (int a = 0; a < d; ++a)
#pragma unroll
                for (int b = a; b < d; ++b) out[o++] = P[a * d + b];
            return;
        }
    }
}

__device__ __forceinline__ bool coef_ok(int ncomp, int d, const double* c) {
    if (ncomp == 1) return c[0] > 0.0;
    return d == 2 ? (c[0] > 0.0 && c[2] > 0.0) : (c[0] > 0.0 && c[3] > 0.0 && c[5] > 0.0);
}

}  // namespace
}  // namespace dogip
