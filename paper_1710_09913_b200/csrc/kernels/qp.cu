// qp.cu -- the quadrature-point matrix-free comparator (PAPER.md "Alternative
// approaches"): the element-wise product A_T u_T evaluated on the fly over the
// integration points, with no stored operator data,
//   grad u(x_q) = J_T^{-T} sum_i gradhat phihat_i(xhat_q) u_{T,i},
//   (A_T u_T)_l = sum_q A(x_q) grad u(x_q) . grad phi_l(x_q) w_q |det J_T|          (EL)
//   (A_T u_T)_l = sum_q m(x_q) u(x_q) phi_l(x_q) w_q |det J_T|                        (WP)
// with the same contract rule Q (reading L10) as the DoGIP weights, so it reproduces
// the same Galerkin matrix A and is parity-tested against the same
// oracle.  It exists to measure the DoGIP-vs-quadrature trade-off the paper argues
// qualitatively on the same hardware: DoGIP streams W_T n_c weights
// per element, the comparator re-evaluates geometry, coefficient and (V_T x n_q) basis
// contractions every apply.
//
// Mapping: one thread = one element (canonical tile order, 32 elements of one simplex
// type per warp, so the gather offsets and the table rows are warp-uniform); the basis
// table phihat(xhat_q) (WP) or gradhat phihat(xhat_q) (EL) of the rule is staged in
// shared memory once per persistent CTA and read per point as a broadcast; geometry from the lattice or the jittered vertex
// array; the coefficient from coef_eval (geometry.cuh) at every point, or once per
// element when it is cell-constant (K_T = |det| R^-1 M R^-T, reading L6).
#include <cuda_runtime.h>

#ifdef DOGIP_GEN_HEADER
#include DOGIP_GEN_HEADER
#else
#include "../generated/bhat_gen.cuh"
#endif
#include "apply.cuh"
#include "common.cuh"
#include "geometry.cuh"

namespace dogip {
namespace {

constexpr int QP_THREADS = 128;
constexpr int QP_SMEM_MAX = 200 * 1024;   // shared-memory budget of the staged basis table

// off[l] = sum_i alpha_i(l) v_i (v_0 = cell origin), compile-time alpha
template <class RE, int L = 0>
__device__ __forceinline__ void alpha_offsets(int* off, int v1, int v2, int v3) {
    if constexpr (L < RE::VT) {
        off[L] = RE::ALPHA[L][0] * v1 + RE::ALPHA[L][1] * v2 + RE::ALPHA[L][2] * v3;
        alpha_offsets<RE, L + 1>(off, v1, v2, v3);
    }
}

// projection-pass read of a basis-table row: an opaque load, so the compiler re-reads the
// row instead of keeping the interpolation pass's D x V_T values live (spills)
__device__ __forceinline__ double ld_again(const double* p) {
    double v;
    asm volatile("ld.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// elements per thread: each basis-table row read from shared memory serves E elements
// (register blocking; E = 2 where u_T, y_T of both fit next to the point work)
template <int VT, int F>
__host__ __device__ constexpr int qp_ept() { return (F == 0 ? VT <= 20 : VT <= 10) ? 2 : 1; }

// per-element state of the comparator
// per-element state of the comparator; the geometry is kept only when the coefficient
// varies inside the element (CC = false: evaluated at every point)
template <int D, int VT, bool CC>
struct QpElem;
template <int D, int VT>
struct QpElem<D, VT, true> {
    int64_t base;
    int s;                       // simplex type (gather / scatter offsets are recomputed)
    uint64_t skip;
    bool valid;
    double K[D * (D + 1) / 2];   // EL: |det| R^-1 M R^-T;  WP: K[0] = |det| m
};
template <int D, int VT>
struct QpElem<D, VT, false> {
    int64_t base;
    int s;
    uint64_t skip;
    bool valid;
    double K[D * (D + 1) / 2];
    Geo G;
};

template <int D, int P, int F, bool DIR, bool CC>
__global__ void __launch_bounds__(QP_THREADS) qp_apply_kernel(QpArgs a, const ApplyTables tab) {
    using RE = dogip_gen::RefElem<D, P, 0, 0>;          // V-side constants (V_T, ALPHA)
    constexpr int VT = RE::VT;
    constexpr int NSYM = D * (D + 1) / 2;
    constexpr int TW = F == 0 ? VT : D * VT;            // table doubles per point
    constexpr int E = CC ? qp_ept<VT, F>() : 1;
    const SlabGeo& g = a.geo;
    // the basis table of the rule, staged once per CTA (persistent grid): per point the
    // warp reads the same row -> shared-memory broadcast, vectorised along l
    // (3D P4 EL exceeds shared memory: points >= nq_s are read from global / L1)
    extern __shared__ __align__(16) double tsm[];
    const double* tglob = F == 0 ? a.phi : a.dphi;
    const int nq_s = a.nq_smem;
    for (int i = threadIdx.x; i < nq_s * TW; i += blockDim.x) tsm[i] = tglob[i];
    __syncthreads();
    // K = |det| R^-1 M R^-T (reading L6, chain rule P:172-175), upper triangle
    auto congruence = [&](const Geo& G, const double* cv, double* Kout) {
        double M[D][D];
        int o = 0;
        if (a.ncomp == 1) {
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int s2 = 0; s2 < D; ++s2) M[r][s2] = r == s2 ? cv[0] : 0.0;
        } else {
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int s2 = r; s2 < D; ++s2) { M[r][s2] = M[s2][r] = cv[o++]; }
        }
        o = 0;
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int s2 = r; s2 < D; ++s2) {
                double v = 0.0;
#pragma unroll
                for (int p2 = 0; p2 < D; ++p2) {
                    double tt = 0.0;
#pragma unroll
                    for (int q2 = 0; q2 < D; ++q2) tt = fma(M[p2][q2], G.Rinv[s2][q2], tt);
                    v = fma(G.Rinv[r][p2], tt, v);
                }
                Kout[o++] = fabs(G.det) * v;
            }
    };
    // element groups: E consecutive tiles x 32 lanes; thread (group, lane) owns element
    // lane of each tile of the group
    const int64_t t_begin = a.tile_begin, t_end = a.tile_end;
    const int64_t ngroups = (t_end - t_begin + E - 1) / E;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    double udot = 0.0;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < ngroups * TILE; it += nthr) {
        const int64_t grp = it / TILE;
        const int lane = (int)(it % TILE);
        QpElem<D, VT, CC> el[E];
        double uT[E][VT], yT[E][VT];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t tile = t_begin + grp * E + e;
            QpElem<D, VT, CC>& X = el[e];
            X.valid = false;
            X.skip = 0;
#pragma unroll
            for (int l = 0; l < VT; ++l) { uT[e][l] = 0.0; yT[e][l] = 0.0; }
            if (tile >= t_end) continue;
            const TileCoord tc = tile_coord(g, tile);
            const int ci = tc.ci0 + lane;
            if (ci >= g.Nx) continue;
            X.valid = true;
            const Geo G = element_geo<D>(g, a.verts, tile * TILE + lane, nullptr);
            if constexpr (!CC) X.G = G;
            X.base = (int64_t)g.p * (ci + g.sy * tc.cj + g.sz * tc.ck);
            X.s = tc.s;
            int off[VT];
            alpha_offsets<RE>(off, tab.vstr[tc.s][0], tab.vstr[tc.s][1], D == 3 ? tab.vstr[tc.s][2] : 0);
            if constexpr (DIR) {
                const unsigned long long* fm = tab.fmask[tc.s];
                if (ci == 0) X.skip |= fm[0];
                if (ci == g.Nx - 1) X.skip |= fm[1];
                if (D == 3) {
                    if (tc.cj == 0) X.skip |= fm[2];
                    if (tc.cj == g.Ny - 1) X.skip |= fm[3];
                    if (tc.ck == 0 && g.bnd_lo) X.skip |= fm[4];
                    if (tc.ck == g.Nz - 1 && g.bnd_hi) X.skip |= fm[5];
                } else {
                    if (tc.cj == 0 && g.bnd_lo) X.skip |= fm[2];
                    if (tc.cj == g.Ny - 1 && g.bnd_hi) X.skip |= fm[3];
                }
            }
#pragma unroll
            for (int l = 0; l < VT; ++l)
                uT[e][l] = ((X.skip >> l) & 1ull) ? 0.0 : __ldg(a.u + X.base + off[l]);
            if constexpr (CC) {
                double cc[6];
                coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, G.S, cc);
                if constexpr (F == 1) congruence(G, cc, X.K);
                else X.K[0] = fabs(G.det) * cc[0];
            }
        }
        auto coef_at = [&](const Geo& G, int q, double* cv) {
            double x[3] = {G.S[0], G.S[1], G.S[2]};
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int c = 0; c < D; ++c) x[r] += G.R[r][c] * __ldg(a.qp + q * D + c);
            coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, x, cv);
        };
        for (int q = 0; q < a.nq; ++q) {
            const double wq = __ldg(a.qw + q);
            if constexpr (F == 0) {
                // WP (eq:bilf_gp P:189): h_q = w_q |det| m(x_q) u(x_q)
                const double* ph = (q < nq_s ? tsm : tglob) + (size_t)q * VT;
                double v[E];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = 0.0;
#pragma unroll
                for (int l = 0; l < VT; ++l) {
                    const double t = ph[l];
#pragma unroll
                    for (int e = 0; e < E; ++e) v[e] = fma(t, uT[e][l], v[e]);
                }
                double h[E];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    double dm = 0.0;          // |det| m(x_q)
                    if constexpr (CC) {
                        dm = el[e].K[0];
                    } else if (el[e].valid) {
                        double cv[6];
                        coef_at(el[e].G, q, cv);
                        dm = fabs(el[e].G.det) * cv[0];
                    }
                    h[e] = el[e].valid ? wq * dm * v[e] : 0.0;
                }
                // the projection re-reads the row (keeping V_T table values live next to
                // u_T and y_T would spill)
#pragma unroll
                for (int l = 0; l < VT; ++l) {
                    const double t = ld_again(ph + l);
#pragma unroll
                    for (int e = 0; e < E; ++e) yT[e][l] = fma(t, h[e], yT[e][l]);
                }
            } else {
                // EL (eq:bilf_se P:316): h_q = w_q K(x_q) gradhat u(x_q)
                const double* dp = (q < nq_s ? tsm : tglob) + (size_t)q * D * VT;
                double gr[E][D];
#pragma unroll
                for (int e = 0; e < E; ++e)
#pragma unroll
                    for (int r = 0; r < D; ++r) gr[e][r] = 0.0;
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int l = 0; l < VT; ++l) {
                        const double t = dp[r * VT + l];
#pragma unroll
                        for (int e = 0; e < E; ++e) gr[e][r] = fma(t, uT[e][l], gr[e][r]);
                    }
                double h[E][D];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    double Kq[NSYM];
#pragma unroll
                    for (int k = 0; k < NSYM; ++k) Kq[k] = 0.0;
                    if constexpr (CC) {
#pragma unroll
                        for (int k = 0; k < NSYM; ++k) Kq[k] = el[e].K[k];
                    } else if (el[e].valid) {
                        double cv[6];
                        coef_at(el[e].G, q, cv);
                        congruence(el[e].G, cv, Kq);
                    }
                    double Kf[D][D];
                    int o = 0;
#pragma unroll
                    for (int r = 0; r < D; ++r)
#pragma unroll
                        for (int s2 = r; s2 < D; ++s2) { Kf[r][s2] = Kf[s2][r] = Kq[o++]; }
#pragma unroll
                    for (int r = 0; r < D; ++r) {
                        double acc = 0.0;
#pragma unroll
                        for (int c = 0; c < D; ++c) acc = fma(Kf[r][c], gr[e][c], acc);
                        h[e][r] = el[e].valid ? wq * acc : 0.0;
                    }
                }
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int l = 0; l < VT; ++l) {
                        const double t = ld_again(dp + r * VT + l);
#pragma unroll
                        for (int e = 0; e < E; ++e) yT[e][l] = fma(t, h[e][r], yT[e][l]);
                    }
            }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (!el[e].valid) continue;
            int off[VT];
            const int sx = el[e].s;
            alpha_offsets<RE>(off, tab.vstr[sx][0], tab.vstr[sx][1], D == 3 ? tab.vstr[sx][2] : 0);
#pragma unroll
            for (int l = 0; l < VT; ++l) {
                if (!((el[e].skip >> l) & 1ull)) red_add_f64(a.y + el[e].base + off[l], yT[e][l]);
                udot = fma(uT[e][l], yT[e][l], udot);
            }
        }
    }
    if (a.dot_partials) {
        for (int o = 16; o > 0; o >>= 1) udot += __shfl_xor_sync(0xffffffffu, udot, o);
        if ((threadIdx.x & 31) == 0) a.dot_partials[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = udot;
    }
}

template <int D, int P, int F, bool DIR, bool CC>
cudaError_t launch_qp_one(const QpArgs& a) {
    auto kern = qp_apply_kernel<D, P, F, DIR, CC>;
    constexpr int VT = dogip_gen::RefElem<D, P, 0, 0>::VT;
    constexpr int TW = F == 0 ? VT : D * VT;
    QpArgs b = a;
    b.nq_smem = a.nq < QP_SMEM_MAX / (int)(8 * TW) ? a.nq : QP_SMEM_MAX / (8 * TW);
    const size_t smem = sizeof(double) * (size_t)b.nq_smem * TW;
    static std::atomic<uint64_t> cfg[MAX_DEVICES];   // per instantiation, per device (keyed on smem)
    int occ = 1;
    if (cudaError_t e = kernel_occupancy(kern, QP_THREADS, smem, cfg, &occ); e != cudaSuccess) return e;
    const int64_t nel = (a.tile_end - a.tile_begin) * TILE;
    constexpr int E = CC ? qp_ept<VT, F>() : 1;
    int64_t grid = (int64_t)a.num_sms * occ;
    const int64_t need = ((a.tile_end - a.tile_begin + E - 1) / E * TILE + QP_THREADS - 1) / QP_THREADS;
    if (grid > need) grid = need;
    constexpr int NW = QP_THREADS / 32;
    if (a.dot_partials) {
        if (grid < 1) grid = 1;
        if (grid * NW > APPLY_MAX_WARPS) grid = APPLY_MAX_WARPS / NW;
        *a.dot_nslots = (int)(grid * NW);
    } else if (nel <= 0) {
        return cudaSuccess;
    }
    kern<<<(unsigned)grid, QP_THREADS, smem, a.stream>>>(b, *a.tab);
    count_launches(1);
    return cudaGetLastError();
}

template <int D, int P, bool CC>
cudaError_t launch_qp_dpc(const QpArgs& a) {
    if (a.form == 0)
        return a.dirichlet ? launch_qp_one<D, P, 0, true, CC>(a) : launch_qp_one<D, P, 0, false, CC>(a);
    return a.dirichlet ? launch_qp_one<D, P, 1, true, CC>(a) : launch_qp_one<D, P, 1, false, CC>(a);
}

template <int D, int P>
cudaError_t launch_qp_dp(const QpArgs& a) {
    const bool cc = a.kind == DOGIP_COEF_CONST || a.kind == DOGIP_COEF_PER_CELL || a.kind == DOGIP_COEF_CONST_TENSOR;
    return cc ? launch_qp_dpc<D, P, true>(a) : launch_qp_dpc<D, P, false>(a);
}

template <int D>
cudaError_t launch_qp_d(const QpArgs& a) {
    switch (a.p) {
        case 1: return launch_qp_dp<D, 1>(a);
        case 2: return launch_qp_dp<D, 2>(a);
        case 3: return launch_qp_dp<D, 3>(a);
        case 4: return launch_qp_dp<D, 4>(a);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_qp_apply(const QpArgs& a) { return a.d == 2 ? launch_qp_d<2>(a) : launch_qp_d<3>(a); }

}  // namespace dogip
