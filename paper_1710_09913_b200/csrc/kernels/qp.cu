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

template <int D, int P, int F, bool DIR>
__global__ void __launch_bounds__(QP_THREADS) qp_apply_kernel(QpArgs a, const ApplyTables tab) {
    using RE = dogip_gen::RefElem<D, P, 0, 0>;          // V-side constants (V_T, ALPHA)
    constexpr int VT = RE::VT;
    constexpr int NSYM = D * (D + 1) / 2;
    constexpr int TW = F == 0 ? VT : D * VT;            // table doubles per point
    const SlabGeo& g = a.geo;
    // the basis table of the rule, staged once per CTA (persistent grid): per point the
    // warp reads the same row -> shared-memory broadcast, vectorised along l
    // (3D P4 EL exceeds shared memory: points >= nq_s are read from global / L1)
    extern __shared__ __align__(16) double tsm[];
    const double* tglob = F == 0 ? a.phi : a.dphi;
    const int nq_s = a.nq_smem;
    for (int i = threadIdx.x; i < nq_s * TW; i += blockDim.x) tsm[i] = tglob[i];
    __syncthreads();
    const int64_t e_begin = a.tile_begin * TILE, e_end = a.tile_end * TILE;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const bool cellconst = a.kind == DOGIP_COEF_CONST || a.kind == DOGIP_COEF_PER_CELL ||
                           a.kind == DOGIP_COEF_CONST_TENSOR;
    double udot = 0.0;
    for (int64_t eK = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; eK < e_end; eK += stride) {
        const int64_t tile = eK / TILE;
        const int lane = (int)(eK % TILE);
        const TileCoord tc = tile_coord(g, tile);
        const int ci = tc.ci0 + lane;
        if (ci >= g.Nx) continue;
        const Geo G = element_geo<D>(g, a.verts, eK, nullptr);
        const int64_t base = (int64_t)g.p * (ci + g.sy * tc.cj + g.sz * tc.ck);
        const int v1 = tab.vstr[tc.s][0], v2 = tab.vstr[tc.s][1], v3 = D == 3 ? tab.vstr[tc.s][2] : 0;
        uint64_t skip = 0;
        if constexpr (DIR) {
            const unsigned long long* fm = tab.fmask[tc.s];
            if (ci == 0) skip |= fm[0];
            if (ci == g.Nx - 1) skip |= fm[1];
            if (D == 3) {
                if (tc.cj == 0) skip |= fm[2];
                if (tc.cj == g.Ny - 1) skip |= fm[3];
                if (tc.ck == 0 && g.bnd_lo) skip |= fm[4];
                if (tc.ck == g.Nz - 1 && g.bnd_hi) skip |= fm[5];
            } else {
                if (tc.cj == 0 && g.bnd_lo) skip |= fm[2];
                if (tc.cj == g.Ny - 1 && g.bnd_hi) skip |= fm[3];
            }
        }
        int off[VT];
        double uT[VT], yT[VT];
        alpha_offsets<RE>(off, v1, v2, v3);
#pragma unroll
        for (int l = 0; l < VT; ++l) {
            uT[l] = ((skip >> l) & 1ull) ? 0.0 : __ldg(a.u + base + off[l]);
            yT[l] = 0.0;
        }
        const double adet = fabs(G.det);
        double cc[6];
        if (cellconst) coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, G.S, cc);
        if constexpr (F == 0) {
            // WP (eq:bilf_gp P:189): h_q = w_q |det| m(x_q) u(x_q)
            for (int q = 0; q < a.nq; ++q) {
                const double* ph = (q < nq_s ? tsm : tglob) + (size_t)q * VT;
                double v = 0.0;
#pragma unroll
                for (int l = 0; l < VT; ++l) v = fma(ph[l], uT[l], v);
                double m = cc[0];
                if (!cellconst) {
                    double x[3] = {G.S[0], G.S[1], G.S[2]};
#pragma unroll
                    for (int r = 0; r < D; ++r)
#pragma unroll
                        for (int c = 0; c < D; ++c) x[r] += G.R[r][c] * __ldg(a.qp + q * D + c);
                    double cv[6];
                    coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, x, cv);
                    m = cv[0];
                }
                const double h = __ldg(a.qw + q) * adet * m * v;
                // the projection re-reads the row from shared memory (keeping V_T table values
                // live next to u_T and y_T would spill for 3D P3/P4)
#pragma unroll
                for (int l = 0; l < VT; ++l) yT[l] = fma(ph[l], h, yT[l]);
            }
        } else {
            // EL (eq:bilf_se P:316): h_q = w_q K(x_q) gradhat u(x_q),
            // K = |det| R^-1 M(x_q) R^-T (chain rule P:172-175)
            double K[NSYM];
            auto congruence = [&](const double* cv, double* Kout) {
                double M[D][D];
                int o = 0;
                if (a.ncomp == 1) {
#pragma unroll
                    for (int r = 0; r < D; ++r)
#pragma unroll
                        for (int s = 0; s < D; ++s) M[r][s] = r == s ? cv[0] : 0.0;
                } else {
#pragma unroll
                    for (int r = 0; r < D; ++r)
#pragma unroll
                        for (int s = r; s < D; ++s) { M[r][s] = M[s][r] = cv[o++]; }
                }
                o = 0;
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int s = r; s < D; ++s) {
                        double v = 0.0;
#pragma unroll
                        for (int p2 = 0; p2 < D; ++p2) {
                            double tt = 0.0;
#pragma unroll
                            for (int q2 = 0; q2 < D; ++q2) tt = fma(M[p2][q2], G.Rinv[s][q2], tt);
                            v = fma(G.Rinv[r][p2], tt, v);
                        }
                        Kout[o++] = adet * v;
                    }
            };
            if (cellconst) congruence(cc, K);
            for (int q = 0; q < a.nq; ++q) {
                const double* dp = (q < nq_s ? tsm : tglob) + (size_t)q * D * VT;
                double gr[D];
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    double s = 0.0;
#pragma unroll
                    for (int l = 0; l < VT; ++l) s = fma(dp[r * VT + l], uT[l], s);
                    gr[r] = s;
                }
                if (!cellconst) {
                    double x[3] = {G.S[0], G.S[1], G.S[2]};
#pragma unroll
                    for (int r = 0; r < D; ++r)
#pragma unroll
                        for (int c = 0; c < D; ++c) x[r] += G.R[r][c] * __ldg(a.qp + q * D + c);
                    double cv[6];
                    coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, x, cv);
                    congruence(cv, K);
                }
                const double wq = __ldg(a.qw + q);
                double h[D];
                int o = 0;
                double Kf[D][D];
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int s = r; s < D; ++s) { Kf[r][s] = Kf[s][r] = K[o++]; }
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    double s = 0.0;
#pragma unroll
                    for (int c = 0; c < D; ++c) s = fma(Kf[r][c], gr[c], s);
                    h[r] = wq * s;
                }
#pragma unroll
                for (int l = 0; l < VT; ++l) {
                    double s = yT[l];
#pragma unroll
                    for (int r = 0; r < D; ++r) s = fma(dp[r * VT + l], h[r], s);
                    yT[l] = s;
                }
            }
        }
#pragma unroll
        for (int l = 0; l < VT; ++l) {
            if (!((skip >> l) & 1ull)) red_add_f64(a.y + base + off[l], yT[l]);
            udot = fma(uT[l], yT[l], udot);
        }
    }
    if (a.dot_partials) {
        for (int o = 16; o > 0; o >>= 1) udot += __shfl_xor_sync(0xffffffffu, udot, o);
        if ((threadIdx.x & 31) == 0) a.dot_partials[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = udot;
    }
}

template <int D, int P, int F, bool DIR>
cudaError_t launch_qp_one(const QpArgs& a) {
    auto kern = qp_apply_kernel<D, P, F, DIR>;
    constexpr int VT = dogip_gen::RefElem<D, P, 0, 0>::VT;
    constexpr int TW = F == 0 ? VT : D * VT;
    QpArgs b = a;
    b.nq_smem = a.nq < QP_SMEM_MAX / (int)(8 * TW) ? a.nq : QP_SMEM_MAX / (8 * TW);
    const size_t smem = sizeof(double) * (size_t)b.nq_smem * TW;
    static size_t configured = 0;
    static int occ = 0;
    if (configured != smem) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, QP_THREADS, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        configured = smem;
    }
    const int64_t nel = (a.tile_end - a.tile_begin) * TILE;
    int64_t grid = (int64_t)a.num_sms * occ;
    const int64_t need = (nel + QP_THREADS - 1) / QP_THREADS;
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

template <int D, int P>
cudaError_t launch_qp_dp(const QpArgs& a) {
    if (a.form == 0) return launch_qp_one<D, P, 0, false>(a);
    return a.dirichlet ? launch_qp_one<D, P, 1, true>(a) : launch_qp_one<D, P, 1, false>(a);
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
