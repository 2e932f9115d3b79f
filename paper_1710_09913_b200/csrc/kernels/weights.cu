// weights.cu -- one-time DoGIP weight kernels (sm_100a).
//
//   WP  a_{T,j} = |det R_T| sum_q w_q m(F_T xq) phi^W_j(xq)               (Theorem 2)
//   EL  A_{T,j} = Rinv_T (|det R_T| sum_q w_q M(F_T xq) phi^W_j(xq)) Rinv_T^T (Theorem 4)
// with the collapsed Gauss-Jacobi rule Q (reading L10).  Three steps per batch
// of elements (K-order = apply-kernel tile order):
//   1. quad_coef : C[e, c, q] = |det R_T| w_q M_c(F_T xq)      (c = coefficient component)
//   2. gemm      : Abar[j, e, c] = sum_q C[e, c, q] Phi[q, j]   (smem-tiled FP64 DMMA GEMM,
//                  stored transposed so step 3 reads it coalesced along e)
//   3. finalize  : congruence with Rinv_T (EL) and the tile-major store [tile][j*NC+c][lane]
// Cell-constant coefficients skip 1-2: Abar = |det R_T| M_T s_j, s_j = sum_q w_q phi^W_j(xq).
#include <cuda_runtime.h>

#include "../../../include/dogip.h"
#include "apply.cuh"
#include "common.cuh"
#include "geometry.cuh"

namespace dogip {
namespace {

// 1. CT[q][e*ncomp + c] = |det| w_q M_c(x_q)   (element index fastest: coalesced stores,
//    and the GEMM's A operand read along M)
template <int D, int KIND>
__global__ void quad_coef_kernel(WeightsArgs a, int64_t e0, int64_t nb) {
    // one thread per element (geometry once), looping over the points; for a fixed point
    // consecutive threads write consecutive elements
    const int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (el >= nb) return;
    const Geo G = element_geo<D>(a.geo, a.verts, e0 + el, a.bad_flag);
    const double adet = G.valid ? fabs(G.det) : 0.0;
    const int64_t M = nb * a.ncomp;
    bool ok = true;
    for (int q = 0; q < a.nq; ++q) {
        double x[3] = {0, 0, 0};
#pragma unroll
        for (int r = 0; r < D; ++r) {
            x[r] = G.S[r];
#pragma unroll
            for (int c = 0; c < D; ++c) x[r] += G.R[r][c] * a.qp[q * D + c];
        }
        double cv[6];
        coef_eval<D>(KIND < 0 ? a.kind : KIND, a.params, a.per_cell, G.cell, x, cv);   // switch folded per KIND
        ok = ok && coef_ok(a.ncomp, D, cv);
        const double sc = adet * a.qw[q];
        for (int c = 0; c < a.ncomp; ++c) a.scratch_c[(int64_t)q * M + el * a.ncomp + c] = sc * cv[c];
    }
    if (G.valid && !ok) atomicOr(a.bad_flag, 2);
}

// 2. C^T (N x M) with C = A^T (K x M)^T * B (K x N), FP64 on the FP64 tensor path
//    (mma.sync.aligned.m8n8k4.f64, DMMA -- sm_100a has no tcgen05 f64 kind): block tile
//    64 (M) x 56 (N), 4 warps each owning 2 x 7 m8n8 accumulator tiles, K in steps of
//    16 through padded shared memory (row stride 68 / 60 doubles: a fragment load is the
//    optimal 2 wavefronts).  N = W_T: 165 (C5) -> 3 column blocks of 56 (2 % padding).
constexpr int GBM = 64, GBN = 56, GK = 16, GPA = GBM + 4, GPB = GBN + 4;
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
#ifndef DOGIP_GEMM_MINB
#define DOGIP_GEMM_MINB 1
#endif
__global__ void __launch_bounds__(128, DOGIP_GEMM_MINB) gemm_kernel(const double* __restrict__ AT, const double* __restrict__ B,
                                                   double* __restrict__ C, int64_t M, int N, int K) {
    __shared__ __align__(16) double As[GK][GPA];
    __shared__ __align__(16) double Bs[GK][GPB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // column tile fastest: the NT CTAs sharing one A row block run together, so the
    // block is read from DRAM once and re-read from L2 (not NT times from DRAM)
    const int NT = (N + GBN - 1) / GBN;
    const int64_t m0 = (int64_t)(blockIdx.x / NT) * GBM;
    const int n0 = (int)(blockIdx.x % NT) * GBN;
    double acc[2][7][2] = {};
    // register-staged double buffering: the next K slab's global loads are in flight
    // while this slab's DMMAs run
    constexpr int LA = GBM * GK / 128, LB = GBN * GK / 128;
    double ra[LA], rb[LB];
    auto load = [&](int k0) {
#pragma unroll
        for (int r = 0; r < LA; ++r) {
            const int i = threadIdx.x + r * 128, kk = i / GBM, mm = i % GBM;
            const int64_t gm = m0 + mm;
            ra[r] = (gm < M && k0 + kk < K) ? AT[(int64_t)(k0 + kk) * M + gm] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < LB; ++r) {
            const int i = threadIdx.x + r * 128, kb = i / GBN, nn = i % GBN;
            rb[r] = (k0 + kb < K && n0 + nn < N) ? B[(int64_t)(k0 + kb) * N + n0 + nn] : 0.0;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int r = 0; r < LA; ++r) {
            const int i = threadIdx.x + r * 128;
            As[i / GBM][i % GBM] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < LB; ++r) {
            const int i = threadIdx.x + r * 128;
            Bs[i / GBN][i % GBN] = rb[r];
        }
    };
    load(0);
    store();
    __syncthreads();
    for (int k0 = 0; k0 < K; k0 += GK) {
        const bool more = k0 + GK < K;
        if (more) load(k0 + GK);
#pragma unroll
        for (int ks = 0; ks < GK / 4; ++ks) {
            const int kr = ks * 4 + (lane & 3);
            double af[2], bf[7];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) af[mt] = As[kr][(warp * 2 + mt) * 8 + (lane >> 2)];
#pragma unroll
            for (int nt = 0; nt < 7; ++nt) bf[nt] = Bs[kr][nt * 8 + (lane >> 2)];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 7; ++nt) dmma_884(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
        __syncthreads();
        if (more) {
            store();
            __syncthreads();
        }
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 7; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t gm = m0 + (warp * 2 + mt) * 8 + (lane >> 2);
                const int gn = n0 + nt * 8 + 2 * (lane & 3) + h;
                if (gm < M && gn < N) C[(int64_t)gn * M + gm] = acc[mt][nt][h];   // C^T: [n][m]
            }
}


// 3. congruence + tile-major store.  direct: cell-constant coefficient.
template <int D>
__global__ void finalize_kernel(WeightsArgs a, int64_t e0, int64_t nb, int direct) {
    const int64_t el = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (el >= nb) return;
    const int64_t eK = e0 + el;
    const Geo G = element_geo<D>(a.geo, a.verts, eK, a.bad_flag);
    constexpr int d = D;
    const int WT = a.WT, NC = a.NC, nc = a.ncomp;
    const int64_t tile = eK / TILE;
    const int lane = (int)(eK % TILE);
    double* out = a.out + (size_t)tile * a.tile_rows * TILE + lane;
    double cconst[6] = {0, 0, 0, 0, 0, 0};
    if (direct) {
        double x[3] = {G.S[0], G.S[1], G.S[2]};
        coef_eval<D>(a.kind, a.params, a.per_cell, G.cell, x, cconst);
        if (G.valid && !coef_ok(nc, d, cconst)) atomicOr(a.bad_flag, 2);
    }
    const double adet = fabs(G.det);
    if (a.store == 1) {
        // isotropic storage (Corollary P:411-428, element-wise): G_T = Rinv Rinv^T, then a_j
        int o = 0;
        for (int r = 0; r < d; ++r)
            for (int s = r; s < d; ++s) {
                double v = 0.0;
                for (int q = 0; q < d; ++q) v += G.Rinv[r][q] * G.Rinv[s][q];
                out[(size_t)o * TILE] = G.valid ? v : 0.0;
                ++o;
            }
        for (int j = 0; j < WT; ++j) {
            const double aj = direct ? adet * cconst[0] * a.sW[j] : a.scratch_a[(size_t)j * nb + el];
            out[(size_t)(a.NG + (a.rowperm ? a.rowperm[j] : j)) * TILE] = G.valid ? aj : 0.0;
        }
        return;
    }
    if (a.sym) {   // symmetry-adapted WP rows: ahat_psi(P) = (1/s) sum_c psi(c) a_{c j0} (STORE 5)
        auto aj = [&](int j) { return direct ? adet * cconst[0] * a.sW[j] : a.scratch_a[(size_t)j * nb + el]; };
        for (int r = 0; r < WT; ++r) {
            double v = 0.0;
            for (int k = 0; k < 4; ++k) {
                const int j = a.symj[r * 4 + k];
                if (j >= 0) v = fma(a.symc[r * 4 + k], aj(j), v);
            }
            out[(size_t)r * TILE] = G.valid ? v : 0.0;
        }
        return;
    }
    for (int j = 0; j < WT; ++j) {
        double ab[6];
        for (int c = 0; c < nc; ++c)
            ab[c] = direct ? adet * cconst[c] * a.sW[j] : a.scratch_a[(size_t)j * nb * nc + el * nc + c];
        const int row = a.rowperm ? a.rowperm[j] : j;   // FULL WP with the symmetry-adapted body: orbit order
        if (!G.valid) {
            for (int c = 0; c < NC; ++c) out[(size_t)(row * NC + c) * TILE] = 0.0;
            continue;
        }
        if (a.form == DOGIP_WP) {
            out[(size_t)row * TILE] = ab[0];
            continue;
        }
        // Abar (symmetric) -> A = Rinv Abar Rinv^T  (A_rs = Rinv_rp Abar_pq Rinv_sq)
        double Ab[3][3];
        if (nc == 1) {
            for (int p = 0; p < d; ++p)
                for (int q = 0; q < d; ++q) Ab[p][q] = p == q ? ab[0] : 0.0;
        } else {
            int o = 0;
            for (int p = 0; p < d; ++p)
                for (int q = p; q < d; ++q) { Ab[p][q] = Ab[q][p] = ab[o++]; }
        }
        int o = 0;
        for (int r = 0; r < d; ++r)
            for (int s = r; s < d; ++s) {
                double v = 0.0;
                for (int p = 0; p < d; ++p) {
                    double t = 0.0;
                    for (int q = 0; q < d; ++q) t += Ab[p][q] * G.Rinv[s][q];
                    v += G.Rinv[r][p] * t;
                }
                out[(size_t)(j * NC + o) * TILE] = v;
                ++o;
            }
    }
}

}  // namespace

cudaError_t launch_weights(const WeightsArgs& a) {
    const int64_t nel = a.geo.ntiles * TILE;
    const bool direct = a.kind == DOGIP_COEF_CONST || a.kind == DOGIP_COEF_PER_CELL ||
                        a.kind == DOGIP_COEF_CONST_TENSOR;
    for (int64_t e0 = 0; e0 < nel; e0 += a.batch) {
        const int64_t nb = (nel - e0) < a.batch ? (nel - e0) : a.batch;
        if (!direct) {
            const unsigned qb = (unsigned)((nb + 127) / 128);
            if (a.d == 2) {
                if (a.kind == DOGIP_COEF_SINCOS2D) quad_coef_kernel<2, DOGIP_COEF_SINCOS2D><<<qb, 128, 0, a.stream>>>(a, e0, nb);
                else if (a.kind == DOGIP_COEF_TANH_RADIAL) quad_coef_kernel<2, DOGIP_COEF_TANH_RADIAL><<<qb, 128, 0, a.stream>>>(a, e0, nb);
                else quad_coef_kernel<2, -1><<<qb, 128, 0, a.stream>>>(a, e0, nb);
            } else {
                if (a.kind == DOGIP_COEF_TANH_RADIAL) quad_coef_kernel<3, DOGIP_COEF_TANH_RADIAL><<<qb, 128, 0, a.stream>>>(a, e0, nb);
                else if (a.kind == DOGIP_COEF_ANISO_FOURIER) quad_coef_kernel<3, DOGIP_COEF_ANISO_FOURIER><<<qb, 128, 0, a.stream>>>(a, e0, nb);
                else quad_coef_kernel<3, -1><<<qb, 128, 0, a.stream>>>(a, e0, nb);
            }
            const int64_t M = nb * a.ncomp;
            const unsigned grid = (unsigned)(((M + GBM - 1) / GBM) * ((a.WT + GBN - 1) / GBN));
            gemm_kernel<<<grid, 128, 0, a.stream>>>(a.scratch_c, a.phiW, a.scratch_a, M, a.WT, a.nq);
        }
        if (a.d == 2) finalize_kernel<2><<<(unsigned)((nb + 127) / 128), 128, 0, a.stream>>>(a, e0, nb, direct ? 1 : 0);
        else finalize_kernel<3><<<(unsigned)((nb + 127) / 128), 128, 0, a.stream>>>(a, e0, nb, direct ? 1 : 0);
        count_launches(direct ? 1 : 3);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// ---------------------------------------------------------- global WP (Theorem 1)
namespace {
// wel != null: wg[l^W_T(j)] += a_{T,j};  wel == null: wg[l^W_T(j)] += 1 (multiplicity)
__global__ void globalize_kernel(SlabGeo g, int WT, const double* __restrict__ wel, const int* __restrict__ offw,
                                 double* wg) {
    const int64_t eK = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (eK >= g.ntiles * TILE) return;
    const int64_t tile = eK / TILE;
    const int lane = (int)(eK % TILE);
    const TileCoord tc = tile_coord(g, tile);
    const int ci = tc.ci0 + lane;
    if (ci >= g.Nx) return;
    const int64_t base = (int64_t)(2 * g.p) * (ci + g.swy * tc.cj + g.swz * tc.ck);
    for (int j = 0; j < WT; ++j)
        red_add_f64(wg + base + offw[tc.s * WT + j], wel ? wel[((size_t)tile * WT + j) * TILE + lane] : 1.0);
}

// natural W lattice (x fastest) -> class-major rows: x = 2p c + k stored at k (Nx+1) + c,
// so the 32 lanes of a tile (cells c .. c+31) read 32 consecutive doubles for every W node
__global__ void permute_w_kernel(SlabGeo g, const double* __restrict__ nat, double* __restrict__ out) {
    const int64_t MW = g.swy, twop = 2 * g.p;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.ndof_w; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / MW, x = i - row * MW;
        const int64_t cc = x / twop, k = x - cc * twop;
        out[row * g.rw + k * (g.Nx + 1) + cc] = nat[i];
    }
}

__global__ void divide_kernel(double* a, const double* b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = b[i] > 0.0 ? a[i] / b[i] : 0.0;
}
}  // namespace

cudaError_t launch_divide(double* a, const double* b, int64_t n, cudaStream_t st) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 4 * 148 * 8) blocks = 4 * 148 * 8;
    divide_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, b, n);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_permute_w(const SlabGeo& g, const double* nat, double* out, cudaStream_t st) {
    int64_t blocks = (g.ndof_w + 255) / 256;
    if (blocks > 4 * 148 * 8) blocks = 4 * 148 * 8;
    permute_w_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, nat, out);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_globalize(const SlabGeo& g, int WT, const double* wel, const int* offw, double* wg,
                             cudaStream_t st) {
    const int64_t n = g.ntiles * TILE;
    globalize_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(g, WT, wel, offw, wg);
    count_launches(1);
    return cudaGetLastError();
}

// ---------------------------------------------------------- load vector (K5)
namespace {
template <int D>
__global__ void load_vector_kernel(SlabGeo g, const double* verts, const double* sV, int VT,
                                   const ApplyTables tab, double f, double* b) {
    const int64_t eK = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (eK >= g.ntiles * TILE) return;
    const Geo G = element_geo<D>(g, verts, eK, nullptr);
    if (!G.valid) return;
    const int64_t tile = eK / TILE;
    const int lane = (int)(eK % TILE);
    const TileCoord tc = tile_coord(g, tile);
    const int ci = tc.ci0 + lane;
    const int64_t base = (int64_t)g.p * (ci + g.sy * tc.cj + g.sz * tc.ck);
    const double sc = f * fabs(G.det);
    for (int l = 0; l < VT; ++l) red_add_f64(b + base + tab.off[tc.s * MAX_VT + l], sc * sV[l]);
}
}  // namespace

cudaError_t launch_load_vector(const SlabGeo& g, int p, const double* verts, const double* sV, int VT,
                               const ApplyTables* tab, double f, double* b, cudaStream_t st) {
    (void)p;
    const int64_t n = g.ntiles * TILE;
    if (g.d == 2) load_vector_kernel<2><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(g, verts, sV, VT, *tab, f, b);
    else load_vector_kernel<3><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(g, verts, sV, VT, *tab, f, b);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace dogip
