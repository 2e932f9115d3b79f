// apply_cell.cuh -- the cell-per-lane apply kernel (sm_100a).  Included by
// apply_impl.cuh inside namespace dogip::(anonymous), after the element kernel whose
// building blocks (Chunking, WarpStream, lockstep policy, generated bodies) it reuses.
#pragma once

// ------------------------------------------------------------------ cell per lane
// Small elements (2D P1-P2, 3D P1-P2): one lane = one CELL (all d! simplices of it), one
// warp = 32 consecutive cells along x ("cell tile" = the d! element tiles of those cells,
// contiguous in the tile-major weight stream).  The lane's cell holds its (p+1)^d DoFs in
// registers; each simplex's u_T / y_T are compile-time views of them, so DoFs shared by
// the simplices of a cell are gathered and scattered once.  The x = p face of a cell is
// the x = 0 face of the next lane's cell: gathered by that lane and passed with one
// shuffle, and its contributions are added into that lane's x = 0 face by one shuffle
// before the scatter.  2D P1 per cell: 2 loads + 2 atomics instead of 6 + 6 (the element
// kernel's 19 us at C2 p = 1 was issue- and L2-atomic-bound,
// profiles/r01_C2_p1_p2_ncu_summary.txt).  Same operator, same weights (FULL storage).
template <class RE>
struct CellRE {     // the ns element tiles of one cell tile, read as one super tile
    static constexpr int VT = RE::VT, WT = RE::NS * RE::WT, NC = RE::NC, NG = 0, NS = RE::NS;
    static constexpr int TILE_ROWS = RE::NS * RE::TILE_ROWS, RALIGN = RE::RALIGN, DOT_IN_BODY = 0;
    static __host__ __device__ constexpr int row_of(int J) {
        return (J / RE::WT) * RE::TILE_ROWS + RE::row_of(J % RE::WT);
    }
};
#ifndef DOGIP_CELL_LOCKSTEP
#define DOGIP_CELL_LOCKSTEP -1  // -1: 2D cell kernels lock-step (C2 p=3 -3 %), 3D do not (C3 neutral,
                                // 24 % of its stall samples sat at the barrier); 0 / 1 force (A/B)
#endif
template <class RE>
struct LockstepPolicy<CellRE<RE>> {
    static constexpr bool value = DOGIP_CELL_LOCKSTEP >= 0 ? DOGIP_CELL_LOCKSTEP != 0 : RE::NS == 2;
};

#ifndef DOGIP_CELL_MAXP_2D
#define DOGIP_CELL_MAXP_2D 3   // 2D: cells of up to (p+1)^2 = 16 DoFs per lane (P4 spills: slower)
#endif
template <int D, int P>
__host__ __device__ constexpr bool cell_kernel_enabled() {
#ifdef DOGIP_NO_CELL_KERNEL
    return false;
#else
    return P <= 2 || (D == 2 && P <= DOGIP_CELL_MAXP_2D);
#endif
}

// simplex S of the cell through the super-tile stream (node J of S = node S WT + J)
template <class WS, int S, int WT, int TR>
struct SubPol {
    WS& ws;
    template <int J>
    __device__ __forceinline__ void begin() { ws.template begin<S * WT + J>(); }
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return ws.w(S * TR + k); }
};
// simplex S of the cell, weights already in registers (direct-weights path)
template <int OFF>
struct RegPolOff {
    const double* wr;
    template <int J>
    __device__ __forceinline__ void begin() {}
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return wr[OFF + k]; }
};

// cell-DoF index (x + (p+1) (y + (p+1) z)) of local DoF L of simplex S
template <int D, int P, class RE, int S, int L>
__host__ __device__ constexpr int cidx() {
    if constexpr (D == 3)
        return RE::LOFF[S][L][0] + (P + 1) * (RE::LOFF[S][L][1] + (P + 1) * RE::LOFF[S][L][2]);
    else
        return RE::LOFF[S][L][0] + (P + 1) * RE::LOFF[S][L][1];
}

template <int D, int P, class RE, int S, int L = 0>
__device__ __forceinline__ void view_in(const double* uc, const double* yc, double* uT, double* yT) {
    if constexpr (L < RE::VT) {
        uT[L] = uc[cidx<D, P, RE, S, L>()];
        yT[L] = yc[cidx<D, P, RE, S, L>()];
        view_in<D, P, RE, S, L + 1>(uc, yc, uT, yT);
    }
}
template <int D, int P, class RE, int S, int L = 0>
__device__ __forceinline__ void view_out(double* yc, const double* yT) {
    if constexpr (L < RE::VT) {
        yc[cidx<D, P, RE, S, L>()] = yT[L];
        view_out<D, P, RE, S, L + 1>(yc, yT);
    }
}

template <int D, int P, class RE, bool DW, class WS, int S = 0>
__device__ __forceinline__ void cell_body(const double* uc, double* yc, WS& ws, const double* wr) {
    if constexpr (S < RE::NS) {
        double uT[RE::VT], yT[RE::VT];
        view_in<D, P, RE, S>(uc, yc, uT, yT);
        if constexpr (DW) {
            RegPolOff<S * RE::TILE_ROWS> pol{wr};
            RE::body(uT, yT, pol);
        } else {
            SubPol<WS, S, RE::WT, RE::TILE_ROWS> pol{ws};
            RE::body(uT, yT, pol);
        }
        view_out<D, P, RE, S>(yc, yT);
        cell_body<D, P, RE, DW, WS, S + 1>(uc, yc, ws, wr);
    }
}

struct CellCtx {
    int64_t base;          // DoF index of the cell origin
    int ci, cj, ck;
    bool valid;            // ci < Nx
    bool load0;            // ci <= Nx: the x = 0 face exists (feeds the left lane's x = p face)
    bool last;             // scatters its own x = p face (last valid cell or lane 31)
};

__device__ __forceinline__ CellCtx cell_ctx(const SlabGeo& g, int64_t ct, int lane, int D) {
    // cell tile ct = xb + nxb (cj + Ny ck); element tile t = s + ns ct
    const uint32_t t = (uint32_t)ct, nxb = (uint32_t)g.nxb;
    const uint32_t r = fdiv(t, g.fd_nxb);
    const int xb = (int)(t - r * nxb);
    CellCtx c;
    if (D == 3) {
        const uint32_t ny = (uint32_t)g.Ny;
        const uint32_t ck = fdiv(r, g.fd_ny);
        c.cj = (int)(r - ck * ny);
        c.ck = (int)ck;
    } else {
        c.cj = (int)r;
        c.ck = 0;
    }
    c.ci = xb * TILE + lane;
    c.valid = c.ci < g.Nx;
    c.load0 = c.ci <= g.Nx;
    c.last = c.valid && (lane == TILE - 1 || c.ci == g.Nx - 1);
    c.base = (int64_t)g.p * (c.ci + g.sy * c.cj + g.sz * c.ck);
    return c;
}

// DoF (x, y, z) of the cell (offsets 0..p) is a Dirichlet boundary DoF (reading L14)
template <int D, int P>
__device__ __forceinline__ bool cell_bnd(const SlabGeo& g, const CellCtx& c, int x, int y, int z) {
    bool b = (x == 0 && c.ci == 0) || (x == P && c.ci == g.Nx - 1);
    if (D == 3) {
        b = b || (y == 0 && c.cj == 0) || (y == P && c.cj == g.Ny - 1);
        b = b || (z == 0 && c.ck == 0 && g.bnd_lo) || (z == P && c.ck == g.Nz - 1 && g.bnd_hi);
    } else {
        b = b || (y == 0 && c.cj == 0 && g.bnd_lo) || (y == P && c.cj == g.Ny - 1 && g.bnd_hi);
    }
    return b;
}

template <int D, int P, bool DIR>
__device__ __forceinline__ void cell_gather(const double* __restrict__ u, const SlabGeo& g, const CellCtx& c,
                                            int lane, double* uc) {
    constexpr int Q = P + 1, NZ = D == 3 ? Q : 1;
#pragma unroll
    for (int z = 0; z < NZ; ++z)
#pragma unroll
        for (int yy = 0; yy < Q; ++yy)
#pragma unroll
            for (int x = 0; x < Q; ++x) {
                const int k = x + Q * (yy + Q * z);
                const int64_t off = c.base + x + g.sy * yy + g.sz * z;
                double v = 0.0;
                if (x == 0) {
                    if (c.load0) v = ldg_f64(u + off);
                } else if (x < P) {
                    if (c.valid) v = ldg_f64(u + off);
                }
                uc[k] = v;
            }
    // x = p face: the next lane's x = 0 face (lane 31 loads its own)
#pragma unroll
    for (int z = 0; z < NZ; ++z)
#pragma unroll
        for (int yy = 0; yy < Q; ++yy) {
            const int k0 = Q * (yy + Q * z);
            double v = __shfl_down_sync(0xffffffffu, uc[k0], 1);
            if (lane == TILE - 1) v = c.valid ? ldg_f64(u + c.base + P + g.sy * yy + g.sz * z) : 0.0;
            uc[k0 + P] = v;
        }
    if constexpr (DIR) {
#pragma unroll
        for (int z = 0; z < NZ; ++z)
#pragma unroll
            for (int yy = 0; yy < Q; ++yy)
#pragma unroll
                for (int x = 0; x < Q; ++x)
                    if (cell_bnd<D, P>(g, c, x, yy, z)) uc[x + Q * (yy + Q * z)] = 0.0;
    }
}

template <int D, int P, bool DIR>
__device__ __forceinline__ void cell_scatter(double* __restrict__ y, const double* __restrict__ u, const SlabGeo& g,
                                             const CellCtx& c, int lane, double* yc, double* udot) {
    constexpr int Q = P + 1, NZ = D == 3 ? Q : 1;
    // the left lane's x = p face joins this lane's x = 0 face
#pragma unroll
    for (int z = 0; z < NZ; ++z)
#pragma unroll
        for (int yy = 0; yy < Q; ++yy) {
            const int k0 = Q * (yy + Q * z);
            const double v = __shfl_up_sync(0xffffffffu, yc[k0 + P], 1);
            if (lane > 0) yc[k0] += v;
        }
    if (!c.valid) return;
#pragma unroll
    for (int z = 0; z < NZ; ++z)
#pragma unroll
        for (int yy = 0; yy < Q; ++yy)
#pragma unroll
            for (int x = 0; x < Q; ++x) {
                if (DIR && cell_bnd<D, P>(g, c, x, yy, z)) {
                    // Dirichlet row y_i = u_i, written once: by the DoF's floor cell (offset < p
                    // on every axis, or the cell on the upper domain face / upper slab end)
                    const bool own = (x < P || c.ci == g.Nx - 1) &&
                                     (yy < P || (c.cj == g.Ny - 1 && (D == 3 || g.bnd_hi))) &&
                                     (D == 2 || z < P || (c.ck == g.Nz - 1 && g.bnd_hi));
                    if (own) {
                        const int64_t i = c.base + x + g.sy * yy + g.sz * z;
                        const double v = ldg_f64(u + i);
                        y[i] = v;
                        if (udot) *udot = fma(v, v, *udot);
                    }
                    continue;
                }
                if (x == P && !c.last) continue;
                red_add_f64(y + c.base + x + g.sy * yy + g.sz * z, yc[x + Q * (yy + Q * z)]);
            }
}

#ifndef DOGIP_CELL_MINB_2D1
#define DOGIP_CELL_MINB_2D1 8   // 2D P1: <= 64 registers, 32 warps per SM (latency-bound gathers)
#endif
#ifndef DOGIP_CELL_MINB_3D2
#define DOGIP_CELL_MINB_3D2 2   // 3D P2: 27 + 27 cell values per lane (3 CTAs/SM spills)
#endif
template <int D, int P>
constexpr int cell_min_blocks() {
    return (D == 3 && P == 2) ? DOGIP_CELL_MINB_3D2 : (D == 2 && P == 4) ? 2 : (D == 2 && P == 1) ? DOGIP_CELL_MINB_2D1 : 3;
}

template <int D, int P, int F, bool DIR>
__global__ void __launch_bounds__(APPLY_THREADS, cell_min_blocks<D, P>())
apply_cell_kernel(const double* __restrict__ u, double* __restrict__ y, const double* __restrict__ w,
                  const SlabGeo geo, const int64_t ct_begin, const int64_t ct_end, double* __restrict__ dot_partials,
                  const double* __restrict__ skip_if) {
    if (skip_if && *skip_if != 0.0) return;
    using RE = dogip_gen::RefElem<D, P, F, 0>;
    using CR = CellRE<RE>;
    using C = Chunking<CR>;
    constexpr int NW = APPLY_THREADS / 32;
    constexpr int Q = P + 1, NCD = D == 3 ? Q * Q * Q : Q * Q;
    constexpr bool DW = direct_weights<RE>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* rings = reinterpret_cast<double*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(rings + (size_t)NW * C::S * C::ROWS * TILE);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = ct_begin + (int64_t)blockIdx.x * NW + warp;
    const int64_t nw = (int64_t)gridDim.x * NW;
    WarpStream<CR> ws;
    ws.ring = rings + (size_t)warp * C::S * C::ROWS * TILE;
    ws.bar0 = smem_u32(bars + warp * C::S);
    ws.lane = lane;
    ws.tptr = w + gw * C::TILE_DBL;
    ws.tstride = nw * C::TILE_DBL;
    ws.tiles_left = gw < ct_end ? (ct_end - gw + nw - 1) / nw : 0;
    ws.cons = 0;
    ws.policy = policy_evict_first();
    if constexpr (!DW) {
        if (lane == 0) {
            for (int s = 0; s < C::S; ++s) mbar_init(ws.bar0 + 8u * s, 1);
            fence_mbar_init();
            ws.prologue();
        }
    }
    __syncwarp();
    double wr[DW ? CR::TILE_ROWS : 1];
    auto loadw = [&](int64_t t) {
        if constexpr (DW) {
            const double* wt = w + t * C::TILE_DBL + lane;
#pragma unroll
            for (int k = 0; k < CR::TILE_ROWS; ++k) wr[k] = ldg_stream_f64(wt + k * TILE);
        }
    };
    double udot = 0.0;
    double uc[NCD];
    CellCtx cur{};
    if (gw < ct_end) {
        cur = cell_ctx(geo, gw, lane, D);
        cell_gather<D, P, DIR>(u, geo, cur, lane, uc);
        loadw(gw);
    }
    for (int64_t ct = gw; ct < ct_end; ct += nw) {
        double yc[NCD];
#pragma unroll
        for (int k = 0; k < NCD; ++k) yc[k] = 0.0;
        cell_body<D, P, RE, DW, WarpStream<CR>>(uc, yc, ws, wr);
        if constexpr (!DW) ws.next_tile();
        if (dot_partials) {     // sum_T u_T^T y_T of the cell's simplices = uc . yc (views)
#pragma unroll
            for (int k = 0; k < NCD; ++k) udot = fma(uc[k], yc[k], udot);
        }
        const CellCtx prev = cur;
        if (ct + nw < ct_end) {                 // next tile's gather overlaps this scatter
            cur = cell_ctx(geo, ct + nw, lane, D);
            cell_gather<D, P, DIR>(u, geo, cur, lane, uc);
            loadw(ct + nw);
        }
        cell_scatter<D, P, DIR>(y, u, geo, prev, lane, yc, dot_partials ? &udot : nullptr);
    }
    if constexpr (!DW) lockstep_tail<CR, C>(gw, ct_end, ct_begin + (int64_t)blockIdx.x * NW, nw);
    if (dot_partials) {
        for (int o = 16; o > 0; o >>= 1) udot += __shfl_xor_sync(0xffffffffu, udot, o);
        if (lane == 0) dot_partials[(int64_t)blockIdx.x * NW + warp] = udot;
    }
}

template <int D, int P, int F, bool DIR>
cudaError_t launch_cell(const ApplyArgs& a) {
    using RE = dogip_gen::RefElem<D, P, F, 0>;
    using C = Chunking<CellRE<RE>>;
    constexpr int NW = APPLY_THREADS / 32;
    constexpr bool DW = direct_weights<RE>();
    const size_t smem = DW ? 0 : (size_t)NW * C::S * C::ROWS * TILE * 8 + (size_t)NW * C::S * 8;
    auto kern = apply_cell_kernel<D, P, F, DIR>;
    static std::atomic<uint64_t> cfg[MAX_DEVICES];
    int occ = 1;
    if (cudaError_t e = kernel_occupancy(kern, APPLY_THREADS, smem, cfg, &occ); e != cudaSuccess) return e;
    const int ns = RE::NS;
    const int64_t c0 = a.tile_begin / ns, c1 = a.tile_end / ns;     // ranges are whole cell tiles
    const int64_t ntiles = c1 - c0;
    int64_t grid = (int64_t)a.num_sms * occ;
    const int64_t need = (ntiles + NW - 1) / NW;
    if (grid > need) grid = need;
    if (a.dot_partials) {
        if (grid < 1) grid = 1;
        if (grid * NW > APPLY_MAX_WARPS) grid = APPLY_MAX_WARPS / NW;
        *a.dot_nslots = (int)(grid * NW);
    } else if (ntiles <= 0) {
        return cudaSuccess;
    }
    kern<<<(unsigned)grid, APPLY_THREADS, smem, a.stream>>>(a.u, a.y, a.w, a.geo, c0, c1, a.dot_partials, a.skip_if);
    if (DIR && a.rows_written) *a.rows_written = true;   // Dirichlet rows written in-kernel
    count_launches(1);
    return cudaGetLastError();
}

// DOGIP_CELL_KERNEL=0 in the environment selects the element-per-lane kernel instead (A/B)
inline bool cell_kernel_env() {
    static const bool on = [] {
        const char* e = std::getenv("DOGIP_CELL_KERNEL");
        return !(e && e[0] == '0');
    }();
    return on;
}

