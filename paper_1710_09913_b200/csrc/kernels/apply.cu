// apply.cu -- the hot DoGIP apply kernel (sm_100a).
//
// y += sum_T P_T^T Bhat^T A_T Bhat P_T u      (Algorithm 1, PAPER.md P:491-511;
//                                              Theorem 2 eq:wp_dogip_mul P:276,
//                                              Theorem 4 eq:ep_dogip_mul P:439)
// Mapping:
//  * one warp = one 32-element tile = 32 consecutive cells along x with the same
//    simplex type s; one lane = one element (gather offsets are warp-uniform and
//    read from the kernel-parameter bank);
//  * the per-element work g = Bhat u_T, h = A_T g, y_T += Bhat^T h is the
//    generated straight-line, sparsity- and +-1-aware FP64 code of
//    generated/bhat_gen.cuh, node by node, so only u_T and y_T sit in registers;
//  * A_T is stored tile-major [tile][W_T * NC][32] (lane fastest) and streamed
//    by each warp through its own S-stage shared-memory ring with 1D bulk
//    copies (cp.async.bulk, the TMA engine) that complete on mbarriers; the
//    stream runs ahead across tile boundaries, so HBM requests stay in flight
//    independently of register pressure;
//  * u_T is gathered with read-only loads (neighbouring lanes share cache
//    lines), y_T is scattered with fire-and-forget red.global.add.f64 (y must
//    be zeroed first); DIRICHLET zeroes boundary DoFs of u_T and skips their
//    scatter (the boundary rows are fixed by dirichlet_fixup).
#include <cuda_runtime.h>

#ifdef DOGIP_GEN_HEADER
#include DOGIP_GEN_HEADER
#else
#include "../generated/bhat_gen.cuh"
#endif
#ifndef DOGIP_UPREFETCH
// cp.async (LDGSTS) prefetch of the next tile's u_T into shared memory.  Measured
// slower than direct read-only gathers on B200 (profiles/r01_ab_variants.log), off.
#define DOGIP_UPREFETCH 0
#endif
#include "apply.cuh"
#include "common.cuh"

namespace dogip {

namespace {

template <class RE>
struct Chunking {
    static constexpr int ROWS = RE::ROWS;                                 // rows per streamed chunk
    static constexpr int TILE_ROWS = RE::TILE_ROWS;                       // rows per tile
    static constexpr int NCH = (TILE_ROWS + ROWS - 1) / ROWS;             // chunks per tile
    static constexpr int S = 4;                                           // ring stages per warp
};

template <class RE>
struct WarpStream {
    using C = Chunking<RE>;
    double* ring;          // this warp's ring in shared memory
    uint32_t bar0;         // smem address of this warp's S mbarriers
    int lane;
    const double* wbase;   // global weights (tile-major)
    int64_t gw, nw, tile_end;
    int64_t g_cons;        // next chunk (warp-global sequence) to consume
    const double* cur;     // current stage + lane
    uint64_t policy;

    __device__ __forceinline__ void issue(int64_t gg) const {   // lane 0 only
        const int64_t it = gg / C::NCH;
        const int c = (int)(gg - it * C::NCH);
        const int64_t tile = gw + it * nw;
        if (tile >= tile_end) return;
        const int rows = (c == C::NCH - 1) ? C::TILE_ROWS - c * C::ROWS : C::ROWS;
        const uint32_t bytes = (uint32_t)rows * TILE * 8u;
        const int st = (int)(gg % C::S);
        const uint32_t bar = bar0 + 8u * st;
        mbar_expect_tx(bar, bytes);
        bulk_g2s_evict_first(smem_u32(ring + (size_t)st * C::ROWS * TILE),
                             wbase + ((size_t)tile * C::TILE_ROWS + (size_t)c * C::ROWS) * TILE,
                             bytes, bar, policy);
    }
    // node J's weights start a new chunk (node 0 also covers the NG leading rows)
    template <int J>
    __device__ __forceinline__ void begin() {
        if constexpr (J == 0 || RE::row_of(J) / C::ROWS != RE::row_of(J - 1) / C::ROWS) {
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_smem();          // prior generic reads of the stage
                issue(g_cons + C::S - 1);          // refill the stage consumed last
            }
            const int st = (int)(g_cons % C::S);
            mbar_wait(bar0 + 8u * st, (uint32_t)((g_cons / C::S) & 1));
            cur = ring + (size_t)st * C::ROWS * TILE + lane;
            ++g_cons;
        }
    }
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return cur[(k % C::ROWS) * TILE]; }
};

// Theorem 1 storage (global WP diagonal over W = C_{N,2p}): the weight of
// double-grid node j of the element is gathered from the global W-lattice vector.
struct GatherPol {
    const double* wg;      // global W weights of this slab
    const int* offw;       // shared-memory W-lattice offsets of this simplex type
    int64_t baseW;         // W-lattice index of the cell origin
    template <int J>
    __device__ __forceinline__ void begin() {}
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return __ldg(wg + baseW + offw[k]); }
};

// 3 CTAs (12 warps) per SM where u_T + y_T fit in <= 170 registers, else 2
#ifndef DOGIP_MINB_LARGE
#define DOGIP_MINB_LARGE 2   // CTAs/SM asked of ptxas when V_T > 20 (3D P4)
#endif
template <int D, int P, int F, int ST>
constexpr int min_blocks() { return dogip_gen::RefElem<D, P, F, ST>::VT <= 20 ? 3 : DOGIP_MINB_LARGE; }

template <int D, int P, int F, int ST, bool DIR, bool GLOB>
__global__ void __launch_bounds__(APPLY_THREADS, min_blocks<D, P, F, ST>())
apply_kernel(const double* __restrict__ u, double* __restrict__ y, const double* __restrict__ w,
             const SlabGeo geo, const ApplyTables tab, const int64_t tile_begin, const int64_t tile_end,
             double* __restrict__ dot_partials, const int* __restrict__ offw_g) {
    using RE = dogip_gen::RefElem<D, P, F, ST>;
    using C = Chunking<RE>;
    constexpr int NW = APPLY_THREADS / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* rings = reinterpret_cast<double*>(smem_raw);
    double* ubufs = rings + (size_t)NW * C::S * C::ROWS * TILE;          // [NW][VT][32]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ubufs + (size_t)NW * RE::VT * TILE);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpStream<RE> ws;
    ws.ring = rings + (size_t)warp * C::S * C::ROWS * TILE;
    ws.bar0 = smem_u32(bars + warp * C::S);
    ws.lane = lane;
    ws.wbase = w;
    ws.gw = tile_begin + (int64_t)blockIdx.x * NW + warp;
    ws.nw = (int64_t)gridDim.x * NW;
    ws.tile_end = tile_end;
    ws.g_cons = 0;
    ws.policy = policy_evict_first();
    double* ubuf = ubufs + (size_t)warp * RE::VT * TILE;
    const uint32_t ubuf_s = smem_u32(ubuf + lane);
    __shared__ int offw_s[GLOB ? MAX_NS * MAX_WT_GLOBAL : 1];
    if constexpr (GLOB) {
        for (int i = threadIdx.x; i < MAX_NS * RE::WT; i += blockDim.x)
            offw_s[(i / RE::WT) * MAX_WT_GLOBAL + i % RE::WT] = offw_g[i];
        __syncthreads();
    } else if (lane == 0) {
        for (int s = 0; s < C::S; ++s) mbar_init(ws.bar0 + 8u * s, 1);
        fence_mbar_init();
        for (int s = 0; s < C::S - 1; ++s) ws.issue(s);      // prologue of the weight stream
    }
    // u_T of a tile -> this lane's column of the warp's u buffer (cp.async, no registers)
    auto prefetch_u = [&](int64_t t) {
        const TileCoord tc = tile_coord(geo, t);
        const int ci = tc.ci0 + lane;
        if (ci < geo.Nx) {
            const double* ub = u + (int64_t)geo.p * (ci + geo.sy * tc.cj + geo.sz * tc.ck);
            const int* off = tab.off + tc.s * MAX_VT;
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) cp_async8(ubuf_s + 8u * TILE * l, ub + off[l]);
        }
        cp_async_commit();
    };
    if (DOGIP_UPREFETCH && ws.gw < tile_end) prefetch_u(ws.gw);
    __syncwarp();

    double udot = 0.0;
    for (int64_t tile = ws.gw; tile < tile_end; tile += ws.nw) {
        const TileCoord tc = tile_coord(geo, tile);
        const int ci = tc.ci0 + lane;
        const bool valid = ci < geo.Nx;
        const int64_t base = (int64_t)geo.p * (ci + geo.sy * tc.cj + geo.sz * tc.ck);
        const int* off = tab.off + tc.s * MAX_VT;
        const int* lof = tab.loff + tc.s * MAX_VT;
        double uT[RE::VT], yT[RE::VT];
        uint64_t bmask = 0;
        if (DOGIP_UPREFETCH) {
            cp_async_wait_all();
            __syncwarp();
        }
#pragma unroll
        for (int l = 0; l < RE::VT; ++l) {
            bool take = valid;
            if constexpr (DIR) {
                const int lo = lof[l];
                const int X = geo.p * ci + (lo & 0xff);
                const int Y = geo.p * tc.cj + ((lo >> 8) & 0xff);
                const int Z = geo.p * tc.ck + ((lo >> 16) & 0xff);
                bool b = X == 0 || X == geo.pmax_x;
                if (D == 3) {
                    b = b || Y == 0 || Y == geo.pmax_y || (Z == 0 && geo.bnd_lo) || (Z == geo.pmax_z && geo.bnd_hi);
                } else {
                    b = b || (Y == 0 && geo.bnd_lo) || (Y == geo.pmax_y && geo.bnd_hi);
                }
                if (b) { bmask |= (1ull << l); take = false; }
            }
            if (DOGIP_UPREFETCH) {
                const double v = ubuf[l * TILE + lane];
                uT[l] = take ? v : 0.0;
            } else {
                uT[l] = take ? ldg_f64(u + base + off[l]) : 0.0;
            }
            yT[l] = 0.0;
        }
        if (DOGIP_UPREFETCH) {
            __syncwarp();
            if (tile + ws.nw < tile_end) prefetch_u(tile + ws.nw);  // overlaps this tile's compute
        }
        if constexpr (GLOB) {
            GatherPol gp{w, offw_s + tc.s * MAX_WT_GLOBAL,
                         (int64_t)(2 * geo.p) * (ci + geo.swy * tc.cj + geo.swz * tc.ck)};
            RE::body(uT, yT, gp);
        } else {
            RE::body(uT, yT, ws);
        }
        if (valid) {
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) {
                if (DIR && ((bmask >> l) & 1ull)) continue;
                red_add_f64(y + base + off[l], yT[l]);
            }
            // u^T A u = sum_T u_T^T (Bhat^T A_T Bhat u_T): the CG dot p.q, element by element
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) udot = fma(uT[l], yT[l], udot);
        }
    }
    if (dot_partials) {     // deterministic: one partial per warp, fixed order reduction later
        for (int o = 16; o > 0; o >>= 1) udot += __shfl_xor_sync(0xffffffffu, udot, o);
        if (lane == 0) dot_partials[(int64_t)blockIdx.x * NW + warp] = udot;
    }
}

template <int D, int P, int F, int ST, bool DIR, bool GLOB>
cudaError_t launch_one(const ApplyArgs& a) {
    using RE = dogip_gen::RefElem<D, P, F, ST>;
    using C = Chunking<RE>;
    constexpr int NW = APPLY_THREADS / 32;
    const size_t smem = (size_t)NW * C::S * C::ROWS * TILE * 8 + (size_t)NW * RE::VT * TILE * 8 +
                        (size_t)NW * C::S * 8;
    auto kern = apply_kernel<D, P, F, ST, DIR, GLOB>;
    static int configured = 0;   // per instantiation
    static int occ = 1;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, APPLY_THREADS, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        configured = 1;
    }
    const int64_t ntiles = a.tile_end - a.tile_begin;
    int64_t grid = (int64_t)a.num_sms * occ;
    const int64_t need = (ntiles + NW - 1) / NW;
    if (grid > need) grid = need;
    if (a.dot_partials) {       // every slot of the partial array must be written
        if (grid < 1) grid = 1;
        if (grid * NW > APPLY_MAX_WARPS) grid = APPLY_MAX_WARPS / NW;
        *a.dot_nslots = (int)(grid * NW);
    } else if (ntiles <= 0) {
        return cudaSuccess;
    }
    kern<<<(unsigned)grid, APPLY_THREADS, smem, a.stream>>>(a.u, a.y, a.w, a.geo, *a.tab, a.tile_begin,
                                                           a.tile_end, a.dot_partials, a.offw);
    count_launches(1);
    return cudaGetLastError();
}

template <int D, int P, int F, int ST>
cudaError_t launch_dir(const ApplyArgs& a) {
    return a.dirichlet ? launch_one<D, P, F, ST, true, false>(a) : launch_one<D, P, F, ST, false, false>(a);
}

template <int D, int P>
cudaError_t launch_form(const ApplyArgs& a) {
    if (a.form == 0 && a.store == 2) return launch_one<D, P, 0, 0, false, true>(a);   // WP has no BC
    if (a.form == 0) return launch_dir<D, P, 0, 0>(a);
    return a.store == 1 ? launch_dir<D, P, 1, 1>(a) : launch_dir<D, P, 1, 0>(a);
}

template <int D>
cudaError_t launch_p(const ApplyArgs& a) {
    switch (a.p) {
        case 1: return launch_form<D, 1>(a);
        case 2: return launch_form<D, 2>(a);
        case 3: return launch_form<D, 3>(a);
        case 4: return launch_form<D, 4>(a);
    }
    return cudaErrorInvalidValue;
}

}  // namespace

std::atomic<long long> g_launches{0};

cudaError_t launch_apply(const ApplyArgs& a) {
    return a.d == 2 ? launch_p<2>(a) : launch_p<3>(a);
}

// Reference-element constants of the generated tables, for the host side.
template <int D, int P, int F, int ST>
static void fill_info(RefInfo& r) {
    using RE = dogip_gen::RefElem<D, P, F, ST>;
    r.VT = RE::VT; r.WT = RE::WT; r.NC = RE::NC; r.NG = RE::NG; r.NS = RE::NS;
    r.tile_rows = RE::TILE_ROWS;
    r.flops = RE::FLOPS; r.nnz = RE::NNZ; r.nnz_pm1 = RE::NNZ_PM1;
    for (int s = 0; s < RE::NS; ++s)
        for (int l = 0; l < RE::VT; ++l)
            for (int ax = 0; ax < 3; ++ax) r.loff[s][l][ax] = ax < D ? RE::LOFF[s][l][ax] : 0;
}

bool ref_info(int d, int p, int form, int store, RefInfo& r) {
#define DOGIP_CASE(D, P)                                                       \
    if (d == D && p == P) {                                                    \
        if (form == 0 && store == 0) { fill_info<D, P, 0, 0>(r); return true; } \
        if (form == 1 && store == 0) { fill_info<D, P, 1, 0>(r); return true; } \
        if (form == 1 && store == 1) { fill_info<D, P, 1, 1>(r); return true; } \
        return false;                                                          \
    }
    DOGIP_CASE(2, 1) DOGIP_CASE(2, 2) DOGIP_CASE(2, 3) DOGIP_CASE(2, 4)
    DOGIP_CASE(3, 1) DOGIP_CASE(3, 2) DOGIP_CASE(3, 3) DOGIP_CASE(3, 4)
#undef DOGIP_CASE
    return false;
}

}  // namespace dogip
