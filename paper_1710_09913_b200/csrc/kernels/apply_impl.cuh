// apply_impl.cuh -- the hot DoGIP apply kernel (sm_100a): templates, included by the
// per-(d, p) translation units apply_<d>_<p>.cu (compiled in parallel).
//
// y += sum_T P_T^T Bhat^T A_T Bhat P_T u      (Algorithm 1, PAPER.md P:491-511;
//                                              Theorem 2 eq:wp_dogip_mul P:276,
//                                              Theorem 4 eq:ep_dogip_mul P:439)
// Mapping:
//  * one warp = one 32-element tile = 32 consecutive cells along x with the same
//    simplex type s; one lane = one element;
//  * the per-element work g = Bhat u_T, h = A_T g, y_T += Bhat^T h is the
//    generated straight-line, sparsity- and +-1-aware FP64 code of
//    generated/bhat_gen.cuh, node by node, so only u_T and y_T sit in registers
//    (3D EL: the projection goes through the barycentric-derivative tables,
//    Bhat_r = D_{r+1} - D_0: 3D P3 3848 instead of 4296 flops; WP SYM storage: block-diagonal
//    by character, see gen_bhat.cpp emit_sym);
//  * A_T is stored tile-major [tile][W_T * NC][32] (lane fastest) and streamed
//    by each warp through its own S-stage shared-memory ring with 1D bulk
//    copies (cp.async.bulk, the TMA engine) that complete on mbarriers; the
//    stream runs ahead across tile boundaries, so HBM requests stay in flight
//    independently of register pressure.  Chunk boundaries are compile-time
//    (node rows), so the refill address is one add off the tile pointer;
//  * gather/scatter offsets are formed in registers: every simplex of the cell
//    has v_0 = cell origin, so off(l) = sum_i alpha_i(l) v_i(s) with compile-time
//    alpha and d per-tile vertex strides (no per-DoF table loads);
//  * the next tile's u_T is gathered (read-only loads) before this tile's y_T is
//    scattered with fire-and-forget red.global.add.f64 (y zeroed first), so the
//    gather latency overlaps the scatter; DIRICHLET zeroes boundary DoFs of u_T
//    and skips their scatter (the boundary rows are fixed by dirichlet_fixup).
//  * 3D EL: warps 2i / 2i+1 hold Kuhn types 2m / 2m+1 of the same cells, which share a
//    face; the even warp hands its y_T on that face to the odd one through shared memory
//    before the scatter (pair combine, 25 % fewer atomics).
// Kernels in this file:
//  * apply_kernel       element per lane (above): p >= 3 (2D p = 4), ISO, SYM, GLOBAL;
//  * apply_cell_kernel  cell per lane (all d! simplices of a cell, DoFs shared on chip,
//                       x faces by shuffles, Dirichlet rows written in-kernel): FULL storage,
//                       p <= 2 and 2D p = 3 (apply_cell.cuh).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

#include <cstdint>
#ifndef DOGIP_SYM_VSMEM
#define DOGIP_SYM_VSMEM 0      // 1: the symmetry-adapted body keeps v in the u_T staging buffer in shared
                               // memory (not registers), at 3 CTAs/SM (A/B builds)
#endif
#if DOGIP_SYM_VSMEM
__device__ __forceinline__ double dogip_lds_f64(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void dogip_sts_f64(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}
#define DOGIP_SYM_VDECL(n) const uint32_t vs_ = pol.vs
#define DOGIP_SYM_VSET(k, slot, e) dogip_sts_f64(vs_ + 256u * (slot), (e))
#define DOGIP_SYM_V(k, slot) dogip_lds_f64(vs_ + 256u * (slot))
#define DOGIP_SYM_U(l) dogip_lds_f64(vs_ + 256u * (l))
#endif
#ifdef DOGIP_GEN_HEADER
#include DOGIP_GEN_HEADER
#else
#include "../generated/bhat_gen.cuh"
#endif
#include "apply.cuh"
#include "common.cuh"

#ifndef DOGIP_ISO_STAGES
#define DOGIP_ISO_STAGES 2      // ring stages of the ISO kernels (0 = DOGIP_STAGES)
#endif
#ifndef DOGIP_LOCKSTEP
#define DOGIP_LOCKSTEP -1      // CTA barrier at every weight chunk (the CTA's warps share I-cache
                               // lines): -1 per-variant policy, 0 never, 1 always (A/B builds)
#endif
#ifndef DOGIP_SYM_UPF
#define DOGIP_SYM_UPF 1        // symmetry-adapted body: stage the next tile's u_T in shared memory
#endif
#ifndef DOGIP_STAGES
#define DOGIP_STAGES 4          // ring stages per warp
#endif
#ifndef DOGIP_ROWS_3CTA
#define DOGIP_ROWS_3CTA 18      // max rows per chunk when 3 CTAs share an SM
#endif
#ifndef DOGIP_ROWS_3CTA_2D
#define DOGIP_ROWS_3CTA_2D 24   // 2D full-storage kernels at 3 CTAs: fewer, larger chunks (C2 p=3/4 -1-2 %)
#endif
#ifndef DOGIP_ROWS_2CTA
#define DOGIP_ROWS_2CTA 24      // ... when 2 CTAs share an SM
#endif

#ifndef DOGIP_FULL_SYM
#define DOGIP_FULL_SYM 1   // 0: FULL WP storage through the plain node-by-node body (A/B builds)
#endif

namespace dogip {

namespace {

// 3 CTAs (12 warps) per SM where u_T + y_T fit in <= 170 registers, else 2
#ifndef DOGIP_MINB_LARGE
#define DOGIP_MINB_LARGE 2   // CTAs/SM asked of ptxas when V_T > 20 (3D P4)
#endif
#ifndef DOGIP_MINB_SMALL
#define DOGIP_MINB_SMALL 3   // CTAs/SM asked of ptxas when V_T <= 10 (2D P1-P3, 3D P1-P2)
#endif
#ifndef DOGIP_ROWS_4CTA
#define DOGIP_ROWS_4CTA 12
#endif
template <class RE>
constexpr int min_blocks128() {   // CTAs of APPLY_THREADS (4 warps) per SM
#ifdef DOGIP_MINB_OVERRIDE
    return DOGIP_MINB_OVERRIDE;
#endif
    // 2D P4 (V_T = 15): 2 CTAs / 255 registers beat 3 / 168 with spills (C2 p=4 -4 %, iso -5 %,
    // profiles/r02_ab_minb.log)
    if (DOGIP_SYM_VSMEM && RE::DOT_IN_BODY) return 3;
    return RE::VT <= 10 ? DOGIP_MINB_SMALL : (RE::VT <= 20 && RE::NS == 6) ? 3 : DOGIP_MINB_LARGE;
}

// Threads per CTA.  The symmetry-adapted bodies at 8 warps/SM (3D P4 WP: SYM, and FULL through
// the same body) run as ONE 8-warp CTA per SM instead of two 4-warp CTAs: the SM's warps then
// hold 8 consecutive tiles (the Kuhn types of the same cells, then the next x-block), so
// their u_T gathers and y atomics share L1 / L2 lines (C5 SYM 1.76 -> 1.69 ms, FULL 1.90 ->
// 1.79 median, profiles/r02_ab_cta256.log).  The other kernels measured neutral or slower.
#ifndef DOGIP_SYM_CTA8
#define DOGIP_SYM_CTA8 1
#endif
template <class RE>
__host__ __device__ constexpr int cta_threads() {
    return (DOGIP_SYM_CTA8 && RE::DOT_IN_BODY && min_blocks128<RE>() == 2) ? 2 * APPLY_THREADS : APPLY_THREADS;
}
template <class RE>
constexpr int min_blocks() {       // CTAs of cta_threads<RE>() per SM asked of ptxas
    return min_blocks128<RE>() * APPLY_THREADS / cta_threads<RE>();
}

// Balanced chunks of whole nodes: NCH = ceil(TILE_ROWS / ROWS_MAX) chunks of ROWS rows
// (a multiple of NC, so a node's NC rows never straddle two chunks; the NG leading
// rows of the iso storage sit in chunk 0), the last chunk shorter.
#ifndef DOGIP_SYM_ROWS
#define DOGIP_SYM_ROWS 24      // rows per chunk of the symmetry-adapted kernel (u_T staging shares smem)
#endif
#ifndef DOGIP_SYM_STAGES
#define DOGIP_SYM_STAGES 2
#endif
#ifndef DOGIP_STAGES_FORCE
#define DOGIP_STAGES_FORCE 0   // > 0: every kernel uses this many stages (A/B builds)
#endif
// Lock-stepping the 4 warps of a CTA at every weight chunk (profiles/r01_ab_lockstep2.log):
// -5 % for the FP64-bound ISO storage (C4 iso 2.47 -> 2.34 ms, C2 p=4 iso -14 %), -1 % for
// the long full tiles of C4 / C5; +3 % for the symmetry-adapted kernel, +2 % for C2 p=4 EL
template <class RE>
struct LockstepPolicy {
    static constexpr bool value = !RE::DOT_IN_BODY && (RE::NG > 0 || RE::TILE_ROWS >= 165);
};
template <class RE>
__host__ __device__ constexpr bool lockstep() {
    if constexpr (DOGIP_LOCKSTEP >= 0) return DOGIP_LOCKSTEP != 0;
    else return LockstepPolicy<RE>::value;
}

template <class RE, int TW = TILE>
struct Chunking {
    // ring stages per (d, p, form, storage), from the B200 A/B of 2/3/4 stages
    // (profiles/r01_ab_ring_stages.log): double buffering wins for the long weight tiles of
    // 3D P3 EL (C4: 3.72 -> 3.45 ms), 2D P4 EL and the symmetry-adapted kernel, 4 stages
    // for the rest (C2 p=2, C3, C5 full lose 1-6 % with 2).  The ISO kernels (NG > 0) run
    // CTA-lockstepped and take 2 (C4 iso 2.17 -> 2.13 ms, r01_ab_bary_deriv.log tail)
    static constexpr int S = DOGIP_STAGES_FORCE > 0 ? DOGIP_STAGES_FORCE
                           : RE::DOT_IN_BODY ? DOGIP_SYM_STAGES
                           : (RE::NC > 1 && RE::TILE_ROWS >= 84) ? 2
                           : (RE::NG > 0 && DOGIP_ISO_STAGES > 0) ? DOGIP_ISO_STAGES
                           : DOGIP_STAGES;
    static constexpr int TILE_ROWS = RE::TILE_ROWS;
    static constexpr int AL = RE::RALIGN;                                  // chunk boundaries fall on rows % AL == 0
    // the symmetry-adapted kernel stages u_T in shared memory too: 16-row chunks keep 2 CTAs/SM
    static constexpr int ROWS_MAX0 = min_blocks<RE>() >= 4 ? DOGIP_ROWS_4CTA
                                     : min_blocks<RE>() >= 3 ? ((RE::NS == 2 && RE::NG == 0) ? DOGIP_ROWS_3CTA_2D : DOGIP_ROWS_3CTA)
                                     : (DOGIP_SYM_UPF && RE::DOT_IN_BODY) ? DOGIP_SYM_ROWS : DOGIP_ROWS_2CTA;
    static constexpr int ROWS_MAX = (ROWS_MAX0 / AL) * AL;
    static constexpr int NCH0 = (TILE_ROWS + ROWS_MAX - 1) / ROWS_MAX;
    static constexpr int ROWS_B = (TILE_ROWS + NCH0 - 1) / NCH0;
    static constexpr int ROWS1 = ((ROWS_B + AL - 1) / AL) * AL;
    static constexpr int ROWS = ROWS1 < RE::NG + RE::NC ? RE::NG + RE::NC : ROWS1;
    static constexpr int NCH = (TILE_ROWS + ROWS - 1) / ROWS;             // chunks per tile
    static constexpr int LAST = TILE_ROWS - (NCH - 1) * ROWS;              // rows of the last chunk
    static constexpr int64_t TILE_DBL = (int64_t)TILE_ROWS * TW;           // doubles per tile
    static_assert(RE::NG == 0 || RE::NG <= ROWS, "iso G rows must sit in chunk 0");
};

template <class RE>
struct WarpStream {
    using C = Chunking<RE>;
    double* ring;          // this warp's ring in shared memory
    uint32_t bar0;         // smem address of this warp's S mbarriers
    int lane;
    const double* tptr;    // weights of the tile being consumed
    int64_t tstride;       // doubles between this warp's consecutive tiles
    int64_t tiles_left;    // this warp's tiles from the current one on
    uint32_t cons;         // chunks consumed so far (stage = cons % S, parity = cons / S)
    const double* cur;     // current stage + lane
    uint64_t policy;
    uint32_t vs;           // DOGIP_SYM_VSMEM: smem address of this lane's u_T / v column

    // chunk-sequence number g (relative: K tiles ahead, chunk c) -> stage g % S
    template <int K, int CI>
    __device__ __forceinline__ void issue(uint32_t stage) const {   // lane 0 only
        if (K >= tiles_left) return;
        constexpr int rows = (CI == C::NCH - 1) ? C::LAST : C::ROWS;
        constexpr uint32_t bytes = (uint32_t)rows * TILE * 8u;
        const uint32_t bar = bar0 + 8u * stage;
        mbar_expect_tx(bar, bytes);
        bulk_g2s_evict_first(smem_u32(ring + (size_t)stage * C::ROWS * TILE),
                             tptr + K * tstride + (int64_t)CI * C::ROWS * TILE, bytes, bar, policy);
    }
    template <int G>
    __device__ __forceinline__ void prologue_one() {
        if constexpr (G < C::S - 1) {
            issue<G / C::NCH, G % C::NCH>((uint32_t)G);
            prologue_one<G + 1>();
        }
    }
    __device__ __forceinline__ void prologue() { prologue_one<0>(); }
    // node J's weights start a new chunk (node 0 also covers the NG leading rows)
    template <int J>
    __device__ __forceinline__ void begin() {
        constexpr int c_cur = RE::row_of(J) / C::ROWS;
        if constexpr (J == 0 || c_cur != RE::row_of(J - 1) / C::ROWS) {
            constexpr int gi = c_cur + C::S - 1;          // chunk refilled now, relative to this tile
            if constexpr (lockstep<RE>()) asm volatile("bar.sync 1, %0;" ::"n"(cta_threads<RE>()) : "memory");
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async_smem();                 // prior generic reads of the stage
                issue<gi / C::NCH, gi % C::NCH>((cons + C::S - 1) % C::S);
            }
            const uint32_t st = cons % C::S;
            mbar_wait(bar0 + 8u * st, (cons / C::S) & 1u);
            cur = ring + (size_t)st * C::ROWS * TILE + lane;
            ++cons;
        }
    }
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return cur[(k % C::ROWS) * TILE]; }
    __device__ __forceinline__ void next_tile() {
        tptr += tstride;
        --tiles_left;
    }
};

#ifndef DOGIP_DIRECT_ROWS
#define DOGIP_DIRECT_ROWS 6    // tiles with at most this many weight rows skip the smem ring
#endif
template <class RE>
__host__ __device__ constexpr bool direct_weights() { return !RE::DOT_IN_BODY && RE::TILE_ROWS <= DOGIP_DIRECT_ROWS; }

// weights already in registers (direct-weights path): node rows are compile-time indices
struct RegPol {
    const double* wr;
    template <int J>
    __device__ __forceinline__ void begin() {}
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) const { return wr[k]; }
};

// LOCKSTEP: a warp with fewer tiles than its CTA's first warp matches the barriers the
// others still execute (NCH per tile)
template <class RE, class C>
__device__ __forceinline__ void lockstep_tail(int64_t gw, int64_t tile_end, int64_t gw0, int64_t nw) {
    if constexpr (lockstep<RE>()) {
        const int64_t mine = gw < tile_end ? (tile_end - gw + nw - 1) / nw : 0;
        const int64_t first = gw0 < tile_end ? (tile_end - gw0 + nw - 1) / nw : 0;
        for (int64_t k = mine; k < first; ++k)
            for (int c = 0; c < C::NCH; ++c) asm volatile("bar.sync 1, %0;" ::"n"(cta_threads<RE>()) : "memory");
    }
}

// Theorem 1 storage (global WP diagonal over W = C_{N,2p}): the weight of
// double-grid node j of the element is gathered from the global W-lattice vector, stored
// class-major along x (x = 2p c + k at k (Nx+1) + c), so a tile's 32 lanes read 32
// consecutive doubles per node; offw holds each node's offset in that layout.
#ifndef DOGIP_GLOB_AHEAD
#define DOGIP_GLOB_AHEAD 4     // W values loaded this many nodes ahead into registers (0 = on demand;
                               // C5 GLOBAL 2.275 -> 2.214 ms at 8, profiles/r02_ab_global_ahead.log;
                               // 2.265 -> 2.195 ms at 4 on the final build, r02_ab_global_ahead_final.log)
#endif
template <int WT>
struct GatherPol {
    static constexpr int D = DOGIP_GLOB_AHEAD;
    const double* wg;      // global W weights of this slab
    const int* offw;       // shared-memory W-lattice offsets of this simplex type
    int64_t baseW;         // W-lattice index of the cell origin
    double buf[D > 0 ? D : 1];   // node k's value sits in buf[k % D] (registers: k is a literal)
    __device__ __forceinline__ double ld(int k) const { return __ldg(wg + baseW + offw[k]); }
    template <int J>
    __device__ __forceinline__ void begin() {
        if constexpr (J == 0 && D > 0) {
#pragma unroll
            for (int k = 0; k < D && k < WT; ++k) buf[k] = ld(k);
        }
    }
    template <int J>
    __device__ __forceinline__ void end() {}
    __device__ __forceinline__ double w(int k) {
        if constexpr (D == 0) return ld(k);
        const double v = buf[k % D];
        if (k + D < WT) buf[k % D] = ld(k + D);   // the load runs while node k is computed
        return v;
    }
};

// Per-tile gather context of one lane's element.
struct ElemCtx {
    int64_t base;          // DoF index of the cell origin
    int v1, v2, v3;        // DoF-lattice offsets of vertices 1..d
    uint64_t skip;         // bit l: local DoF l is not gathered / scattered (Dirichlet)
    bool valid;            // lane holds a real element (ci < Nx)
    int s, ci, cj, ck;
};

template <class RE, int D, bool DIR>
__device__ __forceinline__ ElemCtx elem_ctx(const SlabGeo& geo, const ApplyTables& tab, int64_t t, int lane) {
    const TileCoord tc = tile_coord(geo, t);
    ElemCtx c;
    c.s = tc.s; c.ci = tc.ci0 + lane; c.cj = tc.cj; c.ck = tc.ck;
    c.valid = c.ci < geo.Nx;
    c.base = (int64_t)geo.p * (c.ci + geo.sy * tc.cj + geo.sz * tc.ck);
    c.v1 = tab.vstr[tc.s][0];
    c.v2 = tab.vstr[tc.s][1];
    c.v3 = D == 3 ? tab.vstr[tc.s][2] : 0;
    c.skip = 0;
    if constexpr (DIR) {   // boundary DoFs = DoFs on a cell face that lies on the domain boundary
        const unsigned long long* fm = tab.fmask[tc.s];
        uint64_t b = 0;
        if (c.ci == 0) b |= fm[0];
        if (c.ci == geo.Nx - 1) b |= fm[1];
        if (D == 3) {
            if (tc.cj == 0) b |= fm[2];
            if (tc.cj == geo.Ny - 1) b |= fm[3];
            if (tc.ck == 0 && geo.bnd_lo) b |= fm[4];
            if (tc.ck == geo.Nz - 1 && geo.bnd_hi) b |= fm[5];
        } else {
            if (tc.cj == 0 && geo.bnd_lo) b |= fm[2];
            if (tc.cj == geo.Ny - 1 && geo.bnd_hi) b |= fm[3];
        }
        c.skip = b;
    }
    return c;
}

template <class RE, int L>
__device__ __forceinline__ int dof_off(const ElemCtx& c) {
    return RE::ALPHA[L][0] * c.v1 + RE::ALPHA[L][1] * c.v2 + RE::ALPHA[L][2] * c.v3;
}

template <class RE, int L = 0>
__device__ __forceinline__ void gather(const double* __restrict__ u, const ElemCtx& c, double* uT) {
    if constexpr (L < RE::VT) {
        const bool take = c.valid && !((c.skip >> L) & 1ull);
#ifdef DOGIP_AB_NO_GATHER   // timing experiment only: no u loads (wrong results)
        uT[L] = take ? 1.0 + 1e-3 * (double)(c.base + dof_off<RE, L>(c)) : 0.0;
#else
        uT[L] = take ? ldg_f64(u + c.base + dof_off<RE, L>(c)) : 0.0;
#endif
        gather<RE, L + 1>(u, c, uT);
    }
}

// u_T of a tile -> the warp's [VT][32] shared buffer with cp.async (no registers held)
template <class RE, int L = 0>
__device__ __forceinline__ void gather_async(const double* __restrict__ u, const ElemCtx& c, uint32_t ubuf_lane) {
    if constexpr (L < RE::VT) {
        if (c.valid && !((c.skip >> L) & 1ull)) cp_async8(ubuf_lane + 8u * TILE * L, u + c.base + dof_off<RE, L>(c));
        gather_async<RE, L + 1>(u, c, ubuf_lane);
    }
}

template <class RE, int L = 0>
__device__ __forceinline__ void scatter(double* __restrict__ y, const ElemCtx& c, const double* yT) {
    if constexpr (L < RE::VT) {
#ifdef DOGIP_AB_NO_SCATTER  // timing experiment only: one store per element instead of V_T atomics
        if (L == 0) { double t = 0.0; for (int k = 0; k < RE::VT; ++k) t += yT[k]; if (t == 1.2345) y[c.base] = t; }
#else
        if (!((c.skip >> L) & 1ull)) red_add_f64(y + c.base + dof_off<RE, L>(c), yT[L]);
#endif
        scatter<RE, L + 1>(y, c, yT);
    }
}


// Pair combine (round 2).  The 4 warps of a CTA hold consecutive tiles, and tiles are
// ordered with the simplex type s fastest, so warps 2i and 2i+1 always hold types (2m, 2m+1)
// of the SAME 32 cells (tile ranges start and end on whole cell rows).  Those two simplices
// share a face (3D Kuhn types 0|1, 2|3, 4|5 differ by one adjacent transposition; 2D: the
// diagonal edge), so the even warp hands its y_T values on the shared DoFs to the odd warp
// through shared memory (one 64-thread named barrier per tile, double-buffered) and skips
// their atomics: 3D P4 70 -> 55, 3D P3 40 -> 30 red.global.add.f64 per element pair.
#ifndef DOGIP_PAIR_COMBINE
#define DOGIP_PAIR_COMBINE 1
#endif
template <class RE>
__host__ __device__ constexpr int loff_dim() { return (int)(sizeof(RE::LOFF[0][0]) / sizeof(RE::LOFF[0][0][0])); }
// local DoF of simplex s0 + 1 at the same lattice point as DoF l0 of simplex s0 (-1: none)
template <class RE>
__host__ __device__ constexpr int pair_partner(int s0, int l0) {
    for (int l = 0; l < RE::VT; ++l) {
        bool eq = true;
        for (int a = 0; a < loff_dim<RE>(); ++a)
            if (RE::LOFF[s0][l0][a] != RE::LOFF[s0 + 1][l][a]) eq = false;
        if (eq) return l;
    }
    return -1;
}
template <class RE>
__host__ __device__ constexpr int pair_slot(int s0, int l0) {   // index among the shared DoFs
    int k = 0;
    for (int l = 0; l < l0; ++l) k += pair_partner<RE>(s0, l) >= 0;
    return k;
}
template <class RE>
__host__ __device__ constexpr int pair_shared_max() {
    int m = 0;
    for (int s0 = 0; s0 + 1 < RE::NS; s0 += 2) {
        const int k = pair_slot<RE>(s0, RE::VT);
        m = k > m ? k : m;
    }
    return m;
}
template <class RE>
__host__ __device__ constexpr uint64_t pair_mask(int s0) {
    uint64_t m = 0;
    for (int l = 0; l < RE::VT; ++l)
        if (pair_partner<RE>(s0, l) >= 0) m |= 1ull << l;
    return m;
}
template <class RE, int S0, int L = 0>
__device__ __forceinline__ void pair_put(const double* yT, double* buf) {
    if constexpr (L < RE::VT) {
        if constexpr (pair_partner<RE>(S0, L) >= 0) buf[pair_slot<RE>(S0, L) * TILE] = yT[L];
        pair_put<RE, S0, L + 1>(yT, buf);
    }
}
template <class RE, int S0, int L = 0>
__device__ __forceinline__ void pair_get(double* yT, const double* buf) {
    if constexpr (L < RE::VT) {
        constexpr int l1 = pair_partner<RE>(S0, L);
        if constexpr (l1 >= 0) yT[l1] += buf[pair_slot<RE>(S0, L) * TILE];
        pair_get<RE, S0, L + 1>(yT, buf);
    }
}
// put (even warp): returns the mask of the DoFs handed over; get (odd warp): 0
template <class RE, int S0 = 0>
__device__ __forceinline__ uint64_t pair_dispatch(bool put, int ps, double* yT, double* buf) {
    if constexpr (S0 + 1 < RE::NS) {
        if (ps == S0 / 2) {
            constexpr uint64_t mask = pair_mask<RE>(S0);
            if (put) { pair_put<RE, S0>(yT, buf); return mask; }
            pair_get<RE, S0>(yT, buf);
            return 0;
        }
        return pair_dispatch<RE, S0 + 2>(put, ps, yT, buf);
    }
    return 0;
}
// Before the scatter of a tile of type s (warp-uniform): returns the DoFs this warp must not
// scatter (the even warp's shared DoFs).  buf = this pair's [2][F][32] buffer, par = tile parity.
template <class RE>
__device__ __forceinline__ uint64_t pair_combine(double* yT, double* buf, int par, int s, int warp, int lane) {
    constexpr int F = pair_shared_max<RE>();
    double* b = buf + (size_t)par * F * TILE + lane;
    const bool even = (s & 1) == 0;
    uint64_t m = 0;
    if (even) m = pair_dispatch<RE>(true, s >> 1, yT, b);
    asm volatile("bar.sync %0, 64;" ::"r"(2 + (warp >> 1)) : "memory");
    if (!even) pair_dispatch<RE>(false, s >> 1, yT, b);
    return m;
}
// On for the 3D elliptic kernels (C4 full 3.56 -> 3.53 ms, iso 2.16 -> 2.10); off for WP
// (C5 sym / full / global neutral to +1 %) and 2D (C2 p=4 iso +11 %):
// profiles/r02_ab_pair_combine.log
template <class RE, int D, int F>
__host__ __device__ constexpr bool pair_enabled() {
    return DOGIP_PAIR_COMBINE && D == 3 && F == 1 && !direct_weights<RE>() && cta_threads<RE>() % 64 == 0;
}

template <int D, int P, int F, int ST, bool DIR, bool GLOB>
__global__ void __launch_bounds__(cta_threads<dogip_gen::RefElem<D, P, F, ST>>(), min_blocks<dogip_gen::RefElem<D, P, F, ST>>())
apply_kernel(const double* __restrict__ u, double* __restrict__ y, const double* __restrict__ w,
             const SlabGeo geo, const ApplyTables tab, const int64_t tile_begin, const int64_t tile_end,
             double* __restrict__ dot_partials, const int* __restrict__ offw_g,
             const double* __restrict__ skip_if) {
    if (skip_if && *skip_if != 0.0) return;    // finished CG solve: the weight stream is not read
    using RE = dogip_gen::RefElem<D, P, F, ST>;
    using C = Chunking<RE>;
    constexpr int NW = cta_threads<RE>() / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr bool RING = !(GLOB || direct_weights<RE>());                   // weight ring + mbarriers
    double* rings = reinterpret_cast<double*>(smem_raw);
    uint64_t* bars = reinterpret_cast<uint64_t*>(rings + (RING ? (size_t)NW * C::S * C::ROWS * TILE : 0));
    constexpr bool UPF = DOGIP_SYM_UPF && RE::DOT_IN_BODY && !GLOB;
    double* ubufs = reinterpret_cast<double*>(bars + (RING ? NW * C::S : 0));   // [NW][VT][32] (UPF only)
    constexpr bool PAIRC = pair_enabled<RE, D, F>();
    constexpr int PF = pair_shared_max<RE>();
    double* pbuf = !PAIRC ? nullptr : ubufs + (UPF ? (size_t)NW * RE::VT * TILE : 0) +
                   (size_t)((threadIdx.x >> 5) >> 1) * 2 * PF * TILE;      // [NW/2][2][PF][32]
    int ppar = 0;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gw = tile_begin + (int64_t)blockIdx.x * NW + warp;
    const int64_t nw = (int64_t)gridDim.x * NW;
    WarpStream<RE> ws;
    ws.ring = rings + (size_t)warp * C::S * C::ROWS * TILE;
    ws.bar0 = smem_u32(bars + warp * C::S);
    ws.lane = lane;
    ws.tptr = w + gw * C::TILE_DBL;
    ws.tstride = nw * C::TILE_DBL;
    ws.tiles_left = gw < tile_end ? (tile_end - gw + nw - 1) / nw : 0;
    ws.cons = 0;
    ws.policy = policy_evict_first();
    __shared__ int offw_s[GLOB ? MAX_NS * MAX_WT_GLOBAL : 1];
    constexpr bool DW = direct_weights<RE>() && !GLOB;
    if constexpr (GLOB) {
        for (int i = threadIdx.x; i < RE::NS * RE::WT; i += blockDim.x)   // the table holds NS * WT
            offw_s[(i / RE::WT) * MAX_WT_GLOBAL + i % RE::WT] = offw_g[i];
        __syncthreads();
    } else if (DW) {
    } else if (lane == 0) {
        for (int s = 0; s < C::S; ++s) mbar_init(ws.bar0 + 8u * s, 1);
        fence_mbar_init();
        ws.prologue();                                   // prologue of the weight stream
    }
    __syncwarp();

    double udot = 0.0;
    double uT[RE::VT];
    ElemCtx cur{};
    if constexpr (DW) {
        // tiny tiles (<= DOGIP_DIRECT_ROWS weight rows): each lane reads its element's
        // weights with coalesced read-only loads (one 256 B row per warp load), the next
        // tile's together with its u_T gather -- no ring, barriers or bulk copies
        double wr[RE::TILE_ROWS];
        auto loadw = [&](int64_t t) {
            const double* wt = w + t * C::TILE_DBL + lane;
#pragma unroll
            for (int k = 0; k < RE::TILE_ROWS; ++k) wr[k] = ldg_stream_f64(wt + k * TILE);
        };
        if (gw < tile_end) {
            cur = elem_ctx<RE, D, DIR>(geo, tab, gw, lane);
            gather<RE>(u, cur, uT);
            loadw(gw);
        }
        for (int64_t tile = gw; tile < tile_end; tile += nw) {
            double yT[RE::VT];
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) yT[l] = 0.0;
            RegPol rp{wr};
            RE::body(uT, yT, rp);
            if (dot_partials) {
#pragma unroll
                for (int l = 0; l < RE::VT; ++l) udot = fma(uT[l], yT[l], udot);
            }
            const ElemCtx prev = cur;
            if (tile + nw < tile_end) {
                cur = elem_ctx<RE, D, DIR>(geo, tab, tile + nw, lane);
                gather<RE>(u, cur, uT);
                loadw(tile + nw);
            }
            if (prev.valid) scatter<RE>(y, prev, yT);
        }
    } else if constexpr (UPF) {
        double* ubuf = ubufs + (size_t)warp * RE::VT * TILE;
        const uint32_t ubuf_lane = smem_u32(ubuf + lane);
        if (gw < tile_end) {
            cur = elem_ctx<RE, D, DIR>(geo, tab, gw, lane);
            gather_async<RE>(u, cur, ubuf_lane);
        }
        cp_async_commit();
        for (int64_t tile = gw; tile < tile_end; tile += nw) {
            cp_async_wait_all();
            __syncwarp();
#if DOGIP_SYM_VSMEM
            {
            // v lives in this lane's staging column: zero the slots the gather skipped, run
            // the body on smem, then stage the next tile (after the body's last v read)
            if (!cur.valid || cur.skip) {
#pragma unroll
                for (int l = 0; l < RE::VT; ++l)
                    if (!cur.valid || ((cur.skip >> l) & 1ull)) dogip_sts_f64(ubuf_lane + 256u * l, 0.0);
            }
            const ElemCtx prev = cur;
            double yT[RE::VT];
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) yT[l] = 0.0;
            ws.vs = ubuf_lane;
            RE::body(nullptr, yT, ws, dot_partials ? &udot : nullptr);
            ws.next_tile();
            __syncwarp();
            if (tile + nw < tile_end) {
                cur = elem_ctx<RE, D, DIR>(geo, tab, tile + nw, lane);
                gather_async<RE>(u, cur, ubuf_lane);
            }
            cp_async_commit();
            if (prev.valid) scatter<RE>(y, prev, yT);
            continue;
            }
#endif
#pragma unroll
            for (int l = 0; l < RE::VT; ++l)
                uT[l] = (cur.valid && !((cur.skip >> l) & 1ull)) ? ubuf[l * TILE + lane] : 0.0;
            __syncwarp();
            const ElemCtx prev = cur;
            if (tile + nw < tile_end) {         // next tile's u_T lands in smem during this body
                cur = elem_ctx<RE, D, DIR>(geo, tab, tile + nw, lane);
                gather_async<RE>(u, cur, ubuf_lane);
            }
            cp_async_commit();
            double yT[RE::VT];
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) yT[l] = 0.0;
            if constexpr (RE::DOT_IN_BODY) RE::body(uT, yT, ws, dot_partials ? &udot : nullptr);
            ws.next_tile();
            ElemCtx sc = prev;
            if constexpr (PAIRC) { sc.skip |= pair_combine<RE>(yT, pbuf, ppar, prev.s, warp, lane); ppar ^= 1; }
            if (sc.valid) scatter<RE>(y, sc, yT);
        }
        lockstep_tail<RE, C>(gw, tile_end, tile_begin + (int64_t)blockIdx.x * NW, nw);
    } else {
    if (gw < tile_end) {
        cur = elem_ctx<RE, D, DIR>(geo, tab, gw, lane);
        gather<RE>(u, cur, uT);
    }
    for (int64_t tile = gw; tile < tile_end; tile += nw) {
        double yT[RE::VT];
#pragma unroll
        for (int l = 0; l < RE::VT; ++l) yT[l] = 0.0;
        if constexpr (GLOB) {
            // padding lanes (ci >= Nx) gather the slab's first cell: in bounds and finite
            // (their u_T is 0, so y_T = 0 and the fused p.q stays exact)
            GatherPol<RE::WT> gp{w, offw_s + cur.s * MAX_WT_GLOBAL,
                         cur.valid ? geo.rw * (int64_t)(2 * geo.p) * (cur.cj + geo.swy * cur.ck) + cur.ci : 0};
            RE::body(uT, yT, gp);
        } else {
            if constexpr (RE::DOT_IN_BODY) RE::body(uT, yT, ws, dot_partials ? &udot : nullptr);
            else RE::body(uT, yT, ws);
            ws.next_tile();
        }
        // u^T A u = sum_T u_T^T (Bhat^T A_T Bhat u_T): the CG dot p.q, element by element
        // (padding lanes and Dirichlet DoFs have u_T = 0 and contribute nothing)
        if (!RE::DOT_IN_BODY && dot_partials) {
#pragma unroll
            for (int l = 0; l < RE::VT; ++l) udot = fma(uT[l], yT[l], udot);
        }
        ElemCtx prev = cur;
        if constexpr (PAIRC) { prev.skip |= pair_combine<RE>(yT, pbuf, ppar, prev.s, warp, lane); ppar ^= 1; }
        if (tile + nw < tile_end) {            // next tile's gather overlaps this scatter
            cur = elem_ctx<RE, D, DIR>(geo, tab, tile + nw, lane);
            gather<RE>(u, cur, uT);
        }
        if (prev.valid) scatter<RE>(y, prev, yT);
    }
    if constexpr (!GLOB) lockstep_tail<RE, C>(gw, tile_end, tile_begin + (int64_t)blockIdx.x * NW, nw);
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
    constexpr int NW = cta_threads<RE>() / 32;
    constexpr bool UPF = DOGIP_SYM_UPF && RE::DOT_IN_BODY && !GLOB;
    constexpr bool DW = direct_weights<RE>() && !GLOB;
    const size_t smem = ((GLOB || DW) ? 0 : (size_t)NW * C::S * C::ROWS * TILE * 8 + (size_t)NW * C::S * 8) +
                        (UPF ? (size_t)NW * RE::VT * TILE * 8 : 0) +
                        (pair_enabled<RE, D, F>() ? (size_t)(NW / 2) * 2 * pair_shared_max<RE>() * TILE * 8 : 0);
    auto kern = apply_kernel<D, P, F, ST, DIR, GLOB>;
    static std::atomic<uint64_t> cfg[MAX_DEVICES];   // per instantiation, per device
    int occ = 1;
    if (cudaError_t e = kernel_occupancy(kern, cta_threads<RE>(), smem, cfg, &occ); e != cudaSuccess) return e;
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
    kern<<<(unsigned)grid, cta_threads<RE>(), smem, a.stream>>>(a.u, a.y, a.w, a.geo, *a.tab, a.tile_begin,
                                                           a.tile_end, a.dot_partials, a.offw, a.skip_if);
    count_launches(1);
    return cudaGetLastError();
}

#include "apply_cell.cuh"   // cell-per-lane kernel (p <= 2, 2D p = 3)

template <int D, int P, int F, int ST>
cudaError_t launch_dir(const ApplyArgs& a) {
    if constexpr (ST == 0 && cell_kernel_enabled<D, P>()) {
        const int ns = D == 2 ? 2 : 6;
        if (cell_kernel_env() && a.tile_begin % ns == 0 && a.tile_end % ns == 0)
            return a.dirichlet ? launch_cell<D, P, F, true>(a) : launch_cell<D, P, F, false>(a);
    }
    return a.dirichlet ? launch_one<D, P, F, ST, true, false>(a) : launch_one<D, P, F, ST, false, false>(a);
}

// DOGIP_STORE_FULL of the weighted projection runs the symmetry-adapted body (RefElem<.., 6>:
// the same a_{T,j}, rows in orbit order) where it is instantiated: 3D p >= 3 (C5)
template <int D, int P>
__host__ __device__ constexpr bool full_sym_body() { return DOGIP_FULL_SYM && D == 3 && P >= 3; }

template <int D, int P>
cudaError_t launch_form(const ApplyArgs& a) {
    // every storage has the Dirichlet-elimination instantiation (DOGIP_DIRICHLET_ZERO)
    if (a.form == 0 && a.store == 2)
        return a.dirichlet ? launch_one<D, P, 0, 0, true, true>(a) : launch_one<D, P, 0, 0, false, true>(a);
    if (a.form == 0 && a.store == 5) return launch_dir<D, P, 0, 5>(a);
    if (a.form == 0 && a.store == 6) {   // internal: FULL weights in orbit order, symmetry-adapted body
        if constexpr (full_sym_body<D, P>()) return launch_dir<D, P, 0, 6>(a);
        else return cudaErrorInvalidValue;
    }
    if (a.form == 0) return launch_dir<D, P, 0, 0>(a);
    return a.store == 1 ? launch_dir<D, P, 1, 1>(a) : launch_dir<D, P, 1, 0>(a);
}

// Reference-element constants of the generated tables, for the host side.
template <int D, int P, int F, int ST>
void fill_info(RefInfo& r) {
    using RE = dogip_gen::RefElem<D, P, F, ST>;
    r.VT = RE::VT; r.WT = RE::WT; r.NC = RE::NC; r.NG = RE::NG; r.NS = RE::NS;
    r.tile_rows = RE::TILE_ROWS;
    r.flops = RE::FLOPS; r.nnz = RE::NNZ; r.nnz_pm1 = RE::NNZ_PM1;
    r.sym = ST == 5;
    if constexpr (ST == 5) {
        for (int j = 0; j < RE::WT; ++j)
            for (int k = 0; k < 4; ++k) { r.symj[j][k] = RE::SYMJ[j][k]; r.symc[j][k] = RE::SYMC[j][k]; }
    }
    r.has_rowperm = RE::HAS_ROWPERM;
    for (int j = 0; j < RE::WT && j < MAX_WT_GLOBAL; ++j) {
        if constexpr (RE::HAS_ROWPERM) r.rowperm[j] = RE::ROWPERM[j];
        else r.rowperm[j] = j;
    }
    for (int s = 0; s < RE::NS; ++s)
        for (int l = 0; l < RE::VT; ++l)
            for (int ax = 0; ax < 3; ++ax) r.loff[s][l][ax] = ax < D ? RE::LOFF[s][l][ax] : 0;
}

}  // namespace
}  // namespace dogip
