// common.cuh -- shared device-side definitions of libdogip (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dogip {

constexpr int TILE = 32;       // elements per tile = one warp, one element per lane
constexpr int MAX_VT = 35;     // C(4+3,3)
constexpr int MAX_NS = 6;      // 3! Kuhn simplices per cube

// Geometry of this rank's slab as seen by the kernels.  Cells (ci, cj, ck)
// are LOCAL (ck in [0, Nz) along the slab axis; 2D: ck = 0, cj along the slab
// axis).  DoF lattice strides sx = 1, sy = M, sz = M^2, M = pN + 1.
// q = n / d for 0 <= n < 2^31 as one wide multiply and a shift (round-up method:
// m = ceil(2^(31+l) / d), l = ceil(log2 d), so m < 2^32 and floor(n m / 2^(31+l)) is
// exact for 31-bit n).  Replaces the ~20-instruction runtime integer division in the
// per-tile coordinate decode, which dominated the 2D P1 kernel's instruction count.
struct FastDiv {
    uint32_t m;
    int sh;
};
inline FastDiv make_fastdiv(uint32_t d) {
    int l = 0;
    while ((1ull << l) < d) ++l;
    return FastDiv{(uint32_t)(((1ull << (31 + l)) + d - 1) / d), 31 + l};
}
__device__ __host__ __forceinline__ uint32_t fdiv(uint32_t n, FastDiv f) {
    return (uint32_t)(((uint64_t)n * f.m) >> f.sh);
}

struct SlabGeo {
    int d, p, ns;                  // dimension, order, simplices per cell
    int Nx, Ny, Nz;                // local cells per axis (2D: Nz = 1)
    int nxb;                       // ceil(Nx / 32)
    int64_t ntiles;                // ns * nxb * Ny * Nz
    int64_t sy, sz;                // DoF strides
    int64_t ndof;                  // local DoFs
    int pmax_x, pmax_y, pmax_z;    // last DoF lattice index per axis (local)
    int bnd_lo, bnd_hi;            // slab-axis planes 0 / pmax are domain boundary
    int64_t zoff;                  // global cell offset along the slab axis
    int N;                         // global cells per axis
    int64_t swy, swz;              // W-lattice (order 2p) strides of the global WP storage
    int64_t ndof_w;                // local W-lattice DoFs
    int64_t rw;                    // stored row length of the class-major W layout: 2p (Nx + 1)
    FastDiv fd_ns, fd_nxb, fd_ny;  // divisors of tile_coord (set with the fields above)
};

// Tile t -> (simplex s, x-block, cj, ck).  Tiles are ordered with s fastest,
// then x-blocks, then rows cj, then layers ck (slab axis slowest), so the
// tiles of one cube layer are contiguous.
struct TileCoord {
    int s, ci0, cj, ck;
};
// 32-bit unsigned arithmetic: a slab has < 2^31 tiles (dogip_mesh_setup rejects more),
// and 64-bit division is ~5x the instructions -- it dominated tiny tiles (2D P1).
__device__ __host__ inline TileCoord tile_coord(const SlabGeo& g, int64_t t64) {
    TileCoord c;
    const uint32_t t = (uint32_t)t64, ns = (uint32_t)g.ns, nxb = (uint32_t)g.nxb;
    const uint32_t r1 = fdiv(t, g.fd_ns);
    c.s = (int)(t - r1 * ns);
    const uint32_t r2 = fdiv(r1, g.fd_nxb);
    const int xb = (int)(r1 - r2 * nxb);
    if (g.d == 3) {
        const uint32_t ny = (uint32_t)g.Ny;
        const uint32_t ck = fdiv(r2, g.fd_ny);
        c.cj = (int)(r2 - ck * ny);
        c.ck = (int)ck;
    } else {
        c.cj = (int)r2;
        c.ck = 0;
    }
    c.ci0 = xb * TILE;
    return c;
}

// ------------------------------------------------------- PTX helpers (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}
// 1D bulk copy global -> shared (TMA engine, no tensor map), completes on mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// bulk copy with an L2 evict-first hint: streamed weights are read exactly once
__device__ __forceinline__ void bulk_g2s_evict_first(uint32_t dst, const void* src, uint32_t bytes,
                                                     uint32_t bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }
// streamed read-only load, not kept in L1 (weights read exactly once)
__device__ __forceinline__ double ldg_stream_f64(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Ampere-style async copy global -> shared (LDGSTS), 8 bytes, L1-allocating
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void red_add_f64(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

}  // namespace dogip
