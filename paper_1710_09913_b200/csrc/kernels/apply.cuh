// apply.cuh -- host-visible interface of the kernels in kernels/*.cu
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

#include <atomic>

namespace dogip {

// kernel launches issued by the library (dogip_kernel_launches)
extern std::atomic<long long> g_launches;
inline void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Dynamic-shared-memory opt-in and occupancy of one kernel, cached PER DEVICE (the
// attribute is a per-device property: a second mesh on another device must opt in
// again).  `cache` is a per-kernel static array; slot = (smem + 1) << 16 | occupancy.
// Concurrent first calls may both configure, which is harmless.
constexpr int MAX_DEVICES = 64;
template <class Kern>
inline cudaError_t kernel_occupancy(Kern kern, int threads, size_t smem, std::atomic<uint64_t>* cache, int* occ) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t key = ((uint64_t)smem + 1) << 16;
    std::atomic<uint64_t>* slot = (dev >= 0 && dev < MAX_DEVICES) ? &cache[dev] : nullptr;
    if (slot) {
        const uint64_t v = slot->load(std::memory_order_acquire);
        if ((v & ~0xffffull) == key) { *occ = (int)(v & 0xffff); return cudaSuccess; }
    }
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
    if (e != cudaSuccess) return e;
    if (o < 1) o = 1;
    if (slot) slot->store(key | (uint64_t)(o & 0xffff), std::memory_order_release);
    *occ = o;
    return cudaSuccess;
}

#ifndef DOGIP_APPLY_THREADS
#define DOGIP_APPLY_THREADS 128
#endif
constexpr int APPLY_THREADS = DOGIP_APPLY_THREADS;   // 4 warps = 4 tiles in flight per CTA
constexpr int APPLY_MAX_WARPS = 148 * 8 * 4;   // bound of the per-warp dot partials of one launch

// Warp-uniform gather tables (kernel-parameter bank): off = local DoF index
// offset of local DoF l of simplex s from the cell's base DoF; loff = the
// same offset as packed lattice coordinates x | y << 8 | z << 16.
struct ApplyTables {
    int off[MAX_NS * MAX_VT];
    int loff[MAX_NS * MAX_VT];
    // apply kernel: DoF-lattice offset of vertex i = 1..d of simplex s (v_0 = cell origin),
    // so off[s][l] = sum_i alpha_i(l) vstr[s][i-1] with compile-time alpha
    int vstr[MAX_NS][3];
    // DoFs of simplex s on the cell face "axis a at 0" (bit 2a) / "axis a at p" (2a+1)
    unsigned long long fmask[MAX_NS][6];
};

constexpr int MAX_WT_GLOBAL = 165;   // W_T of P_8 in 3D (global WP storage, p <= 4)

struct ApplyArgs {
    int d, p, form, store;      // store: 0 full A_T blocks, 1 isotropic a_j + G_T (EL), 2 global WP,
                                // 5 symmetry-adapted WP
    bool dirichlet;
    const double* u;
    double* y;
    const double* w;
    SlabGeo geo;
    const ApplyTables* tab;
    int64_t tile_begin, tile_end;
    int num_sms;
    cudaStream_t stream;
    double* dot_partials;      // != null: per-warp partials of u^T A u (APPLY_MAX_WARPS slots)
    int* dot_nslots;           // out: number of partial slots written
    const int* offw;           // global WP: device table [NS][W_T] of W-lattice offsets
    const double* skip_if;     // != null: the kernel returns at once when *skip_if != 0 (an
                               // iteration enqueued after its CG solve finished)
    bool* rows_written;        // out (optional): set when the launched kernel wrote the Dirichlet
                               // rows y_i = u_i itself (cell kernel), so no fix-up is needed
};

cudaError_t launch_apply(const ApplyArgs& a);

// Constants of the generated reference element (generated/bhat_gen.cuh).
struct RefInfo {
    int VT, WT, NC, NG, NS, tile_rows, flops, nnz, nnz_pm1;
    int loff[MAX_NS][MAX_VT][3];
    int has_rowperm;                 // node rows stored permuted (symmetry-adapted ISO)
    int rowperm[MAX_WT_GLOBAL];      // storage row of canonical node j (identity unless has_rowperm)
    int sym;                         // symmetry-adapted WP (STORE 5): row r = sum_k symc[r][k] a_{symj[r][k]}
    int symj[MAX_WT_GLOBAL][4];
    double symc[MAX_WT_GLOBAL][4];
};
bool ref_info(int d, int p, int form, int store, RefInfo& r);

// ----------------------------------------------------------- weights (K1)
struct WeightsArgs {
    int d, p, form, store, nq, WT, NC, ncomp;  // ncomp: coefficient components (1 or d(d+1)/2)
    int NG, tile_rows;                     // leading per-element rows, rows per tile
    int kind;                              // DOGIP_COEF_*
    const double* params;                  // device copy of the coefficient parameters
    int nparams;
    const double* per_cell;                // device, global cell numbering, or null
    const double* verts;                   // device ((N+1)^d, d) or null (lattice)
    const double* qp;                      // device (nq, d) reference points
    const double* qw;                      // device (nq,) weights
    const double* phiW;                    // device (nq, WT) double-grid basis at points
    const double* sW;                      // device (WT,) sum_q w_q phi^W_j(x_q)
    SlabGeo geo;
    double* out;                           // tile-major weights [tile][WT*NC][32]
    double* scratch_c;                     // [nb * ncomp][nq]
    double* scratch_a;                     // [nb * ncomp][WT]
    int64_t batch;                         // elements per batch (multiple of 32)
    int* bad_flag;                         // device int: 1 degenerate element, 2 bad coefficient
    const int* rowperm;                    // device (WT,): storage row of node j (permuted ISO layout)
    int sym;                               // symmetry-adapted WP rows (STORE 5)
    const int* symj;                       // device (WT, 4): canonical nodes of stored row r (-1: none)
    const double* symc;                    // device (WT, 4): their coefficients
    cudaStream_t stream;
};
cudaError_t launch_weights(const WeightsArgs& a);
// global WP (Theorem 1): wg[l^W_T(j)] += a_{T,j} from tile-major element weights
// (wel == null: += 1, the multiplicity of each W node); a /= b elementwise (b > 0)
cudaError_t launch_divide(double* a, const double* b, int64_t n, cudaStream_t st);
cudaError_t launch_globalize(const SlabGeo& g, int WT, const double* wel, const int* offw, double* wg,
                             cudaStream_t st);
// natural W lattice -> the class-major layout the apply reads (geo.rw; padding left untouched)
cudaError_t launch_permute_w(const SlabGeo& g, const double* nat, double* out, cudaStream_t st);

// ----------------------------------------------------------- quadrature-point comparator
// Matrix-free A u over the integration points, no stored operator.
struct QpArgs {
    int d, p, form;
    bool dirichlet;
    const double* u;
    double* y;
    SlabGeo geo;
    const ApplyTables* tab;
    int nq;
    const double* qp;       // device (nq, d) reference points
    const double* qw;       // device (nq,) weights
    const double* phi;      // device (nq, V_T) basis values (WP)
    const double* dphi;     // device (nq, d, V_T) reference gradients (EL)
    int nq_smem;            // points whose table rows are staged in shared memory (set by the launcher)
    int kind, ncomp;        // DOGIP_COEF_*, coefficient components
    const double* params;   // device coefficient parameters
    const double* per_cell; // device per-cell values or null
    const double* verts;    // device vertices or null (lattice)
    int64_t tile_begin, tile_end;
    int num_sms;
    cudaStream_t stream;
    double* dot_partials;
    int* dot_nslots;
};
cudaError_t launch_qp_apply(const QpArgs& a);

// ----------------------------------------------------------- vectors / CG
cudaError_t launch_dirichlet_fixup(const SlabGeo& g, const double* u, double* y, cudaStream_t st);
cudaError_t launch_zero_boundary(const SlabGeo& g, double* y, cudaStream_t st);
// y_i = u_i on the boundary DoFs of slab-axis DoF planes [P0, P1)
cudaError_t launch_dirichlet_planes(const SlabGeo& g, const double* u, double* y, int64_t P0, int64_t P1,
                                    cudaStream_t st);
cudaError_t launch_load_vector(const SlabGeo& g, int p, const double* verts, const double* sV,
                               int VT, const ApplyTables* tab, double f, double* b, cudaStream_t st);

// deterministic two-pass reductions (partials of fixed grid, then one block)
constexpr int RED_BLOCKS = 592;       // 4 x 148 SMs
constexpr int RED_THREADS = 256;
cudaError_t launch_dot(const double* a, const double* b, int64_t i0, int64_t i1, double* partials,
                       double* out, cudaStream_t st);
// x += alpha p, r -= alpha q over [0, n), alpha = scal[RR]/scal[PQ]; partial r.r over [i0, i1)
cudaError_t launch_cg_xr(double* x, double* r, const double* p, const double* q, int64_t n, int64_t i0,
                         int64_t i1, double* scal, double* partials, cudaStream_t st);
// p = r + beta p, beta = scal[RRNEW]/scal[RR]; then scal[RR] = scal[RRNEW]
cudaError_t launch_cg_p(double* p, const double* r, int64_t n, double* scal, cudaStream_t st);
cudaError_t launch_reduce_final(const double* partials, double* out, cudaStream_t st);
cudaError_t launch_axpby(double* y, const double* x, double a, double b, int64_t n, cudaStream_t st);
cudaError_t launch_add_planes(double* y, const double* lo, const double* hi, int64_t plane,
                              int64_t last_plane_off, cudaStream_t st);
cudaError_t launch_fill(double* y, double v, int64_t n, cudaStream_t st);
// sum of n partials in fixed order (+ *extra if non-null) -> *out
cudaError_t launch_sum_partials(const double* partials, int n, const double* extra, double* out, cudaStream_t st);
// Dirichlet rows y_i = u_i on boundary DoFs; if bpart != null also the partial sum of
// u_i^2 over boundary DoFs in [i0, i1), each counted once (RED_BLOCKS slots)
cudaError_t launch_dirichlet_fixup_dot(const SlabGeo& g, const double* u, double* y, int64_t i0, int64_t i1,
                                       double* bpart, cudaStream_t st);
// r -= alpha q (alpha = scal[RR]/scal[PQ]) over [0,n); partial r.r over [i0,i1) -> scal[RRNEW]
cudaError_t launch_cg_r(double* r, const double* q, int64_t n, int64_t i0, int64_t i1, double* scal,
                        double* partials, cudaStream_t st);
// x += alpha p; p = r + beta p (beta = scal[RRNEW]/scal[RR]); then scal[RR] = scal[RRNEW]
cudaError_t launch_cg_px(double* x, double* p, const double* r, int64_t n, double* scal, cudaStream_t st);

// device scalars of a CG solve: S_DONE / S_IT / S_STATUS are the loop state (cg_control)
enum CgScal { S_RR = 0, S_PQ = 1, S_RRNEW = 2, S_BB = 3, S_DONE = 4, S_IT = 5, S_STATUS = 6, S_COUNT = 8 };
// after an iteration: breakdown / count / convergence / maxit -> S_DONE, S_STATUS; with h
// (graph path) also the WHILE node's condition = !S_DONE
cudaError_t launch_cg_control(double* scal, double rtol, int maxit, const cudaGraphConditionalHandle* h,
                              cudaStream_t st);
// S_IT = 0, S_DONE = (||r_0|| <= rtol ||b||), rtol < 0: never converged (fixed-count runs)
cudaError_t launch_cg_init(double* scal, double rtol, cudaStream_t st);
// loopback all-reduce: out[i] = sum_k slots[k stride + i], k = 0..nranks-1 in order
cudaError_t launch_sum_slots(const double* slots, int nranks, int64_t stride, int64_t n, double* out,
                             cudaStream_t st);

}  // namespace dogip
