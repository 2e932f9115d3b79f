// vectors.cu -- CG vector kernels, reductions and boundary handling (sm_100a).
//
// CG (reading L15, Hestenes-Stiefel) needs per iteration: q = A p (apply.cu),
// p.q, x += alpha p, r -= alpha q with r.r, p = r + beta p.  The scalars stay
// on the device (scal[]), so an iteration enqueues without host round trips;
// alpha / beta are formed inside the kernels.  Reductions are deterministic:
// fixed RED_BLOCKS partials, then one block sums them in a fixed order.
#include <cuda_runtime.h>

#include "apply.cuh"

namespace dogip {
namespace {

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[RED_THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < RED_THREADS / 32 ? sh[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t i0, int64_t i1, double* partials) {
    double s = 0.0;
    for (int64_t i = i0 + (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < i1;
         i += (int64_t)gridDim.x * RED_THREADS)
        s = fma(a[i], b[i], s);
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) reduce_final_kernel(const double* partials, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < RED_BLOCKS; i += RED_THREADS) s += partials[i];
    s = block_sum(s);
    if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(RED_THREADS) cg_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ q, int64_t n, int64_t i0,
                                                            int64_t i1, const double* scal, double* partials) {
    const double alpha = scal[S_RR] / scal[S_PQ];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * RED_THREADS) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        if (i >= i0 && i < i1) s = fma(ri, ri, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) cg_p_kernel(double* __restrict__ p, const double* __restrict__ r,
                                                           int64_t n, const double* scal) {
    const double beta = scal[S_RRNEW] / scal[S_RR];
    for (int64_t i = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * RED_THREADS)
        p[i] = fma(beta, p[i], r[i]);
}

__global__ void shift_rr_kernel(double* scal) { scal[S_RR] = scal[S_RRNEW]; }

__global__ void axpby_kernel(double* y, const double* x, double a, double b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = a * x[i] + b * y[i];
}

__global__ void fill_kernel(double* y, double v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = v;
}

__global__ void add_planes_kernel(double* y, const double* lo, const double* hi, int64_t plane,
                                  int64_t last_off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane; i += (int64_t)gridDim.x * blockDim.x) {
        if (lo) y[i] += lo[i];
        if (hi) y[last_off + i] += hi[i];
    }
}

// Boundary DoFs of the local slab, enumerated face by face (duplicates on
// edges are harmless: every face writes the same value).
__device__ __forceinline__ bool boundary_dof(const SlabGeo& g, int64_t t, int64_t& idx) {
    const int64_t nx = g.pmax_x + 1, ny = g.pmax_y + 1, nz = g.pmax_z + 1;
    if (g.d == 2) {
        // faces x = 0, x = pmax_x over y; y = 0 (bnd_lo), y = pmax_y (bnd_hi) over x
        if (t < 2 * ny) { const int64_t Y = t % ny; idx = (t / ny ? g.pmax_x : 0) + Y * g.sy; return true; }
        t -= 2 * ny;
        if (t < nx) { if (!g.bnd_lo) return false; idx = t; return true; }
        t -= nx;
        if (t < nx) { if (!g.bnd_hi) return false; idx = t + (int64_t)g.pmax_y * g.sy; return true; }
        return false;
    }
    const int64_t fx = ny * nz, fy = nx * nz, fz = nx * ny;
    if (t < 2 * fx) {
        const int64_t side = t / fx, r = t % fx;
        idx = (side ? g.pmax_x : 0) + (r % ny) * g.sy + (r / ny) * g.sz;
        return true;
    }
    t -= 2 * fx;
    if (t < 2 * fy) {
        const int64_t side = t / fy, r = t % fy;
        idx = (r % nx) + (side ? (int64_t)g.pmax_y : 0) * g.sy + (r / nx) * g.sz;
        return true;
    }
    t -= 2 * fy;
    if (t < 2 * fz) {
        const int64_t side = t / fz, r = t % fz;
        if (side == 0 && !g.bnd_lo) return false;
        if (side == 1 && !g.bnd_hi) return false;
        idx = (r % nx) + (r / nx) * g.sy + (side ? (int64_t)g.pmax_z : 0) * g.sz;
        return true;
    }
    return false;
}

__host__ __device__ inline int64_t boundary_count(const SlabGeo& g) {
    const int64_t nx = g.pmax_x + 1, ny = g.pmax_y + 1, nz = g.pmax_z + 1;
    if (g.d == 2) return 2 * ny + 2 * nx;
    return 2 * (ny * nz + nx * nz + nx * ny);
}

__global__ void boundary_set_kernel(SlabGeo g, const double* u, double* y) {
    const int64_t n = boundary_count(g);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t idx;
        if (boundary_dof(g, t, idx)) y[idx] = u ? u[idx] : 0.0;
    }
}

inline unsigned grid_for(int64_t n, int threads, int maxb = 4 * 148 * 4) {
    int64_t b = (n + threads - 1) / threads;
    if (b > maxb) b = maxb;
    if (b < 1) b = 1;
    return (unsigned)b;
}

}  // namespace

cudaError_t launch_dot(const double* a, const double* b, int64_t i0, int64_t i1, double* partials, double* out,
                       cudaStream_t st) {
    dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, b, i0, i1, partials);
    reduce_final_kernel<<<1, RED_THREADS, 0, st>>>(partials, out);
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_cg_xr(double* x, double* r, const double* p, const double* q, int64_t n, int64_t i0, int64_t i1,
                         double* scal, double* partials, cudaStream_t st) {
    cg_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(x, r, p, q, n, i0, i1, scal, partials);
    reduce_final_kernel<<<1, RED_THREADS, 0, st>>>(partials, scal + S_RRNEW);
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_cg_p(double* p, const double* r, int64_t n, double* scal, cudaStream_t st) {
    cg_p_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(p, r, n, scal);
    shift_rr_kernel<<<1, 1, 0, st>>>(scal);
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_reduce_final(const double* partials, double* out, cudaStream_t st) {
    reduce_final_kernel<<<1, RED_THREADS, 0, st>>>(partials, out);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_axpby(double* y, const double* x, double a, double b, int64_t n, cudaStream_t st) {
    axpby_kernel<<<grid_for(n, 256), 256, 0, st>>>(y, x, a, b, n);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_fill(double* y, double v, int64_t n, cudaStream_t st) {
    fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(y, v, n);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_add_planes(double* y, const double* lo, const double* hi, int64_t plane, int64_t last_off,
                              cudaStream_t st) {
    add_planes_kernel<<<grid_for(plane, 256), 256, 0, st>>>(y, lo, hi, plane, last_off);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dirichlet_fixup(const SlabGeo& g, const double* u, double* y, cudaStream_t st) {
    boundary_set_kernel<<<grid_for(boundary_count(g), 256), 256, 0, st>>>(g, u, y);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_zero_boundary(const SlabGeo& g, double* y, cudaStream_t st) {
    boundary_set_kernel<<<grid_for(boundary_count(g), 256), 256, 0, st>>>(g, nullptr, y);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace dogip
