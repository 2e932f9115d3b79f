// vectors.cu -- CG vector kernels, reductions and boundary handling (sm_100a).
//
// CG (reading L15, Hestenes-Stiefel) needs per iteration: q = A p (apply_impl.cuh),
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

// Streaming kernels work on double2 pairs (vectors are 16-byte aligned:
// cudaMalloc / torch allocations), U pairs in flight per thread; element i is
// in pair i/2.  The [i0, i1) owned-range mask applies per element.
constexpr int VU = 2;

__global__ void __launch_bounds__(RED_THREADS) dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t i0, int64_t i1, double* partials) {
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    // whole pairs [k0, k1) lie below i1 (no read past element i1 - 1); an odd i1 leaves
    // the tail element i1 - 1, added by one thread below
    const int64_t k0 = i0 / 2, k1 = i1 / 2;
    const int64_t stride = (int64_t)gridDim.x * RED_THREADS;
    double s = 0.0;
    for (int64_t k = k0 + (int64_t)blockIdx.x * RED_THREADS + threadIdx.x; k < k1; k += VU * stride) {
        double2 va[VU], vb[VU];
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk < k1) { va[j] = a2[kk]; vb[j] = b2[kk]; }
            else { va[j] = make_double2(0.0, 0.0); vb[j] = va[j]; }
        }
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t e = 2 * (k + j * stride);
            if (e >= i0 && e < i1) s = fma(va[j].x, vb[j].x, s);
            if (e + 1 >= i0 && e + 1 < i1) s = fma(va[j].y, vb[j].y, s);
        }
    }
    if ((i1 & 1) && i1 - 1 >= i0 && blockIdx.x == 0 && threadIdx.x == 0) s = fma(a[i1 - 1], b[i1 - 1], s);
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) reduce_final_kernel(const double* partials, double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < RED_BLOCKS; i += RED_THREADS) s += partials[i];
    s = block_sum(s);
    if (threadIdx.x == 0) *out = s;
}

// CG step sizes from the device scalars.  The iteration is a no-op once the solve is done
// (S_DONE, set by cg_control: converged, breakdown or maxit -- the eagerly enqueued batches
// of the multi-rank loop run past that point) and on breakdown (p.q <= 0: x is left at the
// last iterate, as the oracle's CG returns it).
__device__ __forceinline__ double cg_alpha(const double* scal) {
    return (scal[S_DONE] != 0.0 || !(scal[S_PQ] > 0.0)) ? 0.0 : scal[S_RR] / scal[S_PQ];
}
__device__ __forceinline__ double cg_beta(const double* scal) {
    return scal[S_RR] > 0.0 ? scal[S_RRNEW] / scal[S_RR] : 0.0;
}

__global__ void __launch_bounds__(RED_THREADS) cg_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p,
                                                            const double* __restrict__ q, int64_t n, int64_t i0,
                                                            int64_t i1, const double* scal, double* partials) {
    const double alpha = cg_alpha(scal);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    const int64_t np = n / 2;
    const int64_t stride = (int64_t)gridDim.x * RED_THREADS;
    const int64_t tid = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x;
    double s = 0.0;
    for (int64_t k = tid; k < np; k += VU * stride) {
        double2 vx[VU], vr[VU], vp[VU], vq[VU];
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk < np) { vx[j] = x2[kk]; vr[j] = r2[kk]; vp[j] = p2[kk]; vq[j] = q2[kk]; }
        }
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk >= np) continue;
            vx[j].x = fma(alpha, vp[j].x, vx[j].x);
            vx[j].y = fma(alpha, vp[j].y, vx[j].y);
            vr[j].x = fma(-alpha, vq[j].x, vr[j].x);
            vr[j].y = fma(-alpha, vq[j].y, vr[j].y);
            x2[kk] = vx[j];
            r2[kk] = vr[j];
            const int64_t e = 2 * kk;
            if (e >= i0 && e < i1) s = fma(vr[j].x, vr[j].x, s);
            if (e + 1 >= i0 && e + 1 < i1) s = fma(vr[j].y, vr[j].y, s);
        }
    }
    if ((n & 1) && tid == 0) {          // odd tail element
        const int64_t e = n - 1;
        x[e] = fma(alpha, p[e], x[e]);
        const double re = fma(-alpha, q[e], r[e]);
        r[e] = re;
        if (e >= i0 && e < i1) s = fma(re, re, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) cg_p_kernel(double* __restrict__ p, const double* __restrict__ r,
                                                           int64_t n, const double* scal) {
    const double beta = cg_beta(scal);
    double2* p2 = reinterpret_cast<double2*>(p);
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const int64_t np = n / 2;
    const int64_t stride = (int64_t)gridDim.x * RED_THREADS;
    const int64_t tid = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x;
    for (int64_t k = tid; k < np; k += VU * stride) {
        double2 vp[VU], vr[VU];
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk < np) { vp[j] = p2[kk]; vr[j] = r2[kk]; }
        }
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk >= np) continue;
            vp[j].x = fma(beta, vp[j].x, vr[j].x);
            vp[j].y = fma(beta, vp[j].y, vr[j].y);
            p2[kk] = vp[j];
        }
    }
    if ((n & 1) && tid == 0) p[n - 1] = fma(beta, p[n - 1], r[n - 1]);
}

__global__ void shift_rr_kernel(double* scal) { scal[S_RR] = scal[S_RRNEW]; }

// Device-side loop control after each CG iteration: a breakdown (p.q <= 0, the iteration
// made no update) ends the solve without counting it; otherwise count the iteration and
// stop on ||r|| <= rtol ||b|| or maxit.  Graph path: also sets the WHILE node's condition.
__global__ void cg_control_kernel(double* scal, double rtol, int maxit, cudaGraphConditionalHandle h, int use_h) {
    if (scal[S_DONE] == 0.0) {
        if (!(scal[S_PQ] > 0.0)) {
            scal[S_DONE] = 1.0;
            scal[S_STATUS] = -9.0;                 // DOGIP_E_BREAKDOWN
        } else {
            const double it = scal[S_IT] + 1.0;
            scal[S_IT] = it;
            if (sqrt(scal[S_RR]) <= rtol * sqrt(scal[S_BB])) {
                scal[S_DONE] = 1.0;
                scal[S_STATUS] = 0.0;              // DOGIP_OK
            } else if (it >= (double)maxit) {
                scal[S_DONE] = 1.0;
                scal[S_STATUS] = 1.0;              // DOGIP_NOT_CONVERGED
            }
        }
    }
    if (use_h) cudaGraphSetConditional(h, scal[S_DONE] == 0.0 ? 1u : 0u);
}

// start of a solve: counters reset; done at once if ||r_0|| <= rtol ||b|| (rtol < 0: never)
__global__ void cg_init_kernel(double* scal, double rtol) {
    scal[S_IT] = 0.0;
    scal[S_STATUS] = 1.0;
    const bool conv = rtol >= 0.0 && sqrt(scal[S_RR]) <= rtol * sqrt(scal[S_BB]);
    scal[S_DONE] = conv ? 1.0 : 0.0;
    if (conv) scal[S_STATUS] = 0.0;
}

// in-process all-reduce of the loopback communicator: out[i] = sum_k slots[k stride + i],
// ranks in fixed order (identical bits on every rank)
__global__ void sum_slots_kernel(const double* slots, int nranks, int64_t stride, int64_t n, double* out) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nranks; ++k) s += slots[k * stride + i];
        out[i] = s;
    }
}

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

// Boundary DoFs of the local slab, enumerated face by face.  Edge / corner DoFs
// appear on several faces; `first` marks the one enumeration that counts them
// (faces in order x0, x1, y0, y1, z0, z1; later faces skip earlier faces' DoFs).
__device__ __forceinline__ bool boundary_dof(const SlabGeo& g, int64_t t, int64_t& idx, bool& first) {
    const int64_t nx = g.pmax_x + 1, ny = g.pmax_y + 1, nz = g.pmax_z + 1;
    first = true;
    if (g.d == 2) {
        // faces x = 0, x = pmax_x over y; y = 0 (bnd_lo), y = pmax_y (bnd_hi) over x
        if (t < 2 * ny) { const int64_t Y = t % ny; idx = (t / ny ? g.pmax_x : 0) + Y * g.sy; return true; }
        t -= 2 * ny;
        const int64_t X = t % nx;
        first = X != 0 && X != g.pmax_x;
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
        const int64_t X = r % nx;
        first = X != 0 && X != g.pmax_x;
        idx = X + (side ? (int64_t)g.pmax_y : 0) * g.sy + (r / nx) * g.sz;
        return true;
    }
    t -= 2 * fy;
    if (t < 2 * fz) {
        const int64_t side = t / fz, r = t % fz;
        if (side == 0 && !g.bnd_lo) return false;
        if (side == 1 && !g.bnd_hi) return false;
        const int64_t X = r % nx, Y = r / nx;
        first = X != 0 && X != g.pmax_x && Y != 0 && Y != g.pmax_y;
        idx = X + Y * g.sy + (side ? (int64_t)g.pmax_z : 0) * g.sz;
        return true;
    }
    return false;
}

__host__ __device__ inline int64_t boundary_count(const SlabGeo& g) {
    const int64_t nx = g.pmax_x + 1, ny = g.pmax_y + 1, nz = g.pmax_z + 1;
    if (g.d == 2) return 2 * ny + 2 * nx;
    return 2 * (ny * nz + nx * nz + nx * ny);
}

__global__ void __launch_bounds__(RED_THREADS) boundary_set_kernel(SlabGeo g, const double* u, double* y,
                                                                   int64_t i0, int64_t i1, double* bpart) {
    const int64_t n = boundary_count(g);
    double s = 0.0;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t idx;
        bool first;
        if (boundary_dof(g, t, idx, first)) {
            const double v = u ? u[idx] : 0.0;
            y[idx] = v;
            if (first && idx >= i0 && idx < i1) s = fma(v, v, s);
        }
    }
    if (bpart) {
        s = block_sum(s);
        if (threadIdx.x == 0) bpart[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(RED_THREADS) sum_partials_kernel(const double* partials, int n, const double* extra,
                                                                   double* out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += RED_THREADS) s += partials[i];
    s = block_sum(s);
    if (threadIdx.x == 0) *out = extra ? s + *extra : s;
}

__global__ void __launch_bounds__(RED_THREADS) cg_r_kernel(double* __restrict__ r, const double* __restrict__ q,
                                                           int64_t n, int64_t i0, int64_t i1, const double* scal,
                                                           double* partials) {
    const double alpha = cg_alpha(scal);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    const int64_t np = n / 2;
    const int64_t stride = (int64_t)gridDim.x * RED_THREADS;
    const int64_t tid = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x;
    double s = 0.0;
    for (int64_t k = tid; k < np; k += VU * stride) {
        double2 vr[VU], vq[VU];
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk < np) { vr[j] = r2[kk]; vq[j] = q2[kk]; }
        }
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk >= np) continue;
            vr[j].x = fma(-alpha, vq[j].x, vr[j].x);
            vr[j].y = fma(-alpha, vq[j].y, vr[j].y);
            r2[kk] = vr[j];
            const int64_t e = 2 * kk;
            if (e >= i0 && e < i1) s = fma(vr[j].x, vr[j].x, s);
            if (e + 1 >= i0 && e + 1 < i1) s = fma(vr[j].y, vr[j].y, s);
        }
    }
    if ((n & 1) && tid == 0) {
        const int64_t e = n - 1;
        const double re = fma(-alpha, q[e], r[e]);
        r[e] = re;
        if (e >= i0 && e < i1) s = fma(re, re, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_THREADS) cg_px_kernel(double* __restrict__ x, double* __restrict__ p,
                                                            const double* __restrict__ r, int64_t n,
                                                            const double* scal) {
    const double alpha = cg_alpha(scal);
    const double beta = cg_beta(scal);
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* p2 = reinterpret_cast<double2*>(p);
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const int64_t np = n / 2;
    const int64_t stride = (int64_t)gridDim.x * RED_THREADS;
    const int64_t tid = (int64_t)blockIdx.x * RED_THREADS + threadIdx.x;
    for (int64_t k = tid; k < np; k += VU * stride) {
        double2 vx[VU], vp[VU], vr[VU];
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk < np) { vx[j] = x2[kk]; vp[j] = p2[kk]; vr[j] = r2[kk]; }
        }
#pragma unroll
        for (int j = 0; j < VU; ++j) {
            const int64_t kk = k + j * stride;
            if (kk >= np) continue;
            vx[j].x = fma(alpha, vp[j].x, vx[j].x);
            vx[j].y = fma(alpha, vp[j].y, vx[j].y);
            vp[j].x = fma(beta, vp[j].x, vr[j].x);
            vp[j].y = fma(beta, vp[j].y, vr[j].y);
            x2[kk] = vx[j];
            p2[kk] = vp[j];
        }
    }
    if ((n & 1) && tid == 0) {
        x[n - 1] = fma(alpha, p[n - 1], x[n - 1]);
        p[n - 1] = fma(beta, p[n - 1], r[n - 1]);
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

cudaError_t launch_cg_control(double* scal, double rtol, int maxit, const cudaGraphConditionalHandle* h,
                              cudaStream_t st) {
    cg_control_kernel<<<1, 1, 0, st>>>(scal, rtol, maxit, h ? *h : cudaGraphConditionalHandle{}, h != nullptr);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_cg_init(double* scal, double rtol, cudaStream_t st) {
    cg_init_kernel<<<1, 1, 0, st>>>(scal, rtol);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_sum_slots(const double* slots, int nranks, int64_t stride, int64_t n, double* out,
                             cudaStream_t st) {
    sum_slots_kernel<<<1, 64, 0, st>>>(slots, nranks, stride, n, out);
    count_launches(1);
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

// Dirichlet rows y_i = u_i restricted to slab-axis DoF planes [P0, P1) (pipelined host apply)
__global__ void __launch_bounds__(RED_THREADS) boundary_planes_kernel(SlabGeo g, const double* __restrict__ u,
                                                                      double* __restrict__ y, int64_t P0, int64_t P1) {
    const int64_t plane = g.d == 3 ? g.sz : g.sy;
    const int64_t n = (P1 - P0) * plane;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = P0 * plane + t;
        const int64_t P = idx / plane, r = idx - P * plane;
        const int64_t X = r % g.sy;
        bool b = X == 0 || X == g.pmax_x || (P == 0 && g.bnd_lo) || (P == (g.d == 3 ? g.pmax_z : g.pmax_y) && g.bnd_hi);
        if (g.d == 3) {
            const int64_t Y = r / g.sy;
            b = b || Y == 0 || Y == g.pmax_y;
        }
        if (b) y[idx] = u[idx];
    }
}

cudaError_t launch_dirichlet_planes(const SlabGeo& g, const double* u, double* y, int64_t P0, int64_t P1,
                                    cudaStream_t st) {
    const int64_t plane = g.d == 3 ? g.sz : g.sy;
    if (P1 <= P0) return cudaSuccess;
    boundary_planes_kernel<<<grid_for((P1 - P0) * plane, RED_THREADS), RED_THREADS, 0, st>>>(g, u, y, P0, P1);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dirichlet_fixup(const SlabGeo& g, const double* u, double* y, cudaStream_t st) {
    boundary_set_kernel<<<grid_for(boundary_count(g), RED_THREADS), RED_THREADS, 0, st>>>(g, u, y, 0, 0, nullptr);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_zero_boundary(const SlabGeo& g, double* y, cudaStream_t st) {
    boundary_set_kernel<<<grid_for(boundary_count(g), RED_THREADS), RED_THREADS, 0, st>>>(g, nullptr, y, 0, 0,
                                                                                          nullptr);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_dirichlet_fixup_dot(const SlabGeo& g, const double* u, double* y, int64_t i0, int64_t i1,
                                       double* bpart, cudaStream_t st) {
    boundary_set_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(g, u, y, i0, i1, bpart);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double* partials, int n, const double* extra, double* out, cudaStream_t st) {
    sum_partials_kernel<<<1, RED_THREADS, 0, st>>>(partials, n, extra, out);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_cg_r(double* r, const double* q, int64_t n, int64_t i0, int64_t i1, double* scal,
                        double* partials, cudaStream_t st) {
    cg_r_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(r, q, n, i0, i1, scal, partials);
    reduce_final_kernel<<<1, RED_THREADS, 0, st>>>(partials, scal + S_RRNEW);
    count_launches(2);
    return cudaGetLastError();
}

cudaError_t launch_cg_px(double* x, double* p, const double* r, int64_t n, double* scal, cudaStream_t st) {
    cg_px_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(x, p, r, n, scal);
    shift_rr_kernel<<<1, 1, 0, st>>>(scal);
    count_launches(2);
    return cudaGetLastError();
}

}  // namespace dogip
