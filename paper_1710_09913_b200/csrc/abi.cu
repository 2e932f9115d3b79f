// abi.cu -- the C ABI of libdogip.so (include/dogip.h): handles, argument
// checking, setup tables, the apply / exchange / CG orchestration on CUDA
// streams.  Every arithmetic step of the path runs in kernels/*.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <memory>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: no-op unless a profiler is attached

#include "../../include/dogip.h"
#include "host/comm.hpp"
#include "host/quadrature.hpp"
#include "host/tables.hpp"
#include "kernels/apply.cuh"

using namespace dogip;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? DOGIP_E_OOM : DOGIP_E_CUDA,       \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                \
    } while (0)
#define NK(call)                                                                            \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            return fail(DOGIP_E_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
    } while (0)
// a collective of the mesh's communicator (comm.hpp); failures carry the backend's message
#define CM(m, call)                                           \
    do {                                                      \
        int rc_ = (call);                                     \
        if (rc_) return fail(rc_, (m)->comm->err);            \
    } while (0)
#define RET(call)                     \
    do {                              \
        int rc_ = (call);             \
        if (rc_ < 0) return rc_;      \
    } while (0)

// host-side NVTX range for the duration of an entry point (nsys / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ handles
struct dogip_mesh_s {
    int d = 0, p = 0, rank = 0, nranks = 1, device = 0, num_sms = 148;
    int64_t N = 0, z0 = 0, z1 = 0;
    SlabGeo geo{};
    ApplyTables tab{};
    RefInfo ref{};          // V-side layout (form independent)
    double* d_verts = nullptr;
    Comm* comm = nullptr;     // NCCL or in-process loopback (owned); null: single rank / partial sums
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_bnd = nullptr, ev_comm = nullptr;
    double* rbuf = nullptr;   // 2 planes: from rank-1, from rank+1
};

struct dogip_op_s {
    dogip_mesh_s* m = nullptr;
    int form = 0, nq = 0, store = 0;
    int kstore = 0;           // storage the apply kernels are instantiated for (6: FULL WP, symmetry-adapted body)
    RefInfo ref{};
    double* d_w = nullptr;
    int64_t w_doubles = 0;
    double* d_sV = nullptr;   // int_ref phi^V_l, for the load vector
    double* r = nullptr;      // CG scratch
    double* pv = nullptr;
    double* q = nullptr;
    double* partials = nullptr;
    double* scal = nullptr;
    double* h_scal = nullptr;  // pinned
    double* hu = nullptr;      // device scratch for the host-buffer apply
    double* hy = nullptr;
    int* d_offw = nullptr;     // global WP: W-lattice offsets [NS][W_T]
    double* dotp = nullptr;    // per-warp partials of p^T A p (3 launches x APPLY_MAX_WARPS)
    double* bpart = nullptr;   // boundary-row partials of the Dirichlet fix-up (RED_BLOCKS)
    float weights_ms = 0.f;
    // quadrature-point comparator (DOGIP_STORE_QP): tables and coefficient data
    double *q_pts = nullptr, *q_wts = nullptr, *q_phi = nullptr, *q_dphi = nullptr, *q_params = nullptr,
           *q_cell = nullptr;
    int q_kind = 0, q_ncomp = 1, q_nq = 0;
    // graph-captured CG loop (single rank): conditional WHILE node around one iteration
    cudaGraph_t cg_graph = nullptr;
    cudaGraphExec_t cg_exec = nullptr;
    cudaStream_t cap_stream = nullptr;   // capture stream (the legacy default stream cannot capture)
    // several ranks (DOGIP_CG_GRAPH_MR=1, capturable communicator): a batch of predicated
    // iterations, NCCL calls included, as one CUDA graph
    cudaGraphExec_t mr_exec = nullptr;
    struct { const double* x = nullptr; unsigned flags = 0; double rtol = 0.0; int maxit = 0, batch = 0; cudaStream_t st = nullptr; } mr_key;
    struct { const double* x = nullptr; unsigned flags = 0; double rtol = 0.0; int maxit = 0; cudaStream_t st = nullptr; } cg_key;
    // pipelined host-buffer apply: copy-in / copy-out streams, one event pair per chunk
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_done;
};

// Makes `dev` current for the scope and restores the caller's device afterwards (setup,
// destroy and synchronous entry points must not leave torch's current device switched).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (dev >= 0 && dev != prev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// Caller vectors are read and written as 16-byte pairs by the CG / reduction kernels.
static int check_vec(const void* p, const char* name) {
    if (!p) return fail(DOGIP_E_INVALID_ARG, std::string("null ") + name);
    if ((reinterpret_cast<uintptr_t>(p) & 15u) != 0)
        return fail(DOGIP_E_INVALID_ARG, std::string(name) + " must be 16-byte aligned");
    return DOGIP_OK;
}

static int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e--) r *= b;
    return r;
}

extern "C" int dogip_version(void) { return 100; }
extern "C" const char* dogip_last_error(void) { return g_err.c_str(); }

extern "C" int dogip_slab_range(int64_t N, int rank, int nranks, int64_t* z0, int64_t* z1) {
    if (nranks < 1 || rank < 0 || rank >= nranks || N < nranks)
        return fail(DOGIP_E_INVALID_SIZE, "slab partition needs N >= nranks >= 1 and 0 <= rank < nranks");
    *z0 = N * rank / nranks;
    *z1 = N * (rank + 1) / nranks;
    return DOGIP_OK;
}

extern "C" int dogip_nccl_unique_id(void* out128) {
    if (!out128) return fail(DOGIP_E_INVALID_ARG, "null output");
    auto& api = nccl();
    if (!api.ok) return fail(DOGIP_E_NCCL, api.err);
    ncclUniqueId id;
    NK(api.GetUniqueId(&id));
    std::memcpy(out128, &id, sizeof id);
    return DOGIP_OK;
}

// ------------------------------------------------------------------ mesh
// ------------------------------------------------------------------ loopback groups
struct dogip_loopback_s {
    LoopbackGroup g;
};

extern "C" int dogip_loopback_create(int nranks, int device, dogip_loopback* out) {
    if (!out) return fail(DOGIP_E_INVALID_ARG, "null output handle");
    *out = nullptr;
    if (nranks < 1) return fail(DOGIP_E_INVALID_SIZE, "loopback group needs nranks >= 1");
    DeviceGuard dg(device);
    auto* L = new dogip_loopback_s();
    L->g.nranks = nranks;
    L->g.device = device;
    L->g.sendbox.resize((size_t)nranks * nranks);
    L->g.donebox.resize((size_t)nranks * nranks);
    L->g.arbox.resize(nranks);
    if (cudaMalloc(&L->g.slots, sizeof(double) * 2 * nranks * LoopbackGroup::SLOT) != cudaSuccess) {
        delete L;
        return fail(DOGIP_E_OOM, "loopback scratch");
    }
    *out = L;
    return DOGIP_OK;
}

extern "C" int dogip_loopback_destroy(dogip_loopback L) {
    if (!L) return DOGIP_OK;
    {
        std::lock_guard<std::mutex> lk(L->g.mu);
        if (L->g.members > 0) return fail(DOGIP_E_INVALID_ARG, "loopback group still has meshes attached");
    }
    DeviceGuard dg(L->g.device);
    cudaFree(L->g.slots);
    delete L;
    return DOGIP_OK;
}

extern "C" int dogip_mesh_setup(int d, int64_t N, int p, const double* vertices, int rank, int nranks,
                                const void* nccl_id, int device, dogip_mesh* out) {
    return dogip_mesh_setup_ex(d, N, p, vertices, rank, nranks, nccl_id ? DOGIP_COMM_NCCL : DOGIP_COMM_NONE,
                               nccl_id, device, out);
}

extern "C" int dogip_mesh_setup_ex(int d, int64_t N, int p, const double* vertices, int rank, int nranks,
                                   int comm_kind, const void* comm_arg, int device, dogip_mesh* out) {
    if (!out) return fail(DOGIP_E_INVALID_ARG, "null output handle");
    if (comm_kind != DOGIP_COMM_NONE && comm_kind != DOGIP_COMM_NCCL && comm_kind != DOGIP_COMM_LOOPBACK)
        return fail(DOGIP_E_INVALID_ARG, "unknown communicator kind");
    if (comm_kind != DOGIP_COMM_NONE && !comm_arg) return fail(DOGIP_E_INVALID_ARG, "communicator argument missing");
    if (comm_kind == DOGIP_COMM_LOOPBACK && device != static_cast<const dogip_loopback_s*>(comm_arg)->g.device)
        return fail(DOGIP_E_INVALID_ARG, "loopback ranks must run on the group's device");
    *out = nullptr;
    if (d != 2 && d != 3) return fail(DOGIP_E_INVALID_DIM, "invalid-dimension: d must be 2 or 3");
    if (N < 1) return fail(DOGIP_E_INVALID_SIZE, "invalid-size: N must be >= 1");
    if (p < 1 || p > 4) return fail(DOGIP_E_UNSUPPORTED_ORDER, "p must be in 1..4");
    if (nranks < 1 || rank < 0 || rank >= nranks || N < nranks)
        return fail(DOGIP_E_INVALID_SIZE, "invalid-size: need N >= nranks >= 1, 0 <= rank < nranks");
    if ((double)ipow(p * N + 1, d) > 9.0e15) return fail(DOGIP_E_INVALID_SIZE, "mesh too large");
    auto* m = new dogip_mesh_s();
    m->d = d; m->N = N; m->p = p; m->rank = rank; m->nranks = nranks; m->device = device;
    dogip_slab_range(N, rank, nranks, &m->z0, &m->z1);
    const int64_t L = m->z1 - m->z0, M = p * N + 1;
    ref_info(d, p, 0, 0, m->ref);
    SlabGeo& g = m->geo;
    g.d = d; g.p = p; g.ns = d == 2 ? 2 : 6; g.N = (int)N;
    g.Nx = (int)N;
    g.Ny = d == 2 ? (int)L : (int)N;
    g.Nz = d == 2 ? 1 : (int)L;
    g.nxb = (int)((N + TILE - 1) / TILE);
    g.ntiles = (int64_t)g.ns * g.nxb * g.Ny * g.Nz;
    g.fd_ns = make_fastdiv((uint32_t)g.ns);
    g.fd_nxb = make_fastdiv((uint32_t)g.nxb);
    g.fd_ny = make_fastdiv((uint32_t)g.Ny);
    if (g.ntiles >= (int64_t)1 << 31) {   // tile_coord's 32-bit arithmetic
        delete m;
        return fail(DOGIP_E_INVALID_SIZE, "invalid-size: 2^31 or more element tiles per rank");
    }
    g.sy = M;
    g.sz = d == 3 ? M * M : 0;
    g.ndof = ipow(M, d - 1) * (p * L + 1);
    g.pmax_x = (int)(p * N);
    g.pmax_y = d == 2 ? (int)(p * L) : (int)(p * N);
    g.pmax_z = d == 2 ? 0 : (int)(p * L);
    g.bnd_lo = m->z0 == 0;
    g.bnd_hi = m->z1 == N;
    g.zoff = m->z0;
    const int64_t MW = 2 * p * N + 1;          // W-lattice of the global WP storage (Theorem 1)
    g.swy = MW;
    g.swz = d == 3 ? MW * MW : 0;
    g.ndof_w = ipow(MW, d - 1) * (2 * p * L + 1);
    g.rw = 2 * p * ((int64_t)g.Nx + 1);
    for (int s = 0; s < g.ns; ++s)
        for (int l = 0; l < m->ref.VT; ++l) {
            const int* o = m->ref.loff[s][l];
            m->tab.off[s * MAX_VT + l] = (int)(o[0] + M * o[1] + (d == 3 ? M * M * o[2] : 0));
            m->tab.loff[s * MAX_VT + l] = o[0] | (o[1] << 8) | (o[2] << 16);
            for (int ax = 0; ax < d; ++ax) {
                if (o[ax] == 0) m->tab.fmask[s][2 * ax] |= 1ull << l;
                if (o[ax] == p) m->tab.fmask[s][2 * ax + 1] |= 1ull << l;
            }
        }
    {
        const auto simp = cell_simplices(d);
        for (int s = 0; s < g.ns; ++s)
            for (int i = 1; i <= d; ++i) {
                const auto& v = simp[s][i];
                m->tab.vstr[s][i - 1] = (int)(v[0] + M * v[1] + (d == 3 ? M * M * v[2] : 0));
            }
    }
    if (device < 0) {   // host-only mesh: partition / numbering introspection, no device work
        *out = m;
        return DOGIP_OK;
    }
    DeviceGuard dg(device);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) { delete m; return fail(DOGIP_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)); }
    cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (vertices) {
        // host-side orientation check of the jittered mesh (E_DEGENERATE_ELEMENT)
        const int64_t nv = ipow(N + 1, d);
        for (int64_t i = 0; i < nv * d; ++i)
            if (!std::isfinite(vertices[i])) { delete m; return fail(DOGIP_E_DEGENERATE_ELEMENT, "non-finite vertex"); }
        e = cudaMalloc(&m->d_verts, sizeof(double) * nv * d);
        if (e == cudaSuccess) e = cudaMemcpy(m->d_verts, vertices, sizeof(double) * nv * d, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(m->d_verts); delete m; return fail(DOGIP_E_OOM, "vertex upload failed"); }
    }
    if (comm_kind != DOGIP_COMM_NONE) {   // also for nranks = 1: exercises the exchange / all-reduce plumbing
        int rc = 0;
        std::string msg;
        if (comm_kind == DOGIP_COMM_NCCL) {
            auto* c = new NcclComm();
            rc = c->init(comm_arg, rank, nranks);
            msg = c->err;
            m->comm = c;
        } else {
            auto* c = new LoopbackComm();
            rc = c->init(&static_cast<dogip_loopback_s*>(const_cast<void*>(comm_arg))->g, rank, nranks);
            msg = c->err;
            m->comm = c;
        }
        if (rc) { dogip_mesh_destroy(m); return fail(rc, msg); }
        cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&m->ev_bnd, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m->ev_comm, cudaEventDisableTiming);
        const int64_t plane = ipow(M, d - 1);
        if (cudaMalloc(&m->rbuf, sizeof(double) * 2 * plane) != cudaSuccess) { dogip_mesh_destroy(m); return fail(DOGIP_E_OOM, "exchange buffers"); }
    }
    *out = m;
    return DOGIP_OK;
}

extern "C" int dogip_mesh_info(dogip_mesh m, dogip_mesh_info_t* o) {
    if (!m || !o) return fail(DOGIP_E_INVALID_ARG, "null argument");
    const int64_t M = m->p * m->N + 1, plane = ipow(M, m->d - 1);
    o->d = m->d; o->p = m->p; o->rank = m->rank; o->nranks = m->nranks;
    o->N = m->N; o->z0 = m->z0; o->z1 = m->z1;
    o->n_elem_local = (m->d == 2 ? 2 : 6) * ipow(m->N, m->d - 1) * (m->z1 - m->z0);
    o->n_elem_global = (m->d == 2 ? 2 : 6) * ipow(m->N, m->d);
    o->ndof_local = m->geo.ndof;
    o->ndof_global = ipow(M, m->d);
    o->plane_size = plane;
    o->dof_offset = m->p * m->z0 * plane;
    o->owned_begin = 0;
    o->owned_end = m->rank < m->nranks - 1 ? m->geo.ndof - plane : m->geo.ndof;
    return DOGIP_OK;
}

extern "C" void dogip_mesh_destroy(dogip_mesh m) {
    if (!m) return;
    if (m->device < 0) { delete m; return; }
    DeviceGuard dg(m->device);
    delete m->comm;
    if (m->comm_stream) cudaStreamDestroy(m->comm_stream);
    if (m->ev_bnd) cudaEventDestroy(m->ev_bnd);
    if (m->ev_comm) cudaEventDestroy(m->ev_comm);
    cudaFree(m->rbuf);
    cudaFree(m->d_verts);
    delete m;
}

// ------------------------------------------------------------------ weights
static int check_coeff(int d, int form, const dogip_coeff* c, int& ncomp) {
    if (!c) return fail(DOGIP_E_BAD_COEFF, "null coefficient");
    const int64_t np = c->nparams;
    auto need = [&](int64_t k) { return np >= k && c->params; };
    ncomp = 1;
    switch (c->kind) {
        case DOGIP_COEF_CONST:
            if (!need(1) || !(c->params[0] > 0)) return fail(DOGIP_E_BAD_COEFF, "CONST needs params[0] > 0");
            return 0;
        case DOGIP_COEF_PER_CELL:
            if (!c->per_cell) return fail(DOGIP_E_BAD_COEFF, "PER_CELL needs per_cell values");
            return 0;
        case DOGIP_COEF_SINCOS2D:
            if (d != 2 || !need(2)) return fail(DOGIP_E_BAD_COEFF, "SINCOS2D needs d = 2 and 2 params");
            return 0;
        case DOGIP_COEF_TANH_RADIAL:
            if (!need(4 + d)) return fail(DOGIP_E_BAD_COEFF, "TANH_RADIAL needs 4 + d params");
            return 0;
        case DOGIP_COEF_ANISO_FOURIER: {
            if (d != 3 || form != DOGIP_EL || !need(4)) return fail(DOGIP_E_BAD_COEFF, "ANISO_FOURIER needs d = 3, EL");
            const int64_t n = (int64_t)c->params[3];
            if (n < 0 || np < 4 + 9 * n) return fail(DOGIP_E_BAD_COEFF, "ANISO_FOURIER parameter count");
            if (!(c->params[0] > 0 && c->params[1] > 0 && c->params[2] > 0)) return fail(DOGIP_E_BAD_COEFF, "eigenvalues must be > 0");
            ncomp = 6;
            return 0;
        }
        case DOGIP_COEF_CONST_TENSOR: {
            if (form != DOGIP_EL || !need(d * d)) return fail(DOGIP_E_BAD_COEFF, "CONST_TENSOR needs EL and d*d params");
            for (int a = 0; a < d; ++a) {
                if (!(c->params[a * d + a] > 0)) return fail(DOGIP_E_BAD_COEFF, "tensor diagonal must be > 0");
                for (int b = 0; b < d; ++b)
                    if (c->params[a * d + b] != c->params[b * d + a]) return fail(DOGIP_E_BAD_COEFF, "tensor not symmetric");
            }
            ncomp = d * (d + 1) / 2;
            return 0;
        }
    }
    return fail(DOGIP_E_BAD_COEFF, "unknown coefficient kind");
}

// Sum the two interface planes (P values each) of a slab vector of length n with the
// neighbours (same plan as the apply exchange); synchronous, setup only.
// An asynchronous communicator failure (dead peer, NCCL error) surfaces at the next call
// on the mesh: the communicator is aborted and E_NCCL returned.
static int comm_check(dogip_mesh_s* m) {
    if (!m->comm) return DOGIP_OK;
    if (const int rc = m->comm->async_error()) {
        const std::string msg = m->comm->err;
        m->comm->abort();
        return fail(rc, msg);
    }
    return DOGIP_OK;
}

// Synchronise `st`.  With a communicator the wait polls the stream and the communicator's
// asynchronous error state; an error, or no progress within DOGIP_COMM_TIMEOUT_S seconds
// (default 600), aborts the communicator (ncclCommAbort releases the blocked kernels) and
// returns E_NCCL instead of hanging on a dead peer.
static int stream_sync(dogip_mesh_s* m, cudaStream_t st) {
    if (!m->comm) {
        CK(cudaStreamSynchronize(st));
        return DOGIP_OK;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) return DOGIP_OK;
        if (e != cudaErrorNotReady) return fail(DOGIP_E_CUDA, std::string("stream: ") + cudaGetErrorString(e));
        RET(comm_check(m));
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (dt > comm_timeout_s()) {
            m->comm->abort();
            return fail(DOGIP_E_NCCL, "timed out waiting for the peers (DOGIP_COMM_TIMEOUT_S); communicator aborted");
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

// Sum the two interface planes (P values each) of a slab vector of length n with the
// neighbours (same plan as the apply exchange); synchronous, setup only.
static int sum_interface_planes(dogip_mesh_s* m, double* v, int64_t P, int64_t n, cudaStream_t st) {
    double* rb = nullptr;
    CK(cudaMalloc(&rb, sizeof(double) * 2 * P));
    struct Free { double* p; ~Free() { cudaFree(p); } } fr{rb};
    CM(m, m->comm->exchange(v, v + n - P, rb, rb + P, P, st));
    CK(launch_add_planes(v, m->rank > 0 ? rb : nullptr, m->rank < m->nranks - 1 ? rb + P : nullptr, P, n - P, st));
    return stream_sync(m, st);
}

// Coefficient parameters as the kernels read them: the caller's array, plus for the
// rotated anisotropic field cos(phi) and sin(phi) of its 3n phases appended (so each point
// needs one sincos per Fourier mode, geometry.cuh coef_eval).
static std::vector<double> device_params(const dogip_coeff* c) {
    std::vector<double> v(c->params, c->params + c->nparams);
    if (c->kind == DOGIP_COEF_ANISO_FOURIER && c->nparams >= 4) {
        const int n = (int)c->params[3];
        const double* phi = c->params + 4 + 3 * n;
        for (int i = 0; i < 3 * n; ++i) v.push_back((double)std::cos((long double)phi[i]));
        for (int i = 0; i < 3 * n; ++i) v.push_back((double)std::sin((long double)phi[i]));
    }
    return v;
}

struct DevBufs {   // frees on scope exit
    std::vector<void*> p;
    ~DevBufs() { for (void* x : p) cudaFree(x); }
    template <class T> cudaError_t alloc(T** out, size_t n) {
        cudaError_t e = cudaMalloc((void**)out, sizeof(T) * std::max<size_t>(n, 1));
        if (e == cudaSuccess) p.push_back(*out);
        return e;
    }
};

extern "C" int dogip_weights(dogip_mesh m, int form, const dogip_coeff* coeff, int quad_n1d, void* stream,
                             dogip_op* out) {
    return dogip_weights_ex(m, form, coeff, quad_n1d, DOGIP_STORE_FULL, stream, out);
}

extern "C" int dogip_weights_ex(dogip_mesh m, int form, const dogip_coeff* coeff, int quad_n1d, int storage,
                                void* stream, dogip_op* out) {
    NvtxRange nv("dogip_weights");
    if (!m || !out) return fail(DOGIP_E_INVALID_ARG, "null argument");
    *out = nullptr;
    if (form != DOGIP_WP && form != DOGIP_EL) return fail(DOGIP_E_INVALID_ARG, "form must be DOGIP_WP or DOGIP_EL");
    if (storage != DOGIP_STORE_FULL && storage != DOGIP_STORE_ISO && storage != DOGIP_STORE_GLOBAL &&
        storage != DOGIP_STORE_QP && storage != DOGIP_STORE_SYM)
        return fail(DOGIP_E_INVALID_ARG, "unknown storage");
    if (storage == DOGIP_STORE_SYM && form != DOGIP_WP)
        return fail(DOGIP_E_INVALID_ARG, "DOGIP_STORE_SYM applies to the weighted projection only");
    if (storage == DOGIP_STORE_ISO && form != DOGIP_EL)
        return fail(DOGIP_E_INVALID_ARG, "DOGIP_STORE_ISO applies to the elliptic form only");
    if (storage == DOGIP_STORE_GLOBAL && form != DOGIP_WP)
        return fail(DOGIP_E_INVALID_ARG, "DOGIP_STORE_GLOBAL (Theorem 1) applies to the weighted projection only");
    if (storage == DOGIP_STORE_GLOBAL && m->nranks > 1 && !m->comm)
        return fail(DOGIP_E_INVALID_ARG, "DOGIP_STORE_GLOBAL on several ranks needs the NCCL communicator");
    if (m->device < 0) return fail(DOGIP_E_INVALID_ARG, "host-only mesh (device < 0) cannot hold an operator");
    int ncomp = 1;
    RET(check_coeff(m->d, form, coeff, ncomp));
    if (storage == DOGIP_STORE_ISO && ncomp != 1)
        return fail(DOGIP_E_BAD_COEFF, "DOGIP_STORE_ISO needs an isotropic coefficient (M = m I)");
    DeviceGuard dg(m->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int d = m->d, p = m->p;
    auto* op = new dogip_op_s();
    op->m = m;
    op->form = form;
    op->store = storage;
    op->kstore = storage;
    // FULL weighted projection: the same a_{T,j} with rows in orbit order where the
    // symmetry-adapted body is instantiated (internal kernel storage 6)
    if (storage == DOGIP_STORE_FULL && form == DOGIP_WP && ref_info(d, p, form, 6, op->ref)) op->kstore = 6;
    else ref_info(d, p, form, (storage == DOGIP_STORE_GLOBAL || storage == DOGIP_STORE_QP) ? 0 : storage, op->ref);
    const int WT = op->ref.WT, NC = op->ref.NC, VT = op->ref.VT;
    const int n1d = quad_n1d > 0 ? quad_n1d : p + 3;
    std::vector<double> pts, wts;
    simplex_rule(d, n1d, pts, wts);
    const int nq = (int)wts.size();
    op->nq = n1d;
    const int kw = form == DOGIP_WP ? 2 * p : 2 * p - 2;
    std::vector<double> phiW((size_t)nq * WT), phiV((size_t)nq * VT), sW(WT), sV(VT);
    eval_basis_ld(d, kw, pts.data(), nq, phiW.data());
    eval_basis_ld(d, p, pts.data(), nq, phiV.data());
    for (int j = 0; j < WT; ++j) {
        long double s = 0;
        for (int q = 0; q < nq; ++q) s += (long double)wts[q] * phiW[(size_t)q * WT + j];
        sW[j] = (double)s;
    }
    for (int l = 0; l < VT; ++l) {
        long double s = 0;
        for (int q = 0; q < nq; ++q) s += (long double)wts[q] * phiV[(size_t)q * VT + l];
        sV[l] = (double)s;
    }
    op->w_doubles = storage == DOGIP_STORE_QP ? 0 : m->geo.ntiles * (int64_t)op->ref.tile_rows * TILE;
    auto cleanup_fail = [&](int code, const std::string& msg) { dogip_op_destroy(op); return fail(code, msg); };
    const std::vector<double> qparams = device_params(coeff);
    if (storage == DOGIP_STORE_QP) {
        // matrix-free comparator: basis values / reference gradients at the n_q points of
        // the same rule, coefficient parameters and per-cell values; nothing per element
        std::vector<double> dphiV((size_t)nq * d * VT);
        eval_grad_ld(d, p, pts.data(), nq, dphiV.data());
        auto up = [&](double** dst, const double* src, size_t n) {
            if (cudaMalloc(dst, sizeof(double) * std::max<size_t>(n, 1)) != cudaSuccess) return false;
            if (n) cudaMemcpy(*dst, src, sizeof(double) * n, cudaMemcpyHostToDevice);
            return true;
        };
        if (!up(&op->d_sV, sV.data(), VT) || !up(&op->q_pts, pts.data(), pts.size()) ||
            !up(&op->q_wts, wts.data(), wts.size()) || !up(&op->q_phi, phiV.data(), phiV.size()) ||
            !up(&op->q_dphi, dphiV.data(), dphiV.size()) ||
            !up(&op->q_params, qparams.data(), qparams.size()))
            return cleanup_fail(DOGIP_E_OOM, "quadrature tables");
        if (coeff->kind == DOGIP_COEF_PER_CELL && !up(&op->q_cell, coeff->per_cell, (size_t)ipow(m->N, d)))
            return cleanup_fail(DOGIP_E_OOM, "per-cell coefficient");
        op->q_kind = coeff->kind;
        op->q_ncomp = ncomp;
        op->q_nq = nq;
        // FP64 flops per element per apply: interpolation + projection at every point
        // (coefficient evaluation and congruence not counted)
        op->ref.flops = form == DOGIP_WP ? nq * (4 * VT + 3) : nq * (4 * d * VT + 2 * d * d + d);
        *out = op;
        return DOGIP_OK;
    }
    if (cudaMalloc(&op->d_w, sizeof(double) * op->w_doubles) != cudaSuccess)
        return cleanup_fail(DOGIP_E_OOM, "weights allocation (" + std::to_string(op->w_doubles * 8) + " bytes)");
    if (cudaMalloc(&op->d_sV, sizeof(double) * VT) != cudaSuccess) return cleanup_fail(DOGIP_E_OOM, "sV");
    cudaMemcpy(op->d_sV, sV.data(), sizeof(double) * VT, cudaMemcpyHostToDevice);

    DevBufs tmp;
    WeightsArgs a{};
    a.d = d; a.p = p; a.form = form;
    a.store = (storage == DOGIP_STORE_GLOBAL || storage == DOGIP_STORE_SYM) ? 0 : storage;
    a.sym = storage == DOGIP_STORE_SYM;
    a.nq = nq; a.WT = WT; a.NC = NC; a.ncomp = ncomp;
    a.NG = op->ref.NG; a.tile_rows = op->ref.tile_rows;
    a.kind = coeff->kind;
    a.nparams = (int)coeff->nparams;
    a.geo = m->geo;
    a.out = op->d_w;
    a.verts = m->d_verts;
    a.stream = st;
    double *dparams = nullptr, *dqp = nullptr, *dqw = nullptr, *dphi = nullptr, *dsW = nullptr, *dcell = nullptr;
    int* dbad = nullptr;
    if (tmp.alloc(&dparams, qparams.size()) || tmp.alloc(&dqp, pts.size()) || tmp.alloc(&dqw, wts.size()) ||
        tmp.alloc(&dphi, phiW.size()) || tmp.alloc(&dsW, WT) || tmp.alloc(&dbad, 1))
        return cleanup_fail(DOGIP_E_OOM, "weight tables");
    if (!qparams.empty()) cudaMemcpy(dparams, qparams.data(), sizeof(double) * qparams.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dqp, pts.data(), sizeof(double) * pts.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dqw, wts.data(), sizeof(double) * wts.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dphi, phiW.data(), sizeof(double) * phiW.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dsW, sW.data(), sizeof(double) * WT, cudaMemcpyHostToDevice);
    cudaMemset(dbad, 0, sizeof(int));
    if (coeff->kind == DOGIP_COEF_PER_CELL) {
        const int64_t ncell = ipow(m->N, d);
        if (tmp.alloc(&dcell, ncell)) return cleanup_fail(DOGIP_E_OOM, "per-cell coefficient");
        cudaMemcpy(dcell, coeff->per_cell, sizeof(double) * ncell, cudaMemcpyHostToDevice);
    }
    a.params = dparams; a.qp = dqp; a.qw = dqw; a.phiW = dphi; a.sW = dsW; a.per_cell = dcell; a.bad_flag = dbad;
    if (a.sym) {
        std::vector<int> hj((size_t)WT * 4);
        std::vector<double> hc((size_t)WT * 4);
        for (int r = 0; r < WT; ++r)
            for (int k = 0; k < 4; ++k) { hj[r * 4 + k] = op->ref.symj[r][k]; hc[r * 4 + k] = op->ref.symc[r][k]; }
        int* dj = nullptr;
        double* dc = nullptr;
        if (tmp.alloc(&dj, hj.size()) || tmp.alloc(&dc, hc.size())) return cleanup_fail(DOGIP_E_OOM, "symmetry tables");
        cudaMemcpy(dj, hj.data(), sizeof(int) * hj.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice);
        a.symj = dj;
        a.symc = dc;
    }
    if (op->ref.has_rowperm) {
        int* drp = nullptr;
        if (tmp.alloc(&drp, WT)) return cleanup_fail(DOGIP_E_OOM, "row permutation");
        cudaMemcpy(drp, op->ref.rowperm, sizeof(int) * WT, cudaMemcpyHostToDevice);
        a.rowperm = drp;
    }
    const bool direct = coeff->kind == DOGIP_COEF_CONST || coeff->kind == DOGIP_COEF_PER_CELL ||
                        coeff->kind == DOGIP_COEF_CONST_TENSOR;
    int64_t batch = (int64_t)(1024ll << 20) / (8ll * ncomp * std::max(nq, WT));   // 1 GB of scratch
    batch = std::max<int64_t>(TILE, batch / TILE * TILE);
    a.batch = batch;
    if (!direct) {
        if (tmp.alloc(&a.scratch_c, (size_t)batch * ncomp * nq) || tmp.alloc(&a.scratch_a, (size_t)batch * ncomp * WT))
            return cleanup_fail(DOGIP_E_OOM, "weight scratch");
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    cudaError_t ce = launch_weights(a);
    cudaEventRecord(e1, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce == cudaSuccess) cudaEventElapsedTime(&op->weights_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ce != cudaSuccess) return cleanup_fail(DOGIP_E_CUDA, std::string("weights kernels: ") + cudaGetErrorString(ce));
    int bad = 0;
    cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost);
    if (bad & 1) return cleanup_fail(DOGIP_E_DEGENERATE_ELEMENT, "an element is degenerate or inverted");
    if (bad & 2) return cleanup_fail(DOGIP_E_BAD_COEFF, "coefficient is not positive at a quadrature point");
    if (storage == DOGIP_STORE_GLOBAL) {
        // Theorem 1: A_ii = int_Omega m phi^W_i = sum over the elements sharing W node i
        std::vector<int> offw((size_t)m->geo.ns * WT);
        const auto AW = multi_indices(d, 2 * p);
        const auto simp = cell_simplices(d);
        const int64_t MW = m->geo.swy;
        for (int s = 0; s < m->geo.ns; ++s)
            for (int j = 0; j < WT; ++j) {
                int o[3] = {0, 0, 0};
                for (int ax = 0; ax < d; ++ax)
                    for (int i = 0; i <= d; ++i) o[ax] += AW[j][i] * simp[s][i][ax];
                offw[(size_t)s * WT + j] = (int)(o[0] + MW * o[1] + (d == 3 ? MW * MW * o[2] : 0));
            }
        // The apply visits a W node once per element sharing it, so the stored diagonal
        // is A_ii / mult_i (u, v continuous at x_i: the sum over those elements gives A_ii).
        double *wg = nullptr, *cnt = nullptr;
        if (cudaMalloc(&op->d_offw, sizeof(int) * offw.size()) != cudaSuccess ||
            cudaMalloc(&wg, sizeof(double) * m->geo.ndof_w) != cudaSuccess ||
            cudaMalloc(&cnt, sizeof(double) * m->geo.ndof_w) != cudaSuccess) {
            cudaFree(wg);
            return cleanup_fail(DOGIP_E_OOM, "global W weights");
        }
        cudaMemcpy(op->d_offw, offw.data(), sizeof(int) * offw.size(), cudaMemcpyHostToDevice);
        cudaMemsetAsync(wg, 0, sizeof(double) * m->geo.ndof_w, st);
        cudaMemsetAsync(cnt, 0, sizeof(double) * m->geo.ndof_w, st);
        ce = launch_globalize(m->geo, WT, op->d_w, op->d_offw, wg, st);
        if (ce == cudaSuccess) ce = launch_globalize(m->geo, WT, nullptr, op->d_offw, cnt, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        cudaFree(op->d_w);
        op->d_w = wg;
        op->w_doubles = m->geo.ndof_w;
        if (ce != cudaSuccess) { cudaFree(cnt); return cleanup_fail(DOGIP_E_CUDA, std::string("globalize: ") + cudaGetErrorString(ce)); }
        if (m->comm) {
            const int64_t PW = m->d == 3 ? MW * MW : MW;
            int rc = sum_interface_planes(m, wg, PW, m->geo.ndof_w, st);
            if (rc >= 0) rc = sum_interface_planes(m, cnt, PW, m->geo.ndof_w, st);
            if (rc < 0) { cudaFree(cnt); dogip_op_destroy(op); return rc; }
        }
        ce = launch_divide(wg, cnt, m->geo.ndof_w, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        cudaFree(cnt);
        if (ce != cudaSuccess) return cleanup_fail(DOGIP_E_CUDA, std::string("globalize: ") + cudaGetErrorString(ce));
        // class-major layout for coalesced gathers: rows of the W lattice (y, z) of length
        // 2p (Nx+1); node offsets re-expressed in it
        const int64_t rows = m->geo.ndof_w / MW;
        double* wp = nullptr;
        if (cudaMalloc(&wp, sizeof(double) * rows * m->geo.rw) != cudaSuccess)
            return cleanup_fail(DOGIP_E_OOM, "global W weights (class-major)");
        cudaMemsetAsync(wp, 0, sizeof(double) * rows * m->geo.rw, st);
        ce = launch_permute_w(m->geo, wg, wp, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        cudaFree(wg);
        op->d_w = wp;
        op->w_doubles = rows * m->geo.rw;
        if (ce != cudaSuccess) return cleanup_fail(DOGIP_E_CUDA, std::string("permute W: ") + cudaGetErrorString(ce));
        const int twop = 2 * p;
        for (auto& o : offw) {
            const int64_t ox = o % MW, oy = (o / MW) % MW, oz = d == 3 ? o / (MW * MW) : 0;
            o = (int)(m->geo.rw * (oy + MW * oz) + (ox % twop) * (m->geo.Nx + 1) + ox / twop);
        }
        cudaMemcpy(op->d_offw, offw.data(), sizeof(int) * offw.size(), cudaMemcpyHostToDevice);
    }
    *out = op;
    return DOGIP_OK;
}

extern "C" int dogip_op_info(dogip_op op, dogip_op_info_t* o) {
    if (!op || !o) return fail(DOGIP_E_INVALID_ARG, "null argument");
    o->form = op->form; o->d = op->m->d; o->p = op->m->p;
    o->V_T = op->ref.VT; o->W_T = op->ref.WT;
    o->n_c = op->form == DOGIP_WP ? 1 : op->m->d * (op->m->d + 1) / 2;
    o->storage = op->store;
    o->stream_doubles_per_elem =
        (op->store == DOGIP_STORE_GLOBAL || op->store == DOGIP_STORE_QP) ? 0 : op->ref.tile_rows;
    o->flops_per_elem = op->ref.flops;
    o->quad_n1d = op->nq;
    o->n_tiles = op->m->geo.ntiles;
    o->weight_bytes = op->w_doubles * 8;
    o->weights_ms = op->weights_ms;
    return DOGIP_OK;
}

extern "C" void dogip_op_destroy(dogip_op op) {
    if (!op) return;
    DeviceGuard dg(op->m->device);
    for (double* x : {op->d_w, op->d_sV, op->r, op->pv, op->q, op->partials, op->scal, op->hu, op->hy, op->dotp,
                      op->bpart})
        cudaFree(x);
    cudaFree(op->d_offw);
    for (double* x : {op->q_pts, op->q_wts, op->q_phi, op->q_dphi, op->q_params, op->q_cell}) cudaFree(x);
    if (op->h_scal) cudaFreeHost(op->h_scal);
    if (op->cg_exec) cudaGraphExecDestroy(op->cg_exec);
    if (op->mr_exec) cudaGraphExecDestroy(op->mr_exec);
    if (op->cg_graph) cudaGraphDestroy(op->cg_graph);
    if (op->cap_stream) cudaStreamDestroy(op->cap_stream);
    for (cudaEvent_t e : op->ev_in) cudaEventDestroy(e);
    for (cudaEvent_t e : op->ev_done) cudaEventDestroy(e);
    if (op->s_h2d) cudaStreamDestroy(op->s_h2d);
    if (op->s_d2h) cudaStreamDestroy(op->s_d2h);
    delete op;
}

// ------------------------------------------------------------------ apply
static int exchange_planes(dogip_mesh_s* m, double* y, cudaEvent_t ready) {
    NvtxRange nv("dogip_exchange");
    // sum this rank's partial interface planes with the neighbours' (A8)
    const int64_t P = m->d == 3 ? m->geo.sy * m->geo.sy : m->geo.sy;
    const int64_t last = m->geo.ndof - P;
    CK(cudaStreamWaitEvent(m->comm_stream, ready, 0));
    CM(m, m->comm->exchange(y, y + last, m->rbuf, m->rbuf + P, P, m->comm_stream));
    CK(cudaEventRecord(m->ev_comm, m->comm_stream));
    return DOGIP_OK;
}

static int finish_exchange(dogip_mesh_s* m, double* y, cudaStream_t st) {
    const int64_t P = m->d == 3 ? m->geo.sy * m->geo.sy : m->geo.sy;
    CK(cudaStreamWaitEvent(st, m->ev_comm, 0));
    CK(launch_add_planes(y, m->rank > 0 ? m->rbuf : nullptr, m->rank < m->nranks - 1 ? m->rbuf + P : nullptr, P,
                         m->geo.ndof - P, st));
    return DOGIP_OK;
}

// the comparator's launch arguments for the same tile range / flags as an apply
static QpArgs qp_args(dogip_op op, const ApplyArgs& a) {
    QpArgs q{};
    q.d = a.d; q.p = a.p; q.form = a.form; q.dirichlet = a.dirichlet;
    q.u = a.u; q.y = a.y; q.geo = a.geo; q.tab = a.tab;
    q.nq = op->q_nq; q.qp = op->q_pts; q.qw = op->q_wts; q.phi = op->q_phi; q.dphi = op->q_dphi;
    q.kind = op->q_kind; q.ncomp = op->q_ncomp; q.params = op->q_params; q.per_cell = op->q_cell;
    q.verts = op->m->d_verts;
    q.tile_begin = a.tile_begin; q.tile_end = a.tile_end;
    q.num_sms = a.num_sms; q.stream = a.stream;
    q.dot_partials = a.dot_partials; q.dot_nslots = a.dot_nslots;
    return q;
}

// y = A u (+ exchange); with dot != null also *dot = u^T y over this rank's elements
// (+ boundary rows owned by this rank), fused into the apply kernel (CG's p.q).
constexpr int MAX_APPLY_LAUNCHES = 3;   // per apply: boundary layers (2) + interior

static int apply_impl(dogip_op op, const double* u, double* y, unsigned flags, cudaStream_t st,
                      double* dot = nullptr, const double* skip_if = nullptr) {
    dogip_mesh_s* m = op->m;
    const SlabGeo& g = m->geo;
    const bool xchg = m->comm && !(flags & DOGIP_NO_EXCHANGE);
    CK(cudaMemsetAsync(y, 0, sizeof(double) * g.ndof, st));
    ApplyArgs a{};
    a.d = m->d; a.p = m->p; a.form = op->form; a.store = op->kstore;
    a.offw = op->d_offw;
    a.dirichlet = (flags & DOGIP_DIRICHLET_ZERO) != 0;
    a.u = u; a.y = y; a.w = op->d_w; a.geo = g; a.tab = &m->tab;
    a.num_sms = m->num_sms;
    a.stream = st;
    a.skip_if = skip_if;
    bool rows_written = false;
    a.rows_written = &rows_written;
    int nslots[MAX_APPLY_LAUNCHES] = {};
    int nl = 0;
    if (dot && !op->dotp) {
        CK(cudaMalloc(&op->dotp, sizeof(double) * MAX_APPLY_LAUNCHES * APPLY_MAX_WARPS));
        CK(cudaMalloc(&op->bpart, sizeof(double) * RED_BLOCKS));
    }
    int64_t slot0 = 0;   // the launches' per-warp partials of p.q are packed back to back
    auto launch = [&](int64_t t0, int64_t t1) -> cudaError_t {
        a.tile_begin = t0;
        a.tile_end = t1;
        a.dot_partials = dot ? op->dotp + slot0 : nullptr;
        a.dot_nslots = &nslots[nl];
        const cudaError_t e = op->store == DOGIP_STORE_QP ? launch_qp_apply(qp_args(op, a)) : launch_apply(a);
        slot0 += nslots[nl];
        ++nl;
        return e;
    };
    if (!xchg) {
        CK(launch(0, g.ntiles));
    } else {
        // boundary cube layers first, exchange overlapped with the interior layers
        const int64_t layers = m->z1 - m->z0;
        const int64_t tpl = g.ntiles / layers;
        if (layers <= 2) {
            CK(launch(0, g.ntiles));
            CK(cudaEventRecord(m->ev_bnd, st));
            RET(exchange_planes(m, y, m->ev_bnd));
        } else {
            CK(launch(0, tpl));
            CK(launch(g.ntiles - tpl, g.ntiles));
            CK(cudaEventRecord(m->ev_bnd, st));
            RET(exchange_planes(m, y, m->ev_bnd));
            CK(launch(tpl, g.ntiles - tpl));
        }
        RET(finish_exchange(m, y, st));
    }
    if (dot) {
        CK(launch_sum_partials(op->dotp, (int)slot0, nullptr, dot, st));
    }
    // the cell-per-lane kernel (p <= 2) writes the Dirichlet rows itself (one owner per row,
    // its u_i^2 in the fused dot); the other kernels take the separate fix-up
    if (a.dirichlet && !rows_written) {
        if (dot) {
            dogip_mesh_info_t info;
            dogip_mesh_info(m, &info);
            CK(launch_dirichlet_fixup_dot(g, u, y, info.owned_begin, info.owned_end, op->bpart, st));
            CK(launch_sum_partials(op->bpart, RED_BLOCKS, dot, dot, st));
        } else {
            CK(launch_dirichlet_fixup(g, u, y, st));
        }
    }
    return DOGIP_OK;
}

extern "C" int dogip_apply(dogip_op op, const double* u, double* y, unsigned flags, void* stream) {
    NvtxRange nv("dogip_apply");
    if (!op) return fail(DOGIP_E_INVALID_ARG, "null argument");
    RET(check_vec(u, "u"));
    RET(check_vec(y, "y"));
    if (u == y) return fail(DOGIP_E_INVALID_ARG, "u and y must not alias");
    if (flags & ~(DOGIP_DIRICHLET_ZERO | DOGIP_NO_EXCHANGE)) return fail(DOGIP_E_INVALID_ARG, "unknown flags");
    RET(comm_check(op->m));
    return apply_impl(op, u, y, flags, (cudaStream_t)stream);
}

// Host-buffer apply, pipelined over chunks of cube layers along the slab axis (single
// rank): the copy-in of chunk c+1's u planes, the apply kernel of chunk c's elements
// and the copy-out of the y planes chunk c completed run on three streams.  Tiles are
// ordered with the slab axis slowest, so chunk c = layers [a, b) = tiles [a tpl, b tpl)
// reads DoF planes [p a, p b] and completes planes [p a, p b) (the last chunk also p b).
// Dirichlet rows (y_i = u_i) are written per completed plane range (the cell kernel writes
// them itself, in the chunk holding the row's floor cell); the DIRICHLET kernels never
// scatter into boundary DoFs, so the order against later chunks is free.
static int apply_host_pipelined(dogip_op op, const double* u_host, double* y_host, unsigned flags,
                                cudaStream_t st) {
    dogip_mesh_s* m = op->m;
    const SlabGeo& g = m->geo;
    const int64_t layers = g.d == 3 ? g.Nz : g.Ny;
    const int64_t tpl = g.ntiles / layers;
    const int64_t plane = g.d == 3 ? g.sz : g.sy;
    const int p = m->p;
    int kmax = 24;                                   // chunks (DOGIP_HOST_CHUNKS overrides, A/B;
                                                     // 24 vs 16 / 32: +2.4 % / +4 % e2e on C4)
    if (const char* e = std::getenv("DOGIP_HOST_CHUNKS")) kmax = std::max(1, std::atoi(e));
    const int K = (int)std::min<int64_t>(layers, kmax);
    const bool dir = (flags & DOGIP_DIRICHLET_ZERO) != 0;
    if (!op->s_h2d) {
        CK(cudaStreamCreateWithFlags(&op->s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&op->s_d2h, cudaStreamNonBlocking));
    }
    while ((int)op->ev_in.size() < K + 1) {
        cudaEvent_t a, b;
        CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        op->ev_in.push_back(a);
        op->ev_done.push_back(b);
    }
    // the caller's stream orders us after its prior work; y starts from zero (atomics)
    CK(cudaEventRecord(op->ev_in[K], st));
    CK(cudaStreamWaitEvent(op->s_h2d, op->ev_in[K], 0));
    CK(cudaMemsetAsync(op->hy, 0, sizeof(double) * g.ndof, st));
    int64_t in_end = 0, out_end = 0;   // DoF planes copied in / out so far
    for (int c = 0; c < K; ++c) {
        const int64_t a = layers * c / K, b = layers * (c + 1) / K;
        const int64_t need = p * b + 1;                         // planes [0, p b] resident
        CK(cudaMemcpyAsync(op->hu + in_end * plane, u_host + in_end * plane,
                           sizeof(double) * (need - in_end) * plane, cudaMemcpyHostToDevice, op->s_h2d));
        in_end = need;
        CK(cudaEventRecord(op->ev_in[c], op->s_h2d));
        CK(cudaStreamWaitEvent(st, op->ev_in[c], 0));
        ApplyArgs aa{};
        aa.d = m->d; aa.p = p; aa.form = op->form; aa.store = op->kstore;
        aa.offw = op->d_offw;
        aa.dirichlet = dir;
        aa.u = op->hu; aa.y = op->hy; aa.w = op->d_w; aa.geo = g; aa.tab = &m->tab;
        aa.num_sms = m->num_sms;
        aa.stream = st;
        aa.tile_begin = a * tpl;
        aa.tile_end = b * tpl;
        bool rows_written = false;
        aa.rows_written = &rows_written;
        CK(op->store == DOGIP_STORE_QP ? launch_qp_apply(qp_args(op, aa)) : launch_apply(aa));
        const int64_t done = c == K - 1 ? p * b + 1 : p * b;    // planes [out_end, done) are final
        // Dirichlet rows: written by the cell kernel of the chunk owning them, else here
        if (dir && !rows_written) CK(launch_dirichlet_planes(g, op->hu, op->hy, out_end, done, st));
        CK(cudaEventRecord(op->ev_done[c], st));
        CK(cudaStreamWaitEvent(op->s_d2h, op->ev_done[c], 0));
        CK(cudaMemcpyAsync(y_host + out_end * plane, op->hy + out_end * plane,
                           sizeof(double) * (done - out_end) * plane, cudaMemcpyDeviceToHost, op->s_d2h));
        out_end = done;
    }
    CK(cudaStreamSynchronize(op->s_d2h));
    CK(cudaStreamSynchronize(st));
    return DOGIP_OK;
}

extern "C" int dogip_apply_host(dogip_op op, const double* u_host, double* y_host, unsigned flags, void* stream) {
    NvtxRange nv("dogip_apply_host");
    if (!op || !u_host || !y_host) return fail(DOGIP_E_INVALID_ARG, "null argument");
    if (flags & ~(DOGIP_DIRICHLET_ZERO | DOGIP_NO_EXCHANGE)) return fail(DOGIP_E_INVALID_ARG, "unknown flags");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = op->m->geo.ndof;
    DeviceGuard dg(op->m->device);
    if (!op->hu) {
        CK(cudaMalloc(&op->hu, sizeof(double) * n));
        CK(cudaMalloc(&op->hy, sizeof(double) * n));
    }
    const bool xchg = op->m->comm && !(flags & DOGIP_NO_EXCHANGE);
    if (!xchg) return apply_host_pipelined(op, u_host, y_host, flags, st);
    CK(cudaMemcpyAsync(op->hu, u_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    RET(dogip_apply(op, op->hu, op->hy, flags, stream));
    CK(cudaMemcpyAsync(y_host, op->hy, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    RET(stream_sync(op->m, st));
    return DOGIP_OK;
}

extern "C" int dogip_load_vector(dogip_op op, double f, double* b, unsigned flags, void* stream) {
    NvtxRange nv("dogip_load_vector");
    if (!op) return fail(DOGIP_E_INVALID_ARG, "null argument");
    RET(check_vec(b, "b"));
    RET(comm_check(op->m));
    cudaStream_t st = (cudaStream_t)stream;
    dogip_mesh_s* m = op->m;
    CK(cudaMemsetAsync(b, 0, sizeof(double) * m->geo.ndof, st));
    CK(launch_load_vector(m->geo, m->p, m->d_verts, op->d_sV, op->ref.VT, &m->tab, f, b, st));
    if (m->comm && !(flags & DOGIP_NO_EXCHANGE)) {
        CK(cudaEventRecord(m->ev_bnd, st));
        RET(exchange_planes(m, b, m->ev_bnd));
        RET(finish_exchange(m, b, st));
    }
    if (flags & DOGIP_DIRICHLET_ZERO) CK(launch_zero_boundary(m->geo, b, st));
    return DOGIP_OK;
}

// ------------------------------------------------------------------ CG
static int allreduce_scalar(dogip_mesh_s* m, double* s, cudaStream_t st) {
    if (m->comm) CM(m, m->comm->allreduce_sum(s, 1, st));
    return DOGIP_OK;
}

extern "C" int64_t dogip_kernel_launches(void) { return (int64_t)g_launches.load(); }

// One CG iteration (Hestenes-Stiefel, reading L15), every step on the device:
//   q = A p, p.q fused into the apply            [all-reduce p.q]
//   r -= alpha q, r.r                            [all-reduce r.r]
//   x += alpha p, p = r + beta p
//   control: breakdown / count / convergence / maxit -> S_DONE (graph path: WHILE condition)
// An iteration enqueued after the solve finished is a no-op (the apply kernel returns at
// once and alpha = 0), so batches of iterations are enqueued without a host round trip.
static int cg_iteration(dogip_op op, double* x, unsigned aflags, double rtol, int maxit,
                        const cudaGraphConditionalHandle* h, cudaStream_t st, cudaEvent_t ev0 = nullptr,
                        cudaEvent_t ev1 = nullptr) {
    dogip_mesh_s* m = op->m;
    dogip_mesh_info_t info;
    dogip_mesh_info(m, &info);
    const int64_t n = m->geo.ndof;
    if (ev0) CK(cudaEventRecord(ev0, st));
    RET(apply_impl(op, op->pv, op->q, aflags, st, op->scal + S_PQ, op->scal + S_DONE));   // q = A p
    if (ev1) CK(cudaEventRecord(ev1, st));
    RET(allreduce_scalar(m, op->scal + S_PQ, st));
    CK(launch_cg_r(op->r, op->q, n, info.owned_begin, info.owned_end, op->scal, op->partials, st));
    RET(allreduce_scalar(m, op->scal + S_RRNEW, st));
    CK(launch_cg_px(x, op->pv, op->r, n, op->scal, st));
    CK(launch_cg_control(op->scal, rtol, maxit, h, st));
    return DOGIP_OK;
}

// The CG iterations of a single-rank solve as one CUDA graph: a conditional WHILE node
// whose body is one cg_iteration; its control kernel sets the condition, so the loop runs
// without a host round trip.  Rebuilt when x, the flags, rtol, maxit or the stream change.
static int cg_graph_build(dogip_op op, double* x, double rtol, int maxit, unsigned aflags, cudaStream_t st) {
    auto& k = op->cg_key;
    if (!op->cg_exec || k.x != x || k.flags != aflags || k.rtol != rtol || k.maxit != maxit || k.st != st) {
        if (op->cg_exec) { cudaGraphExecDestroy(op->cg_exec); op->cg_exec = nullptr; }
        if (op->cg_graph) { cudaGraphDestroy(op->cg_graph); op->cg_graph = nullptr; }
        CK(cudaGraphCreate(&op->cg_graph, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, op->cg_graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, op->cg_graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        if (!op->cap_stream) CK(cudaStreamCreateWithFlags(&op->cap_stream, cudaStreamNonBlocking));
        cudaStream_t cs = op->cap_stream;
        CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        const int rc = cg_iteration(op, x, aflags, rtol, maxit, &h, cs);
        cudaGraph_t captured = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(cs, &captured);
        if (rc < 0) return rc;
        CK(ee);
        CK(cudaGraphInstantiate(&op->cg_exec, op->cg_graph, 0));
        k.x = x; k.flags = aflags; k.rtol = rtol; k.maxit = maxit; k.st = st;
    }
    return DOGIP_OK;
}

// Several ranks: `batch` predicated iterations -- exchange and all-reduces of the
// communicator included -- captured once as a plain CUDA graph (opt-in, DOGIP_CG_GRAPH_MR=1;
// validated with a 1-rank NCCL communicator on the one-GPU pool).  Rebuilt when x, the flags,
// rtol, maxit, the batch or the stream change.
static int cg_batch_graph_build(dogip_op op, double* x, double rtol, int maxit, unsigned aflags, cudaStream_t st,
                                int batch) {
    auto& k = op->mr_key;
    if (op->mr_exec && k.x == x && k.flags == aflags && k.rtol == rtol && k.maxit == maxit && k.batch == batch &&
        k.st == st)
        return DOGIP_OK;
    if (op->mr_exec) { cudaGraphExecDestroy(op->mr_exec); op->mr_exec = nullptr; }
    if (!op->cap_stream) CK(cudaStreamCreateWithFlags(&op->cap_stream, cudaStreamNonBlocking));
    cudaStream_t cs = op->cap_stream;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = DOGIP_OK;
    for (int i = 0; i < batch && rc >= 0; ++i) rc = cg_iteration(op, x, aflags, rtol, maxit, nullptr, cs);
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(cs, &g);
    if (rc < 0) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    CK(ee);
    const cudaError_t ie = cudaGraphInstantiate(&op->mr_exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) { op->mr_exec = nullptr; CK(ie); }
    k.x = x; k.flags = aflags; k.rtol = rtol; k.maxit = maxit; k.batch = batch; k.st = st;
    return DOGIP_OK;
}

extern "C" int dogip_cg(dogip_op op, const double* b, double* x, double rtol, int maxit, unsigned flags,
                        void* stream, dogip_cg_result* res) {
    NvtxRange nv("dogip_cg");
    if (!op || !res) return fail(DOGIP_E_INVALID_ARG, "null argument");
    RET(check_vec(b, "b"));
    RET(check_vec(x, "x"));
    if (flags & ~(DOGIP_DIRICHLET_ZERO | DOGIP_CG_RESUME)) return fail(DOGIP_E_INVALID_ARG, "unknown flags");
    cudaStream_t st = (cudaStream_t)stream;
    dogip_mesh_s* m = op->m;
    RET(comm_check(m));
    const int64_t n = m->geo.ndof;
    dogip_mesh_info_t info;
    dogip_mesh_info(m, &info);
    const int64_t o0 = info.owned_begin, o1 = info.owned_end;
    const bool resume = (flags & DOGIP_CG_RESUME) != 0;
    if (resume && !op->r) return fail(DOGIP_E_INVALID_ARG, "DOGIP_CG_RESUME without a previous dogip_cg call");
    if (!op->r) {
        CK(cudaMalloc(&op->r, sizeof(double) * n));
        CK(cudaMalloc(&op->pv, sizeof(double) * n));
        CK(cudaMalloc(&op->q, sizeof(double) * n));
        CK(cudaMalloc(&op->partials, sizeof(double) * RED_BLOCKS));
        CK(cudaMalloc(&op->scal, sizeof(double) * S_COUNT));
        CK(cudaMallocHost(&op->h_scal, sizeof(double) * S_COUNT));
    }
    if (!op->dotp) {
        CK(cudaMalloc(&op->dotp, sizeof(double) * MAX_APPLY_LAUNCHES * APPLY_MAX_WARPS));
        CK(cudaMalloc(&op->bpart, sizeof(double) * RED_BLOCKS));
    }
    const unsigned aflags = flags & DOGIP_DIRICHLET_ZERO;
    const bool bench = maxit < 0;
    const int nit = bench ? -maxit : maxit;
    const double rtol_dev = bench ? -1.0 : rtol;      // fixed-count runs never test convergence
    cudaEvent_t t0, t1;
    CK(cudaEventCreate(&t0));
    CK(cudaEventCreate(&t1));
    std::vector<cudaEvent_t> aev;
    struct EvGuard {
        cudaEvent_t a, b;
        std::vector<cudaEvent_t>* v;
        ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); for (auto e : *v) cudaEventDestroy(e); }
    } guard{t0, t1, &aev};
    if (bench) {
        aev.resize(2 * (size_t)nit);
        for (auto& e : aev) CK(cudaEventCreate(&e));
    }
    // single rank: the graph-captured loop is built (or reused) before the timed region
    const bool graph = !bench && nit > 0 && !m->comm && std::getenv("DOGIP_CG_NO_GRAPH") == nullptr;
    if (graph) RET(cg_graph_build(op, x, rtol_dev, nit, aflags, st));
    int batch = 32;
    if (const char* e = std::getenv("DOGIP_CG_BATCH")) batch = std::max(1, std::atoi(e));
    const char* mre = std::getenv("DOGIP_CG_GRAPH_MR");
    const bool mr_graph = !bench && nit > 0 && m->comm && m->comm->capturable() && mre && mre[0] == '1';
    if (mr_graph) RET(cg_batch_graph_build(op, x, rtol_dev, nit, aflags, st, batch));
    CK(cudaEventRecord(t0, st));
    if (!resume) {
        // r = b - A x ; p = r
        RET(apply_impl(op, x, op->q, aflags, st));
        CK(cudaMemcpyAsync(op->r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        CK(launch_axpby(op->r, op->q, -1.0, 1.0, n, st));
        CK(cudaMemcpyAsync(op->pv, op->r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        CK(launch_dot(op->r, op->r, o0, o1, op->partials, op->scal + S_RR, st));
        RET(allreduce_scalar(m, op->scal + S_RR, st));
    }
    CK(launch_dot(b, b, o0, o1, op->partials, op->scal + S_BB, st));
    RET(allreduce_scalar(m, op->scal + S_BB, st));
    CK(launch_cg_init(op->scal, rtol_dev, st));
    if (!bench) {
        // one host read per solve: b = 0 returns x untouched; ||r_0|| small enough stops here
        CK(cudaMemcpyAsync(op->h_scal, op->scal, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st));
        RET(stream_sync(m, st));
        if (op->h_scal[S_BB] == 0.0) {
            res->iters = 0; res->status = DOGIP_OK; res->rel_res = 0.0; res->seconds = 0.0; res->apply_seconds = 0.0;
            return DOGIP_OK;
        }
        if (op->h_scal[S_DONE] == 0.0 && nit > 0) {
            if (graph) {
                CK(cudaGraphLaunch(op->cg_exec, st));
            } else {
                // batches of predicated iterations (eager, or one captured graph per batch),
                // one host read of the device's done flag per batch
                for (int enq = 0; enq < nit;) {
                    const int kk = mr_graph ? batch : std::min(batch, nit - enq);
                    if (mr_graph) CK(cudaGraphLaunch(op->mr_exec, st));
                    else for (int i = 0; i < kk; ++i) RET(cg_iteration(op, x, aflags, rtol_dev, nit, nullptr, st));
                    enq += kk;
                    CK(cudaMemcpyAsync(op->h_scal, op->scal, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st));
                    RET(stream_sync(m, st));
                    if (op->h_scal[S_DONE] != 0.0) break;
                }
            }
        }
    } else {
        for (int i = 0; i < nit; ++i) RET(cg_iteration(op, x, aflags, rtol_dev, nit, nullptr, st, aev[2 * i], aev[2 * i + 1]));
    }
    CK(cudaEventRecord(t1, st));
    CK(cudaMemcpyAsync(op->h_scal, op->scal, sizeof(double) * S_COUNT, cudaMemcpyDeviceToHost, st));
    RET(stream_sync(m, st));
    const double* hs = op->h_scal;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    double aps = 0.0;
    for (int i = 0; i < (bench ? nit : 0); ++i) {
        float a = 0.f;
        cudaEventElapsedTime(&a, aev[2 * i], aev[2 * i + 1]);
        aps += a * 1e-3;
    }
    int status = (int)hs[S_STATUS];
    if (hs[S_DONE] == 0.0) status = DOGIP_NOT_CONVERGED;        // maxit = 0, or batches exhausted
    if (bench && status == DOGIP_NOT_CONVERGED) status = DOGIP_OK;
    res->iters = (int)hs[S_IT];
    res->status = status;
    res->rel_res = hs[S_BB] > 0 ? std::sqrt(hs[S_RR]) / std::sqrt(hs[S_BB]) : 0.0;
    res->seconds = ms * 1e-3;
    res->apply_seconds = aps;
    if (status == DOGIP_E_BREAKDOWN) return fail(DOGIP_E_BREAKDOWN, "CG breakdown: p^T A p <= 0");
    return status;
}

// ------------------------------------------------------------------ introspection
extern "C" int dogip_reference_table(int d, int p, int form, double* out, int64_t cap) {
    if ((d != 2 && d != 3)) return fail(DOGIP_E_INVALID_DIM, "d must be 2 or 3");
    if (p < 1 || p > 8) return fail(DOGIP_E_UNSUPPORTED_ORDER, "p must be in 1..8 for tables");
    if (form != DOGIP_WP && form != DOGIP_EL) return fail(DOGIP_E_INVALID_ARG, "bad form");
    Table t;
    try { t = bhat_table(d, p, form); } catch (const std::exception& e) { return fail(DOGIP_E_INVALID_ARG, e.what()); }
    const int64_t n = (int64_t)t.v.size();
    if (out) {
        if (cap < n) return fail(DOGIP_E_INVALID_SIZE, "capacity too small");
        for (int64_t i = 0; i < n; ++i) out[i] = t.v[i].to_double();
    }
    return (int)n;
}

extern "C" int dogip_reference_nnz(int d, int p, int form, int64_t* nnz, int64_t* pm1) {
    if ((d != 2 && d != 3)) return fail(DOGIP_E_INVALID_DIM, "d must be 2 or 3");
    if (p < 1 || p > 8) return fail(DOGIP_E_UNSUPPORTED_ORDER, "p must be in 1..8 for tables");
    if (form != DOGIP_WP && form != DOGIP_EL) return fail(DOGIP_E_INVALID_ARG, "bad form");
    Table t;
    try { t = bhat_table(d, p, form); } catch (const std::exception& e) { return fail(DOGIP_E_INVALID_ARG, e.what()); }
    int64_t a = 0, b = 0;
    for (auto& v : t.v) { a += !v.is_zero(); b += v.is_pm1(); }
    if (nnz) *nnz = a;
    if (pm1) *pm1 = b;
    return DOGIP_OK;
}

// exact count of distinct DoF pairs sharing an element, structured mesh of n cells
static int64_t csr_nnz_direct(int d, int64_t n, int p) {
    const auto A = multi_indices(d, p);
    const auto simp = cell_simplices(d);
    struct RI {
        int VT;
        std::vector<std::array<std::array<int, 3>, 128>> loff;   // [s][l][axis], V_T <= 84
    } ri;
    ri.VT = (int)A.size();
    ri.loff.resize(simp.size());
    for (size_t s = 0; s < simp.size(); ++s)
        for (int l = 0; l < ri.VT; ++l)
            for (int ax = 0; ax < 3; ++ax) {
                int o = 0;
                for (int i = 0; i <= d; ++i) o += A[l][i] * simp[s][i][ax];
                ri.loff[s][l][ax] = ax < d ? o : 0;
            }
    const int64_t M = p * n + 1;
    const int ns = d == 2 ? 2 : 6;
    const int64_t ncell = d == 2 ? n * n : n * n * n;
    std::vector<uint64_t> keys;
    keys.reserve((size_t)ncell * ns * ri.VT * ri.VT);
    const uint64_t nd = (uint64_t)(d == 2 ? M * M : M * M * M);
    std::vector<int64_t> ids(ri.VT);
    for (int64_t c = 0; c < ncell; ++c) {
        const int64_t ci = c % n, cj = (c / n) % n, ck = d == 3 ? c / (n * n) : 0;
        for (int s = 0; s < ns; ++s) {
            for (int l = 0; l < ri.VT; ++l) {
                const auto& o = ri.loff[s][l];
                ids[l] = (p * ci + o[0]) + M * (p * cj + o[1]) + (d == 3 ? M * M * (p * ck + o[2]) : 0);
            }
            for (int i = 0; i < ri.VT; ++i)
                for (int j = 0; j < ri.VT; ++j) keys.push_back((uint64_t)ids[i] * nd + (uint64_t)ids[j]);
        }
    }
    std::sort(keys.begin(), keys.end());
    return (int64_t)(std::unique(keys.begin(), keys.end()) - keys.begin());
}

extern "C" int dogip_csr_nnz(int d, int64_t N, int p, int64_t* nnz) {
    if (d != 2 && d != 3) return fail(DOGIP_E_INVALID_DIM, "d must be 2 or 3");
    if (p < 1 || p > 8 || (d == 3 && p > 6)) return fail(DOGIP_E_UNSUPPORTED_ORDER, "p must be in 1..8 (2D), 1..6 (3D)");
    if (N < 1 || !nnz) return fail(DOGIP_E_INVALID_SIZE, "N must be >= 1");
    if (N <= d + 3) { *nnz = csr_nnz_direct(d, N, p); return DOGIP_OK; }
    // nnz(N) is an exact polynomial of degree d for N >= 2: Lagrange through N = 2..d+3,
    // checked on the extra point d+3 from the first d+1 samples
    const int npt = d + 2;
    std::vector<int64_t> xs(npt), ys(npt);
    for (int i = 0; i < npt; ++i) { xs[i] = 2 + i; ys[i] = csr_nnz_direct(d, xs[i], p); }
    auto lagrange = [&](int64_t x, int m) {
        Rat acc(0);
        for (int i = 0; i < m; ++i) {
            Rat t(ys[i]);
            for (int j = 0; j < m; ++j)
                if (j != i) t = t * Rat(x - xs[j], xs[i] - xs[j]);
            acc = acc + t;
        }
        return acc;
    };
    if (lagrange(xs[npt - 1], npt - 1) != Rat(ys[npt - 1]))
        return fail(DOGIP_E_INVALID_ARG, "pattern count is not polynomial in N");
    const Rat v = lagrange(N, npt);
    if (v.d != 1) return fail(DOGIP_E_INVALID_ARG, "non-integer pattern count");
    *nnz = v.n;
    return DOGIP_OK;
}

extern "C" int dogip_quadrature(int d, int n1d, double* pts, double* wts, int64_t cap) {
    if (d != 2 && d != 3) return fail(DOGIP_E_INVALID_DIM, "d must be 2 or 3");
    if (n1d < 1 || n1d > 64) return fail(DOGIP_E_INVALID_SIZE, "n1d must be in 1..64");
    std::vector<double> P, W;
    simplex_rule(d, n1d, P, W);
    const int64_t n = (int64_t)W.size();
    if (pts || wts) {
        if (cap < n) return fail(DOGIP_E_INVALID_SIZE, "capacity too small");
        if (pts) std::memcpy(pts, P.data(), sizeof(double) * P.size());
        if (wts) std::memcpy(wts, W.data(), sizeof(double) * W.size());
    }
    return (int)n;
}

// K-order (tile, lane) -> canonical local element index; -1 for padding lanes
static int64_t canonical_elem(const SlabGeo& g, int64_t tile, int lane) {
    const TileCoord tc = tile_coord(g, tile);
    const int ci = tc.ci0 + lane;
    if (ci >= g.Nx) return -1;
    const int64_t cell = g.d == 2 ? ci + (int64_t)g.Nx * tc.cj : ci + (int64_t)g.Nx * (tc.cj + (int64_t)g.Ny * tc.ck);
    return cell * g.ns + tc.s;
}

extern "C" int dogip_export_weights(dogip_op op, double* host, int64_t cap) {
    if (!op || !host) return fail(DOGIP_E_INVALID_ARG, "null argument");
    if (op->store == DOGIP_STORE_QP) return fail(DOGIP_E_INVALID_ARG, "DOGIP_STORE_QP stores no weights");
    dogip_mesh_info_t info;
    dogip_mesh_info(op->m, &info);
    const int d = op->m->d, WT = op->ref.WT, TR = op->ref.tile_rows;
    const int NC = op->form == DOGIP_WP ? 1 : d * (d + 1) / 2;
    if (cap < info.n_elem_local * WT * NC) return fail(DOGIP_E_INVALID_SIZE, "capacity too small");
    std::vector<double> w(op->w_doubles);
    DeviceGuard dg(op->m->device);
    CK(cudaMemcpy(w.data(), op->d_w, sizeof(double) * op->w_doubles, cudaMemcpyDeviceToHost));
    const SlabGeo& g = op->m->geo;
    std::vector<int> offw;
    if (op->store == DOGIP_STORE_GLOBAL) {
        offw.resize((size_t)g.ns * WT);
        CK(cudaMemcpy(offw.data(), op->d_offw, sizeof(int) * offw.size(), cudaMemcpyDeviceToHost));
    }
    for (int64_t t = 0; t < g.ntiles; ++t)
        for (int lane = 0; lane < TILE; ++lane) {
            const int64_t e = canonical_elem(g, t, lane);
            if (e < 0) continue;
            if (op->store == DOGIP_STORE_GLOBAL) {     // the global weights each element sees
                const TileCoord tc = tile_coord(g, t);
                const int64_t bw = g.rw * (int64_t)(2 * g.p) * (tc.cj + g.swy * tc.ck) + tc.ci0 + lane;
                for (int j = 0; j < WT; ++j) host[e * WT + j] = w[bw + offw[(size_t)tc.s * WT + j]];
                continue;
            }
            auto at = [&](int row) { return w[((size_t)t * TR + row) * TILE + lane]; };
            if (op->store == DOGIP_STORE_SYM) {
                // a_j = sum over the rows r of j's orbit of s_r c_{r,j} ahat_r  (the character
                // matrix of an orbit is orthogonal: X X^T = s I)
                for (int j = 0; j < WT; ++j) host[e * WT + j] = 0.0;
                for (int r = 0; r < WT; ++r) {
                    int sz = 0;
                    for (int k = 0; k < 4; ++k) sz += op->ref.symj[r][k] >= 0;
                    for (int k = 0; k < 4; ++k) {
                        const int j = op->ref.symj[r][k];
                        if (j >= 0) host[e * WT + j] += sz * op->ref.symc[r][k] * at(r);
                    }
                }
                continue;
            }
            for (int j = 0; j < WT; ++j)
                for (int c = 0; c < NC; ++c)
                    host[(e * WT + j) * NC + c] =
                        op->store == DOGIP_STORE_ISO ? at(op->ref.NG + op->ref.rowperm[j]) * at(c) : at(op->ref.rowperm[j] * NC + c);
        }
    return DOGIP_OK;
}

extern "C" int dogip_test_perturb_weight(dogip_op op, int64_t elem, int j, int c, double delta) {
    if (!op) return fail(DOGIP_E_INVALID_ARG, "null argument");
    if (op->store != DOGIP_STORE_FULL) return fail(DOGIP_E_INVALID_ARG, "perturbation hook: DOGIP_STORE_FULL only");
    const SlabGeo& g = op->m->geo;
    dogip_mesh_info_t info;
    dogip_mesh_info(op->m, &info);
    const int NC = op->ref.NC;
    if (elem < 0 || elem >= info.n_elem_local || j < 0 || j >= op->ref.WT || c < 0 || c >= NC)
        return fail(DOGIP_E_INVALID_SIZE, "perturbation hook: index out of range");
    // canonical e = ns * cell + s, cell = ci + Nx (cj + Ny ck) -> tile (s fastest, then x-block,
    // row, layer) and lane ci % 32, the inverse of canonical_elem
    const int64_t s = elem % g.ns, cell = elem / g.ns;
    const int64_t ci = cell % g.Nx, cj = (cell / g.Nx) % g.Ny, ck = cell / ((int64_t)g.Nx * g.Ny);
    const int64_t tile = s + g.ns * (ci / TILE + g.nxb * (cj + (int64_t)g.Ny * ck));
    const size_t idx = ((size_t)tile * op->ref.tile_rows + (size_t)(op->ref.rowperm[j] * NC + c)) * TILE + (size_t)(ci % TILE);
    DeviceGuard dg(op->m->device);
    double v = 0.0;
    CK(cudaMemcpy(&v, op->d_w + idx, sizeof(double), cudaMemcpyDeviceToHost));
    v += delta;
    CK(cudaMemcpy(op->d_w + idx, &v, sizeof(double), cudaMemcpyHostToDevice));
    return DOGIP_OK;
}

extern "C" int dogip_export_dofmap(dogip_mesh m, int64_t* host, int64_t cap) {
    if (!m || !host) return fail(DOGIP_E_INVALID_ARG, "null argument");
    dogip_mesh_info_t info;
    dogip_mesh_info(m, &info);
    const int VT = m->ref.VT;
    if (cap < info.n_elem_local * VT) return fail(DOGIP_E_INVALID_SIZE, "capacity too small");
    const SlabGeo& g = m->geo;
    for (int64_t t = 0; t < g.ntiles; ++t)
        for (int lane = 0; lane < TILE; ++lane) {
            const int64_t e = canonical_elem(g, t, lane);
            if (e < 0) continue;
            const TileCoord tc = tile_coord(g, t);
            const int64_t base = (int64_t)g.p * (tc.ci0 + lane + g.sy * tc.cj + g.sz * tc.ck);
            for (int l = 0; l < VT; ++l) host[e * VT + l] = base + m->tab.off[tc.s * MAX_VT + l];
        }
    return DOGIP_OK;
}
