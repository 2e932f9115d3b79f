/*
 * dogip.h -- C ABI of the B200-native DoGIP apply + CG library (libdogip.so).
 *
 * DoGIP = "double-grid integration with interpolation-projection"
 * (arXiv 1710.09913, /root/reference/PAPER.md, cited as P:<line>).  The
 * library applies the FEM system matrix of two forms on simplicial Lagrange
 * P_p elements without assembling it:
 *
 *     y = A u = sum_T P_T^T  Bhat^T A_T^DoGIP Bhat  P_T u      (Algorithm 1)
 *
 *   WP  weighted projection  a(u,v) = int m u v               (eq:bilf_gp)
 *       A_T^DoGIP = diag_j int_T m phi^W_j, W = P_2p           (Theorem 2)
 *   EL  scalar elliptic      a(u,v) = int M grad u . grad v   (eq:bilf_se)
 *       A_T,j = Rinv_T (int_T M phi^W_j) Rinv_T^T, W = P_2p-2  (Theorem 4)
 *
 * and solves A x = b with plain conjugate gradients.
 *
 * Conventions (all calls):
 *  - fp64 everywhere.  Return value: 0 = OK, > 0 non-fatal status, < 0 error;
 *    the message of the last error of the calling thread is dogip_last_error().
 *  - Vectors passed to apply/cg/load_vector are CALLER-OWNED DEVICE pointers
 *    (e.g. torch CUDA tensors), contiguous, 16-byte aligned (the vector kernels
 *    move fp64 pairs; a misaligned pointer returns E_INVALID_ARG), of length
 *    ndof_local; the library never frees them.  Handles are library-owned
 *    (destroy with *_destroy).  Setup / destroy / synchronous calls restore the
 *    caller's current CUDA device on return.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Work is asynchronous on that stream, except dogip_cg and the *_host
 *    entry points, which synchronise it.  dogip_apply / dogip_load_vector /
 *    dogip_cg launch on the caller's current CUDA device, which must be the
 *    mesh's `device` (the Python binding makes it current around each call).
 *  - Concurrency: an op is read-only after dogip_weights, so single-rank
 *    dogip_apply calls on one op may run concurrently on different streams
 *    with distinct y.  Calls that use library-owned scratch are
 *    NOT re-entrant per handle: dogip_apply_host and dogip_cg (per op), and
 *    any call that exchanges interface planes (mesh with a communicator) --
 *    serialise those on one stream / thread per handle.
 *  - Multi-GPU (nranks > 1): one process per GPU; every call is collective and
 *    must be made by all ranks in the same order.  The mesh is split into
 *    slabs of whole cube layers along the LAST axis (z in 3D, y in 2D); rank r
 *    holds the DoF planes [p*z0, p*z1] of its slab, both interface planes
 *    included, which is a contiguous range of the global DoF vector.
 *
 * Mesh, numbering and layout (readings L3-L6):
 *  - unit square / cube, N cells per axis; 2D cell (i,j) -> triangles
 *    (v00,v10,v11), (v00,v11,v01); 3D cell -> 6 Kuhn tetrahedra, one per
 *    permutation of the axes in lexicographic order; canonical element id
 *    e = d! * cell + s, cell = i + N j (+ N^2 k).
 *  - vertices and DoFs lexicographic with x fastest: id = i + M j (+ M^2 k),
 *    M = N+1 (vertices) or p*N+1 (DoFs).
 *  - local DoF order: barycentric multi-index (alpha_1..alpha_d), alpha_1
 *    fastest, alpha_0 = p - sum.
 */
#ifndef DOGIP_H
#define DOGIP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- forms (P:184-209 WP, P:305-339 EL) -------------------------------- */
#define DOGIP_WP 0
#define DOGIP_EL 1

/* ---- coefficient models (BASELINE.json configs) ------------------------ */
#define DOGIP_COEF_CONST          0  /* m = params[0]; EL: M = m I                         */
#define DOGIP_COEF_PER_CELL       1  /* m = per_cell[cell], N^d host values, isotropic      */
#define DOGIP_COEF_SINCOS2D       2  /* m = params[0] + params[1] sin(2 pi x) cos(2 pi y)   */
#define DOGIP_COEF_TANH_RADIAL    3  /* m = a0 + a1 tanh(k (|x - c| - r0)),
                                        params = {a0, a1, k, r0, c_1..c_d}                  */
#define DOGIP_COEF_ANISO_FOURIER  4  /* 3D only: M = R(x) diag(e) R(x)^T, R = Rodrigues(w(x)),
                                        w_i(x) = sum_m c[m,i] cos(2 pi kappa_m . x + phi[m,i]);
                                        params = {e_1,e_2,e_3, n, kappa(n*3), phi(n*3), c(n*3)} */
#define DOGIP_COEF_CONST_TENSOR   5  /* M = params[0..d*d) row-major, symmetric (EL only)   */

/* ---- weight storage (dogip_weights_ex) ---------------------------------- */
#define DOGIP_STORE_FULL  0  /* WP: a_{T,j}; EL: symmetric A_{T,j} (d(d+1)/2 per node).
                                The device layout is internal (3D WP p >= 3: node rows in the
                                orbit order of DOGIP_STORE_SYM, applied through the same
                                block-diagonal body); dogip_export_weights returns canonical order */
#define DOGIP_STORE_ISO   1  /* EL with isotropic M = m I (Corollary, element-wise):
                                A_{T,j} = a_{T,j} G_T, a_{T,j} = int_T m phi^W_j, G_T = Rinv Rinv^T;
                                stores W_T + d(d+1)/2 doubles per element instead of W_T d(d+1)/2 */
#define DOGIP_STORE_GLOBAL 2 /* WP only (Theorem 1): one global diagonal over the
                                double-grid space W = C_{N,2p}, A_ii = int_Omega m phi^W_i, stored
                                as a W-lattice vector ((2pN+1)^d values) holding A_ii / mult_i
                                (mult_i = elements sharing W node i, each visits it once) and
                                gathered per element; kept class-major along x (x = 2p c + k at
                                k (N+1) + c: rows of 2p(N+1) doubles) so a tile's lanes gather
                                consecutive values; multi-rank needs a communicator */
#define DOGIP_STORE_SYM    5 /* WP only: the same weights in symmetry-adapted form -- per orbit P of
                                the double-grid nodes under the barycentric involutions
                                G = <(0 1), (2 3)> (3D) / <(0 1)> (2D), ahat_psi(P) = (1/|G|) sum_g
                                psi(g) a_{g j0}; the apply runs Bhat block-diagonally by character
                                (3D P4: 784 instead of 1729 nonzeros); same bytes; in 3D p >= 3
                                DOGIP_STORE_FULL runs the same body on the plain values (~10 %
                                more FP64 operations than this storage) */
#define DOGIP_STORE_QP     4 /* no DoGIP weights: the quadrature-point matrix-free comparator
                                ("alternative approaches") -- geometry, coefficient and the
                                basis contractions at the n_q points of the contract rule (L10) are
                                evaluated on the fly every apply; same operator A up to rounding.
                                Stores only the basis tables and the coefficient data; does not
                                validate coefficient positivity or element orientation */

/* ---- status codes ------------------------------------------------------- */
#define DOGIP_OK                     0
#define DOGIP_NOT_CONVERGED          1  /* CG hit maxit (x holds the last iterate)           */
#define DOGIP_E_INVALID_DIM         -1  /* d not in {2,3}                                    */
#define DOGIP_E_INVALID_SIZE        -2  /* N < 1, N < nranks, bad rank, bad buffer capacity  */
#define DOGIP_E_UNSUPPORTED_ORDER   -3  /* p not in 1..4                                     */
#define DOGIP_E_DEGENERATE_ELEMENT  -4  /* det R_T == 0 (or orientation flipped by jitter)  */
#define DOGIP_E_BAD_COEFF           -5  /* unknown kind, wrong parameter count, tensor for WP,
                                           non-symmetric tensor, non-positive samples        */
#define DOGIP_E_OOM                 -6  /* device allocation failed                          */
#define DOGIP_E_CUDA                -7  /* CUDA runtime error (message has the detail)       */
#define DOGIP_E_NCCL                -8  /* NCCL missing or failed                            */
#define DOGIP_E_BREAKDOWN           -9  /* CG: p^T A p <= 0 (operator not SPD)               */
#define DOGIP_E_INVALID_ARG        -10  /* NULL handle / pointer, bad form or flags          */

/* ---- apply / cg / load-vector flags ------------------------------------ */
#define DOGIP_DIRICHLET_ZERO  1u  /* symmetric elimination of all boundary DoFs (reading L14):
                                     y_i = (A (D u))_i on interior DoFs, y_i = u_i on the
                                     boundary; load vector zeroed on the boundary           */
#define DOGIP_NO_EXCHANGE     2u  /* multi-rank: return this rank's partial sums on the
                                     interface planes (no NCCL exchange) -- tests only      */
#define DOGIP_CG_RESUME       4u  /* dogip_cg: continue from the state (x, r, p, r.r) the
                                     previous dogip_cg call on this op left, skipping the
                                     initial residual -- times exactly |maxit| iterations  */

typedef struct dogip_mesh_s* dogip_mesh;
typedef struct dogip_op_s*   dogip_op;
typedef struct dogip_loopback_s* dogip_loopback;

/* ---- communicator kinds (dogip_mesh_setup_ex) ---------------------------- */
#define DOGIP_COMM_NONE      0  /* single rank, or partial sums only (DOGIP_NO_EXCHANGE)     */
#define DOGIP_COMM_NCCL      1  /* comm_arg = 128-byte ncclUniqueId: one process per GPU     */
#define DOGIP_COMM_LOOPBACK  2  /* comm_arg = dogip_loopback: every rank in THIS process, one
                                   host thread per rank, same device; planes and scalars are
                                   moved with cudaMemcpyAsync, host threads rendezvous per
                                   collective (tests of the multi-rank path on one GPU)     */

typedef struct {
    int      d, p, rank, nranks;
    int64_t  N;                 /* cells per axis (global)                                   */
    int64_t  z0, z1;            /* this rank's cube layers [z0, z1) along the last axis      */
    int64_t  n_elem_local;      /* d! N^(d-1) (z1 - z0)                                      */
    int64_t  n_elem_global;     /* d! N^d                                           */
    int64_t  ndof_local;        /* (pN+1)^(d-1) (p (z1-z0) + 1)                               */
    int64_t  ndof_global;       /* (pN+1)^d                                                  */
    int64_t  dof_offset;        /* global id of local DoF 0 = p z0 (pN+1)^(d-1)               */
    int64_t  plane_size;        /* (pN+1)^(d-1) DoFs per interface plane                     */
    int64_t  owned_begin, owned_end; /* local DoF range this rank owns for reductions:
                                     the upper interface plane belongs to the rank above     */
} dogip_mesh_info_t;

typedef struct {
    int         kind;           /* DOGIP_COEF_*                                              */
    const double* params;       /* host array, see the kinds above                           */
    int64_t     nparams;
    const double* per_cell;     /* host array of N^d values (GLOBAL cell numbering) or NULL  */
} dogip_coeff;

typedef struct {
    int     form, d, p;
    int     V_T;                /* C(p+d, d) local primal DoFs                               */
    int     W_T;                /* C(2p+d, d) (WP) or C(2p-2+d, d) (EL) double-grid nodes    */
    int     n_c;                /* stored weights per node: 1 (WP), d(d+1)/2 (EL, reading L11)*/
    int     quad_n1d;           /* points per direction of the weight rule (reading L10)     */
    int     storage;            /* DOGIP_STORE_*                                             */
    int     stream_doubles_per_elem; /* doubles the apply streams per element               */
    int     flops_per_elem;     /* fp64 flops of the generated element body                  */
    int64_t n_tiles;            /* 32-element tiles of the apply kernel                      */
    int64_t weight_bytes;       /* device bytes of the streamed weights (incl. tile padding) */
    double  weights_ms;         /* device time of the one-time weights kernels               */
} dogip_op_info_t;

typedef struct {
    int     iters;              /* CG iterations performed                                   */
    int     status;             /* DOGIP_OK, DOGIP_NOT_CONVERGED or DOGIP_E_BREAKDOWN        */
    double  rel_res;            /* ||r_k||_2 / ||b||_2 of the recursively updated residual  */
    double  seconds;            /* device time of the iteration loop                         */
    double  apply_seconds;      /* device time spent in the applies (maxit < 0 only, else 0) */
} dogip_cg_result;

/* Version of the ABI (major*100 + minor). */
int dogip_version(void);

/* Message of the last error raised on the calling thread ("" if none). */
const char* dogip_last_error(void);

/*
 * dogip_mesh_setup -- structured mesh M_N, P_p DoF plan and
 * slab partition; with nccl_id also the NCCL communicator.
 *   d, N, p     dimension (2|3), cells per axis (>= 1, >= nranks), order (1..4)
 *   vertices    host array ((N+1)^d, d) of vertex coordinates in vertex order,
 *               or NULL for the lattice {0,1/N,..,1}^d (copied; caller keeps it)
 *   rank/nranks this process and the world size (0/1 for one GPU)
 *   nccl_id     128-byte ncclUniqueId created by rank 0 and broadcast by the
 *               caller (torch.distributed); NULL when the caller only wants partial
 *               sums (DOGIP_NO_EXCHANGE) or runs one rank without NCCL.  Any non-NULL
 *               id (also with nranks = 1) creates the communicator, and every apply /
 *               load vector / CG then runs the exchange and all-reduce path (a 1-rank
 *               communicator makes them identities: a single-GPU check of the plumbing)
 *   device      CUDA device ordinal used by every later call on this mesh; -1 builds a
 *               host-only mesh (info / dofmap introspection, no device work)
 * Errors: E_INVALID_DIM, E_INVALID_SIZE, E_UNSUPPORTED_ORDER,
 *         E_DEGENERATE_ELEMENT (a Kuhn/right simplex lost its orientation),
 *         E_NCCL, E_CUDA, E_OOM.
 */
int dogip_mesh_setup(int d, int64_t N, int p, const double* vertices, int rank, int nranks,
                     const void* nccl_id, int device, dogip_mesh* out);

/*
 * dogip_mesh_setup_ex -- dogip_mesh_setup with an explicit communicator kind
 * (DOGIP_COMM_*).  dogip_mesh_setup(..., nccl_id, ...) is dogip_mesh_setup_ex with
 * DOGIP_COMM_NCCL when nccl_id != NULL, else DOGIP_COMM_NONE.  With DOGIP_COMM_LOOPBACK
 * every later collective call (apply / load vector / CG / GLOBAL weights) of each rank
 * must be made from that rank's own host thread, concurrently with the other ranks.
 * Errors: as dogip_mesh_setup; E_INVALID_ARG (unknown kind, missing comm_arg, loopback
 * group of another device or size).
 */
int dogip_mesh_setup_ex(int d, int64_t N, int p, const double* vertices, int rank, int nranks,
                        int comm_kind, const void* comm_arg, int device, dogip_mesh* out);

/* In-process loopback group of nranks ranks on `device` (DOGIP_COMM_LOOPBACK): serves ONE
 * mesh per rank (the ranks' collectives are matched by call order).  Destroy after every
 * mesh using it (else E_INVALID_ARG). */
int dogip_loopback_create(int nranks, int device, dogip_loopback* out);
int dogip_loopback_destroy(dogip_loopback group);

int dogip_mesh_info(dogip_mesh mesh, dogip_mesh_info_t* out);

/* Rank 0 creates the 128-byte ncclUniqueId passed to dogip_mesh_setup by
 * every rank (the caller broadcasts it, e.g. with torch.distributed). */
int dogip_nccl_unique_id(void* out128);

/* Host-only slab partition rule (no device work): cube layers of `rank`. */
int dogip_slab_range(int64_t N, int rank, int nranks, int64_t* z0, int64_t* z1);

/*
 * dogip_weights -- one-time kernels computing A_T^DoGIP for every local element:
 *   WP  a_{T,j}  = |det R_T| sum_q w_q m(F_T xq) phi^W_j(xq)
 *   EL  A_{T,j}  = Rinv_T ( |det R_T| sum_q w_q M(F_T xq) phi^W_j(xq) ) Rinv_T^T
 * with the collapsed Gauss-Jacobi rule of quad_n1d points per direction
 * (0 = the contract default p+3, reading L10).  Weights are stored in the
 * apply kernel's tile-major layout.  Synchronises `stream`.
 * Errors: E_INVALID_ARG (form), E_BAD_COEFF, E_OOM, E_CUDA.
 */
int dogip_weights(dogip_mesh mesh, int form, const dogip_coeff* coeff, int quad_n1d,
                  void* stream, dogip_op* out);

/* dogip_weights with an explicit storage variant (DOGIP_STORE_*).  DOGIP_STORE_ISO
 * needs form = DOGIP_EL (else E_INVALID_ARG) and an isotropic coefficient kind
 * (else E_BAD_COEFF); DOGIP_STORE_GLOBAL and _SYM need form = DOGIP_WP (else
 * E_INVALID_ARG); DOGIP_STORE_QP takes both forms and stores no weights.  The apply
 * result is the same operator up to rounding for every storage.
 * dogip_export_weights returns a_{T,j} / A_{T,j} in canonical order for FULL, ISO
 * and SYM (converted back from the stored layout), per element the stored values
 * of its W nodes, A_{l^W_T(j), l^W_T(j)} / mult_{l^W_T(j)}, for GLOBAL, and
 * E_INVALID_ARG for QP. */
int dogip_weights_ex(dogip_mesh mesh, int form, const dogip_coeff* coeff, int quad_n1d, int storage,
                     void* stream, dogip_op* out);

int dogip_op_info(dogip_op op, dogip_op_info_t* out);

/*
 * dogip_apply -- y = A u on this rank's DoFs (Algorithm 1, with the
 * transpose of reading L8).  u: device, ndof_local, its interface planes must be
 * consistent across ranks; y: device, ndof_local, overwritten; with nranks > 1
 * y's interface planes are summed over both owners on return (NCCL exchange
 * overlapped with interior elements) unless DOGIP_NO_EXCHANGE.  u and y must
 * not alias.  Asynchronous on `stream`.  Errors: E_INVALID_ARG, E_CUDA, E_NCCL
 * (an asynchronous communicator failure of an earlier call is reported here and the
 * communicator aborted).
 */
int dogip_apply(dogip_op op, const double* u, double* y, unsigned flags, void* stream);

/*
 * dogip_apply_host -- the same apply with HOST buffers u_host, y_host (ndof_local
 * doubles each, caller-owned; pinned memory is needed for the copies to overlap).
 * Single rank: pipelined over up to 24 chunks of cube layers along the slab axis --
 * copy-in of the next chunk's u planes, the apply kernel of this chunk's elements and
 * copy-out of the y planes it completed run concurrently on three streams (library-
 * owned device scratch and copy streams, ordered after prior work on `stream`).
 * Several ranks with exchange: copy in, dogip_apply, copy out.  Synchronises.
 * Errors: E_INVALID_ARG (null buffer, unknown flags), E_OOM, E_CUDA, E_NCCL.
 */
int dogip_apply_host(dogip_op op, const double* u_host, double* y_host, unsigned flags,
                     void* stream);

/*
 * dogip_load_vector -- b_i = int f phi_i for constant f (eq:linsys_gp P:207,
 * eq:linsys_se P:337), zero on boundary DoFs with DOGIP_DIRICHLET_ZERO.
 * b: device, ndof_local; interface planes are summed across ranks.
 */
int dogip_load_vector(dogip_op op, double f, double* b, unsigned flags, void* stream);

/*
 * dogip_cg -- unpreconditioned Hestenes-Stiefel CG (reading L15) on A (or its
 * Dirichlet-eliminated version with DOGIP_DIRICHLET_ZERO): x0 = caller's x,
 * stops when ||r_k||_2 <= rtol ||b||_2 (recursive residual) or after maxit
 * iterations (maxit < 0: run exactly -maxit iterations, no convergence test --
 * benchmarking).  b, x: device, ndof_local.  Dots run over owned DoFs and are
 * all-reduced.  Synchronises `stream`.  Returns DOGIP_OK, DOGIP_NOT_CONVERGED
 * or DOGIP_E_BREAKDOWN (also in res->status; on breakdown x holds the last iterate).
 * The stopping test runs on the device after every iteration (no host round trip
 * per iteration).  Single rank, maxit > 0: the iterations run as one CUDA graph
 * (conditional WHILE node around one iteration; built once per (x, flags, rtol,
 * maxit, stream) and cached in the op, outside the timed res->seconds).  Otherwise
 * (several ranks, or DOGIP_CG_NO_GRAPH=1) batches of DOGIP_CG_BATCH (default 32)
 * iterations are enqueued at once and the host reads the device's done flag once
 * per batch; iterations enqueued after the stop are no-ops (the apply kernel returns
 * at once).  With an NCCL communicator and DOGIP_CG_GRAPH_MR=1 a batch, NCCL calls
 * included, is captured once as a CUDA graph and replayed.  With a communicator every wait polls its asynchronous error state: a
 * dead peer or no progress within DOGIP_COMM_TIMEOUT_S seconds (default 600) aborts
 * the communicator and returns E_NCCL.
 */
int dogip_cg(dogip_op op, const double* b, double* x, double rtol, int maxit, unsigned flags,
             void* stream, dogip_cg_result* res);

/* Number of CUDA kernels this library has launched in this process (all
 * devices); the difference around a timed region is its kernel count. */
int64_t dogip_kernel_launches(void);

/* ---- introspection (tests; host only unless stated) --------------------- */

/* Exact reference table rounded to fp64: WP Bhat (W_T x V_T), EL Bhat
 * (d x W_T x V_T).  cap = capacity in doubles.  Returns the element count. */
int dogip_reference_table(int d, int p, int form, double* out, int64_t cap);

/* nnz and nnz_{+-1} of the reference table (eq:comp_eff; reading L12). */
int dogip_reference_nnz(int d, int p, int form, int64_t* nnz, int64_t* nnz_pm1);

/* Structural nonzeros of the assembled CSR matrix A of C_{N,p} on M_N (pairs of
 * DoFs sharing an element, the full pattern), exact: counted for small N and
 * extended through the exact degree-d polynomial in N it follows.  With the
 * paper's memory model mem A = 2 nnz + nrows this reproduces the `mem A`
 * column of Tables 3/4.  p <= 8 (2D), <= 6 (3D).  Host only. */
int dogip_csr_nnz(int d, int64_t N, int p, int64_t* nnz);

/* The collapsed Gauss-Jacobi rule: pts (n1d^d x d), wts (n1d^d).  Returns n1d^d. */
int dogip_quadrature(int d, int n1d, double* pts, double* wts, int64_t cap);

/* Weights of this rank in canonical layout [n_elem_local][W_T][n_c] (EL:
 * upper triangle row-major: 2D a11 a12 a22, 3D a11 a12 a13 a22 a23 a33), local
 * canonical element order e = d! (cell_local) + s.  Copies device -> host. */
int dogip_export_weights(dogip_op op, double* host_out, int64_t cap);

/* l_T of this rank: (n_elem_local, V_T) LOCAL DoF ids, canonical element order. */
int dogip_export_dofmap(dogip_mesh mesh, int64_t* host_out, int64_t cap);

/* TEST HOOK (negative control of the parity tests, not for production): adds `delta`
 * to the stored weight A_{T,j} component c (canonical order of dogip_export_weights) of
 * local element `elem`, in place on the device.  DOGIP_STORE_FULL only (else
 * E_INVALID_ARG); E_INVALID_SIZE for an index out of range.  Synchronous. */
int dogip_test_perturb_weight(dogip_op op, int64_t elem, int j, int c, double delta);

void dogip_op_destroy(dogip_op op);
void dogip_mesh_destroy(dogip_mesh mesh);

#ifdef __cplusplus
}
#endif
#endif /* DOGIP_H */
