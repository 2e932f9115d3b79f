"""Thin Python API over the C ABI (argument marshalling only; every step runs
in libdogip.so).  torch is used for device memory and streams only.

    mesh = Mesh(d=3, N=128, p=3)                    # dogip_mesh_setup
    op   = Operator(mesh, EL, coeff)                # dogip_weights
    y    = op.apply(u)                              # dogip_apply
    b    = op.load_vector(1.0, dirichlet=True)      # dogip_load_vector
    res  = op.cg(b, x, rtol=1e-10, dirichlet=True)  # dogip_cg
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import DOGIP_DIRICHLET_ZERO, DOGIP_EL, DOGIP_NO_EXCHANGE, DOGIP_WP, DogipError, check, load

__all__ = ["Mesh", "Operator", "LoopbackGroup", "CoeffSpec", "DOGIP_WP", "DOGIP_EL", "DogipError",
           "reference_table", "reference_nnz", "quadrature", "slab_range", "nccl_unique_id"]


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_lib.c_dp)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _tensor_ptr(t, n: int, device: Optional[int] = None) -> int:
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    if t.numel() != n:
        raise ValueError(f"expected {n} entries, got {t.numel()}")
    if device is not None and t.device.index != device:
        raise ValueError(f"tensor on cuda:{t.device.index}, mesh on cuda:{device}")
    if t.data_ptr() % 16:
        raise ValueError("vector must be 16-byte aligned (the C ABI reads fp64 pairs)")
    return t.data_ptr()


@dataclass
class CoeffSpec:
    """Coefficient model (include/dogip.h DOGIP_COEF_*)."""
    kind: int
    params: np.ndarray
    per_cell: Optional[np.ndarray] = None

    @classmethod
    def from_obj(cls, c) -> "CoeffSpec":
        return cls(int(c.kind), np.ascontiguousarray(c.params, dtype=np.float64),
                   None if c.per_cell is None else np.ascontiguousarray(c.per_cell, dtype=np.float64))


def kernel_launches() -> int:
    return int(load().dogip_kernel_launches())


def slab_range(N: int, rank: int, nranks: int):
    z0, z1 = C.c_int64(), C.c_int64()
    check(load().dogip_slab_range(N, rank, nranks, C.byref(z0), C.byref(z1)))
    return z0.value, z1.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(load().dogip_nccl_unique_id(buf))
    return buf.raw


def reference_table(d: int, p: int, form: int) -> np.ndarray:
    lib = load()
    n = check(lib.dogip_reference_table(d, p, form, None, 0), allow_positive=True)
    out = np.empty(n)
    check(lib.dogip_reference_table(d, p, form, _dptr(out), n), allow_positive=True)
    return out


def reference_nnz(d: int, p: int, form: int):
    a, b = C.c_int64(), C.c_int64()
    check(load().dogip_reference_nnz(d, p, form, C.byref(a), C.byref(b)))
    return a.value, b.value


def quadrature(d: int, n1d: int):
    lib = load()
    n = check(lib.dogip_quadrature(d, n1d, None, None, 0), allow_positive=True)
    pts, wts = np.empty((n, d)), np.empty(n)
    check(lib.dogip_quadrature(d, n1d, _dptr(pts), _dptr(wts), n), allow_positive=True)
    return pts, wts


class LoopbackGroup:
    """In-process communicator of `nranks` ranks on one device (DOGIP_COMM_LOOPBACK): each
    rank's mesh is driven from its own host thread; the library moves interface planes and
    CG scalars between the ranks with cudaMemcpyAsync (tests of the multi-rank path)."""

    def __init__(self, nranks: int, device: int = 0):
        self._lib = load()
        h = C.c_void_p()
        check(self._lib.dogip_loopback_create(int(nranks), int(device), C.byref(h)))
        self.handle, self.nranks, self.device = h, nranks, device

    def close(self):
        if getattr(self, "handle", None):
            check(self._lib.dogip_loopback_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Mesh:
    """Structured simplex mesh M_N + P_p DoF plan (+ slab partition, NCCL or loopback comm)."""

    def __init__(self, d: int, N: int, p: int, vertices: Optional[np.ndarray] = None, rank: int = 0,
                 nranks: int = 1, nccl_id: Optional[bytes] = None, device: int = 0,
                 loopback: Optional[LoopbackGroup] = None):
        lib = load()
        self._lib = lib
        self._verts = None if vertices is None else np.ascontiguousarray(vertices, dtype=np.float64)
        h = C.c_void_p()
        if loopback is not None:
            if nccl_id is not None:
                raise ValueError("pass either nccl_id or loopback")
            self._group = loopback          # the group must outlive the mesh
            check(lib.dogip_mesh_setup_ex(d, N, p, _dptr(self._verts), rank, nranks, _lib.DOGIP_COMM_LOOPBACK,
                                          loopback.handle, device, C.byref(h)))
        else:
            idbuf = None if nccl_id is None else C.create_string_buffer(nccl_id, 128)
            check(lib.dogip_mesh_setup(d, N, p, _dptr(self._verts), rank, nranks, idbuf, device, C.byref(h)))
        self.handle = h
        self.device = device
        info = _lib.MeshInfo()
        check(lib.dogip_mesh_info(h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _lib.MeshInfo._fields_}
        self.ndof = self.info["ndof_local"]

    def dofmap(self) -> np.ndarray:
        vt = {2: {1: 3, 2: 6, 3: 10, 4: 15}, 3: {1: 4, 2: 10, 3: 20, 4: 35}}[self.info["d"]][self.info["p"]]
        out = np.empty((self.info["n_elem_local"], vt), dtype=np.int64)
        check(self._lib.dogip_export_dofmap(self.handle, out.ctypes.data_as(_lib.c_i64p), out.size))
        return out

    def close(self):
        if getattr(self, "handle", None):
            self._lib.dogip_mesh_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """A^DoGIP of one form on a mesh (dogip_weights) + apply / load vector / CG."""

    def __init__(self, mesh: Mesh, form: int, coeff, quad_n1d: int = 0, stream=None, storage: int = 0):
        self.mesh = mesh
        self._lib = mesh._lib
        self.coeff = coeff if isinstance(coeff, CoeffSpec) else CoeffSpec.from_obj(coeff)
        cs = _lib.Coeff(self.coeff.kind, _dptr(self.coeff.params), self.coeff.params.size,
                        _dptr(self.coeff.per_cell))
        h = C.c_void_p()
        check(self._lib.dogip_weights_ex(mesh.handle, form, C.byref(cs), quad_n1d, storage,
                                         C.c_void_p(_stream_ptr(stream)), C.byref(h)))
        self.handle = h
        oi = _lib.OpInfo()
        check(self._lib.dogip_op_info(h, C.byref(oi)))
        self.info = {f: getattr(oi, f) for f, _ in _lib.OpInfo._fields_}
        self.ndof = mesh.ndof
        self.form = form

    # -- apply ---------------------------------------------------------------
    def _device(self):
        """The mesh's CUDA device made current for a call (the C ABI launches on the
        caller's current device / stream)."""
        import torch
        return torch.cuda.device(self.mesh.device)

    def apply(self, u, y=None, dirichlet: bool = False, exchange: bool = True, stream=None):
        import torch
        if y is None:
            y = torch.empty_like(u)
        flags = (DOGIP_DIRICHLET_ZERO if dirichlet else 0) | (0 if exchange else DOGIP_NO_EXCHANGE)
        with self._device():
            check(self._lib.dogip_apply(self.handle, C.c_void_p(_tensor_ptr(u, self.ndof, self.mesh.device)),
                                        C.c_void_p(_tensor_ptr(y, self.ndof, self.mesh.device)), flags,
                                        C.c_void_p(_stream_ptr(stream))))
        return y

    def apply_host(self, u: np.ndarray, y: Optional[np.ndarray] = None, dirichlet: bool = False, stream=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.size != self.ndof:
            raise ValueError("size mismatch")
        if y is None:
            y = np.empty_like(u)
        if not (isinstance(y, np.ndarray) and y.dtype == np.float64 and y.flags.c_contiguous and y.size == self.ndof):
            raise TypeError(f"y must be a contiguous float64 array of {self.ndof} entries")
        flags = DOGIP_DIRICHLET_ZERO if dirichlet else 0
        with self._device():
            check(self._lib.dogip_apply_host(self.handle, u.ctypes.data, y.ctypes.data, flags,
                                             C.c_void_p(_stream_ptr(stream))))
        return y

    def apply_host_ptr(self, u_ptr: int, y_ptr: int, dirichlet: bool = False, stream=None):
        """Host-buffer apply on raw (pinned) host pointers."""
        flags = DOGIP_DIRICHLET_ZERO if dirichlet else 0
        with self._device():
            check(self._lib.dogip_apply_host(self.handle, C.c_void_p(u_ptr), C.c_void_p(y_ptr), flags,
                                             C.c_void_p(_stream_ptr(stream))))

    def load_vector(self, f: float = 1.0, dirichlet: bool = False, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty(self.ndof, dtype=torch.float64, device=f"cuda:{self.mesh.device}")
        flags = DOGIP_DIRICHLET_ZERO if dirichlet else 0
        with self._device():
            check(self._lib.dogip_load_vector(self.handle, float(f),
                                              C.c_void_p(_tensor_ptr(out, self.ndof, self.mesh.device)), flags,
                                              C.c_void_p(_stream_ptr(stream))))
        return out

    def cg(self, b, x, rtol: float = 1e-10, maxit: int = 10000, dirichlet: bool = False, stream=None,
           resume: bool = False) -> dict:
        """maxit < 0: exactly |maxit| iterations without convergence checks
        (benchmarking); resume: continue the previous call's iteration."""
        res = _lib.CgResult()
        flags = (DOGIP_DIRICHLET_ZERO if dirichlet else 0) | (_lib.DOGIP_CG_RESUME if resume else 0)
        with self._device():
            rc = self._lib.dogip_cg(self.handle, C.c_void_p(_tensor_ptr(b, self.ndof, self.mesh.device)),
                                    C.c_void_p(_tensor_ptr(x, self.ndof, self.mesh.device)), float(rtol), int(maxit),
                                    flags, C.c_void_p(_stream_ptr(stream)), C.byref(res))
        if rc < 0 and rc != -9:
            check(rc)
        return {"iters": res.iters, "status": _lib.STATUS.get(res.status, res.status),
                "rel_res": res.rel_res, "seconds": res.seconds, "apply_seconds": res.apply_seconds}

    def export_weights(self) -> np.ndarray:
        i = self.info
        out = np.empty((self.mesh.info["n_elem_local"], i["W_T"], i["n_c"]))
        check(self._lib.dogip_export_weights(self.handle, _dptr(out), out.size))
        return out

    def _test_perturb_weight(self, elem: int, j: int, c: int, delta: float):
        """Test hook (negative control): A_{T,j}[c] += delta on the device (FULL storage)."""
        check(self._lib.dogip_test_perturb_weight(self.handle, int(elem), int(j), int(c), float(delta)))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.dogip_op_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
