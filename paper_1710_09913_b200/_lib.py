"""ctypes binding of libdogip.so (include/dogip.h) -- argument marshalling only.

The library is built in-tree by paper_1710_09913_b200/build.py.  There is no
fallback: if the shared library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdogip.so")

DOGIP_WP, DOGIP_EL = 0, 1
DOGIP_STORE_FULL, DOGIP_STORE_ISO, DOGIP_STORE_GLOBAL, DOGIP_STORE_QP, DOGIP_STORE_SYM = 0, 1, 2, 4, 5
DOGIP_DIRICHLET_ZERO, DOGIP_NO_EXCHANGE, DOGIP_CG_RESUME = 1, 2, 4
DOGIP_COMM_NONE, DOGIP_COMM_NCCL, DOGIP_COMM_LOOPBACK = 0, 1, 2
STATUS = {0: "OK", 1: "NOT_CONVERGED", -1: "E_INVALID_DIM", -2: "E_INVALID_SIZE",
          -3: "E_UNSUPPORTED_ORDER", -4: "E_DEGENERATE_ELEMENT", -5: "E_BAD_COEFF", -6: "E_OOM",
          -7: "E_CUDA", -8: "E_NCCL", -9: "E_BREAKDOWN", -10: "E_INVALID_ARG"}

c_i64p = C.POINTER(C.c_int64)
c_dp = C.POINTER(C.c_double)


class MeshInfo(C.Structure):
    _fields_ = [("d", C.c_int), ("p", C.c_int), ("rank", C.c_int), ("nranks", C.c_int),
                ("N", C.c_int64), ("z0", C.c_int64), ("z1", C.c_int64),
                ("n_elem_local", C.c_int64), ("n_elem_global", C.c_int64),
                ("ndof_local", C.c_int64), ("ndof_global", C.c_int64), ("dof_offset", C.c_int64),
                ("plane_size", C.c_int64), ("owned_begin", C.c_int64), ("owned_end", C.c_int64)]


class Coeff(C.Structure):
    _fields_ = [("kind", C.c_int), ("params", c_dp), ("nparams", C.c_int64), ("per_cell", c_dp)]


class OpInfo(C.Structure):
    _fields_ = [("form", C.c_int), ("d", C.c_int), ("p", C.c_int), ("V_T", C.c_int), ("W_T", C.c_int),
                ("n_c", C.c_int), ("quad_n1d", C.c_int), ("storage", C.c_int),
                ("stream_doubles_per_elem", C.c_int), ("flops_per_elem", C.c_int), ("n_tiles", C.c_int64),
                ("weight_bytes", C.c_int64), ("weights_ms", C.c_double)]


class CgResult(C.Structure):
    _fields_ = [("iters", C.c_int), ("status", C.c_int), ("rel_res", C.c_double), ("seconds", C.c_double),
                ("apply_seconds", C.c_double)]


# (name, restype, argtypes) for every symbol of include/dogip.h
SIGNATURES = [
    ("dogip_version", C.c_int, []),
    ("dogip_last_error", C.c_char_p, []),
    ("dogip_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("dogip_slab_range", C.c_int, [C.c_int64, C.c_int, C.c_int, c_i64p, c_i64p]),
    ("dogip_mesh_setup", C.c_int, [C.c_int, C.c_int64, C.c_int, c_dp, C.c_int, C.c_int, C.c_void_p,
                                   C.c_int, C.POINTER(C.c_void_p)]),
    ("dogip_mesh_setup_ex", C.c_int, [C.c_int, C.c_int64, C.c_int, c_dp, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                      C.c_int, C.POINTER(C.c_void_p)]),
    ("dogip_loopback_create", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("dogip_loopback_destroy", C.c_int, [C.c_void_p]),
    ("dogip_mesh_info", C.c_int, [C.c_void_p, C.POINTER(MeshInfo)]),
    ("dogip_weights", C.c_int, [C.c_void_p, C.c_int, C.POINTER(Coeff), C.c_int, C.c_void_p,
                                C.POINTER(C.c_void_p)]),
    ("dogip_weights_ex", C.c_int, [C.c_void_p, C.c_int, C.POINTER(Coeff), C.c_int, C.c_int, C.c_void_p,
                                   C.POINTER(C.c_void_p)]),
    ("dogip_op_info", C.c_int, [C.c_void_p, C.POINTER(OpInfo)]),
    ("dogip_apply", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]),
    ("dogip_apply_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]),
    ("dogip_load_vector", C.c_int, [C.c_void_p, C.c_double, C.c_void_p, C.c_uint, C.c_void_p]),
    ("dogip_cg", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_uint,
                           C.c_void_p, C.POINTER(CgResult)]),
    ("dogip_kernel_launches", C.c_int64, []),
    ("dogip_reference_table", C.c_int, [C.c_int, C.c_int, C.c_int, c_dp, C.c_int64]),
    ("dogip_reference_nnz", C.c_int, [C.c_int, C.c_int, C.c_int, c_i64p, c_i64p]),
    ("dogip_csr_nnz", C.c_int, [C.c_int, C.c_int64, C.c_int, c_i64p]),
    ("dogip_quadrature", C.c_int, [C.c_int, C.c_int, c_dp, c_dp, C.c_int64]),
    ("dogip_export_weights", C.c_int, [C.c_void_p, c_dp, C.c_int64]),
    ("dogip_export_dofmap", C.c_int, [C.c_void_p, c_i64p, C.c_int64]),
    ("dogip_test_perturb_weight", C.c_int, [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_double]),
    ("dogip_op_destroy", None, [C.c_void_p]),
    ("dogip_mesh_destroy", None, [C.c_void_p]),
]

_lib = None


class DogipError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def load() -> C.CDLL:
    """Load libdogip.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("DOGIP_LIB", LIB_PATH)     # A/B experiments: libdogip_<variant>.so
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, allow_positive: bool = False) -> int:
    if rc < 0 or (rc > 0 and not allow_positive):
        raise DogipError(rc, load().dogip_last_error().decode())
    return rc
