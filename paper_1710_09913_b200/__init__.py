"""B200-native DoGIP apply + CG (arXiv 1710.09913).

The compute path is libdogip.so (hand-written CUDA for sm_100a behind the C
ABI of include/dogip.h); this package only binds it (``_lib``, ``api``) and
builds it (``build``).  There is no CPU fallback.
"""
from .api import (DOGIP_EL, DOGIP_WP, CoeffSpec, DogipError, Mesh, Operator,  # noqa: F401
                  nccl_unique_id, quadrature, reference_nnz, reference_table, slab_range)
