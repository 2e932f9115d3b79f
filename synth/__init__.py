"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the DoGIP method: it only draws random
numbers and names the benchmark configurations (BASELINE.json ``configs``).
Both ``oracle/`` (tests) and ``paper_1710_09913_b200`` (product path) consume
the arrays it returns; neither side imports the other.  The recipes follow
the input readings L19-L23 recorded in DESIGN.md.
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .generators import (  # noqa: F401
    u_vector,
    grf_per_cell,
    rotation_field_params,
    vertex_jitter,
)
