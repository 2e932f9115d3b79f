"""Host-side checks of libdogip.so on CPU (no GPU calls).

* the library loads and exports every symbol include/dogip.h declares;
* its exact reference tables equal the oracle's rationals rounded to fp64
  BITWISE (two independent exact implementations);
* its quadrature equals the oracle's scipy-based rule to a few ulp;
* slab partition, host-only mesh info and DoF map agree with the oracle;
* argument errors map to the documented status codes.
"""
import os
import re

import numpy as np
import pytest

from oracle import mesh as om
from oracle import quadrature as oq
from oracle import reference as ref
from paper_1710_09913_b200 import _lib
from paper_1710_09913_b200.api import (DogipError, Mesh, quadrature, reference_nnz, reference_table,
                                       slab_range)

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "dogip.h")


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    decl = set(re.findall(r"\b(dogip_[a-z_0-9]+)\s*\(", open(HEADER).read()))
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(lib, name), name
    assert decl == {n for n, _, _ in _lib.SIGNATURES}
    assert lib.dogip_version() >= 100


@pytest.mark.parametrize("d,p", [(2, p) for p in range(1, 9)] + [(3, p) for p in range(1, 5)])
def test_reference_tables_bitwise(d, p):
    for form in (0, 1):
        got = reference_table(d, p, form)
        want = (ref.bhat_wp(d, p) if form == 0 else ref.bhat_el(d, p)).ravel()
        assert got.shape == want.shape
        assert np.array_equal(got, want), (d, p, form)
        nnz, pm1 = reference_nnz(d, p, form)
        assert (nnz, pm1) == ref.nnz_counts(ref.bhat_wp_exact(d, p) if form == 0 else ref.bhat_el_exact(d, p))


@pytest.mark.parametrize("d,n", [(2, 1), (2, 4), (2, 7), (3, 4), (3, 6), (3, 7), (3, 11)])
def test_quadrature_matches_oracle(d, n):
    """Same points to 2 ulp; weights within scipy's own accuracy (its
    Golub-Welsch weights are off by up to ~2e-14 at n = 11, ours ~1e-15,
    both measured against the exact simplex moments below)."""
    import itertools
    from fractions import Fraction
    from math import factorial
    pts, wts = quadrature(d, n)
    opts, owts = oq.simplex_rule(d, n)
    assert np.allclose(pts, opts, rtol=0, atol=4e-16)
    assert np.allclose(wts, owts, rtol=1e-13, atol=0)
    P = np.asarray(pts, dtype=np.longdouble)
    W = np.asarray(wts, dtype=np.longdouble)
    for al in itertools.product(range(2 * n), repeat=d):
        if sum(al) <= 2 * n - 1:
            ex = Fraction(int(np.prod([factorial(a) for a in al])), factorial(sum(al) + d))
            v = float(np.sum(W * np.prod(P ** np.array(al), axis=1)))
            assert abs(v - float(ex)) <= 4e-15 * float(ex), al


@pytest.mark.parametrize("N,n", [(128, 1), (128, 2), (128, 8), (96, 8), (7, 3), (5, 5)])
def test_slab_ranges_tile_the_axis(N, n):
    z = [slab_range(N, r, n) for r in range(n)]
    assert z[0][0] == 0 and z[-1][1] == N
    assert all(a[1] == b[0] for a, b in zip(z, z[1:]))
    assert max(b - a for a, b in z) - min(b - a for a, b in z) <= 1


@pytest.mark.parametrize("d,N,p,nranks", [(2, 5, 2, 1), (2, 33, 1, 1), (3, 3, 3, 1), (3, 4, 2, 2), (2, 6, 3, 3),
                                          (3, 33, 1, 2), (2, 97, 2, 3)])
def test_host_mesh_info_and_dofmap(d, N, p, nranks):
    lT = om.dof_map(om.structured_mesh(d, N), p)
    ns = 2 if d == 2 else 6
    M = p * N + 1
    plane = M ** (d - 1)
    for r in range(nranks):
        m = Mesh(d, N, p, rank=r, nranks=nranks, device=-1)
        info = m.info
        z0, z1 = slab_range(N, r, nranks)
        assert (info["z0"], info["z1"]) == (z0, z1)
        assert info["ndof_local"] == plane * (p * (z1 - z0) + 1)
        assert info["dof_offset"] == p * z0 * plane
        assert info["n_elem_global"] == ns * N ** d
        assert info["owned_end"] == info["ndof_local"] - (plane if r < nranks - 1 else 0)
        got = m.dofmap() + info["dof_offset"]
        cells_per_layer = N ** (d - 1)
        e0 = ns * cells_per_layer * z0
        e1 = ns * cells_per_layer * z1
        assert np.array_equal(got, lT[e0:e1])


@pytest.mark.parametrize("args,code", [((4, 3, 1), -1), ((2, 0, 1), -2), ((2, 3, 5), -3), ((3, 2, 0), -3)])
def test_mesh_argument_errors(args, code):
    with pytest.raises(DogipError) as ei:
        Mesh(*args, device=-1)
    assert ei.value.code == code


def test_mesh_tile_count_limit():
    """2^31 or more element tiles per rank (tile_coord's 31-bit multiply-shift decode)
    is rejected at setup, before any allocation."""
    with pytest.raises(DogipError) as ei:
        Mesh(3, 2600, 1, device=-1)                          # 6 * 82 * 2600^2 = 3.3e9 tiles
    assert ei.value.code == -2 and "2^31" in str(ei.value)
    m = Mesh(3, 2600, 1, rank=0, nranks=2, device=-1)      # half the layers: accepted
    assert m.info["n_elem_local"] == 6 * 2600 ** 2 * 1300
    m.close()


def test_slab_error_and_operator_on_host_mesh():
    with pytest.raises(DogipError) as ei:
        Mesh(3, 2, 1, rank=0, nranks=3, device=-1)
    assert ei.value.code == -2
    from paper_1710_09913_b200.api import CoeffSpec, Operator
    m = Mesh(2, 2, 1, device=-1)
    with pytest.raises(DogipError) as ei:
        Operator(m, 0, CoeffSpec(0, np.array([1.0])))
    assert ei.value.code == -10


def test_report_reproduces_paper_tables():
    """NEXT item 4: the library's own report reproduces Tables 3/4 entirely and
    every Table 1/2 column except mem A for k >= 2 (reading L13)."""
    import json
    from paper_1710_09913_b200 import report
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables_1_4.json")))
    rows = {(r["form"], r["d"], r["k"]): r for r in report.tables()}
    for t, grows in gold["tables"].items():
        form, d = t[:2], int(t[2])
        for g in grows:
            r = rows[(form, d, g["k"])]
            for key in ("mem_A_T", "mem_A_dogip", "mem_A_dogip_T", "nnz_Bhat"):
                assert r[key] == g[key], (t, g["k"], key)
            if form == "EL" or g["k"] == 1 and d == 2:
                assert r["mem_A"] == g["mem_A"], (t, g["k"])
                assert abs(r["mem_eff"] - g["mem_eff"]) <= 0.005 + 1e-12
                assert abs(r["comp_eff"] - g["comp_eff"]) <= 0.005 + 1e-12
            else:
                assert r["mem_A"] >= g["mem_A"]


def test_header_constants_match_binding():
    """#define values of include/dogip.h (storage variants, flags, status codes) equal the
    binding's constants -- the ABI cannot drift silently."""
    text = open(HEADER).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(DOGIP_[A-Z0-9_]+)\s+(-?\d+)", text)}
    for name in ("DOGIP_STORE_FULL", "DOGIP_STORE_ISO", "DOGIP_STORE_GLOBAL",
                 "DOGIP_STORE_QP", "DOGIP_STORE_SYM", "DOGIP_DIRICHLET_ZERO", "DOGIP_NO_EXCHANGE",
                 "DOGIP_CG_RESUME"):
        assert name in defs, name
        assert getattr(_lib, name) == defs[name], name
    for code, label in _lib.STATUS.items():
        assert defs.get("DOGIP_" + label) == code, label
