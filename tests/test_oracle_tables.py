"""Oracle pins against the integers the paper prints (Tables 1-4).

Fixture: tests/golden/paper_tables_1_4.json, transcribed from PAPER.md with the
line of every row.  These pin: node layout + reference simplex (nnz B-hat,
reading L1/L2), W spaces (mem A_T^DoGIP, reading L7/L11), mesh topology + DoF
map (mem A of Tables 3/4, readings L3/L4) and the cost model (eq:memory_eff,
eq:comp_eff with nnz_{+-1} = entries exactly +-1, reading L12).
"""
import json
import os

import pytest

from oracle import metrics
from oracle.reference import bhat_el_exact, bhat_wp_exact, dim_P, nnz_counts

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                   "paper_tables_1_4.json")))
CASES = [(t, r) for t, rows in GOLD["tables"].items() for r in rows]
IDS = [f"{t}-k{r['k']}" for t, r in CASES]


def _dform(t):
    return (2 if t.endswith("2D") else 3), (0 if t.startswith("WP") else 1)


def _bhat(t, k):
    d, form = _dform(t)
    return bhat_wp_exact(d, k) if form == 0 else bhat_el_exact(d, k)


@pytest.mark.parametrize("t,row", CASES, ids=IDS)
def test_nnz_bhat(t, row):
    nnz, _ = nnz_counts(_bhat(t, row["k"]))
    assert nnz == row["nnz_Bhat"], f"P:{row['paper_line']}"


@pytest.mark.parametrize("t,row", CASES, ids=IDS)
def test_element_storage_columns(t, row):
    d, form = _dform(t)
    k, N = row["k"], row["N"]
    assert dim_P(d, k) ** 2 == row["mem_A_T"]
    assert metrics.nnz_AT_dogip(d, k, form) == row["mem_A_dogip_T"]
    assert metrics.nnz_AT_dogip(d, k, form) * metrics.n_elem(d, N) == row["mem_A_dogip"]


@pytest.mark.parametrize("t,row", CASES, ids=IDS)
def test_dim_V_captions(t, row):
    d, _ = _dform(t)
    assert metrics.dim_V(d, row["N"], row["k"]) == GOLD["dim_V"][f"{d}D"]["value"]


MEM_A_PINNED = [(t, r) for t, r in CASES
                if t.startswith("EL") or (t == "WP2D" and r["k"] == 1)]


@pytest.mark.parametrize("t,row", MEM_A_PINNED,
                         ids=[f"{t}-k{r['k']}" for t, r in MEM_A_PINNED])
def test_mem_A_full_pattern(t, row):
    """Tables 3/4 (and Table 1 k=1): CSR memory of the full coupling pattern."""
    d, _ = _dform(t)
    k, N = row["k"], row["N"]
    nnz = metrics.nnz_A_pattern(d, N, k)
    assert metrics.mem_csr(nnz, metrics.dim_V(d, N, k)) == row["mem_A"]


@pytest.mark.parametrize("t,row", [(t, r) for t, r in CASES if t.startswith("WP") and r["k"] > 1],
                         ids=[f"{t}-k{r['k']}" for t, r in CASES if t.startswith("WP") and r["k"] > 1])
def test_wp_mem_A_is_below_full_pattern(t, row):
    """Tables 1/2 k>=2 drop coefficient-dependent sub-1e-14 entries (reading L13):
    the printed value can only be below the full pattern (parity unpinned)."""
    d, _ = _dform(t)
    k, N = row["k"], row["N"]
    full = metrics.mem_csr(metrics.nnz_A_pattern(d, N, k), metrics.dim_V(d, N, k))
    assert row["mem_A"] <= full


@pytest.mark.parametrize("t,row", CASES, ids=IDS)
def test_efficiencies_two_decimals(t, row):
    d, form = _dform(t)
    k, N = row["k"], row["N"]
    nnzB, pm1 = nnz_counts(_bhat(t, k))
    me = metrics.memory_efficiency(d, N, k, form, row["mem_A"])
    ce = metrics.comp_efficiency(d, N, k, form, row["mem_A"], nnzB, pm1)
    assert abs(me - row["mem_eff"]) <= 0.005 + 1e-12, (me, row)
    assert abs(ce - row["comp_eff"]) <= 0.005 + 1e-12, (ce, row)


def test_nnz_pm1_wp_unit_rows():
    """WP: rows of B-hat at double-grid nodes that coincide with primal nodes
    are unit rows (P:283 with the delta property) -> >= V_T entries +-1."""
    for d, ks in ((2, (1, 2, 3, 4)), (3, (1, 2, 3))):
        for k in ks:
            _, pm1 = nnz_counts(bhat_wp_exact(d, k))
            assert pm1 >= dim_P(d, k)
