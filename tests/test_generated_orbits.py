"""FULL WP storage through the symmetry-adapted body (RefElem<d, p, 0, 6> in the generated
header): the stored row of W node j is ROWPERM[j].  The body assumes that the rows come in
whole orbits of the barycentric involutions G = <(0 1), (2 3)> (3D) / <(0 1)> (2D) -- the
group under which Bhat is equivariant (product basis) -- sorted by decreasing
orbit size, with the k-th row of a 4-orbit holding g_k(rep) for g_0 = id, g_1 = (0 1),
g_2 = (2 3), g_3 = (0 1)(2 3) (its butterflies form ahat_psi = (1/4) sum_k psi(g_k) a_k).

This checks those invariants against the oracle's own node numbering (reading L5,
oracle.reference.multi_indices), independently of the generator's orbit code.  CPU only;
skipped when the library has not been built (the header is a build product)."""
import os
import re

import pytest

from oracle.reference import multi_indices

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "paper_1710_09913_b200", "csrc", "generated", "bhat_gen.cuh")


def _rowperm(text: str, d: int, p: int):
    m = re.search(r"struct RefElem<%d, %d, 0, 6> \{(.*?)\n\};" % (d, p), text, re.S)
    assert m, f"RefElem<{d}, {p}, 0, 6> missing"
    body = m.group(1)
    wt = int(re.search(r"WT = (\d+)", body).group(1))
    rp = re.search(r"ROWPERM\[(\d+)\] = \{([^}]*)\}", body)
    assert rp and int(rp.group(1)) == wt
    return [int(x) for x in rp.group(2).split(",")]


def _act(g, a):
    """barycentric index permutation g (tuple of images) applied to multi-index a"""
    return tuple(a[g[i]] for i in range(len(a)))


@pytest.mark.skipif(not os.path.exists(HEADER), reason="library not built (no generated header)")
@pytest.mark.parametrize("d,p", [(2, 1), (2, 2), (2, 3), (2, 4), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_full_wp_rows_in_orbit_order(d, p):
    text = open(HEADER).read()
    perm = _rowperm(text, d, p)
    W = list(multi_indices(d, 2 * p))
    assert sorted(perm) == list(range(len(W))), "ROWPERM is not a permutation"
    node_at = [None] * len(W)
    for j, r in enumerate(perm):
        node_at[r] = W[j]
    if d == 3:
        gens = [(0, 1, 2, 3), (1, 0, 2, 3), (0, 1, 3, 2), (1, 0, 3, 2)]   # id, (0 1), (2 3), both
    else:
        gens = [(0, 1, 2), (1, 0, 2)]
    orbit = {a: frozenset(_act(g, a) for g in gens) for a in W}
    sizes = [len(orbit[node_at[r]]) for r in range(len(W))]
    assert sizes == sorted(sizes, reverse=True), "orbits not sorted by decreasing size"
    r = 0
    while r < len(W):
        s = sizes[r]
        block = node_at[r:r + s]
        assert r % s == 0, "an orbit straddles an alignment boundary"
        assert frozenset(block) == orbit[block[0]], f"rows {r}..{r + s - 1} are not one G-orbit"
        if s == len(gens):   # full orbit: member k = g_k(rep)
            assert block == [_act(g, block[0]) for g in gens]
        r += s
