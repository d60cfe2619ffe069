"""GPU parity at the SCC-size boundaries of the kernels' mask widths:
32 / 33 (uint32 -> uint64 masks), 63 / 64 / 65 (the last one-word mask, the first
two-word one), 128 / 129 (two -> three words) and 256 (four words), on the DFS engine in
both modes (materialized arrays element by element, COUNT_HASH counts, E_canon and digest)
and, for 32 / 33 / 64, on the frontier engine.  Each size comes closed (no arc leaves the
SCC) and with arcs into and out of it (head / tail / transit segments).  Expected values
come from oracle/ only."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")

SIZES = [32, 33, 63, 64, 65, 128, 129, 256]


def _scc(n, open_):
    """A ring of n vertices with three chords (a handful of cycles, O(n^2) paths); open_:
    a source vertex n -> 0 and n // 2, and exits n // 3 -> n + 1, (n - 1) -> n + 1."""
    arcs = [(i, (i + 1) % n) for i in range(n)]
    arcs += [(0, n // 2), (n // 3, n // 8), (3 * n // 4, n // 5)]
    m = n
    if open_:
        arcs += [(n, 0), (n, n // 2), (n // 3, n + 1), (n - 1, n + 1)]
        m = n + 2
    return gen.from_arcs(m, sorted(set(arcs)), name=f"ring{n}{'-open' if open_ else ''}")


def _oracle(g):
    ro, rv = oracle.prime_paths(g)
    return {"n_paths": len(ro) - 1, "total_vertices": int(ro[-1]), "n_extensions": oracle.ext_count(g),
            "digest": oracle.digest(ro, rv)}, ro, rv


def _stats(st):
    return {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"], "n_extensions": st["n_extensions"],
            "digest": (st["hash_lo"], st["hash_hi"])}


@pytest.mark.parametrize("open_", [False, True])
@pytest.mark.parametrize("n", SIZES)
def test_dfs_engine_at_mask_boundaries(n, open_):
    g = _scc(n, open_)
    ref, ro, rv = _oracle(g)
    ps = tp.prime_paths(g, digest=True)
    off, vert = ps.to_numpy()
    np.testing.assert_array_equal(off, ro, err_msg=g.name)
    np.testing.assert_array_equal(vert, rv, err_msg=g.name)
    assert _stats(ps.stats) == ref, g.name
    assert ps.stats["max_scc"] == n
    cnt = tp.prime_paths(g, mode="count", digest=True).stats
    assert _stats(cnt) == ref, g.name


@pytest.mark.parametrize("open_", [False, True])
@pytest.mark.parametrize("n", [32, 33, 64])
def test_frontier_engine_at_mask_boundaries(n, open_):
    g = _scc(n, open_)
    ref, _, _ = _oracle(g)
    st = tp.prime_paths(g, mode="count", digest=True, engine="frontier").stats
    assert _stats(st) == ref, g.name


def test_frontier_rejects_65():
    g = _scc(65, False)
    with pytest.raises(Exception):
        tp.prime_paths(g, mode="count", digest=True, engine="frontier")
