"""Out-degree-2 normalization (tpgen_normalize_outdeg2, host C++; Fig. 5;
DESIGN.md R24).  Host-only, so these run without a GPU.  Pins: the result's shape (out-degree
<= 2, the chain of d - 2 new vertices, unchanged rows of vertices with d <= 2), and -- by brute
force on small graphs, not by re-deriving the construction -- that the simple paths between the
input's vertices are exactly those of the normalized graph with the new vertices deleted, and
that the input vertices' reachability is unchanged."""
import itertools

import numpy as np
import pytest

from workloads import generators as gen

tp = pytest.importorskip("paper_2210_16998_b200")


def _rows(n, off, tgt):
    return [list(tgt[off[v]:off[v + 1]]) for v in range(n)]


def _simple_paths(rows, n_orig):
    """Every simple path (as a tuple of vertex ids, cycles v..v included) of the graph, with the
    vertices >= n_orig deleted, keeping those that start and end at vertices < n_orig."""
    out = set()

    def walk(path, seen):
        u = path[-1]
        if path[0] < n_orig and u < n_orig:
            out.add(tuple(x for x in path if x < n_orig))
        for w in rows[u]:
            if w == path[0]:  # a cycle closure (a self-loop closes <s, s>)
                if w < n_orig:
                    out.add(tuple(x for x in path + [w] if x < n_orig))
            elif w not in seen:
                seen.add(w)
                walk(path + [w], seen)
                seen.discard(w)

    for s in range(len(rows)):
        if s < n_orig:
            walk([s], {s})
    return out


def _reach(rows):
    n = len(rows)
    R = np.zeros((n, n), dtype=bool)
    for s in range(n):
        st, R[s, s] = [s], True
        while st:
            u = st.pop()
            for w in rows[u]:
                if not R[s, w]:
                    R[s, w] = True
                    st.append(w)
    return R


def _graphs():
    yield gen.fig1b()
    yield gen.dense_scc(6, 4, 3)
    yield gen.dense_scc(7, 3, 5)
    yield gen.from_arcs(5, [(0, 1), (0, 2), (0, 3), (0, 4), (4, 0), (3, 3)])
    rng = np.random.default_rng(11)
    for i in range(25):
        yield gen.random_digraph(int(rng.integers(2, 8)), 0.45, 300 + i, self_loops=bool(i % 2))


def test_shape():
    for g in _graphs():
        h = tp.normalize_outdeg2(g)
        deg = np.diff(g.offsets)
        extra = int(np.maximum(deg - 2, 0).sum())
        assert h.n == g.n + extra and len(h.targets) == g.m + extra, g.name
        assert np.all(np.diff(h.offsets) <= 2), g.name
        assert np.all(h.origin[:g.n] == np.arange(g.n))
        for v in range(g.n):
            row = sorted(g.targets[g.offsets[v]:g.offsets[v + 1]])
            hrow = list(h.targets[h.offsets[v]:h.offsets[v + 1]])
            if len(row) <= 2:
                assert hrow == row, (g.name, v)
            else:
                assert hrow[0] == row[0] and hrow[1] >= g.n and h.origin[hrow[1]] == v
                assert int(np.sum(h.origin[g.n:] == v)) == len(row) - 2
        for x in range(g.n, h.n):  # a new vertex has one predecessor (its chain's previous link)
            assert int(np.sum(h.targets == x)) == 1


def test_identity_on_outdegree_two():
    g = gen.fig1b()  # a CFG of out-degree <= 2
    assert np.all(np.diff(g.offsets) <= 2)
    h = tp.normalize_outdeg2(g)
    assert h.n == g.n
    np.testing.assert_array_equal(h.offsets, g.offsets)
    np.testing.assert_array_equal(h.targets, g.targets)


def test_simple_paths_and_reachability_preserved():
    for g in _graphs():
        if g.n > 9:
            continue
        h = tp.normalize_outdeg2(g)
        rg = [sorted(r) for r in _rows(g.n, g.offsets, g.targets)]
        rh = _rows(h.n, h.offsets, h.targets)
        assert _simple_paths(rh, g.n) == _simple_paths(rg, g.n), g.name
        np.testing.assert_array_equal(_reach(rh)[:g.n, :g.n], _reach(rg), err_msg=g.name)


def test_invalid_graphs():
    with pytest.raises(Exception):
        tp.normalize_outdeg2((np.array([0, 2], dtype=np.int64), np.array([0, 0], dtype=np.int32)))  # duplicate arc
    with pytest.raises(Exception):
        tp.normalize_outdeg2((np.array([0, 1], dtype=np.int64), np.array([3], dtype=np.int32)))  # out of range
