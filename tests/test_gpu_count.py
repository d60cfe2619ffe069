"""GPU parity of COUNT_HASH mode (counts, vertices, E_canon, digest without the output;
the DFS's count modes, dfs.cuh) and the full-size comparisons of the two largest
configurations against the oracle (SURVEY 8(d) "Comparison"; Thm. 3).

Expected values come only from oracle/: oracle.pp_stats streams every start vertex's
prime paths through the same digest (oracle_pp_stats, pinned in tests/test_oracle.py
against the materialized oracle blocks), run on the host's cores."""
import os

import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")

M64 = (1 << 64) - 1


def _tot(st_rows):
    """Totals of oracle.pp_stats rows: (n_paths, vertices, hash_lo, hash_hi)."""
    a = st_rows[:, :4].astype(object)
    return (int(a[:, 0].sum()), int(a[:, 1].sum()), int(a[:, 2].sum()) & M64, int(a[:, 3].sum()) & M64)


def _gpu_tot(st):
    return (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"])


def _count(g, **kw):
    return tp.prime_paths(g, mode="count", digest=True, **kw).stats


def _corpus():
    rng = np.random.default_rng(11)
    for i in range(60):
        n = int(rng.integers(1, 12))
        yield gen.random_digraph(n, float(rng.choice([0.1, 0.2, 0.3, 0.45])), 700 + i,
                                 self_loops=bool(rng.random() < 0.5))
    yield gen.fig1b()
    yield gen.config2()
    yield gen.config4(K=30)
    yield gen.k_seq_loops(5, 4)
    yield gen.k_nested_if(5)
    for n, d, seed in ((12, 3, 1), (16, 3, 2), (20, 3, 7)):
        yield gen.dense_scc(n, d, seed)
    yield gen.parallel_sccs(3, 24, 9)  # SCCs with entry and exit arcs (config 5's shape, small)
    yield gen.parallel_sccs(2, 40, 3)  # ... with 64-bit masks


def test_count_mode_matches_oracle():
    """Every graph of the corpus: counts, vertices, digest and E_canon of the count-mode
    DFS equal the oracle's; the counts-only variant gives the same counts."""
    for g in _corpus():
        st = _count(g)
        ref = oracle.pp_stats(g)
        assert _gpu_tot(st) == _tot(ref), g.name
        assert st["n_extensions"] == oracle.ext_count(g), g.name
        st2 = tp.prime_paths(g, mode="count", digest=False).stats
        assert (st2["n_paths"], st2["total_vertices"], st2["n_extensions"]) == (st["n_paths"], st["total_vertices"],
                                                                               st["n_extensions"]), g.name
        if tp.components(g)[0].size and max(np.bincount(tp.components(g)[0])) <= 64:
            assert st2["n_cross"] == st["n_cross"], g.name  # (n_cross needs the digest pass above 64)


def test_count_mode_per_start_blocks():
    """Start-vertex ranges in count mode equal the oracle's per-start rows."""
    g = gen.parallel_sccs(3, 24, 9)
    ref = oracle.pp_stats(g)
    plan = tp.Plan(g)
    for v in range(g.n):
        st = plan.prime_paths(mode="count", digest=True, start_range=(v, v + 1)).stats
        assert _gpu_tot(st) == tuple(int(x) for x in ref[v]), v
    plan.close()


def test_count_mode_head_overflow_retry(monkeypatch):
    """A head buffer too small for the call's head segments is grown and the phase rerun."""
    g = gen.parallel_sccs(4, 30, 2)
    ref = _tot(oracle.pp_stats(g))
    monkeypatch.setenv("TPGEN_TEST_HEADCAP", "300")
    st = _count(g)
    assert _gpu_tot(st) == ref
    assert st["n_count_rounds"] >= 3  # segment phase + an overflowed and a rerun prime-path phase


@pytest.mark.timeout(1200)
def test_config3_whole_list_vs_oracle():
    """Config 3 at full size in the bench's launch configuration: all 22 start-vertex
    blocks element by element, and the whole list's n_paths, total vertices, E_canon and
    digest -- materialized and in count mode."""
    g = gen.config3()
    ref = oracle.pp_stats_parallel(g, chunk=1)
    plan = tp.Plan(g)
    ps = plan.prime_paths(digest=True)
    st = ps.stats
    assert _gpu_tot(st) == _tot(ref)
    e_canon = oracle.ext_count(g)
    assert st["n_extensions"] == e_canon == int(ref[:, 4].sum())
    off, vert = ps.offsets, ps.vertices
    first = vert[off[:-1]].cpu().numpy()
    assert np.all(np.diff(first) >= 0)
    counts = np.bincount(first, minlength=g.n)
    for s in range(g.n):
        assert counts[s] == int(ref[s, 0]), s
        ro, rv = oracle.prime_paths(g, v_lo=s, v_hi=s + 1)
        idx = np.nonzero(first == s)[0]
        a, b = int(idx[0]), int(idx[-1]) + 1
        o = off[a:b + 1].cpu().numpy()
        np.testing.assert_array_equal(o - o[0], ro, err_msg=f"start {s}")
        np.testing.assert_array_equal(vert[o[0]:o[-1]].cpu().numpy(), rv, err_msg=f"start {s}")
    del ps
    cs = plan.prime_paths(mode="count", digest=True).stats
    assert _gpu_tot(cs) == _tot(ref) and cs["n_extensions"] == e_canon
    plan.close()


@pytest.mark.timeout(2400)
def test_config5_every_start_vertex_vs_oracle():
    """Config 5 (16 parallel 56-vertex SCCs, ~1.3e10 extensions) on one GPU: for every one
    of its start vertices, (n_paths, total vertices, E_canon, digest) of a count-mode call
    on that start vertex equal the oracle's streamed per-start row; the whole-graph count
    call equals the oracle's totals (no GPU result is compared with another GPU result)."""
    g = gen.config5()
    ref = oracle.pp_stats_parallel(g, chunk=2)
    plan = tp.Plan(g)
    whole = plan.prime_paths(mode="count", digest=True).stats
    assert _gpu_tot(whole) == _tot(ref)
    assert whole["n_extensions"] == int(ref[:, 4].sum()) > 10 ** 10
    for v in range(g.n):
        st = plan.prime_paths(mode="count", digest=True, start_range=(v, v + 1)).stats
        assert _gpu_tot(st) == tuple(int(x) for x in ref[v, :4]), v
        assert st["n_extensions"] == int(ref[v, 4]), v
    plan.close()


# ------------------------------------------------------------ test paths, COUNT_HASH
def _tp_graphs():
    yield gen.fig1b()
    yield gen.config2()
    yield gen.k_seq_loops(4, 3)
    yield gen.config4(K=30)
    yield gen.parallel_sccs(3, 24, 9)
    yield gen.parallel_sccs(2, 40, 3)


def test_tp_count_mode_matches_oracle():
    """tpgen_test_paths in COUNT_HASH mode (each prime path's R15 test path hashed when the
    path is found, never written) equals the oracle's streamed TP statistics; the list path
    (test paths of a given prime-path list) gives the same numbers."""
    for g in _tp_graphs():
        ref = _tot(oracle.pp_stats(g, tp=(g.entry, g.exit)))
        st = tp.test_paths(g, g.entry, g.exit, mode="count").stats
        assert _gpu_tot(st) == ref, g.name
        pps = tp.prime_paths(g)
        st2 = tp.test_paths(g, g.entry, g.exit, pps, mode="count").stats
        assert _gpu_tot(st2) == ref, g.name


def test_tp_count_mode_unreachable():
    g = gen.from_arcs(4, [(0, 1), (1, 0), (2, 3)])
    with pytest.raises(tp.TpgenError) as ei:
        tp.test_paths(g, 0, 1, mode="count")
    assert ei.value.status_name == "TPGEN_ERR_UNREACHABLE"


@pytest.mark.timeout(1200)
def test_config4_full_test_paths_element_by_element():
    """Config 4 at full size (K = 150 loops): every test path, element by element, against
    oracle.test_paths (R15) of the oracle's prime paths; and the COUNT_HASH digest."""
    g = gen.config4()
    ro, rv = oracle.prime_paths(g)
    to, tv = oracle.test_paths(g, ro, rv, g.entry, g.exit)
    ts = tp.test_paths(g, g.entry, g.exit)
    o, v = ts.to_numpy()
    np.testing.assert_array_equal(o, to)
    np.testing.assert_array_equal(v, tv)
    st = tp.test_paths(g, g.entry, g.exit, mode="count").stats
    assert (st["n_paths"], st["total_vertices"]) == (len(to) - 1, int(to[-1]))
    assert (st["hash_lo"], st["hash_hi"]) == oracle.digest(to, tv)


@pytest.mark.timeout(1800)
def test_config3_and_config5_test_path_digests():
    """Configs 3 and 5 at full size: the COUNT_HASH test-path count, vertices and digest equal
    the oracle's streamed TP statistics over every start vertex (host cores)."""
    for g, entry, exit_ in ((gen.config3(), 0, 21), (gen.config5(), None, None)):
        entry = g.entry if entry is None else entry
        exit_ = g.exit if exit_ is None else exit_
        ref = oracle.pp_stats_parallel(g, tp=(entry, exit_), chunk=2)
        st = tp.test_paths(g, entry, exit_, mode="count").stats
        assert _gpu_tot(st) == _tot(ref), g.name
