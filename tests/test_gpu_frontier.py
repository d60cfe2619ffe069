"""GPU parity of the level-synchronous frontier engine (TPGEN_ENGINE_FRONTIER, DESIGN.md
§6.6): counts, E_canon and the order-free digest vs the CPU oracle (expected values from
oracle/ only), and vs the DFS engine at config 3's full size."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")


def _oracle_stats(g, v_lo=0, v_hi=None):
    ro, rv = oracle.prime_paths(g, v_lo=v_lo, v_hi=v_hi)
    return {"n_paths": len(ro) - 1, "total_vertices": int(ro[-1]),
            "n_extensions": oracle.ext_count(g, v_lo=v_lo, v_hi=v_hi), "digest": oracle.digest(ro, rv)}


def _frontier(g, **kw):
    st = tp.prime_paths(g, mode="count", digest=True, engine="frontier", **kw).stats
    return {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"],
            "n_extensions": st["n_extensions"], "digest": (st["hash_lo"], st["hash_hi"])}


def _lean_corpus():
    yield gen.from_arcs(1, [(0, 0)])                       # self-loop: [0, 0]
    yield gen.from_arcs(2, [(0, 1), (1, 0)])               # 2-cycle
    yield gen.from_arcs(3, [])                             # isolated vertices only
    for n, d, seed in ((5, 2, 1), (8, 3, 2), (12, 3, 3), (14, 4, 4), (16, 3, 5)):
        yield gen.dense_scc(n, d, seed)
    ring = [(i, (i + 1) % 32) for i in range(32)] + [(i, (i + 5) % 32) for i in range(0, 32, 4)]
    yield gen.from_arcs(32, ring)                          # a 32-vertex SCC: every mask bit in use
    parts = [gen.dense_scc(6 + i % 5, 2 + i % 2, 50 + i) for i in range(12)]
    parts += [gen.from_arcs(1, [(0, 0)]), gen.from_arcs(2, []), gen.from_arcs(2, [(0, 1), (1, 0)])]
    yield gen.disjoint_union(parts, name="lean-union")


def test_frontier_matches_oracle():
    for g in _lean_corpus():
        assert _frontier(g) == _oracle_stats(g), g.name


def _wide_corpus():
    """SCCs of 33..64 vertices: the 64-bit-mask records (24 bytes: mask, meta | S)."""
    yield gen.dense_scc(36, 2, 3)
    yield gen.dense_scc(40, 2, 4)
    yield gen.from_arcs(64, [(i, (i + 1) % 64) for i in range(64)] + [(i, (i + 7) % 64) for i in range(0, 64, 8)])
    yield gen.disjoint_union([gen.dense_scc(34, 2, 9), gen.dense_scc(7, 3, 10), gen.from_arcs(1, [(0, 0)]),
                              gen.from_arcs(2, [])], name="wide-union")


def test_frontier_wide_masks_match_oracle():
    for g in _wide_corpus():
        assert _frontier(g) == _oracle_stats(g), g.name


def test_frontier_wide_masks_chunked(monkeypatch):
    monkeypatch.setenv("TPGEN_FRONTIER_CHUNK", "512")
    g = gen.dense_scc(36, 2, 3)
    st = tp.prime_paths(g, mode="count", digest=True, engine="frontier").stats
    assert st["n_count_rounds"] > st["max_scc"] + 1  # chunks (one persistent launch walks them)
    assert {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"],
            "n_extensions": st["n_extensions"], "digest": (st["hash_lo"], st["hash_hi"])} == _oracle_stats(g)


def test_frontier_counts_only(monkeypatch):
    """digest=False: records without the digest sum (8 bytes for 32-bit masks, 16 for
    64-bit) and no hashing; counts and E_canon equal to the oracle's, in one pass and
    DFS-chunked."""
    graphs = list(_lean_corpus()) + list(_wide_corpus())
    for chunk in (None, "300"):
        if chunk:
            monkeypatch.setenv("TPGEN_FRONTIER_CHUNK", chunk)
        for g in graphs:
            st = tp.prime_paths(g, mode="count", digest=False, engine="frontier").stats
            ref = _oracle_stats(g)
            assert (st["n_paths"], st["total_vertices"], st["n_extensions"]) == \
                (ref["n_paths"], ref["total_vertices"], ref["n_extensions"]), (g.name, chunk)
            assert (st["hash_lo"], st["hash_hi"]) == (0, 0)


def test_frontier_start_ranges_add_up():
    g = gen.disjoint_union([gen.dense_scc(10, 3, 7), gen.from_arcs(3, [(0, 0), (1, 2), (2, 1)]),
                            gen.dense_scc(9, 3, 8)], name="ranges")
    whole = _frontier(g)
    assert whole == _oracle_stats(g)
    cuts = [0, 4, 10, 11, 15, g.n]
    tot = [0, 0, 0, 0, 0]
    for a, b in zip(cuts[:-1], cuts[1:]):
        part = _frontier(g, start_range=(a, b))
        assert part == _oracle_stats(g, a, b), (a, b)
        tot = [tot[0] + part["n_paths"], tot[1] + part["total_vertices"], tot[2] + part["n_extensions"],
               (tot[3] + part["digest"][0]) % 2**64, (tot[4] + part["digest"][1]) % 2**64]
    assert tot == [whole["n_paths"], whole["total_vertices"], whole["n_extensions"], *whole["digest"]]


def test_frontier_overflow_retry(monkeypatch):
    """A record buffer far too small: every call retries with a larger one until it fits."""
    monkeypatch.setenv("TPGEN_FRONTIER_CAP", "64")
    g = gen.dense_scc(13, 3, 11)
    plan = tp.Plan(g)
    st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    assert st["n_count_rounds"] >= 1
    assert {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"],
            "n_extensions": st["n_extensions"], "digest": (st["hash_lo"], st["hash_hi"])} == _oracle_stats(g)
    plan.close()


@pytest.mark.parametrize("walk", ["persistent", "graph"])
def test_frontier_dfs_chunked(monkeypatch, walk):
    """The DFS-chunked frontier (level buffers of a few hundred records, chunks of
    capacity / out-degree records, each level drained before its parent's next chunk)
    gives the oracle's counts, E_canon and digest -- walked by the persistent kernel (one
    grid barrier per chunk) and by the CUDA-graph WHILE loop (scheduler + level launch)."""
    monkeypatch.setenv("TPGEN_FRONTIER_CHUNK", "256")
    monkeypatch.setenv("TPGEN_FRONTIER_WALK", walk)
    for g in (gen.dense_scc(13, 3, 11), gen.dense_scc(16, 3, 5),
              gen.disjoint_union([gen.dense_scc(9, 3, 60), gen.from_arcs(2, [(0, 1), (1, 0)]),
                                  gen.from_arcs(1, [])], name="chunk-union")):
        st = tp.prime_paths(g, mode="count", digest=True, engine="frontier").stats
        assert st["n_count_rounds"] > st["max_scc"] + 1  # more than one chunk per level
        assert {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"],
                "n_extensions": st["n_extensions"], "digest": (st["hash_lo"], st["hash_hi"])} == \
            _oracle_stats(g), g.name


def test_frontier_rejects_wide_sccs_and_materialize():
    with pytest.raises(tp.TpgenError) as e:
        _frontier(gen.from_arcs(70, [(i, (i + 1) % 70) for i in range(70)]))  # a 70-vertex SCC
    assert e.value.status_name.endswith("INVALID_ARGUMENT")
    with pytest.raises(tp.TpgenError):
        tp.prime_paths(gen.dense_scc(8, 2, 1), engine="frontier")  # materialize: counts only


def _seg_corpus():
    """Graphs whose arcs leave SCCs: heads, tail / transit items, cross prime paths."""
    yield gen.fig1b()
    yield gen.config2()  # (a 71-vertex SCC: skipped below)
    yield gen.k_seq_loops(5, 4)
    yield gen.config4(K=30)
    yield gen.parallel_sccs(3, 24, 9)
    yield gen.parallel_sccs(2, 40, 3)  # 64-bit masks
    yield gen.config5(K=2, n=30)
    rng = np.random.default_rng(29)
    for i in range(50):
        n = int(rng.integers(2, 12))
        yield gen.random_digraph(n, float(rng.choice([0.15, 0.25, 0.35])), 900 + i, self_loops=bool(rng.random() < 0.5))


def test_frontier_with_segment_events_matches_oracle():
    """The frontier engine on graphs whose arcs leave SCCs: the segment phase and
    the prime-path phase as level-synchronous passes writing items and heads, then the count-mode
    DP and stitch -- counts, vertices, E_canon and digest equal to the oracle's; counts only too."""
    for g in _seg_corpus():
        comp = tp.components(g)[0]
        if comp.size and np.bincount(comp).max() > 64:
            continue
        ref = _oracle_stats(g)
        assert _frontier(g) == ref, g.name
        st = tp.prime_paths(g, mode="count", digest=False, engine="frontier").stats
        assert (st["n_paths"], st["total_vertices"], st["n_extensions"]) == \
            (ref["n_paths"], ref["total_vertices"], ref["n_extensions"]), g.name


def test_frontier_segment_events_dfs_chunked(monkeypatch):
    """The DFS-chunked walk (one persistent launch, per-level rings) on graphs whose arcs leave
    SCCs: forced with rings of max(256, n) records (TPGEN_FRONTIER_CHUNK), and reached by itself under a
    device-memory budget too small for one level (TPGEN_FRONTIER_BUDGET); equal to the oracle."""
    graphs = [g for g in _seg_corpus() if not (tp.components(g)[0].size and
                                               np.bincount(tp.components(g)[0]).max() > 64)]
    for g in graphs:
        monkeypatch.setenv("TPGEN_FRONTIER_CHUNK", str(max(256, g.n)))  # (a ring holds every root)
        assert _frontier(g) == _oracle_stats(g), g.name
    monkeypatch.delenv("TPGEN_FRONTIER_CHUNK")
    g = gen.config4(K=40)
    monkeypatch.setenv("TPGEN_FRONTIER_BUDGET", str(2 << 20))  # 2 MB: rings of ~2000 records per level
    plan = tp.Plan(g)
    st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    plan.close()
    assert {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"], "n_extensions": st["n_extensions"],
            "digest": (st["hash_lo"], st["hash_hi"])} == _oracle_stats(g)


@pytest.mark.timeout(1200)
def test_frontier_config5_full_size():
    """Config 5 in COUNT_HASH through the frontier engine equals the count-mode DFS (itself equal to
    the oracle for every start vertex, tests/test_gpu_count.py) and the oracle's totals."""
    tp.release_cache()  # (workspaces the earlier tests' one-shot calls keep: this test needs ~100 GB)
    g = gen.config5()
    ref = oracle.pp_stats_parallel(g, chunk=4)
    a = ref[:, :4].astype(object)
    tot = (int(a[:, 0].sum()), int(a[:, 1].sum()), int(a[:, 2].sum()) & ((1 << 64) - 1),
           int(a[:, 3].sum()) & ((1 << 64) - 1))
    plan = tp.Plan(g)
    st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    assert (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"]) == tot
    assert st["n_extensions"] == int(ref[:, 4].sum())
    plan.close()


def test_frontier_config3_full_size():
    """config 3 in the bench's launch configuration: equal to the DFS engine's count mode
    (itself bit-exact against the oracle), E_canon equal to the oracle's counter, and two
    start vertices' counts and digests equal to the oracle's."""
    g = gen.config3()
    plan = tp.Plan(g)
    f = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    d = plan.prime_paths(mode="count", digest=True).stats
    for k in ("n_paths", "total_vertices", "n_extensions", "hash_lo", "hash_hi"):
        assert f[k] == d[k], k
    # the DFS-chunked frontier at full size (4 M records per level buffer, peak level ~3.4e7)
    import os
    os.environ["TPGEN_FRONTIER_CHUNK"] = str(1 << 22)
    try:
        c = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    finally:
        del os.environ["TPGEN_FRONTIER_CHUNK"]
    assert c["n_count_rounds"] > 20 and c["gpu_launches"] <= 3  # wavefront steps walked inside one launch
    for k in ("n_paths", "total_vertices", "n_extensions", "hash_lo", "hash_hi"):
        assert c[k] == f[k], k
    n = plan.prime_paths(mode="count", digest=False, engine="frontier").stats  # counts only
    for k in ("n_paths", "total_vertices", "n_extensions"):
        assert n[k] == f[k], k
    assert f["n_extensions"] == oracle.ext_count(g)
    for s in (3, 17):
        st = plan.prime_paths(mode="count", digest=True, engine="frontier", start_range=(s, s + 1)).stats
        assert {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"],
                "n_extensions": st["n_extensions"], "digest": (st["hash_lo"], st["hash_hi"])} == \
            _oracle_stats(g, s, s + 1)
    plan.close()


def test_frontier_memory_budget_switches_to_chunks(monkeypatch):
    """A device-memory budget too small for one level (TPGEN_FRONTIER_BUDGET, bytes) makes the
    call switch to the DFS-chunked frontier by itself (the budget counts the exact
    buffer sizes); the results stay equal to the oracle's."""
    g = gen.dense_scc(14, 4, 4)
    ref = _oracle_stats(g)
    monkeypatch.setenv("TPGEN_FRONTIER_BUDGET", str(1 << 20))
    plan = tp.Plan(g)
    st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    plan.close()
    got = {"n_paths": st["n_paths"], "total_vertices": st["total_vertices"], "n_extensions": st["n_extensions"],
           "digest": (st["hash_lo"], st["hash_hi"])}
    assert got == ref
    assert st["n_count_rounds"] > 40  # many chunks, not one per level
