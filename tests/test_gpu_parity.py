"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Expected values come only from oracle/ (itself pinned by tests/test_oracle.py)."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")


def _gpu(g, **kw):
    ps = tp.prime_paths(g, digest=True, **kw)
    off, vert = ps.to_numpy()
    return off, vert, ps.stats


def _assert_same(g, **kw):
    off, vert, st = _gpu(g, **kw)
    ro, rv = oracle.prime_paths(g)
    assert off.shape == ro.shape, (g.name, off.shape, ro.shape)
    np.testing.assert_array_equal(off, ro, err_msg=g.name)
    np.testing.assert_array_equal(vert, rv, err_msg=g.name)
    assert (st["hash_lo"], st["hash_hi"]) == oracle.digest(ro, rv)
    assert st["n_extensions"] == oracle.ext_count(g), g.name
    return st


def test_fig1b_bit_exact():
    st = _assert_same(gen.fig1b())
    assert st["n_paths"] == 19 and st["total_vertices"] == 114
    assert st["n_extensions"] == 42
    assert st["n_cross"] == 8  # 2 complete + 4 exit + 2 entry


def test_random_corpus_individual():
    rng = np.random.default_rng(42)
    for i in range(120):
        n = int(rng.integers(1, 12))
        g = gen.random_digraph(n, float(rng.choice([0.1, 0.2, 0.3, 0.45])), 100 + i,
                               self_loops=bool(rng.random() < 0.5))
        _assert_same(g)


def test_random_corpus_batched_union():
    """Many small graphs as disjoint components of one call: many SCCs per launch."""
    rng = np.random.default_rng(7)
    parts = []
    for i in range(300):
        n = int(rng.integers(1, 10))
        parts.append(gen.random_digraph(n, float(rng.choice([0.15, 0.25, 0.4])), 5000 + i))
    g = gen.disjoint_union(parts, name="union300")
    _assert_same(g)


def test_multi_scc_chains():
    for seed in range(40):
        parts = [gen.random_digraph(4, 0.5, 11 * seed + j) for j in range(4)]
        u = gen.disjoint_union(parts)
        arcs = u.arcs() + [(3, 4), (7, 8), (11, 12), (1, 6), (0, 9), (5, 14)]
        _assert_same(gen.from_arcs(u.n, arcs))


@pytest.mark.parametrize("K,N", [(1, 3), (3, 3), (6, 4), (20, 5)])
def test_seq_loops(K, N):
    st = _assert_same(gen.k_seq_loops(K, N))
    assert st["n_paths"] == 1 + K * N + 2 * K + K * (K - 1) // 2


def test_config2_structured():
    _assert_same(gen.config2())


def test_config4_loop_chain():
    st = _assert_same(gen.config4())
    assert st["n_cross"] > 0.9 * st["n_paths"]


@pytest.mark.parametrize("n,d,seed", [(12, 3, 1), (16, 3, 2), (18, 3, 3), (14, 4, 4)])
def test_dense_scc_medium(n, d, seed):
    """Dense SCCs big enough to force truncation/refinement rounds."""
    st = _assert_same(gen.dense_scc(n, d, seed))
    assert st["n_units"] >= 2  # the work was split across lanes


def test_cycle_64_and_limit():
    st = _assert_same(gen.single_loop(64))
    assert st["n_paths"] == 64
    with pytest.raises(tp.TpgenError) as ei:
        tp.prime_paths(gen.single_loop(257))
    assert ei.value.status_name == "TPGEN_ERR_UNSUPPORTED"


def test_edge_cases():
    empty = gen.from_arcs(0, [])
    ps = tp.prime_paths(empty)
    assert ps.n_paths == 0 and ps.offsets.cpu().tolist() == [0]
    _assert_same(gen.from_arcs(1, []))            # isolated vertex -> <v>
    _assert_same(gen.from_arcs(1, [(0, 0)]))      # self-loop -> <v,v>
    _assert_same(gen.from_arcs(5, []))            # no arcs
    _assert_same(gen.from_arcs(3, [(0, 0), (0, 1), (1, 1), (1, 2), (2, 2)]))


def test_invalid_graph_errors():
    with pytest.raises(tp.TpgenError) as ei:
        tp.prime_paths((np.array([0, 2, 2]), np.array([1, 1])))
    assert ei.value.status_name == "TPGEN_ERR_INVALID_GRAPH"
    with pytest.raises(tp.TpgenError):
        tp.prime_paths((np.array([0, 1]), np.array([3])))


def test_shards_concatenate_to_whole():
    g = gen.disjoint_union([gen.dense_scc(12, 3, s) for s in range(4)] + [gen.config2()], name="shards")
    ro, rv = oracle.prime_paths(g)
    offs, verts = [], []
    lo_prev = 0
    for r in range(3):
        ps = tp.prime_paths(g, shard=(r, 3))
        o, v = ps.to_numpy()
        assert ps.stats["shard_lo"] == lo_prev
        lo_prev = ps.stats["shard_hi"]
        offs.append(o)
        verts.append(v)
    assert lo_prev == g.n
    cat_v = np.concatenate(verts)
    np.testing.assert_array_equal(cat_v, rv)
    cat_o = [0]
    for o in offs:
        cat_o += (o[1:] + cat_o[-1]).tolist()
    np.testing.assert_array_equal(np.asarray(cat_o), ro)


@pytest.mark.parametrize("env", [{}, {"TPGEN_NO_PRESPLIT": "1"}, {"TPGEN_NO_LEAN": "1"}],
                         ids=["lean+presplit", "lean", "generic"])
def test_dfs_kernel_variants(env, monkeypatch):
    """Graphs where no arc leaves an SCC take the LEAN DFS (rem-mask stacks) with host
    pre-split roots; the same graphs through the generic kernel must agree."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for n, d, seed in [(12, 3, 1), (16, 3, 2), (20, 3, 3), (31, 2, 4), (2, 1, 1)]:
        _assert_same(gen.dense_scc(n, d, seed))
    _assert_same(gen.disjoint_union([gen.dense_scc(10, 3, s) for s in range(6)], name="sccs6"))
    _assert_same(gen.disjoint_union([gen.dense_scc(8, 2, 1), gen.random_digraph(1, 0.0, 1)], name="scc+isolated"))


def test_lean_plan_shards_reuse_presplit_cache():
    """One Plan, several start ranges: the pre-split roots are cached per range."""
    g = gen.disjoint_union([gen.dense_scc(14, 3, s) for s in range(3)], name="lean_shards")
    ro, rv = oracle.prime_paths(g)
    plan = tp.Plan(g)
    for _ in range(2):
        verts, n_ext = [], 0
        for r in range(3):
            ps = plan.prime_paths(shard=(r, 3), digest=True)
            verts.append(ps.to_numpy()[1])
            n_ext += ps.stats["n_extensions"]
        np.testing.assert_array_equal(np.concatenate(verts), rv)
        assert n_ext == oracle.ext_count(g)
        o, v = plan.prime_paths().to_numpy()
        np.testing.assert_array_equal(o, ro)
        np.testing.assert_array_equal(v, rv)


def test_one_shot_plan_cache_detects_graph_change():
    """One-shot calls reuse the previous plan only when the CSR is byte-identical."""
    g1 = gen.dense_scc(12, 3, 1)
    t2 = np.asarray(g1.targets).copy()
    row = np.asarray(g1.offsets)
    v = 0
    succ = set(t2[row[v]:row[v + 1]].tolist())
    t2[row[v]] = next(w for w in range(1, g1.n) if w not in succ)  # same offsets, one arc moved
    t2[row[v]:row[v + 1]] = np.sort(t2[row[v]:row[v + 1]])
    g2 = gen.Graph(g1.n, np.asarray(g1.offsets), t2.astype(np.int32), g1.entry, g1.exit, "moved_arc", {})
    for g in (g1, g1, g2, g2, g1):
        _assert_same(g)


def test_host_output_and_plan_reuse():
    g = gen.config2()
    ro, rv = oracle.prime_paths(g)
    ps = tp.prime_paths(g, output="host")
    o, v = ps.to_numpy()
    np.testing.assert_array_equal(o, ro)
    np.testing.assert_array_equal(v, rv)
    plan = tp.Plan(g)
    for _ in range(3):
        o2, v2 = plan.prime_paths().to_numpy()
        np.testing.assert_array_equal(o2, ro)
        np.testing.assert_array_equal(v2, rv)
    plan.close()


def test_config3_sampled_blocks():
    """Full config 3 in the bench's launch configuration; blocks of sampled start
    vertices compared element by element, totals against the oracle's counters."""
    g = gen.config3()
    plan = tp.Plan(g)
    ps = plan.prime_paths(digest=True)
    off = ps.offsets
    vert = ps.vertices
    st = ps.stats
    assert st["n_extensions"] == oracle.ext_count(g)
    first = vert[off[:-1]].cpu().numpy()
    assert np.all(np.diff(first) >= 0)
    for s in (0, 11, 21):
        ro, rv = oracle.prime_paths(g, v_lo=s, v_hi=s + 1)
        idx = np.nonzero(first == s)[0]
        a, b = int(idx[0]), int(idx[-1]) + 1
        o = off[a:b + 1].cpu().numpy()
        np.testing.assert_array_equal(o - o[0], ro)
        np.testing.assert_array_equal(vert[o[0]:o[-1]].cpu().numpy(), rv)
    plan.close()


def test_test_paths_fig1b_and_config2():
    for g in (gen.fig1b(), gen.config2()):
        ro, rv = oracle.prime_paths(g)
        to, tv = oracle.test_paths(g, ro, rv, g.entry, g.exit)
        pp = tp.prime_paths(g)
        ts = tp.test_paths(g, g.entry, g.exit, pp)
        o, v = ts.to_numpy()
        np.testing.assert_array_equal(o, to)
        np.testing.assert_array_equal(v, tv)
        ts2 = tp.test_paths(g, g.entry, g.exit)  # computes the PPs itself
        o2, v2 = ts2.to_numpy()
        np.testing.assert_array_equal(o2, to)
        np.testing.assert_array_equal(v2, tv)


def test_test_paths_unreachable():
    g = gen.from_arcs(4, [(0, 1), (1, 0), (2, 3)])
    with pytest.raises(tp.TpgenError) as ei:
        tp.test_paths(g, 0, 1)
    assert ei.value.status_name == "TPGEN_ERR_UNREACHABLE"


@pytest.mark.timeout(900)
def test_config5_sampled_blocks_and_shards():
    """Config 5 (16 parallel 56-vertex SCCs, ~1.3e10 extensions) at full size on one GPU.

    * blocks of sampled start vertices (an SCC entry, interior vertices, an SCC
      exit, a trivial vertex with an empty block) vs the oracle, element by
      element, with their E_canon and digest;
    * COUNT_HASH over the whole graph (the one-GPU configuration: the full output
      is ~200 GB) equals the sum of 8 materialized start-vertex shards, whose
      digests add up to the count-mode digest."""
    g = gen.config5()
    plan = tp.Plan(g)
    for s in (5, 17, 205, 464, 887):
        ps = plan.prime_paths(start_range=(s, s + 1), digest=True)
        o, v = ps.to_numpy()
        ro, rv = oracle.prime_paths(g, v_lo=s, v_hi=s + 1)
        np.testing.assert_array_equal(o, ro, err_msg=f"start {s}")
        np.testing.assert_array_equal(v, rv, err_msg=f"start {s}")
        assert ps.stats["n_extensions"] == oracle.ext_count(g, v_lo=s, v_hi=s + 1)
        assert (ps.stats["hash_lo"], ps.stats["hash_hi"]) == oracle.digest(ro, rv)
        del ps
    whole = plan.prime_paths(mode="count", digest=True).stats
    tot_pp = tot_v = tot_e = 0
    h_lo = h_hi = 0
    for r in range(8):
        ps = plan.prime_paths(shard=(r, 8), digest=True)
        st = ps.stats
        tot_pp += st["n_paths"]
        tot_v += st["total_vertices"]
        tot_e += st["n_extensions"]
        h_lo = (h_lo + st["hash_lo"]) % (1 << 64)
        h_hi = (h_hi + st["hash_hi"]) % (1 << 64)
        del ps
    assert whole["n_paths"] == tot_pp and whole["total_vertices"] == tot_v
    assert whole["n_extensions"] == tot_e > 10 ** 10
    assert (whole["hash_lo"], whole["hash_hi"]) == (h_lo, h_hi)
    plan.close()


@pytest.mark.parametrize("qcap,pool", [(16, 4), (200, 64), (4096, 2)])
def test_overflow_retry_paths(monkeypatch, qcap, pool):
    """The work queue and the record pool overflow and are retried bigger (test
    hooks cap what a DFS phase may use); results stay bit-exact, including graphs
    whose segment phase and prime-path phase both overflow."""
    monkeypatch.setenv("TPGEN_TEST_QCAP", str(qcap))
    monkeypatch.setenv("TPGEN_TEST_POOL", str(pool))
    rounds = 0
    for g in (gen.fig1b(), gen.config2(), gen.config4(K=40), gen.dense_scc(14, 3, 1), gen.k_seq_loops(4, 5)):
        st = _assert_same(g)
        rounds += st["n_count_rounds"]
    assert rounds > 10  # the caps forced retries


@pytest.mark.parametrize("n,chords", [(100, [(0, 50), (70, 10)]), (150, [(0, 75), (100, 20), (40, 120)]),
                                      (230, [(5, 200), (150, 7)])])
def test_large_scc_masks(n, chords):
    """SCCs of 65-256 vertices: multi-word visited masks (W = 2, 4) and the
    sequential writer; materialized and COUNT_HASH digests agree with the oracle."""
    arcs = [(i, (i + 1) % n) for i in range(n)] + chords
    g = gen.from_arcs(n, arcs)
    st = _assert_same(g)
    cnt = tp.prime_paths(g, mode="count", digest=True).stats
    assert (cnt["n_paths"], cnt["total_vertices"], cnt["hash_lo"], cnt["hash_hi"]) == \
        (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"])


def test_count_mode_digest_matches_oracle():
    """COUNT_HASH (hash-mode writers, no output) gives the oracle's counts and digest on
    graphs with segment items and head blocks (mixed batches) and without."""
    rng = np.random.default_rng(7)
    graphs = [gen.fig1b(), gen.config2(), gen.config4(K=40), gen.dense_scc(14, 3, 1), gen.k_seq_loops(4, 5)]
    graphs += [gen.random_digraph(int(rng.integers(3, 10)), 0.3, 900 + i) for i in range(20)]
    for g in graphs:
        ro, rv = oracle.prime_paths(g)
        st = tp.prime_paths(g, mode="count", digest=True).stats
        assert st["n_paths"] == len(ro) - 1, g.name
        assert st["total_vertices"] == int(ro[-1]), g.name
        assert (st["hash_lo"], st["hash_hi"]) == oracle.digest(ro, rv), g.name
        assert st["n_extensions"] == oracle.ext_count(g), g.name


def test_test_paths_config4():
    g = gen.config4(K=40)
    ro, rv = oracle.prime_paths(g)
    to, tv = oracle.test_paths(g, ro, rv, g.entry, g.exit)
    ts = tp.test_paths(g, g.entry, g.exit)
    o, v = ts.to_numpy()
    np.testing.assert_array_equal(o, to)
    np.testing.assert_array_equal(v, tv)


def test_long_paths_and_many_sccs():
    """Paths far longer than one SCC (a 20000-vertex chain: one prime path of 20000
    vertices, stitched from 20000 one-vertex segments), 2^16 source-sink paths of a
    ladder DAG, and a chain of 3000 three-cycles (many small SCCs)."""
    n = 20000
    _assert_same(gen.from_arcs(n, [(i, i + 1) for i in range(n - 1)]))
    k = 16  # ladder: i -> (i+1 top, i+1 bottom) for both rails
    arcs = []
    for i in range(k):
        for a in (2 * i, 2 * i + 1):
            arcs += [(a, 2 * i + 2), (a, 2 * i + 3)]
    st = _assert_same(gen.from_arcs(2 * k + 2, arcs))
    assert st["n_paths"] == 2 * 2 ** k  # 2 sources x 2^k rail choices (each ending in one of the 2 sinks)
    arcs = []
    for c in range(3000):
        b = 3 * c
        arcs += [(b, b + 1), (b + 1, b + 2), (b + 2, b)]
        if c + 1 < 3000:
            arcs.append((b + 2, b + 3))
    _assert_same(gen.from_arcs(9000, arcs))


def test_plan_test_paths():
    """tpgen_plan_test_paths (the plan's graph, no re-planning) equals the oracle, with the
    prime paths given (device) or computed by the call."""
    for g in (gen.fig1b(), gen.config2(), gen.config4(K=30)):
        ro, rv = oracle.prime_paths(g)
        to, tv = oracle.test_paths(g, ro, rv, g.entry, g.exit)
        plan = tp.Plan(g)
        for pin in (plan.prime_paths(), None):
            o, v = plan.test_paths(g.entry, g.exit, pin).to_numpy()
            np.testing.assert_array_equal(o, to, err_msg=g.name)
            np.testing.assert_array_equal(v, tv, err_msg=g.name)
        plan.close()


def test_pp_class_report():
    """tpgen_plan_classify (five-class report, R19) equals the oracle's per-path
    classification, for device and host prime-path lists."""
    rng = np.random.default_rng(3)
    graphs = [gen.fig1b(), gen.k_seq_loops(5, 3), gen.config2(), gen.config4(K=40)]
    graphs += [gen.random_digraph(int(rng.integers(4, 10)), 0.3, 700 + i) for i in range(10)]
    for g in graphs:
        start = g.entry if g.entry >= 0 else 0
        end = g.exit if g.exit >= 0 else g.n - 1
        ro, rv = oracle.prime_paths(g)
        _, want = oracle.pp_classes(g, ro, rv, start, end)
        plan = tp.Plan(g)
        ps = plan.prime_paths()
        assert plan.classify(ps, start, end) == want, g.name
        host = tp.PathSet(ro, rv, len(ro) - 1, False, {})
        assert plan.classify(host, start, end) == want, g.name
        plan.close()


def test_greedy_test_path_cover():
    """TPGEN_TP_GREEDY (host greedy cover with linear-time marking) equals the oracle's
    plain greedy cover (naive containment scans), element by element."""
    for g in (gen.fig1b(), gen.config2(), gen.k_seq_loops(4, 3), gen.k_nested_if(5), gen.config4(K=12)):
        ro, rv = oracle.prime_paths(g)
        to, tv = oracle.greedy_test_paths(g, ro, rv, g.entry, g.exit)
        o, v = tp.test_paths(g, g.entry, g.exit, cover="greedy").to_numpy()
        np.testing.assert_array_equal(o, to, err_msg=g.name)
        np.testing.assert_array_equal(v, tv, err_msg=g.name)
        plan = tp.Plan(g)
        o2, v2 = plan.test_paths(g.entry, g.exit, plan.prime_paths(), cover="greedy").to_numpy()
        np.testing.assert_array_equal(o2, to, err_msg=g.name)
        np.testing.assert_array_equal(v2, tv, err_msg=g.name)
        plan.close()


def test_sharded_prime_paths_nccl_single_rank():
    """The distributed helper on the real path (NCCL, world size 1 on cuda:0): the block
    is the whole list, totals and digest match the oracle."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2210_16998_b200.distributed import sharded_prime_paths

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        g = gen.config2()
        res = sharded_prime_paths(g)
        ro, rv = oracle.prime_paths(g)
        o, v = res.paths.to_numpy()
        np.testing.assert_array_equal(o, ro)
        np.testing.assert_array_equal(v, rv)
        assert res.pp_base == 0 and res.vertex_base == 0 and res.n_paths == len(ro) - 1
        assert res.digest == oracle.digest(ro, rv)
        g = gen.dense_scc(14, 3, 9)  # the frontier engine's count mode through the same exchange
        res = sharded_prime_paths(g, mode="count", engine="frontier")
        ro, rv = oracle.prime_paths(g)
        assert res.n_paths == len(ro) - 1 and res.total_vertices == int(ro[-1])
        assert res.n_extensions == oracle.ext_count(g) and res.digest == oracle.digest(ro, rv)
    finally:
        dist.destroy_process_group()
