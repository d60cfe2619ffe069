"""Pins for the CPU oracle (oracle/) against things other than itself.

Every expected value here comes from the paper (cited), a closed form, a
textbook special case, or brute force on tiny inputs -- never from the oracle
under test or from the CUDA path.
"""
import itertools

import numpy as np
import pytest

import oracle
from oracle import brute
from tests.conftest import load_golden
from workloads import generators as gen


def _pp_list(g, **kw):
    off, vert = oracle.prime_paths(g, **kw)
    return oracle.as_list(off, vert)


# --------------------------------------------------------------- worked example
def test_fig1b_prime_paths_equal_paper():
    """the 19 PPs quoted in the paper."""
    rows = load_golden("fig1b_prime_paths.txt")
    paper = sorted(p for _, p in rows)
    assert len(paper) == 19  # P:255 "we reach 19 PPs"
    got = _pp_list(gen.fig1b())
    assert got == paper  # same set, and oracle order is lexicographic
    assert got == sorted(got)


def test_fig1b_class_counts():
    """11 internal, 2 complete, 4 exit, 2 entry."""
    rows = load_golden("fig1b_prime_paths.txt")
    counts = {}
    for tag, _ in rows:
        counts[tag] = counts.get(tag, 0) + 1
    assert counts == {"internal": 11, "complete": 2, "exit": 4, "entry": 2}


def test_fig1b_tier0_equals_paper():
    rows = load_golden("fig1b_prime_paths.txt")
    g = gen.fig1b()
    assert brute.prime_paths(g.n, brute.graph_succ(g)) == sorted(p for _, p in rows)


def test_fig1b_graph_matches_paper_counts():
    """E = 13, V = 11, CC = 13 - 11 + 2 = 4."""
    g = gen.fig1b()
    assert (g.n, g.m, g.m - g.n + 2) == (11, 13, 4)


def test_fig1b_scc():
    """Fig. 2(a) / P:150: the one nontrivial SCC is {2,3,4,5,6,8}."""
    lab = oracle.scc_labels(gen.fig1b())
    members = [v for v in range(11) if lab[v] == lab[2]]
    assert members == [2, 3, 4, 5, 6, 8]
    assert len(set(lab.tolist())) == 6  # that SCC + 5 singletons


def test_fig1b_ext_count():
    """E_canon on Fig. 1(b) = 42: the per-start counts 8,9,6,6,6,7 are brute-forced here."""
    g = gen.fig1b()
    scc = {2, 3, 4, 5, 6, 8}
    succ = brute.graph_succ(g)
    sp = brute.simple_paths(g.n, [[w for w in succ[v] if w in scc and v in scc] for v in range(g.n)])
    per = {s: sum(1 for p in sp if p[0] == s and len(p) >= 2) for s in scc}
    assert per == {2: 8, 3: 9, 4: 6, 5: 6, 6: 6, 8: 7}
    assert oracle.ext_count(g) == 42 == sum(per.values())


def test_fig1b_segments_reading(golden):
    """DESIGN.md reading R8/R9 reproduce the paper's intermediate path sets:
    head = non-entry first, pred(first) within path, last an exit;
    transit = entry first, exit last (all acyclic simple paths, Def. 6);
    tail = entry first, succ(last) within path."""
    g = gen.fig1b()
    rows = golden("fig1b_segments.txt")
    scc = set(dict(rows)["scc"])
    succ = brute.graph_succ(g)
    pred = [[u for u in range(g.n) if v in succ[u]] for v in range(g.n)]
    entries = {v for v in scc if any(u not in scc for u in pred[v])}
    exits = {v for v in scc if any(w not in scc for w in succ[v])}
    assert sorted(entries) == list(dict(rows)["entries"])
    assert sorted(exits) == list(dict(rows)["exits"])
    inner = [[w for w in succ[v] if w in scc] if v in scc else [] for v in range(g.n)]
    paths = [p for p in brute.simple_paths(g.n, inner)
             if p[0] in scc and not (len(p) > 1 and p[0] == p[-1])]
    head = sorted(p for p in paths if p[0] not in entries and set(pred[p[0]]) <= set(p) and p[-1] in exits)
    transit = sorted(p for p in paths if p[0] in entries and p[-1] in exits)
    tail = sorted(p for p in paths if p[0] in entries and set(succ[p[-1]]) <= set(p))
    assert head == sorted(p for t, p in rows if t == "head")
    assert transit == sorted(p for t, p in rows if t == "transit")
    assert tail == sorted(p for t, p in rows if t == "tail")


# ---------------------------------------------------------- closed forms
@pytest.mark.parametrize("K", [1, 2, 3, 4, 5])
def test_nested_if_closed_form(K):
    """K nested if-then -> K+1 prime paths."""
    assert len(_pp_list(gen.k_nested_if(K))) == K + 1


@pytest.mark.parametrize("K", [1, 2, 3, 4, 6, 8])
def test_seq_if_closed_form(K):
    """K if-then in sequence -> 2^K prime paths."""
    assert len(_pp_list(gen.k_seq_if(K))) == 2 ** K


@pytest.mark.parametrize("K", [1, 2, 3, 5, 9])
def test_single_loop_closed_form(K):
    """a single loop of length K -> K prime paths (one rotation per vertex);
    E_canon = K^2 (K starts x K-1 acyclic extensions + 1 closure)."""
    g = gen.single_loop(K)
    pps = _pp_list(g)
    assert len(pps) == K
    assert all(p[0] == p[-1] and len(p) == K + 1 for p in pps)
    assert oracle.ext_count(g) == K * K


@pytest.mark.parametrize("K,N,expect", [(1, 3, 6), (2, 3, 12), (3, 3, 19), (3, 2, 16), (4, 3, 27)])
def test_seq_loops_count(K, N, expect):
    """K loops in sequence: 1 complete + K*N internal + K exit + K entry + K(K-1)/2 SCC->SCC.
    (The paper's K((N+1)+(K-1)/2) at P:636 is wrong -- DESIGN.md reading R7.)
    Cross-checked against tier-0 brute force where it is small enough."""
    g = gen.k_seq_loops(K, N)
    assert 1 + K * N + 2 * K + K * (K - 1) // 2 == expect
    pps = _pp_list(g)
    assert len(pps) == expect
    if g.n <= 11:
        assert pps == brute.prime_paths(g.n, brute.graph_succ(g))


def _count_st_paths(g):
    """#Start->End paths of a DAG by memoised recursion (Npath for DAGs)."""
    memo = {}

    def f(v):
        if v == g.exit:
            return 1
        if v not in memo:
            memo[v] = sum(f(int(w)) for w in g.succ(v))
        return memo[v]

    return f(g.entry)


@pytest.mark.parametrize("seed", range(12))
def test_dag_pp_equals_npath(seed):
    """for acyclic CFGs the PP count equals the Npath complexity (= #Start->End paths
    when every vertex lies on such a path), and every PP is a Start->End path."""
    g = gen.random_dag_cfg(8 + seed, seed)
    pps = _pp_list(g)
    assert len(pps) == _count_st_paths(g)
    assert all(p[0] == g.entry and p[-1] == g.exit for p in pps)


# ------------------------------------------------------- tier-0 equivalence corpus
def _corpus(count, seed0=1000):
    rng = np.random.default_rng(seed0)
    for i in range(count):
        n = int(rng.integers(1, 9))
        p = float(rng.choice([0.12, 0.2, 0.3, 0.4]))
        yield gen.random_digraph(n, p, seed0 + i, self_loops=bool(rng.random() < 0.5))


def test_tier1_equals_tier0_random_corpus():
    """Def. 1 brute force vs the DFS oracle (with and without the exact prunes A', B)."""
    total = 0
    for g in _corpus(700):
        ref = brute.prime_paths(g.n, brute.graph_succ(g))
        assert _pp_list(g, prunes=True) == ref, g.name
        assert _pp_list(g, prunes=False) == ref, g.name
        total += len(ref)
    assert total > 3000


def test_tier1_equals_tier0_multi_scc():
    """Chains of small SCCs (exercise SCC->SCC prime paths and prunes)."""
    for seed in range(60):
        parts = [gen.random_digraph(3, 0.5, 7 * seed + j) for j in range(3)]
        u = gen.disjoint_union(parts)
        arcs = u.arcs() + [(2, 3), (5, 6), (1, 4), (0, 7)]
        g = gen.from_arcs(u.n, arcs)
        assert _pp_list(g) == brute.prime_paths(g.n, brute.graph_succ(g))


def test_ext_count_matches_bruteforce():
    for g in _corpus(200, seed0=5000):
        lab = oracle.scc_labels(g)
        succ = brute.graph_succ(g)
        cnt = 0
        for s in range(g.n):
            comp = {v for v in range(g.n) if lab[v] == lab[s]}
            nontriv = len(comp) > 1 or s in succ[s]
            if not nontriv:
                continue
            inner = [[w for w in succ[v] if w in comp] if v in comp else [] for v in range(g.n)]
            cnt += sum(1 for p in brute.simple_paths(g.n, inner) if p[0] == s and len(p) >= 2)
        assert oracle.ext_count(g) == cnt


def test_scc_labels_mutual_reachability():
    for g in _corpus(100, seed0=9000):
        lab = oracle.scc_labels(g)
        succ = brute.graph_succ(g)
        reach = []
        for a in range(g.n):
            seen, st = {a}, [a]
            while st:
                v = st.pop()
                for w in succ[v]:
                    if w not in seen:
                        seen.add(w)
                        st.append(w)
            reach.append(seen)
        for a, b in itertools.product(range(g.n), repeat=2):
            assert (lab[a] == lab[b]) == (b in reach[a] and a in reach[b])


# ------------------------------------------------------------------ invariants
def test_invariants_simple_antichain_coverage():
    """Every PP is simple; no PP is a proper subpath of another; every simple path is a
    contiguous subpath of some PP (north_star invariants)."""
    for g in _corpus(150, seed0=7000):
        pps = _pp_list(g)
        pset = set(pps)
        for p in pps:
            body = p[:-1] if len(p) > 1 and p[0] == p[-1] else p
            assert len(set(body)) == len(body)
            for i in range(len(p)):
                for j in range(i + 1, len(p) + 1):
                    if j - i < len(p):
                        assert p[i:j] not in pset
        subs = set()
        for p in pps:
            for i in range(len(p)):
                for j in range(i + 1, len(p) + 1):
                    subs.add(p[i:j])
        for sp in brute.simple_paths(g.n, brute.graph_succ(g)):
            assert sp in subs


def test_lexicographic_order_and_blocks():
    g = gen.config2()
    off, vert = oracle.prime_paths(g)
    pps = oracle.as_list(off, vert)
    assert pps == sorted(pps)
    # per-start-vertex blocks concatenate to the whole list
    parts = []
    for lo, hi in [(0, 10), (10, 31), (31, g.n)]:
        parts += _pp_list(g, v_lo=lo, v_hi=hi)
    assert parts == pps


# ---------------------------------------------------------------------- digest
def test_digest_order_independent_and_sensitive():
    g = gen.fig1b()
    off, vert = oracle.prime_paths(g)
    d = oracle.digest(off, vert)
    pps = oracle.as_list(off, vert)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(pps))
    pv = [pps[i] for i in perm]
    off2 = np.cumsum([0] + [len(p) for p in pv]).astype(np.int64)
    vert2 = np.asarray([v for p in pv for v in p], dtype=np.int32)
    assert oracle.digest(off2, vert2) == d
    vert3 = vert2.copy()
    vert3[3] ^= 1
    assert oracle.digest(off2, vert3) != d
    # splitting one path differently changes the digest (length is hashed)
    off4 = off2.copy()
    off4[1] += 1
    assert oracle.digest(off4, vert2) != d


# ------------------------------------------------------------------ test paths
def test_tp_tables_are_lexmin_shortest_walks():
    """The prefix/suffix rule (R15) equals 'lexicographically smallest among
    minimum-hop walks', checked by brute force on tiny graphs."""
    checks = 0
    for g in _corpus(150, seed0=3000):
        if g.n < 2:
            continue
        succ = brute.graph_succ(g)
        entry, exit_ = 0, g.n - 1
        pre, suf = oracle.tp_tables(g, entry, exit_)
        for v in range(g.n):
            assert pre[v] == brute.lexmin_shortest_walk(succ, entry, v)
            assert suf[v] == brute.lexmin_shortest_walk(succ, v, exit_)
            checks += 2
    assert checks > 1000


def test_fig1b_test_paths():
    """S:536 example: PP <8,2,3,4,8> -> TP <S,1,2,3,4,8,2,3,4,8,2,9,E>; every TP runs
    entry->exit along arcs and contains its PP; 19 aligned, 10 distinct."""
    g = gen.fig1b()
    off, vert = oracle.prime_paths(g)
    toff, tvert = oracle.test_paths(g, off, vert, g.entry, g.exit)
    pps = oracle.as_list(off, vert)
    tps = oracle.as_list(toff, tvert)
    assert len(tps) == 19
    assert tps[pps.index((8, 2, 3, 4, 8))] == (0, 1, 2, 3, 4, 8, 2, 3, 4, 8, 2, 9, 10)
    arcs = set(g.arcs())
    for p, t in zip(pps, tps):
        assert t[0] == g.entry and t[-1] == g.exit
        assert all((a, b) in arcs for a, b in zip(t[:-1], t[1:]))
        assert any(t[i:i + len(p)] == p for i in range(len(t) - len(p) + 1))
    assert len(set(tps)) == 10


def test_fig1b_pp_classes_match_paper():
    """Every one of the 19 PPs gets the class the paper prints for it."""
    rows = load_golden("fig1b_prime_paths.txt")
    tag = {tuple(p): t for t, p in rows}
    g = gen.fig1b()
    off, vert = oracle.prime_paths(g)
    labels, counts = oracle.pp_classes(g, off, vert, g.entry, g.exit)
    for i, lab in enumerate(labels):
        p = tuple(int(v) for v in vert[off[i]:off[i + 1]])
        assert tag[p] == lab, (p, tag[p], lab)
    assert counts == {"complete": 2, "entry": 2, "exit": 4, "internal": 11, "transit": 0}


@pytest.mark.parametrize("K,N", [(1, 3), (3, 3), (4, 2), (6, 3)])
def test_seq_loops_pp_classes(K, N):
    """K loops in sequence (R7): 1 complete, K*N internal, K exit, K entry and
    K(K-1)/2 SCC->SCC transit prime paths."""
    g = gen.k_seq_loops(K, N)
    off, vert = oracle.prime_paths(g)
    _, counts = oracle.pp_classes(g, off, vert, g.entry, g.exit)
    assert counts == {"complete": 1, "entry": K, "exit": K, "internal": K * N, "transit": K * (K - 1) // 2}


def _check_greedy_cover(g):
    off, vert = oracle.prime_paths(g)
    pps = oracle.as_list(off, vert)
    to, tv = oracle.greedy_test_paths(g, off, vert, g.entry, g.exit)
    tps = oracle.as_list(to, tv)
    succ = {v: set(g.succ(v).tolist()) for v in range(g.n)}
    for t in tps:  # entry -> exit walks along arcs
        assert t[0] == g.entry and t[-1] == g.exit
        assert all(b in succ[a] for a, b in zip(t, t[1:]))
    for q in pps:  # every prime path is covered
        assert any(oracle._contains(list(t), list(q)) for t in tps), q
    # the seeds: the longest uncovered PP at each step, in order; never more TPs than PPs
    assert len(tps) <= len(pps)
    return pps, tps


def test_greedy_cover_fig1b():
    """Fig. 1(b): every PP covered by entry->exit walks; the first TP extends the first
    (lexicographically) of the longest PPs, <Start,1,2,3,5,6,8> (length 7), and
    also covers the exit PP <3,5,6,8,2,9,End>; fewer TPs than the 19 per-PP ones."""
    pps, tps = _check_greedy_cover(gen.fig1b())
    assert tps[0] == (0, 1, 2, 3, 5, 6, 8, 2, 9, 10)
    assert len(tps) < len(pps)


def test_greedy_cover_dag_is_identity():
    """In a DAG with one source and one sink every PP is a complete Start->End path
    (P:604): each is its own TP, in length-then-lexicographic order."""
    for K in (3, 5):
        g = gen.k_seq_if(K)
        off, vert = oracle.prime_paths(g)
        to, tv = oracle.greedy_test_paths(g, off, vert, g.entry, g.exit)
        pps = oracle.as_list(off, vert)
        tps = oracle.as_list(to, tv)
        assert sorted(tps) == sorted(pps)
        assert [len(t) for t in tps] == sorted((len(p) for p in pps), reverse=True)


def test_greedy_cover_invariants():
    for g in (gen.config2(), gen.k_seq_loops(3, 3), gen.k_nested_if(4)):
        _check_greedy_cover(g)


# ---------------------------------------------------------------- K7: sorted-unique test paths
def _is_subpath(t, q):  # (plain scan written here, independent of the oracle's helpers)
    return any(list(t[i:i + len(q)]) == list(q) for i in range(len(t) - len(q) + 1))


def _check_unique(g):
    off, vert = oracle.prime_paths(g)
    uo, uv = oracle.unique_test_paths(g, off, vert, g.entry, g.exit)
    tps = oracle.as_list(uo, uv)
    arcs = {(u, int(w)) for u in range(g.n) for w in g.targets[g.offsets[u]:g.offsets[u + 1]]}
    for t in tps:  # entry -> exit walks along arcs
        assert t[0] == g.entry and t[-1] == g.exit
        assert all((t[i], t[i + 1]) in arcs for i in range(len(t) - 1))
    for a, b in zip(tps, tps[1:]):  # strictly increasing: sorted, no duplicates
        assert tuple(a) < tuple(b)
    for p in oracle.as_list(off, vert):  # "the set of TPs covering all PPs"
        assert any(_is_subpath(t, p) for t in tps), p
    return oracle.as_list(off, vert), tps


def test_unique_test_paths_fig1b():
    """Fig. 1(b): the 19 per-PP test paths collapse to 10 distinct ones (SURVEY §8(d),
    config 1: "19 TPs (10 unique)"), each an entry->exit walk, together covering all 19 PPs."""
    pps, tps = _check_unique(gen.fig1b())
    assert len(pps) == 19 and len(tps) == 10


def test_unique_test_paths_dag_are_the_prime_paths():
    """One-source one-sink DAG: every PP is a complete Start->End path and is its own
    test path, so the unique set is the PP list itself (already in lexicographic order)."""
    for K in (3, 5):
        g = gen.k_seq_if(K)
        pps, tps = _check_unique(g)
        assert tps == pps and len(tps) == 2 ** K


def test_unique_test_paths_invariants():
    for g in (gen.config2(), gen.k_seq_loops(3, 3), gen.k_nested_if(4), gen.config4(K=6)):
        _check_unique(g)


# ---------------------------------------------------------------- digest (R20)
def _flat(paths):
    off = np.zeros(len(paths) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(p) for p in paths])
    vert = np.asarray([v for p in paths for v in p], dtype=np.int32)
    return off, vert


def _dig(paths):
    return oracle.digest(*_flat(paths))


def test_digest_order_independent_and_additive():
    """The set digest is a sum over paths: any order, and shards add up (mod 2^64)."""
    rng = np.random.default_rng(3)
    paths = [list(rng.integers(0, 50, size=int(rng.integers(1, 12)))) for _ in range(200)]
    whole = _dig(paths)
    perm = [paths[i] for i in rng.permutation(len(paths))]
    assert _dig(perm) == whole
    a, b = _dig(paths[:77]), _dig(paths[77:])
    assert ((a[0] + b[0]) % 2**64, (a[1] + b[1]) % 2**64) == whole
    assert _dig([]) == (0, 0)


def test_digest_sensitive_to_vertices_order_and_binding():
    """A changed vertex, a reorder inside a path, a rotation, and two paths that swap
    their suffixes (same multiset of (position, vertex) pairs) all change the digest."""
    p, q = [3, 1, 4, 1, 5], [9, 2, 6, 5, 3]
    base = _dig([p, q])
    assert _dig([[3, 1, 4, 1, 6], q]) != base
    assert _dig([[1, 3, 4, 1, 5], q]) != base
    assert _dig([[1, 4, 1, 5, 3], q]) != base
    assert _dig([[3, 1, 6, 5, 3], [9, 2, 4, 1, 5]]) != base  # suffixes swapped at position 2
    assert _dig([p + [7], q]) != base and _dig([p[:-1], q]) != base
    assert _dig([p]) != _dig([p, p])  # multiplicity counts


# ------------------------------------------------- per-start statistics (streamed)
def _stats_graphs():
    gs = [gen.fig1b(), gen.config2(), gen.k_seq_loops(3, 3), gen.k_nested_if(4), gen.config4(K=12),
          gen.dense_scc(9, 3, 2)]
    gs += [g for g in _corpus(60, seed0=9100)]
    return gs


def test_pp_stats_equal_materialized_blocks():
    """oracle_pp_stats (prime paths hashed while enumerated, nothing stored) equals, per
    start vertex, the count, vertex total and digest of the materialized block
    (oracle_prime_paths, pinned above) -- the streaming comparison of SURVEY 8(d)."""
    for g in _stats_graphs():
        st = oracle.pp_stats(g)
        for v in range(g.n):
            o, vv = oracle.prime_paths(g, v_lo=v, v_hi=v + 1)
            assert (int(st[v, 0]), int(st[v, 1])) == (len(o) - 1, int(o[-1])), (g.name, v)
            assert (int(st[v, 2]), int(st[v, 3])) == oracle.digest(o, vv), (g.name, v)
        o, vv = oracle.prime_paths(g)
        lo, hi = oracle.digest(o, vv)
        assert (int(st[:, 2].sum(dtype=np.uint64)), int(st[:, 3].sum(dtype=np.uint64))) == (lo, hi)


def test_tp_stats_equal_materialized_test_paths():
    """oracle_tp_stats hashes every prime path's test path (R15) as it is formed: per start
    vertex equal to the materialized test paths (oracle.test_paths, pinned by the brute-force
    lexmin walks and the S:536 example above) of that start's prime paths."""
    for g in (gen.fig1b(), gen.config2(), gen.k_seq_loops(3, 3), gen.config4(K=8)):
        st = oracle.pp_stats(g, tp=(g.entry, g.exit))
        for v in range(g.n):
            o, vv = oracle.prime_paths(g, v_lo=v, v_hi=v + 1)
            to, tv = oracle.test_paths(g, o, vv, g.entry, g.exit)
            assert (int(st[v, 0]), int(st[v, 1])) == (len(to) - 1, int(to[-1])), (g.name, v)
            assert (int(st[v, 2]), int(st[v, 3])) == oracle.digest(to, tv), (g.name, v)
    g = gen.from_arcs(4, [(0, 1), (1, 0), (2, 3)])  # vertices 2, 3 unreachable from entry 0
    with pytest.raises(ValueError):
        oracle.pp_stats(g, tp=(0, 1))


def test_pp_stats_parallel_equals_serial():
    g = gen.config2()
    par = oracle.pp_stats_parallel(g, procs=3, chunk=7)
    assert np.array_equal(par[:, :4], oracle.pp_stats(g))
    assert [int(x) for x in par[:, 4]] == [oracle.ext_count(g, v, v + 1) for v in range(g.n)]
    assert int(par[:, 4].sum()) == oracle.ext_count(g)
    assert np.array_equal(oracle.pp_stats_parallel(g, 5, 40, tp=(g.entry, g.exit), procs=2, chunk=3)[:, :4],
                          oracle.pp_stats(g, 5, 40, tp=(g.entry, g.exit)))


def test_digest_single_vertex_and_cycle_closed_forms():
    """Closed forms of R20 (S = sum_i mix(v_i)(2i+1)): a path <v> and its repetition
    <v, v> differ only by the weight of the second position, so for every v the two
    digests differ; a K-cycle's K rotations are K distinct paths with K distinct digests."""
    ones = [_dig([[v]]) for v in range(50)]
    assert len(set(ones)) == 50
    assert all(_dig([[v]]) != _dig([[v, v]]) for v in range(50))
    K = 7
    rot = [[(i + j) % K for j in range(K)] + [i] for i in range(K)]
    assert len({_dig([r]) for r in rot}) == K


# ---------------------------------------------------------------- Npath (NEXT #3)
def test_npath_closed_forms():
    """Npath of the paper's examples: 4 for Fig. 1(b) (the loop body runs at
    most once: <S,1,2,9,E>, <S,..,3,4,8,2,9,E>, <S,..,3,5,6,8,2,9,E>, <S,..,3,5,7,E>);
    K sequential if-then-else: 2^K; a DAG: the number of start -> end paths."""
    g = gen.fig1b()
    assert brute.npath(g.n, brute.graph_succ(g), g.entry, g.exit) == 4
    for K in (1, 3, 5):
        g = gen.k_seq_if(K)
        assert brute.npath(g.n, brute.graph_succ(g), g.entry, g.exit) == 2 ** K
    for seed in range(4):
        g = gen.random_dag_cfg(8 + seed, seed)
        assert brute.npath(g.n, brute.graph_succ(g), g.entry, g.exit) == _count_st_paths(g)
