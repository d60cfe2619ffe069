"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/tpgen.h declares, and its host-only component-graph entry point
(tpgen_components) matches the definitions (Defs. 3-5 P:137-156)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from oracle import brute
from tests.conftest import ROOT
from workloads import generators as gen

import paper_2210_16998_b200 as tp
from paper_2210_16998_b200 import _abi


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "tpgen.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(tpgen_[a-z0-9_]+)\s*\(", src))
    return {n for n in names if not n.endswith("_fn")}


def test_library_exports_every_declared_symbol():
    lib = tp.library()
    declared = _declared_functions()
    assert declared == set(_abi.SYMBOLS), declared ^ set(_abi.SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tpgen_\w+)", out))
    assert declared <= exported


def test_version_and_status_strings():
    lib = tp.library()
    assert b"sm_100a" in lib.tpgen_version()
    for code in range(9):
        assert lib.tpgen_status_string(code)


def test_abi_struct_sizes_match_header():
    """The ctypes mirror must match the C layout (compiled probe, no GPU)."""
    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "tpgen.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(tpgen_options), sizeof(tpgen_stats), sizeof(tpgen_paths),
 offsetof(tpgen_stats, ms_plan), offsetof(tpgen_options, host_out), offsetof(tpgen_options, engine),
 offsetof(tpgen_options, shard_prefix), offsetof(tpgen_stats, unit_lo), offsetof(tpgen_options, prune));return 0;}
'''
    tmpd = os.path.join(ROOT, "build")
    os.makedirs(tmpd, exist_ok=True)
    c = os.path.join(tmpd, "abi_probe.c")
    exe = os.path.join(tmpd, "abi_probe")
    open(c, "w").write(probe)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
    vals = [int(x) for x in subprocess.check_output([exe]).split()]
    assert vals == [ctypes.sizeof(_abi.Options), ctypes.sizeof(_abi.Stats), ctypes.sizeof(_abi.Paths),
                    _abi.Stats.ms_plan.offset, _abi.Options.host_out.offset, _abi.Options.engine.offset,
                    _abi.Options.shard_prefix.offset, _abi.Stats.unit_lo.offset, _abi.Options.prune.offset]


def _corpus(count, seed0):
    rng = np.random.default_rng(seed0)
    for i in range(count):
        n = int(rng.integers(1, 12))
        yield gen.random_digraph(n, float(rng.choice([0.1, 0.2, 0.35])), seed0 + i)


def test_components_match_definitions():
    graphs = list(_corpus(200, 11)) + [gen.fig1b(), gen.config2(), gen.config4()]
    for g in graphs:
        comp, flags, nscc = tp.components(g)
        lab = oracle.scc_labels(g)
        # same partition as mutual reachability
        for a in range(g.n):
            for b in range(g.n):
                assert (comp[a] == comp[b]) == (lab[a] == lab[b])
        assert nscc == len(set(comp.tolist()))
        succ = brute.graph_succ(g)
        for v in range(g.n):
            size = int((comp == comp[v]).sum())
            entry = any(comp[u] != comp[v] for u in range(g.n) if v in succ[u])
            exit_ = any(comp[w] != comp[v] for w in succ[v])
            nontriv = size > 1 or v in succ[v]
            assert flags[v] == (1 if entry else 0) | (2 if exit_ else 0) | (4 if nontriv else 0)
            for w in succ[v]:  # reverse topological ids
                assert comp[w] <= comp[v]


def test_components_fig1b():
    comp, flags, nscc = tp.components(gen.fig1b())
    scc = [v for v in range(11) if comp[v] == comp[2]]
    assert scc == [2, 3, 4, 5, 6, 8] and nscc == 6
    assert [v for v in scc if flags[v] & 1] == [2]
    assert [v for v in scc if flags[v] & 2] == [2, 5]


@pytest.mark.parametrize("so,st,n,code", [
    ([1, 1], [0], 1, 2),             # offsets[0] != 0
    ([0, 2, 1], [1, 0], 2, 2),       # decreasing
    ([0, 1], [5], 1, 2),             # target out of range
    ([0, 2, 2], [1, 1], 2, 2),       # duplicate arc
])
def test_components_rejects_invalid_graphs(so, st, n, code):
    with pytest.raises(tp.TpgenError) as ei:
        tp.components((np.asarray(so), np.asarray(st)))
    assert ei.value.status == code


def test_compute_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        tp.prime_paths(gen.fig1b())


def test_frontier_engine_option_checks():
    """TPGEN_ENGINE_FRONTIER computes counts + digest only; the option checks run before
    any device work (include/tpgen.h tpgen_options.engine)."""
    lib = tp.library()
    g = gen.fig1b()
    so, st = g.offsets, g.targets
    for engine, mode in ((_abi.ENGINE_FRONTIER, _abi.OUT_MATERIALIZE), (7, _abi.OUT_COUNT_HASH)):
        o = _abi.Options()
        lib.tpgen_options_init(ctypes.byref(o))
        assert o.engine == _abi.ENGINE_DFS
        o.engine, o.output_mode = engine, mode
        paths, stats = _abi.Paths(), _abi.Stats()
        r = lib.tpgen_prime_paths(so.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), g.n, ctypes.byref(o),
                                  ctypes.byref(paths), ctypes.byref(stats))
        assert r == 1  # TPGEN_ERR_INVALID_ARGUMENT
        assert paths.n_paths == 0
    with pytest.raises(ValueError):
        tp.prime_paths(g, mode="count", engine="bfs")
    for engine, mode in ((_abi.ENGINE_DFS, _abi.OUT_MATERIALIZE), (_abi.ENGINE_FRONTIER, _abi.OUT_COUNT_HASH)):
        o = _abi.Options()  # pruning (NEXT #2): the DFS engine's COUNT_HASH mode only
        lib.tpgen_options_init(ctypes.byref(o))
        assert o.prune == 0
        o.engine, o.output_mode, o.prune = engine, mode, 1
        paths, stats = _abi.Paths(), _abi.Stats()
        r = lib.tpgen_prime_paths(so.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), g.n, ctypes.byref(o),
                                  ctypes.byref(paths), ctypes.byref(stats))
        assert r == 1
    for engine in (_abi.ENGINE_FRONTIER, _abi.ENGINE_ALG3):  # prefix-unit shards: a DFS-engine option
        o = _abi.Options()
        lib.tpgen_options_init(ctypes.byref(o))
        assert o.shard_prefix == 0
        o.engine, o.output_mode, o.shard_prefix, o.shard_count = engine, _abi.OUT_COUNT_HASH, 1, 2
        paths, stats = _abi.Paths(), _abi.Stats()
        r = lib.tpgen_prime_paths(so.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  st.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), g.n, ctypes.byref(o),
                                  ctypes.byref(paths), ctypes.byref(stats))
        assert r == 1


def test_metrics_fig1b_and_loops():
    """Table-1 structure metrics on the host: Fig. 1(b) has CC = 4, one SCC
    {2,3,4,5,6,8} with 7 internal arcs; K sequential loops of N vertices: K SCCs."""
    import paper_2210_16998_b200 as tp
    from workloads import generators as gen
    m = tp.metrics(gen.fig1b())
    assert m["nodes"] == 11 and m["edges"] == 13 and m["cc"] == 4
    assert m["sccs"] == 1 and m["scc_nodes"] == 6 and m["scc_edges"] == 7
    m = tp.metrics(gen.k_seq_loops(3, 4))
    assert m["sccs"] == 3 and m["cc"] == m["edges"] - m["nodes"] + 2


def test_metrics_npath_vs_oracle():
    """tpgen_metrics_compute's Npath (acyclic DP / arc-simple walk search) equals the tier-0
    recursion on the arc set (oracle/brute.py, pinned to P:592)."""
    import paper_2210_16998_b200 as tp
    from workloads import generators as gen
    assert tp.metrics(gen.fig1b())["npath"] == 4
    graphs = [gen.fig1b(), gen.k_seq_if(4), gen.k_nested_if(3), gen.k_seq_loops(2, 3), gen.config2()]
    graphs += [gen.random_dag_cfg(9, s) for s in range(3)]
    for g in graphs:
        m = tp.metrics(g)
        if m["npath_status"] != "exact":
            continue
        assert m["npath"] == brute.npath(g.n, brute.graph_succ(g), g.entry, g.exit), g.name
    for i, g in enumerate(_corpus(80, 77)):
        if g.n < 2 or g.n > 7:
            continue
        m = tp.metrics(g, start=0, end=g.n - 1)
        assert m["npath_status"] == "exact"
        assert m["npath"] == brute.npath(g.n, brute.graph_succ(g), 0, g.n - 1), g.name
        assert m["cc"] == m["edges"] - m["nodes"] + 2 * m["weak_components"]


def test_shard_range_partitions_the_starts():
    import paper_2210_16998_b200 as tp
    from workloads import generators as gen
    g = gen.config5()
    for world in (1, 2, 3, 8):
        cuts = [tp.shard_range(g, r, world) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == g.n
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))


def test_shard_units_tile_the_split():
    """Prefix-unit shards (tpgen_shard_units): on graphs with no arc leaving an SCC
    and SCCs of <= 32 vertices the ranks' unit ranges tile [0, n_units) in rank order, heavy start
    vertices are cut into prefix units (more units than start vertices, every rank non-empty even
    when there are more ranks than start vertices), the start ranges are monotone; elsewhere the
    split is the start-vertex one."""
    g = gen.config3()
    for world in (1, 2, 8, 40):
        cuts = [tp.shard_units(g, r, world) for r in range(world)]
        assert all(c["applies"] for c in cuts)
        n_units = cuts[0]["n_units"]
        assert all(c["n_units"] == n_units for c in cuts)
        assert cuts[0]["unit_lo"] == 0 and cuts[-1]["unit_hi"] == n_units
        assert all(a["unit_hi"] == b["unit_lo"] for a, b in zip(cuts, cuts[1:]))
        assert all(c["unit_hi"] > c["unit_lo"] for c in cuts)
        assert all(a["lo"] <= b["lo"] and a["hi"] <= b["hi"] and a["hi"] - 1 <= b["lo"]
                   for a, b in zip(cuts, cuts[1:]))
        assert cuts[0]["lo"] == 0 and cuts[-1]["hi"] == g.n
        if world > 1:
            assert n_units > g.n
    assert tp.shard_units(g, 0, 1)["n_units"] == g.n  # one shard: nothing is heavy enough to cut
    g5 = gen.config5()  # 56-vertex SCCs with arcs leaving them: the start-vertex split
    for r in range(4):
        c = tp.shard_units(g5, r, 4)
        assert not c["applies"] and (c["lo"], c["hi"]) == tp.shard_range(g5, r, 4)
        assert c["unit_lo"] == c["unit_hi"] == c["n_units"] == 0
    with pytest.raises(tp.TpgenError):
        tp.shard_units(g, 3, 3)


def _unit_of(pp, units):
    """Index of the prefix unit a prime path belongs to (tpgen_shard_unit_paths semantics)."""
    hits = [i for i, (path, clo) in enumerate(units)
            if (clo and pp == path + (path[0],)) or (not clo and pp[:len(path)] == path)]
    assert len(hits) == 1, (pp, hits)
    return hits[0]


@pytest.mark.parametrize("world", [2, 5, 16])
def test_prefix_units_partition_the_oracle_list(world):
    """The prefix-unit split on the host, pinned by the oracle: the units of all shards, in rank
    order, partition the oracle's canonical prime-path list into contiguous runs in unit order
    (so shard r's output is block r of the global list), and each shard's units are the
    [unit_lo, unit_hi) range tpgen_shard_units reports."""
    for g in (gen.dense_scc(12, 3, 7), gen.dense_scc(9, 4, 3),
              gen.disjoint_union([gen.dense_scc(10, 3, 1), gen.dense_scc(7, 3, 2)], name="pfx_union")):
        units, bounds = [], []
        for r in range(world):
            u = tp.shard_unit_paths(g, r, world)
            c = tp.shard_units(g, r, world)
            assert c["applies"] and len(u) == c["unit_hi"] - c["unit_lo"] and c["unit_lo"] == len(units)
            if u:
                assert (u[0][0][0], u[-1][0][0] + 1) == (c["lo"], c["hi"])
            units += u
            bounds.append(len(units))
        assert len(units) == tp.shard_units(g, 0, world)["n_units"]
        off, vert = oracle.prime_paths(g)
        idx = [_unit_of(tuple(vert[off[i]:off[i + 1]].tolist()), units) for i in range(len(off) - 1)]
        assert idx == sorted(idx), g.name  # canonical order = unit order
    assert tp.shard_unit_paths(gen.config5(), 0, 4) == []  # arcs leave its SCCs: no prefix split
