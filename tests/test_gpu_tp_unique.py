"""K7 (TPGEN_TP_UNIQUE): the distinct per-PP test paths in lexicographic order (device merge
sort with a sequence comparator, adjacent duplicates dropped, compacted) -- element by element
against oracle.unique_test_paths (expected values from oracle/ only)."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")


def _check(g, ref=None, **kw):
    if ref is None:
        ro, rv = oracle.prime_paths(g)
        ref = oracle.unique_test_paths(g, ro, rv, g.entry, g.exit)
    uo, uv = ref
    ts = tp.test_paths(g, g.entry, g.exit, cover="unique", **kw)
    o, v = ts.to_numpy()
    np.testing.assert_array_equal(o, uo, err_msg=g.name)
    np.testing.assert_array_equal(v, uv, err_msg=g.name)
    assert ts.stats["n_paths"] == len(uo) - 1 and ts.stats["total_vertices"] == int(uo[-1])
    return ts


def test_unique_fig1b():
    ts = _check(gen.fig1b())
    assert ts.stats["n_paths"] == 10  # 19 per-PP test paths, 10 distinct


def test_unique_corpus():
    for g in (gen.config2(), gen.k_seq_loops(3, 3), gen.k_nested_if(4), gen.k_seq_if(6), gen.config4(K=40)):
        _check(g)


def test_unique_config4_full_and_given_prime_list_and_host_output():
    g = gen.config4()  # K = 150
    ro, rv = oracle.prime_paths(g)
    ref = oracle.unique_test_paths(g, ro, rv, g.entry, g.exit)
    _check(g, ref)
    pp = tp.prime_paths(g)
    _check(g, ref, prime=pp)
    _check(g, ref, output="host")


def test_unique_rejects_count_mode():
    g = gen.fig1b()
    with pytest.raises(Exception):
        tp.test_paths(g, g.entry, g.exit, cover="unique", mode="count")
