"""GPU parity of NEXT #2 reachability pruning (tpgen_options.prune, not in the
paper): the pruned count-mode DFS gives the oracle's prime-path counts, vertices and digest,
with no more extensions than E_canon (and strictly fewer where a subtree holds no event).

Expected values come only from oracle/ (oracle.pp_stats, oracle.ext_count)."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")

M64 = (1 << 64) - 1


def _tot(rows):
    a = rows[:, :4].astype(object)
    return (int(a[:, 0].sum()), int(a[:, 1].sum()), int(a[:, 2].sum()) & M64, int(a[:, 3].sum()) & M64)


def _corpus():
    rng = np.random.default_rng(23)
    for i in range(50):
        n = int(rng.integers(2, 13))
        yield gen.random_digraph(n, float(rng.choice([0.15, 0.25, 0.35])), 900 + i,
                                 self_loops=bool(rng.random() < 0.4))
    yield gen.fig1b()
    yield gen.config2()
    yield gen.config4(K=30)
    for n, d, seed in ((12, 3, 1), (16, 3, 2), (20, 2, 5), (24, 2, 8)):
        yield gen.dense_scc(n, d, seed)
    yield gen.parallel_sccs(3, 24, 9)
    yield gen.parallel_sccs(2, 40, 3)  # 64-bit masks


def test_pruned_count_mode_matches_oracle():
    fewer = 0
    for g in _corpus():
        st = tp.prime_paths(g, mode="count", digest=True, prune=True).stats
        ref = oracle.pp_stats(g)
        assert (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"]) == _tot(ref), g.name
        e = oracle.ext_count(g)
        assert st["n_extensions"] <= e, g.name
        fewer += st["n_extensions"] < e
        nd = tp.prime_paths(g, mode="count", digest=False, prune=True).stats  # counts-only variant
        assert (nd["n_paths"], nd["total_vertices"], nd["n_extensions"]) == \
            (st["n_paths"], st["total_vertices"], st["n_extensions"]), g.name
    assert fewer > 0  # the rule fires somewhere in the corpus


@pytest.mark.parametrize("name", ["config3", "config5"])
def test_pruned_full_size_equals_unpruned(name):
    """Configs 3 and 5 at full size: pruned counts and digest equal the unpruned call's (itself
    equal to the oracle's in tests/test_gpu_count.py), with fewer extensions made."""
    g = getattr(gen, name)()
    plan = tp.Plan(g)
    a = plan.prime_paths(mode="count", digest=True).stats
    b = plan.prime_paths(mode="count", digest=True, prune=True).stats
    assert (b["n_paths"], b["total_vertices"], b["hash_lo"], b["hash_hi"]) == \
        (a["n_paths"], a["total_vertices"], a["hash_lo"], a["hash_hi"])
    assert b["n_extensions"] <= a["n_extensions"]
    plan.close()


def test_prune_option_checks():
    g = gen.fig1b()
    with pytest.raises(tp.TpgenError):
        tp.prime_paths(g, prune=True)  # materialize: not supported
    with pytest.raises(tp.TpgenError):
        tp.prime_paths(g, mode="count", engine="frontier", prune=True)
