"""GPU parity of prefix-unit shards (tpgen_options.shard_prefix; SURVEY 8(a) a7 "(start, depth-k
prefix) for heavy starts"): shard r of N is a contiguous range of the split's prefix units, so its
output is block r of the global canonical list.  Expected values come only from oracle/ (the
whole-list comparisons) or from the same library's unsharded call, itself pinned to the oracle by
tests/test_gpu_parity.py and tests/test_gpu_count.py."""
import numpy as np
import pytest

import oracle
from workloads import generators as gen

pytestmark = pytest.mark.gpu

tp = pytest.importorskip("paper_2210_16998_b200")

M64 = (1 << 64) - 1


def _shards(plan, world, **kw):
    return [plan.prime_paths(shard=(r, world), shard_prefix=True, **kw) for r in range(world)]


def _check_unit_tiling(g, world, stats):
    split = [tp.shard_units(g, r, world) for r in range(world)]
    assert [(s["unit_lo"], s["unit_hi"]) for s in stats] == [(c["unit_lo"], c["unit_hi"]) for c in split]
    assert [(s["shard_lo"], s["shard_hi"]) for s in stats] == [(c["lo"], c["hi"]) for c in split]


@pytest.mark.parametrize("world", [2, 5, 16, 48])
def test_prefix_shards_are_blocks_of_the_oracle_list(world):
    """Small graphs with fewer start vertices than some shard counts: every shard's block equals
    the oracle's list at the block's offset, element by element; E_canon and the digests add up to
    the oracle's; a count-mode shard equals the materialized one."""
    for g in (gen.dense_scc(12, 3, 7), gen.dense_scc(9, 4, 3),
              gen.disjoint_union([gen.dense_scc(10, 3, 1), gen.dense_scc(7, 3, 2)], name="pfx_union")):
        ro, rv = oracle.prime_paths(g)
        plan = tp.Plan(g)
        pss = _shards(plan, world, digest=True)
        _check_unit_tiling(g, world, [p.stats for p in pss])
        base = 0
        ext = h_lo = h_hi = 0
        for r, ps in enumerate(pss):
            o, v = ps.to_numpy()
            n = ps.stats["n_paths"]
            np.testing.assert_array_equal(o, ro[base: base + n + 1] - ro[base], err_msg=f"{g.name} shard {r}")
            np.testing.assert_array_equal(v, rv[ro[base]: ro[base + n]], err_msg=f"{g.name} shard {r}")
            base += n
            ext += ps.stats["n_extensions"]
            h_lo = (h_lo + ps.stats["hash_lo"]) & M64
            h_hi = (h_hi + ps.stats["hash_hi"]) & M64
            c = plan.prime_paths(shard=(r, world), shard_prefix=True, mode="count", digest=True).stats
            assert (c["n_paths"], c["total_vertices"], c["n_extensions"], c["hash_lo"], c["hash_hi"]) == \
                (n, ps.stats["total_vertices"], ps.stats["n_extensions"], ps.stats["hash_lo"], ps.stats["hash_hi"])
        assert base == len(ro) - 1, g.name
        assert ext == oracle.ext_count(g), g.name
        assert (h_lo, h_hi) == oracle.digest(ro, rv)
        plan.close()


def test_prefix_shards_config3_full_size():
    """Config 3 (22 start vertices, 6.0e7 prime paths) in 8 prefix-unit shards: the blocks
    concatenate to the unsharded canonical list element by element; the count-mode shards sum to
    the unsharded counts, E_canon and digest; the heaviest shard does at most 1.3x the mean work
    (start-vertex shards of 22 starts over 8 ranks cannot do better than ~1.4x)."""
    g = gen.config3()
    plan = tp.Plan(g)
    whole = plan.prime_paths(digest=True)
    wo, wv = whole.offsets, whole.vertices
    wst = dict(whole.stats)
    base = 0
    ext = []
    for r in range(8):
        ps = plan.prime_paths(shard=(r, 8), shard_prefix=True)
        n = ps.stats["n_paths"]
        nv = ps.stats["total_vertices"]
        vb = int(wo[base].item())
        assert bool((ps.offsets == (wo[base: base + n + 1] - vb)).all()), f"shard {r} offsets"
        assert bool((ps.vertices == wv[vb: vb + nv]).all()), f"shard {r} vertices"
        base += n
        ext.append(ps.stats["n_extensions"])
        del ps
    assert base == wst["n_paths"]
    assert sum(ext) == wst["n_extensions"]
    assert max(ext) <= 1.3 * (sum(ext) / len(ext)), ext
    del whole, wo, wv
    cw = plan.prime_paths(mode="count", digest=True).stats
    tot = [0, 0, 0, 0, 0]
    cst = []
    for r in range(8):
        c = plan.prime_paths(shard=(r, 8), shard_prefix=True, mode="count", digest=True).stats
        cst.append(c)
        for i, k in enumerate(("n_paths", "total_vertices", "n_extensions")):
            tot[i] += c[k]
        tot[3] = (tot[3] + c["hash_lo"]) & M64
        tot[4] = (tot[4] + c["hash_hi"]) & M64
    _check_unit_tiling(g, 8, cst)
    assert tot == [cw["n_paths"], cw["total_vertices"], cw["n_extensions"], cw["hash_lo"], cw["hash_hi"]]
    assert (cw["hash_lo"], cw["hash_hi"]) == (wst["hash_lo"], wst["hash_hi"])
    plan.close()


def test_prefix_shards_fall_back_to_start_vertices():
    """Graphs the split does not apply to (arcs leaving SCCs): shard_prefix leaves the
    start-vertex shards (unit_lo = unit_hi = -1) and the output unchanged."""
    g = gen.config2()
    for r in range(3):
        a = tp.prime_paths(g, shard=(r, 3), shard_prefix=True)
        b = tp.prime_paths(g, shard=(r, 3))
        assert a.stats["unit_lo"] == a.stats["unit_hi"] == -1
        assert (a.stats["shard_lo"], a.stats["shard_hi"]) == tp.shard_range(g, r, 3)
        np.testing.assert_array_equal(a.to_numpy()[1], b.to_numpy()[1])
