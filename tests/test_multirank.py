"""World-size-2 `gloo` test of the multi-rank path, CPU only.

bench.py's N>1 run gives rank r start-vertex shard (r, N) of the planner's
cost-balanced split (tpgen_shard_range) and reduces counts (sum) and times (max)
over the ranks.  Here each rank computes its block with the ORACLE (no GPU on
this box) and the test checks, across two real processes talking over gloo:
  * the rank blocks concatenate to the canonical list of the whole union graph
    (shards are contiguous blocks of the global order);
  * bench.rank_reduce sums the counts and maxes the times;
  * the order-independent digests of the blocks add up to the whole digest.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cut(g, world):
    """Start-vertex shard boundaries: the library's planner split (tpgen_shard_range, a host call)."""
    import sys

    sys.path.insert(0, ROOT)
    import paper_2210_16998_b200 as tp

    return [tp.shard_range(g, r, world)[0] for r in range(world)] + [g.n]


def _worker(rank: int, world: int, port: int, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench
    import oracle
    from workloads import generators as gen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gen.parallel_sccs(3, 7, 4)  # config 5's shape, small: Start -> d_i -> SCC_i -> J -> End
        lo, hi = _cut(g, world)[rank], _cut(g, world)[rank + 1]
        off, vert = oracle.prime_paths(g, v_lo=lo, v_hi=hi)
        n_pp = len(off) - 1
        ext = oracle.ext_count(g, v_lo=lo, v_hi=hi)
        (tot_pp, tot_ext), (ms_max, e2e_max) = bench.rank_reduce(dist, world, [float(n_pp), float(ext)],
                                                                 [1.0 + rank, 10.0 * (rank + 1)], "cpu")
        # gather the blocks to rank 0 (object collective over gloo)
        blocks = [None] * world
        dist.all_gather_object(blocks, (off.tolist(), vert.tolist()))
        h = oracle.digest(off, vert)
        hs = torch.tensor([h[0] & 0xFFFFFFFF, h[0] >> 32, h[1] & 0xFFFFFFFF, h[1] >> 32], dtype=torch.float64)
        parts = [torch.zeros_like(hs) for _ in range(world)]
        dist.all_gather(parts, hs)
        if rank == 0:
            q.put(dict(tot_pp=tot_pp, tot_ext=tot_ext, ms_max=ms_max, e2e_max=e2e_max, blocks=blocks,
                       parts=[p.tolist() for p in parts], n=g.n))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_shards_and_reduce():
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    from workloads import generators as gen
    import bench

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    g = gen.parallel_sccs(3, 7, 4)
    off, vert = oracle.prime_paths(g)
    # concatenation of the rank blocks == the whole canonical list
    cat_off, cat_vert = [0], []
    for bo, bv in res["blocks"]:
        shift = cat_off[-1]
        cat_off.extend(shift + np.asarray(bo[1:], dtype=np.int64))
        cat_vert.extend(bv)
    assert np.array_equal(np.asarray(cat_off, dtype=np.int64), off)
    assert np.array_equal(np.asarray(cat_vert, dtype=np.int32), vert)
    # reductions: counts summed, times maxed
    assert res["tot_pp"] == float(len(off) - 1)
    assert res["tot_ext"] == float(oracle.ext_count(g))
    assert res["ms_max"] == 2.0 and res["e2e_max"] == 20.0
    # digest is additive over shards (mod 2^64)
    lo = sum(int(p[0]) | (int(p[1]) << 32) for p in res["parts"]) % (1 << 64)
    hi = sum(int(p[2]) | (int(p[3]) << 32) for p in res["parts"]) % (1 << 64)
    assert (lo, hi) == oracle.digest(off, vert)
    # strong scaling: both ranks got work
    assert len(res["blocks"][0][1]) > 0 and len(res["blocks"][1][1]) > 0


def _worker_sharded(rank: int, world: int, port: int, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle
    from paper_2210_16998_b200 import PathSet
    from paper_2210_16998_b200.distributed import sharded_prime_paths
    from workloads import generators as gen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gen.config2()
        cut = [0, 30, g.n]  # stand-in for the planner's cost-balanced shard boundaries

        def compute(r, w):  # the oracle's block for this rank's start-vertex range
            off, vert = oracle.prime_paths(g, v_lo=cut[r], v_hi=cut[r + 1])
            lo, hi = oracle.digest(off, vert)
            st = {"n_paths": len(off) - 1, "total_vertices": int(off[-1]),
                  "n_extensions": oracle.ext_count(g, v_lo=cut[r], v_hi=cut[r + 1]), "hash_lo": lo, "hash_hi": hi}
            return PathSet(off, vert, len(off) - 1, False, st)

        res = sharded_prime_paths(g, compute=compute, gather=True)
        if rank == 0:
            q.put(dict(whole=(res.whole[0].tolist(), res.whole[1].tolist())))
        if rank == 1:
            q.put(dict(pp_base=res.pp_base, vertex_base=res.vertex_base, n_paths=res.n_paths,
                       total_vertices=res.total_vertices, n_extensions=res.n_extensions, digest=res.digest,
                       local=(res.paths.offsets.tolist(), res.paths.vertices.tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_prime_paths_gloo():
    """paper_2210_16998_b200.distributed: the one all_gather gives each rank the global
    offsets of its block, the totals and the set digest of the whole list."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    from workloads import generators as gen

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240), q.get(timeout=240)]
    res = next(x for x in got if "local" in x)
    whole = next(x for x in got if "whole" in x)["whole"]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gen.config2()
    off, vert = oracle.prime_paths(g)
    lo_off, lo_vert = res["local"]
    a = res["pp_base"]
    # rank 1's block sits at its global offsets in the whole canonical list
    assert np.array_equal(np.asarray(lo_off, dtype=np.int64) + res["vertex_base"], off[a:a + len(lo_off)])
    assert np.array_equal(np.asarray(lo_vert, dtype=np.int32), vert[res["vertex_base"]:int(off[-1])])
    assert res["n_paths"] == len(off) - 1 and res["total_vertices"] == int(off[-1])
    assert res["n_extensions"] == oracle.ext_count(g)
    assert tuple(res["digest"]) == oracle.digest(off, vert)
    # C4: rank 0 holds the whole canonical list, element by element
    assert np.array_equal(np.asarray(whole[0], dtype=np.int64), off)
    assert np.array_equal(np.asarray(whole[1], dtype=np.int32), vert)


def _worker_prefix(rank: int, world: int, port: int, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle
    import paper_2210_16998_b200 as tp
    from paper_2210_16998_b200 import PathSet
    from paper_2210_16998_b200.distributed import sharded_prime_paths
    from workloads import generators as gen

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gen.dense_scc(9, 4, 3)  # 9 start vertices, one SCC: prefix units cut the heavy starts

        def compute(r, w):  # the oracle's prime paths of this rank's prefix units (the host split)
            units = tp.shard_unit_paths(g, r, w)
            off, vert = oracle.prime_paths(g)
            keep = []
            for i in range(len(off) - 1):
                pp = tuple(vert[off[i]:off[i + 1]].tolist())
                if any((c and pp == p + (p[0],)) or (not c and pp[:len(p)] == p) for p, c in units):
                    keep.append(pp)
            o = np.zeros(len(keep) + 1, dtype=np.int64)
            o[1:] = np.cumsum([len(p) for p in keep])
            v = np.asarray([x for p in keep for x in p], dtype=np.int32)
            lo, hi = oracle.digest(o, v)
            st = {"n_paths": len(keep), "total_vertices": int(o[-1]), "n_extensions": 0,
                  "hash_lo": lo, "hash_hi": hi}
            return PathSet(o, v, len(keep), False, st)

        res = sharded_prime_paths(g, compute=compute, gather=True, shard_prefix=True)
        q.put(dict(rank=rank, pp_base=res.pp_base, n_paths=res.n_paths, digest=res.digest,
                   local=len(res.paths.offsets) - 1,
                   whole=(res.whole[0].tolist(), res.whole[1].tolist()) if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_prefix_shards_gloo():
    """Prefix-unit shards (tpgen_options.shard_prefix) through the same exchange: each rank's
    block is its units' prime paths, the blocks' global offsets tile the list, and the C4 gather
    on rank 0 equals the oracle's whole canonical list element by element."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    from workloads import generators as gen

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_prefix, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=240), q.get(timeout=240)], key=lambda x: x["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gen.dense_scc(9, 4, 3)
    off, vert = oracle.prime_paths(g)
    assert got[0]["pp_base"] == 0 and got[1]["pp_base"] == got[0]["local"]
    assert got[0]["local"] > 0 and got[1]["local"] > 0
    assert got[0]["local"] + got[1]["local"] == len(off) - 1 == got[1]["n_paths"]
    assert tuple(got[1]["digest"]) == oracle.digest(off, vert)
    whole = got[0]["whole"]
    assert np.array_equal(np.asarray(whole[0], dtype=np.int64), off)
    assert np.array_equal(np.asarray(whole[1], dtype=np.int32), vert)
