"""Multi-GPU prime paths: one process per GPU over torch.distributed.

Every rank enumerates the prime paths whose first vertex lies in its start-vertex
shard (``tpgen_options.shard_rank / shard_count``: contiguous ranges balanced by
the planner's cost estimates).  The per-start trees are independent and a
shard's output is a contiguous block of the global canonical list, so the only
exchange is one all_gather of five words per rank (SURVEY §8(e) C1 + C2): the
block's global prime-path and vertex offsets, the totals, and the
order-independent digest.  Results stay where they were computed unless
``gather=True``: then rank 0 also receives the whole canonical
list -- the ranks' blocks concatenated in rank order, which is the global order
(every block is a contiguous range of start vertices) -- through one all_gather
of the padded blocks; for outputs that fit one GPU (config 5's ~230 GB does not).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

from . import PathSet, prime_paths

_MASK64 = (1 << 64) - 1


@dataclass
class ShardResult:
    paths: PathSet          # this rank's contiguous block of the global canonical list
    pp_base: int            # global index of its first prime path
    vertex_base: int        # global offset of its first vertex
    n_paths: int            # totals over all ranks
    total_vertices: int
    n_extensions: int
    digest: Tuple[int, int]  # set digest of the whole list (sum mod 2^64 of the ranks' digests)
    whole: Optional[Tuple] = None  # gather=True, rank 0: (offsets, vertices) of the whole list


def _signed(u: int) -> int:
    u &= _MASK64
    return u - (1 << 64) if u >= (1 << 63) else u


def _gather_blocks(ps: PathSet, rows, rank: int, world: int, group, dev):
    """C4: every rank's block (offsets relative to its block, vertices) to rank 0, as one
    all_gather of a padded int64 buffer [n_paths, offsets..., vertices...] per rank."""
    import torch
    import torch.distributed as dist

    n_max = max(r[0] for r in rows)
    v_max = max(r[1] for r in rows)
    size = 1 + (n_max + 1) + v_max
    buf = torch.zeros(size, dtype=torch.int64, device=dev)
    off, vert = ps.offsets, ps.vertices
    if not torch.is_tensor(off):
        off, vert = torch.as_tensor(off), torch.as_tensor(vert)
    n = int(off.numel()) - 1
    buf[0] = n
    buf[1:n + 2] = off.to(dev, torch.int64)
    buf[1 + n_max + 1:1 + n_max + 1 + int(vert.numel())] = vert.to(dev, torch.int64)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return None
    offs, verts, vbase = [torch.zeros(1, dtype=torch.int64, device=dev)], [], 0
    for r, p in enumerate(parts):
        k, nv = int(rows[r][0]), int(rows[r][1])
        offs.append(p[2:k + 2] + vbase)
        verts.append(p[1 + n_max + 1:1 + n_max + 1 + nv].to(torch.int32))
        vbase += nv
    return torch.cat(offs), torch.cat(verts) if verts else torch.zeros(0, dtype=torch.int32, device=dev)


def sharded_prime_paths(graph, group=None, *, device: Optional[int] = None, mode: str = "materialize",
                        digest: bool = True, compute: Optional[Callable[[int, int], PathSet]] = None,
                        engine: str = "dfs", gather: bool = False, shard_prefix: bool = False) -> ShardResult:
    """This rank's prime paths plus their place in the global list.

    ``engine="frontier"`` (with ``mode="count"``) runs the level-synchronous engine on
    this rank's start vertices; the exchange is the same.
    ``gather=True`` (materialize mode): rank 0 also gets the whole list in ``whole`` (C4).
    ``shard_prefix=True``: the ranks split prefix units of heavy start vertices
    (tpgen_options.shard_prefix; a graph with fewer start vertices than ranks still balances);
    the blocks are still contiguous in rank order, so the exchange is the same.
    ``compute(rank, world)`` replaces the GPU call (a test seam: the gloo tests run
    the collective logic on CPU with the oracle's shards)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if compute is None:
        dev = torch.cuda.current_device() if device is None else device
        ps = prime_paths(graph, device=dev, shard=(rank, world), mode=mode, digest=digest, engine=engine,
                         shard_prefix=shard_prefix)
    else:
        ps = compute(rank, world)
    st = ps.stats
    words = [int(st["n_paths"]), int(st["total_vertices"]), int(st["n_extensions"]),
             _signed(int(st.get("hash_lo", 0))), _signed(int(st.get("hash_hi", 0)))]
    on_gpu = dist.get_backend(group) == "nccl"
    cdev = torch.device("cuda", torch.cuda.current_device() if device is None else device) if on_gpu else \
        torch.device("cpu")  # NCCL tensors on the GPU this rank computes on
    t = torch.tensor(words, dtype=torch.int64, device=cdev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    rows = [[int(x) for x in r.cpu().tolist()] for r in out]
    whole = None
    if gather:
        if mode != "materialize":
            raise ValueError("gather=True needs mode='materialize'")
        whole = _gather_blocks(ps, rows, rank, world, group, cdev)
    return ShardResult(
        paths=ps,
        pp_base=sum(r[0] for r in rows[:rank]),
        vertex_base=sum(r[1] for r in rows[:rank]),
        n_paths=sum(r[0] for r in rows),
        total_vertices=sum(r[1] for r in rows),
        n_extensions=sum(r[2] for r in rows),
        digest=(sum(r[3] for r in rows) & _MASK64, sum(r[4] for r in rows) & _MASK64),
        whole=whole,
    )
