"""B200-native prime-path / test-path engine (TPGen hot path, arXiv 2210.16998).

Thin Python binding over the C ABI in ``include/tpgen.h`` (``libtpgen.so``):
argument marshalling only -- every step of the path runs in the library's
CUDA kernels.  PyTorch supplies device memory (output buffers come from the
caching allocator), streams and, in bench.py, process groups.  There is no
CPU fallback: without the built library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any, Dict, Optional, Tuple

import numpy as np

from . import _abi

__all__ = ["TpgenError", "PathSet", "Plan", "prime_paths", "test_paths", "components", "metrics", "shard_range", "shard_units", "shard_unit_paths",
           "library", "version"]


class TpgenError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.status_name = _abi.STATUS_NAMES.get(status, str(status))
        super().__init__(f"{self.status_name}: {msg}")


def library():
    return _abi.load()


def version() -> str:
    return library().tpgen_version().decode()


@dataclass
class PathSet:
    """Canonical flat path array: ``offsets[n_paths+1]`` (int64), ``vertices`` (int32).

    On device these are torch CUDA tensors, on the host numpy arrays."""

    offsets: Any
    vertices: Any
    n_paths: int
    on_device: bool
    stats: Dict[str, Any] = field(default_factory=dict)

    def to_numpy(self) -> Tuple[np.ndarray, np.ndarray]:
        if self.on_device:
            return self.offsets.cpu().numpy(), self.vertices.cpu().numpy()
        return np.asarray(self.offsets), np.asarray(self.vertices)

    def as_list(self):
        off, vert = self.to_numpy()
        return [tuple(vert[off[i]:off[i + 1]].tolist()) for i in range(len(off) - 1)]


def _csr(graph) -> Tuple[np.ndarray, np.ndarray, int]:
    if hasattr(graph, "offsets") and hasattr(graph, "targets"):
        so, st, n = graph.offsets, graph.targets, graph.n
    else:
        so, st = graph[0], graph[1]
        n = len(so) - 1
    so = np.ascontiguousarray(so, dtype=np.int64)
    st = np.ascontiguousarray(st, dtype=np.int32)
    if st.size == 0:
        st = np.zeros(1, dtype=np.int32)  # valid pointer for an arc-free graph
    return so, st, int(n)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


class _PathsOwner:
    """Owns a library-allocated tpgen_paths (device pool memory); frees it when the
    last tensor view is gone."""

    def __init__(self, paths: _abi.Paths):
        self.paths = paths

    def __del__(self):
        try:
            library().tpgen_paths_free(ctypes.byref(self.paths))
        except Exception:
            pass


class _DeviceArray:
    """Zero-copy view of library device memory for torch (``__cuda_array_interface__``)."""

    def __init__(self, owner: _PathsOwner, ptr: int, n: int, typestr: str):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 2, "strides": None}


def _as_tensor(owner: _PathsOwner, ptr: int, n: int, typestr: str, device: int):
    import torch

    return torch.as_tensor(_DeviceArray(owner, ptr, n, typestr), device=torch.device("cuda", device))


class _TorchAllocator:
    """Output allocator backed by torch's caching allocator (device memory only)."""

    def __init__(self, device: int):
        import torch

        self.torch = torch
        self.device = torch.device("cuda", device)
        self.live: Dict[int, Any] = {}
        self.alloc_fn = _abi.ALLOC_FN(self._alloc)
        self.free_fn = _abi.FREE_FN(self._free)

    def _alloc(self, nbytes, stream, ctx):
        t = self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.device)
        p = t.data_ptr()
        self.live[p] = t
        return p

    def _free(self, ptr, stream, ctx):
        self.live.pop(int(ptr or 0), None)

    def take(self, ptr: int):
        return self.live.pop(ptr)


def _options(device: int, output: str, mode: str, shard: Tuple[int, int], digest: bool, max_paths: int,
             max_extensions: int, stream, alloc: Optional[_TorchAllocator], host_out=None,
             start_range: Optional[Tuple[int, int]] = None, engine: str = "dfs",
             plan_cache: bool = True, shard_prefix: bool = False, prune: bool = False) -> _abi.Options:
    lib = library()
    o = _abi.Options()
    lib.tpgen_options_init(ctypes.byref(o))
    o.device = device
    o.stream = stream
    o.output_on_device = 1 if output == "device" else 0
    o.output_mode = _abi.OUT_COUNT_HASH if mode == "count" else _abi.OUT_MATERIALIZE
    o.shard_rank, o.shard_count = shard
    if start_range is not None:
        o.start_lo, o.start_hi = start_range
    o.max_paths = max_paths
    o.max_extensions = max_extensions
    o.compute_digest = 1 if digest else 0
    o.engine = _engine(engine)
    o.no_plan_cache = 0 if plan_cache else 1
    o.shard_prefix = 1 if shard_prefix else 0
    o.prune = 1 if prune else 0
    if alloc is not None:
        o.device_alloc = alloc.alloc_fn
        o.device_free = alloc.free_fn
    if host_out is not None:
        o.host_out = host_out.data_ptr()
        o.host_out_bytes = host_out.numel() * host_out.element_size()
    return o


_ENGINES = {"dfs": _abi.ENGINE_DFS, "frontier": _abi.ENGINE_FRONTIER, "alg3": _abi.ENGINE_ALG3}


def _engine(engine: str) -> int:
    if engine not in _ENGINES:
        raise ValueError(f"engine must be one of {sorted(_ENGINES)}, not {engine!r}")
    return _ENGINES[engine]


def _stream_handle(device: int, stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _check(status: int):
    if status != _abi.TPGEN_OK:
        raise TpgenError(status, library().tpgen_last_error_message().decode())


def _wrap(paths: _abi.Paths, stats: _abi.Stats, alloc: Optional[_TorchAllocator], host_out=None) -> PathSet:
    lib = library()
    n = int(paths.n_paths)
    st = stats.as_dict()
    nv = int(st.get("total_vertices", 0))
    if not ctypes.cast(paths.offsets, ctypes.c_void_p).value:  # count-only mode: stats, no arrays
        return PathSet(None, None, int(st.get("n_paths", 0)), False, st)
    if paths.on_device:
        p_off = ctypes.cast(paths.offsets, ctypes.c_void_p).value
        p_v = ctypes.cast(paths.vertices, ctypes.c_void_p).value
        if alloc is None:  # library pool memory, viewed zero-copy; freed with the last view
            owner = _PathsOwner(paths)
            off = _as_tensor(owner, p_off, n + 1, "<i8", int(paths.device))
            vert = _as_tensor(owner, p_v, nv, "<i4", int(paths.device))
            return PathSet(off, vert, n, True, st)
        off = alloc.take(p_off).view(alloc.torch.int64)[: n + 1]
        vert = alloc.take(p_v).view(alloc.torch.int32)[:nv]
        lib.tpgen_paths_free(ctypes.byref(paths))
        return PathSet(off, vert, n, True, st)
    if host_out is not None and ctypes.cast(paths.offsets, ctypes.c_void_p).value == host_out.data_ptr():
        import torch

        off = host_out[: 8 * (n + 1)].view(torch.int64)
        vert = host_out[8 * (n + 1): 8 * (n + 1) + 4 * nv].view(torch.int32)
        lib.tpgen_paths_free(ctypes.byref(paths))
        return PathSet(off, vert, n, False, st)
    off = np.ctypeslib.as_array(paths.offsets, shape=(n + 1,)).copy()
    vert = (np.ctypeslib.as_array(paths.vertices, shape=(nv,)).copy() if nv else np.zeros(0, dtype=np.int32))
    lib.tpgen_paths_free(ctypes.byref(paths))
    return PathSet(off, vert, n, False, st)


def prime_paths(graph, *, device: int = 0, output: str = "device", mode: str = "materialize",
                shard: Tuple[int, int] = (0, 1), digest: bool = False, max_paths: int = 0,
                max_extensions: int = 0, stream=None, host_out=None,
                start_range: Optional[Tuple[int, int]] = None, engine: str = "dfs",
                plan_cache: bool = True, shard_prefix: bool = False, prune: bool = False) -> PathSet:
    """All prime paths of ``graph`` (Def. 1), canonical order.

    ``graph``: a ``workloads.Graph`` or ``(offsets, targets)`` successor CSR (host).
    ``engine``: "dfs" (default), "frontier" (level-synchronous, ``mode="count"`` only;
    include/tpgen.h TPGEN_ENGINE_FRONTIER) or "alg3" (the paper's vertex-centric
    self-stabilizing Alg. 3 as a comparison engine, ``mode="count"``, <= 128 vertices;
    TPGEN_ENGINE_ALG3).  ``plan_cache=False``: plan and upload the graph
    anew even if the previous call passed the same CSR (tpgen_options.no_plan_cache).
    ``shard_prefix=True``: ``shard`` splits prefix units of heavy start vertices, not whole
    start vertices (tpgen_options.shard_prefix; see ``shard_units``).  ``prune=True``
    (``mode="count"``): NEXT #2 reachability pruning (tpgen_options.prune; n_extensions
    then counts the extensions made)."""
    lib = library()
    _engine(engine)
    so, st, n = _csr(graph)
    alloc = None  # outputs come from the library's device memory pool (no Python callback while timing)
    o = _options(device, output, mode, shard, digest, max_paths, max_extensions, _stream_handle(device, stream),
                 alloc, host_out, start_range, engine, plan_cache, shard_prefix, prune)
    paths, stats = _abi.Paths(), _abi.Stats()
    _check(lib.tpgen_prime_paths(_p64(so), _p32(st), n, ctypes.byref(o), ctypes.byref(paths), ctypes.byref(stats)))
    return _wrap(paths, stats, alloc, host_out)


def test_paths(graph, entry: int, exit: int, prime: Optional[PathSet] = None, *, device: int = 0,
               output: str = "device", stream=None, cover: str = "per_pp", mode: str = "materialize") -> PathSet:
    """Entry->exit test paths (R15): one per prime path,
    aligned with the prime-path list (cover="per_pp"), their distinct set in lexicographic order
    (cover="unique", K7; materialized only), or the greedy cover -- longest
    uncovered prime path first, every prime path contained in a TP covered (cover="greedy").
    ``mode="count"``: COUNT_HASH -- the test paths' count, vertices and R20 digest in the
    stats, nothing written (fused into the count-mode enumeration when ``prime`` is None)."""
    lib = library()
    so, st, n = _csr(graph)
    alloc = None
    o = _options(device, output, mode, (0, 1), mode == "count", 0, 0, _stream_handle(device, stream), alloc)
    o.tp_mode = _tp_mode(cover)
    keep = []
    pin = _paths_in(prime, device, keep)
    paths, stats = _abi.Paths(), _abi.Stats()
    _check(lib.tpgen_test_paths(_p64(so), _p32(st), n, ctypes.byref(pin) if pin is not None else None, entry, exit,
                                ctypes.byref(o), ctypes.byref(paths), ctypes.byref(stats)))
    return _wrap(paths, stats, alloc)


_TP_MODES = {"per_pp": _abi.TP_PER_PP, "unique": _abi.TP_UNIQUE, "greedy": _abi.TP_GREEDY}


def _tp_mode(cover: str) -> int:
    if cover not in _TP_MODES:
        raise ValueError("cover must be 'per_pp', 'unique' or 'greedy'")
    return _TP_MODES[cover]


def _paths_in(prime: Optional[PathSet], device: int, keep: list):
    """A PathSet as the ABI's tpgen_paths input (device views or host arrays kept alive in `keep`)."""
    if prime is None:
        return None
    pin = _abi.Paths()
    pin.n_paths = prime.n_paths
    if prime.on_device:
        pin.offsets = ctypes.cast(prime.offsets.data_ptr(), ctypes.POINTER(ctypes.c_int64))
        pin.vertices = ctypes.cast(prime.vertices.data_ptr(), ctypes.POINTER(ctypes.c_int32))
        pin.on_device = 1
    else:
        a = np.ascontiguousarray(prime.offsets, dtype=np.int64)
        b = np.ascontiguousarray(prime.vertices, dtype=np.int32)
        if b.size == 0:
            b = np.zeros(1, dtype=np.int32)
        keep += [a, b]
        pin.offsets = _p64(a)
        pin.vertices = _p32(b)
        pin.on_device = 0
    pin.device = device
    return pin


def components(graph):
    """Component graph on the host (``tpgen_components``): (comp[v], flags[v], n_scc).
    flags: 1 = SCC entry vertex (Def. 4), 2 = SCC exit vertex (Def. 5), 4 = nontrivial SCC."""
    lib = library()
    so, st, n = _csr(graph)
    comp = np.zeros(max(n, 1), dtype=np.int32)
    flags = np.zeros(max(n, 1), dtype=np.int32)
    nscc = ctypes.c_int32()
    _check(lib.tpgen_components(_p64(so), _p32(st), n, _p32(comp), _p32(flags), ctypes.byref(nscc)))
    return comp[:n], flags[:n], int(nscc.value)


def shard_range(graph, rank: int, count: int) -> Tuple[int, int]:
    """Start-vertex range [lo, hi) of shard ``rank`` of ``count`` (``tpgen_shard_range``, host):
    the planner's contiguous, cost-balanced split that ``shard=(rank, count)`` selects."""
    lib = library()
    so, st, n = _csr(graph)
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    _check(lib.tpgen_shard_range(_p64(so), _p32(st), n, rank, count, ctypes.byref(lo), ctypes.byref(hi)))
    return int(lo.value), int(hi.value)


def shard_units(graph, rank: int, count: int) -> Dict[str, Any]:
    """Prefix-unit shard ``rank`` of ``count`` (``tpgen_shard_units``, host; what
    ``shard=(rank, count), shard_prefix=True`` selects): ``applies``, the unit range
    ``[unit_lo, unit_hi)`` of ``n_units`` and the start vertices ``[lo, hi)`` it touches."""
    lib = library()
    so, st, n = _csr(graph)
    ap, lo, hi = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    ul, uh, nu = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib.tpgen_shard_units(_p64(so), _p32(st), n, rank, count, ctypes.byref(ap), ctypes.byref(ul),
                                 ctypes.byref(uh), ctypes.byref(nu), ctypes.byref(lo), ctypes.byref(hi)))
    return {"applies": bool(ap.value), "unit_lo": int(ul.value), "unit_hi": int(uh.value),
            "n_units": int(nu.value), "lo": int(lo.value), "hi": int(hi.value)}


def shard_unit_paths(graph, rank: int, count: int):
    """The prefix units of shard ``rank`` of ``count`` (``tpgen_shard_unit_paths``, host): a list of
    ``(path, closure)`` -- ``path`` the unit's global vertex ids (start first); ``closure`` True:
    the cyclic prime path path + [start], False: every prime path with ``path`` as a prefix."""
    lib = library()
    so, st, n = _csr(graph)
    nu, nv = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.tpgen_shard_unit_paths(_p64(so), _p32(st), n, rank, count, None, None, None, 0, 0,
                                      ctypes.byref(nu), ctypes.byref(nv)))
    off = np.zeros(nu.value + 1, dtype=np.int64)
    vert = np.zeros(max(nv.value, 1), dtype=np.int32)
    clo = np.zeros(max(nu.value, 1), dtype=np.int32)
    _check(lib.tpgen_shard_unit_paths(_p64(so), _p32(st), n, rank, count, _p64(off), _p32(vert), _p32(clo),
                                      nu.value, nv.value, ctypes.byref(nu), ctypes.byref(nv)))
    return [(tuple(vert[off[i]:off[i + 1]].tolist()), bool(clo[i])) for i in range(nu.value)]


def release_cache() -> None:
    """Frees what one-shot calls keep between calls (``tpgen_release_cache``): the cached plan and
    its device workspaces per device, the cached output blocks; trims the device memory pool."""
    library().tpgen_release_cache()


@dataclass
class CSRGraph:
    """A CSR graph returned by the library (host arrays)."""
    n: int
    offsets: np.ndarray
    targets: np.ndarray
    origin: np.ndarray  # normalize_outdeg2: the input vertex each vertex stands for
    name: str = ""


def normalize_outdeg2(graph) -> CSRGraph:
    """Out-degree-2 normalization (``tpgen_normalize_outdeg2``, host C++; PAPER.md P:272-290,
    Fig. 5): every vertex with d > 2 successors w1 < ... < wd keeps v -> w1 and gets a chain of
    d - 2 new vertices x_i -> w_{i+1}, x_{i+1} (the last one -> w_{d-1}, w_d)."""
    lib = library()
    so, st, n = _csr(graph)
    N, M = ctypes.c_int32(), ctypes.c_int64()
    z = ctypes.POINTER(ctypes.c_int64)()
    _check(lib.tpgen_normalize_outdeg2(_p64(so), _p32(st), n, ctypes.byref(N), ctypes.byref(M), z,
                                       ctypes.POINTER(ctypes.c_int32)(), ctypes.POINTER(ctypes.c_int32)()))
    off = np.zeros(N.value + 1, dtype=np.int64)
    tgt = np.zeros(max(M.value, 1), dtype=np.int32)
    org = np.zeros(max(N.value, 1), dtype=np.int32)
    _check(lib.tpgen_normalize_outdeg2(_p64(so), _p32(st), n, ctypes.byref(N), ctypes.byref(M), _p64(off),
                                       _p32(tgt), _p32(org)))
    return CSRGraph(int(N.value), off, tgt[:M.value], org[:N.value],
                    name=getattr(graph, "name", "graph") + "-outdeg2")


NPATH_STATUS = {0: "exact", 1: "saturated at 2^62", 2: "not computed (cyclic, search budget exceeded)"}


def metrics(graph, start: Optional[int] = None, end: Optional[int] = None) -> Dict[str, Any]:
    """Structure metrics of Table 1 from ``tpgen_metrics_compute`` (host
    C++): Nodes, Edges, SCCs (nontrivial), SccNodes, SccEdges, weakly connected components P,
    CC = E - V + 2P and Npath = start -> end walks using every arc at most once
    (P:592-601).  ``start`` / ``end`` default to the graph's entry / exit."""
    lib = library()
    so, st, n = _csr(graph)
    start = getattr(graph, "entry", 0) if start is None else start
    end = getattr(graph, "exit", n - 1) if end is None else end
    if n and (start is None or start < 0):
        start = 0
    if n and (end is None or end < 0):
        end = n - 1
    m = _abi.Metrics()
    _check(lib.tpgen_metrics_compute(_p64(so), _p32(st), n, int(start or 0), int(end or 0), ctypes.byref(m)))
    return {"nodes": m.nodes, "edges": m.edges, "sccs": m.sccs, "scc_nodes": m.scc_nodes,
            "scc_edges": m.scc_edges, "weak_components": m.weak_components, "cc": m.cc, "npath": int(m.npath),
            "npath_status": NPATH_STATUS[m.npath_status]}


class Plan:
    """Host plan + device-resident graph tables (``tpgen_plan_create``); ``prime_paths()``
    then runs device-only (what bench.py times as ``value``)."""

    def __init__(self, graph, device: int = 0, stream=None):
        lib = library()
        so, st, n = _csr(graph)
        self.device = device
        self.n = n
        o = _options(device, "device", "materialize", (0, 1), False, 0, 0, _stream_handle(device, stream), None)
        h = ctypes.c_void_p()
        _check(lib.tpgen_plan_create(_p64(so), _p32(st), n, ctypes.byref(o), ctypes.byref(h)))
        self._h = h

    def prime_paths(self, *, output: str = "device", mode: str = "materialize", shard: Tuple[int, int] = (0, 1),
                    digest: bool = False, max_paths: int = 0, stream=None, host_out=None,
                    start_range: Optional[Tuple[int, int]] = None, engine: str = "dfs",
                    shard_prefix: bool = False, prune: bool = False) -> PathSet:
        lib = library()
        alloc = None
        o = _options(self.device, output, mode, shard, digest, max_paths, 0, _stream_handle(self.device, stream),
                     alloc, host_out, start_range, engine, shard_prefix=shard_prefix, prune=prune)
        paths, stats = _abi.Paths(), _abi.Stats()
        _check(lib.tpgen_plan_prime_paths(self._h, ctypes.byref(o), ctypes.byref(paths), ctypes.byref(stats)))
        return _wrap(paths, stats, alloc, host_out)

    def test_paths(self, entry: int, exit: int, prime: Optional[PathSet] = None, *, output: str = "device",
                   stream=None, cover: str = "per_pp", mode: str = "materialize") -> PathSet:
        """Test paths of the plan's graph (tpgen_plan_test_paths): no re-planning per call."""
        lib = library()
        o = _options(self.device, output, mode, (0, 1), mode == "count", 0, 0,
                     _stream_handle(self.device, stream), None)
        o.tp_mode = _tp_mode(cover)
        keep = []
        pin = _paths_in(prime, self.device, keep)
        paths, stats = _abi.Paths(), _abi.Stats()
        _check(lib.tpgen_plan_test_paths(self._h, ctypes.byref(pin) if pin is not None else None, entry, exit,
                                         ctypes.byref(o), ctypes.byref(paths), ctypes.byref(stats)))
        return _wrap(paths, stats, None)

    def classify(self, prime: PathSet, start: int, end: int, stream=None) -> Dict[str, int]:
        """Five-class report of a prime-path list (tpgen_plan_classify; R19)."""
        lib = library()
        o = _options(self.device, "device", "materialize", (0, 1), False, 0, 0, _stream_handle(self.device, stream),
                     None)
        keep = []
        pin = _paths_in(prime, self.device, keep)
        counts = (ctypes.c_int64 * 5)()
        _check(lib.tpgen_plan_classify(self._h, ctypes.byref(pin), start, end, ctypes.byref(o), counts))
        return dict(zip(("complete", "entry", "exit", "internal", "transit"), (int(c) for c in counts)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            library().tpgen_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
