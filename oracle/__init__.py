"""CPU oracle for TPGen's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2210_16998_b200``) never imports it and shares no code
with it.

Contents
  * ``oracle.c`` (tier 1): DFS prime-path enumerator following Def. 1
     with the operational maximality test, E_canon counter,
    digest, lexmin-shortest prefix/suffix tables for test paths.
  * ``brute.py`` (tier 0): the definition itself -- all simple paths, minus the
    proper contiguous subpaths of other simple paths -- for tiny graphs.
  * this module: ctypes wrappers + test-path assembly (a plain loop).

Parity status: PP set, E_canon, digest and the TP
prefix/suffix tables are pinned by tests/test_oracle.py (worked example P:230-255,
closed forms P:626-643, DAG = Npath P:604, tier-0 brute force, brute-force
lexmin walks, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        lib.oracle_prime_paths.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32),
                                           ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           P(P(ctypes.c_int64)), P(P(ctypes.c_int32)),
                                           P(ctypes.c_int64), P(ctypes.c_int64)]
        lib.oracle_prime_paths.restype = ctypes.c_int
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        lib.oracle_ext_count.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32),
                                         ctypes.c_int32, ctypes.c_int32]
        lib.oracle_ext_count.restype = ctypes.c_int64
        lib.oracle_scc_labels.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32),
                                          P(ctypes.c_int32)]
        lib.oracle_digest.argtypes = [ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int32),
                                      P(ctypes.c_uint64)]
        lib.oracle_tp_tables.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32),
                                         ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int32),
                                         P(ctypes.c_int32), P(ctypes.c_int32), P(ctypes.c_int32)]
        lib.oracle_pp_stats.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32), ctypes.c_int32,
                                        ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_uint64)]
        lib.oracle_pp_stats.restype = ctypes.c_int
        lib.oracle_tp_stats.argtypes = [ctypes.c_int32, P(ctypes.c_int64), P(ctypes.c_int32), ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P(ctypes.c_int64),
                                        P(ctypes.c_uint64)]
        lib.oracle_tp_stats.restype = ctypes.c_int
        _lib = lib
    return _lib


def _csr(g):
    so = np.ascontiguousarray(g.offsets, dtype=np.int64)
    st = np.ascontiguousarray(g.targets, dtype=np.int32)
    if st.size == 0:
        st = np.zeros(1, dtype=np.int32)
    return so, st


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def prime_paths(g, v_lo: int = 0, v_hi: Optional[int] = None, prunes: bool = True
                ) -> Tuple[np.ndarray, np.ndarray]:
    """Prime paths with first vertex in [v_lo, v_hi), lexicographic order.

    Returns (offsets int64[n_paths+1] starting at 0, vertices int32)."""
    lib = _load()
    so, st = _csr(g)
    v_hi = g.n if v_hi is None else v_hi
    po = ctypes.POINTER(ctypes.c_int64)()
    pv = ctypes.POINTER(ctypes.c_int32)()
    npaths = ctypes.c_int64()
    nvert = ctypes.c_int64()
    rc = lib.oracle_prime_paths(g.n, _p64(so), _p32(st), v_lo, v_hi, int(prunes), ctypes.byref(po),
                                ctypes.byref(pv), ctypes.byref(npaths), ctypes.byref(nvert))
    if rc != 0:
        raise MemoryError("oracle_prime_paths failed")
    try:
        off = np.ctypeslib.as_array(po, shape=(npaths.value + 1,)).copy()
        vert = (np.ctypeslib.as_array(pv, shape=(nvert.value,)).copy() if nvert.value
                else np.zeros(0, dtype=np.int32))
    finally:
        lib.oracle_free(ctypes.cast(po, ctypes.c_void_p))
        lib.oracle_free(ctypes.cast(pv, ctypes.c_void_p))
    return off, vert


def ext_count(g, v_lo: int = 0, v_hi: Optional[int] = None) -> int:
    """E_canon restricted to start vertices in [v_lo, v_hi)."""
    lib = _load()
    so, st = _csr(g)
    return int(lib.oracle_ext_count(g.n, _p64(so), _p32(st), v_lo, g.n if v_hi is None else v_hi))


def scc_labels(g) -> np.ndarray:
    lib = _load()
    so, st = _csr(g)
    lab = np.zeros(max(g.n, 1), dtype=np.int32)
    lib.oracle_scc_labels(g.n, _p64(so), _p32(st), _p32(lab))
    return lab[:g.n]


def digest(offsets: np.ndarray, vertices: np.ndarray) -> Tuple[int, int]:
    lib = _load()
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    vert = np.ascontiguousarray(vertices, dtype=np.int32)
    if vert.size == 0:
        vert = np.zeros(1, dtype=np.int32)
    out = (ctypes.c_uint64 * 2)()
    lib.oracle_digest(off.shape[0] - 1, _p64(off), _p32(vert), out)
    return int(out[0]), int(out[1])


def pp_stats(g, v_lo: int = 0, v_hi: Optional[int] = None, tp: Optional[Tuple[int, int]] = None) -> np.ndarray:
    """Per start vertex v in [v_lo, v_hi): (n_paths, n_vertices, hash_lo, hash_hi) of the prime
    paths whose first vertex is v -- or, with ``tp=(entry, exit)``, of their test paths (R15) --
    hashed while they are enumerated (oracle_pp_stats / oracle_tp_stats; nothing stored).
    Returns a uint64 array [v_hi - v_lo, 4]."""
    lib = _load()
    so, st = _csr(g)
    v_hi = g.n if v_hi is None else v_hi
    k = max(v_hi - v_lo, 0)
    cnt = np.zeros(2 * max(k, 1), dtype=np.int64)
    hs = np.zeros(2 * max(k, 1), dtype=np.uint64)
    ph = hs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    if tp is None:
        rc = lib.oracle_pp_stats(g.n, _p64(so), _p32(st), v_lo, v_hi, _p64(cnt), ph)
    else:
        rc = lib.oracle_tp_stats(g.n, _p64(so), _p32(st), v_lo, v_hi, int(tp[0]), int(tp[1]), _p64(cnt), ph)
    if rc == -2:
        raise ValueError("a prime path's endpoints are unreachable from entry / to exit")
    if rc != 0:
        raise MemoryError("oracle_pp_stats failed")
    out = np.zeros((k, 4), dtype=np.uint64)
    out[:, 0] = cnt[0:2 * k:2]
    out[:, 1] = cnt[1:2 * k:2]
    out[:, 2] = hs[0:2 * k:2]
    out[:, 3] = hs[1:2 * k:2]
    return out


def _stats_worker(a):
    n, so, st, lo, hi, tp = a

    class _G:
        pass

    g = _G()
    g.n, g.offsets, g.targets = n, so, st
    rows = pp_stats(g, lo, hi, tp)
    ext = np.asarray([ext_count(g, v, v + 1) for v in range(lo, hi)], dtype=np.uint64).reshape(-1, 1)
    return lo, np.concatenate([rows, ext], axis=1)


def pp_stats_parallel(g, v_lo: int = 0, v_hi: Optional[int] = None, tp: Optional[Tuple[int, int]] = None,
                      procs: Optional[int] = None, chunk: int = 4) -> np.ndarray:
    """``pp_stats`` over [v_lo, v_hi) split into blocks of ``chunk`` start vertices, run on
    ``procs`` host processes (the per-start enumerations are independent), plus a fifth
    column: each start vertex's E_canon (``ext_count``).  uint64 array [v_hi - v_lo, 5]."""
    import multiprocessing as mp

    v_hi = g.n if v_hi is None else v_hi
    procs = procs or max(1, os.cpu_count() or 1)
    so, st = _csr(g)
    jobs = [(g.n, so, st, lo, min(lo + chunk, v_hi), tp) for lo in range(v_lo, v_hi, chunk)]
    out = np.zeros((max(v_hi - v_lo, 0), 5), dtype=np.uint64)
    if not jobs:
        return out
    build()
    with mp.get_context("spawn").Pool(min(procs, len(jobs))) as pool:
        for lo, part in pool.imap_unordered(_stats_worker, jobs):
            out[lo - v_lo: lo - v_lo + part.shape[0]] = part
    return out


def tp_tables(g, entry: int, exit: int):
    """Lexmin-shortest prefix (entry->v) and suffix (v->exit) walks per vertex.

    Returns (pre: list[list[int] | None], suf: list[list[int] | None])."""
    lib = _load()
    so, st = _csr(g)
    n = g.n
    pre_len = np.zeros(n, dtype=np.int32)
    suf_len = np.zeros(n, dtype=np.int32)
    pre_tab = np.zeros(n * n, dtype=np.int32)
    suf_tab = np.zeros(n * n, dtype=np.int32)
    lib.oracle_tp_tables(n, _p64(so), _p32(st), entry, exit, _p32(pre_len), _p32(pre_tab),
                         _p32(suf_len), _p32(suf_tab))
    pre = [None if pre_len[v] < 0 else pre_tab[v * n: v * n + pre_len[v]].tolist() for v in range(n)]
    suf = [None if suf_len[v] < 0 else suf_tab[v * n: v * n + suf_len[v]].tolist() for v in range(n)]
    return pre, suf


def test_paths(g, offsets: np.ndarray, vertices: np.ndarray, entry: int, exit: int
               ) -> Tuple[np.ndarray, np.ndarray]:
    """TP_i = prefix[first_i][:-1] + PP_i + suffix[last_i][1:], aligned with the PP list
    (reading R15).  Raises ValueError if an endpoint is unreachable."""
    pre, suf = tp_tables(g, entry, exit)
    out_off = [0]
    out_v = []
    for i in range(len(offsets) - 1):
        p = vertices[offsets[i]:offsets[i + 1]].tolist()
        a, b = pre[p[0]], suf[p[-1]]
        if a is None or b is None:
            raise ValueError(f"PP {i} endpoints unreachable from entry / to exit")
        tp = a[:-1] + p + b[1:]
        out_v.extend(tp)
        out_off.append(len(out_v))
    return np.asarray(out_off, dtype=np.int64), np.asarray(out_v, dtype=np.int32)


def unique_test_paths(g, offsets: np.ndarray, vertices: np.ndarray, entry: int, exit: int
                      ) -> Tuple[np.ndarray, np.ndarray]:
    """K7: the distinct test paths of ``test_paths`` -- "the set of TPs
    covering all PPs" -- in lexicographic order of the vertex sequences
    (R14: Python's list order, a proper prefix first)."""
    to, tv = test_paths(g, offsets, vertices, entry, exit)
    tps = sorted({tuple(tv[to[i]:to[i + 1]].tolist()) for i in range(len(to) - 1)})
    out_off = np.zeros(len(tps) + 1, dtype=np.int64)
    for i, t in enumerate(tps):
        out_off[i + 1] = out_off[i] + len(t)
    out_v = np.array([x for t in tps for x in t], dtype=np.int32)
    return out_off, out_v


def _contains(t, q) -> bool:
    """q is a contiguous subsequence of t (plain scan)."""
    m = len(q)
    for i in range(len(t) - m + 1):
        if t[i:i + m] == q:
            return True
    return False


def greedy_test_paths(g, offsets: np.ndarray, vertices: np.ndarray, entry: int, exit: int
                      ) -> Tuple[np.ndarray, np.ndarray]:
    """Greedy test-path cover ("starts with the
    longest PP ... extends every PP to visit initial and final nodes").
    Prime paths in order of decreasing length, ties in canonical (lexicographic)
    order; the first one not yet covered becomes TP = prefix ++ PP ++ suffix (the
    R15 walks); every prime path that is a contiguous subpath of that TP is covered.
    Plain loops with a naive containment scan -- small graphs only."""
    pre, suf = tp_tables(g, entry, exit)
    pps = [vertices[offsets[i]:offsets[i + 1]].tolist() for i in range(len(offsets) - 1)]
    order = sorted(range(len(pps)), key=lambda i: (-len(pps[i]), i))
    covered = [False] * len(pps)
    out_off, out_v = [0], []
    for i in order:
        if covered[i]:
            continue
        p = pps[i]
        a, b = pre[p[0]], suf[p[-1]]
        if a is None or b is None:
            raise ValueError(f"PP {i} endpoints unreachable from entry / to exit")
        tp = a[:-1] + p + b[1:]
        out_v.extend(tp)
        out_off.append(len(out_v))
        for j, q in enumerate(pps):
            if not covered[j] and len(q) <= len(tp) and _contains(tp, q):
                covered[j] = True
    return np.asarray(out_off, dtype=np.int64), np.asarray(out_v, dtype=np.int32)


def as_list(offsets: np.ndarray, vertices: np.ndarray):
    return [tuple(vertices[offsets[i]:offsets[i + 1]].tolist()) for i in range(len(offsets) - 1)]


PP_CLASSES = ("complete", "entry", "exit", "internal", "transit")


def pp_class(first: int, last: int, start: int, end: int, scc: np.ndarray) -> str:
    """The paper's PP taxonomy (reading R19): complete = Start ... End
    (Def. 2); entry = from Start into an SCC (Def. 11, P:182-186 read as
    Start -> SCC, R7); exit = from an SCC to End (Def. 10); internal = inside one SCC
    (Def. 9); transit = SCC -> SCC, the class Defs. 2-11 miss (R7).  A
    path cannot leave an SCC and come back, so "inside one SCC" is scc[first] ==
    scc[last]."""
    if first == start and last == end:
        return "complete"
    if first == start:
        return "entry"
    if last == end:
        return "exit"
    if scc[first] == scc[last]:
        return "internal"
    return "transit"


def pp_classes(g, offsets: np.ndarray, vertices: np.ndarray, start: int, end: int):
    """Class of every prime path (a plain loop) and the counts per class."""
    scc = scc_labels(g)
    labels = []
    for i in range(len(offsets) - 1):
        a, b = int(offsets[i]), int(offsets[i + 1])
        labels.append(pp_class(int(vertices[a]), int(vertices[b - 1]), start, end, scc))
    counts = {c: 0 for c in PP_CLASSES}
    for c in labels:
        counts[c] += 1
    return labels, counts
