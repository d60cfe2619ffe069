"""Seeded CFG generators (no method arithmetic; see package docstring).

Recipes follow SURVEY.md §8(d) "Configs as concrete synthetic inputs" and
Appendix A/B; DESIGN.md §"Input recipe" restates them.  All randomness comes
from ``numpy.random.default_rng(seed)`` so every graph is reproducible.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


@dataclass
class Graph:
    """Successor CSR of a directed graph; rows sorted ascending, no duplicate arcs."""

    n: int
    offsets: np.ndarray  # int64[n+1]
    targets: np.ndarray  # int32[m]
    entry: int = -1      # Start vertex (TP entry), -1 if none
    exit: int = -1       # End vertex (TP exit), -1 if none
    name: str = ""
    meta: Dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.targets.shape[0])

    def succ(self, v: int) -> np.ndarray:
        return self.targets[self.offsets[v]:self.offsets[v + 1]]

    def arcs(self) -> List[Tuple[int, int]]:
        out = []
        for v in range(self.n):
            for w in self.succ(v):
                out.append((v, int(w)))
        return out


def from_arcs(n: int, arcs: Sequence[Tuple[int, int]], entry: int = -1, exit: int = -1,
              name: str = "", meta: Optional[Dict] = None) -> Graph:
    rows: List[set] = [set() for _ in range(n)]
    for a, b in arcs:
        if not (0 <= a < n and 0 <= b < n):
            raise ValueError(f"arc {(a, b)} out of range for n={n}")
        rows[a].add(int(b))
    offsets = np.zeros(n + 1, dtype=np.int64)
    tg: List[int] = []
    for v in range(n):
        r = sorted(rows[v])
        tg.extend(r)
        offsets[v + 1] = offsets[v] + len(r)
    return Graph(n, offsets, np.asarray(tg, dtype=np.int32), entry, exit, name, dict(meta or {}))


# ----------------------------------------------------------------------------
# Config 1: the paper's worked example, Fig. 1(b) (arcs
# recovered from the paths quoted at P:129-185).
# Ids: Start=0, blocks 1..9, End=10.
# ----------------------------------------------------------------------------
FIG1B_ARCS = [(0, 1), (1, 2), (2, 3), (2, 9), (3, 4), (3, 5), (4, 8), (5, 6), (5, 7),
              (6, 8), (8, 2), (9, 10), (7, 10)]


def fig1b() -> Graph:
    return from_arcs(11, FIG1B_ARCS, entry=0, exit=10, name="config1_fig1b")


# ----------------------------------------------------------------------------
# Structured-program CFGs (configs 2 and 4): grammar {block, if, if-else,
# while, do-while} with optional conditional break/continue arcs.
# ----------------------------------------------------------------------------
class _Builder:
    def __init__(self, rng: np.random.Generator):
        self.rng = rng
        self.n = 0
        self.arcs: List[Tuple[int, int]] = []

    def new(self) -> int:
        self.n += 1
        return self.n - 1

    def arc(self, a: int, b: int) -> None:
        self.arcs.append((a, b))


def _stmt(b: _Builder, cur: int, depth: int, loops: List[Tuple[int, int]],
          allow_loops: bool, p_brk: float, p_cont: float, max_seq: int) -> int:
    rng = b.rng
    kinds = ["block", "if", "ifelse"]
    if allow_loops and depth > 0:
        kinds += ["while", "dowhile"]
    if depth <= 0:
        kinds = ["block"]
    k = kinds[int(rng.integers(len(kinds)))]
    if k == "block":
        v = b.new()
        b.arc(cur, v)
        if loops:
            head, lexit = loops[-1]
            if rng.random() < p_brk:
                b.arc(v, lexit)
            elif rng.random() < p_cont:
                b.arc(v, head)
        return v
    if k in ("if", "ifelse"):
        t0 = b.new()
        b.arc(cur, t0)
        t1 = _seq(b, t0, depth - 1, loops, allow_loops, p_brk, p_cont, max_seq)
        j = b.new()
        b.arc(t1, j)
        if k == "if":
            b.arc(cur, j)
        else:
            e0 = b.new()
            b.arc(cur, e0)
            e1 = _seq(b, e0, depth - 1, loops, allow_loops, p_brk, p_cont, max_seq)
            b.arc(e1, j)
        return j
    if k == "while":
        h = b.new()
        b.arc(cur, h)
        x = b.new()
        b0 = b.new()
        b.arc(h, b0)
        b1 = _seq(b, b0, depth - 1, loops + [(h, x)], allow_loops, p_brk, p_cont, max_seq)
        b.arc(b1, h)
        b.arc(h, x)
        return x
    # do-while
    b0 = b.new()
    b.arc(cur, b0)
    c = b.new()
    x = b.new()
    b1 = _seq(b, b0, depth - 1, loops + [(c, x)], allow_loops, p_brk, p_cont, max_seq)
    b.arc(b1, c)
    b.arc(c, b0)
    b.arc(c, x)
    return x


def _seq(b: _Builder, cur: int, depth: int, loops, allow_loops, p_brk, p_cont, max_seq) -> int:
    cnt = 1 + int(b.rng.integers(max_seq))
    for _ in range(cnt):
        cur = _stmt(b, cur, depth, loops, allow_loops, p_brk, p_cont, max_seq)
    return cur


def structured_cfg(seed: int, depth: int = 4, max_seq: int = 3, p_brk: float = 0.06,
                   p_cont: float = 0.06, allow_loops: bool = True) -> Graph:
    rng = np.random.default_rng(seed)
    b = _Builder(rng)
    s = b.new()
    last = _seq(b, s, depth, [], allow_loops, p_brk, p_cont, max_seq)
    e = b.new()
    b.arc(last, e)
    g = from_arcs(b.n, b.arcs, entry=s, exit=e, name=f"structured_s{seed}")
    g.meta["cc"] = g.m - g.n + 2
    return g


def config2(seed0: int = 0) -> Graph:
    """first seed with V in [50,75] and CC=E-V+2 in [15,26]."""
    seed = seed0
    while True:
        g = structured_cfg(seed)
        cc = g.m - g.n + 2
        if 50 <= g.n <= 75 and 15 <= cc <= 26:
            g.name = f"config2_structured_s{seed}"
            g.meta.update(seed=seed, cc=cc)
            return g
        seed += 1


# ----------------------------------------------------------------------------
# Dense random SCCs (config 3) -- exact out-degree d, no self-loops,
# successors uniform without replacement, rejection until strongly connected.
# ----------------------------------------------------------------------------
def _strongly_connected(n: int, succ: List[List[int]]) -> bool:
    if n == 0:
        return True
    pred: List[List[int]] = [[] for _ in range(n)]
    for v in range(n):
        for w in succ[v]:
            pred[w].append(v)
    for adj in (succ, pred):
        seen = [False] * n
        seen[0] = True
        st = [0]
        while st:
            v = st.pop()
            for w in adj[v]:
                if not seen[w]:
                    seen[w] = True
                    st.append(w)
        if not all(seen):
            return False
    return True


def dense_scc(n: int, d: int, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    while True:
        succ = []
        for v in range(n):
            others = [u for u in range(n) if u != v]
            pick = rng.choice(len(others), size=d, replace=False)
            succ.append(sorted(others[i] for i in pick))
        if _strongly_connected(n, succ):
            break
    arcs = [(v, w) for v in range(n) for w in succ[v]]
    return from_arcs(n, arcs, entry=0, exit=n - 1, name=f"dense_n{n}_d{d}_s{seed}",
                     meta=dict(seed=seed, n_scc=n, d=d))


CONFIG3_SEED = 1


def config3(seed: int = CONFIG3_SEED) -> Graph:
    """single dense SCC, n=22, exact out-degree 4."""
    g = dense_scc(22, 4, seed)
    g.name = f"config3_dense22_d4_s{seed}"
    return g


# ----------------------------------------------------------------------------
# Config 4: chain of K while loops with structured depth-1 bodies and
# straight-line glue.
# ----------------------------------------------------------------------------
def loop_chain(K: int, seed: int, body_depth: int = 1, glue_max: int = 12,
               body_max_seq: int = 3) -> Graph:
    rng = np.random.default_rng(seed)
    b = _Builder(rng)
    start = b.new()
    cur = start
    for _ in range(K):
        for _ in range(int(rng.integers(glue_max + 1))):
            v = b.new()
            b.arc(cur, v)
            cur = v
        h = b.new()
        b.arc(cur, h)
        b0 = b.new()
        b.arc(h, b0)
        b1 = _seq(b, b0, body_depth, [], False, 0.0, 0.0, body_max_seq)
        b.arc(b1, h)
        cur = h
    for _ in range(int(rng.integers(glue_max + 1))):
        v = b.new()
        b.arc(cur, v)
        cur = v
    end = b.new()
    b.arc(cur, end)
    g = from_arcs(b.n, b.arcs, entry=start, exit=end, name=f"loopchain_K{K}_s{seed}")
    g.meta.update(K=K, seed=seed, cc=g.m - g.n + 2)
    return g


def config4(seed: int = 0, K: int = 150) -> Graph:
    g = loop_chain(K, seed)
    g.name = f"config4_loopchain_K{K}_s{seed}"
    return g


# ----------------------------------------------------------------------------
# Config 5: Start -> d1 -> ... -> dK -> J -> End; d_i -> SCC_i.v0;
# SCC_i.v(n-1) -> J.  Each SCC_i: random Hamiltonian cycle plus one extra
# random arc per vertex (strongly connected, out-degree 2, no self-loops).
# ----------------------------------------------------------------------------
def _ham_plus_one(n: int, rng: np.random.Generator) -> List[List[int]]:
    perm = rng.permutation(n)
    succ: List[set] = [set() for _ in range(n)]
    for i in range(n):
        succ[int(perm[i])].add(int(perm[(i + 1) % n]))
    for v in range(n):
        while len(succ[v]) < 2:
            w = int(rng.integers(n))
            if w != v:
                succ[v].add(w)
    return [sorted(s) for s in succ]


def parallel_sccs(K: int, n: int, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    start = 0
    ds = list(range(1, K + 1))
    base = K + 1
    J = base + K * n
    end = J + 1
    arcs: List[Tuple[int, int]] = []
    prev = start
    for d in ds:
        arcs.append((prev, d))
        prev = d
    arcs.append((prev, J))
    arcs.append((J, end))
    for i in range(K):
        off = base + i * n
        succ = _ham_plus_one(n, rng)
        for v in range(n):
            for w in succ[v]:
                arcs.append((off + v, off + w))
        arcs.append((ds[i], off + 0))
        arcs.append((off + n - 1, J))
    g = from_arcs(end + 1, arcs, entry=start, exit=end, name=f"parallel_K{K}_n{n}_s{seed}")
    g.meta.update(K=K, n_scc=n, seed=seed, cc=g.m - g.n + 2)
    return g


def config5(K: int = 16, n: int = 56, seed: int = 5) -> Graph:
    g = parallel_sccs(K, n, seed)
    g.name = f"config5_parallel_K{K}_n{n}_s{seed}"
    return g


# ----------------------------------------------------------------------------
# Small graphs for the oracle pins and the random parity corpus.
# ----------------------------------------------------------------------------
def random_digraph(n: int, p: float, seed: int, self_loops: bool = True) -> Graph:
    rng = np.random.default_rng(seed)
    arcs = []
    for a in range(n):
        for b in range(n):
            if a == b and not self_loops:
                continue
            if rng.random() < p:
                arcs.append((a, b))
    return from_arcs(n, arcs, name=f"rand_n{n}_p{p}_s{seed}")


def disjoint_union(graphs: Sequence[Graph], name: str = "") -> Graph:
    arcs = []
    base = 0
    for g in graphs:
        for a, b in g.arcs():
            arcs.append((a + base, b + base))
        base += g.n
    out = from_arcs(base, arcs, name=name or "union")
    return out


def k_nested_if(K: int) -> Graph:
    """K nested if-then: Start=c_1, c_i -> c_{i+1} (then), c_i -> j_i (skip),
    innermost then-block t -> j_K, j_i -> j_{i-1}, j_1 -> End."""
    # vertices: c_1..c_K = 0..K-1, t = K, j_K..j_1 = K+1..2K, End = 2K+1
    arcs = []
    c = list(range(K))
    t = K
    j = {i: 2 * K - i + 1 for i in range(1, K + 1)}  # j_K = K+1, j_1 = 2K
    end = 2 * K + 1
    for i in range(1, K + 1):
        nxt = c[i] if i < K else t
        arcs.append((c[i - 1], nxt))
        arcs.append((c[i - 1], j[i]))
    arcs.append((t, j[K]))
    for i in range(K, 1, -1):
        arcs.append((j[i], j[i - 1]))
    arcs.append((j[1], end))
    return from_arcs(2 * K + 2, arcs, entry=0, exit=end, name=f"nested_if_K{K}")


def k_seq_if(K: int) -> Graph:
    """K if-then in sequence: c_i -> t_i -> c_{i+1}, c_i -> c_{i+1}."""
    arcs = []
    # c_i = 2i, t_i = 2i+1 for i in 0..K-1, End = 2K
    for i in range(K):
        c, t, nxt = 2 * i, 2 * i + 1, 2 * i + 2
        arcs += [(c, t), (t, nxt), (c, nxt)]
    return from_arcs(2 * K + 1, arcs, entry=0, exit=2 * K, name=f"seq_if_K{K}")


def single_loop(K: int) -> Graph:
    """Pure K-cycle: 0 -> 1 -> ... -> K-1 -> 0."""
    arcs = [(i, (i + 1) % K) for i in range(K)]
    return from_arcs(K, arcs, name=f"cycle_K{K}")


def k_seq_loops(K: int, N: int) -> Graph:
    """K loops in sequence, each header + N-1 body vertices (SURVEY §4.1 wiring):
    Start -> h_1, h_i -> body_i,1 -> ... -> body_i,N-1 -> h_i, h_i -> h_{i+1}, h_K -> End."""
    arcs = []
    start = 0
    nxt_id = 1
    heads = []
    bodies = []
    for _ in range(K):
        h = nxt_id
        nxt_id += 1
        bd = list(range(nxt_id, nxt_id + N - 1))
        nxt_id += N - 1
        heads.append(h)
        bodies.append(bd)
    end = nxt_id
    arcs.append((start, heads[0]))
    for i in range(K):
        chain = [heads[i]] + bodies[i] + [heads[i]]
        for a, b in zip(chain[:-1], chain[1:]):
            arcs.append((a, b))
        arcs.append((heads[i], heads[i + 1] if i + 1 < K else end))
    return from_arcs(end + 1, arcs, entry=start, exit=end, name=f"seq_loops_K{K}_N{N}")


def random_dag_cfg(n: int, seed: int, extra: float = 0.3) -> Graph:
    """Random DAG where every vertex lies on a Start(0) -> End(n-1) path."""
    rng = np.random.default_rng(seed)
    arcs = set()
    for v in range(1, n):
        arcs.add((int(rng.integers(v)), v))           # a predecessor
    for v in range(n - 1):
        arcs.add((v, int(rng.integers(v + 1, n))))    # a successor
    for _ in range(int(extra * n)):
        a = int(rng.integers(n - 1))
        b = int(rng.integers(a + 1, n))
        arcs.add((a, b))
    return from_arcs(n, sorted(arcs), entry=0, exit=n - 1, name=f"dag_n{n}_s{seed}")


CONFIGS = {
    1: "paper's worked-example CFG (Fig. 1(b))",
    2: "synthetic structured CFG ~60 vertices, cyclomatic ~20",
    3: "single dense SCC of 22 vertices, exact out-degree 4",
    4: "chain of 150 while loops, ~2000 vertices, 150 SCCs",
    5: "parallel 56-vertex out-degree-2 SCCs behind a dispatch chain (high Npath)",
}


def make_config(idx: int, **kw) -> Graph:
    return {1: fig1b, 2: config2, 3: config3, 4: config4, 5: config5}[idx](**kw)
