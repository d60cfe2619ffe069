"""Tier-0 oracle: Def. 1 written out literally (TEST INFRASTRUCTURE ONLY).

PAPER.md P:106 (simple path: v1..vk, k > 0, no repeated vertex unless v1 = vk),
P:127-130 (Def. 1: a PP is a maximal simple path), P:28 ("a simple path that is
not included in any other simple path").  "Included" is read as contiguous
subpath (reading R3).

Algorithm: enumerate every simple path (DFS from every vertex, extending the
tail; a step back to v1 closes a cycle and stops), collect every proper
contiguous subpath of every simple path, and return the simple paths that are
not in that collection.  Exponential -- tiny graphs only (n <= ~11).
"""
from __future__ import annotations

from typing import List, Sequence, Set, Tuple


def simple_paths(n: int, succ: Sequence[Sequence[int]]) -> List[Tuple[int, ...]]:
    out: List[Tuple[int, ...]] = []

    def rec(path: List[int]):
        out.append(tuple(path))
        if len(path) >= 2 and path[0] == path[-1]:
            return  # a closed cycle cannot be extended and stay simple
        for w in succ[path[-1]]:
            if w == path[0] or w not in path:
                path.append(w)
                rec(path)
                path.pop()

    for v in range(n):
        rec([v])
    return out


def prime_paths(n: int, succ: Sequence[Sequence[int]]) -> List[Tuple[int, ...]]:
    sp = simple_paths(n, succ)
    covered: Set[Tuple[int, ...]] = set()
    for q in sp:
        L = len(q)
        for i in range(L):
            for j in range(i + 1, L + 1):
                if j - i < L:
                    covered.add(q[i:j])
    return sorted(p for p in set(sp) if p not in covered)


def graph_succ(g) -> List[List[int]]:
    return [g.succ(v).tolist() for v in range(g.n)]


def lexmin_shortest_walk(succ, a: int, b: int):
    """Brute force: all walks a->b of minimum hop count; return the lexicographically
    smallest (for pinning the TP prefix/suffix rule).  None if unreachable."""
    frontier = [(a,)]
    seen_len = 0
    while frontier:
        done = [w for w in frontier if w[-1] == b]
        if done:
            return list(min(done))
        seen_len += 1
        if seen_len > len(succ) + 1:
            return None
        nxt = []
        for w in frontier:
            for x in succ[w[-1]]:
                nxt.append(w + (x,))
        frontier = nxt
    return None


def npath(n: int, succ: Sequence[Sequence[int]], start: int, end: int) -> int:
    """Npath written out: Npath(end, G) = 1 and
    Npath(v, G) = sum over arcs (v, w) of Npath(w, G - (v, w)) -- the number of start -> end
    walks that use every arc at most once, by plain recursion on the arc set.  Tiny graphs only."""
    def rec(v: int, removed: frozenset) -> int:
        if v == end:
            return 1
        total = 0
        for w in succ[v]:
            if (v, w) not in removed:
                total += rec(w, removed | {(v, w)})
        return total

    return rec(start, frozenset())
