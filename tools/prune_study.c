// prune_study.c -- host measurement behind DESIGN.md §6.5 "Reachability pruning"
// (SURVEY §8(f) NEXT #2): how many nodes of the per-start simple-path tries lie
// in subtrees that emit no prime path, and how many of them a reachability
// test removes at what cost.  Plain C, <= 64-vertex graphs; not part of the
// library.  Input: "n\n" then per vertex "d w1 .. wd" (successor lists), n <= 64.
//   gcc -O2 -o /tmp/prune_study tools/prune_study.c && /tmp/prune_study g.txt 20 [n_starts]
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

static int n, s, D;
static uint64_t sin_[64], pin_[64], ps;
static long long nodes, dead_roots, dead_nodes, tests, iters, pruned;

// emissions in the subtree of (u, M) including u's own event; *sub = its node count
static long long dfs_dead(int u, uint64_t M, int depth, long long *sub) {
    nodes++;
    long long e = 0, below = 0, bn = 0;
    const uint64_t c = sin_[u] & (~M | (1ull << s));
    if (depth > 0 && c == 0 && (ps & ~(M & ~(1ull << u))) == 0) e++;
    for (uint64_t cc = c; cc; cc &= cc - 1) {
        const int w = __builtin_ctzll(cc);
        if (w == s) { below++; continue; }
        long long k = 0;
        below += dfs_dead(w, M | (1ull << w), depth + 1, &k);
        bn += k;
    }
    if (below == 0 && bn > 0) { dead_roots++; dead_nodes += bn; }
    *sub = 1 + bn;
    return e + below;
}

static uint64_t reach(int u, uint64_t M) {
    uint64_t R = 0, F = sin_[u] & ~M;
    while (F) {
        const int v = __builtin_ctzll(F);
        F &= F - 1;
        iters++;
        if (R >> v & 1) continue;
        R |= 1ull << v;
        F |= sin_[v] & ~M & ~R;
    }
    return R;
}

// the same walk with the test applied at depths 1..D
static long long dfs_pruned(int u, uint64_t M, int depth) {
    nodes++;
    long long e = 0;
    const uint64_t c = sin_[u] & (~M | (1ull << s));
    if (depth > 0 && c == 0 && (ps & ~(M & ~(1ull << u))) == 0) e++;
    if (c && depth > 0 && depth <= D) {
        tests++;
        const uint64_t R = reach(u, M);
        const int closure_possible = ((ps >> u) & 1) || (ps & R);
        const int acyclic_possible = (ps & ~M & ~R) == 0;
        if (!closure_possible && !acyclic_possible) { pruned++; return e; }
    }
    for (uint64_t cc = c; cc; cc &= cc - 1) {
        const int w = __builtin_ctzll(cc);
        if (w == s) { e++; continue; }
        e += dfs_pruned(w, M | (1ull << w), depth + 1);
    }
    return e;
}

int main(int argc, char **argv) {
    if (argc < 3) return 2;
    FILE *f = fopen(argv[1], "r");
    if (!f || fscanf(f, "%d", &n) != 1 || n > 64) return 1;
    D = atoi(argv[2]);
    for (int v = 0; v < n; v++) {
        int d;
        if (fscanf(f, "%d", &d) != 1) return 1;
        for (int j = 0; j < d; j++) {
            int w;
            if (fscanf(f, "%d", &w) != 1) return 1;
            sin_[v] |= 1ull << w;
            pin_[w] |= 1ull << v;
        }
    }
    long long pp = 0, sub;
    for (s = 0; s < (argc > 3 ? atoi(argv[3]) : n); s++) { ps = pin_[s]; pp += dfs_dead(s, 1ull << s, 0, &sub); }
    printf("nodes %lld prime_paths %lld dead_subtree_roots %lld nodes_in_dead_subtrees %lld (%.1f%%)\n", nodes, pp,
           dead_roots, dead_nodes, 100.0 * dead_nodes / nodes);
    const long long all = nodes;
    nodes = 0;
    pp = 0;
    for (s = 0; s < (argc > 3 ? atoi(argv[3]) : n); s++) { ps = pin_[s]; pp += dfs_pruned(s, 1ull << s, 0); }
    printf("test at depth <= %d: nodes %lld (%.1f%% removed) prime_paths %lld tests %lld bfs_steps %lld pruned %lld\n", D,
           nodes, 100.0 * (all - nodes) / all, pp, tests, iters, pruned);
    return 0;
}
