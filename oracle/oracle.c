/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for TPGen's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * library.  It shares no code, header, table or constant generator with the
 * CUDA path in paper_2210_16998_b200/ (and never includes include/tpgen.h).
 *
 * What it computes (citations: PAPER.md line numbers, "P:n"):
 *   - PP(G): the prime paths of G.  A simple path v1..vk (k >= 1) may repeat
 *     only v1 = vk.  A prime path is a simple path that is not a proper
 *     (contiguous) subpath of another simple path (Def. 1; P:28
 *     "a simple path that is not included in any other simple path").
 *     Operational form used here (reading R3):
 *       * a cyclic path (k >= 2, v1 = vk) is always maximal;
 *       * an acyclic path is maximal iff every successor of vk lies in
 *         {v2..vk} and every predecessor of v1 lies in {v1..v(k-1)}
 *         (a proper super-path must extend p by one arc at its head or tail,
 *         and that one-arc extension is itself simple).
 *     Enumeration: for v1 = 0..n-1 ascending, DFS over simple paths starting
 *     at v1, successors ascending, extending at the tail only; a successor equal
 *     to v1 closes a cycle (emitted, never extended).  This is Ammann-Offutt's
 *     "extend while simple" generation with the maximality test applied
 *     per path instead of a final pairwise prune.  Emission order is therefore
 *     lexicographic (preorder of a successor-sorted trie over a prefix-free set).
 *   - Two exact prunes (both derived from Def. 1; tier-0 brute force in
 *     tests/ checks them on thousands of graphs):
 *       A'  if v1 has a predecessor outside SCC(v1), no acyclic path starting at
 *           v1 is maximal (that predecessor can be prepended: it cannot already
 *           be on the path, else it would share v1's SCC), so only cycles are
 *           searched, and cycles through v1 stay inside SCC(v1);
 *       B   once the path leaves SCC(v1) it can never return, so no cycle can
 *           close and head-closure (pred(v1) on the path) is frozen; if it does
 *           not hold at the step out, the subtree emits nothing.
 *     With use_prunes = 0 the plain search is run (slow; small graphs only).
 *   - SCCs for the prunes: mutual reachability by BFS from every vertex
 *     ("for any pair vi, vj ... reachable from each other").
 *   - E_canon: sum over nontrivial SCCs C (|C| > 1 or a self-loop) and s in C
 *     of the number of simple paths with >= 2 vertices inside C starting at s,
 *     cycle closures included (the number of ExtendPath calls of Alg. 4,
 *     P:459-472, restricted to one SCC).  Counted by its own DFS.
 *   - Digest: per path, S = sum over positions i of mix(i << 32 | v_i) and
 *     z = mix(S ^ (seed + len)); set digest = sum over paths mod 2^64
 *     (reading R20), two seeds.
 *   - Test paths: prefix[v] = lexicographically-first shortest
 *     walk entry -> v (BFS from entry, successors ascending, first discoverer is
 *     the parent); suffix[v] = v then repeatedly the smallest successor w with
 *     dist_to_exit[w] = dist_to_exit[cur] - 1.  TP_i = prefix[first_i] minus its
 *     last vertex, then PP_i, then suffix[last_i] minus its first vertex
 *     (reading R15).  parity of TPs is pinned by that rule only
 *     (the paper prints no TP); tests check it against brute-force lexmin walks.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t len, cap;
    int32_t *a;
} ovec32;
typedef struct {
    int64_t len, cap;
    int64_t *a;
} ovec64;

static int v32_push(ovec32 *v, int32_t x) {
    if (v->len == v->cap) {
        int64_t nc = v->cap ? v->cap * 2 : 1024;
        int32_t *na = (int32_t *)realloc(v->a, (size_t)nc * sizeof(int32_t));
        if (!na) return -1;
        v->a = na;
        v->cap = nc;
    }
    v->a[v->len++] = x;
    return 0;
}
static int v64_push(ovec64 *v, int64_t x) {
    if (v->len == v->cap) {
        int64_t nc = v->cap ? v->cap * 2 : 1024;
        int64_t *na = (int64_t *)realloc(v->a, (size_t)nc * sizeof(int64_t));
        if (!na) return -1;
        v->a = na;
        v->cap = nc;
    }
    v->a[v->len++] = x;
    return 0;
}

/* ---------------------------------------------------------------- graph */
typedef struct {
    int32_t n;
    const int64_t *so;  /* successor offsets */
    const int32_t *st;  /* successor targets (ascending per row) */
    int64_t *po;        /* predecessor offsets */
    int32_t *pt;        /* predecessor sources */
    int32_t *scc;       /* scc label (smallest member id) */
    uint8_t *nontriv;   /* per vertex: its SCC has >1 vertex or v has a self-loop */
} ograph;

static int g_init(ograph *g, int32_t n, const int64_t *so, const int32_t *st) {
    memset(g, 0, sizeof(*g));
    g->n = n;
    g->so = so;
    g->st = st;
    int64_t m = n ? so[n] : 0;
    g->po = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->pt = (int32_t *)malloc((size_t)(m ? m : 1) * sizeof(int32_t));
    g->scc = (int32_t *)malloc((size_t)(n ? n : 1) * sizeof(int32_t));
    g->nontriv = (uint8_t *)calloc((size_t)(n ? n : 1), 1);
    if (!g->po || !g->pt || !g->scc || !g->nontriv) return -1;
    for (int32_t v = 0; v < n; v++)
        for (int64_t e = so[v]; e < so[v + 1]; e++) g->po[st[e] + 1]++;
    for (int32_t v = 0; v < n; v++) g->po[v + 1] += g->po[v];
    int64_t *fill = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!fill) return -1;
    memcpy(fill, g->po, ((size_t)n + 1) * sizeof(int64_t));
    for (int32_t v = 0; v < n; v++) /* sources ascending because v ascends */
        for (int64_t e = so[v]; e < so[v + 1]; e++) g->pt[fill[st[e]]++] = v;
    free(fill);

    /* SCC by mutual reachability: reach[a*n+b] = b reachable from a. */
    uint8_t *reach = (uint8_t *)calloc((size_t)n * (size_t)n + 1, 1);
    int32_t *queue = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    if (!reach || !queue) return -1;
    for (int32_t a = 0; a < n; a++) {
        uint8_t *r = reach + (size_t)a * n;
        int64_t qh = 0, qt = 0;
        r[a] = 1;
        queue[qt++] = a;
        while (qh < qt) {
            int32_t v = queue[qh++];
            for (int64_t e = so[v]; e < so[v + 1]; e++) {
                int32_t w = st[e];
                if (!r[w]) { r[w] = 1; queue[qt++] = w; }
            }
        }
    }
    for (int32_t a = 0; a < n; a++) {
        g->scc[a] = a;
        for (int32_t b = 0; b < a; b++)
            if (reach[(size_t)a * n + b] && reach[(size_t)b * n + a]) { g->scc[a] = g->scc[b]; break; }
    }
    for (int32_t a = 0; a < n; a++) {
        for (int32_t b = 0; b < n; b++)
            if (b != a && g->scc[b] == g->scc[a]) g->nontriv[a] = 1;
        for (int64_t e = so[a]; e < so[a + 1]; e++)
            if (st[e] == a) g->nontriv[a] = 1;
    }
    free(reach);
    free(queue);
    return 0;
}

static void g_free(ograph *g) {
    free(g->po);
    free(g->pt);
    free(g->scc);
    free(g->nontriv);
}

/* -------------------------------------------------------------- digest */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}

#define SEED_A 0x9E3779B97F4A7C15ULL
#define SEED_B 0xD1B54A32D192ED03ULL

/* DESIGN.md reading R20: S = sum_i mix(v_i) * (2i + 1), path digest = mix(S ^ (seed + len)). */
static uint64_t path_hash(uint64_t seed, const int32_t *v, int64_t len) {
    uint64_t S = 0;
    for (int64_t i = 0; i < len; i++) S += mix64((uint64_t)(uint32_t)v[i]) * (2 * (uint64_t)i + 1);
    return mix64(S ^ (seed + (uint64_t)len));
}

/* ------------------------------------------------------- prime paths */
/* Test-path context of oracle_tp_stats: the prefix / suffix walks (R15). */
typedef struct {
    const int32_t *pre_len, *pre_tab, *suf_len, *suf_tab;
    int32_t n;
    int32_t *buf;  /* room for one test path (3n vertices) */
    int unreachable;
} otp;

typedef struct {
    ovec64 off;      /* path start offsets (n_paths + 1 once finished) */
    ovec32 vert;     /* concatenated vertices */
    int stats_only;  /* 1: hash every emitted path instead of storing it */
    int64_t n_paths, n_vert;
    uint64_t ha, hb;
    otp *tp;         /* non-NULL: hash the prime path's test path instead of the path */
} opaths;

static void hash_into(opaths *out, const int32_t *p, int64_t len) {
    out->n_paths++;
    out->n_vert += len;
    out->ha += path_hash(SEED_A, p, len);
    out->hb += path_hash(SEED_B, p, len);
}

/* Stats mode: the emitted prime path (closing vertex appended), or its test path
 * prefix[first] minus its last vertex ++ PP ++ suffix[last] minus its first vertex. */
static void emit_stats(opaths *out, const int32_t *path, int32_t k, int32_t closing) {
    otp *t = out->tp;
    int32_t last = closing >= 0 ? closing : path[k - 1];
    if (!t) {
        int32_t buf[k + 1];
        for (int32_t i = 0; i < k; i++) buf[i] = path[i];
        if (closing >= 0) buf[k] = closing;
        hash_into(out, buf, closing >= 0 ? k + 1 : k);
        return;
    }
    int32_t first = path[0];
    if (t->pre_len[first] < 0 || t->suf_len[last] < 0) {
        t->unreachable = 1;
        return;
    }
    int64_t m = 0;
    for (int32_t i = 0; i + 1 < t->pre_len[first]; i++) t->buf[m++] = t->pre_tab[(size_t)first * t->n + i];
    for (int32_t i = 0; i < k; i++) t->buf[m++] = path[i];
    if (closing >= 0) t->buf[m++] = closing;
    for (int32_t i = 1; i < t->suf_len[last]; i++) t->buf[m++] = t->suf_tab[(size_t)last * t->n + i];
    hash_into(out, t->buf, m);
}

static int emit(opaths *out, const int32_t *path, int32_t k, int32_t closing) {
    if (out->stats_only) {
        emit_stats(out, path, k, closing);
        return 0;
    }
    if (v64_push(&out->off, out->vert.len)) return -1;
    for (int32_t i = 0; i < k; i++)
        if (v32_push(&out->vert, path[i])) return -1;
    if (closing >= 0 && v32_push(&out->vert, closing)) return -1;
    return 0;
}

/* Operational maximality test for an acyclic simple path (see header). */
static int is_maximal_acyclic(const ograph *g, const int32_t *path, int32_t k, const uint8_t *on) {
    int32_t v1 = path[0], vk = path[k - 1];
    for (int64_t e = g->so[vk]; e < g->so[vk + 1]; e++) {
        int32_t w = g->st[e];
        if (!on[w] || w == v1) return 0; /* w outside {v2..vk} (v1 != vk here) */
    }
    for (int64_t e = g->po[v1]; e < g->po[v1 + 1]; e++) {
        int32_t u = g->pt[e];
        if (!on[u] || (u == vk && k > 1)) return 0; /* u outside {v1..v(k-1)} */
        if (u == vk && k == 1) return 0;            /* self-loop: <v> extends to <v,v> */
    }
    return 1;
}

/* DFS from v1; emits maximal paths in lexicographic order. */
static int pp_from(const ograph *g, int32_t v1, int use_prunes, opaths *out,
                   int32_t *path, int64_t *nxt, uint8_t *on) {
    int32_t n = g->n;
    int cycles_only = 0;
    if (use_prunes) {
        for (int64_t e = g->po[v1]; e < g->po[v1 + 1]; e++)
            if (g->scc[g->pt[e]] != g->scc[v1]) cycles_only = 1;  /* prune A' */
    }
    int32_t k = 1;
    path[0] = v1;
    on[v1] = 1;
    nxt[0] = g->so[v1];
    if (!cycles_only && is_maximal_acyclic(g, path, 1, on))
        if (emit(out, path, 1, -1)) return -1;
    while (k > 0) {
        int32_t vk = path[k - 1];
        if (nxt[k - 1] < g->so[vk + 1]) {
            int32_t w = g->st[nxt[k - 1]++];
            if (w == v1) {                       /* cycle closure: always prime */
                if (emit(out, path, k, v1)) return -1;
                continue;
            }
            if (on[w]) continue;                 /* not simple */
            if (cycles_only && g->scc[w] != g->scc[v1]) continue;  /* prune A' */
            if (use_prunes && g->scc[w] != g->scc[v1] && g->scc[vk] == g->scc[v1]) {
                /* prune B: first step out of SCC(v1); head-closure frozen from here */
                int closed = 1;
                for (int64_t e = g->po[v1]; e < g->po[v1 + 1]; e++)
                    if (!on[g->pt[e]]) closed = 0;
                if (!closed) continue;
            }
            path[k] = w;
            on[w] = 1;
            nxt[k] = g->so[w];
            k++;
            if (!cycles_only && is_maximal_acyclic(g, path, k, on))
                if (emit(out, path, k, -1)) return -1;
        } else {
            on[vk] = 0;
            k--;
        }
    }
    (void)n;
    return 0;
}

/*
 * oracle_prime_paths: all prime paths whose first vertex lies in [v_lo, v_hi),
 * in lexicographic order.  Returns 0 on success, -1 on OOM.  *out_off has
 * n_paths + 1 entries (relative to the block), *out_vert holds the vertices;
 * release both with oracle_free.
 */
int oracle_prime_paths(int32_t n, const int64_t *so, const int32_t *st, int32_t v_lo, int32_t v_hi,
                       int32_t use_prunes, int64_t **out_off, int32_t **out_vert, int64_t *n_paths,
                       int64_t *n_vert) {
    ograph g;
    if (g_init(&g, n, so, st)) return -1;
    opaths out;
    memset(&out, 0, sizeof(out));
    int32_t *path = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int64_t *nxt = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    uint8_t *on = (uint8_t *)calloc((size_t)n + 1, 1);
    int rc = (!path || !nxt || !on) ? -1 : 0;
    if (v_lo < 0) v_lo = 0;
    if (v_hi > n) v_hi = n;
    for (int32_t v = v_lo; v < v_hi && rc == 0; v++) rc = pp_from(&g, v, use_prunes, &out, path, nxt, on);
    if (rc == 0) rc = v64_push(&out.off, out.vert.len);
    free(path);
    free(nxt);
    free(on);
    g_free(&g);
    if (rc) {
        free(out.off.a);
        free(out.vert.a);
        return -1;
    }
    *n_paths = out.off.len - 1;
    *n_vert = out.vert.len;
    *out_off = out.off.a;
    *out_vert = out.vert.a ? out.vert.a : (int32_t *)malloc(sizeof(int32_t));
    return 0;
}

void oracle_free(void *p) { free(p); }

int oracle_tp_tables(int32_t n, const int64_t *so, const int32_t *st, int32_t entry, int32_t exit_v,
                     int32_t *pre_len, int32_t *pre_tab, int32_t *suf_len, int32_t *suf_tab);

/*
 * oracle_pp_stats: for every start vertex v in [v_lo, v_hi), the prime paths
 * whose first vertex is v, hashed as they are enumerated (same DFS and test as
 * oracle_prime_paths, nothing stored): cnt[2*(v-v_lo)] = number of paths,
 * cnt[2*(v-v_lo)+1] = their vertices, hash[2*(v-v_lo)], hash[..+1] = digest.
 * With entry >= 0 the TEST PATH of every prime path (R15, entry -> exit) is
 * hashed instead (returns -2 if some prime path's TP does not exist).
 */
static int pp_stats_impl(int32_t n, const int64_t *so, const int32_t *st, int32_t v_lo, int32_t v_hi,
                         int32_t entry, int32_t exit_v, int64_t *cnt, uint64_t *hash) {
    ograph g;
    if (g_init(&g, n, so, st)) return -1;
    int32_t *path = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int64_t *nxt = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    uint8_t *on = (uint8_t *)calloc((size_t)n + 1, 1);
    otp tp;
    memset(&tp, 0, sizeof(tp));
    int32_t *tabs = NULL;
    int rc = (!path || !nxt || !on) ? -1 : 0;
    if (rc == 0 && entry >= 0) {
        tabs = (int32_t *)malloc(((size_t)2 * n * n + 5 * (size_t)n + 3) * sizeof(int32_t));
        if (!tabs) rc = -1;
        else {
            int32_t *pl = tabs, *sl = tabs + n, *pt = tabs + 2 * (size_t)n, *stb = pt + (size_t)n * n;
            tp.buf = stb + (size_t)n * n;
            oracle_tp_tables(n, so, st, entry, exit_v, pl, pt, sl, stb);
            tp.pre_len = pl;
            tp.suf_len = sl;
            tp.pre_tab = pt;
            tp.suf_tab = stb;
            tp.n = n;
        }
    }
    if (v_lo < 0) v_lo = 0;
    if (v_hi > n) v_hi = n;
    for (int32_t v = v_lo; v < v_hi && rc == 0; v++) {
        opaths out;
        memset(&out, 0, sizeof(out));
        out.stats_only = 1;
        out.tp = entry >= 0 ? &tp : NULL;
        rc = pp_from(&g, v, 1, &out, path, nxt, on);
        cnt[2 * (size_t)(v - v_lo)] = out.n_paths;
        cnt[2 * (size_t)(v - v_lo) + 1] = out.n_vert;
        hash[2 * (size_t)(v - v_lo)] = out.ha;
        hash[2 * (size_t)(v - v_lo) + 1] = out.hb;
    }
    if (rc == 0 && tp.unreachable) rc = -2;
    free(tabs);
    free(path);
    free(nxt);
    free(on);
    g_free(&g);
    return rc;
}

int oracle_pp_stats(int32_t n, const int64_t *so, const int32_t *st, int32_t v_lo, int32_t v_hi, int64_t *cnt,
                    uint64_t *hash) {
    return pp_stats_impl(n, so, st, v_lo, v_hi, -1, -1, cnt, hash);
}

int oracle_tp_stats(int32_t n, const int64_t *so, const int32_t *st, int32_t v_lo, int32_t v_hi, int32_t entry,
                    int32_t exit_v, int64_t *cnt, uint64_t *hash) {
    if (entry < 0 || entry >= n || exit_v < 0 || exit_v >= n) return -3;
    return pp_stats_impl(n, so, st, v_lo, v_hi, entry, exit_v, cnt, hash);
}

/* ------------------------------------------------------------ E_canon */
static int64_t count_in_scc(const ograph *g, int32_t s, int32_t *path, int64_t *nxt, uint8_t *on) {
    int64_t cnt = 0;
    int32_t k = 1;
    path[0] = s;
    on[s] = 1;
    nxt[0] = g->so[s];
    while (k > 0) {
        int32_t vk = path[k - 1];
        if (nxt[k - 1] < g->so[vk + 1]) {
            int32_t w = g->st[nxt[k - 1]++];
            if (g->scc[w] != g->scc[s]) continue;
            if (w == s) { cnt++; continue; }     /* closure counts as an extension */
            if (on[w]) continue;
            cnt++;
            path[k] = w;
            on[w] = 1;
            nxt[k] = g->so[w];
            k++;
        } else {
            on[vk] = 0;
            k--;
        }
    }
    return cnt;
}

int64_t oracle_ext_count(int32_t n, const int64_t *so, const int32_t *st, int32_t v_lo, int32_t v_hi) {
    ograph g;
    if (g_init(&g, n, so, st)) return -1;
    int32_t *path = (int32_t *)malloc(((size_t)n + 1) * sizeof(int32_t));
    int64_t *nxt = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    uint8_t *on = (uint8_t *)calloc((size_t)n + 1, 1);
    int64_t total = 0;
    if (v_lo < 0) v_lo = 0;
    if (v_hi > n) v_hi = n;
    for (int32_t s = v_lo; s < v_hi; s++)
        if (g.nontriv[s]) total += count_in_scc(&g, s, path, nxt, on);
    free(path);
    free(nxt);
    free(on);
    g_free(&g);
    return total;
}

/* SCC labels as computed by the oracle (smallest member id). */
int oracle_scc_labels(int32_t n, const int64_t *so, const int32_t *st, int32_t *label) {
    ograph g;
    if (g_init(&g, n, so, st)) return -1;
    memcpy(label, g.scc, (size_t)n * sizeof(int32_t));
    g_free(&g);
    return 0;
}

/* -------------------------------------------------------------- digest */
void oracle_digest(int64_t n_paths, const int64_t *off, const int32_t *vert, uint64_t *out2) {
    uint64_t a = 0, b = 0;
    for (int64_t i = 0; i < n_paths; i++) {
        a += path_hash(SEED_A, vert + off[i], off[i + 1] - off[i]);
        b += path_hash(SEED_B, vert + off[i], off[i + 1] - off[i]);
    }
    out2[0] = a;
    out2[1] = b;
}

/* ----------------------------------------------------------- test paths */
/*
 * Builds prefix (entry -> v) and suffix (v -> exit) walks for every vertex.
 * pre_len[v] / suf_len[v] = number of vertices, -1 if unreachable.  Walks are
 * stored at v * (n) .. in the caller-provided n*n tables pre_tab / suf_tab.
 */
int oracle_tp_tables(int32_t n, const int64_t *so, const int32_t *st, int32_t entry, int32_t exit_v,
                     int32_t *pre_len, int32_t *pre_tab, int32_t *suf_len, int32_t *suf_tab) {
    ograph g;
    if (g_init(&g, n, so, st)) return -1;
    int32_t *parent = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *dist = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *tmp = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    for (int32_t v = 0; v < n; v++) { parent[v] = -2; pre_len[v] = -1; suf_len[v] = -1; dist[v] = -1; }
    /* BFS from entry; successors ascending; first discoverer is the parent */
    int64_t qh = 0, qt = 0;
    parent[entry] = -1;
    queue[qt++] = entry;
    while (qh < qt) {
        int32_t v = queue[qh++];
        for (int64_t e = so[v]; e < so[v + 1]; e++) {
            int32_t w = st[e];
            if (parent[w] == -2) { parent[w] = v; queue[qt++] = w; }
        }
    }
    for (int32_t v = 0; v < n; v++) {
        if (parent[v] == -2) continue;
        int32_t len = 0;
        for (int32_t c = v; c != -1; c = parent[c]) tmp[len++] = c;
        pre_len[v] = len;
        for (int32_t i = 0; i < len; i++) pre_tab[(size_t)v * n + i] = tmp[len - 1 - i];
    }
    /* reverse BFS distances to exit */
    qh = qt = 0;
    dist[exit_v] = 0;
    queue[qt++] = exit_v;
    while (qh < qt) {
        int32_t v = queue[qh++];
        for (int64_t e = g.po[v]; e < g.po[v + 1]; e++) {
            int32_t u = g.pt[e];
            if (dist[u] < 0) { dist[u] = dist[v] + 1; queue[qt++] = u; }
        }
    }
    for (int32_t v = 0; v < n; v++) {
        if (dist[v] < 0) continue;
        int32_t cur = v, len = 0;
        suf_tab[(size_t)v * n + len++] = cur;
        while (cur != exit_v) {
            int32_t best = -1;
            for (int64_t e = so[cur]; e < so[cur + 1]; e++) {
                int32_t w = st[e];
                if (dist[w] == dist[cur] - 1 && (best < 0 || w < best)) best = w;
            }
            cur = best;
            suf_tab[(size_t)v * n + len++] = cur;
        }
        suf_len[v] = len;
    }
    free(parent);
    free(dist);
    free(queue);
    free(tmp);
    g_free(&g);
    return 0;
}
