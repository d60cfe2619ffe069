/*
 * tpgen.h -- C ABI of the B200-native prime-path / test-path engine.
 *
 * Reference: "TPGen: A Self-Stabilizing GPU-Based Method for Prime and Test
 * Paths Generation" (arXiv 2210.16998), cited as PAPER.md line numbers (P:n).
 *
 * Problem 1: input a CFG G = (V, E), start s, end e; output the
 * prime paths of G and a set of test paths covering them.  The prime-path set
 * does not depend on s and e (Def. 1), so the ABI has two calls:
 *   tpgen_prime_paths -- all prime paths (maximal simple paths, simple cycles
 *                        included), canonical order;
 *   tpgen_test_paths  -- one entry->exit test path per prime path.
 *
 * Conventions (all calls)
 *   - Graph input is a SUCCESSOR CSR in HOST memory, borrowed for the call:
 *     csr_offsets int64[n_vertices+1] (offsets[0] = 0, non-decreasing),
 *     csr_targets int32[offsets[n]] (each in [0, n_vertices)).  Rows need not be
 *     sorted; duplicate arcs in a row are rejected (TPGEN_ERR_INVALID_GRAPH);
 *     self-loops are allowed.  (The paper's CSR is predecessor-oriented, P:300;
 *     predecessor masks are derived internally.)
 *   - Vertex ids are int32, path offsets int64, counts uint64 internally
 *     (overflow -> TPGEN_ERR_LIMIT_EXCEEDED, detected before any output
 *     allocation).
 *   - Canonical output order: lexicographic on int32 sequences.  Prime-path
 *     sets are prefix-free, so the order is total.  Output arrays:
 *       offsets  int64[n_paths + 1], offsets[0] = 0, non-decreasing;
 *       vertices int32[offsets[n_paths]] (global vertex ids).
 *     A cyclic prime path v1..vk repeats v1 at the end (v1 = vk).
 *   - Outputs are allocated by the library, on the device (opt->device) through
 *     opt->device_alloc (or cudaMallocAsync on opt->stream when NULL), or in
 *     pinned host memory when output_on_device = 0.  Release with
 *     tpgen_paths_free.  On any error *out is zeroed.
 *   - Work is enqueued on opt->stream (a cudaStream_t; NULL = legacy default
 *     stream) and the call returns after the stream has been synchronised.
 *   - Errors: a tpgen_status; tpgen_status_string gives a static message and
 *     tpgen_last_error_message a thread-local detail string.
 *   - There is no CPU fallback: without a usable CUDA device every call that
 *     computes returns TPGEN_ERR_CUDA.
 */
#ifndef TPGEN_H
#define TPGEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TPGEN_OK = 0,
    TPGEN_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, n < 0, bad entry/exit, bad shard spec */
    TPGEN_ERR_INVALID_GRAPH = 2,    /* offsets[0] != 0, decreasing offsets, target out of range, duplicate arc */
    TPGEN_ERR_LIMIT_EXCEEDED = 3,   /* n_paths > max_paths, extensions > max_extensions, or a count >= 2^62 */
    TPGEN_ERR_OUT_OF_MEMORY = 4,    /* host or device allocation failed */
    TPGEN_ERR_UNREACHABLE = 5,      /* tpgen_test_paths: a PP's first vertex is not reachable from entry,
                                       or its last vertex cannot reach exit */
    TPGEN_ERR_CUDA = 6,             /* CUDA runtime error (no device, launch failure, ...) */
    TPGEN_ERR_INTERNAL = 7,         /* invariant violated inside the library */
    TPGEN_ERR_UNSUPPORTED = 8       /* a strongly connected component with more than 256 vertices */
} tpgen_status;

enum { TPGEN_OUT_MATERIALIZE = 0, TPGEN_OUT_COUNT_HASH = 1 };
enum { TPGEN_TP_PER_PP = 0, TPGEN_TP_UNIQUE = 1, TPGEN_TP_GREEDY = 2 };
/* Enumeration engine (tpgen_options.engine). */
enum { TPGEN_ENGINE_DFS = 0, TPGEN_ENGINE_FRONTIER = 1, TPGEN_ENGINE_ALG3 = 2 };

/* Canonical flat path array (see conventions). */
typedef struct {
    int64_t n_paths;
    int64_t *offsets;   /* n_paths + 1 entries */
    int32_t *vertices;  /* offsets[n_paths] entries */
    int32_t on_device;  /* 1: device pointers on `device`; 0: pinned host pointers */
    int32_t device;
    void *_owner;       /* library-private */
} tpgen_paths;

typedef void *(*tpgen_alloc_fn)(size_t bytes, void *stream, void *ctx);
typedef void (*tpgen_free_fn)(void *ptr, void *stream, void *ctx);

typedef struct {
    int32_t device;            /* CUDA ordinal; -1 = current device */
    void *stream;              /* cudaStream_t; NULL = legacy default stream */
    int32_t output_on_device;  /* 1 (default): device output; 0: pinned host output */
    int32_t output_mode;       /* TPGEN_OUT_MATERIALIZE (default) | TPGEN_OUT_COUNT_HASH (counts + digest only) */
    int32_t shard_rank;        /* start-vertex shard (0-based); with shard_count = 1 the whole graph */
    int32_t shard_count;       /* >= 1 */
    int32_t start_lo, start_hi;  /* explicit start-vertex range [lo, hi) instead of the shard split when
                                    start_hi > start_lo (e.g. one rank per independent component); combined
                                    with shard_count > 1: TPGEN_ERR_INVALID_ARGUMENT */
    int64_t max_paths;         /* 0 = unlimited */
    int64_t max_extensions;    /* 0 = unlimited */
    int32_t tp_mode;           /* TPGEN_TP_PER_PP: one TP per PP, aligned; TPGEN_TP_UNIQUE (K7, SURVEY §8(a)
                                  a6): the set of distinct per-PP TPs ("the set of TPs covering all PPs",
                                  P:269) in lexicographic order of the int32 sequences -- materialized output
                                  only (COUNT_HASH: TPGEN_ERR_INVALID_ARGUMENT); TPGEN_TP_GREEDY: greedy cover
                                  -- longest uncovered PP first (ties lexicographic), extended by the R15
                                  walks, every PP contained in it covered */
    int32_t compute_digest;    /* 1: fill stats->hash_lo/hi (extra pass over the output) */
    tpgen_alloc_fn device_alloc;  /* output allocator; NULL -> cudaMallocAsync */
    tpgen_free_fn device_free;
    void *alloc_ctx;
    void *host_out;            /* optional caller-owned (ideally pinned) host buffer for output_on_device = 0:
                                  offsets are placed at host_out, vertices right after them; used when
                                  host_out_bytes >= 8*(n_paths+1) + 4*n_vertices, else pinned memory is
                                  allocated by the library.  The caller keeps ownership. */
    size_t host_out_bytes;
    int32_t engine;            /* TPGEN_ENGINE_DFS (default): depth-first walk, on-chip path stacks, every
                                  output mode.  TPGEN_ENGINE_FRONTIER: level-synchronous frontier extension
                                  (Alg. 4 ExtendPath applied to every simple path of length l at once,
                                  P:459-472; the north-star's level-by-level kernel): path records
                                  {visited mask, last, first, position-keyed digest sum} streamed through HBM,
                                  ping-pong buffers, block-scan compaction; on graphs with arcs leaving SCCs
                                  the levels also write head segments and (for SCC entries) transit / tail
                                  segments, stitched by the same completion DP as the DFS count mode.
                                  Requires output_mode = TPGEN_OUT_COUNT_HASH (counts, E_canon and -- with
                                  compute_digest = 1 -- the digest; compute_digest = 0 drops the digest sum
                                  from the records of graphs without arcs leaving SCCs) and SCCs of <= 64
                                  vertices (else TPGEN_ERR_INVALID_ARGUMENT).  A level that does not fit
                                  in the device memory budget switches the call (or pass) to the
                                  DFS-chunked frontier; TPGEN_ERR_OUT_OF_MEMORY when
                                  even the per-level rings cannot hold the roots.  TPGEN_ENGINE_ALG3: the paper's vertex-centric self-stabilizing
                                  algorithm (Alg. 1-4) as a comparison engine -- one cooperative
                                  launch, one CTA per vertex owning the list of the simple paths ending at
                                  it, every simple path of the graph held in HBM at once; COUNT_HASH
                                  only, no shards or start ranges, graphs of <= 128 vertices (and <= the
                                  SM count), else TPGEN_ERR_INVALID_ARGUMENT; TPGEN_ERR_OUT_OF_MEMORY when
                                  the lists do not fit.  Its n_extensions is the number of ExtendPath calls
                                  (every simple path of >= 2 vertices), equal to E_canon on strongly
                                  connected graphs. */
    int32_t no_plan_cache;     /* one-shot calls (tpgen_prime_paths / tpgen_test_paths) keep the last graph's plan
                                  and device tables per device and reuse them when the next call passes a
                                  byte-identical CSR; 1 = always plan and upload anew (what an end-to-end timing of a
                                  fresh graph measures).  Ignored by the tpgen_plan_* calls. */
    int32_t shard_prefix;      /* 1: with shard_count > 1, shards are contiguous ranges of PREFIX UNITS instead of
                                  start vertices ("(start, depth-k prefix) for heavy starts"):
                                  a heavy start vertex's path trie is cut at its depth-k prefixes (each unit the
                                  subtree under path[0..k], or the closing arc of a cycle) until no unit holds
                                  more than 1/(16 count) of the Knuth-estimated work, so a graph with fewer start
                                  vertices than shards (config 3: 22 starts) still balances.  Units keep the
                                  canonical order, so shard r's output is still block r of the global list
                                  (tpgen_shard_units gives the split).  Applies to graphs with one mask word (SCCs
                                  of <= 32 vertices) and no arc leaving an SCC on the DFS engine (materialize
                                  additionally needs the LEAN table in shared memory: n_vertices <= 1024);
                                  elsewhere the start-vertex split is used and stats.unit_lo = unit_hi = -1.
                                  Other engines: TPGEN_ERR_INVALID_ARGUMENT.  0 (default): start-vertex shards. */
    int32_t prune;             /* 1: reachability pruning (not in the paper) in the COUNT_HASH
                                  prime-path phase of the DFS engine: a child w is not entered when w is not a
                                  predecessor of the start s, some predecessor of s is off the path, and no
                                  predecessor of s off the path is reachable from w in the SCC minus the path
                                  (bitset BFS) -- its subtree holds no closure, internal prime path or head
                                  segment (Def. 1; Def. 6).  Counts, vertices and digest are
                                  unchanged; stats.n_extensions then counts the extensions MADE (<= E_canon).
                                  Graphs with SCCs of > 64 vertices and the segment / test-path phases do not
                                  prune.  Requires output_mode = TPGEN_OUT_COUNT_HASH and the DFS engine, else
                                  TPGEN_ERR_INVALID_ARGUMENT.  0 (default): off (measured slower). */
} tpgen_options;

typedef struct {
    int64_t n_paths;         /* paths returned (this shard) */
    int64_t total_vertices;  /* offsets[n_paths] */
    int64_t n_extensions;    /* E_canon of this shard's start vertices */
    int64_t n_cross;         /* prime paths spanning >= 2 SCCs */
    int64_t n_units;         /* DFS work units (roots + donated) */
    int64_t n_heads;         /* head segments (cross-PP blocks) */
    int64_t n_segments;      /* transit + tail segment items */
    uint64_t hash_lo, hash_hi;  /* order-independent multiset digest */
    int32_t n_scc, n_scc_nontrivial, max_scc, n_count_rounds;
    int64_t gpu_launches;    /* kernels this call launched */
    int32_t shard_lo, shard_hi;  /* start-vertex range of this shard */
    double ms_plan;          /* host planning (Tarjan, tables) */
    double ms_count;         /* device: DFS phases + linearization (ms_device - ms_write - ms_stitch) */
    double ms_write;         /* device: canonical writer (expand_kernel) */
    double ms_stitch;        /* device: segment scans + stitch writer */
    double ms_device;        /* device time of the whole pipeline (CUDA events) */
    double ms_total;         /* wall clock of the call */
    double ms_dfs_write;     /* device time of the dominant kernel (dfs_kernel, both phases) */
    double ms_dfs_count;     /* same as ms_dfs_write (kept for ABI stability) */
    double ms_linearize;     /* device: linearization of the unit forest (canonical offsets) */
    double ms_dominant;      /* device time of the prime-path phase's enumeration kernel (the dominant launch) */
    int64_t ext_dominant;    /* extensions (E_canon terms) that launch made */
    int64_t unit_lo, unit_hi;  /* shard_prefix: this shard's prefix-unit range [unit_lo, unit_hi) of the
                                  split (tpgen_shard_units); -1 / -1 otherwise */
} tpgen_stats;

void tpgen_options_init(tpgen_options *opt);
const char *tpgen_status_string(tpgen_status s);
const char *tpgen_last_error_message(void);
const char *tpgen_version(void);

/*
 * All prime paths of G (Def. 1) whose first vertex lies in this
 * shard's start-vertex range, in canonical order.  Shards partition the global
 * canonical list into contiguous blocks in rank order.
 */
tpgen_status tpgen_prime_paths(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                               const tpgen_options *opt, tpgen_paths *out, tpgen_stats *stats);

/*
 * Test paths ("the set of TPs covering all PPs"; "extends every PP
 * to visit initial and final nodes"): TP_i = prefix[first_i] (minus its last
 * vertex) ++ PP_i ++ suffix[last_i] (minus its first vertex), aligned 1:1 with
 * the prime-path list.  prefix[v] is the lexicographically smallest
 * minimum-hop walk entry -> v, suffix[v] the one v -> exit (R15).
 * prime_paths: a canonical list (host or device), or NULL to compute it.
 */
tpgen_status tpgen_test_paths(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                              const tpgen_paths *prime_paths, int32_t entry, int32_t exit,
                              const tpgen_options *opt, tpgen_paths *out, tpgen_stats *stats);

/*
 * Component graph (host only, no device needed): Tarjan SCCs of G.
 * comp[v] = SCC id of v, ids in reverse topological order of the component
 * DAG (Def. 3): every arc between two SCCs goes from a larger id to
 * a smaller one.  flags[v] = 1 if v is an SccEntryVertex (Def. 4),
 * | 2 if an SccExitVertex (Def. 5), | 4 if its SCC is nontrivial
 * (more than one vertex or a self-loop).  comp and flags are caller-owned
 * int32[n_vertices]; *n_scc receives the number of SCCs.  Same validation and
 * error codes as tpgen_prime_paths (TPGEN_ERR_UNSUPPORTED is not raised here).
 */
tpgen_status tpgen_components(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                              int32_t *comp, int32_t *flags, int32_t *n_scc);

/*
 * Start-vertex shard of a graph (host only): [*lo, *hi) of shard `rank` of `count`, the planner's
 * contiguous ranges balanced by its per-start cost estimates (what tpgen_options.shard_rank /
 * shard_count select).  Same validation and errors as tpgen_components.
 */
tpgen_status tpgen_shard_range(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                               int32_t rank, int32_t count, int32_t *lo, int32_t *hi);

/*
 * Prefix-unit shard of a graph (host only; tpgen_options.shard_prefix): the split
 * has *n_units units in canonical order; shard `rank` of `count` takes [*unit_lo, *unit_hi) and
 * touches start vertices [*lo, *hi) (its first / last unit's start; neighbouring shards may share
 * one).  *applies = 0 when the graph does not qualify (SCCs of > 32 vertices or arcs leaving SCCs):
 * the unit outputs are then 0 and lo / hi are tpgen_shard_range's.  Any output pointer may be NULL
 * except applies.  Same validation and errors as tpgen_components.
 */
tpgen_status tpgen_shard_units(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                               int32_t rank, int32_t count, int32_t *applies, int64_t *unit_lo,
                               int64_t *unit_hi, int64_t *n_units, int32_t *lo, int32_t *hi);

/*
 * The units of prefix-unit shard `rank` of `count` (host only; what tpgen_shard_units counts):
 * unit i is the path vertices[offsets[i] .. offsets[i+1]) (global ids, the start first); closure[i]
 * = 1: the unit is the closing arc of that path back to its start (one cyclic prime path), 0: the
 * trie subtree under the path (every prime path that has it as a prefix).  Two-call pattern:
 * *n_units_out / *n_vertices_out are always set; the arrays (n_units + 1 offsets, n_units closure
 * flags, n_vertices ids) are written when every pointer is non-NULL and the capacities suffice,
 * else TPGEN_ERR_INVALID_ARGUMENT (graphs the split does not apply to: 0 units).
 */
tpgen_status tpgen_shard_unit_paths(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                                    int32_t rank, int32_t count, int64_t *offsets, int32_t *vertices,
                                    int32_t *closure, int64_t cap_units, int64_t cap_vertices,
                                    int64_t *n_units_out, int64_t *n_vertices_out);

/* Structure metrics of a CFG (Table 1; host only). */
typedef struct {
    int64_t nodes, edges;      /* V, E */
    int64_t sccs;              /* nontrivial SCCs (more than one vertex, or a self-loop) */
    int64_t scc_nodes;         /* vertices in nontrivial SCCs */
    int64_t scc_edges;         /* arcs with both ends in the same nontrivial SCC */
    int64_t weak_components;   /* P: weakly connected components */
    int64_t cc;                /* cyclomatic complexity E - V + 2P */
    uint64_t npath;            /* Npath: start -> end paths that use every arc at most once (
                                  Npath(end) = 1, Npath(v) = sum over arcs (v,w) of Npath(w) in G minus the arc) */
    int32_t npath_status;      /* 0: exact; 1: >= 2^62 (npath saturated at 2^62); 2: not computed -- the graph
                                  has cycles and the arc-simple walk search exceeded its budget (10^8 steps) */
    int32_t pad;
} tpgen_metrics;

tpgen_status tpgen_metrics_compute(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                                   int32_t start, int32_t end, tpgen_metrics *out);

/* Stream-ordered release; safe on a zeroed struct. */
void tpgen_paths_free(tpgen_paths *p);

/*
 * Plan API: host planning + host->device upload of the graph tables once, then
 * device-resident calls (what bench.py times as `value`).
 */
typedef struct tpgen_plan tpgen_plan;
tpgen_status tpgen_plan_create(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                               const tpgen_options *opt, tpgen_plan **plan);
tpgen_status tpgen_plan_prime_paths(tpgen_plan *plan, const tpgen_options *opt, tpgen_paths *out,
                                    tpgen_stats *stats);
/*
 * Five-class report of a canonical prime-path list of the plan's graph (
 * DESIGN.md R19): counts[0..4] = complete (Start ... End, Def. 2), entry
 * (Start into an SCC, Def. 11), exit (an SCC to End, Def. 10), internal (inside one
 * SCC, Def. 9), transit (SCC to SCC, the class the paper's taxonomy misses).
 * prime_paths: host or device arrays; counts: caller-owned int64[5].
 */
tpgen_status tpgen_plan_classify(tpgen_plan *plan, const tpgen_paths *prime_paths, int32_t start, int32_t end,
                                 const tpgen_options *opt, int64_t counts[5]);
/* Test paths of the plan's graph (same contract as tpgen_test_paths, no re-planning). */
tpgen_status tpgen_plan_test_paths(tpgen_plan *plan, const tpgen_paths *prime_paths, int32_t entry, int32_t exit,
                                   const tpgen_options *opt, tpgen_paths *out, tpgen_stats *stats);
void tpgen_plan_destroy(tpgen_plan *plan);
/* Releases what one-shot calls keep between calls: the per-device cached plans
 * with their device workspaces and the library's cached output blocks, then trims the device
 * memory pool.  Plans created with tpgen_plan_create are not affected.  Safe to call at any
 * time outside a running call. */
void tpgen_release_cache(void);

/* Out-degree-2 normalization (Fig. 5: "we can convert a vertex v with an out-degree
 * greater than 2 ... to a vertex with out-degree 2 by adding some new intermediate vertices between
 * v and its successor vertices"; the figure itself is not in the text -- DESIGN.md R24 reads it as a
 * chain).  A vertex v with successors w1 < ... < wd, d > 2, keeps the arcs v -> w1 and v -> x1;
 * the new vertex x_i (i = 1..d-2) has the arcs x_i -> w_{i+1} and x_i -> x_{i+1}, and x_{d-2}
 * has x_{d-2} -> w_{d-1}, x_{d-2} -> w_d.  New vertices are numbered n, n+1, ... in order of v,
 * then i.  Every other vertex and arc is kept.  Host-only (the graph is KB-sized).
 *   csr_offsets / csr_targets / n_vertices: the input CSR (host, borrowed; validated like
 *     tpgen_prime_paths: TPGEN_ERR_INVALID_GRAPH on decreasing offsets, out-of-range targets or
 *     duplicate arcs in a row; NULL pointers with n_vertices > 0 -> TPGEN_ERR_INVALID_ARGUMENT).
 *   *out_n, *out_m: set to the normalized vertex and arc counts (always, when non-NULL).
 *   out_offsets (out_n + 1 entries), out_targets (out_m), origin (out_n: the input vertex whose
 *     successor list each vertex splits; itself for the input's vertices): caller-owned host
 *     arrays, filled when non-NULL (call once with NULLs to size them).  Successor lists of the
 *     result are ascending. */
tpgen_status tpgen_normalize_outdeg2(const int64_t *csr_offsets, const int32_t *csr_targets, int32_t n_vertices,
                                     int32_t *out_n, int64_t *out_m, int64_t *out_offsets, int32_t *out_targets,
                                     int32_t *origin);

#ifdef __cplusplus
}
#endif
#endif /* TPGEN_H */
