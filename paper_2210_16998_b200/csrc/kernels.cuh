// kernels.cuh -- device code of libtpgen (sm_100a): the DFS enumerator.
//
// Hot path: per start vertex s, depth-first
// enumeration of the simple paths inside SCC(s) (tail extension along CSR
// arcs, a W-word visited mask per path, cycle closure back to s -- PAPER.md
// Alg. 4 "ExtendPath" P:459-472, Ammann-Offutt generation P:865), fused with
// the maximality / segment classification (Def. 1, Defs. 6-9
// P:158-176 under DESIGN.md readings R8/R9) and the canonical writer.
//
// Design: one lane owns one work unit (a subtree of the
// per-start trie, or a terminal event) and walks it depth-first; the lane's
// path lives in shared memory ([level][lane] bytes), its visited set in
// registers.  Lanes refill from a global unit counter (warp-aggregated
// atomic).  Emission is warp-cooperative: every emitting lane's path is
// written by the whole warp as one coalesced store stream.  Exact output
// offsets come from a count pass with the same step function, a scan, and the
// write pass.  Units that exceed a step budget in the count pass are split into
// a counted piece (replayed for exactly that many steps by the write pass) plus
// the untried sibling subtrees on its stack, which keeps lexicographic order
// and bounds every unit's work.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

// Bounds checks of debug builds (TPGEN_KERNEL_DEBUG=1 python paper_2210_16998_b200/build.py --force):
// a failed check prints its site and traps; release builds compile them away.
#ifdef TPGEN_KERNEL_DEBUG
#include <cstdio>
#define TPG_DCHECK(cond, what)                                                          \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            printf("tpgen device check failed: %s (%s:%d)\n", what, __FILE__, __LINE__); \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define TPG_DCHECK(cond, what) \
    do {                       \
    } while (0)
#endif

namespace tpg {

enum UnitKind : uint8_t { K_NODE = 0, K_SELF = 1, K_CLOSURE = 2, K_OUT = 3 };
enum UnitStatus : uint8_t { ST_PENDING = 0, ST_DONE = 1, ST_TRUNC = 2 };
enum EvType : int { EV_NONE = 0, EV_PP = 1, EV_HEAD = 2, EV_TAIL = 3, EV_TRANSIT = 4 };
enum Pass : int { PASS_COUNT = 0, PASS_WRITE = 1 };
enum Cnt : int { C_PP = 0, C_VERT = 1, C_ITEMS = 2, C_ITEMV = 3, C_HEADS = 4, C_HEADV = 5, C_NUM = 6 };

// ------------------------------------------------------------------ masks
template <int W>
struct Mask {
    uint64_t w[W];
};

template <int W>
__device__ __forceinline__ Mask<W> mzero() {
    Mask<W> m;
#pragma unroll
    for (int i = 0; i < W; i++) m.w[i] = 0;
    return m;
}
template <int W>
__device__ __forceinline__ void mset(Mask<W> &m, int b) {
#pragma unroll
    for (int i = 0; i < W; i++)
        if (i == (b >> 6)) m.w[i] |= 1ull << (b & 63);
}
template <int W>
__device__ __forceinline__ void mclr(Mask<W> &m, int b) {
#pragma unroll
    for (int i = 0; i < W; i++)
        if (i == (b >> 6)) m.w[i] &= ~(1ull << (b & 63));
}
template <int W>
__device__ __forceinline__ Mask<W> mbit(int b) {
    Mask<W> m = mzero<W>();
    mset(m, b);
    return m;
}
// (a & ~b) == 0
template <int W>
__device__ __forceinline__ bool msubset(const Mask<W> &a, const Mask<W> &b) {
    uint64_t r = 0;
#pragma unroll
    for (int i = 0; i < W; i++) r |= a.w[i] & ~b.w[i];
    return r == 0;
}
template <int W>
__device__ __forceinline__ Mask<W> operator|(const Mask<W> &a, const Mask<W> &b) {
    Mask<W> r;
#pragma unroll
    for (int i = 0; i < W; i++) r.w[i] = a.w[i] | b.w[i];
    return r;
}
// lowest set bit >= k of (sin & (~M | sbit)); 64*W if none
template <int W>
__device__ __forceinline__ int mnext(const Mask<W> &sin, const Mask<W> &M, const Mask<W> &sbit, int k) {
    int res = 64 * W;
#pragma unroll
    for (int i = W - 1; i >= 0; i--) {
        uint64_t c = sin.w[i] & (~M.w[i] | sbit.w[i]);
        const int lo = i * 64;
        if (k >= lo + 64) c = 0;
        else if (k > lo) c = (c >> (k - lo)) << (k - lo);
        if (c) res = lo + __ffsll((long long)c) - 1;
    }
    return res;
}

// ------------------------------------------------------------------ tables
// One vertex of an SCC in SCC-local order (device copy of the HostPlan slot).
template <int W>
struct __align__(16) Slot {
    uint64_t sin[W];  // in-SCC successors (local bits; a self-loop sets the own bit)
    uint64_t pin[W];  // in-SCC predecessors
    int32_t gid, out_off, out_cnt, flags;
};

// A work unit: a trie node (K_NODE: the whole subtree under it), or one
// terminal event of a trie node (K_CLOSURE: the cycle path(+)s, K_OUT: the arc
// to an out-of-SCC successor).
template <int W>
struct __align__(16) Unit {
    uint8_t path[64 * W];  // local vertex ids, path[0..depth]
    int32_t scc;           // (16-byte aligned: read as one int4)
    int32_t e;             // K_OUT: out-arc index
    uint32_t nsteps;       // write pass: replay exactly this many steps (0 = to completion)
    uint8_t depth, kind, k, o;
    uint64_t M[W];         // visited mask of path[0..depth]
    uint8_t rdepth;        // stop states: root depth of the unit
    uint8_t pad[3];
};

// Canonical offsets of one units outputs (linearization, aux_kernels.cuh).
struct __align__(16) LinNode {
    uint64_t v[C_NUM];  // offsets (relative to the jump target until the jumping ends)
    int64_t jmp;        // ancestor still to be added (-1: none)
    int64_t pad;
};

struct DevGraph {
    const void *slots;  // Slot<W>[n]
    const int32_t *slot_gid;
    const int32_t *out_gid;
    const int32_t *out_pos;
    const int32_t *scc_vbase;
    const int32_t *scc_out_base;
    const int32_t *scc_nout;
    const int64_t *scc_pair_base;
    const int32_t *slot_eidx;
    const uint64_t *Wc;  // completions per entry vertex (global id)
    const uint64_t *Wv;  // total vertices of those completions
    const int32_t *scc_gbase;  // global id of local 0 when an SCC's ids are contiguous, else -1
    const uint64_t *slot_mix;  // per slot: mix64(global id), the vertex's digest value (R20)
    const uint64_t *vmix;      // per global vertex id: mix64(id)
    const uint64_t *scc_exm;   // per SCC (<= 64 vertices): local bits of its exit vertices (Def. 5)
    const uint64_t *slot_d2;   // in-SCC out-degree <= 2 everywhere: {t0 | t1 << 32 | exit << 40, mix} per slot, else null
    const int32_t *v_slot;     // per global vertex id: its slot
    const int32_t *comp;       // per global vertex id: its SCC
    int32_t shard_lo, shard_hi;
};

// Count-mode head segment (cnt_kernel, count.cuh): the digest sum S of the head h, |h|
// and the slot of h's last vertex (an SCC exit); the cross prime paths h (+) w (+) ...
// over every out-of-SCC arc of that vertex are counted by head_count_kernel and hashed by
// stitch_hash_s_kernel.  x < 0 marks an unused slot of a warp's block.
struct TPG_ALIGN(16) HeadS {
    uint64_t S;
    int32_t len;
    int32_t x;
};

// Test-path digest terms of a vertex v (COUNT_HASH test paths, R15 + R20): prefix[v] minus
// its last vertex contributes S_pre (positions 0..), suffix[v] minus its first vertex
// contributes A_suf + 2 o B_suf when it starts at position o.  pre_len / suf_len are the
// walks' vertex counts (-1: no walk).  With them the TP of a path p (digest sum S, sum of
// mix B, L vertices, first f, last w) has
//   S_tp = S_pre[f] + S + 2 (pre_len[f] - 1) B + A_suf[w] + 2 (pre_len[f] - 1 + L) B_suf[w],
//   |TP| = pre_len[f] - 1 + L + suf_len[w] - 1.
struct TPG_ALIGN(16) TpTerm {
    uint64_t S_pre, A_suf, B_suf;
    int32_t pre_len, suf_len;
};

__device__ __forceinline__ uint64_t mul64x32_(uint64_t m, uint32_t w) {
    return (uint64_t)(uint32_t)m * w + ((uint64_t)((uint32_t)(m >> 32) * w) << 32);
}
// prefix part of a test path: S' = S_pre[f] + S + 2 o B, positions consumed o + L; false if no walk
__device__ __forceinline__ bool tp_head(const TpTerm *tp, int f, uint64_t &S, uint64_t B, uint32_t &len) {
    const TpTerm t = tp[f];
    if (t.pre_len < 0) return false;
    const uint32_t o = (uint32_t)t.pre_len - 1u;
    S = t.S_pre + S + mul64x32_(B, 2u * o);
    len += o;
    return true;
}
// suffix part: S += A_suf[w] + 2 L B_suf[w], L = positions so far; false if no walk
__device__ __forceinline__ bool tp_tail(const TpTerm *tp, int w, uint64_t &S, uint32_t &len) {
    const TpTerm t = tp[w];
    if (t.suf_len < 0) return false;
    S += t.A_suf + mul64x32_(t.B_suf, 2u * len);
    len += (uint32_t)t.suf_len - 1u;
    return true;
}

// Count-mode segment item (cnt_kernel's segment phase) of the entry vertex ent (global id):
// a tail segment (x < 0), or a transit segment ending at the exit vertex of slot x, followed
// by any of that vertex's out-of-SCC arcs (in arc order, W(y) completions each).  With the
// R20 terms mix(v) * (2 pos + 1) the item's contribution to a path's digest sum at offset o
// is A + 2 o B (A = its own sum from position 0, B = the sum of its mix(v)), so no vertex
// list is kept.  ent < 0 marks an unused slot of a warp's block.
struct TPG_ALIGN(16) ItemS {
    uint64_t A, B;
    int32_t len;
    int32_t x;
    int32_t ent;
    int32_t last;  // slot of its last vertex (the path's last vertex when it is a tail)
};

struct DfsArgs {
    DevGraph G;
    void *units;              // Unit<W>[qcap]: the work queue (roots pre-filled by the host)
    unsigned int *ready;      // per queue slot: 1 once the unit record is written
    unsigned long long *qhead;  // claims (own 128-byte line)
    unsigned long long *qtd;    // tail (pushed) << 32 | done (finished) (own 128-byte line)
    unsigned long long qcap;  // queue capacity (slots)
    // per-unit results, indexed by queue slot
    uint64_t *cnt[C_NUM];
    uint64_t *ext;
    int64_t *rfirst;          // first record chunk of the unit
    int64_t *rcount;          // records of the unit
    int64_t *child_head;      // latest block of units donated by the unit (-1: none)
    int64_t *blk_first;       // donated block: first unit
    int32_t *blk_count;       // donated block: number of units
    int64_t *blk_next;        // donated block: the unit's previous block (-1: none)
    int32_t *gen;             // donation generation (roots 0)
    int64_t *parent;          // donor of the unit (roots: -1, set by the host)
    int32_t *nchild;          // number of units the unit donated
    int *maxgen;
    unsigned long long *agg_tail_cnt, *agg_tail_len, *agg_pair_cnt, *agg_pair_len;
    unsigned int *overflow;   // bit 0: count overflow, bit 1: record pool exhausted, bit 2: queue full
    // record pool
    uint64_t *chunks;
    unsigned long long *chunk_next;
    unsigned long long chunk_cap;
    uint32_t split_min;       // steps a unit runs before it may be split
    uint32_t low_water;       // split when fewer queued units than this are waiting to be claimed
    int32_t eager_gens;       // donation generations that split at once (the ramp-up from one root per start)
    uint32_t split_min_starve;  // ... split_min while more than starve_lanes lanes wait for work
    int32_t starve_lanes;
    unsigned long long *dbg;  // TPGEN_KERNEL_DEBUG builds: iterations, idle iterations, lane-steps, donations
    int n_slots;              // slot table size (copied to shared memory by the TS kernels)
    // count modes (no records): totals [0] prime paths, [1] vertices, [2] E_canon, [3] digest a,
    // [4] digest b, [5] head slots reserved, [6] cross-SCC prime paths; heads go to heads[0 .. head_cap)
    unsigned long long *cacc;
    HeadS *heads;
    unsigned long long head_cap;
    ItemS *items;                 // count modes, segment phase: items go to items[0 .. item_cap)
    unsigned long long item_cap;  //   (cacc[7] = item slots reserved)
    const TpTerm *tp;             // count modes: non-null = hash the prime paths' TEST PATHS (per slot)
    int32_t prune;                // count modes, prime-path phase: NEXT #2 reachability pruning (P_PRUNE)
    uint32_t k2, k8, k16;         // = 2, 8, 16: multipliers the count kernel keeps opaque to ptxas (count.cuh)
};

// 256 threads per block for W <= 2; 128 for W = 4 (the per-lane path needs 64*W bytes of smem)
template <int W>
struct DfsCfg {
    static constexpr int threads = (W <= 2) ? 256 : 128;
    static constexpr int warps = threads / 32;
    static constexpr int min_blocks = (W == 1) ? 3 : ((W == 2) ? 2 : 3);
};
constexpr unsigned kFull = 0xffffffffu;

template <int W>
__device__ __forceinline__ const Slot<W> *slot_ptr(const DevGraph &G, int i) {
    return reinterpret_cast<const Slot<W> *>(G.slots) + i;
}
template <int W>
__device__ __forceinline__ Mask<W> ld_sin(const Slot<W> *p) {
    Mask<W> m;
    if (W == 1) {
        m.w[0] = __ldg(&p->sin[0]);
    } else {
#pragma unroll
        for (int i = 0; i < W; i += 2) {
            const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(&p->sin[i]));
            m.w[i] = v.x;
            m.w[i + 1] = v.y;
        }
    }
    return m;
}
template <int W>
__device__ __forceinline__ Mask<W> ld_pin(const Slot<W> *p) {
    Mask<W> m;
#pragma unroll
    for (int i = 0; i < W; i++) m.w[i] = __ldg(&p->pin[i]);
    return m;
}
template <int W>
__device__ __forceinline__ int4 ld_meta(const Slot<W> *p) {
    return __ldg(reinterpret_cast<const int4 *>(&p->gid));
}

__device__ __forceinline__ int count_out_le(const DevGraph &G, int out_off, int out_cnt, int w) {
    int o = 0;
    while (o < out_cnt && __ldg(G.out_pos + out_off + o) <= w) o++;
    return o;
}

// dataflow hand-off: the decrement releases the caller's earlier additions and
// acquires those of every earlier decrementer
__device__ __forceinline__ int atom_dec_acq_rel(int *p) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
    return old;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Digest (reading R20): a path v_0..v_{k-1} has the position-weighted
// sum S = sum_i mix(v_i) * (2i + 1) (mod 2^64) and the two digests a = mix(S ^ (SEED_A + k)),
// b = mix(S ^ (SEED_B + k)); the set digest is the sum over paths mod 2^64 (order
// independent, so shards add up).  The terms of S are independent (no per-vertex chain) and
// a vertex's term at any position is its per-vertex value mix(v) times an odd weight, so a
// DFS keeps S in a register: one table load and a multiply-add per push or pop.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finalizer
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}
// position weight of the digest term of the vertex at position p (R20)
__device__ __forceinline__ uint64_t pos_weight(uint32_t p) { return 2 * (uint64_t)p + 1; }
constexpr uint64_t kSeedA = 0x9E3779B97F4A7C15ull, kSeedB = 0xD1B54A32D192ED03ull;
struct PathHash {
    uint64_t a, b;  // the path's digests after fin() (accumulators: sums of them)
    uint64_t s;     // position-keyed vertex sum
    uint32_t p, n;  // next position, path length
    __device__ __forceinline__ void init(uint64_t len) {
        s = 0;
        p = 0;
        n = (uint32_t)len;
    }
    __device__ __forceinline__ void add(int32_t v) {
        s += mix64((uint64_t)(uint32_t)v) * (2 * (uint64_t)p + 1);
        p++;
    }
    __device__ __forceinline__ void fin() {
        a = mix64(s ^ (0x9E3779B97F4A7C15ull + (uint64_t)n));
        b = mix64(s ^ (0xD1B54A32D192ED03ull + (uint64_t)n));
    }
};

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b, unsigned int *ovf) {
    uint64_t r = a + b;
    if (r < a || r >= (1ull << 62)) {
        atomicOr(ovf, 1u);
        r = (1ull << 62);
    }
    return r;
}
__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t b, unsigned int *ovf) {
    uint64_t hi = __umul64hi(a, b), lo = a * b;
    if (hi || lo >= (1ull << 62)) {
        atomicOr(ovf, 1u);
        return (1ull << 62);
    }
    return lo;
}

}  // namespace tpg
