// dfs.cuh -- the DFS enumerator kernel (K1) of libtpgen.
//
// Hot path: per start vertex s, depth-first
// enumeration of the simple paths inside SCC(s) (tail extension along CSR
// arcs, a visited bit mask per path, cycle closure back to s -- PAPER.md
// Alg. 4 "ExtendPath" P:459-472, Ammann-Offutt generation P:865), fused with
// the maximality / segment classification (Def. 1, Defs. 6-9
// P:158-176 under DESIGN.md readings R8/R9).
//
// One lane owns one work unit (a subtree of the per-start trie, or a terminal
// event) and walks it depth-first.  Its path lives in shared memory, laid out
// [level/4][lane][level%4] so that the 32 lanes of a warp touching their own
// path never conflict on a bank; its visited set lives in a register (32-bit
// when the largest SCC has <= 32 vertices).  Lanes refill from a global unit
// counter (warp-aggregated atomic).
//
// Output is a per-unit stream of 64-bit *path-delta records* (lane-local
// stores, no warp cooperation): "truncate the path to c vertices, append n
// bytes, then emit" -- consecutive prime paths of a DFS share long prefixes,
// so a record carries only the few vertices pushed since the previous one.
// Records live in 512-byte chunks linked through their last word, allocated
// from a pool by atomic bump.  The expand kernel (expand.cuh) replays the
// streams into the canonical offsets/vertices arrays at exact offsets obtained
// from the per-unit counters this kernel also produces.
#pragma once

#include "kernels.cuh"

namespace tpg {

// ---------------------------------------------------------------- mask traits
template <class T>
struct MT;

template <>
struct MT<uint32_t> {
    static constexpr int W = 1, BITS = 32;
    static __device__ __forceinline__ uint32_t bit(int b) { return 1u << b; }
    static __device__ __forceinline__ void set(uint32_t &m, int b) { m |= 1u << b; }
    static __device__ __forceinline__ void clr(uint32_t &m, int b) { m &= ~(1u << b); }
    static __device__ __forceinline__ bool subset(uint32_t a, uint32_t b) { return (a & ~b) == 0u; }
    static __device__ __forceinline__ uint32_t andnot(uint32_t a, uint32_t b) { return a & ~b; }
    // lowest set bit >= k of (sin & (~M | sbit)), BITS if none
    static __device__ __forceinline__ int next(uint32_t sin, uint32_t M, uint32_t sbit, int k) {
        // k <= 32; the 64-bit shift clears everything for k = 32; ctz(0) = 32 = none
        const uint32_t c = sin & (~M | sbit) & (uint32_t)(0xffffffffull << k);
        return __clz(__brev(c));
    }
    static __device__ __forceinline__ uint32_t load(const uint64_t *w) { return (uint32_t)__ldg(w); }
    static __device__ __forceinline__ uint32_t from(const uint64_t *w) { return (uint32_t)w[0]; }
    static __device__ __forceinline__ void store(uint32_t m, uint64_t *w) { w[0] = m; }
};

template <>
struct MT<uint64_t> {
    static constexpr int W = 1, BITS = 64;
    static __device__ __forceinline__ uint64_t bit(int b) { return 1ull << b; }
    static __device__ __forceinline__ void set(uint64_t &m, int b) { m |= 1ull << b; }
    static __device__ __forceinline__ void clr(uint64_t &m, int b) { m &= ~(1ull << b); }
    static __device__ __forceinline__ bool subset(uint64_t a, uint64_t b) { return (a & ~b) == 0ull; }
    static __device__ __forceinline__ uint64_t andnot(uint64_t a, uint64_t b) { return a & ~b; }
    static __device__ __forceinline__ int next(uint64_t sin, uint64_t M, uint64_t sbit, int k) {
        const uint64_t c = sin & (~M | sbit) & ((k < 64) ? (~0ull << k) : 0ull);
        return __clzll(__brevll(c));  // 64 = none
    }
    static __device__ __forceinline__ uint64_t load(const uint64_t *w) { return __ldg(w); }
    static __device__ __forceinline__ uint64_t from(const uint64_t *w) { return w[0]; }
    static __device__ __forceinline__ void store(uint64_t m, uint64_t *w) { w[0] = m; }
};

template <int WW>
struct MT<Mask<WW>> {
    using T = Mask<WW>;
    static constexpr int W = WW, BITS = 64 * WW;
    static __device__ __forceinline__ T bit(int b) { return mbit<WW>(b); }
    static __device__ __forceinline__ void set(T &m, int b) { mset(m, b); }
    static __device__ __forceinline__ void clr(T &m, int b) { mclr(m, b); }
    static __device__ __forceinline__ bool subset(const T &a, const T &b) { return msubset(a, b); }
    static __device__ __forceinline__ T andnot(const T &a, const T &b) {
        T r;
#pragma unroll
        for (int i = 0; i < WW; i++) r.w[i] = a.w[i] & ~b.w[i];
        return r;
    }
    static __device__ __forceinline__ int next(const T &sin, const T &M, const T &sbit, int k) {
        return mnext(sin, M, sbit, k);
    }
    static __device__ __forceinline__ T load(const uint64_t *w) {
        T m;
#pragma unroll
        for (int i = 0; i < WW; i++) m.w[i] = __ldg(w + i);
        return m;
    }
    static __device__ __forceinline__ T from(const uint64_t *w) {
        T m;
#pragma unroll
        for (int i = 0; i < WW; i++) m.w[i] = w[i];
        return m;
    }
    static __device__ __forceinline__ void store(const T &m, uint64_t *w) {
#pragma unroll
        for (int i = 0; i < WW; i++) w[i] = m.w[i];
    }
};

// ---------------------------------------------------------------- records
// 64-bit path-delta record:
//   bits 0-2 type, bit 3 closure flag, bits 4-12 c (truncate the path to c
//   vertices), bits 13-15 n (number of appended vertices, <= 5),
//   bits 16-55 the n appended local vertex ids (one byte each).
// R_ARG carries the out-arc index of the HEAD / TRANSIT record directly after it, in bits 32-63.
enum RecType : int { R_PATH = 0, R_PP = EV_PP, R_HEAD = EV_HEAD, R_TAIL = EV_TAIL, R_TRANSIT = EV_TRANSIT, R_ARG = 6 };
constexpr int kChunkRecs = 64;  // records per chunk; the last word links to the next chunk
constexpr int kRecBytes = 5;    // appended vertices carried by one record
constexpr int kStepsPerIter = 16;// DFS steps per pass of the persistent loop
#ifndef GEN_POP2
#define GEN_POP2 1  // generic step: pop a second exhausted level in the same step
#endif
#ifndef TPGEN_LEAN_BLOCKS
#define TPGEN_LEAN_BLOCKS 3
#endif
constexpr int kLeanBlocks = TPGEN_LEAN_BLOCKS;  // resident LEAN blocks per SM (4 at 64 registers: faster DFS, more units, slower step)
constexpr int kEagerGens = 4;    // donation generations that split without waiting split_min steps (default)

// Event codes inside the DFS: type in bits 0-2, closure flag bit 3, path length in bits 8+.
constexpr int EV_CLO = 8;
__device__ __forceinline__ int ev_type(int ev) { return ev & 7; }
__device__ __forceinline__ int ev_len(int ev) { return ev >> 8; }

// shared-memory path layout: byte of level l of lane q at ((l>>2)*32 + q)*4 + (l&3)
__device__ __forceinline__ int pidx(int l) { return ((l >> 2) << 7) | (l & 3); }

// path bytes are addressed with 32-bit shared-window addresses
__device__ __forceinline__ int lds_u8(uint32_t a) {
    int v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ int lds_u32(uint32_t a) {
    int v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, int v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Up to 5 consecutive path bytes starting at position p (shared-memory layout of
// pidx): two 32-bit words of the lane's column, funnel-shifted.  Bytes past the
// record's count are left in place (decoders read only the first n); the word
// after the last level is a spare row of the path array.
__device__ __forceinline__ uint64_t path_bytes(uint32_t mp, int p) {
    const uint32_t a = mp + ((p >> 2) << 7);
    uint32_t lo, hi;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(a) : "memory");
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(a + 128) : "memory");
    return (((uint64_t)hi << 32) | lo) >> (8 * (p & 3));
}

template <class T>
struct Lane {
    T M, sbit, ps, sin;  // visited set, bit of s, pred(s) in SCC, succ(u) in SCC
    int32_t vb, s, u, l, r, k, o, ooff, ocnt, flags;
    uint32_t steps;
    bool active, done, seg, emit;
    // record stream state: the decoder knows path[0..base) (base <= l+1); the bytes
    // path[base..l] are read from the shared-memory path when the next record is written
    int32_t base;
    uint64_t S;  // count modes: digest sum of path[0..l] (R20), kept up to date by push and pop
};

// Per-slot digest values mix64(gid) (R20): staged in shared memory next to the slot table
// (TS), else read through L1.
template <bool TS>
struct MixTab {
    const uint64_t *g;
    uint32_t sb;  // TS: shared-window address
    __device__ __forceinline__ uint64_t operator()(int i) const {
        if (TS) {
            uint64_t v;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sb + (uint32_t)i * 8u) : "memory");
            return v;
        }
        return __ldg(g + i);
    }
};

// DFS kernel modes: M_REC writes the path-delta record streams (materialize, and the
// segment phase); M_CNT counts and digests every prime path in the walk itself (no
// records; COUNT_HASH); M_CNT_NOHASH counts only.
enum DfsMode : int { M_REC = 0, M_CNT = 1, M_CNT_NOHASH = 2 };

// View of the slot table: staged in shared memory (TS) when it fits, else read through L1.
// The shared copy is addressed through a 32-bit shared-window base kept in a register.
template <class T, bool TS>
struct ShTab {  // generic fallback (masks of several words): through the generic pointer
    static __device__ __forceinline__ T sin(const void *p, uint32_t, int i) {
        return MT<T>::from(reinterpret_cast<const Slot<MT<T>::W> *>(p)[i].sin);
    }
};
template <>
struct ShTab<uint32_t, true> {
    static __device__ __forceinline__ uint32_t sin(const void *, uint32_t sb, int i) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sb + (uint32_t)i * 32u) : "memory");
        return v;
    }
};
template <>
struct ShTab<uint64_t, true> {
    static __device__ __forceinline__ uint64_t sin(const void *, uint32_t sb, int i) {
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sb + (uint32_t)i * 32u) : "memory");
        return v;
    }
};
template <int W, bool TS>
struct TabView {
    const Slot<W> *p;
    uint32_t sb;  // TS: shared-window address of the table
    template <class T>
    __device__ __forceinline__ T sin(int i) const {
        if (TS && W == 1) return ShTab<T, true>::sin(p, sb, i);
        return TS ? MT<T>::from(p[i].sin) : MT<T>::load(p[i].sin);
    }
    template <class T>
    __device__ __forceinline__ T pin(int i) const {
        return TS ? MT<T>::from(p[i].pin) : MT<T>::load(p[i].pin);
    }
    __device__ __forceinline__ int4 meta(int i) const {
        if (TS && W == 1) {
            int4 v;
            asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(sb + (uint32_t)i * 32u + 16u)
                         : "memory");
            return v;
        }
        return TS ? *reinterpret_cast<const int4 *>(&p[i].gid) : ld_meta(p + i);
    }
};

template <class T, bool TS>
__device__ __forceinline__ void load_slot(const TabView<MT<T>::W, TS> &tab, Lane<T> &L, int u) {
    L.sin = tab.template sin<T>(L.vb + u);
    const int4 m = tab.meta(L.vb + u);
    L.ooff = m.y;
    L.ocnt = m.z;
    L.flags = m.w;
}

// Own event of a node whose last vertex is w (evaluated when the node is created).
//  PP mode (s not an SCC entry): internal acyclic prime path iff
//    succ(w) within {v2..vk} and pred(s) within {v1..v(k-1)}   (Def. 1 / Def. 9)
//  segment mode (s an SCC entry): tail segment iff succ(w) within the path  (R8)
template <class T>
__device__ __forceinline__ int node_event(const Lane<T> &L, int w) {
    using O = MT<T>;
    const int len = (L.l + 1) << 8;
    const bool tail = O::subset(L.sin, L.M);
    const bool pp = O::subset(L.sin, O::andnot(L.M, L.sbit)) && O::subset(L.ps, O::andnot(L.M, O::bit(w)));
    const int ev = L.seg ? (tail ? (EV_TAIL | len) : 0) : ((L.emit && pp) ? (EV_PP | len) : 0);
    return (L.flags & F_EXIT) ? 0 : ev;
}

// Arc to an out-of-SCC successor from the current node.
//  segment mode: transit segment item (Def. 6 -- all entry->exit paths, R9)
//  PP mode: a head segment iff pred(s) lies on the path (R8) -> cross block
template <class T>
__device__ __forceinline__ int out_event(const Lane<T> &L) {
    const int len = (L.l + 1) << 8;
    if (L.seg) return EV_TRANSIT | len;
    return MT<T>::subset(L.ps, L.M) ? (EV_HEAD | len) : 0;
}

// A lane writes the records of all its units into one chain of chunks: a unit
// starts wherever the previous one ended (rfirst = global record index), so
// starting a unit costs no allocation.  When a chunk fills, the lane switches to
// the chunk it reserved at its previous switch and reserves the next one (the
// atomic's result is needed only one chunk later).
struct RecWriter {
    uint64_t *cur;   // current chunk
    int fill;        // records used in it (kChunkRecs - 1: full, the next record needs a new chunk)
    long long next;  // chunk reserved for the next switch (-1: none)
    int count;       // records of the current unit
};

__device__ __forceinline__ void rec_switch(const DfsArgs &A, RecWriter &R) {
    unsigned long long nc = (R.next >= 0) ? (unsigned long long)R.next : atomicAdd(A.chunk_next, 1ull);
    R.next = (long long)atomicAdd(A.chunk_next, 1ull);
    if (nc >= A.chunk_cap) {  // pool exhausted: the phase is retried with a bigger pool;
        atomicOr(A.overflow, 2u);  // meanwhile write into the sink chunk past the end
        nc = A.chunk_cap;
    }
    TPG_DCHECK(nc <= A.chunk_cap, "dfs: chunk out of range");
    R.cur[kChunkRecs - 1] = nc;  // link
    R.cur = A.chunks + nc * kChunkRecs;
    R.fill = 0;
}

__device__ __forceinline__ void rec_put(const DfsArgs &A, RecWriter &R, uint64_t rec) {
    if (R.fill == kChunkRecs - 1) rec_switch(A, R);
    R.cur[R.fill++] = rec;
    R.count++;
}

// One step of the depth-first walk.  Children of a node are visited in
// ascending global id: in-SCC successors (local bits; ascending local id ==
// ascending global id), the closing arc back to s, and out-of-SCC successors
// (merged by their rank out_pos among the SCC members).  Returns the event.
// A step that exhausts a node pops it and, unless the parent still has
// out-of-SCC arcs to merge, moves on to the parent's next child in the same
// step (a pop costs no step of its own).
template <class T, bool TS, bool CNT>
__device__ __forceinline__ int dfs_step(const DfsArgs &A, const DevGraph &G, const TabView<MT<T>::W, TS> &tab,
                                        const MixTab<TS> &mt, Lane<T> &L, RecWriter &R, uint32_t mp, int &e_out,
                                        uint32_t &ext) {
    using O = MT<T>;
    int w = O::next(L.sin, L.M, L.sbit, L.k);
    if (L.o < L.ocnt) {  // exit vertex with out-of-SCC arcs still to visit
        const int e = L.ooff + L.o;
        if (__ldg(G.out_pos + e) <= w) {
            L.o++;
            e_out = e;
            return out_event(L);
        }
    }
    // straight-line, predicated: [pop] then [closure | push]
    const bool none = w >= O::BITS;
    const bool fin = none && L.l == L.r;  // subtree of the unit's root exhausted
    if (none && !fin) {  // pop, then the parent's next child (unless the parent merges out-arcs)
        const int wold = L.u;
        const int parent = lds_u8(mp + pidx(L.l - 1));
        L.M = O::andnot(L.M, O::bit(wold));
        if (CNT) L.S -= mt(L.vb + wold) * pos_weight((uint32_t)L.l);
        L.l -= 1;
        L.u = parent;
        load_slot(tab, L, parent);
        L.k = wold + 1;
        L.base = min(L.base, L.l + 1);  // the record decoder's known prefix shortens
        if (L.ocnt > 0) L.o = count_out_le(G, L.ooff, L.ocnt, wold);  // rare: an exit vertex
        w = (L.ocnt > 0) ? O::BITS : O::next(L.sin, L.M, L.sbit, L.k);
        if (GEN_POP2 && w >= O::BITS && L.ocnt == 0 && L.l > L.r) {  // the parent is exhausted too: one more level
            const int wold2 = L.u;
            const int parent2 = lds_u8(mp + pidx(L.l - 1));
            L.M = O::andnot(L.M, O::bit(wold2));
            if (CNT) L.S -= mt(L.vb + wold2) * pos_weight((uint32_t)L.l);
            L.l -= 1;
            L.u = parent2;
            load_slot(tab, L, parent2);
            L.k = wold2 + 1;
            L.base = min(L.base, L.l + 1);
            if (L.ocnt > 0) L.o = count_out_le(G, L.ooff, L.ocnt, wold2);
            w = (L.ocnt > 0) ? O::BITS : O::next(L.sin, L.M, L.sbit, L.k);
        }
    }
    if (fin) L.done = true;
    const bool go = !fin && w < O::BITS;
    const bool clo = go && w == L.s;  // cycle closure: always prime (Alg. 4 l.4-6)
    const bool push = go && !clo;
    if (go && L.emit) ext++;
    int ev = (clo && L.emit) ? (EV_PP | EV_CLO | ((L.l + 2) << 8)) : 0;
    if (clo) L.k = w + 1;
    if (push) {
        sts_u8(mp + pidx(L.l + 1), w);
        if (CNT) L.S += mt(L.vb + w) * pos_weight((uint32_t)(L.l + 1));
        L.M = L.M | O::bit(w);
        L.k = 0;
        L.l += 1;
        L.u = w;
        load_slot(tab, L, w);
        L.o = 0;
        ev = node_event(L, w);
    }
    return ev;
}

// ---------------------------------------------------------------- lean step
// LEAN kernels (engine.cu picks them): prime-path mode only, 32-bit masks, and
// no vertex of the call has an arc leaving its SCC -- so there are no head,
// tail or transit events and a node's children are exactly the bits of
// succ(u) & (~M | {s}) in ascending local (= global) id, the bit of s being the
// closing arc (Alg. 4 l.4-6).  The lane keeps the untried children
// of its current node in L.sin and those of every ancestor in a shared-memory
// stack rem[level] (one 32-bit word per level, [level][lane] so the lanes of a
// warp never share a bank): a pop is two independent shared loads, a push two
// shared stores and one slot-table load, with no next-child search.
#ifndef LEAN_POPS
#define LEAN_POPS 2  // levels a LEAN step may pop (measured: 1 -> 2 saves 5 % of the DFS)
#endif
__device__ __forceinline__ uint32_t lane_rem(uint32_t rp, int l) { return (uint32_t)lds_u32(rp + ((uint32_t)l << 7)); }

// Own event of a node reached by pushing w (c = its children, Mp = the mask before w):
// internal prime path iff succ(w) within {v2..vk} (c == 0: no child, no closure)
// and pred(s) within {v1..v(k-1)} (Def. 1 / Def. 9; R3).
__device__ __forceinline__ int lean_node_event(uint32_t c, uint32_t ps, uint32_t Mp, int l, bool emit) {
    return (emit && c == 0u && (ps & ~Mp) == 0u) ? (EV_PP | ((l + 1) << 8)) : 0;
}

#ifndef LEAN_PRED
#define LEAN_PRED 1  // 1: the LEAN step as one straight-line predicated stream (pops, then the take);
                     // config 3 materialized dfs_kernel 2.655 -> 2.460 ms (A/B on one box)
#endif
template <bool TS, bool CNT>
__device__ __forceinline__ int lean_step(const TabView<1, TS> &tab, const MixTab<TS> &mt, Lane<uint32_t> &L,
                                         uint32_t mp, uint32_t rp, uint32_t &ext) {
#if LEAN_PRED
    // the same moves as below, without branches: every lane executes every instruction, the
    // predicates select (the walk order, hence the record stream, is unchanged)
#pragma unroll
    for (int x = 0; x < LEAN_POPS; x++) {
        const bool pk = (L.sin == 0u) & (L.l > L.r);
        const int u = lds_u8(mp + pidx(L.l));
        if (CNT) L.S -= pk ? mt(L.vb + u) * pos_weight((uint32_t)L.l) : 0ull;
        const int lp = pk ? L.l - 1 : L.l;
        const uint32_t rem = lane_rem(rp, lp);
        L.sin = pk ? rem : L.sin;
        L.M &= pk ? ~(1u << u) : ~0u;
        L.base = pk ? min(L.base, lp + 1) : L.base;
        L.l = lp;
    }
    const bool empty = L.sin == 0u;
    if (empty & (L.l == L.r)) L.done = true;
    const bool take = !empty;
    const int w = __ffs(L.sin) - 1;  // (take)
    const int wv = take ? w : 0;     // (lanes that do not take read local vertex 0: a valid slot)
    const uint32_t rest = L.sin & (L.sin - 1u);
    ext += (take & L.emit) ? 1u : 0u;
    const bool clo = take & (w == L.s);
    const bool push = take & !clo;
    if (push) {
        sts_u32(rp + ((uint32_t)L.l << 7), rest);
        sts_u8(mp + pidx(L.l + 1), w);
    }
    if (CNT) L.S += push ? mt(L.vb + wv) * pos_weight((uint32_t)(L.l + 1)) : 0ull;
    const uint32_t Mp = L.M;
    const uint32_t Mn = Mp | (1u << wv);
    const uint32_t cw = tab.template sin<uint32_t>(L.vb + wv) & (~Mn | L.sbit);
    L.M = push ? Mn : Mp;
    L.l += push ? 1 : 0;
    L.sin = push ? cw : (take ? rest : L.sin);
    const int evc = L.emit ? (EV_PP | EV_CLO | ((L.l + 2) << 8)) : 0;
    const int evn = lean_node_event(cw, L.ps, Mp, L.l, L.emit);
    return clo ? evc : (push ? evn : 0);
#endif
    const bool pop = L.sin == 0u;
    const bool fin = pop && L.l == L.r;  // the unit's subtree is exhausted
    if (pop && !fin) {                   // back to the parent and its untried children
        const int u = lds_u8(mp + pidx(L.l));
        if (CNT) L.S -= mt(L.vb + u) * pos_weight((uint32_t)L.l);
        L.l -= 1;
        L.sin = lane_rem(rp, L.l);
        L.M &= ~(1u << u);
        L.base = min(L.base, L.l + 1);  // the record decoder's known prefix shortens
#pragma unroll
        for (int x = 1; x < LEAN_POPS; x++) {  // exhausted ancestors: more levels in the same step
            if (L.sin == 0u && L.l > L.r) {
                const int u2 = lds_u8(mp + pidx(L.l));
                if (CNT) L.S -= mt(L.vb + u2) * pos_weight((uint32_t)L.l);
                L.l -= 1;
                L.sin = lane_rem(rp, L.l);
                L.M &= ~(1u << u2);
                L.base = min(L.base, L.l + 1);
            }
        }
    }
    if (fin) L.done = true;
    int ev = 0;
    if (!fin && L.sin != 0u) {
        const int w = __ffs(L.sin) - 1;
        L.sin &= L.sin - 1u;
        if (L.emit) ext++;
        if (w == L.s) {  // cycle closure: always prime (Alg. 4 l.4-6)
            ev = L.emit ? (EV_PP | EV_CLO | ((L.l + 2) << 8)) : 0;
        } else {
            sts_u32(rp + ((uint32_t)L.l << 7), L.sin);
            sts_u8(mp + pidx(L.l + 1), w);
            if (CNT) L.S += mt(L.vb + w) * pos_weight((uint32_t)(L.l + 1));
            const uint32_t Mp = L.M;
            L.M |= 1u << w;
            L.l += 1;
            L.sin = tab.template sin<uint32_t>(L.vb + w) & (~L.M | L.sbit);
            ev = lean_node_event(L.sin, L.ps, Mp, L.l, L.emit);
        }
    }
    return ev;
}

// Donation for LEAN lanes: the untried children of the shallowest level j0 in
// [r, l] that has any (rem[j0], or L.sin when j0 == l), as units in ascending id.
template <bool TS, bool WRITE>
__device__ int lean_donate(const Lane<uint32_t> &L, uint32_t mp, uint32_t rp, int uscc, int &j0, Unit<1> *out) {
    if (!WRITE) {
        for (int j = L.r; j <= L.l; j++) {
            const uint32_t c = (j == L.l) ? L.sin : lane_rem(rp, j);
            if (c) {
                j0 = j;
                return __popc(c);
            }
        }
        return 0;
    }
    uint32_t c = (j0 == L.l) ? L.sin : lane_rem(rp, j0);
    uint32_t M = L.M;  // the mask of path[0..j0]
    for (int j = j0 + 1; j <= L.l; j++) M &= ~(1u << lds_u8(mp + pidx(j)));
    int n = 0;
    while (c) {
        const int w = __ffs(c) - 1;
        c &= c - 1u;
        const int kind = (w == L.s) ? K_CLOSURE : K_NODE;
        Unit<1> &U = out[n];
        uint32_t *pw = reinterpret_cast<uint32_t *>(U.path);
        for (int q = 0; q <= (j0 >> 2); q++) pw[q] = (uint32_t)lds_u32(mp + (q << 7));
        uint64_t Mu = M;
        if (kind == K_NODE) {
            U.path[j0 + 1] = (uint8_t)w;
            Mu |= 1ull << w;
        }
        U.M[0] = Mu;
        const int depth = (kind == K_NODE) ? j0 + 1 : j0;
        *reinterpret_cast<int4 *>(&U.scc) = make_int4(uscc, -1, 0, depth | (kind << 8));
        n++;
    }
    return n;
}

template <class T>
struct DfsTraits {
    static constexpr int W = MT<T>::W;
    static constexpr int threads = DfsCfg<W>::threads;
    static constexpr int warps = DfsCfg<W>::warps;
    static constexpr int min_blocks = DfsCfg<W>::min_blocks;
};

// queue counters are polled with GPU-scope relaxed loads (a volatile load would be system scope)
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_flags(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// hand-off of queued units between lanes of different SMs: the producer fences once after
// writing a block of units, then sets their ready flags with relaxed stores
__device__ __forceinline__ void st_relaxed(unsigned int *p, unsigned int v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// The consumer polls the flag with a relaxed load; once it sees the flag set it
// issues a fence.acq_rel (the acquire half of the hand-off: one per claimed unit)
// and then its L2 (.cg) loads of the unit payload.
__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Donation: the untried events (children in ascending global id) of the
// shallowest node on the lane's stack that still has any -- the largest
// subtrees left in the unit.  WRITE=false finds that level (j0) and counts the
// events; WRITE=true writes them as units.  The lane keeps everything below
// level j0 and stops when its walk returns to depth j0+1, so its remaining
// output precedes the donated units in lexicographic order.
template <class T, bool TS, bool WRITE>
__device__ int lane_donate(const DevGraph &G, const TabView<MT<T>::W, TS> &tab, const Lane<T> &L, uint32_t mp,
                           int uscc, int &j0, Unit<MT<T>::W> *out) {
    using O = MT<T>;
    constexpr int W = O::W;
    T M = L.M;
    int best = 0;
    for (int j = L.l; j >= L.r; j--) {
        const int u = lds_u8(mp + pidx(j));
        const T sin = tab.template sin<T>(L.vb + u);
        const int4 meta = tab.meta(L.vb + u);
        int k, o;
        if (j == L.l) {
            k = L.k;
            o = L.o;
        } else {
            const int wc = lds_u8(mp + pidx(j + 1));
            O::clr(M, wc);
            k = wc + 1;
            o = count_out_le(G, meta.y, meta.z, wc);
        }
        if (WRITE && j != j0) continue;
        int n = 0;
        while (true) {
            const int w = O::next(sin, M, L.sbit, k);
            int kind = -1, e = -1;
            if (o < meta.z && __ldg(G.out_pos + meta.y + o) <= w) {
                e = meta.y + o;
                o++;
                if (L.seg || O::subset(L.ps, M)) kind = K_OUT;
            } else {
                if (w >= O::BITS) break;
                k = w + 1;
                kind = (w == L.s) ? K_CLOSURE : K_NODE;
            }
            if (kind < 0) continue;
            if (WRITE) {
                Unit<W> &U = out[n];
                const int depth = (kind == K_NODE) ? j + 1 : j;
                uint32_t *pw = reinterpret_cast<uint32_t *>(U.path);
                for (int q = 0; q <= (j >> 2); q++) pw[q] = (uint32_t)lds_u32(mp + (q << 7));
                T Mu = M;
                if (kind == K_NODE) {
                    U.path[j + 1] = (uint8_t)w;
                    O::set(Mu, w);
                }
                O::store(Mu, U.M);
                *reinterpret_cast<int4 *>(&U.scc) = make_int4(uscc, e, 0, depth | (kind << 8));
            }
            n++;
        }
        if (WRITE) return n;
        if (n > 0) {
            best = n;
            j0 = j;
        }
    }
    return best;
}

// Persistent DFS kernel with an in-kernel work queue.  Idle lanes claim the
// units that are queued (warp-aggregated atomic on the head); a running lane
// whose unit has taken at least split_min steps splits it when the backlog of
// queued, unclaimed units falls below low_water: its walk so far becomes a
// finished piece and the untried siblings on its stack are pushed as new units
// (children of the piece in the unit forest).  The kernel ends when every
// pushed unit has finished (done == tail; both live in one 64-bit word so a
// single load gives a consistent snapshot).
//
// Count modes (MODE = M_CNT / M_CNT_NOHASH; COUNT_HASH calls, prime-path phase): no
// record stream and no per-unit results.  The lane keeps the digest sum S of its path
// in a register (push: + mix(v) * (2l+1), pop: the same subtracted; R20); a prime path
// found by a step is queued per warp (S, length) and the warp hashes 32 queued paths at
// once, one per lane, so the two splitmix64 finalizers never run divergently.  A head
// segment (an exit vertex with out-of-SCC arcs, pred(s) on the path) adds its W(x)
// cross prime paths to the counts and is written as a HeadS {S, |h|, x} into the warp's
// current block of 256 head slots (one atomic per block) for stitch_hash_s_kernel.
// Totals are reduced per warp into A.cacc when the kernel ends.
template <class T, bool TS, bool LEAN, int MODE>
__global__ void __launch_bounds__(DfsTraits<T>::threads, LEAN ? kLeanBlocks : DfsTraits<T>::min_blocks) dfs_kernel(DfsArgs A) {
    using O = MT<T>;
    constexpr int W = O::W;
    constexpr int WARPS = DfsTraits<T>::warps;
    constexpr bool CNT = MODE != M_REC;
    constexpr bool HSH = MODE == M_CNT;
    static_assert(!LEAN || MT<T>::BITS == 32, "LEAN kernels use 32-bit masks");
    static_assert(!CNT || W == 1, "count modes use one mask word");
    constexpr int PLEV = LEAN ? 32 : 64 * W;  // path levels per lane
    __shared__ __align__(16) uint8_t spath[WARPS * PLEV * 32 + 128];  // + a spare row (path_bytes)
    __shared__ __align__(16) uint32_t srem[LEAN ? WARPS * 32 * 32 : 1];  // LEAN: rem[level][lane] per warp
    __shared__ __align__(16) uint64_t sqS[HSH ? WARPS * 64 : 1];  // count mode: per warp, queued prime paths' S
    __shared__ uint16_t sqL[HSH ? WARPS * 64 : 1];                // ... and their lengths
    extern __shared__ __align__(16) uint8_t stab[];  // slot table copy (TS); count modes: then the mix table
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t mp;  // this lane's column of the shared path array (opaque: not recomputed in the loop)
    asm volatile("mov.b32 %0, %1;" : "=r"(mp) : "r"((uint32_t)__cvta_generic_to_shared(spath + wid * PLEV * 32) + lane * 4));
    uint32_t rp;  // LEAN: this lane's column of the rem stack (level l at rp + 128 l)
    asm volatile("mov.b32 %0, %1;" : "=r"(rp) : "r"((uint32_t)__cvta_generic_to_shared(srem + (LEAN ? wid * 32 * 32 : 0)) + (LEAN ? lane * 4 : 0)));
    const DevGraph &G = A.G;
    TabView<W, TS> tab;
    MixTab<TS> mt;
    mt.g = G.slot_mix;
    mt.sb = 0;
    if (TS) {
        const int4 *src = reinterpret_cast<const int4 *>(G.slots);
        int4 *dst = reinterpret_cast<int4 *>(stab);
        for (int i = threadIdx.x; i < A.n_slots * (int)(sizeof(Slot<W>) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
        if (CNT) {
            uint64_t *dm = reinterpret_cast<uint64_t *>(stab + (size_t)A.n_slots * sizeof(Slot<W>));
            for (int i = threadIdx.x; i < A.n_slots; i += blockDim.x) dm[i] = __ldg(G.slot_mix + i);
        }
        __syncthreads();
        tab.p = reinterpret_cast<const Slot<W> *>(stab);
        asm volatile("mov.b32 %0, %1;" : "=r"(tab.sb) : "r"((uint32_t)__cvta_generic_to_shared(stab)));
        mt.sb = tab.sb + (uint32_t)((size_t)A.n_slots * sizeof(Slot<W>));
    } else {
        tab.p = reinterpret_cast<const Slot<W> *>(G.slots);
        tab.sb = 0;
    }
    // count modes: the warp's prime-path queue, per-lane totals, the warp's head-slot block
    uint64_t *qS = sqS + (HSH ? wid * 64 : 0);
    uint16_t *qL = sqL + (HSH ? wid * 64 : 0);
    uint32_t qn = 0;                                  // queued prime paths (warp-uniform, < 32 between drains)
    uint64_t t_pp = 0, t_vert = 0, t_ext = 0, t_ha = 0, t_hb = 0, t_cross = 0;
    unsigned long long hblk = 0, hblk_end = 0;       // warp-uniform: next free / end of the warp's head block
    const uint32_t lt_mask = (1u << lane) - 1u;
    Unit<W> *units = reinterpret_cast<Unit<W> *>(A.units);

    Lane<T> L;
    L.active = false;
    L.done = false;
    bool waiting = false, exited = false;
    int64_t slot = -1;
    int32_t uscc = 0, ugen = 0;
    uint64_t c_pp = 0, c_vert = 0;                          // per-unit counters (C_PP, C_VERT)
    uint32_t c_it = 0, c_itv = 0, c_hd = 0, c_hdv = 0, ext = 0;  // C_ITEMS, C_ITEMV, C_HEADS, C_HEADV, E_canon
    RecWriter R;
    R.cur = A.chunks + A.chunk_cap * kChunkRecs;  // the sink chunk, marked full: the first record allocates
    R.fill = kChunkRecs - 1;
    R.next = -1;
    R.count = 0;

    int64_t child_head = -1;  // latest donated block of the running unit
    int nchild = 0;           // units donated by the running unit
#ifdef TPGEN_KERNEL_DEBUG
    unsigned long long d_it = 0, d_act = 0, d_don = 0, d_last = 0, d_prev = 0, d_lt = 0;
    const unsigned long long t0 = A.dbg ? A.dbg[7] : 0;
#endif
    uint32_t last_split = 0;
    uint32_t iter = 0;
    // Queue traffic is software-pipelined: every global load or atomic whose
    // result the warp needs is issued in one iteration and consumed in the next,
    // so its L2 round trip overlaps a DFS step instead of stalling the warp.
    unsigned rdy = 0;                       // waiting lanes: ready flag of `slot`, loaded last iteration
    bool claim_pending = false;             // warp-uniform: a claim atomic is in flight
    unsigned claim_mask = 0;                // lanes the claim is for
    int claim_leader = 0;
    unsigned long long claim_res = 0;       // leader: first claimed slot
    bool snap_pending = false;              // warp-uniform: lane 0 loaded the queue words last iteration
    unsigned long long snap_td = 0, snap_head = 0;
    unsigned snap_ov = 0;
    bool qdone = false;                     // every pushed unit finished (or the pool/queue overflowed)
    bool prev_active = true;
    __shared__ unsigned long long s_td, s_head;  // warp 0's latest queue snapshot
    __shared__ unsigned s_ov;
    if (threadIdx.x == 0) {
        s_td = 1ull << 32;  // until warp 0's first snapshot: work pending (tail 1, done 0) and lanes
        s_head = 1ull << 20;  // waiting for it (backlog negative), so the first units split at once
        s_ov = 0;
    }
    __syncthreads();
    while (true) {
        int ev = 0, e = -1;
        iter++;
        // ---------------- consume last iteration's queue snapshot / claim
        // The queue words are polled by warp 0 of each block only (the lines they live on are
        // hot: every claim, push and completion is an atomic on them); it publishes its
        // snapshot in shared memory, where the other warps read it.
        bool feed = false;
        uint32_t split_need = A.split_min;  // steps a unit runs before it may donate
        {
            bool have = false;
            unsigned long long td = 0, hd = 0;
            unsigned ov = 0;
            if (wid == 0) {
                if (snap_pending) {
                    td = __shfl_sync(kFull, snap_td, 0);
                    hd = __shfl_sync(kFull, snap_head, 0);
                    ov = __shfl_sync(kFull, snap_ov, 0);
                    if (lane == 0) {
                        *reinterpret_cast<volatile unsigned long long *>(&s_td) = td;
                        *reinterpret_cast<volatile unsigned long long *>(&s_head) = hd;
                        *reinterpret_cast<volatile unsigned *>(&s_ov) = ov;
                    }
                    snap_pending = false;
                    have = true;
                }
            } else if (((iter & 1u) == 0u) || !prev_active) {
                td = *reinterpret_cast<volatile unsigned long long *>(&s_td);
                hd = *reinterpret_cast<volatile unsigned long long *>(&s_head);
                ov = *reinterpret_cast<volatile unsigned *>(&s_ov);
                have = true;
            }
            if (have) {
                qdone = ((td >> 32) == (td & 0xffffffffull)) || ((ov & 6u) != 0u);
                // donate when the backlog of queued, unclaimed units is below the low-water mark
                const long long backlog = (long long)(td >> 32) - (long long)hd;
                feed = backlog < (long long)A.low_water;
                // many lanes waiting for work (the end game): split after few steps
                if (backlog < -(long long)A.starve_lanes) split_need = A.split_min_starve;
            }
        }
        // ---------------- waiting lanes: start the unit once written, or stop when all work is done
        if (waiting) {
            if (rdy != 0u) {
                waiting = false;
                // acquire: the producer's unit stores (released by its fence before the flag) are
                // visible to the loads below (Theorem-2-style race freedom of the hand-off)
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                // queue slots are written by other SMs during this launch: read them at L2 (ld.cg)
                TPG_DCHECK(slot >= 0 && slot < (int64_t)A.qcap, "dfs: claimed slot out of range");
                const Unit<W> *U = units + slot;
                const int4 h = __ldcg(reinterpret_cast<const int4 *>(&U->scc));  // scc, e, -, depth|kind
                {
                    uint64_t mw[W];
#pragma unroll
                    for (int i = 0; i < W; i++) mw[i] = __ldcg(reinterpret_cast<const unsigned long long *>(U->M) + i);
                    L.M = O::from(mw);
                }
                uscc = h.x;
                ugen = __ldcg(A.gen + slot);
                const int kind = (h.w >> 8) & 0xff;
                const int depth = h.w & 0xff;
                L.l = L.r = depth;
                const uint4 *p4 = reinterpret_cast<const uint4 *>(U->path);
#pragma unroll 1
                for (int q = 0; q * 16 <= depth; q++) {
                    const uint4 v = __ldcg(p4 + q);
                    const uint32_t wa = mp + pidx(q * 16);  // 4 levels per 32-bit smem word
                    sts_u32(wa, v.x);
                    if (q * 16 + 4 <= depth) sts_u32(wa + 128, v.y);
                    if (q * 16 + 8 <= depth) sts_u32(wa + 256, v.z);
                    if (q * 16 + 12 <= depth) sts_u32(wa + 384, v.w);
                }
                const int s = lds_u8(mp);
                const int u = lds_u8(mp + pidx(depth));
                L.s = s;
                L.u = u;
                L.sbit = O::bit(s);
                L.vb = __ldg(G.scc_vbase + uscc);
                L.ps = tab.template pin<T>(L.vb + s);
                const int4 sm = tab.meta(L.vb + s);
                L.seg = (sm.w & F_ENTRY) != 0;
                L.emit = sm.x >= G.shard_lo && sm.x < G.shard_hi;
                L.k = 0;
                L.o = 0;
                L.steps = 0;
                L.done = false;
                L.active = true;
                child_head = -1;
                nchild = 0;
                last_split = 0;
                L.base = depth + 1;
                ext = 0;
                c_pp = c_vert = 0;
                c_it = c_itv = c_hd = c_hdv = 0;
                if constexpr (CNT) {  // the digest sum of the unit's root path
                    uint64_t S0 = 0;
                    for (int i = 0; i <= depth; i++) S0 += mt(L.vb + lds_u8(mp + pidx(i))) * pos_weight((uint32_t)i);
                    L.S = S0;
                } else {
                    if (R.fill == kChunkRecs - 1) rec_switch(A, R);
                    A.rfirst[slot] = (int64_t)(R.cur - A.chunks) + R.fill;  // global record index
                    R.count = 0;
                }
                // the unit's root event (no step is counted for it)
                bool lean_root = false;
                if constexpr (LEAN) {  // the root's children; its own event
                    if (kind == K_NODE) {
                        L.sin = tab.template sin<T>(L.vb + u) & (~L.M | L.sbit);
                        if (depth > 0 && L.emit) ext++;
                        ev = lean_node_event(L.sin, L.ps, L.M & ~O::bit(u), depth, L.emit);
                        lean_root = true;
                    }
                }
                if (lean_root) {
                } else if (kind == K_NODE) {
                    load_slot(tab, L, u);
                    if (depth > 0 && L.emit) ext++;
                    ev = node_event(L, u);
                } else if (kind == K_CLOSURE) {
                    L.done = true;
                    if (L.emit) {
                        ext++;
                        ev = EV_PP | EV_CLO | ((depth + 2) << 8);
                    }
                } else {  // K_OUT
                    L.done = true;
                    e = h.y;
                    ev = out_event(L);
                }
            } else if (qdone) {
                // nothing is running that could still push this slot (done == tail implies slot >= tail)
                waiting = false;
                exited = true;
            } else if (slot < (int64_t)A.qcap) {
                rdy = ld_relaxed(A.ready + slot);  // consumed next iteration
            }
        }
        // ---------------- the claim issued last iteration: take the slots, poll their flags next iteration
        if (claim_pending) {
            const unsigned long long base = __shfl_sync(kFull, claim_res, claim_leader);
            if ((claim_mask >> lane) & 1u) {
                slot = (int64_t)(base + __popc(claim_mask & ((1u << lane) - 1u)));
                waiting = true;  // the slot may lie beyond the tail: wait until it is pushed
                rdy = (slot < (int64_t)A.qcap) ? ld_relaxed(A.ready + slot) : 0u;
            }
            claim_pending = false;
        }
        // ---------------- idle lanes claim the next slots (one atomic per warp, consumed next iteration)
        {
            const unsigned need = __ballot_sync(kFull, !L.active && !waiting && !exited);
            if (need && !claim_pending) {
                claim_leader = __ffs(need) - 1;
                claim_mask = need;
                claim_pending = true;
                if (lane == claim_leader) claim_res = atomicAdd(A.qhead, (unsigned long long)__popc(need));
            }
        }
        // ---------------- queue snapshot for donation / termination (lane 0, consumed next iteration)
        const bool any_active = __ballot_sync(kFull, L.active) != 0;
        prev_active = any_active;
        if (wid == 0 && !snap_pending && (((iter & 1u) == 0u) || !any_active)) {
            if (lane == 0) {
                snap_td = ld_volatile(A.qtd);
                snap_head = ld_volatile(A.qhead);
                snap_ov = ld_flags(A.overflow);
            }
            snap_pending = true;
        }
#ifdef TPGEN_KERNEL_DEBUG
        d_it++;
        {
            const int na = __popc(__ballot_sync(kFull, L.active));
            d_act += na;
            if (A.dbg && lane == 0) {  // time-weighted timeline: 64 buckets of 0.1 ms
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (d_last == 0) {
                    d_last = now;
                } else {
                    d_lt += (unsigned long long)na * (now - d_prev);  // lanes busy since the last pass
                    if (now - d_last > 2000ull) {                     // flush about every 2 us
                        const unsigned long long bkt = min((now - t0) / 100000ull, 63ull);
                        atomicAdd(A.dbg + 8 + 2 * bkt, d_lt);
                        atomicAdd(A.dbg + 9 + 2 * bkt, 32ull * (now - d_last));
                        d_lt = 0;
                        d_last = now;
                    }
                }
                d_prev = now;
            }
        }
#endif
        if (!any_active) {
            if (__ballot_sync(kFull, !exited) == 0) break;
            __nanosleep(128);
            continue;
        }

        // ---------------- kStepsPerIter DFS steps for every running lane; the queue housekeeping
        // above runs once per kStepsPerIter steps (lanes that just started emit their root event first)
#pragma unroll 1
        // (the event of a step is written at the top of the next pass of this loop; a unit
        // that just started carries its root event into the first pass; pass kStepsPerIter
        // only writes the last step's event)
        for (int t = 0; t <= kStepsPerIter; t++) {
            // ---------------- event: counters + one record (lane-local)
            if constexpr (CNT) {
                // count modes: prime paths into the warp queue, head segments into the head block
                const int ty = ev ? ev_type(ev) : 0;
                const uint32_t len = (uint32_t)ev_len(ev);
                const bool is_pp = ev && (LEAN || ty == EV_PP);
                const bool is_head = !LEAN && ev && ty == EV_HEAD;
                uint64_t Sx = L.S;
                if (is_pp) {
                    if (ev & EV_CLO) Sx += mt(L.vb + L.s) * pos_weight(len - 1);  // the closing vertex s
                    t_pp += 1;
                    t_vert += len;
                }
                if constexpr (HSH) {
                    const uint32_t bal = __ballot_sync(kFull, is_pp);
                    if (bal) {
                        if (is_pp) {
                            const uint32_t j = qn + __popc(bal & lt_mask);
                            qS[j] = Sx;
                            qL[j] = (uint16_t)len;
                        }
                        qn += __popc(bal);
                        if (qn >= 32) {
                            __syncwarp();
                            qn -= 32;
                            const uint64_t z = qS[qn + lane];
                            const uint64_t n = qL[qn + lane];
                            t_ha += mix64(z ^ (kSeedA + n));
                            t_hb += mix64(z ^ (kSeedB + n));
                            __syncwarp();
                        }
                    }
                }
                if constexpr (!LEAN) {
                    const uint32_t hb = HSH ? __ballot_sync(kFull, is_head) : 0u;
                    if (!HSH && is_head) {  // counts only: no head records
                        const int32_t x = __ldg(G.out_gid + e);
                        const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                        t_pp = sat_add(t_pp, Wx, A.overflow);
                        t_cross = sat_add(t_cross, Wx, A.overflow);
                        t_vert = sat_add(t_vert, sat_add(sat_mul((uint64_t)len, Wx, A.overflow), Vx, A.overflow),
                                         A.overflow);
                    }
                    if (hb) {
                        const uint32_t need = __popc(hb);
                        if (hblk + need > hblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                            for (unsigned long long j = hblk + lane; j < hblk_end; j += 32)
                                if (j < A.head_cap) A.heads[j].x = -1;
                            unsigned long long b = 0;
                            if (lane == 0) b = atomicAdd(A.cacc + 5, 256ull);
                            b = __shfl_sync(kFull, b, 0);
                            hblk = b;
                            hblk_end = b + 256;
                            if (b + 256 > A.head_cap && lane == 0) atomicOr(A.overflow, 8u);
                        }
                        if (is_head) {
                            const unsigned long long j = hblk + __popc(hb & lt_mask);
                            const int32_t x = __ldg(G.out_gid + e);
                            if (j < A.head_cap) {
                                HeadS hr;
                                hr.S = Sx;
                                hr.len = (int32_t)len;
                                hr.x = x;
                                *reinterpret_cast<ulonglong2 *>(A.heads + j) =
                                    *reinterpret_cast<const ulonglong2 *>(&hr);
                            }
                            const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                            t_pp = sat_add(t_pp, Wx, A.overflow);
                            t_cross = sat_add(t_cross, Wx, A.overflow);
                            t_vert = sat_add(t_vert, sat_add(sat_mul((uint64_t)len, Wx, A.overflow), Vx, A.overflow),
                                             A.overflow);
                        }
                        hblk += need;
                    }
                }
            } else if (ev) {
                const int ty = ev_type(ev);
                const uint64_t len = (uint64_t)ev_len(ev);
                // the bytes path[base..l] the decoder lacks, <= kRecBytes per record
                int nb = L.l + 1 - L.base;
                while (nb > kRecBytes) {  // continuation records
                    rec_put(A, R, (uint64_t)R_PATH | ((uint64_t)L.base << 4) | ((uint64_t)kRecBytes << 13) |
                                      (path_bytes(mp, L.base) << 16));
                    L.base += kRecBytes;
                    nb -= kRecBytes;
                }
                // HEAD / TRANSIT carry their out-arc in an R_ARG record written directly before them
                if (!LEAN && (ty == EV_HEAD || ty == EV_TRANSIT)) rec_put(A, R, (uint64_t)R_ARG | ((uint64_t)(uint32_t)e << 32));
                rec_put(A, R, (uint64_t)ty | (uint64_t)(ev & EV_CLO) | ((uint64_t)L.base << 4) | ((uint64_t)nb << 13) |
                                  (path_bytes(mp, L.base) << 16));
                L.base = L.l + 1;
                if (LEAN || ty == EV_PP) {
                    c_pp += 1;
                    c_vert += len;
                } else if (ty == EV_HEAD) {
                    const int32_t x = __ldg(G.out_gid + e);
                    const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                    c_pp = sat_add(c_pp, Wx, A.overflow);
                    c_vert = sat_add(c_vert, sat_add(sat_mul(len, Wx, A.overflow), Vx, A.overflow), A.overflow);
                    c_hd += 1;
                    c_hdv += (uint32_t)len;
                } else if (ty == EV_TAIL) {
                    c_it += 1;
                    c_itv += (uint32_t)len;
                    atomicAdd(A.agg_tail_cnt + L.vb + L.s, 1ull);
                    atomicAdd(A.agg_tail_len + L.vb + L.s, (unsigned long long)len);
                } else {  // EV_TRANSIT
                    c_it += 1;
                    c_itv += (uint32_t)len;
                    const int32_t nout = __ldg(G.scc_nout + uscc);
                    const int64_t pair = __ldg(G.scc_pair_base + uscc) +
                                         (int64_t)__ldg(G.slot_eidx + L.vb + L.s) * nout - __ldg(G.scc_out_base + uscc) + e;
                    atomicAdd(A.agg_pair_cnt + pair, 1ull);
                    atomicAdd(A.agg_pair_len + pair, (unsigned long long)len);
                }
            }
            ev = 0;
            if (t < kStepsPerIter && L.active && !L.done) {
                if constexpr (LEAN) {
                    ev = lean_step<TS, CNT>(tab, mt, L, mp, rp, ext);
                } else {
                    ev = dfs_step<T, TS, CNT>(A, G, tab, mt, L, R, mp, e, ext);
                }
            }
        }
        if (L.active) L.steps += kStepsPerIter;  // (approximate: only the donation policy reads it)

        // ---------------- donate on demand (feed: set by this iteration's queue snapshot)
        // (the first generations split at once: the walk starts from one unit per start
        // vertex and every lane of the GPU needs work)
        if (feed && L.active && !L.done && (L.steps - last_split >= split_need || ugen < A.eager_gens)) {
            // backlog of queued, unclaimed units below the low-water mark: donate the shallowest siblings
            int j0 = -1;
            int m;
            if constexpr (LEAN) m = lean_donate<TS, false>(L, mp, rp, uscc, j0, nullptr);
            else m = lane_donate<T, TS, false>(G, tab, L, mp, uscc, j0, nullptr);
            if (m > 0) {
                const unsigned long long base = atomicAdd(A.qtd, (unsigned long long)m << 32) >> 32;
                const unsigned long long b = base;  // a block is named by its first slot
                if (base + m > A.qcap) {
                    atomicOr(A.overflow, 4u);
                } else {
                    if constexpr (LEAN) lean_donate<TS, true>(L, mp, rp, uscc, j0, units + base);
                    else lane_donate<T, TS, true>(G, tab, L, mp, uscc, j0, units + base);
                    for (int i = 0; i < m; i++) A.gen[base + i] = ugen + 1;
                    if constexpr (!CNT) {  // the unit forest (canonical order of the records)
                        for (int i = 0; i < m; i++) {
                            A.child_head[base + i] = -1;
                            A.parent[base + i] = slot;
                        }
                        A.blk_first[b] = (int64_t)base;
                        A.blk_count[b] = m;
                        A.blk_next[b] = child_head;
                        child_head = (int64_t)b;
                        nchild += m;
                    }
                    atomicMax(A.maxgen, ugen + 1);
                    __threadfence();  // unit data before the ready flags
                    for (int i = 0; i < m; i++) st_relaxed(A.ready + base + i, 1u);
                    if (j0 == L.l) L.done = true;  // nothing left below the donated level
                    else L.r = j0 + 1;             // the walk now ends when it returns to depth j0+1
                    last_split = L.steps;
#ifdef TPGEN_KERNEL_DEBUG
                    d_don++;
#endif
                }
            }
        }

        // ---------------- unit completion
        if (CNT && L.active && L.done) {
            t_ext += ext;
            ext = 0;
            atomicAdd(A.qtd, 1ull);  // done += 1
            L.active = false;
            L.done = false;
        }
        if (!CNT && L.active && L.done) {
            A.cnt[C_PP][slot] = c_pp;
            A.cnt[C_VERT][slot] = c_vert;
            A.cnt[C_ITEMS][slot] = c_it;
            A.cnt[C_ITEMV][slot] = c_itv;
            A.cnt[C_HEADS][slot] = c_hd;
            A.cnt[C_HEADV][slot] = c_hdv;
            A.ext[slot] = ext;
            A.rcount[slot] = R.count;
            A.child_head[slot] = child_head;
            A.nchild[slot] = nchild;
            atomicAdd(A.qtd, 1ull);  // done += 1 (same word as the tail: termination needs no fence)
            L.active = false;
            L.done = false;
        }
    }
    if constexpr (CNT) {  // the queue's remainder, the head block's unused slots, then the totals
        if constexpr (HSH) {
            __syncwarp();
            if (lane < qn) {
                const uint64_t z = qS[lane];
                const uint64_t n = qL[lane];
                t_ha += mix64(z ^ (kSeedA + n));
                t_hb += mix64(z ^ (kSeedB + n));
            }
        }
        for (unsigned long long j = hblk + lane; j < hblk_end; j += 32)
            if (j < A.head_cap) A.heads[j].x = -1;
        uint64_t v[7] = {t_pp, t_vert, t_ext, t_ha, t_hb, 0, t_cross};
        bool ovf = false;  // prime-path totals >= 2^62 (or a wrapped sum): LIMIT_EXCEEDED, like the unit counters
#pragma unroll
        for (int q = 0; q < 7; q++) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t r = v[q] + __shfl_xor_sync(kFull, v[q], o);
                if (q < 2 && (r < v[q] || r >= (1ull << 62))) ovf = true;
                v[q] = r;
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < 7; q++) {
                if (!v[q] || q == 5) continue;
                const unsigned long long old = atomicAdd(A.cacc + q, (unsigned long long)v[q]);
                if (q < 2 && (old + v[q] < old || old + v[q] >= (1ull << 62))) ovf = true;
            }
        }
        if (__any_sync(kFull, ovf) && lane == 0) atomicOr(A.overflow, 1u);
    }
#ifdef TPGEN_KERNEL_DEBUG
    if (A.dbg) {
        if (lane == 0) {
            atomicAdd(A.dbg + 0, d_it);
            atomicAdd(A.dbg + 1, d_act);
        }
        atomicAdd(A.dbg + 2, d_don);
    }
#endif
}

}  // namespace tpg
