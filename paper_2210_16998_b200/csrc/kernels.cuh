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
// to an out-of-SCC successor).  Stop states of truncated units use the same
// record (k, o, rdepth).
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
    int32_t shard_lo, shard_hi;
};

struct DfsArgs {
    DevGraph G;
    const void *units;  // Unit<W>[n_units]
    int64_t n_units;
    const int64_t *work;  // count pass: indices of the units to process
    const unsigned long long *n_work;
    unsigned long long *next;  // grab counter (zeroed before launch)
    // count pass
    uint64_t *cnt[C_NUM];
    uint64_t *ext;
    uint8_t *status;
    void *stop;  // Unit<W>[n_units]
    uint32_t budget;
    unsigned long long *n_trunc;
    unsigned long long *agg_tail_cnt, *agg_tail_len, *agg_pair_cnt, *agg_pair_len;
    unsigned int *overflow;
    // write pass
    const uint64_t *off[C_NUM];
    int64_t *out_off;
    int32_t *out_vert;
    HeadRec *heads;
    int32_t *head_pool;
    ItemRec *items;
    int32_t *item_pool;
};

// 256 threads per block for W <= 2; 128 for W = 4 (the per-lane path needs 64*W bytes of smem)
template <int W>
struct DfsCfg {
    static constexpr int threads = (W <= 2) ? 256 : 128;
    static constexpr int warps = threads / 32;
    static constexpr int min_blocks = (W == 1) ? 4 : ((W == 2) ? 2 : 3);
};
constexpr unsigned kFull = 0xffffffffu;

template <int W>
struct Lane {
    Mask<W> M, sbit, ps, sin;  // visited set, bit of s, pred(s) in SCC, succ(u) in SCC
    int32_t vb, gadd, sgid, s, u, l, r, k, o, ooff, ocnt, flags;
    uint32_t steps, limit;
    bool active, done, seg, emit;
};

// Event codes: type in bits 0-2, closure flag bit 3, path length in bits 8+.
constexpr int EV_CLO = 8;
__device__ __forceinline__ int ev_type(int ev) { return ev & 7; }
__device__ __forceinline__ int ev_len(int ev) { return ev >> 8; }

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

// Own event of a node whose last vertex is w (evaluated when the node is created).
//  PP mode (s not an SCC entry): internal acyclic prime path iff
//    succ(w) within {v2..vk} and pred(s) within {v1..v(k-1)}    (Def. 1 / Def. 9)
//  segment mode (s an SCC entry): tail segment iff succ(w) within the path  (R8)
template <int W>
__device__ __forceinline__ int node_event(const Lane<W> &L, int w) {
    if (L.flags & F_EXIT) return 0;
    const int len = (L.l + 1) << 8;
    if (L.seg) return msubset(L.sin, L.M) ? (EV_TAIL | len) : 0;
    if (!L.emit) return 0;
    Mask<W> inner_t = L.M, inner_h = L.M;
#pragma unroll
    for (int i = 0; i < W; i++) inner_t.w[i] &= ~L.sbit.w[i];
    mclr(inner_h, w);
    return (msubset(L.sin, inner_t) && msubset(L.ps, inner_h)) ? (EV_PP | len) : 0;
}

// Arc to an out-of-SCC successor from the current node.
//  segment mode: transit segment item (Def. 6 -- all entry->exit paths, R9)
//  PP mode: a head segment iff pred(s) lies on the path (R8) -> cross block
template <int W>
__device__ __forceinline__ int out_event(const Lane<W> &L) {
    const int len = (L.l + 1) << 8;
    if (L.seg) return EV_TRANSIT | len;
    return msubset(L.ps, L.M) ? (EV_HEAD | len) : 0;
}

__device__ __forceinline__ int count_out_le(const DevGraph &G, int out_off, int out_cnt, int w) {
    int o = 0;
    while (o < out_cnt && __ldg(G.out_pos + out_off + o) <= w) o++;
    return o;
}

template <int W>
__device__ __forceinline__ void load_slot(const DevGraph &G, Lane<W> &L, int u) {
    const Slot<W> *sp = slot_ptr<W>(G, L.vb + u);
    L.sin = ld_sin(sp);
    const int4 m = ld_meta(sp);
    L.ooff = m.y;
    L.ocnt = m.z;
    L.flags = m.w;
}

// One step of the depth-first walk (branch-light: push, closure and pop share
// one predicated update).  Children of a node are visited in ascending global
// id: in-SCC successors (local bits; ascending local id == ascending global
// id), the closing arc back to s, and out-of-SCC successors (merged by their
// rank out_pos among the SCC members).  Returns the event of this step.
template <int W>
__device__ __forceinline__ int dfs_step(const DevGraph &G, Lane<W> &L, uint8_t *mypath, int &e_out, uint64_t &ext) {
    const int w = mnext(L.sin, L.M, L.sbit, L.k);
    if (L.o < L.ocnt) {  // exit vertex with out-of-SCC arcs still to visit
        const int e = L.ooff + L.o;
        if (__ldg(G.out_pos + e) <= w) {
            L.o++;
            e_out = e;
            return out_event(L);
        }
    }
    const bool has = w < 64 * W;
    if (!has && L.l == L.r) {
        L.done = true;
        return 0;
    }
    const bool clo = has && (w == L.s);
    const bool push = has && !clo;
    const int wold = L.u;
    const int parent = mypath[(L.l > 0 ? L.l - 1 : 0) * 32];
    if (push) mypath[(L.l + 1) * 32] = (uint8_t)w;
    if (push) mset(L.M, w);
    if (!has) mclr(L.M, wold);
    L.k = push ? 0 : (has ? w + 1 : wold + 1);
    L.l += push ? 1 : (has ? 0 : -1);
    if (clo) {  // cycle closure: always prime (Alg. 4 l.4-6)
        if (L.emit) {
            ext++;
            return EV_PP | EV_CLO | ((L.l + 2) << 8);
        }
        return 0;
    }
    L.u = push ? w : parent;
    load_slot(G, L, L.u);
    if (push) {
        L.o = 0;
        if (L.emit) ext++;
        return node_event(L, w);
    }
    L.o = count_out_le(G, L.ooff, L.ocnt, wold);
    return 0;
}

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

template <int W, int PASS>
__global__ void __launch_bounds__(DfsCfg<W>::threads, DfsCfg<W>::min_blocks) dfs_kernel(DfsArgs A) {
    __shared__ uint8_t spath[DfsCfg<W>::warps * 64 * W * 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *wpath = spath + wid * 64 * W * 32;  // [level][lane]
    uint8_t *mypath = wpath + lane;
    const DevGraph &G = A.G;
    const Unit<W> *units = reinterpret_cast<const Unit<W> *>(A.units);
    const int64_t nwork = (PASS == PASS_COUNT) ? (int64_t)*A.n_work : A.n_units;

    Lane<W> L;
    L.active = false;
    L.done = false;
    bool exhausted = false;
    int64_t uidx = -1;
    int32_t uscc = 0;
    uint64_t c[C_NUM];
    uint64_t ext = 0;
    int64_t pair_row = 0;
    int32_t s_slot = 0;
#pragma unroll
    for (int i = 0; i < C_NUM; i++) c[i] = 0;

    while (true) {
        int ev = 0, e = -1;
        // ---------------- refill idle lanes (warp-aggregated grab)
        const unsigned idle = __ballot_sync(kFull, !L.active && !exhausted);
        if (idle) {
            const int leader = __ffs(idle) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(A.next, (unsigned long long)__popc(idle));
            base = __shfl_sync(kFull, base, leader);
            if (!L.active && !exhausted) {
                const int64_t my = (int64_t)base + __popc(idle & ((1u << lane) - 1));
                if (my >= nwork) {
                    exhausted = true;
                } else {
                    uidx = (PASS == PASS_COUNT) ? A.work[my] : my;
                    const Unit<W> *U = units + uidx;
                    const int4 h = *reinterpret_cast<const int4 *>(&U->scc);  // scc, e, nsteps, depth|kind|k|o
#pragma unroll
                    for (int i = 0; i < W; i++) L.M.w[i] = U->M[i];
                    uscc = h.x;
                    const int kind = (h.w >> 8) & 0xff;
                    const int depth = h.w & 0xff;
                    L.l = L.r = depth;
                    const uint4 *p4 = reinterpret_cast<const uint4 *>(U->path);
                    int s = 0, u = 0;
#pragma unroll 1
                    for (int q = 0; q * 16 <= depth; q++) {
                        const uint4 v = p4[q];
                        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int b = 0; b < 16; b++) {
                            const int j = q * 16 + b;
                            if (j <= depth) {
                                const uint8_t byte = (uint8_t)(wv[b >> 2] >> ((b & 3) * 8));
                                mypath[j * 32] = byte;
                                if (j == 0) s = byte;
                                if (j == depth) u = byte;
                            }
                        }
                    }
                    L.s = s;
                    L.u = u;
                    L.sbit = mbit<W>(s);
                    L.vb = __ldg(G.scc_vbase + uscc);
                    L.gadd = __ldg(G.scc_gbase + uscc);
                    s_slot = L.vb + s;
                    const Slot<W> *ss = slot_ptr<W>(G, s_slot);
                    L.ps = ld_pin(ss);
                    const int4 sm = ld_meta(ss);
                    L.seg = (sm.w & F_ENTRY) != 0;
                    L.sgid = sm.x;
                    L.emit = sm.x >= G.shard_lo && sm.x < G.shard_hi;
                    L.k = 0;
                    L.o = 0;
                    L.steps = 0;
                    L.done = false;
                    L.active = true;
                    if (PASS == PASS_COUNT) {
                        L.limit = A.budget;
#pragma unroll
                        for (int i = 0; i < C_NUM; i++) c[i] = 0;
                        ext = 0;
                        if (L.seg) {
                            const int32_t nout = __ldg(G.scc_nout + uscc);
                            pair_row = __ldg(G.scc_pair_base + uscc) +
                                       (int64_t)__ldg(G.slot_eidx + s_slot) * nout - __ldg(G.scc_out_base + uscc);
                        }
                    } else {
                        const uint32_t nsteps = (uint32_t)h.z;
                        L.limit = nsteps ? nsteps : 0xffffffffu;
#pragma unroll
                        for (int i = 0; i < C_NUM; i++) c[i] = A.off[i][uidx];
                    }
                    // the unit's root event (no step is counted for it)
                    if (kind == K_NODE) {
                        load_slot(G, L, u);
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
                }
            }
        }
        if (__ballot_sync(kFull, L.active) == 0) break;

        // ---------------- steps until some lane has an event, finishes or hits its budget
        if (__ballot_sync(kFull, ev != 0 || (L.active && L.done)) == 0) {
            while (true) {
                if (L.active) {
                    ev = dfs_step<W>(G, L, mypath, e, ext);
                    L.steps++;
                }
                if (__ballot_sync(kFull, L.active && (ev != 0 || L.done || L.steps >= L.limit))) break;
            }
        }

        // ---------------- events
        if (PASS == PASS_COUNT) {
            if (ev) {
                const int ty = ev_type(ev);
                const uint64_t len = (uint64_t)ev_len(ev);
                if (ty == EV_PP) {
                    c[C_PP] += 1;
                    c[C_VERT] += len;
                } else if (ty == EV_HEAD) {
                    const int32_t x = __ldg(G.out_gid + e);
                    const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                    c[C_PP] = sat_add(c[C_PP], Wx, A.overflow);
                    c[C_VERT] = sat_add(c[C_VERT], sat_add(sat_mul(len, Wx, A.overflow), Vx, A.overflow),
                                        A.overflow);
                    c[C_HEADS] += 1;
                    c[C_HEADV] += len;
                } else if (ty == EV_TAIL) {
                    c[C_ITEMS] += 1;
                    c[C_ITEMV] += len;
                    atomicAdd(A.agg_tail_cnt + s_slot, 1ull);
                    atomicAdd(A.agg_tail_len + s_slot, (unsigned long long)len);
                } else {  // EV_TRANSIT
                    c[C_ITEMS] += 1;
                    c[C_ITEMV] += len;
                    atomicAdd(A.agg_pair_cnt + pair_row + e, 1ull);
                    atomicAdd(A.agg_pair_len + pair_row + e, (unsigned long long)len);
                }
            }
        } else {
            int32_t *dst = nullptr;
            if (ev) {
                const int ty = ev_type(ev);
                const uint64_t len = (uint64_t)ev_len(ev);
                if (ty == EV_PP) {
                    dst = A.out_vert + c[C_VERT];
                    A.out_off[c[C_PP]] = (int64_t)c[C_VERT];
                    c[C_PP] += 1;
                    c[C_VERT] += len;
                } else if (ty == EV_HEAD) {
                    const int32_t x = __ldg(G.out_gid + e);
                    dst = A.head_pool + c[C_HEADV];
                    HeadRec hr;
                    hr.pp_off = c[C_PP];
                    hr.v_off = c[C_VERT];
                    hr.hv_off = c[C_HEADV];
                    hr.len = (int32_t)len;
                    hr.x = x;
                    A.heads[c[C_HEADS]] = hr;
                    const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                    c[C_PP] += Wx;
                    c[C_VERT] += len * Wx + Vx;
                    c[C_HEADS] += 1;
                    c[C_HEADV] += len;
                } else {  // EV_TAIL / EV_TRANSIT
                    dst = A.item_pool + c[C_ITEMV];
                    ItemRec it;
                    it.pool_off = (int64_t)c[C_ITEMV];
                    it.len = (int32_t)len;
                    it.y = (ty == EV_TRANSIT) ? __ldg(G.out_gid + e) : -1;
                    it.ent = L.sgid;
                    it.pad = 0;
                    A.items[c[C_ITEMS]] = it;
                    c[C_ITEMS] += 1;
                    c[C_ITEMV] += len;
                }
            }
            // warp-cooperative copy: each emitting lane's path is written by the whole warp
            unsigned em = __ballot_sync(kFull, ev != 0);
            while (em) {
                const int src = __ffs(em) - 1;
                em &= em - 1;
                int32_t *d = reinterpret_cast<int32_t *>(__shfl_sync(kFull, (unsigned long long)dst, src));
                const int evs = __shfl_sync(kFull, ev, src);
                const int vb = __shfl_sync(kFull, L.vb, src);
                const int ga = __shfl_sync(kFull, L.gadd, src);
                const uint8_t *sp = wpath + src;
                const int len = ev_len(evs);
                const int plen = len - ((evs & EV_CLO) ? 1 : 0);
                for (int j = lane; j < len; j += 32) {
                    const int loc = sp[(j < plen ? j : 0) * 32];
                    d[j] = (ga >= 0) ? ga + loc : __ldg(G.slot_gid + vb + loc);
                }
            }
        }

        // ---------------- unit completion / budget
        if (L.active && (L.done || L.steps >= L.limit)) {
            if (PASS == PASS_COUNT) {
                const bool trunc = !L.done;
#pragma unroll
                for (int i = 0; i < C_NUM; i++) A.cnt[i][uidx] = c[i];
                A.ext[uidx] = ext;
                A.status[uidx] = trunc ? ST_TRUNC : ST_DONE;
                if (trunc) {
                    Unit<W> *S = reinterpret_cast<Unit<W> *>(A.stop) + uidx;
#pragma unroll
                    for (int i = 0; i < W; i++) S->M[i] = L.M.w[i];
                    int4 h;
                    h.x = uscc;
                    h.y = -1;
                    h.z = (int)L.steps;
                    h.w = L.l | ((int)K_NODE << 8) | (L.k << 16) | (L.o << 24);
                    *reinterpret_cast<int4 *>(&S->scc) = h;
                    S->rdepth = (uint8_t)L.r;
                    for (int j = 0; j <= L.l; j++) S->path[j] = mypath[j * 32];
                    atomicAdd(A.n_trunc, 1ull);
                }
            }
            L.active = false;
            L.done = false;
        }
    }
}

// ------------------------------------------------------------- refinement
// Remainder of a truncated unit: the untried events of every node on its stop
// stack, deepest level first (lexicographic order of the rest of the walk).
template <int W, bool WRITE>
__device__ int remainder_events(const DevGraph &G, const Unit<W> &S, Unit<W> *out) {
    const int vb = __ldg(G.scc_vbase + S.scc);
    const int s = S.path[0];
    const Mask<W> sbit = mbit<W>(s);
    const Slot<W> *ss = slot_ptr<W>(G, vb + s);
    const bool seg = (__ldg(&ss->flags) & F_ENTRY) != 0;
    const Mask<W> ps = ld_pin(ss);
    Mask<W> M;
#pragma unroll
    for (int i = 0; i < W; i++) M.w[i] = S.M[i];
    int n = 0;
    for (int j = S.depth; j >= (int)S.rdepth; j--) {
        const int u = S.path[j];
        const Slot<W> *su = slot_ptr<W>(G, vb + u);
        const int4 meta = ld_meta(su);
        const Mask<W> sin = ld_sin(su);
        int k, o;
        if (j == S.depth) {
            k = S.k;
            o = S.o;
        } else {
            const int wc = S.path[j + 1];
            mclr(M, wc);
            k = wc + 1;
            o = count_out_le(G, meta.y, meta.z, wc);
        }
        while (true) {
            const int w = mnext(sin, M, sbit, k);
            if (o < meta.z && __ldg(G.out_pos + meta.y + o) <= w) {
                const int e = meta.y + o;
                o++;
                if (seg || msubset(ps, M)) {
                    if (WRITE) {
                        Unit<W> &U = out[n];
                        U = S;
#pragma unroll
                        for (int i = 0; i < W; i++) U.M[i] = M.w[i];
                        U.e = e;
                        U.nsteps = 0;
                        U.depth = (uint8_t)j;
                        U.kind = K_OUT;
                        U.k = U.o = U.rdepth = 0;
                    }
                    n++;
                }
                continue;
            }
            if (w >= 64 * W) break;
            k = w + 1;
            if (WRITE) {
                Unit<W> &U = out[n];
                U = S;
                U.nsteps = 0;
                U.k = U.o = U.rdepth = 0;
                U.e = -1;
#pragma unroll
                for (int i = 0; i < W; i++) U.M[i] = M.w[i];
                if (w == s) {
                    U.depth = (uint8_t)j;
                    U.kind = K_CLOSURE;
                } else {
                    U.M[w >> 6] |= 1ull << (w & 63);
                    U.depth = (uint8_t)(j + 1);
                    U.path[j + 1] = (uint8_t)w;
                    U.kind = K_NODE;
                }
            }
            n++;
        }
    }
    return n;
}

}  // namespace tpg
