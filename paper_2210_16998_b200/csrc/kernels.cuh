// kernels.cuh -- device code of libtpgen (sm_100a).
//
// Hot path: per start vertex s, depth-first
// enumeration of the simple paths inside SCC(s) (tail extension along CSR
// arcs, one 64-bit visited mask per path, cycle closure back to s -- PAPER.md
// Alg. 4 "ExtendPath" P:459-472, Ammann-Offutt generation P:865), fused with
// the maximality / segment classification (Def. 1, Defs. 6-9
// P:158-176 under DESIGN.md readings R8/R9) and the canonical writer.
//
// Design: one lane owns one work unit (a subtree of the
// per-start trie, or a terminal event) and walks it depth-first; the lane's
// path lives in shared memory ([level][lane] bytes), its visited set in a
// register.  Lanes refill from a global unit counter (warp-aggregated atomic).
// Emission is warp-cooperative: every emitting lane's path is written by the
// whole warp as one coalesced store stream.  Exact output offsets come from a
// count pass with the same step function, a scan, and the write pass.  Units
// that exceed a step budget in the count pass are split into a counted piece
// (replayed for exactly that many steps by the write pass) plus the untried
// sibling subtrees on its stack, which keeps lexicographic order and bounds
// every unit's work.
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

// A work unit: a trie node (K_NODE: the whole subtree under it), or one
// terminal event of a trie node (K_SELF: the node's own leaf/tail event,
// K_CLOSURE: the cycle path(+)s, K_OUT: the arc to an out-of-SCC successor).
struct __align__(16) Unit {
    uint64_t M;       // visited mask of path[0..depth] (local bits)
    int32_t scc;
    int32_t e;        // K_OUT: out-arc index
    uint32_t nsteps;  // write pass: replay exactly this many steps (0 = to completion)
    uint8_t depth;    // path = path[0..depth]
    uint8_t kind;
    uint8_t k, o;     // stop states only: cursor at level `depth`
    uint8_t rdepth;   // stop states only: root depth of the unit
    uint8_t pad[7];
    uint8_t path[64]; // local vertex ids
};
static_assert(sizeof(Unit) == 96, "Unit layout");

struct DevGraph {
    const Slot *slots;
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
    int32_t shard_lo, shard_hi;
};

struct DfsArgs {
    DevGraph G;
    const Unit *units;
    int64_t n_units;
    const int64_t *work;  // count pass: indices of the units to process
    const unsigned long long *n_work;
    unsigned long long *next;  // grab counter (zeroed before launch)
    // count pass
    uint64_t *cnt[C_NUM];
    uint64_t *ext;
    uint8_t *status;
    Unit *stop;
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

constexpr int kDfsThreads = 256;
constexpr int kDfsWarps = kDfsThreads / 32;
constexpr unsigned kFull = 0xffffffffu;

enum LanePhase : int { PH_IDLE = 0, PH_ROOT = 1, PH_RUN = 2, PH_DONE = 3, PH_EXHAUSTED = 4 };

struct Lane {
    uint64_t M, sbit, ps;
    int32_t vb, sgid, s, u, l, r, k, o, kind, e, phase;
    uint32_t steps, limit;
    bool seg, emit;
};

struct Event {
    int type, len, clo, e;
};

__device__ __forceinline__ Slot ld_slot(const Slot *p) {
    Slot s;
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2 *>(p));
    const int4 b = __ldg(reinterpret_cast<const int4 *>(p) + 1);
    s.sin = a.x;
    s.pin = a.y;
    s.gid = b.x;
    s.out_off = b.y;
    s.out_cnt = b.z;
    s.flags = b.w;
    return s;
}

// Own event of the node whose last vertex is w (called on creation).
//  PP mode (s not an SCC entry): internal acyclic prime path iff
//    succ(w) within {v2..vk} and pred(s) within {v1..v(k-1)}    (Def. 1 / Def. 9)
//  segment mode (s an SCC entry): tail segment iff succ(w) within the path  (R8)
__device__ __forceinline__ void node_event(const DevGraph &G, const Lane &L, int w, Event &ev) {
    const Slot sw = ld_slot(G.slots + L.vb + w);
    if (sw.flags & F_EXIT) return;
    if (L.seg) {
        if ((sw.sin & ~L.M) == 0) ev = Event{EV_TAIL, L.l + 1, 0, -1};
    } else if (L.emit && (sw.sin & ~(L.M & ~L.sbit)) == 0 && (L.ps & ~(L.M & ~(1ull << w))) == 0) {
        ev = Event{EV_PP, L.l + 1, 0, -1};
    }
}

// Arc to an out-of-SCC successor (out-arc e) from the current node.
//  segment mode: transit segment item (Def. 6, all entry->exit paths, R9)
//  PP mode: a head segment iff pred(s) lies on the path (R8) -> cross block
__device__ __forceinline__ void out_event(const Lane &L, int e, Event &ev) {
    if (L.seg) ev = Event{EV_TRANSIT, L.l + 1, 0, e};
    else if ((L.ps & ~L.M) == 0) ev = Event{EV_HEAD, L.l + 1, 0, e};
}

__device__ __forceinline__ int count_out_le(const DevGraph &G, const Slot &su, int w) {
    int o = 0;
    while (o < su.out_cnt && __ldg(G.out_pos + su.out_off + o) <= w) o++;
    return o;
}

// One step of the depth-first walk.  Children of a node are visited in
// ascending global id: in-SCC successors (local bits, ascending local id ==
// ascending global id), the closing arc back to s, and out-of-SCC successors
// (merged by their rank out_pos among the SCC members).
__device__ __forceinline__ void dfs_step(const DevGraph &G, Lane &L, uint8_t *mypath, Event &ev, uint64_t &ext) {
    if (L.phase == PH_ROOT) {
        switch (L.kind) {
            case K_NODE:
                L.phase = PH_RUN;
                if (L.l > 0 && L.emit) ext++;
                node_event(G, L, L.u, ev);
                return;
            case K_SELF:
                L.phase = PH_DONE;
                node_event(G, L, L.u, ev);
                return;
            case K_CLOSURE:
                L.phase = PH_DONE;
                if (L.emit) {
                    ext++;
                    ev = Event{EV_PP, L.l + 2, 1, -1};
                }
                return;
            default:
                L.phase = PH_DONE;
                out_event(L, L.e, ev);
                return;
        }
    }
    const Slot su = ld_slot(G.slots + L.vb + L.u);
    uint64_t cand = su.sin & (~L.M | L.sbit);
    cand = (L.k >= 64) ? 0ull : (cand >> L.k) << L.k;
    const int w = cand ? (__ffsll((long long)cand) - 1) : 64;
    if (L.o < su.out_cnt) {
        const int e = su.out_off + L.o;
        if (__ldg(G.out_pos + e) <= w) {
            L.o++;
            out_event(L, e, ev);
            return;
        }
    }
    if (w < 64) {
        L.k = w + 1;
        if (w == L.s) {  // cycle closure: always prime (Alg. 4 l.4-6)
            if (L.emit) {
                ext++;
                ev = Event{EV_PP, L.l + 2, 1, -1};
            }
            return;
        }
        L.l++;
        mypath[L.l * 32] = (uint8_t)w;
        L.M |= 1ull << w;
        L.u = w;
        L.k = 0;
        L.o = 0;
        if (L.emit) ext++;
        node_event(G, L, w, ev);
        return;
    }
    if (L.l == L.r) {
        L.phase = PH_DONE;
        return;
    }
    const int wold = L.u;
    L.M &= ~(1ull << wold);
    L.l--;
    L.u = mypath[L.l * 32];
    L.k = wold + 1;
    const Slot sp = ld_slot(G.slots + L.vb + L.u);
    L.o = count_out_le(G, sp, wold);
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

template <int PASS>
__global__ void __launch_bounds__(kDfsThreads, 4) dfs_kernel(DfsArgs A) {
    __shared__ uint8_t spath[kDfsWarps * 64 * 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *wpath = spath + wid * 64 * 32;  // [level][lane]
    uint8_t *mypath = wpath + lane;
    const DevGraph &G = A.G;
    const int64_t nwork = (PASS == PASS_COUNT) ? (int64_t)*A.n_work : A.n_units;

    Lane L;
    L.phase = PH_IDLE;
    int64_t uidx = -1;
    uint64_t c[C_NUM];
    uint64_t ext = 0;
    int64_t pair_row = 0;
    int32_t s_slot = 0;
#pragma unroll
    for (int i = 0; i < C_NUM; i++) c[i] = 0;

    while (true) {
        const unsigned idle = __ballot_sync(kFull, L.phase == PH_IDLE);
        if (idle) {
            const int leader = __ffs(idle) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(A.next, (unsigned long long)__popc(idle));
            base = __shfl_sync(kFull, base, leader);
            if (L.phase == PH_IDLE) {
                const int64_t my = (int64_t)base + __popc(idle & ((1u << lane) - 1));
                if (my < nwork) {
                    uidx = (PASS == PASS_COUNT) ? A.work[my] : my;
                    const Unit *U = A.units + uidx;
                    const uint4 h0 = *reinterpret_cast<const uint4 *>(U);
                    const uint4 h1 = *(reinterpret_cast<const uint4 *>(U) + 1);
                    L.M = ((uint64_t)h0.y << 32) | h0.x;
                    const int32_t scc = (int32_t)h0.z;
                    L.e = (int32_t)h0.w;
                    const uint32_t nsteps = h1.x;
                    const int depth = h1.y & 0xff;
                    L.kind = (h1.y >> 8) & 0xff;
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
                    L.sbit = 1ull << s;
                    L.vb = __ldg(G.scc_vbase + scc);
                    s_slot = L.vb + s;
                    const Slot ss = ld_slot(G.slots + s_slot);
                    L.ps = ss.pin;
                    L.seg = (ss.flags & F_ENTRY) != 0;
                    L.sgid = ss.gid;
                    L.emit = ss.gid >= G.shard_lo && ss.gid < G.shard_hi;
                    L.k = 0;
                    L.o = 0;
                    L.steps = 0;
                    L.phase = PH_ROOT;
                    if (PASS == PASS_COUNT) {
                        L.limit = A.budget;
#pragma unroll
                        for (int i = 0; i < C_NUM; i++) c[i] = 0;
                        ext = 0;
                        if (L.seg) {
                            const int32_t nout = __ldg(G.scc_nout + scc);
                            pair_row = __ldg(G.scc_pair_base + scc) +
                                       (int64_t)__ldg(G.slot_eidx + s_slot) * nout - __ldg(G.scc_out_base + scc);
                        }
                    } else {
                        L.limit = nsteps ? nsteps : 0xffffffffu;
#pragma unroll
                        for (int i = 0; i < C_NUM; i++) c[i] = A.off[i][uidx];
                    }
                } else {
                    L.phase = PH_EXHAUSTED;
                }
            }
        }
        const bool active = (L.phase == PH_ROOT || L.phase == PH_RUN);
        if (__ballot_sync(kFull, active) == 0) break;

        Event ev;
        ev.type = EV_NONE;
        if (active) {
            dfs_step(G, L, mypath, ev, ext);
            L.steps++;
        }

        if (PASS == PASS_COUNT) {
            if (ev.type == EV_PP) {
                c[C_PP] += 1;
                c[C_VERT] += (uint64_t)ev.len;
            } else if (ev.type == EV_HEAD) {
                const int32_t x = __ldg(G.out_gid + ev.e);
                const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                c[C_PP] = sat_add(c[C_PP], Wx, A.overflow);
                c[C_VERT] = sat_add(c[C_VERT], sat_add(sat_mul((uint64_t)ev.len, Wx, A.overflow), Vx, A.overflow),
                                    A.overflow);
                c[C_HEADS] += 1;
                c[C_HEADV] += (uint64_t)ev.len;
            } else if (ev.type == EV_TAIL) {
                c[C_ITEMS] += 1;
                c[C_ITEMV] += (uint64_t)ev.len;
                atomicAdd(A.agg_tail_cnt + s_slot, 1ull);
                atomicAdd(A.agg_tail_len + s_slot, (unsigned long long)ev.len);
            } else if (ev.type == EV_TRANSIT) {
                c[C_ITEMS] += 1;
                c[C_ITEMV] += (uint64_t)ev.len;
                atomicAdd(A.agg_pair_cnt + pair_row + ev.e, 1ull);
                atomicAdd(A.agg_pair_len + pair_row + ev.e, (unsigned long long)ev.len);
            }
        } else {
            // ---- warp-cooperative emission ----
            int32_t *dst = nullptr;
            if (ev.type == EV_PP) {
                dst = A.out_vert + c[C_VERT];
                A.out_off[c[C_PP]] = (int64_t)c[C_VERT];
                c[C_PP] += 1;
                c[C_VERT] += (uint64_t)ev.len;
            } else if (ev.type == EV_HEAD) {
                const int32_t x = __ldg(G.out_gid + ev.e);
                dst = A.head_pool + c[C_HEADV];
                HeadRec h;
                h.pp_off = c[C_PP];
                h.v_off = c[C_VERT];
                h.hv_off = c[C_HEADV];
                h.len = ev.len;
                h.x = x;
                A.heads[c[C_HEADS]] = h;
                const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                c[C_PP] += Wx;
                c[C_VERT] += (uint64_t)ev.len * Wx + Vx;
                c[C_HEADS] += 1;
                c[C_HEADV] += (uint64_t)ev.len;
            } else if (ev.type == EV_TAIL || ev.type == EV_TRANSIT) {
                dst = A.item_pool + c[C_ITEMV];
                ItemRec it;
                it.pool_off = (int64_t)c[C_ITEMV];
                it.len = ev.len;
                it.y = (ev.type == EV_TRANSIT) ? __ldg(G.out_gid + ev.e) : -1;
                it.ent = L.sgid;
                it.pad = 0;
                A.items[c[C_ITEMS]] = it;
                c[C_ITEMS] += 1;
                c[C_ITEMV] += (uint64_t)ev.len;
            }
            unsigned em = __ballot_sync(kFull, ev.type != EV_NONE);
            while (em) {
                const int src = __ffs(em) - 1;
                em &= em - 1;
                int32_t *d = reinterpret_cast<int32_t *>(__shfl_sync(kFull, (unsigned long long)dst, src));
                const int len = __shfl_sync(kFull, ev.len, src);
                const int clo = __shfl_sync(kFull, ev.clo, src);
                const int vb = __shfl_sync(kFull, L.vb, src);
                const uint8_t *sp = wpath + src;
                const int plen = len - clo;
                for (int j = lane; j < len; j += 32) {
                    const int loc = sp[(j < plen ? j : 0) * 32];
                    d[j] = __ldg(G.slot_gid + vb + loc);
                }
            }
        }

        if (active) {
            if (L.phase == PH_DONE || L.steps >= L.limit) {
                if (PASS == PASS_COUNT) {
                    const bool trunc = (L.phase != PH_DONE);
#pragma unroll
                    for (int i = 0; i < C_NUM; i++) A.cnt[i][uidx] = c[i];
                    A.ext[uidx] = ext;
                    A.status[uidx] = trunc ? ST_TRUNC : ST_DONE;
                    if (trunc) {
                        Unit *S = A.stop + uidx;
                        uint4 h0, h1;
                        h0.x = (uint32_t)L.M;
                        h0.y = (uint32_t)(L.M >> 32);
                        h0.z = (uint32_t)A.units[uidx].scc;
                        h0.w = 0;
                        h1.x = L.steps;
                        h1.y = (uint32_t)L.l | ((uint32_t)K_NODE << 8) | ((uint32_t)L.k << 16) | ((uint32_t)L.o << 24);
                        h1.z = (uint32_t)L.r;
                        h1.w = 0;
                        reinterpret_cast<uint4 *>(S)[0] = h0;
                        reinterpret_cast<uint4 *>(S)[1] = h1;
                        for (int j = 0; j <= L.l; j++) S->path[j] = mypath[j * 32];
                        atomicAdd(A.n_trunc, 1ull);
                    }
                }
                L.phase = PH_IDLE;
            }
        }
    }
}

// ------------------------------------------------------------- refinement
// Remainder of a truncated unit: the untried events of every node on its stop
// stack, deepest level first (lexicographic order of the rest of the walk).
template <bool WRITE>
__device__ int remainder_events(const DevGraph &G, const Unit &S, Unit *out) {
    const int vb = __ldg(G.scc_vbase + S.scc);
    const int s = S.path[0];
    const uint64_t sbit = 1ull << s;
    const Slot ss = ld_slot(G.slots + vb + s);
    const bool seg = (ss.flags & F_ENTRY) != 0;
    const uint64_t ps = ss.pin;
    uint64_t M = S.M;
    int n = 0;
    for (int j = S.depth; j >= (int)S.rdepth; j--) {
        const int u = S.path[j];
        const Slot su = ld_slot(G.slots + vb + u);
        int k, o;
        if (j == S.depth) {
            k = S.k;
            o = S.o;
        } else {
            const int wc = S.path[j + 1];
            M &= ~(1ull << wc);
            k = wc + 1;
            o = count_out_le(G, su, wc);
        }
        uint64_t cand = su.sin & (~M | sbit);
        cand = (k >= 64) ? 0ull : (cand >> k) << k;
        while (true) {
            const int w = cand ? (__ffsll((long long)cand) - 1) : 64;
            if (o < su.out_cnt && __ldg(G.out_pos + su.out_off + o) <= w) {
                const int e = su.out_off + o;
                o++;
                if (seg || (ps & ~M) == 0) {
                    if (WRITE) {
                        Unit &U = out[n];
                        U = S;
                        U.M = M;
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
            if (w == 64) break;
            cand &= cand - 1;
            if (WRITE) {
                Unit &U = out[n];
                U = S;
                U.nsteps = 0;
                U.k = U.o = U.rdepth = 0;
                U.e = -1;
                if (w == s) {
                    U.M = M;
                    U.depth = (uint8_t)j;
                    U.kind = K_CLOSURE;
                } else {
                    U.M = M | (1ull << w);
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
