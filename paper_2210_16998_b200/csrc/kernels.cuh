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
    const int64_t *work;  // indices of the units to process
    const unsigned long long *n_work;
    unsigned long long *next;  // grab counter (zeroed before launch)
    // per-unit results
    uint64_t *cnt[C_NUM];
    uint64_t *ext;
    uint8_t *status;
    int64_t *rfirst;  // first record chunk of the unit
    int64_t *rcount;  // records of the unit
    void *stop;       // Unit<W>[n_units]: stop states of truncated units
    uint32_t budget;
    unsigned long long *n_trunc;
    unsigned long long *agg_tail_cnt, *agg_tail_len, *agg_pair_cnt, *agg_pair_len;
    unsigned int *overflow;  // bit 0: count overflow, bit 1: record pool exhausted
    // record pool
    uint64_t *chunks;
    unsigned long long *chunk_next;
    unsigned long long chunk_cap;
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
