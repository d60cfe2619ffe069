// count.cuh -- the count-mode enumerator (COUNT_HASH calls, prime-path phase) of libtpgen.
//
// Same walk as dfs.cuh (per start vertex s, depth-first over the simple paths inside
// SCC(s); Alg. 4 "ExtendPath"; the maximality test of Def. 1, P:127-130,
// in its operational form R3), but without the path-delta records: in COUNT_HASH mode
// the order of the walk is irrelevant (every output is a sum), so a step is written as
// ONE straight-line, predicated instruction stream that every lane of a warp executes
// with its own data -- the divergent push / pop / closure / record regions of the
// record-writing step (each executed by the whole warp whenever any lane needs it)
// are gone.  Per pass every lane makes exactly one move:
//   * a pop, if its current node has no untried child left (at the unit's root: the
//     unit is finished), or
//   * the take of the lowest untried child w of its current node (one extension): w = s
//     is a cycle closure, a prime path; otherwise the child's own untried
//     children c_w = succ(w) & (~(M + w) | {s}) are computed at once and
//       c_w == 0, pred(s) within M, w not an SCC exit  -> internal prime path (R3);
//       w an exit, pred(s) within M + w                 -> head segment(s) (R8);
//       c_w != 0                                        -> the walk descends into w
//     so a leaf child never costs a push and a pop.
// Both moves are the same operations on the moved vertex v (the popped one or the
// child): its digest term mix(v) * (2 pos + 1) (R20) added or subtracted, its visited
// bit toggled, the depth moved by one.
// The digest sum S of the current path (R20: sum of mix(v) * (2 pos + 1)) is kept in a
// register; a prime path found in a pass is queued per warp (S, length) and the warp
// hashes 32 queued paths at once.  Head segments (rare: exit vertices only) are written
// as HeadS records into the warp's block of head slots, for stitch_hash_s_kernel.
//
// Masks: 32-bit (SCCs <= 32 vertices) keep the untried children of every level on a
// shared-memory stack (rem[level][lane]); 64-bit recompute them on a pop from the
// parent's successor set (children are taken in ascending id, so the untried ones are
// the successors above the child just finished).
//
// Work distribution is the persistent work queue of dfs_kernel (claims, ready flags,
// donation of the shallowest untried children when the queue runs low), with units
// that carry no per-unit results.
#pragma once

#include "dfs.cuh"

namespace tpg {

#ifndef CNT_MINB_PP64H
#define CNT_MINB_PP64H 4  // resident blocks per SM of the 64-bit hashing prime-path / test-path kernels (64
                          // registers: measured 151.5 -> 142.6 ms on config 5; the other variants lose at 4)
#endif
#ifndef CNT_POP2
#define CNT_POP2 0  // 1: a pop whose parent has no untried child left pops the parent in the same pass
#endif
#ifndef CNT_QUEUE
#define CNT_QUEUE 1  // 1: prime paths into a per-warp queue (ballot), hashed 32 at a time; 0: per-lane rings
#endif
#ifndef CNT_D2_POPS
#define CNT_D2_POPS 2  // D2: 0 -- one move per pass (a pop or a take); k > 0 -- up to k pops, then a take, per pass
                       // (config 5 cnt_kernel, one box: k = 0 / 1 / 2 / 3 / 4 -> 123.8 / 118.1 / 112.0 / 118.7 / 130.1 ms)
#endif
#ifndef CNT_D2_SELFREE
#define CNT_D2_SELFREE 0  // D2 pops: predicates folded into the multiplier / shift instead of 64-bit selects
#endif
#ifndef CNT_PASSES
#define CNT_PASSES 32  // passes of the step between two rounds of queue housekeeping
#endif

template <class T>
struct CntLane {
    T M, rem, sbit, ps, exm;  // visited set, untried children of the current node, bit of s, pred(s), SCC exits
    int32_t l, r, s, vb;      // depth, unit root depth, start vertex (local), slot base of the SCC
    uint64_t S;               // digest sum of path[0..l]
    uint64_t B;               // segment phase: sum of mix(v) over path[0..l] (an item's offset slope)
    uint32_t cur;             // D2: the current node's untried children as bytes (byte 0 taken next; 0xff: none)
    bool active, done, emit;  // emit (segment phase): s lies in the call's start range
};

// Event kinds of a lane's ring (tag bits 29-31; bits 8-28 the slot of the path's last
// vertex, bits 0-7 the path length): a prime path, a head segment (prime-path phase), a
// tail segment or the transit segments over an exit vertex's out-of-SCC arcs (segment phase).
enum CntEv : uint32_t { EK_PP = 0, EK_HEAD = 1, EK_TAIL = 2, EK_TRANSIT = 3 };

// Hot-loop table per slot: in-SCC successor bits and the digest value mix64(gid) (R20),
// staged in shared memory as {sin, mix} pairs (TS) or read from the global copies.
template <class T, bool TS>
struct CntTab {
    const Slot<1> *g;
    const uint64_t *gm;
    uint32_t sb;  // TS: shared-window address of the {sin (8 B), mix (8 B)} table
    __device__ __forceinline__ T sin(int i) const {
        if (TS) {
            if (sizeof(T) == 4) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sb + (uint32_t)i * 16u) : "memory");
                return (T)v;
            }
            uint64_t v;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sb + (uint32_t)i * 16u) : "memory");
            return (T)v;
        }
        return (T)__ldg(&g[i].sin[0]);
    }
    __device__ __forceinline__ T pin(int i) const { return (T)__ldg(&g[i].pin[0]); }
    __device__ __forceinline__ uint64_t mix(int i) const {
        if (TS) {
            uint64_t v;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(sb + (uint32_t)i * 16u + 8u) : "memory");
            return v;
        }
        return __ldg(gm + i);
    }
};

__device__ __forceinline__ int ffs_t(uint32_t x) { return __ffs(x) - 1; }
__device__ __forceinline__ int ffs_t(uint64_t x) { return __ffsll((long long)x) - 1; }
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// D2: a set of at most 2 children as bytes (0xff: none) -> a mask
template <class T>
__device__ __forceinline__ T d2_mask(uint32_t c) {
    const uint32_t b0 = c & 0xffu, b1 = (c >> 8) & 0xffu;
    return (b0 != 0xffu ? (T)1 << b0 : (T)0) | (b1 != 0xffu ? (T)1 << b1 : (T)0);
}
// ... and back (ascending)
template <class T>
__device__ __forceinline__ uint32_t d2_bytes(T m) {
    const uint32_t b0 = m ? (uint32_t)ffs_t(m) : 0xffu;
    const T m1 = m & (m - 1);
    const uint32_t b1 = m1 ? (uint32_t)ffs_t(m1) : 0xffu;
    return b0 | (b1 << 8);
}
// m * w mod 2^64 for a 32-bit w: one wide multiply of the low word, one of the high word
#ifndef CNT_MUL_PTX
#define CNT_MUL_PTX 1  // 1 (measured: config 5 cnt_kernel 111.95 -> 110.87 ms): the product as two PTX multiplies (mul.wide.u32 + mad.lo.u32 into the high word)
#endif
__device__ __forceinline__ uint64_t mul64x32(uint64_t m, uint32_t w) {
#if CNT_MUL_PTX
    uint32_t lo, hi;
    asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %4;\n\tmov.b64 {%0, %1}, t;\n\tmad.lo.u32 %1, %3, %4, %1;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"((uint32_t)m), "r"((uint32_t)(m >> 32)), "r"(w));
    return ((uint64_t)hi << 32) | lo;
#else
    const uint64_t lo = (uint64_t)(uint32_t)m * w;
    return lo + ((uint64_t)((uint32_t)(m >> 32) * w) << 32);
#endif
}

// NEXT #2 (not in the paper): may the subtree under the path node w (path mask Mw,
// w included; untried children cw) hold an event?  Every event below w ends at a vertex x
// reachable from w in C \ path: a closure needs x in pred(s), an internal prime path or a head
// segment needs pred(s) on the path (Def. 1 / R3, Def. 6).  No when w is not in pred(s), some of
// pred(s) is off the path, and none of that part is reachable from w in C \ path (bitset BFS).
// CNT_PRUNE_MAXD: the deepest path position tested (a subtree a shallow test did not cut is still
// cut where a deeper test fires; deep subtrees are small, the test's cost is not).
#ifndef CNT_PRUNE_MAXD
#define CNT_PRUNE_MAXD 64
#endif
template <class T, class Tab>
__device__ __forceinline__ bool prune_keep(const Tab &tab, int vb, T ps, int w, T Mw, T cw) {
    if ((ps >> w) & 1) return true;
    const T need = ps & ~Mw;
    if (need == 0) return true;
    T R = Mw | cw, F = cw;
    bool hit = (cw & need) != 0;
    while (!hit && F != 0) {
        T N = 0;
        for (T f = F; f != 0; f &= f - 1) N |= tab.sin(vb + ffs_t(f));
        N &= ~R;
        hit = (N & need) != 0;
        R |= N;
        F = N;
    }
    return hit;
}

// 2 x + 1, the digest weight of path position x (R20), as one multiply-add (the FMA pipe; the
// compiler's shift-or form takes an ALU-pipe LOP3, the pipe the D2 pass is bound on)
#ifndef CNT_ODD_MAD
#define CNT_ODD_MAD 1
#endif
// CNT_OPAQUE_K: the D2 pass's constant multipliers (2 for the weight, 16 for the table stride)
// come from blockDim.x (= 256, unknown to ptxas), so the products stay IMADs (FMA pipe) instead
// of being strength-reduced to LEA / shift-or (ALU pipe)
#ifndef CNT_PASS_UNROLL
#define CNT_PASS_UNROLL 2  // passes per iteration of the pass loop (config 5 cnt_kernel 103.46 -> 102.78 ms at 2)
#endif
constexpr int kCntPassUnroll = CNT_PASS_UNROLL;
#ifndef CNT_POP_PRED
#define CNT_POP_PRED 0  // D2: the pops' shared loads predicated on the pop (see the pass)
#endif
#ifndef CNT_ACT_REG
#define CNT_ACT_REG 1  // (config 5 cnt_kernel 102.79 -> 101.07 ms) D2: the lane's stepping flag kept across the passes, L.done written after them
#endif
#ifndef CNT_BIT_TAB_TAKE
#define CNT_BIT_TAB_TAKE 1  // the take's bit from the table too (0: two shifts on the ALU pipe instead)
#endif
#ifndef CNT_BIT_TAB
#define CNT_BIT_TAB 1  // D2: one-bit masks from a 512-byte shared table (no SHF / SEL on the ALU pipe)
#endif
#ifndef CNT_OPAQUE_K
#define CNT_OPAQUE_K 1
#endif
__device__ __forceinline__ uint32_t odd2(uint32_t x, uint32_t k2 = 2u) {
#if CNT_ODD_MAD
    uint32_t r;
    if (CNT_OPAQUE_K) asm("mad.lo.u32 %0, %1, %2, 1;" : "=r"(r) : "r"(x), "r"(k2));
    else asm("mad.lo.u32 %0, %1, 2, 1;" : "=r"(r) : "r"(x));
    return r;
#else
    return 2u * x + 1u;
#endif
}
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

template <class T>
struct CntCfg {
    static constexpr bool RS = sizeof(T) == 4;  // untried children on a shared-memory stack
    static constexpr int PLEV = RS ? 32 : 64;   // path levels per lane
    static constexpr int threads = 256, warps = 8, min_blocks = 3;
    static constexpr int ring = 8;              // passes between two warp drains of the lanes' rings
    static constexpr int ring_slots = ring + 1; // events a lane holds between drains: one per pass + its unit
                                                // root's (put when the unit starts, before the passes)
};

// Shared-memory layouts (per warp, [row][lane] so the 32 lanes of a row never conflict):
// the lanes' event rings -- digest sums [slot][lane] (8 B), tags [slot][lane] (4 B), and in
// the segment phase the B sums [slot][lane] (8 B) --, the untried-children stack
// [level][lane] (32-bit masks) and the path bytes [level][lane].
// Dynamic shared memory a cnt_kernel block needs beyond the staged table:
// The event ring is needed only without CNT_QUEUE (for the prime paths): head segments (prime-path
// phase) and items (segment phase) are written at once, in warp blocks of slots.
#ifndef CNT_SEG_RING
#define CNT_SEG_RING 0  // 1: the segment phase's items go through the ring (round-2 first version)
#endif
constexpr bool cnt_uses_ring(bool seg) { return (seg && CNT_SEG_RING) || !CNT_QUEUE; }
template <class T>
constexpr size_t cnt_smem_block(bool seg, bool d2 = false) {
    return (size_t)CntCfg<T>::warps * ((cnt_uses_ring(seg) ? CntCfg<T>::ring_slots * 32 * (seg ? 20 : 12) : 0) +
                                       (CntCfg<T>::RS ? 32 * 32 * 4 : 0) + CntCfg<T>::PLEV * 32 * (d2 ? 2 : 1) +
                                       (CNT_QUEUE ? 64 * 12 : 0));
}

// PH: the phase -- P_PP, the prime-path phase; P_TP, the same hashing every prime path's test
// path instead (the lanes then also keep the sum B of mix(v) over their path); P_SEG, the
// segment phase -- the trees of the SCC entry vertices: their cycles are prime paths (when the
// entry lies in the call's start range; their test paths when A.tp is set), their tail and
// transit segments (R8/R9) become ItemS records for the completion DP and the stitch.
// P_PRUNE: P_PP with NEXT #2's reachability pruning (tpgen_options.prune).
enum CntPhase : int { P_PP = 0, P_TP = 1, P_SEG = 2, P_PRUNE = 3 };
#ifndef CNT_MINB_SEG
#define CNT_MINB_SEG 3
#endif
template <class T>
constexpr int cnt_min_blocks(bool seg, bool hsh) {
    return seg ? CNT_MINB_SEG : ((sizeof(T) == 8 && hsh) ? CNT_MINB_PP64H : CntCfg<T>::min_blocks);
}

// D2 (prime-path phase, table in shared memory, G.slot_d2 set: every in-SCC out-degree <= 2, the
// normal form of the paper's Fig. 5, and config 5's SCCs): a node has at most two
// untried children, kept as two bytes instead of a mask (the take is a byte extract, not a 64-bit
// find-first-set and clear), and a push stores the parent's remaining child next to the child's
// path byte (one u16 per level), so a pop reads the popped vertex and the parent's untried child
// with ONE shared load instead of recomputing them from the parent's successor set.
template <class T, bool TS, bool HSH, bool HX, int PH, bool D2 = false>
__global__ void __launch_bounds__(CntCfg<T>::threads, cnt_min_blocks<T>(PH == P_SEG, HSH)) cnt_kernel(DfsArgs A) {
    static_assert(!D2 || (TS && PH != P_TP && PH != P_PRUNE), "D2: prime-path or segment phase with the table in shared memory");
    constexpr uint32_t PST = D2 ? 64u : 32u;  // bytes per path level of a warp's column block
    constexpr bool SEG = PH == P_SEG;
    constexpr bool TRACK_B = PH == P_TP || PH == P_SEG;
    constexpr int PASS_UNROLL = D2 ? kCntPassUnroll : 1;  // (the generic pass: 1; config 3 count 2.22 vs 2.66 ms at 2)
    using C = CntCfg<T>;
    constexpr bool RS = C::RS;
    constexpr int WARPS = C::warps;
    constexpr int PLEV = C::PLEV;
    constexpr int RING = C::ring;
    constexpr bool USE_RING = cnt_uses_ring(SEG);
    constexpr int RSLOTS = USE_RING ? C::ring_slots : 0;
    __shared__ unsigned long long s_td, s_head;
    __shared__ unsigned s_ov;
    extern __shared__ __align__(16) uint8_t stab[];  // [TS: {sin, mix}[n_slots]] then the block's areas
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *dyn = stab + (TS ? (size_t)A.n_slots * 16 : 0);
    uint64_t *sring = reinterpret_cast<uint64_t *>(dyn);                             // [warp][slot][lane]
    uint32_t *sringt = reinterpret_cast<uint32_t *>(dyn + WARPS * RSLOTS * 32 * 8);    // [warp][slot][lane]
    uint32_t *srem = sringt + WARPS * RSLOTS * 32;                                      // [warp][level][lane]
    uint8_t *spath = reinterpret_cast<uint8_t *>(srem + (RS ? WARPS * 32 * 32 : 0));  // [warp][level][lane]
    uint64_t *sq = reinterpret_cast<uint64_t *>(spath + WARPS * PLEV * PST);           // CNT_QUEUE: [warp][64]
    uint32_t *sql = reinterpret_cast<uint32_t *>(sq + (CNT_QUEUE ? WARPS * 64 : 0));  //            [warp][64]
    uint64_t *sringb = reinterpret_cast<uint64_t *>(sql + (CNT_QUEUE ? WARPS * 64 : 0));  // SEG: [warp][slot][lane]
    const DevGraph &G = A.G;
    // 32-bit shared-window addresses of this lane's columns (opaque: kept in registers)
    uint32_t pb, rb, qb, lb, bb = 0;
    if (SEG) asm volatile("mov.b32 %0, %1;" : "=r"(bb) : "r"((uint32_t)__cvta_generic_to_shared(sringb + wid * RSLOTS * 32) + lane * 8));
    asm volatile("mov.b32 %0, %1;" : "=r"(pb) : "r"((uint32_t)__cvta_generic_to_shared(spath + wid * PLEV * PST) + lane * (PST / 32u)));
    asm volatile("mov.b32 %0, %1;" : "=r"(rb) : "r"((uint32_t)__cvta_generic_to_shared(srem + (RS ? wid * 32 * 32 : 0)) + (RS ? lane * 4 : 0)));
    asm volatile("mov.b32 %0, %1;" : "=r"(qb) : "r"((uint32_t)__cvta_generic_to_shared(sring + wid * RSLOTS * 32) + lane * 8));
    asm volatile("mov.b32 %0, %1;" : "=r"(lb) : "r"((uint32_t)__cvta_generic_to_shared(sringt + wid * RSLOTS * 32) + lane * 4));
#define k2 A.k2    // 2 and 16 as kernel parameters (CNT_OPAQUE_K): constant-bank operands of the IMADs
#define k16 A.k16
#define k8 A.k8
    uint32_t bitb = 0;  // CNT_BIT_TAB (D2): shared table of the 64 one-bit masks 1 << i
    if constexpr (D2 && CNT_BIT_TAB) {
        __shared__ uint64_t s_bits[64];
        if (threadIdx.x < 64) s_bits[threadIdx.x] = 1ull << threadIdx.x;
        asm volatile("mov.b32 %0, %1;" : "=r"(bitb) : "r"((uint32_t)__cvta_generic_to_shared(s_bits)));
    }
    CntTab<T, TS> tab;
    tab.g = reinterpret_cast<const Slot<1> *>(G.slots);
    tab.gm = G.slot_mix;
    tab.sb = 0;
    if (TS) {
        uint64_t *d = reinterpret_cast<uint64_t *>(stab);
        for (int i = threadIdx.x; i < A.n_slots; i += blockDim.x) {
            d[2 * i] = D2 ? __ldg(G.slot_d2 + 2 * i) : __ldg(&tab.g[i].sin[0]);
            d[2 * i + 1] = __ldg(G.slot_mix + i);
        }
        asm volatile("mov.b32 %0, %1;" : "=r"(tab.sb) : "r"((uint32_t)__cvta_generic_to_shared(stab)));
    }
    for (int i = threadIdx.x; i < WARPS * PLEV * (int)PST; i += blockDim.x) spath[i] = 0;  // idle lanes read vertex 0
    if (threadIdx.x == 0) {
        s_td = 1ull << 32;
        s_head = 1ull << 20;
        s_ov = 0;
    }
    __syncthreads();
    Unit<1> *units = reinterpret_cast<Unit<1> *>(A.units);
    uint64_t t_pp = 0, t_vert = 0, t_ext = 0, t_ha = 0, t_hb = 0, t_cross = 0;
    uint32_t rc = 0;  // prime paths in this lane's ring
    unsigned long long hblk = 0, hblk_end = 0;  // warp-uniform: the warp's block of head slots
    unsigned long long iblk = 0, iblk_end = 0;  // ... of item slots (segment phase)

    CntLane<T> L;
    L.active = false;
    L.done = false;
    L.l = L.r = L.s = L.vb = 0;
    L.M = L.rem = L.sbit = L.ps = L.exm = 0;
    L.S = L.B = 0;
    L.cur = 0xffffu;
    L.emit = true;
    bool waiting = false, exited = false;
    int64_t slot = -1;
    int32_t uscc = 0, ugen = 0;
    uint32_t steps = 0, last_split = 0, iter = 0;
    unsigned rdy = 0;
    bool claim_pending = false;
    unsigned claim_mask = 0;
    int claim_leader = 0;
    unsigned long long claim_res = 0;
    bool snap_pending = false;
    unsigned long long snap_td = 0, snap_head = 0;
    unsigned snap_ov = 0;
    bool qdone = false, prev_active = true;

    // an event of this lane into its ring (see CntEv): prime paths are counted at once and, with
    // CNT_QUEUE, go to the warp's queue instead; everything else waits for the drain
    bool ring_ev = false;  // warp-uniform: some lane's ring holds an event other than a prime path
    uint32_t qSa, qLa;  // CNT_QUEUE: shared-window addresses of the warp's queue (opaque: kept in registers)
    asm volatile("mov.b32 %0, %1;" : "=r"(qSa) : "r"((uint32_t)__cvta_generic_to_shared(sq + (CNT_QUEUE ? wid * 64 : 0))));
    asm volatile("mov.b32 %0, %1;" : "=r"(qLa) : "r"((uint32_t)__cvta_generic_to_shared(sql + (CNT_QUEUE ? wid * 64 : 0))));
    uint32_t qn = 0;  // CNT_QUEUE: queued prime paths of the warp (warp-uniform, < 32 between hashes)
    const uint32_t ltm = (1u << lane) - 1u;
    constexpr bool CQ = D2 && PH == P_PP && HSH && HX && CNT_QUEUE && !USE_RING;
    uint32_t r_pp = 0, r_vert = 0;  // prime paths / their vertices since the last flush into t_pp / t_vert
    // CQ: one queued event per lane (warp-uniform call): a prime path is hashed (the two finalizers,
    // R20); a head segment (tag bit 31; bits 8-30 the slot of its last vertex, 0-7 |h|) becomes a
    // HeadS in the warp's block of head slots
    auto cq_flush = [&](bool valid, uint64_t z, uint32_t tag) {
        const bool hd = valid && (tag >> 31) != 0u;
        if (valid && !hd) {
            const uint64_t n = tag & 0xffu;
            t_ha += mix64(z ^ (kSeedA + n));
            t_hb += mix64(z ^ (kSeedB + n));
        }
        const uint32_t hbm = __ballot_sync(kFull, hd);
        if (hbm) {
            const uint32_t need = __popc(hbm);
            if (hblk + need > hblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                for (unsigned long long q = hblk + lane; q < hblk_end; q += 32)
                    if (q < A.head_cap) A.heads[q].x = -1;
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(A.cacc + 5, 256ull);
                b = __shfl_sync(kFull, b, 0);
                hblk = b;
                hblk_end = b + 256;
                if (b + 256 > A.head_cap && lane == 0) atomicOr(A.overflow, 8u);
            }
            const unsigned long long q = hblk + __popc(hbm & ltm);
            if (hd && q < A.head_cap) {
                HeadS hr;
                hr.S = z;
                hr.len = (int32_t)(tag & 0xffu);
                hr.x = (int32_t)((tag >> 8) & 0x7fffffu);
                *reinterpret_cast<ulonglong2 *>(A.heads + q) = *reinterpret_cast<const ulonglong2 *>(&hr);
            }
            hblk += need;
        }
    };
    auto put_ev = [&](bool pp, bool other, uint32_t kind, uint64_t Sx, uint64_t Bx, uint32_t len, int slot_) {
        if ((PH == P_TP || (SEG && A.tp != nullptr)) && (pp || (other && kind == EK_HEAD))) {
            // test paths instead (R15): the prefix walk of s before the path, the suffix walk of its
            // last vertex after it (a head's suffix comes at the end of each completion; its tag keeps
            // |h|, the drain adds the prefix's vertices)
            uint32_t lt = len;
            bool ok = tp_head(A.tp, L.vb + L.s, Sx, Bx, lt);
            if (pp) ok = ok && tp_tail(A.tp, slot_, Sx, lt);
            if (!ok) atomicOr(A.overflow, 16u);
            if (pp) len = lt;
        }
        if (pp) {  // (32-bit per round of passes; added to the 64-bit totals after the passes)
            r_pp += 1;
            r_vert += len;
        }
        if constexpr (CQ) {  // D2 + digest + exits: prime paths AND head segments through the warp's queue
            const bool ev = pp || other;
            const uint32_t bal = __ballot_sync(kFull, ev);
            if (ev) {
                const uint32_t j = qn + __popc(bal & ltm);
                TPG_DCHECK(j < 64, "cnt: warp queue overflow");
                const uint32_t tag = other ? (0x80000000u | ((uint32_t)slot_ << 8) | len) : len;
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(qSa + j * 8u), "l"(Sx) : "memory");
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(qLa + j * 4u), "r"(tag) : "memory");
            }
            qn += __popc(bal);
            if (qn >= 32) {
                __syncwarp();
                qn -= 32;
                uint64_t z;
                uint32_t tag;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(z) : "r"(qSa + (qn + lane) * 8u) : "memory");
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tag) : "r"(qLa + (qn + lane) * 4u) : "memory");
                __syncwarp();
                cq_flush(true, z, tag);
            }
        } else if constexpr (HSH && CNT_QUEUE) {
            const uint32_t bal = __ballot_sync(kFull, pp);
            if (pp) {
                const uint32_t j = qn + __popc(bal & ltm);
                TPG_DCHECK(j < 64, "cnt: warp queue overflow");
                asm volatile("st.shared.u64 [%0], %1;" ::"r"(qSa + j * 8u), "l"(Sx) : "memory");
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(qLa + j * 4u), "r"(len) : "memory");
            }
            qn += __popc(bal);
            if (qn >= 32) {
                __syncwarp();
                qn -= 32;
                uint64_t z;
                uint32_t n32;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(z) : "r"(qSa + (qn + lane) * 8u) : "memory");
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(n32) : "r"(qLa + (qn + lane) * 4u) : "memory");
                const uint64_t n = n32;
                t_ha += mix64(z ^ (kSeedA + n));
                t_hb += mix64(z ^ (kSeedB + n));
                __syncwarp();
            }
        }
        if constexpr (HX && !SEG && !USE_RING && !CQ) {  // a head segment: written at once (one HeadS per head node)
            const uint32_t hbm = __ballot_sync(kFull, other);
            if (hbm) {
                const uint32_t need = __popc(hbm);
                if (hblk + need > hblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                    for (unsigned long long q = hblk + lane; q < hblk_end; q += 32)
                        if (q < A.head_cap) A.heads[q].x = -1;
                    unsigned long long b = 0;
                    if (lane == 0) b = atomicAdd(A.cacc + 5, 256ull);
                    b = __shfl_sync(kFull, b, 0);
                    hblk = b;
                    hblk_end = b + 256;
                    if (b + 256 > A.head_cap && lane == 0) atomicOr(A.overflow, 8u);
                }
                const unsigned long long q = hblk + __popc(hbm & ltm);
                if (other && q < A.head_cap) {
                    HeadS hr;
                    hr.S = Sx;
                    hr.len = (int32_t)len + (PH == P_TP ? A.tp[L.vb + L.s].pre_len - 1 : 0);
                    hr.x = slot_;
                    *reinterpret_cast<ulonglong2 *>(A.heads + q) = *reinterpret_cast<const ulonglong2 *>(&hr);
                }
                hblk += need;
            }
        }
        if constexpr (SEG && !USE_RING) {  // a tail / transit segment: an ItemS written at once
            const uint32_t ibm = __ballot_sync(kFull, other);
            if (ibm) {
                const uint32_t need = __popc(ibm);
                if (iblk + need > iblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                    for (unsigned long long q = iblk + lane; q < iblk_end; q += 32)
                        if (q < A.item_cap) A.items[q].ent = -1;
                    unsigned long long b = 0;
                    if (lane == 0) b = atomicAdd(A.cacc + 7, 256ull);
                    b = __shfl_sync(kFull, b, 0);
                    iblk = b;
                    iblk_end = b + 256;
                    if (b + 256 > A.item_cap && lane == 0) atomicOr(A.overflow, 8u);
                }
                const unsigned long long q = iblk + __popc(ibm & ltm);
                if (other && q < A.item_cap) {
                    const Slot<1> *gsl = reinterpret_cast<const Slot<1> *>(G.slots);
                    const int32_t ent = __ldg(&gsl[L.vb + L.s].gid);
                    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(A.items + q);
                    d[0] = make_ulonglong2(Sx, Bx);
                    d[1] = make_ulonglong2(
                        (unsigned long long)len | ((unsigned long long)(uint32_t)(kind == EK_TAIL ? -1 : slot_) << 32),
                        (unsigned long long)(uint32_t)ent | ((unsigned long long)(uint32_t)slot_ << 32));
                }
                iblk += need;
            }
        }
        const bool to_ring = USE_RING && (((HSH && !CNT_QUEUE) && pp) || ((HX || SEG) && other));
        if (to_ring) {
            TPG_DCHECK(rc < (uint32_t)RSLOTS, "cnt: event ring overflow");
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(qb + rc * 256u), "l"(Sx) : "memory");
            if constexpr (SEG) asm volatile("st.shared.u64 [%0], %1;" ::"r"(bb + rc * 256u), "l"(Bx) : "memory");
            const uint32_t tag = (pp ? (EK_PP << 29) : (kind << 29)) | ((uint32_t)slot_ << 8) | len;
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(lb + rc * 128u), "r"(tag) : "memory");
            rc++;
        }
        if constexpr (USE_RING && (HX || SEG)) ring_ev |= __any_sync(kFull, other);
    };
    // warp-uniform: every lane hashes the prime paths in its ring (the two finalizers, R20),
    // then the warp writes the head segments (prime-path phase) or the items (segment phase)
    auto drain = [&]() {
        if constexpr (!USE_RING) return;
        const uint32_t mx = __reduce_max_sync(kFull, rc);
        for (uint32_t j = 0; j < mx; j++) {
            uint64_t z = 0;
            uint32_t tag = 0;
            if (j < rc) {
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(z) : "r"(qb + j * 256u) : "memory");
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tag) : "r"(lb + j * 128u) : "memory");
            }
            const uint32_t kind = tag >> 29, len = tag & 0xffu;
            const int tslot = (int)((tag >> 8) & 0x1fffffu);
            if (HSH && !CNT_QUEUE && j < rc && kind == EK_PP) {
                t_ha += mix64(z ^ (kSeedA + (uint64_t)len));
                t_hb += mix64(z ^ (kSeedB + (uint64_t)len));
            }
            if constexpr (HX && !SEG) {
                if (ring_ev) {  // head segments: one HeadS per head node, in the warp's block of slots
                    const bool h = j < rc && kind == EK_HEAD;
                    const uint32_t hb = __ballot_sync(kFull, h);
                    if (hb) {
                        const uint32_t need = __popc(hb);
                        if (hblk + need > hblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                            for (unsigned long long q = hblk + lane; q < hblk_end; q += 32)
                                if (q < A.head_cap) A.heads[q].x = -1;
                            unsigned long long b = 0;
                            if (lane == 0) b = atomicAdd(A.cacc + 5, 256ull);
                            b = __shfl_sync(kFull, b, 0);
                            hblk = b;
                            hblk_end = b + 256;
                            if (b + 256 > A.head_cap && lane == 0) atomicOr(A.overflow, 8u);
                        }
                        const unsigned long long q = hblk + __popc(hb & ((1u << lane) - 1u));
                        if (h && q < A.head_cap) {
                            HeadS hr;
                            hr.S = z;
                            hr.len = (int32_t)len + (PH == P_TP ? A.tp[L.vb + L.s].pre_len - 1 : 0);
                            hr.x = tslot;
                            *reinterpret_cast<ulonglong2 *>(A.heads + q) = *reinterpret_cast<const ulonglong2 *>(&hr);
                        }
                        hblk += need;
                    }
                }
            }
            if constexpr (SEG) {
                if (ring_ev) {  // items: a tail segment, or a transit segment over an exit vertex's arcs
                    const bool it = j < rc && (kind == EK_TAIL || kind == EK_TRANSIT);
                    const uint32_t ib = __ballot_sync(kFull, it);
                    if (ib) {
                        const uint32_t need = __popc(ib);
                        if (iblk + need > iblk_end) {  // a new block of 256 slots (the rest of the old one: holes)
                            for (unsigned long long q = iblk + lane; q < iblk_end; q += 32)
                                if (q < A.item_cap) A.items[q].ent = -1;
                            unsigned long long b = 0;
                            if (lane == 0) b = atomicAdd(A.cacc + 7, 256ull);
                            b = __shfl_sync(kFull, b, 0);
                            iblk = b;
                            iblk_end = b + 256;
                            if (b + 256 > A.item_cap && lane == 0) atomicOr(A.overflow, 8u);
                        }
                        const unsigned long long q = iblk + __popc(ib & ((1u << lane) - 1u));
                        if (it && q < A.item_cap) {
                            uint64_t Bx;
                            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(Bx) : "r"(bb + j * 256u) : "memory");
                            const Slot<1> *gsl = reinterpret_cast<const Slot<1> *>(G.slots);
                            const int32_t ent = __ldg(&gsl[L.vb + L.s].gid);
                            const int32_t lastv = tslot;  // (a slot: the test-path terms are per slot)
                            ulonglong2 *d = reinterpret_cast<ulonglong2 *>(A.items + q);
                            d[0] = make_ulonglong2(z, Bx);
                            d[1] = make_ulonglong2(
                                (unsigned long long)len | ((unsigned long long)(uint32_t)(kind == EK_TAIL ? -1 : tslot) << 32),
                                (unsigned long long)(uint32_t)ent | ((unsigned long long)(uint32_t)lastv << 32));
                        }
                        iblk += need;
                    }
                }
            }
        }
        rc = 0;
        ring_ev = false;
    };

    while (true) {
        iter++;
        bool feed = false;
        uint32_t split_need = A.split_min;
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
                const long long backlog = (long long)(td >> 32) - (long long)hd;
                feed = backlog < (long long)A.low_water;
                if (backlog < -(long long)A.starve_lanes) split_need = A.split_min_starve;
            }
        }
        // ---------------- waiting lanes: start the claimed unit once it is written
        bool st_pp = false, st_other = false;  // the unit root's event (a prime path, or see CntEv)
        uint32_t st_kind = 0;
        uint64_t st_S = 0, st_B = 0;
        uint32_t st_len = 0;
        int st_slot = 0;
        if (waiting) {
            if (rdy != 0u) {
                waiting = false;
                // acquire: the producer's unit stores (made visible by its fence) before our reads
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                const Unit<1> *U = units + slot;
                const int4 h = __ldcg(reinterpret_cast<const int4 *>(&U->scc));
                L.M = (T)__ldcg(reinterpret_cast<const unsigned long long *>(U->M));
                uscc = h.x;
                ugen = __ldcg(A.gen + slot);
                const int kind = (h.w >> 8) & 0xff;
                const int depth = h.w & 0xff;
                L.l = L.r = depth;
                L.vb = __ldg(G.scc_vbase + uscc);
                const uint32_t *p4 = reinterpret_cast<const uint32_t *>(U->path);
                uint64_t S0 = 0, B0 = 0;
                int u = 0;
#pragma unroll 1
                for (int q = 0; q * 4 <= depth; q++) {  // path bytes into the lane's column, S of the path
                    const uint32_t wv = __ldcg(p4 + q);
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        const int i = q * 4 + b;
                        if (i <= depth) {
                            const int x = (int)((wv >> (8 * b)) & 0xffu);
                            sts_u8(pb + (uint32_t)i * PST, x);
                            const uint64_t mx = tab.mix(L.vb + x);
                            S0 += mul64x32(mx, 2u * (uint32_t)i + 1u);
                            B0 += mx;
                            u = x;
                        }
                    }
                }
                L.s = (int)(__ldcg(p4) & 0xffu);
                L.sbit = (T)1 << L.s;
                L.ps = tab.pin(L.vb + L.s);
                if constexpr (!D2) L.exm = (HX || SEG) ? (T)__ldg(G.scc_exm + uscc) : (T)0;
                L.S = S0;
                L.B = B0;
                if constexpr (SEG) {
                    const int32_t sg = __ldg(&reinterpret_cast<const Slot<1> *>(G.slots)[L.vb + L.s].gid);
                    L.emit = sg >= G.shard_lo && sg < G.shard_hi;
                }
                steps = 0;
                last_split = 0;
                L.active = true;
                if (kind == K_CLOSURE) {  // the closing arc of path[0..depth] back to s
                    t_ext += L.emit ? 1 : 0;
                    st_pp = L.emit;
                    const uint64_t ms_ = tab.mix(L.vb + L.s);
                    st_S = S0 + mul64x32(ms_, 2u * (uint32_t)depth + 3u);
                    st_B = B0 + ms_;
                    st_len = (uint32_t)depth + 2;
                    st_slot = L.vb + L.s;
                    L.rem = 0;
                    L.cur = 0xffffu;
                    L.done = true;
                } else {  // K_NODE: the node's own event, then its subtree
                    if (depth > 0 && L.emit) t_ext += 1;
                    const T ub = (T)1 << u;
                    const T su = D2 ? (T)__ldg(&tab.g[L.vb + u].sin[0]) : tab.sin(L.vb + u);
                    L.rem = su & (~L.M | L.sbit);
                    if constexpr (PH == P_PRUNE) {  // NEXT #2: the root of a donated unit, as at a push
                        if (depth > 0 && depth <= CNT_PRUNE_MAXD && L.rem != 0 && !prune_keep<T>(tab, L.vb, L.ps, u, L.M, L.rem))
                            L.rem = 0;
                    }
                    if constexpr (D2) L.cur = d2_bytes<T>(L.rem);
                    const bool ex = D2 ? ((__ldg(G.slot_d2 + 2 * (L.vb + u)) >> 40) & 1) != 0 : ((L.exm >> u) & 1) != 0;
                    if constexpr (SEG) {  // tail segment (succ(u) on the path) or transit segments (R8, R9)
                        st_other = ex || (su & ~L.M) == 0;
                        st_kind = ex ? EK_TRANSIT : EK_TAIL;
                    } else {
                        st_pp = L.rem == 0 && (L.ps & ~(L.M & ~ub)) == 0 && !ex;
                        st_other = ex && (L.ps & ~L.M) == 0;
                        st_kind = EK_HEAD;
                    }
                    st_S = S0;
                    st_B = B0;
                    st_len = (uint32_t)depth + 1;
                    st_slot = L.vb + u;
                    L.done = L.rem == 0;
                }
            } else if (qdone) {
                waiting = false;
                exited = true;
            } else if (slot < (int64_t)A.qcap) {
                rdy = ld_relaxed(A.ready + slot);
            }
        }
        put_ev(st_pp, st_other, st_kind, st_S, st_B, st_len, st_slot);  // (the ring is empty: drained after the passes)
        // ---------------- the claim issued last iteration
        if (claim_pending) {
            const unsigned long long base = __shfl_sync(kFull, claim_res, claim_leader);
            if ((claim_mask >> lane) & 1u) {
                slot = (int64_t)(base + __popc(claim_mask & ((1u << lane) - 1u)));
                waiting = true;
                rdy = (slot < (int64_t)A.qcap) ? ld_relaxed(A.ready + slot) : 0u;
            }
            claim_pending = false;
        }
        {
            const unsigned need = __ballot_sync(kFull, !L.active && !waiting && !exited);
            if (need && !claim_pending) {
                claim_leader = __ffs(need) - 1;
                claim_mask = need;
                claim_pending = true;
                if (lane == claim_leader) claim_res = atomicAdd(A.qhead, (unsigned long long)__popc(need));
            }
        }
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
        if (!any_active) {
            drain();
            if (__ballot_sync(kFull, !exited) == 0) break;
            __nanosleep(128);
            continue;
        }

        // ---------------- passes of the unified step: every stepping lane makes exactly one
        // move per pass -- a pop (its node has no untried child left) or the take of its
        // node's lowest untried child -- through ONE instruction stream: the moved vertex v
        // (the popped one or the child), its digest term mix(v)*(2 pos+1), the visited-bit
        // toggle and the depth change are the same operations either way
        uint32_t ext32 = 0;
        bool actp = L.active && !L.done;  // (D2, CNT_ACT_REG) stepping, kept across the passes; L.done after them
#pragma unroll 1
        for (int blk = 0; blk < CNT_PASSES / RING; blk++) {
#pragma unroll PASS_UNROLL
            for (int t = 0; t < RING; t++) {
              if constexpr (D2) {
                const bool act = CNT_ACT_REG ? actp : (L.active && !L.done);
#pragma unroll
                for (int k = 0; k < CNT_D2_POPS; k++) {  // pops first (straight-line, predicated)
                    const bool pk = act & (((~L.cur) & 0xffu) == 0u) & (L.l > L.r);
#if CNT_POP_PRED
                    // only popping lanes touch shared memory (the LSU pipe is the busiest: 85 %); the
                    // others read 0 (vertex 0, weight 0)
                    uint32_t ek;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tmov.u32 %0, 0;\n\t@p ld.shared.u16 %0, [%1];\n\t}"
                                 : "=r"(ek) : "r"(pb + (uint32_t)L.l * PST), "r"((uint32_t)pk) : "memory");
                    const int uk = (int)(ek & 0xffu);
                    uint64_t mk;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tmov.b64 %0, 0;\n\t@p ld.shared.u64 %0, [%1];\n\t}"
                                 : "=l"(mk) : "r"(mad_u32((uint32_t)(L.vb + uk), k16, tab.sb + 8u)), "r"((uint32_t)pk) : "memory");
#else
                    const uint32_t ek = lds_u16(pb + (uint32_t)L.l * PST);
                    const int uk = (int)(ek & 0xffu);
                    uint64_t mk;
                    if (CNT_OPAQUE_K)
                        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(mk) : "r"(mad_u32((uint32_t)(L.vb + uk), k16, tab.sb + 8u)) : "memory");
                    else
                        mk = tab.mix(L.vb + uk);
#endif
#if CNT_BIT_TAB
                    // the popped vertex's bit from the shared bit table by a predicated load (0 when this
                    // lane does not pop), the weight 0 when it does not: no shifts, no 64-bit selects
                    uint64_t ubk;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tmov.b64 %0, 0;\n\t@p ld.shared.u64 %0, [%1];\n\t}"
                                 : "=l"(ubk) : "r"(mad_u32((uint32_t)uk, k8, bitb)), "r"((uint32_t)pk) : "memory");
                    const uint64_t prk = mul64x32(mk, pk ? odd2((uint32_t)L.l, k2) : 0u);
                    L.M ^= (T)ubk;
                    L.S -= prk;
#elif CNT_D2_SELFREE
                    // predicate folded into the operands (no 64-bit selects on the ALU pipe, the kernel's
                    // limiting pipe): the multiplier is 0 and the shift 64 (PTX clamps: a zero bit) when
                    // this lane does not pop
                    const uint64_t prk = mul64x32(mk, pk ? 2u * (uint32_t)L.l + 1u : 0u);
                    uint64_t ubk;
                    asm("shl.b64 %0, %1, %2;" : "=l"(ubk) : "l"(1ull), "r"(pk ? (uint32_t)uk : 64u));
                    L.M ^= (T)ubk;
                    L.S -= prk;
#else
                    const uint64_t prk = mul64x32(mk, odd2((uint32_t)L.l, k2));
                    const T ubk = (T)1 << uk;
                    L.M = pk ? (L.M ^ ubk) : L.M;
                    L.S = pk ? (L.S - prk) : L.S;
#endif
                    if constexpr (TRACK_B) L.B = pk ? (L.B - mk) : L.B;
                    L.l -= pk ? 1 : 0;
                    L.cur = pk ? ((ek >> 8) | 0xff00u) : L.cur;
                }
                const uint32_t cur = L.cur;
                const int l = L.l;
                const uint32_t a = cur & 0xffu;  // (take) the child
                const bool empty = ((~cur) & 0xffu) == 0u;
                if (CNT_ACT_REG) actp = act & !(empty & (l == L.r));  // the unit's subtree is finished
                else if (act & empty & (l == L.r)) L.done = true;
                const bool pop = (CNT_D2_POPS == 0) & act & empty & (l > L.r);
                TPG_DCHECK(!act || (l >= L.r && l < PLEV), "cnt: depth out of range");
                const bool take = act & !empty;
                const uint32_t e = CNT_D2_POPS == 0 ? lds_u16(pb + (uint32_t)l * PST) : 0u;  // {path[l], the untried child of level l-1}
                const int v = take ? (int)a : (int)(e & 0xffu);     // the child, or the vertex popped
                const int vslot = L.vb + v;
                uint64_t wd, mv;  // {t0 | t1 << 32 | exit << 40, mix64(gid)} of v
                asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(wd), "=l"(mv)
                             : "r"(CNT_OPAQUE_K ? mad_u32((uint32_t)vslot, k16, tab.sb) : tab.sb + (uint32_t)vslot * 16u) : "memory");
                const uint64_t prod = mul64x32(mv, odd2((uint32_t)(take ? l + 1 : l), k2));
#if CNT_BIT_TAB && CNT_BIT_TAB_TAKE
                T vbit;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(vbit) : "r"(mad_u32((uint32_t)v, k8, bitb)) : "memory");
#else
                const T vbit = (T)1 << v;
#endif
                const T Mw = L.M | vbit;
                const T avail = ~Mw | L.sbit;  // vertices a child of v may move to
                const uint32_t w1 = (uint32_t)(wd >> 32);
                const uint32_t t0 = (uint32_t)wd, t1 = w1 & 0xffu;  // (a missing one is v: never available)
                // straight-line (bitwise, no short-circuit branches): the availability bits of t0, t1
                const uint32_t ok0 = (uint32_t)(avail >> t0) & 1u, ok1 = (uint32_t)(avail >> t1) & 1u;
                const uint32_t first = ok0 ? t0 : (ok1 ? t1 : 0xffu);
                const uint32_t cw = first | ((ok0 & ok1) ? (t1 << 8) : 0xff00u);
                const bool clo = (int)a == L.s;
                const bool ex = HX && (w1 & 0x100u) != 0;
                const bool leaf = (ok0 | ok1) == 0u;
                const bool pok = (L.ps & ~L.M) == 0;   // pred(s) within path[0..l]
                const bool pokw = (L.ps & ~Mw) == 0;   // ... within path[0..l] + v
                bool pp, other;
                if constexpr (SEG) {  // cycles are prime paths; tail / transit segments become items (R8, R9)
                    const uint32_t in0 = (uint32_t)(Mw >> t0) & 1u, in1 = (uint32_t)(Mw >> t1) & 1u;
                    pp = take & clo & L.emit;
                    other = take & !clo & (ex | ((in0 & in1) != 0u));
                } else {
                    pp = take & (clo | (leaf & pok & !ex));
                    other = HX & take & !clo & ex & pokw;  // a head segment
                }
                const bool push = take & !clo & !leaf;
                const uint64_t Sw = L.S + prod;
                const uint64_t Bw = L.B + mv;
                if (push) {
                    TPG_DCHECK(l + 1 < PLEV, "cnt: path deeper than the lane's column");
                    sts_u16(pb + (uint32_t)(l + 1) * PST, cur);  // {w, the untried child left at level l}
                }
                ext32 += (take && (!SEG || L.emit)) ? 1u : 0u;
                L.M = (push | pop) ? (L.M ^ vbit) : L.M;
                L.S = push ? Sw : (pop ? L.S - prod : L.S);
                if constexpr (TRACK_B) L.B = push ? Bw : (pop ? L.B - mv : L.B);
                L.l = l + (push ? 1 : 0) - (pop ? 1 : 0);
                L.cur = push ? cw : (pop ? ((e >> 8) | 0xff00u) : (take ? ((cur >> 8) | 0xff00u) : cur));
                put_ev(pp, other, SEG ? (ex ? EK_TRANSIT : EK_TAIL) : EK_HEAD, Sw, Bw, (uint32_t)l + 2, vslot);
              } else {
                const bool act = L.active && !L.done;
                const T rem = L.rem;
                const int l = L.l;
                const bool empty = rem == 0;
                if (act && empty && l == L.r) L.done = true;  // the unit's subtree is finished
                const bool pop = act && empty && l > L.r;
                TPG_DCHECK(!act || (l >= L.r && l < PLEV), "cnt: depth out of range");
                const bool take = act && !empty;
                const int w = ffs_t(rem);                     // (take) the child
                const int u = lds_u8(pb + (uint32_t)l * PST);  // (pop) the vertex popped
                const int v = take ? w : u;
                const int vslot = L.vb + v;                   // (idle lanes: a valid slot of their last SCC)
                const uint64_t mv = tab.mix(vslot);
                const uint64_t prod = mul64x32(mv, 2u * (uint32_t)(take ? l + 1 : l) + 1u);
                const T vbit = (T)1 << v;
                const T sn = tab.sin(vslot);
                const bool clo = w == L.s;
                const T Mw = L.M | vbit;
                const T cw = clo ? (T)0 : (sn & (~Mw | L.sbit));  // (take) the child's own untried children
                bool ex = false;
                if constexpr (HX || SEG) ex = ((L.exm >> v) & 1) != 0;
                bool pp, other;
                uint32_t kind;
                if constexpr (SEG) {  // cycles are prime paths; tail / transit segments become items
                    pp = take && clo && L.emit;
                    other = take && !clo && (ex || (sn & ~Mw) == 0);
                    kind = ex ? EK_TRANSIT : EK_TAIL;
                } else {
                    pp = take && (clo || (cw == 0 && (L.ps & ~L.M) == 0 && !ex));
                    other = HX && take && !clo && ex && (L.ps & ~Mw) == 0;  // a head segment
                    kind = EK_HEAD;
                }
                bool push = take && cw != 0;
                if constexpr (PH == P_PRUNE) {
                    // NEXT #2 (not in the paper): a child w whose subtree can hold no prime
                    // path is not entered.  Every event below w ends at a vertex x reachable from w in
                    // C \ path: a closure needs x in pred(s), an internal prime path or a head segment
                    // needs pred(s) on the path (Def. 1 / R3, Def. 6).  So when w is not in pred(s),
                    // some of pred(s) is off the path, and no vertex of pred(s) off the path is
                    // reachable from w in C \ path (bitset BFS), the subtree is empty of events.
                    // (a donated unit's root gets the same test when it starts: the extensions made
                    // do not depend on the donation pattern)
                    if (push && l + 1 <= CNT_PRUNE_MAXD) push = prune_keep<T>(tab, L.vb, L.ps, v, Mw, cw);
                }
                const uint64_t Sw = L.S + prod;  // (take) the digest sum of path + w
                T rem_pop = 0;
                if constexpr (RS) {
                    if (pop) rem_pop = (T)lds_u32(rb + (uint32_t)(l - 1) * 128u);
                } else {
                    if (pop) {  // the parent's successors above u that are still open
                        const int p = lds_u8(pb + (uint32_t)(l - 1) * PST);
                        const T above = (u >= 63) ? (T)0 : ((~(T)0) << (u + 1));
                        rem_pop = tab.sin(L.vb + p) & (~(L.M & ~vbit) | L.sbit) & above;
                    }
                }
                if (push) {
                    TPG_DCHECK(l + 1 < PLEV, "cnt: path deeper than the lane's column");
                    if constexpr (RS) sts_u32(rb + (uint32_t)l * 128u, (uint32_t)(rem & (rem - 1)));
                    sts_u8(pb + (uint32_t)(l + 1) * PST, w);
                }
                ext32 += (take && (!SEG || L.emit)) ? 1u : 0u;
                L.M = (push || pop) ? (L.M ^ vbit) : L.M;
                L.S = push ? Sw : (pop ? L.S - prod : L.S);
                const uint64_t Bw = L.B + mv;  // (the sum of mix: test-path digests and segment items)
                if constexpr (TRACK_B) L.B = push ? Bw : (pop ? L.B - mv : L.B);
                L.l = l + (push ? 1 : 0) - (pop ? 1 : 0);
                L.rem = push ? cw : (pop ? rem_pop : (take ? (rem & (rem - 1)) : rem));
#if CNT_POP2
                if (pop && L.rem == 0 && L.l > L.r) {  // the parent has nothing left either: pop it too
                    const int l2 = L.l;
                    const int u2 = lds_u8(pb + (uint32_t)l2 * 32u);
                    const T vb2 = (T)1 << u2;
                    const uint64_t mv2 = tab.mix(L.vb + u2);
                    T rp2;
                    if constexpr (RS) {
                        rp2 = (T)lds_u32(rb + (uint32_t)(l2 - 1) * 128u);
                    } else {
                        const int p2 = lds_u8(pb + (uint32_t)(l2 - 1) * 32u);
                        const T above2 = (u2 >= 63) ? (T)0 : ((~(T)0) << (u2 + 1));
                        rp2 = tab.sin(L.vb + p2) & (~(L.M & ~vb2) | L.sbit) & above2;
                    }
                    L.M ^= vb2;
                    L.S -= mul64x32(mv2, 2u * (uint32_t)l2 + 1u);
                    if constexpr (TRACK_B) L.B -= mv2;
                    L.l = l2 - 1;
                    L.rem = rp2;
                }
#endif
                put_ev(pp, other, kind, Sw, Bw, (uint32_t)l + 2, vslot);
              }
            }
            drain();
        }
        if (D2 && CNT_ACT_REG && L.active && !actp) L.done = true;
        t_ext += ext32;
        t_pp += r_pp;
        t_vert += r_vert;
        r_pp = r_vert = 0;
        if (L.active) steps += CNT_PASSES;

        // ---------------- donate on demand: the untried children of the shallowest open level
        if (feed && L.active && !L.done && (steps - last_split >= split_need || ugen < A.eager_gens)) {
            int j0 = -1;
            T c0 = 0;
            {
                T M = L.M;
                for (int j = L.l; j >= L.r; j--) {
                    T c;
                    if (j == L.l) {
                        c = D2 ? d2_mask<T>(L.cur) : L.rem;
                    } else {
                        const int wc = lds_u8(pb + (uint32_t)(j + 1) * PST);  // the child of level j on the path
                        M &= ~((T)1 << wc);
                        if constexpr (D2) {
                            c = d2_mask<T>((uint32_t)lds_u8(pb + (uint32_t)(j + 1) * PST + 1u) | 0xff00u);
                        } else if constexpr (RS) {
                            c = (T)lds_u32(rb + (uint32_t)j * 128u);
                        } else {
                            const int p = lds_u8(pb + (uint32_t)j * PST);
                            const T above = (wc >= 63) ? (T)0 : ((~(T)0) << (wc + 1));
                            c = tab.sin(L.vb + p) & (~M | L.sbit) & above;
                        }
                    }
                    if (c) {
                        j0 = j;
                        c0 = c;
                    }
                }
            }
            const int m = j0 >= 0 ? (sizeof(T) == 4 ? __popc((uint32_t)c0) : __popcll((uint64_t)c0)) : 0;
            if (m > 0) {
                const unsigned long long base = atomicAdd(A.qtd, (unsigned long long)m << 32) >> 32;
                if (base + m > A.qcap) {
                    atomicOr(A.overflow, 4u);
                } else {
                    T M = L.M;  // the mask of path[0..j0]
                    for (int j = j0 + 1; j <= L.l; j++) M &= ~((T)1 << lds_u8(pb + (uint32_t)j * PST));
                    T c = c0;
                    for (int n = 0; n < m; n++) {
                        const int w = ffs_t(c);
                        c &= c - 1;
                        const int kind = (w == L.s) ? K_CLOSURE : K_NODE;
                        Unit<1> &U = units[base + n];
                        for (int q = 0; q <= (j0 >> 2); q++) {
                            uint32_t wv = 0;
#pragma unroll
                            for (int b = 0; b < 4; b++)
                                if (q * 4 + b <= j0) wv |= (uint32_t)lds_u8(pb + (uint32_t)(q * 4 + b) * PST) << (8 * b);
                            reinterpret_cast<uint32_t *>(U.path)[q] = wv;
                        }
                        uint64_t Mu = (uint64_t)M;
                        if (kind == K_NODE) {
                            U.path[j0 + 1] = (uint8_t)w;
                            Mu |= 1ull << w;
                        }
                        U.M[0] = Mu;
                        const int depth = (kind == K_NODE) ? j0 + 1 : j0;
                        *reinterpret_cast<int4 *>(&U.scc) = make_int4(uscc, -1, 0, depth | (kind << 8));
                        A.gen[base + n] = ugen + 1;
                    }
                    __threadfence();  // unit data before the ready flags
                    for (int n = 0; n < m; n++) st_relaxed(A.ready + base + n, 1u);
                    if (j0 == L.l) L.done = true;  // nothing left below the donated level
                    else L.r = j0 + 1;             // the walk now ends when it returns to depth j0+1
                    last_split = steps;
                }
            }
        }
        if (L.active && L.done) {
            atomicAdd(A.qtd, 1ull);  // done += 1
            L.active = false;
            L.done = false;
        }
    }
    t_pp += r_pp;
    t_vert += r_vert;
    if constexpr (CQ) {  // the queue's remainder
        __syncwarp();
        uint64_t z = 0;
        uint32_t tag = 0;
        if (lane < qn) {
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(z) : "r"(qSa + lane * 8u) : "memory");
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tag) : "r"(qLa + lane * 4u) : "memory");
        }
        cq_flush(lane < qn, z, tag);
    } else if constexpr (HSH && CNT_QUEUE) {  // the queue's remainder
        __syncwarp();
        if (lane < qn) {
            uint64_t z;
            uint32_t n32;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(z) : "r"(qSa + lane * 8u) : "memory");
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(n32) : "r"(qLa + lane * 4u) : "memory");
            t_ha += mix64(z ^ (kSeedA + (uint64_t)n32));
            t_hb += mix64(z ^ (kSeedB + (uint64_t)n32));
        }
    }
    // the rings were drained; the head block's unused slots, then the totals
    for (unsigned long long j = hblk + lane; j < hblk_end; j += 32)
        if (j < A.head_cap) A.heads[j].x = -1;
    for (unsigned long long j = iblk + lane; j < iblk_end; j += 32)
        if (j < A.item_cap) A.items[j].ent = -1;
    uint64_t v[7] = {t_pp, t_vert, t_ext, t_ha, t_hb, 0, t_cross};
    bool ovf = false;  // prime-path totals >= 2^62 (or a wrapped sum): LIMIT_EXCEEDED
#pragma unroll
    for (int q = 0; q < 7; q++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t r = v[q] + __shfl_xor_sync(kFull, v[q], o);
            if ((q < 2 || q == 6) && (r < v[q] || r >= (1ull << 62))) ovf = true;
            v[q] = r;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 7; q++) {
            if (!v[q] || q == 5) continue;
            const unsigned long long old = atomicAdd(A.cacc + q, (unsigned long long)v[q]);
            if ((q < 2 || q == 6) && (old + v[q] < old || old + v[q] >= (1ull << 62))) ovf = true;
        }
    }
    if (__any_sync(kFull, ovf) && lane == 0) atomicOr(A.overflow, 1u);
}
#undef k2
#undef k16
#undef k8

}  // namespace tpg
