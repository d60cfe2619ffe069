// frontier.cuh -- level-synchronous frontier extension (TPGEN_ENGINE_FRONTIER;
// DESIGN.md §6.6).
//
// Alg. 4 "ExtendPath" applied to every simple path of l+1 vertices
// at once: level l's frontier is a flat array of 16-byte path records in HBM,
// each launch reads it once and writes level l+1's frontier once (the paper's
// level-by-level shape, without its per-vertex path lists).  A record
// carries what the extension and the maximality test need -- the visited mask M
// (<= 32 SCC-local vertices), the last vertex u, the first vertex s and the SCC's
// slot base -- plus S, the position-keyed digest sum of the path so far (R20), so
// that a prime path's digest is finished at the moment it is recognised and no
// path is ever re-read.  Events, as in the LEAN DFS step (R3, Def. 1):
//   child w == s            -> cycle closure, a prime path of l+2 vertices;
//   child w not in M        -> new path p' = p + w with untried-child mask
//                              c' = succ(w) & (~M' | {s}); p' is an internal prime
//                              path iff c' == 0 and pred(s) within M (= M' \ {w});
//                              p' joins level l+1 only if c' != 0 (a record with
//                              no child would be read for nothing).
// Compaction: block scan of the per-thread child counts, one atomicAdd per tile
// on the level's record counter (the frontier's order is irrelevant: counts,
// E_canon and the order-free digest are all sums).  Prime paths found in the
// (divergent) child loop are queued per warp and hashed 32 at a time.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace tpg {

template <class T>
struct FSlot {        // per SCC slot (local ids ascend with global ids)
    T sin;            // in-SCC successor bits (local)
    T pin;            // in-SCC predecessor bits (local)
    int32_t gid;      // global vertex id
    int32_t flags;    // F_EXIT (an arc leaves its SCC), F_ENTRY
};

// Records.  32-bit masks (SCCs of <= 32 vertices): one 16-byte record
//   {key = mask | last << 32 | first << 37 | slot base << 42, S}.
// 64-bit masks (<= 64 vertices): a 16-byte record {mask, last | first << 6 |
// slot base << 12} plus S in a parallel array (24 bytes per record).
__device__ __forceinline__ uint64_t fkey(uint32_t M, uint32_t u, uint32_t s, uint32_t vb) {
    return (uint64_t)M | ((uint64_t)u << 32) | ((uint64_t)s << 37) | ((uint64_t)vb << 42);
}

struct FrontierArgs {
    const void *tab;             // FSlot<T>[n_tab]
    int32_t n_tab;
    const ulonglong2 *in;        // level l records {key, S}
    ulonglong2 *out;             // level l+1 records
    const uint64_t *in_S;        // 64-bit masks: S of the level l records
    uint64_t *out_S;             //               S of the level l+1 records
    const uint64_t *in_B;        // segment phase: sum of mix(v) of the level l paths (item slopes, R20)
    uint64_t *out_B;
    // graphs whose arcs leave SCCs (count modes): heads of the prime-path phase and
    // items of the segment phase, in warp blocks of 256 slots (holes marked), counted in hcnt[0] / hcnt[1]
    HeadS *heads;
    unsigned long long head_cap;
    ItemS *items;
    unsigned long long item_cap;
    unsigned long long *hcnt;
    const uint64_t *slot_mix;    // per slot mix64(gid) (the segment phase's B sums)
    int32_t shard_lo, shard_hi;  // segment phase: cycles through entries in this range are counted
    const unsigned long long *cnt_in;
    unsigned long long *cnt_out;
    unsigned long long cap;      // records per buffer
    unsigned long long lim;      // records of the input to process (chunked mode), ~0 = all
    unsigned long long ring;     // chunked walk: the output is a ring of `ring` records, appends start at
    unsigned long long ring_off; //   ring_off (0 = a flat buffer; cap then bounds the appends)
    unsigned long long *acc;     // [0] prime paths, [1] vertices, [2] extensions, [3] digest a, [4] digest b
    unsigned int *overflow;
    int32_t l;                   // input paths have l + 1 vertices
};

struct FAcc {
    unsigned long long pp = 0, vert = 0, ext = 0, ha = 0, hb = 0;
    __device__ __forceinline__ void emit(uint64_t S, uint32_t len) {
        pp++;
        vert += len;
        ha += mix64(S ^ (0x9E3779B97F4A7C15ull + (uint64_t)len));
        hb += mix64(S ^ (0xD1B54A32D192ED03ull + (uint64_t)len));
    }
    __device__ __forceinline__ void flush(unsigned long long *acc) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pp += __shfl_down_sync(0xffffffffu, pp, o);
            vert += __shfl_down_sync(0xffffffffu, vert, o);
            ext += __shfl_down_sync(0xffffffffu, ext, o);
            ha += __shfl_down_sync(0xffffffffu, ha, o);
            hb += __shfl_down_sync(0xffffffffu, hb, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (pp) atomicAdd(acc + 0, pp);
            if (vert) atomicAdd(acc + 1, vert);
            if (ext) atomicAdd(acc + 2, ext);
            atomicAdd(acc + 3, ha);
            atomicAdd(acc + 4, hb);
        }
    }
};

template <class T>
struct FT;
template <>
struct FT<uint32_t> {
    __device__ static int ffs(uint32_t x) { return __ffs(x); }
    __device__ static int popc(uint32_t x) { return __popc(x); }
    template <bool HASH>
    __device__ static ulonglong2 ld(const FrontierArgs &A, unsigned long long i, uint64_t &S) {
        TPG_DCHECK(i < A.cap, "frontier: record read beyond the level buffer");
        if constexpr (!HASH) {  // counts only: 8-byte records (the key)
            S = 0;
            return make_ulonglong2(__ldcs(reinterpret_cast<const unsigned long long *>(A.in) + i), 0);
        }
        const ulonglong2 r = __ldcs(A.in + i);
        S = r.y;
        return r;
    }
    __device__ static void dec(const ulonglong2 &r, uint32_t &M, uint32_t &u, uint32_t &s, uint32_t &vb) {
        M = (uint32_t)r.x;
        u = (uint32_t)(r.x >> 32) & 31u;
        s = (uint32_t)(r.x >> 37) & 31u;
        vb = (uint32_t)(r.x >> 42);
    }
    template <bool HASH>
    __device__ static void st(const FrontierArgs &A, unsigned long long j, uint32_t M, uint32_t w, uint32_t s,
                              uint32_t vb, uint64_t S) {
        TPG_DCHECK(j < (A.ring ? A.ring : A.cap), "frontier: record write beyond the level buffer");
        if constexpr (HASH) __stcs(A.out + j, make_ulonglong2(fkey(M, w, s, vb), S));
        else __stcs(reinterpret_cast<unsigned long long *>(A.out) + j, (unsigned long long)fkey(M, w, s, vb));
    }
};
template <>
struct FT<uint64_t> {
    __device__ static int ffs(uint64_t x) { return __ffsll((long long)x); }
    __device__ static int popc(uint64_t x) { return __popcll(x); }
    template <bool HASH>
    __device__ static ulonglong2 ld(const FrontierArgs &A, unsigned long long i, uint64_t &S) {
        S = HASH ? __ldcs(reinterpret_cast<const unsigned long long *>(A.in_S) + i) : 0ull;
        return __ldcs(A.in + i);
    }
    __device__ static void dec(const ulonglong2 &r, uint64_t &M, uint32_t &u, uint32_t &s, uint32_t &vb) {
        M = r.x;
        u = (uint32_t)r.y & 63u;
        s = (uint32_t)(r.y >> 6) & 63u;
        vb = (uint32_t)(r.y >> 12);
    }
    template <bool HASH>
    __device__ static void st(const FrontierArgs &A, unsigned long long j, uint64_t M, uint32_t w, uint32_t s,
                              uint32_t vb, uint64_t S) {
        __stcs(A.out + j, make_ulonglong2(M, (uint64_t)w | ((uint64_t)s << 6) | ((uint64_t)vb << 12)));
        if constexpr (HASH) __stcs(reinterpret_cast<unsigned long long *>(A.out_S) + j, (unsigned long long)S);
    }
};

// Warp-aggregated event slots (heads, items): the warp takes blocks of 256 slots with one
// atomic and marks the unused rest of a block (mark(q)) before the next or at the end.
struct EvBlk {
    unsigned long long next = 0, end = 0;
    template <class Mark>
    __device__ __forceinline__ unsigned long long take(uint32_t bal, unsigned long long *ctr, unsigned long long cap,
                                                       unsigned int *ovf, Mark mark) {
        const uint32_t need = __popc(bal);
        const unsigned lane = threadIdx.x & 31;
        if (next + need > end) {
            for (unsigned long long q = next + lane; q < end; q += 32)
                if (q < cap) mark(q);
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(ctr, 256ull);
            b = __shfl_sync(0xffffffffu, b, 0);
            next = b;
            end = b + 256;
            if (b + 256 > cap && lane == 0) atomicOr(ovf, 2u);
        }
        const unsigned long long q = next + __popc(bal & ((1u << lane) - 1u));
        next += need;
        return q;
    }
    template <class Mark>
    __device__ __forceinline__ void close(unsigned long long cap, Mark mark) {
        for (unsigned long long q = next + (threadIdx.x & 31); q < end; q += 32)
            if (q < cap) mark(q);
        next = end;
    }
};

__device__ __forceinline__ void put_head(const FrontierArgs &A, EvBlk &hb, bool hd, uint64_t S, uint32_t len,
                                         int32_t slot) {
    const uint32_t bal = __ballot_sync(0xffffffffu, hd);
    if (!bal) return;
    const unsigned long long q = hb.take(bal, A.hcnt, A.head_cap, A.overflow, [&](unsigned long long i) { A.heads[i].x = -1; });
    if (hd && q < A.head_cap) {
        HeadS h;
        h.S = S;
        h.len = (int32_t)len;
        h.x = slot;
        *reinterpret_cast<ulonglong2 *>(A.heads + q) = *reinterpret_cast<const ulonglong2 *>(&h);
    }
}
__device__ __forceinline__ void put_item(const FrontierArgs &A, EvBlk &ib, bool it, uint64_t S, uint64_t B,
                                         uint32_t len, int32_t x, int32_t ent, int32_t last) {
    const uint32_t bal = __ballot_sync(0xffffffffu, it);
    if (!bal) return;
    const unsigned long long q = ib.take(bal, A.hcnt + 1, A.item_cap, A.overflow, [&](unsigned long long i) { A.items[i].ent = -1; });
    if (it && q < A.item_cap) {
        ulonglong2 *d = reinterpret_cast<ulonglong2 *>(A.items + q);
        d[0] = make_ulonglong2(S, B);
        d[1] = make_ulonglong2((unsigned long long)len | ((unsigned long long)(uint32_t)x << 32),
                               (unsigned long long)(uint32_t)ent | ((unsigned long long)(uint32_t)last << 32));
    }
}

// Roots: one record per start vertex (a child record only if the start has an in-SCC successor).
// The root's own event: without arcs leaving SCCs an isolated vertex is itself a prime path;
// with them (HX) a non-entry start is a prime path when it has no arc at all, a head <s> when
// it is an exit whose predecessors lie on <s>; segment phase (SEG, entry starts): a tail <s>
// (no successor but itself) or a transit <s> (an exit).
template <class T, bool HASH, bool HX = false, bool SEG = false>
__global__ void frontier_root_kernel(FrontierArgs A, const int32_t *root_slot, const int32_t *root_vb, int32_t n) {
    FAcc f;
    unsigned int write = 0;
    uint32_t s = 0, vb = 0;
    uint64_t S = 0, B = 0;
    bool hd = false, it = false, ex = false;
    int32_t slot = 0, gid = 0;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        slot = root_slot[i];
        vb = (uint32_t)root_vb[i];
        const FSlot<T> t = static_cast<const FSlot<T> *>(A.tab)[slot];
        s = (uint32_t)slot - vb;
        gid = t.gid;
        const T sbit = (T)1 << s;
        const uint64_t m = mix64((uint64_t)(uint32_t)t.gid);  // position 0 (weight 1)
        S = (HASH || HX || SEG) ? m : 0ull;
        B = m;
        ex = (HX || SEG) && (t.flags & F_EXIT);
        if constexpr (SEG) {
            it = ex || (t.sin & ~sbit) == 0;
        } else {
            if (t.sin == 0 && !ex && (!HX || t.pin == 0)) {
                if constexpr (HASH) f.emit(S, 1);
                else f.pp++, f.vert++;
            }
            hd = HX && ex && (t.pin & ~sbit) == 0;
        }
        write = t.sin != 0;
    }
    if constexpr (HX && !SEG) {
        EvBlk hb;
        put_head(A, hb, hd, S, 1, slot);
        hb.close(A.head_cap, [&](unsigned long long q) { A.heads[q].x = -1; });
    }
    if constexpr (SEG) {
        EvBlk ib;
        put_item(A, ib, it, S, B, 1, ex ? slot : -1, gid, slot);
        ib.close(A.item_cap, [&](unsigned long long q) { A.items[q].ent = -1; });
    }
    const unsigned int lane = threadIdx.x & 31;
    const unsigned int bal = __ballot_sync(0xffffffffu, write);
    unsigned long long base = 0;
    if (lane == 0 && bal) base = atomicAdd(A.cnt_out, (unsigned long long)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (write) {
        const unsigned long long j = base + __popc(bal & ((1u << lane) - 1u));
        if (j < A.cap) {
            FT<T>::template st<HASH || HX || SEG>(A, j, (T)1 << s, s, s, vb, S);
            if constexpr (SEG) A.out_B[j] = B;
        } else {
            atomicOr(A.overflow, 1u);
        }
    }
    f.flush(A.acc);
}

// One level: every record of level l, every untried child.  Persistent grid;
// a block takes tiles of kFTile records (kFRec per thread, coalesced per k) and
// reserves the tile's surviving children with ONE atomicAdd (block scan): the
// record counter is a single address, and one atomic per warp serialised there
// (1.5 atomics/ns measured: a warp-per-atomic level kernel ran at 1.1 TB/s).
// TS: slot table in shared memory as {sin, pin, mix(gid) * (2(l+1)+1), flags} -- the
// digest term of a vertex at this level's position is computed once per block.
// HX (arcs leave SCCs): an exit child is never an internal prime path; an exit child whose
// start's predecessors lie on the path is a head segment (HeadS).  SEG (the
// segment phase, entry starts): cycles are prime paths when the start lies in the call's range,
// tail / transit segments become ItemS records, the records also carry B = sum of mix(v).
constexpr int kFThreads = 256;
constexpr int kFRec = 4;
constexpr int kFTile = kFThreads * kFRec;

template <class T>
struct FSm {  // shared-memory slot entry
    T sin, pin;
    uint64_t mix;    // digest term of the vertex at position l+1: mix64(gid) * (2(l+1) + 1)
    int32_t flags;   // F_EXIT, bit 2: the start vertex lies in the call's range (segment phase)
    int32_t pad;
};

template <class T, bool TS, bool HASH, bool HX, bool SEG>
__device__ __forceinline__ void frontier_level_body(const FrontierArgs &A, FAcc &f, unsigned int vblk) {
    constexpr bool NEED_S = HASH || HX || SEG;  // heads and items carry their digest sums
    extern __shared__ int4 fsm[];
    FSm<T> *st = reinterpret_cast<FSm<T> *>(fsm);
    const FSlot<T> *tab = static_cast<const FSlot<T> *>(A.tab);
    __shared__ uint32_t wsum[2][kFThreads / 32];
    __shared__ unsigned long long bbase[2];
    __shared__ uint64_t pqs[kFThreads / 32][64];  // per warp: digest sums S of prime paths awaiting their hash
    const uint64_t pw = pos_weight((uint32_t)(A.l + 1));  // digest weight of the new vertex's position
    const unsigned long long n_in = min(min(A.cnt_in ? *A.cnt_in : ~0ull, A.cap), A.lim);
    if ((unsigned long long)vblk * kFTile >= n_in) return;
    if constexpr (TS) {
        for (int i = threadIdx.x; i < A.n_tab; i += blockDim.x) {
            const FSlot<T> t = tab[i];
            const int32_t inr = (t.gid >= A.shard_lo && t.gid < A.shard_hi) ? 4 : 0;
            st[i] = FSm<T>{t.sin, t.pin, mix64((uint64_t)(uint32_t)t.gid) * pw, t.flags | inr, 0};
        }
        __syncthreads();
    }
    auto sinof = [&](uint32_t i) -> T {
        if constexpr (TS) return st[i].sin;
        else return __ldg(&tab[i].sin);
    };
    auto pinof = [&](uint32_t i) -> T {
        if constexpr (TS) return st[i].pin;
        else return __ldg(&tab[i].pin);
    };
    auto mixof = [&](uint32_t i) -> uint64_t {
        if constexpr (TS) return st[i].mix;
        else return mix64((uint64_t)(uint32_t)__ldg(&tab[i].gid)) * pw;
    };
    auto flagsof = [&](uint32_t i) -> int32_t {
        if constexpr (TS) return st[i].flags;
        const int32_t g = __ldg(&tab[i].gid);
        return __ldg(&tab[i].flags) | ((g >= A.shard_lo && g < A.shard_hi) ? 4 : 0);
    };
    const unsigned int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t len = (uint32_t)A.l + 2;  // vertices of a child path (every prime path found at this level)
    uint64_t *pq = pqs[warp];
    uint32_t qn = 0;  // queued prime paths (warp-uniform, < 32 between drains)
    EvBlk hblk, iblk;
    int par = 0;
    for (unsigned long long t0 = (unsigned long long)vblk * kFTile; t0 < n_in;
         t0 += (unsigned long long)gridDim.x * kFTile, par ^= 1) {
        T M[kFRec], keep[kFRec];
        uint32_t sv[kFRec], vb[kFRec];
        uint64_t S[kFRec], Bv[kFRec];
        ulonglong2 r[kFRec];
#pragma unroll
        for (int k = 0; k < kFRec; k++) {  // all loads first: kFRec records in flight per thread
            const unsigned long long i = t0 + k * kFThreads + threadIdx.x;
            S[k] = 0;
            Bv[k] = 0;
            r[k] = i < n_in ? FT<T>::template ld<NEED_S>(A, i, S[k]) : make_ulonglong2(0, 0);
            if constexpr (SEG) Bv[k] = i < n_in ? __ldcs(reinterpret_cast<const unsigned long long *>(A.in_B) + i) : 0ull;
        }
        uint32_t nk = 0;
#pragma unroll
        for (int k = 0; k < kFRec; k++) {
            const unsigned long long i = t0 + k * kFThreads + threadIdx.x;
            uint32_t u, s;
            FT<T>::dec(r[k], M[k], u, s, vb[k]);
            sv[k] = s;
            keep[k] = 0;
            T cc = 0;
            bool head_closed = false, emit = true;
            const T sbit = (T)1 << s;
            T ps = 0;
            if (i < n_in) {
                cc = sinof(vb[k] + u) & (~M[k] | sbit);
                ps = pinof(vb[k] + s);
                head_closed = (ps & ~M[k]) == 0;  // pred(s) within M = M' \ {w}
                if constexpr (SEG) emit = (flagsof(vb[k] + s) & 4) != 0;
                if (emit) f.ext += FT<T>::popc(cc);
            }
            // warp-uniform child loop; prime paths are queued and hashed 32 at a time
            const int maxc = (int)__reduce_max_sync(0xffffffffu, (unsigned)FT<T>::popc(cc));
            for (int it = 0; it < maxc; it++) {
                bool em = false, hd = false, itm = false, ex = false;
                uint64_t Sx = 0, Bx = 0;
                int32_t wsl = 0;
                if (cc) {
                    const uint32_t w = FT<T>::ffs(cc) - 1;
                    cc &= cc - 1;
                    const T wb = (T)1 << w;
                    const bool clo = w == s;
                    const T snw = clo ? (T)0 : sinof(vb[k] + w);
                    const T cw = snw & (~(M[k] | wb) | sbit);
                    if constexpr (HX || SEG) ex = (flagsof(vb[k] + w) & F_EXIT) != 0;
                    if (cw) keep[k] |= wb;
                    if constexpr (SEG) {
                        em = clo && emit;
                        itm = !clo && (ex || (snw & ~(M[k] | wb)) == 0);  // transit, or tail (R8, R9)
                    } else {
                        em = !cw && (clo || (head_closed && !ex));  // cycle closure, or an internal prime path
                        hd = HX && !clo && ex && (ps & ~(M[k] | wb)) == 0;
                    }
                    wsl = (int32_t)(vb[k] + w);
                    if constexpr (NEED_S) Sx = S[k] + mixof(vb[k] + w);
                    if constexpr (SEG) Bx = Bv[k] + __ldg(A.slot_mix + vb[k] + w);
                }
                if constexpr (!HASH) {  // counts only
                    if (em) f.pp++, f.vert += len;
                } else {
                    const uint32_t bal = __ballot_sync(0xffffffffu, em);
                    if (em) pq[qn + __popc(bal & lt)] = Sx;
                    qn += __popc(bal);
                    if (qn >= 32) {
                        __syncwarp();
                        qn -= 32;
                        f.emit(pq[qn + lane], len);
                        __syncwarp();
                    }
                }
                if constexpr (HX && !SEG) put_head(A, hblk, hd, Sx, len, wsl);
                if constexpr (SEG)
                    put_item(A, iblk, itm, Sx, Bx, len, ex ? wsl : -1, __ldg(&tab[vb[k] + s].gid), wsl);
            }
            nk += FT<T>::popc(keep[k]);
        }
        // block compaction: warp scans, one atomicAdd per tile
        uint32_t inc = nk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (unsigned)o) inc += t;
        }
        if (lane == 31) wsum[par][warp] = inc;
        __syncthreads();
        uint32_t woff = 0, btot = 0;
#pragma unroll
        for (int x = 0; x < kFThreads / 32; x++) {
            const uint32_t v = wsum[par][x];
            woff += (x < (int)warp) ? v : 0u;
            btot += v;
        }
        if (threadIdx.x == 0) bbase[par] = btot ? atomicAdd(A.cnt_out, (unsigned long long)btot) : 0ull;
        __syncthreads();
        const unsigned long long bb = bbase[par];
        if (btot) {
            if (bb + btot > A.cap) {
                if (threadIdx.x == 0) atomicOr(A.overflow, 1u);
            } else {
                unsigned long long j = bb + woff + (inc - nk);
#pragma unroll
                for (int k = 0; k < kFRec; k++) {
                    T kp = keep[k];
                    while (kp) {
                        const uint32_t w = FT<T>::ffs(kp) - 1;
                        kp &= kp - 1;
                        uint64_t Sw = 0;
                        if constexpr (NEED_S) Sw = S[k] + mixof(vb[k] + w);
                        unsigned long long jj = j;  // ring buffer (the chunked walk): wrap the append index
                        if (A.ring) {
                            jj += A.ring_off;
                            if (jj >= A.ring) jj -= A.ring;
                        }
                        FT<T>::template st<NEED_S>(A, jj, M[k] | ((T)1 << w), w, sv[k], vb[k], Sw);
                        if constexpr (SEG) A.out_B[jj] = Bv[k] + __ldg(A.slot_mix + vb[k] + w);
                        j++;
                    }
                }
            }
        }
    }
    __syncwarp();
    if (HASH && lane < qn) f.emit(pq[lane], len);  // the queue's remainder
    if constexpr (HX && !SEG) hblk.close(A.head_cap, [&](unsigned long long q) { A.heads[q].x = -1; });
    if constexpr (SEG) iblk.close(A.item_cap, [&](unsigned long long q) { A.items[q].ent = -1; });
}

// Block reduction of the accumulators, one set of atomics per block.
__device__ __forceinline__ void frontier_flush(const FrontierArgs &A, const FAcc &f) {
    __shared__ unsigned long long red[5][kFThreads / 32];
    const unsigned int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long v[5] = {f.pp, f.vert, f.ext, f.ha, f.hb};
#pragma unroll
    for (int q = 0; q < 5; q++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
        if (lane == 0) red[q][warp] = v[q];
    }
    __syncthreads();
    if (threadIdx.x < 5) {
        unsigned long long a = 0;
#pragma unroll
        for (int x = 0; x < kFThreads / 32; x++) a += red[threadIdx.x][x];
        if (a || threadIdx.x >= 3) atomicAdd(A.acc + threadIdx.x, a);
    }
}

template <class T, bool TS, bool HASH, bool HX = false, bool SEG = false>
__global__ void __launch_bounds__(kFThreads) frontier_level_kernel(FrontierArgs A) {
    // once a level has overflowed the attempt is discarded (the call retries bigger or goes
    // chunked): the buffer holds unwritten gaps, so no later level reads it
    if (*reinterpret_cast<volatile const unsigned int *>(A.overflow) & 1u) return;
    const unsigned long long n_in = min(min(*A.cnt_in, A.cap), A.lim);
    if ((unsigned long long)blockIdx.x * kFTile >= n_in) return;  // small levels: idle blocks leave at once
    FAcc f;
    frontier_level_body<T, TS, HASH, HX, SEG>(A, f, blockIdx.x);
    frontier_flush(A, f);
}

// DFS-chunked frontier, scheduled on the device: a CUDA graph whose
// conditional WHILE node runs [frontier_sched_kernel -> frontier_chunk_kernel] until the walk
// over chunks of levels ends, so no chunk waits for a host round trip.  FChunk is the walk's
// state (cur / nl: records consumed / produced per level) plus the next chunk's parameters.
constexpr int kFMaxLevels = 66;  // levels 0..64 (masks of <= 64 vertices) + 1
struct FChunk {
    const ulonglong2 *in;
    const uint64_t *in_S;
    ulonglong2 *out;
    uint64_t *out_S;
    unsigned long long lim;     // records of level l to process
    int32_t l;                  // the chunk's level
    int32_t done;               // the walk has ended (the body's level launch returns at once)
    int32_t started;
    int32_t pad;
    unsigned long long steps;   // chunks scheduled
    unsigned long long recs;    // records written over all levels
    unsigned long long cur[kFMaxLevels], nl[kFMaxLevels];
    unsigned long long oc[3][kFMaxLevels];  // persistent walk: step t's appends to level l: oc[t % 3][l]
    unsigned long long bar;     // persistent walk: grid-barrier arrivals
};
struct FSchedArgs {
    FChunk *c;
    unsigned long long *ctr;    // ctr[8 + l]: records written to level l's buffer
    ulonglong2 *base;           // level l's key array at base + l * capc (16-byte stride)
    uint64_t *baseS;            // level l's S array at baseS + l * capc (64-bit masks)
    uint64_t *baseB;            // segment pass: level l's B array at baseB + l * capc
    unsigned long long capc;    // records per level buffer
    unsigned long long chunk;   // records per chunk (capc / the largest out-degree)
    unsigned long long chunk_div;  // the largest out-degree D (a chunk of k records has <= k * D children)
    uint32_t key_b;             // bytes per record in the key array (8: u32 masks, counts only)
    int32_t Lmax;
};

// One thread: account for the chunk that just ran, pick the next one (the deepest level with
// unconsumed records), or end the while loop.
__global__ void frontier_sched_kernel(FSchedArgs a, cudaGraphConditionalHandle h) {
    if (threadIdx.x != 0) return;
    FChunk &c = *a.c;
    int l;
    if (!c.started) {
        c.started = 1;
        c.nl[0] = a.ctr[8];
        c.cur[0] = 0;
        c.recs = c.nl[0];
        l = 0;
    } else {
        l = c.l;
        c.cur[l] += c.lim;
        if (l + 1 < a.Lmax) {  // level l+1's records can have children: descend
            c.nl[l + 1] = a.ctr[8 + l + 1];
            c.cur[l + 1] = 0;
            c.recs += c.nl[l + 1];
            l++;
        }
    }
    while (l >= 0 && c.cur[l] >= c.nl[l]) l--;
    if (l < 0) {
        c.done = 1;
        cudaGraphSetConditional(h, 0);
        return;
    }
    const unsigned long long k = min(c.nl[l] - c.cur[l], a.chunk);
    a.ctr[8 + l + 1] = 0;
    c.in = reinterpret_cast<const ulonglong2 *>(reinterpret_cast<const char *>(a.base + (size_t)l * a.capc) +
                                                c.cur[l] * a.key_b);
    c.in_S = a.baseS + (size_t)l * a.capc + c.cur[l];
    c.out = a.base + (size_t)(l + 1) * a.capc;
    c.out_S = a.baseS + (size_t)(l + 1) * a.capc;
    c.lim = k;
    c.l = l;
    c.steps++;
}

// The level kernel on the chunk FChunk names (cnt_in = ctr[8 + l] >= lim, so lim bounds it).
template <class T, bool TS, bool HASH>
__global__ void __launch_bounds__(kFThreads) frontier_chunk_kernel(FrontierArgs A, const FChunk *c) {
    const FChunk *cv = c;
    if (*reinterpret_cast<volatile const int32_t *>(&cv->done)) return;
    FrontierArgs B = A;
    B.in = cv->in;
    B.in_S = cv->in_S;
    B.out = cv->out;
    B.out_S = cv->out_S;
    B.lim = cv->lim;
    B.l = cv->l;
    B.cnt_in = A.acc + 8 + B.l;
    B.cnt_out = A.acc + 8 + B.l + 1;
    if ((unsigned long long)blockIdx.x * kFTile >= B.lim) return;
    FAcc f;
    frontier_level_body<T, TS, HASH, false, false>(B, f, blockIdx.x);
    frontier_flush(A, f);
}

// The DFS-chunked frontier as ONE persistent launch (grid = the co-resident blocks), a
// wavefront over the levels: in each step EVERY level with pending records takes a chunk of
// them -- as many as its child level's free space / D guarantees room for (D = the largest
// out-degree) -- so the walk needs about (records / buffer space) steps, not one step per chunk
// of one level.  Level l's buffer is filled from its start (tail[l]) and consumed in order
// (head[l]); an empty buffer restarts at 0.  The deepest level with pending records always has
// an empty (restarted) child buffer, so every step makes progress.  Every block keeps its own
// copy of head / tail and takes the same decisions from the same counters; a step ends at a
// grid barrier.  Step t's appends to level l are counted in oc[t % 3][l]; block 0 zeroes
// oc[(t + 1) % 3] during step t (last read right after the barrier that ended step t - 2).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <class T, bool TS, bool HASH, bool HX = false, bool SEG = false>
__global__ void __launch_bounds__(kFThreads) frontier_walk_kernel(FrontierArgs A, FSchedArgs sa) {
    __shared__ unsigned long long head[kFMaxLevels], tail[kFMaxLevels], take[kFMaxLevels];
    __shared__ unsigned long long s_cnt[kFMaxLevels];
    FChunk *c = sa.c;
    const int Lm = sa.Lmax;
    for (int i = threadIdx.x; i < kFMaxLevels; i += blockDim.x) head[i] = tail[i] = take[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) tail[0] = *reinterpret_cast<volatile unsigned long long *>(sa.ctr + 8);
    __syncthreads();
    unsigned long long recs = tail[0], step = 0;
    FAcc f;  // accumulated over all steps, flushed once
    for (;;) {
        // plan the step (thread 0; the same decisions in every block).  head / tail count records
        // consumed / appended since the start; a level's buffer is a ring of capc records.
        if (threadIdx.x == 0) {
            bool any = false;
            for (int l = 0; l < Lm; l++) {
                const unsigned long long pend = tail[l] - head[l];
                any |= pend != 0;
                unsigned long long k = min(pend, sa.capc - head[l] % sa.capc);  // (a chunk does not wrap)
                if (l + 1 < Lm) k = min(k, (sa.capc - (tail[l + 1] - head[l + 1])) / sa.chunk_div);
                take[l] = k;
            }
            take[kFMaxLevels - 1] = any;
        }
        __syncthreads();
        if (!take[kFMaxLevels - 1]) break;
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < kFMaxLevels; i += blockDim.x) c->oc[(step + 1) % 3][i] = 0;
        unsigned int rot = 0;  // tiles of the step's earlier levels: level l's first tile goes to the next block
        for (int l = 0; l < Lm; l++) {
            const unsigned long long k = take[l];
            if (k == 0) continue;
            const unsigned int vblk = (blockIdx.x + gridDim.x - rot % gridDim.x) % gridDim.x;
            rot += (unsigned int)((k + kFTile - 1) / kFTile);
            if ((unsigned long long)vblk * kFTile >= k) continue;  // no tile of this level for this block
            FrontierArgs B = A;
            const unsigned long long h0 = head[l] % sa.capc;
            B.in = reinterpret_cast<const ulonglong2 *>(reinterpret_cast<const char *>(sa.base + (size_t)l * sa.capc) +
                                                        h0 * sa.key_b);
            B.in_S = sa.baseS + (size_t)l * sa.capc + h0;
            // (level Lm - 1 has no children: level Lm's buffer is never written)
            B.out = sa.base + (size_t)(l + 1) * sa.capc;
            B.out_S = sa.baseS + (size_t)(l + 1) * sa.capc;
            if constexpr (SEG) {
                B.in_B = sa.baseB + (size_t)l * sa.capc + h0;
                B.out_B = sa.baseB + (size_t)(l + 1) * sa.capc;
            }
            B.ring = sa.capc;
            B.ring_off = tail[l + 1] % sa.capc;
            B.cap = sa.capc - (tail[l + 1] - head[l + 1]);  // free records of the ring
            B.lim = k;
            B.l = l;
            B.cnt_in = nullptr;  // (lim bounds the input)
            B.cnt_out = &c->oc[step % 3][l + 1];
            frontier_level_body<T, TS, HASH, HX, SEG>(B, f, vblk);
            __syncthreads();  // (the body's shared memory is reused by the next level)
        }
        // grid barrier: every block's children of this step are written and counted
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(&c->bar, 1ull);
            const unsigned long long target = (unsigned long long)gridDim.x * (step + 1);
            while (ld_acquire_u64(&c->bar) < target) __nanosleep(32);
        }
        __syncthreads();
        for (int i = threadIdx.x; i <= Lm; i += blockDim.x)
            s_cnt[i] = *reinterpret_cast<volatile unsigned long long *>(&c->oc[step % 3][i]);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int l = 0; l < Lm; l++) {
                head[l] += take[l];
                if (l + 1 < Lm) tail[l + 1] += s_cnt[l + 1];
            }
        for (int l = 1; l < Lm; l++) recs += s_cnt[l];
        step++;
        __syncthreads();
    }
    frontier_flush(A, f);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c->recs = recs;
        c->steps = step;
    }
}

}  // namespace tpg
