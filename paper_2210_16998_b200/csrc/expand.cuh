// expand.cuh -- canonical writer (K4) of libtpgen: replays the per-unit
// path-delta record streams written by dfs_kernel into the canonical
// offsets/vertices arrays, head records (cross-SCC
// blocks, filled later by stitch_kernel) and segment items (a5).
//
// One warp per unit.  Two kernels:
//
//  expand_fast_kernel<NPW> (every SCC has at most 31 vertices, so a path fits
//  in NPW <= 8 32-bit words of local ids): the warp takes 32 records at a time,
//  lane j owning record j.  Each lane turns its record into the bytes it writes
//  (positions c..c+n-1) plus a byte mask, and an inclusive warp scan whose
//  operator is "later record overwrites earlier bytes" gives every lane the full
//  path of its record (bytes no record of the batch wrote come from the path the
//  previous batch ended with).  Emitting lanes place their paths in a per-warp
//  shared-memory stage at offsets from a warp scan of their lengths, and the
//  warp streams the stage to HBM with coalesced stores.  Batches that contain
//  other record kinds (segment items, head blocks; they occur only at SCC exits)
//  are emitted lane-parallel too: warp scans of the cursor increments give each
//  lane the offsets of its own record, which it writes directly.
//
//  expand_kernel<W, NP> (any SCC size): sequential replay, the current path
//  distributed over the lanes' registers (lane q holds positions q, q+32, ...);
//  records are fetched 32 at a time and broadcast by shuffle.
#pragma once

#include "dfs.cuh"

namespace tpg {

struct ExpandArgs {
    DevGraph G;
    const void *units;  // Unit<W>[n_units]
    int64_t n_units;
    const int64_t *rfirst;
    const int64_t *rcount;
    const LinNode *off;  // canonical exclusive offsets of each unit's outputs
    const uint64_t *chunks;
    int64_t *out_off;
    int32_t *out_vert;
    HeadRec *heads;
    int32_t *head_pool;
    ItemRec *items;
    int32_t *item_pool;
    unsigned long long *hash_acc;  // HASH kernels: digest of the prime paths instead of writing them
    uint64_t lim[C_NUM];           // totals of the call (debug-build bounds checks)
};

constexpr int kExpandThreads = 256;

__device__ __forceinline__ void st_global_cs(int32_t *p, int v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// TMA bulk copy shared -> global (cp.async.bulk, SASS UBLKCP): 16-byte aligned ends, a
// multiple of 16 bytes; tracked in bulk groups of the issuing thread.
__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, uint32_t bytes) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(ssrc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(s), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the bulk groups issued before the last `n` have finished reading their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (the bulk copy's reads)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Output cursors of one unit (canonical exclusive offsets, advanced as records are replayed).
struct Cursor {
    uint64_t pp, vv, it, itv, hd, hdv;
    int arg;  // out-arc of the pending HEAD / TRANSIT (from the R_ARG record before it)
};

__device__ __forceinline__ Cursor unit_cursor(const ExpandArgs &A, int64_t u) {
    const LinNode *on = A.off + u;
    Cursor cu;
    cu.pp = on->v[C_PP];
    cu.vv = on->v[C_VERT];
    cu.it = on->v[C_ITEMS];
    cu.itv = on->v[C_ITEMV];
    cu.hd = on->v[C_HEADS];
    cu.hdv = on->v[C_HEADV];
    cu.arg = -1;
    return cu;
}

// Record stream reader: 32 records per fetch (lane j gets record r0 + j).
struct RecReader {
    const uint64_t *ch;  // current chunk
    int slot;            // next record slot in it
    int64_t left;        // records of the unit not yet fetched
    uint64_t link;       // the current chunk's link word, loaded when the reader entered the chunk (if the
                         // unit continues past it), so crossing into the next chunk is one load, not two
};

// PREF = false (HASH kernels, short of registers): the link word is read when the chunk is crossed.
template <bool PREF = true>
__device__ __forceinline__ RecReader rec_reader(const ExpandArgs &A, int64_t rfirst, int64_t nrec) {
    RecReader rd;
    rd.ch = A.chunks + (rfirst & ~(int64_t)(kChunkRecs - 1));
    rd.slot = (int)(rfirst & (kChunkRecs - 1));
    rd.left = nrec;
    rd.link = (PREF && rd.slot + nrec > kChunkRecs - 1) ? rd.ch[kChunkRecs - 1] : 0ull;
    return rd;
}

template <bool PREF = true>
__device__ __forceinline__ uint64_t fetch32(const ExpandArgs &A, RecReader &rd, int nb, int lane) {
    const bool cross = rd.slot + nb >= kChunkRecs - 1;
    // the next chunk (its address is only followed when the unit has records beyond this one)
    const uint64_t *nxt = cross ? A.chunks + (PREF ? rd.link : rd.ch[kChunkRecs - 1]) * kChunkRecs : rd.ch;
    uint64_t myrec = 0;
    if (lane < nb) {
        const int sj = rd.slot + lane;
        myrec = (sj < kChunkRecs - 1) ? rd.ch[sj] : nxt[sj - (kChunkRecs - 1)];
    }
    if (PREF) rd.left -= nb;
    if (cross) {
        rd.slot = rd.slot + nb - (kChunkRecs - 1);
        rd.ch = nxt;
        if (PREF && rd.slot + rd.left > kChunkRecs - 1) rd.link = nxt[kChunkRecs - 1];  // prefetch the next link
    } else {
        rd.slot += nb;
    }
    return myrec;
}

// Sequential replay of one record (warp-uniform `rec`); P = the current path
// distributed over the lanes (lane q holds positions q + 32 r).
template <int NP, bool HASH>
__device__ __forceinline__ void replay_one(const ExpandArgs &A, uint64_t rec, int (&P)[NP], Cursor &cu, int lane,
                                           int ga, int vb, int sgid, PathHash &acc) {
    const DevGraph &G = A.G;
    const int ty = (int)(rec & 7);
    if (ty == R_ARG) {
        cu.arg = (int)(rec >> 32);
        return;
    }
    const int cc = (int)((rec >> 4) & 0x1ff);
    const int n = (int)((rec >> 13) & 7);
#pragma unroll
    for (int r = 0; r < NP; r++) {
        const int d = lane + 32 * r - cc;
        if (d >= 0 && d < n) P[r] = (int)((rec >> (16 + 8 * d)) & 0xff);
    }
    if (ty == R_PATH) return;
    const int len = cc + n;
    const int tot = len + (int)((rec >> 3) & 1);
    int32_t *dst;
    if (HASH && ty == R_PP) {  // digest only (R20): lane q adds the terms of positions q + 32 r, one warp sum
        const int s0 = __shfl_sync(kFull, P[0], 0);
        uint64_t part = 0;
#pragma unroll
        for (int r = 0; r < NP; r++) {
            const int pos = lane + 32 * r;
            if (pos < tot) part += __ldg(G.slot_mix + vb + ((pos < len) ? P[r] : s0)) * (2ull * (uint64_t)pos + 1ull);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
        if (lane == 0) {
            acc.a += mix64(part ^ (kSeedA + (uint64_t)tot));
            acc.b += mix64(part ^ (kSeedB + (uint64_t)tot));
        }
        cu.pp += 1;
        cu.vv += (uint64_t)tot;
        return;
    }
    if (ty == R_PP) {
        TPG_DCHECK(cu.pp < A.lim[C_PP] && cu.vv + tot <= A.lim[C_VERT], "replay: prime path out of range");
        dst = A.out_vert + cu.vv;
        if (lane == 0) A.out_off[cu.pp] = (int64_t)cu.vv;
        cu.pp += 1;
        cu.vv += (uint64_t)tot;
    } else if (ty == R_HEAD) {
        TPG_DCHECK(cu.arg >= 0 && cu.hd < A.lim[C_HEADS] && cu.hdv + len <= A.lim[C_HEADV], "replay: head out of range");
        const int32_t x = __ldg(G.out_gid + cu.arg);
        dst = A.head_pool + cu.hdv;
        if (lane == 0) {
            HeadRec hr;
            hr.pp_off = cu.pp;
            hr.v_off = cu.vv;
            hr.hv_off = cu.hdv;
            hr.len = len;
            hr.x = x;
            A.heads[cu.hd] = hr;
        }
        const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
        cu.pp += Wx;
        cu.vv += (uint64_t)len * Wx + Vx;
        cu.hd += 1;
        cu.hdv += (uint64_t)len;
    } else {  // R_TAIL / R_TRANSIT
        TPG_DCHECK(cu.it < A.lim[C_ITEMS] && cu.itv + len <= A.lim[C_ITEMV], "replay: item out of range");
        dst = A.item_pool + cu.itv;
        if (lane == 0) {
            ItemRec ir;
            ir.pool_off = (int64_t)cu.itv;
            ir.len = len;
            ir.y = (ty == R_TRANSIT) ? __ldg(G.out_gid + cu.arg) : -1;
            ir.ent = sgid;
            ir.pad = 0;
            A.items[cu.it] = ir;
        }
        cu.it += 1;
        cu.itv += (uint64_t)len;
    }
    const int s0 = __shfl_sync(kFull, P[0], 0);  // closing vertex of a cycle
    if (ga >= 0) {  // SCC with contiguous global ids (warp-uniform branch)
#pragma unroll
        for (int r = 0; r < NP; r++) {
            const int pos = lane + 32 * r;
            if (pos < tot) st_global_cs(dst + pos, ga + ((pos < len) ? P[r] : s0));
        }
    } else {
#pragma unroll
        for (int r = 0; r < NP; r++) {
            const int pos = lane + 32 * r;
            if (pos < tot) st_global_cs(dst + pos, __ldg(G.slot_gid + vb + ((pos < len) ? P[r] : s0)));
        }
    }
}

// NP = path registers per lane: ceil((longest emitted path + closing vertex) / 32).
__device__ __forceinline__ void flush_hash(const ExpandArgs &A, PathHash &acc) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        acc.a += __shfl_xor_sync(kFull, acc.a, d);
        acc.b += __shfl_xor_sync(kFull, acc.b, d);
    }
    if ((threadIdx.x & 31) == 0 && (acc.a | acc.b)) {
        atomicAdd(A.hash_acc, (unsigned long long)acc.a);
        atomicAdd(A.hash_acc + 1, (unsigned long long)acc.b);
    }
}

template <int W, int NP, bool HASH>
__global__ void __launch_bounds__(kExpandThreads) expand_kernel(ExpandArgs A) {
    const int lane = threadIdx.x & 31;
    const DevGraph &G = A.G;
    const Unit<W> *units = reinterpret_cast<const Unit<W> *>(A.units);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;

    PathHash acc{0, 0, 0, 0, 0};
    for (int64_t u = gw; u < A.n_units; u += nw) {
        const Unit<W> *U = units + u;
        const int4 h = *reinterpret_cast<const int4 *>(&U->scc);
        const int depth = h.w & 0xff;
        int P[NP];
#pragma unroll
        for (int r = 0; r < NP; r++) {
            const int pos = lane + 32 * r;
            P[r] = (pos <= depth) ? U->path[pos] : 0;
        }
        const int vb = __ldg(G.scc_vbase + h.x);
        const int ga = __ldg(G.scc_gbase + h.x);
        const int sgid = __ldg(G.slot_gid + vb + __shfl_sync(kFull, P[0], 0));
        Cursor cu = unit_cursor(A, u);
        const int64_t nrec = A.rcount[u];
        RecReader rd = rec_reader(A, A.rfirst[u], nrec);
        for (int64_t r0 = 0; r0 < nrec; r0 += 32) {
            const int nb = (nrec - r0 < 32) ? (int)(nrec - r0) : 32;
            const uint64_t myrec = fetch32(A, rd, nb, lane);
            for (int i = 0; i < nb; i++)
                replay_one<NP, HASH>(A, __shfl_sync(kFull, myrec, i), P, cu, lane, ga, vb, sgid, acc);
        }
    }
    if (HASH) flush_hash(A, acc);
}

// ---------------------------------------------------------------- fast path
constexpr int kFastMaxScc = 63;  // a path of local ids fits NPW <= 16 32-bit words (W = 1 masks)

#ifndef EXP_MINB
#define EXP_MINB 4  // min resident blocks per SM of the fast writer (launch bounds; 64 registers at 256 threads)
#endif
#ifndef EXP_BUFS
#define EXP_BUFS 2  // bulk-store stages per warp
#endif
template <int NPW>
struct FastCfg {
    static constexpr int threads = (NPW > 8) ? 128 : 256;
    static constexpr int max_out = 4 * NPW + 1;  // output vertices per path (incl. the closing vertex)
    // ints per warp stage: HASH, each lane's path bytes; else one batch's vertices + the 16-byte phase shift
    static constexpr int stage_ints(bool hash) { return hash ? 32 * NPW : (32 * max_out + 4 + 3) / 4 * 4; }
    static constexpr size_t smem_bytes(bool hash) {
        return (size_t)(threads / 32) * (hash ? 1 : EXP_BUFS) * stage_ints(hash) * sizeof(int32_t);
    }
};

__device__ __forceinline__ uint32_t lop_merge(uint32_t mine, uint32_t other, uint32_t mask) {
    return (mine & mask) | (other & ~mask);  // one LOP3
}

// HASH mode: a lane's path digest.  The bytes go through the lane's slice of the
// warp's stage so that the per-vertex loop is a rolled loop (unrolled over up to
// 64 positions with two splitmix64 chains each, the kernel outgrows the
// instruction cache).
template <int NPW>
__device__ __forceinline__ void hash_path(const DevGraph &G, const uint32_t (&D)[NPW], int32_t *stage, int lane, int len,
                                          int tot, int ga, int vb, int s0g, PathHash &acc) {
    uint32_t *mine = reinterpret_cast<uint32_t *>(stage) + lane * NPW;
#pragma unroll
    for (int w = 0; w < NPW; w++)
        if (4 * w < len) mine[w] = D[w];
    const uint8_t *bytes = reinterpret_cast<const uint8_t *>(mine);
    uint64_t S = 0;  // R20: the terms from the per-slot mix table (no splitmix64 per vertex)
#pragma unroll 2
    for (int p = 0; p < len; p++) S += __ldg(G.slot_mix + vb + bytes[p]) * (2ull * (uint64_t)p + 1ull);
    if (len < tot) S += __ldg(G.slot_mix + vb + bytes[0]) * (2ull * (uint64_t)len + 1ull);  // the cycle's closing s
    acc.a += mix64(S ^ (kSeedA + (uint64_t)tot));
    acc.b += mix64(S ^ (kSeedB + (uint64_t)tot));
}

// MIXED = false: the call has no segment items and no head blocks (e.g. a graph
// that is one SCC), so every batch is prime paths and path continuations only.
template <int NPW, bool HASH, bool MIXED>
__global__ void __launch_bounds__(FastCfg<NPW>::threads, EXP_MINB) expand_fast_kernel(ExpandArgs A) {
    constexpr int kWarps = FastCfg<NPW>::threads / 32;
    // one batch of paths (HASH: each lane's path bytes, NPW words)
    // (!HASH: two stages per warp, each shifted by the output offset's alignment -- up to 3 ints --
    // so that the middle of a batch leaves with one TMA bulk store while the next batch is staged)
    constexpr int kStage = FastCfg<NPW>::stage_ints(HASH);
    constexpr int kBufs = HASH ? 1 : EXP_BUFS;
    extern __shared__ __align__(16) int32_t stage_dyn[];  // [kWarps][kBufs][kStage] (launch_fast sizes it)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t *const stage_w = stage_dyn + (size_t)wid * kBufs * kStage;
    int32_t *stage = stage_w;
    int sbuf = 0;  // the stage the next batch fills
    const DevGraph &G = A.G;
    const Unit<1> *units = reinterpret_cast<const Unit<1> *>(A.units);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    PathHash acc{0, 0, 0, 0, 0};

    // the next unit's header, record range and count are loaded one unit ahead
    int4 h_next = make_int4(0, 0, 0, 0);
    int64_t rf_next = 0, rc_next = 0;
    if (!HASH && gw < A.n_units) {
        h_next = *reinterpret_cast<const int4 *>(&units[gw].scc);
        rf_next = A.rfirst[gw];
        rc_next = A.rcount[gw];
    }
    for (int64_t u = gw; u < A.n_units; u += nw) {
        const Unit<1> *U = units + u;
        int4 h;
        int64_t rfirst, nrec;
        if (HASH) {  // (HASH kernels: registers are scarce; the digest chain bounds them, not latency)
            h = *reinterpret_cast<const int4 *>(&U->scc);
            rfirst = A.rfirst[u];
            nrec = A.rcount[u];
        } else {
            h = h_next;
            rfirst = rf_next;
            nrec = rc_next;
        }
        if (!HASH && u + nw < A.n_units) {
            h_next = *reinterpret_cast<const int4 *>(&units[u + nw].scc);
            rf_next = A.rfirst[u + nw];
            rc_next = A.rcount[u + nw];
        }
        // carry = the current path as bytes (positions 0..depth valid; the others are
        // always written by a record before an emitted path reads them)
        uint32_t carry[NPW];
        {
            const uint4 *p4 = reinterpret_cast<const uint4 *>(U->path);
#pragma unroll
            for (int q = 0; q < (NPW + 3) / 4; q++) {
                const uint4 v = p4[q];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; j++)
                    if (4 * q + j < NPW) carry[4 * q + j] = w4[j];
            }
        }
        const int vb = __ldg(G.scc_vbase + h.x);
        const int ga = __ldg(G.scc_gbase + h.x);
        const int s0 = (int)(carry[0] & 0xff);
        const int s0g = (ga >= 0) ? ga + s0 : __ldg(G.slot_gid + vb + s0);  // global id of the start vertex
        Cursor cu = unit_cursor(A, u);
        RecReader rd = rec_reader<!HASH>(A, rfirst, nrec);
        // records are fetched one batch ahead: the next batch's loads overlap this batch's work
        uint64_t nextrec = (nrec > 0) ? fetch32<!HASH>(A, rd, (nrec < 32) ? (int)nrec : 32, lane) : 0ull;
        for (int64_t r0 = 0; r0 < nrec; r0 += 32) {
            const int nb = (nrec - r0 < 32) ? (int)(nrec - r0) : 32;
            const uint64_t myrec = nextrec;  // lanes >= nb: 0 = an empty R_PATH
            if (r0 + 32 < nrec) nextrec = fetch32<!HASH>(A, rd, (nrec - r0 - 32 < 32) ? (int)(nrec - r0 - 32) : 32, lane);
            const int ty = (int)(myrec & 7);
            // ---- this lane's bytes: positions cc .. cc+n-1 of the path
            const int cc = (int)((myrec >> 4) & 0x1ff);
            const int n = (int)((myrec >> 13) & 7);
            const int sh = 8 * (cc & 3);
            const uint64_t nm = (1ull << (8 * n)) - 1ull;
            const uint64_t pay = ((myrec >> 16) & nm) << sh;
            const uint64_t pm = nm << sh;
            const int w0 = cc >> 2;
            uint32_t D[NPW], M[NPW];
#pragma unroll
            for (int w = 0; w < NPW; w++) {
                D[w] = (w == w0) ? (uint32_t)pay : ((w == w0 + 1) ? (uint32_t)(pay >> 32) : 0u);
                M[w] = (w == w0) ? (uint32_t)pm : ((w == w0 + 1) ? (uint32_t)(pm >> 32) : 0u);
            }
            const int len = cc + n;
            // Words below the batch's smallest common prefix are the carry's in every lane, and
            // words from the longest path on are never read: only [wlo, whi) take part
            // (warp-uniform bounds, so the skipped words cost a uniform branch each).
            const int wlo = __reduce_min_sync(kFull, (unsigned)(n > 0 ? cc : 4 * NPW)) >> 2;
            const int whi = (__reduce_max_sync(kFull, (unsigned)len) + 3) >> 2;
            // ---- inclusive scan: later records overwrite earlier bytes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int w = 0; w < NPW; w++) {
                    if (w >= wlo && w < whi) {
                        const uint32_t dn = __shfl_up_sync(kFull, D[w], o);
                        const uint32_t mn = __shfl_up_sync(kFull, M[w], o);
                        if (lane >= o) {
                            D[w] = lop_merge(D[w], dn, M[w]);
                            M[w] |= mn;
                        }
                    }
                }
            }
#pragma unroll
            for (int w = 0; w < NPW; w++) {
                if (w < whi) {
                    D[w] = (w >= wlo) ? lop_merge(D[w], carry[w], M[w]) : carry[w];
                    if (w >= wlo) carry[w] = __shfl_sync(kFull, D[w], 31);
                }
            }
            if (!MIXED || __all_sync(kFull, ty == R_PP || ty == R_PATH)) {
                const bool emit = (ty == R_PP);
                const int tot = emit ? len + (int)((myrec >> 3) & 1) : 0;
                const unsigned em = __ballot_sync(kFull, emit);
                if (HASH) {
                    // ---- digest only: every emitting lane hashes its own path
                    if (emit) hash_path<NPW>(G, D, stage, lane, len, tot, ga, vb, s0g, acc);
                    int T = tot;
#pragma unroll
                    for (int o = 16; o; o >>= 1) T += __shfl_xor_sync(kFull, T, o);
                    cu.pp += (uint64_t)__popc(em);
                    cu.vv += (uint64_t)T;
                    continue;
                }
                // ---- emitting lanes: offsets by a warp scan of the path lengths
                int ex = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(kFull, ex, o);
                    if (lane >= o) ex += t;
                }
                const int T = __shfl_sync(kFull, ex, 31);
                ex -= tot;
                TPG_DCHECK(cu.pp + __popc(em) <= A.lim[C_PP] && cu.vv + (uint64_t)T <= A.lim[C_VERT],
                           "expand: batch out of range");
                if (emit) A.out_off[cu.pp + __popc(em & lt_mask)] = (int64_t)(cu.vv + (uint64_t)ex);
                // ---- stage the vertices (global ids) at the output's 16-byte phase, then the
                // aligned middle leaves in ONE bulk store (TMA), the <= 3 + 3 ragged ends per lane
                if (T == 0) continue;
                const int al = (int)(cu.vv & 3);
                int32_t *stg = stage_w + sbuf * kStage + al;
                if (lane == 0) bulk_wait_read<EXP_BUFS - 1>();  // this stage's previous bulk store has read it
                __syncwarp();
                if (ga >= 0) {
#pragma unroll
                    for (int p = 0; p < 4 * NPW; p++)
                        if (p < tot) stg[ex + p] = ga + (int)((D[p >> 2] >> (8 * (p & 3))) & 0xff);
                } else {
#pragma unroll
                    for (int p = 0; p < 4 * NPW; p++)
                        if (p < tot) stg[ex + p] = __ldg(G.slot_gid + vb + (int)((D[p >> 2] >> (8 * (p & 3))) & 0xff));
                }
                if (len < tot) stg[ex + len] = s0g;  // closing vertex of a cycle (after the byte loop)
                fence_proxy_async_smem();
                __syncwarp();
                int32_t *dst = A.out_vert + cu.vv;
                const int h = min(T, (4 - al) & 3);           // ints before the first 16-byte boundary
                const int nb = ((T - h) >> 2) << 2;           // the aligned middle
                if (lane < h) st_global_cs(dst + lane, stg[lane]);
                if (lane < T - h - nb) st_global_cs(dst + h + nb + lane, stg[h + nb + lane]);
                if (lane == 0) {  // one bulk group per batch (empty without a middle): wait_read<1> counts batches
                    if (nb > 0) bulk_store(dst + h, stg + h, (uint32_t)nb * 4u);
                    bulk_commit();
                }
                if (kBufs > 1) sbuf ^= 1;
                cu.pp += (uint64_t)__popc(em);
                cu.vv += (uint64_t)T;
            } else {
                // ---- segment items / head blocks in this batch: lane-parallel, every lane
                // emits its own record at offsets from warp scans of the cursor increments
                const int myarg = (int)(myrec >> 32);
                int argv = __shfl_up_sync(kFull, myarg, 1);  // an R_ARG record precedes its HEAD / TRANSIT
                if (lane == 0) argv = cu.arg;
                const int lastty = __shfl_sync(kFull, ty, 31);
                const int lastarg = __shfl_sync(kFull, myarg, 31);
                if (lastty == R_ARG) cu.arg = lastarg;
                const bool isPP = ty == R_PP, isH = ty == R_HEAD, isI = ty == R_TAIL || ty == R_TRANSIT;
                const int tot = len + (isPP ? (int)((myrec >> 3) & 1) : 0);
                int32_t x = 0;
                uint64_t dpp = 0, dvv = 0;
                if (isPP) {
                    dpp = 1;
                    dvv = (uint64_t)tot;
                } else if (isH) {
                    x = __ldg(G.out_gid + argv);
                    const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                    dpp = Wx;
                    dvv = (uint64_t)len * Wx + Vx;
                }
                const uint32_t dhd = isH ? 1u : 0u, dhdv = isH ? (uint32_t)len : 0u;
                const uint32_t dit = isI ? 1u : 0u, ditv = isI ? (uint32_t)len : 0u;
                // inclusive warp scans, then exclusive = inclusive - own
                uint64_t spp = dpp, svv = dvv;
                uint32_t shd = dhd, shdv = dhdv, sit = dit, sitv = ditv;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t a1 = __shfl_up_sync(kFull, spp, o), a2 = __shfl_up_sync(kFull, svv, o);
                    const uint32_t b1 = __shfl_up_sync(kFull, shd, o), b2 = __shfl_up_sync(kFull, shdv, o);
                    const uint32_t c1 = __shfl_up_sync(kFull, sit, o), c2 = __shfl_up_sync(kFull, sitv, o);
                    if (lane >= o) {
                        spp += a1;
                        svv += a2;
                        shd += b1;
                        shdv += b2;
                        sit += c1;
                        sitv += c2;
                    }
                }
                const uint64_t pp = cu.pp + spp - dpp, vv = cu.vv + svv - dvv;
                const uint64_t hd = cu.hd + shd - dhd, hdv = cu.hdv + shdv - dhdv;
                const uint64_t it = cu.it + sit - dit, itv = cu.itv + sitv - ditv;
                TPG_DCHECK(!isPP || (pp < A.lim[C_PP] && vv + tot <= A.lim[C_VERT]), "expand: mixed pp out of range");
                TPG_DCHECK(!isH || (argv >= 0 && hd < A.lim[C_HEADS] && hdv + len <= A.lim[C_HEADV]),
                           "expand: mixed head out of range");
                TPG_DCHECK(!isI || (it < A.lim[C_ITEMS] && itv + len <= A.lim[C_ITEMV]), "expand: mixed item out of range");
                int32_t *dst = nullptr;
                if (isPP && !HASH) {
                    A.out_off[pp] = (int64_t)vv;
                    dst = A.out_vert + vv;
                } else if (isH) {
                    HeadRec hr;
                    hr.pp_off = pp;
                    hr.v_off = vv;
                    hr.hv_off = hdv;
                    hr.len = len;
                    hr.x = x;
                    A.heads[hd] = hr;
                    dst = A.head_pool + hdv;
                } else if (isI) {
                    ItemRec ir;
                    ir.pool_off = (int64_t)itv;
                    ir.len = len;
                    ir.y = (ty == R_TRANSIT) ? __ldg(G.out_gid + argv) : -1;
                    ir.ent = s0g;
                    ir.pad = 0;
                    A.items[it] = ir;
                    dst = A.item_pool + itv;
                }
                if (HASH && isPP) hash_path<NPW>(G, D, stage, lane, len, tot, ga, vb, s0g, acc);
                if (dst) {
#pragma unroll
                    for (int p = 0; p < 4 * NPW; p++) {
                        if (p < len) {
                            const int loc = (int)((D[p >> 2] >> (8 * (p & 3))) & 0xff);
                            dst[p] = (ga >= 0) ? ga + loc : __ldg(G.slot_gid + vb + loc);
                        }
                    }
                    if (len < tot) dst[len] = s0g;  // closing vertex of a cycle
                }
                cu.pp += __shfl_sync(kFull, spp, 31);
                cu.vv += __shfl_sync(kFull, svv, 31);
                cu.hd += __shfl_sync(kFull, shd, 31);
                cu.hdv += __shfl_sync(kFull, shdv, 31);
                cu.it += __shfl_sync(kFull, sit, 31);
                cu.itv += __shfl_sync(kFull, sitv, 31);
            }
        }
    }
    if (HASH) flush_hash(A, acc);
    if (!HASH && lane == 0) bulk_wait_all();  // (the stages must outlive the bulk stores' reads)
}

}  // namespace tpg
