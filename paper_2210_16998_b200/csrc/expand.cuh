// expand.cuh -- canonical writer (K4) of libtpgen: replays the per-unit
// path-delta record streams written by dfs_kernel into the canonical
// offsets/vertices arrays, head records (cross-SCC
// blocks, filled later by stitch_kernel) and segment items (a5).
//
// One warp per unit.  The current path lives in registers, distributed over
// the warp (lane q holds positions q, q+32, ...); records are fetched 32 at a
// time (one coalesced load, then broadcast by shuffle), so the replay has no
// dependent global loads and no shared-memory round trips.  Emitting records
// are written as one coalesced streaming store per 32 vertices at the exact
// offsets produced by the linearization of the per-unit counters.
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
};

constexpr int kExpandThreads = 256;

__device__ __forceinline__ void st_global_cs(int32_t *p, int v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// NP = path registers per lane: ceil((longest emitted path + closing vertex) / 32).
template <int W, int NP>
__global__ void __launch_bounds__(kExpandThreads) expand_kernel(ExpandArgs A) {
    const int lane = threadIdx.x & 31;
    const DevGraph &G = A.G;
    const Unit<W> *units = reinterpret_cast<const Unit<W> *>(A.units);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;

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
        const LinNode *on = A.off + u;
        uint64_t pp = on->v[C_PP], vv = on->v[C_VERT];
        uint64_t it = on->v[C_ITEMS], itv = on->v[C_ITEMV];
        uint64_t hd = on->v[C_HEADS], hdv = on->v[C_HEADV];
        const int64_t nrec = A.rcount[u];
        const uint64_t *ch = A.chunks + A.rfirst[u] * kChunkRecs;
        int slot = 0;  // next record slot in chunk `ch`
        int arg = -1;
        for (int64_t r0 = 0; r0 < nrec; r0 += 32) {
            // ---- fetch the next (up to) 32 records: lane j takes record r0 + j
            const int nb = (nrec - r0 < 32) ? (int)(nrec - r0) : 32;
            // link word of a full chunk (read, but only followed when the unit has records beyond it)
            const uint64_t *nxt = (slot + nb >= kChunkRecs - 1) ? A.chunks + ch[kChunkRecs - 1] * kChunkRecs : ch;
            uint64_t myrec = 0;
            if (lane < nb) {
                const int sj = slot + lane;
                myrec = (sj < kChunkRecs - 1) ? ch[sj] : nxt[sj - (kChunkRecs - 1)];
            }
            if (slot + nb >= kChunkRecs - 1) {
                slot = slot + nb - (kChunkRecs - 1);
                ch = nxt;
            } else {
                slot += nb;
            }
            // ---- replay them in order
            for (int i = 0; i < nb; i++) {
                const uint64_t rec = __shfl_sync(kFull, myrec, i);
                const int ty = (int)(rec & 7);
                if (ty == R_ARG) {
                    arg = (int)(rec >> 32);
                    continue;
                }
                const int cc = (int)((rec >> 4) & 0x1ff);
                const int n = (int)((rec >> 13) & 7);
#pragma unroll
                for (int r = 0; r < NP; r++) {
                    const int d = lane + 32 * r - cc;
                    if (d >= 0 && d < n) P[r] = (int)((rec >> (16 + 8 * d)) & 0xff);
                }
                if (ty == R_PATH) continue;
                const int len = cc + n;
                const int tot = len + (int)((rec >> 3) & 1);
                int32_t *dst;
                if (ty == R_PP) {
                    dst = A.out_vert + vv;
                    if (lane == 0) A.out_off[pp] = (int64_t)vv;
                    pp += 1;
                    vv += (uint64_t)tot;
                } else if (ty == R_HEAD) {
                    const int32_t x = __ldg(G.out_gid + arg);
                    dst = A.head_pool + hdv;
                    if (lane == 0) {
                        HeadRec hr;
                        hr.pp_off = pp;
                        hr.v_off = vv;
                        hr.hv_off = hdv;
                        hr.len = len;
                        hr.x = x;
                        A.heads[hd] = hr;
                    }
                    const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                    pp += Wx;
                    vv += (uint64_t)len * Wx + Vx;
                    hd += 1;
                    hdv += (uint64_t)len;
                } else {  // R_TAIL / R_TRANSIT
                    dst = A.item_pool + itv;
                    if (lane == 0) {
                        ItemRec ir;
                        ir.pool_off = (int64_t)itv;
                        ir.len = len;
                        ir.y = (ty == R_TRANSIT) ? __ldg(G.out_gid + arg) : -1;
                        ir.ent = sgid;
                        ir.pad = 0;
                        A.items[it] = ir;
                    }
                    it += 1;
                    itv += (uint64_t)len;
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
        }
    }
}

}  // namespace tpg
