// expand.cuh -- canonical writer (K4) of libtpgen: replays the per-unit
// path-delta record streams written by dfs_kernel into the canonical
// offsets/vertices arrays, head records (cross-SCC
// blocks, filled later by stitch_kernel) and segment items (a5).
//
// One warp per unit.  The warp keeps the unit's current path in shared memory;
// for every record it truncates/appends (lane j writes appended byte j) and,
// for an emitting record, writes the path as one coalesced store stream at the
// exact offsets from the scan of the per-unit counters.  Units are independent,
// so the kernel is a pure streaming writer (output bytes dominate).
#pragma once

#include "dfs.cuh"

namespace tpg {

struct ExpandArgs {
    DevGraph G;
    const void *units;  // Unit<W>[n_units]
    int64_t n_units;
    const int64_t *rfirst;
    const int64_t *rcount;
    const uint64_t *off[C_NUM];  // exclusive scans of the per-unit counters
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

template <int W>
__global__ void __launch_bounds__(kExpandThreads) expand_kernel(ExpandArgs A) {
    constexpr int WARPS = kExpandThreads / 32;
    constexpr int PMAX = 64 * W;
    __shared__ __align__(16) uint8_t spath[WARPS][PMAX + 16];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *P = spath[wid];
    const DevGraph &G = A.G;
    const Unit<W> *units = reinterpret_cast<const Unit<W> *>(A.units);
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;

    for (int64_t u = gw; u < A.n_units; u += nw) {
        const Unit<W> *U = units + u;
        const int4 h = *reinterpret_cast<const int4 *>(&U->scc);
        const int depth = h.w & 0xff;
        for (int j = lane; j <= depth; j += 32) P[j] = U->path[j];
        const int vb = __ldg(G.scc_vbase + h.x);
        const int ga = __ldg(G.scc_gbase + h.x);
        uint64_t pp = A.off[C_PP][u], vv = A.off[C_VERT][u];
        uint64_t it = A.off[C_ITEMS][u], itv = A.off[C_ITEMV][u];
        uint64_t hd = A.off[C_HEADS][u], hdv = A.off[C_HEADV][u];
        const int64_t nrec = A.rcount[u];
        const uint64_t *ch = A.chunks + A.rfirst[u] * kChunkRecs;
        int slot = 0;
        int sgid = -1;
        __syncwarp();
        for (int64_t r = 0; r < nrec; r++) {
            if (slot == kChunkRecs - 1) {
                ch = A.chunks + ch[kChunkRecs - 1] * kChunkRecs;
                slot = 0;
            }
            const uint64_t rec = ch[slot++];
            const int ty = (int)(rec & 7);
            const int cc = (int)((rec >> 4) & 0xff);
            const int n = (int)((rec >> 12) & 7);
            if (lane < n) P[cc + lane] = (uint8_t)(rec >> (16 + 8 * lane));
            const int len = cc + n;
            __syncwarp();
            if (ty == R_PATH) continue;
            int arg = -1;
            if (ty == R_HEAD || ty == R_TRANSIT) {  // followed by its R_ARG record
                if (slot == kChunkRecs - 1) {
                    ch = A.chunks + ch[kChunkRecs - 1] * kChunkRecs;
                    slot = 0;
                }
                arg = (int)(ch[slot++] >> 32);
                r++;
            }
            const int clo = (int)((rec >> 3) & 1);
            const int tot = len + clo;
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
                if (sgid < 0) sgid = __ldg(G.slot_gid + vb + P[0]);
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
            if (ga >= 0) {
                for (int j = lane; j < tot; j += 32) st_global_cs(dst + j, ga + P[j < len ? j : 0]);
            } else {
                for (int j = lane; j < tot; j += 32) st_global_cs(dst + j, __ldg(G.slot_gid + vb + P[j < len ? j : 0]));
            }
            __syncwarp();
        }
        __syncwarp();
    }
}

}  // namespace tpg
