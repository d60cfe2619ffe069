// aux_kernels.cuh -- scans, refinement scatter, segment tables, cross-SCC
// stitch writer (K5), test-path writer (K6) and digest (K8) for libtpgen.
#pragma once

#include "kernels.cuh"

namespace tpg {

// ------------------------------------------------------------------- scan
// Exclusive prefix sums of up to 8 uint64 arrays of the same length, in place.
constexpr int kScanThreads = 256;
constexpr int kScanIpt = 8;
constexpr int kScanTile = kScanThreads * kScanIpt;

struct ScanArrays {
    uint64_t *a[8];
    int na;
};

__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint64_t t = __shfl_up_sync(kFull, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread (kScanThreads threads).
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *sm, uint64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t inc = warp_incl_scan(v);
    if (lane == 31) sm[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t w = (lane < kScanThreads / 32) ? sm[lane] : 0;
        const uint64_t wi = warp_incl_scan(w);
        if (lane < kScanThreads / 32) sm[lane] = wi - w;
        if (lane == kScanThreads / 32 - 1) sm[16] = wi;
    }
    __syncthreads();
    const uint64_t r = inc - v + sm[wid];
    total = sm[16];
    __syncthreads();
    return r;
}

__global__ void scan_reduce_kernel(ScanArrays S, int64_t n, uint64_t *bsum, int nb) {
    __shared__ uint64_t sm[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    for (int a = 0; a < S.na; a++) {
        uint64_t s = 0;
#pragma unroll
        for (int i = 0; i < kScanIpt; i++)
            if (base + i < n) s += S.a[a][base + i];
        uint64_t tot;
        block_excl_scan(s, sm, tot);
        if (threadIdx.x == 0) bsum[(int64_t)a * nb + blockIdx.x] = tot;
    }
}

__global__ void scan_bsum_kernel(uint64_t *bsum, int nb, int na, uint64_t *totals) {
    __shared__ uint64_t sm[32];
    for (int a = 0; a < na; a++) {
        uint64_t carry = 0;
        for (int b0 = 0; b0 < nb; b0 += kScanThreads) {
            const int b = b0 + threadIdx.x;
            const uint64_t v = (b < nb) ? bsum[(int64_t)a * nb + b] : 0;
            uint64_t tot;
            const uint64_t ex = block_excl_scan(v, sm, tot);
            if (b < nb) bsum[(int64_t)a * nb + b] = ex + carry;
            carry += tot;
        }
        if (threadIdx.x == 0) totals[a] = carry;
    }
}

__global__ void scan_down_kernel(ScanArrays S, int64_t n, const uint64_t *bsum, int nb) {
    __shared__ uint64_t sm[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanIpt;
    for (int a = 0; a < S.na; a++) {
        uint64_t v[kScanIpt];
        uint64_t s = 0;
#pragma unroll
        for (int i = 0; i < kScanIpt; i++) {
            v[i] = (base + i < n) ? S.a[a][base + i] : 0;
            s += v[i];
        }
        uint64_t tot;
        uint64_t run = block_excl_scan(s, sm, tot) + bsum[(int64_t)a * nb + blockIdx.x];
#pragma unroll
        for (int i = 0; i < kScanIpt; i++) {
            if (base + i < n) S.a[a][base + i] = run;
            run += v[i];
        }
    }
}

// ---------------------------------------------------------- linearization
// The units form a forest: roots are the start vertices (canonical order =
// ascending global id), and a unit's children are the units it donated, which
// follow all of its own output in lexicographic order -- blocks donated later
// come from deeper levels and so come first (the block list is newest-first).
// Canonical output order is the preorder of that forest, so each unit's output
// offset is  off(root) + sum over the edges on its root path of the position of
// the child inside its parent's output.  Three steps, independent of the
// forest depth in launches:
//   lin_up_flow: subtree totals bottom-up as a dataflow (the last child to
//     finish closes its parent; one launch, one decrement per edge);
//   lin_roots + lin_rel: the position of every unit relative to its parent
//     (the roots: their canonical offset);
//   lin_jump: pointer jumping along parent links (ceil(log2(depth+1))
//     launches), which sums the relative positions along each root path.
struct LinArgs {
    const uint64_t *cnt[C_NUM];  // own counts
    uint64_t *sub[C_NUM];        // subtree totals
    LinNode *node;               // relative offsets / jump links (input of the first jump round)
    uint64_t *acc[C_NUM];        // sums of the children's subtree totals (zeroed before lin_up_flow)
    const int64_t *parent;       // donor of each unit (-1: a root)
    int32_t *pending;            // children whose subtree totals are still open (consumed)
    const int64_t *child_head;
    const int64_t *blk_first;
    const int32_t *blk_count;
    const int64_t *blk_next;
    int64_t n;
    const int64_t *roots;        // root units in canonical order
    int64_t n_roots;
    uint64_t *totals;            // [C_NUM]
};

// Leaves start; every unit passes its subtree total to its donor with plain
// atomic adds, then decrements the donor's open-children count -- whoever
// closes the donor continues with it.  One launch; the critical path is one
// atomic round trip per level of the deepest donation chain.
__global__ void lin_up_flow_kernel(LinArgs A) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x) {
        if (A.child_head[i] >= 0) continue;
        int64_t cur = i;
        uint64_t t[C_NUM];
#pragma unroll
        for (int c = 0; c < C_NUM; c++) t[c] = A.cnt[c][cur];
        for (;;) {
#pragma unroll
            for (int c = 0; c < C_NUM; c++) A.sub[c][cur] = t[c];
            const int64_t p = A.parent[cur];
            if (p < 0) break;
#pragma unroll
            for (int c = 0; c < C_NUM; c++)
                if (t[c]) atomicAdd(reinterpret_cast<unsigned long long *>(A.acc[c] + p), (unsigned long long)t[c]);
            if (atom_dec_acq_rel(A.pending + p) != 1) break;
            cur = p;
#pragma unroll
            for (int c = 0; c < C_NUM; c++) t[c] = A.cnt[c][cur] + ld_relaxed_u64(A.acc[c] + cur);
        }
    }
}

// One block: exclusive scan of the root subtree totals in canonical root order.
__global__ void lin_roots_kernel(LinArgs A) {
    __shared__ uint64_t sm[32];
    for (int c = 0; c < C_NUM; c++) {
        uint64_t carry = 0;
        for (int64_t b0 = 0; b0 < A.n_roots; b0 += kScanThreads) {
            const int64_t j = b0 + threadIdx.x;
            const uint64_t v = (j < A.n_roots) ? A.sub[c][A.roots[j]] : 0;
            uint64_t tot;
            const uint64_t ex = block_excl_scan(v, sm, tot);
            if (j < A.n_roots) {
                A.node[A.roots[j]].v[c] = ex + carry;
                if (c == 0) A.node[A.roots[j]].jmp = -1;
            }
            carry += tot;
        }
        if (threadIdx.x == 0) A.totals[c] = carry;
    }
}

// Many roots: tmp[c][j] = subtree total of root j; scanned device-wide, then scattered.
__global__ void lin_roots_gather_kernel(LinArgs A, uint64_t *tmp) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < A.n_roots; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = A.roots[j];
#pragma unroll
        for (int c = 0; c < C_NUM; c++) tmp[(int64_t)c * A.n_roots + j] = A.sub[c][r];
    }
}
__global__ void lin_roots_scatter_kernel(LinArgs A, const uint64_t *tmp) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < A.n_roots; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = A.roots[j];
#pragma unroll
        for (int c = 0; c < C_NUM; c++) A.node[r].v[c] = tmp[(int64_t)c * A.n_roots + j];
        A.node[r].jmp = -1;
    }
}

// Children placed after their parent's own output, newest block first.
__global__ void lin_rel_kernel(LinArgs A) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x) {
        if (A.child_head[i] < 0) continue;
        uint64_t base[C_NUM];
#pragma unroll
        for (int c = 0; c < C_NUM; c++) base[c] = A.cnt[c][i];
        for (int64_t b = A.child_head[i]; b >= 0; b = A.blk_next[b]) {
            const int64_t cf = A.blk_first[b];
            const int32_t cc = A.blk_count[b];
            for (int32_t k = 0; k < cc; k++) {
                LinNode nd;
#pragma unroll
                for (int c = 0; c < C_NUM; c++) {
                    nd.v[c] = base[c];
                    base[c] += A.sub[c][cf + k];
                }
                nd.jmp = i;
                nd.pad = 0;
                A.node[cf + k] = nd;
            }
        }
    }
}

// One round of pointer jumping (Wyllie): v += v[jmp], jmp = jmp[jmp].
__global__ void lin_jump_kernel(const LinNode *in, LinNode *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        LinNode a = in[i];
        if (a.jmp >= 0) {
            const LinNode b = in[a.jmp];
#pragma unroll
            for (int c = 0; c < C_NUM; c++) a.v[c] += b.v[c];
            a.jmp = b.jmp;
        }
        out[i] = a;
    }
}

__global__ void sum_kernel(const uint64_t *a, int64_t n, unsigned long long *out) {
    uint64_t s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += a[i];
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

// --------------------------------------------------- segment tables (a5)
// Items of entry vertex x are the items of the subtree of x's root unit.
__global__ void item_bounds_kernel(const int64_t *roots, const int32_t *root_gid, int64_t n_roots,
                                   const LinNode *off, const uint64_t *sub_items, int64_t *ibeg, int64_t *iend) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_roots; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = roots[j];
        ibeg[root_gid[j]] = (int64_t)off[r].v[C_ITEMS];
        iend[root_gid[j]] = (int64_t)(off[r].v[C_ITEMS] + sub_items[r]);
    }
}

__global__ void item_weight_kernel(DevGraph G, const ItemRec *items, int64_t n, uint64_t *cw, uint64_t *vw) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const ItemRec it = items[i];
        if (it.y < 0) {
            cw[i] = 1;
            vw[i] = (uint64_t)it.len;
        } else {
            const uint64_t W = __ldg(G.Wc + it.y), V = __ldg(G.Wv + it.y);
            cw[i] = W;
            vw[i] = (uint64_t)it.len * W + V;
        }
    }
}

__global__ void head_weight_kernel(DevGraph G, const HeadRec *heads, int64_t n, uint64_t *hw) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        hw[i] = __ldg(G.Wc + heads[i].x);
}

struct StitchArgs {
    const HeadRec *heads;
    int64_t n_heads;
    const uint64_t *comp_off;  // exclusive scan of W(x_h) over heads
    uint64_t n_comp;
    const ItemRec *items;
    const uint64_t *cum, *vcum;  // global exclusive scans of item weights
    const int64_t *ibeg, *iend;  // per entry vertex (global id)
    const int32_t *head_pool, *item_pool;
    int64_t *out_off;
    int32_t *out_vert;
    uint64_t n_pp, n_vert;  // output sizes (debug-build bounds checks)
};

__device__ __forceinline__ int64_t upper_bound_u64(const uint64_t *a, int64_t lo, int64_t hi, uint64_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// K5: one warp per cross prime path h (+) completion_k(x).  The k-th
// completion is unranked through the entry tables (mixed radix over the DP
// counts), its output position follows from the per-item vertex prefix sums.
__global__ void stitch_kernel(StitchArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t g = (uint64_t)wg; g < A.n_comp; g += (uint64_t)nw) {
        const int64_t h = upper_bound_u64(A.comp_off, 0, A.n_heads, g) - 1;
        const HeadRec H = A.heads[h];
        const uint64_t k = g - A.comp_off[h];
        // pass 1: vertex offset of completion k inside the block
        uint64_t vrel = 0, kk = k;
        int32_t x = H.x;
        while (true) {
            const int64_t b = A.ibeg[x], e = A.iend[x];
            const uint64_t bc = A.cum[b], bv = A.vcum[b];
            const int64_t i = upper_bound_u64(A.cum, b, e, bc + kk) - 1;
            const uint64_t k2 = kk - (A.cum[i] - bc);
            const ItemRec it = A.items[i];
            vrel += A.vcum[i] - bv;
            if (it.y < 0) break;
            vrel += k2 * (uint64_t)it.len;
            x = it.y;
            kk = k2;
        }
        const uint64_t vstart = H.v_off + k * (uint64_t)H.len + vrel;
        TPG_DCHECK(H.pp_off + k < A.n_pp && vstart + H.len <= A.n_vert, "stitch: path out of range");
        if (lane == 0) A.out_off[H.pp_off + k] = (int64_t)vstart;
        int32_t *dst = A.out_vert + vstart;
        for (int j = lane; j < H.len; j += 32) dst[j] = A.head_pool[H.hv_off + j];
        dst += H.len;
        // pass 2: copy the segments
        kk = k;
        x = H.x;
        while (true) {
            const int64_t b = A.ibeg[x], e = A.iend[x];
            const uint64_t bc = A.cum[b];
            const int64_t i = upper_bound_u64(A.cum, b, e, bc + kk) - 1;
            const uint64_t k2 = kk - (A.cum[i] - bc);
            const ItemRec it = A.items[i];
            const int32_t *src = A.item_pool + it.pool_off;
            for (int j = lane; j < it.len; j += 32) dst[j] = src[j];
            dst += it.len;
            if (it.y < 0) break;
            x = it.y;
            kk = k2;
        }
    }
}

// Cross-SCC writer by ranges: warp w writes the completions [g0, g1) of the
// global cross-PP index space (an even split).  It unranks g0 once (binary
// searches over the cumulative item weights, level by level) into a stack of
// (entry, item, prefix length) per level, then steps through the following
// completions in lexicographic order like an odometer: the deepest level that
// still has a next item advances and the levels below restart at the first item
// of their entry; when a head's completions run out, the next head starts from
// its entry's first items.  Consecutive completions are adjacent in the output
// and share the prefix up to the changed level, which the warp copies from the
// path it wrote just before (coalesced, L2-resident); only the changed items
// come from the segment pool.  (Every item leads to at least one completion: a
// sink SCC always has a tail, so no zero-weight item needs skipping.)
struct StitchRangeArgs {
    StitchArgs S;
    int64_t *scratch;  // per warp: 3 * dmax int64 (entry, item, prefix length per level)
    int dmax;
};

__global__ void stitch_range_kernel(StitchRangeArgs C) {
    const StitchArgs &A = C.S;
    const int lane = threadIdx.x & 31;
    const uint64_t wg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    int64_t *sx = C.scratch + wg * 3 * (uint64_t)C.dmax;  // entry of each level
    int64_t *si = sx + C.dmax;                            // item of each level
    int64_t *sp = si + C.dmax;                            // path length before each level's item
    const uint64_t q = A.n_comp / nw, r = A.n_comp % nw;
    const uint64_t g0 = q * wg + (wg < r ? wg : r), g1 = g0 + q + (wg < r ? 1 : 0);
    if (g0 >= g1) return;
    int64_t h = upper_bound_u64(A.comp_off, 0, A.n_heads, g0) - 1;
    HeadRec H = A.heads[h];
    uint64_t k = g0 - A.comp_off[h];
    uint64_t wh = ((h + 1 < A.n_heads) ? A.comp_off[h + 1] : A.n_comp) - A.comp_off[h];
    // ---- unrank completion k of head h (lane 0) into the stack; its vertex offset inside the head block
    int depth = 0;
    int64_t total = 0;
    uint64_t vrel = 0;
    if (lane == 0) {
        uint64_t kk = k;
        int32_t x = H.x;
        int64_t pl = H.len;
        while (true) {
            const int64_t b = A.ibeg[x], e = A.iend[x];
            const uint64_t bc = A.cum[b], bv = A.vcum[b];
            const int64_t i = upper_bound_u64(A.cum, b, e, bc + kk) - 1;
            const uint64_t k2 = kk - (A.cum[i] - bc);
            const ItemRec it = A.items[i];
            vrel += A.vcum[i] - bv;
            TPG_DCHECK(depth < C.dmax, "stitch: stack depth");
            sx[depth] = x;
            si[depth] = i;
            sp[depth] = pl;
            depth++;
            pl += it.len;
            if (it.y < 0) break;
            vrel += k2 * (uint64_t)it.len;
            x = it.y;
            kk = k2;
        }
        total = pl;
    }
    depth = __shfl_sync(kFull, depth, 0);
    total = __shfl_sync(kFull, total, 0);
    vrel = __shfl_sync(kFull, vrel, 0);
    __syncwarp();
    uint64_t vstart = H.v_off + k * (uint64_t)H.len + vrel, pstart = 0;
    int changed = 0;  // first level that differs from the previous completion (0 with a new head: all of it)
    bool fresh = true;
    for (uint64_t g = g0; g < g1; g++) {
        if (g > g0) {
            // ---- advance: the next completion of this head, or the first one of the next head
            int64_t ntotal = 0;
            int nchanged = 0;
            bool nfresh = false;
            if (lane == 0) {
                int j = -1;
                int64_t i = 0;
                int32_t x = 0;
                if (k + 1 < wh) {
                    j = depth - 1;
                    i = si[j] + 1;
                    x = (int32_t)sx[j];
                    while (i >= A.iend[x]) {  // this level is exhausted: advance the one above
                        j--;
                        TPG_DCHECK(j >= 0, "stitch: odometer underflow");
                        i = si[j] + 1;
                        x = (int32_t)sx[j];
                    }
                } else {  // next head: its entry's first items
                    nfresh = true;
                }
                int d = nfresh ? 0 : j;
                int64_t pl = nfresh ? 0 : sp[j];
                if (nfresh) {
                    const HeadRec Hn = A.heads[h + 1];
                    x = Hn.x;
                    i = A.ibeg[x];
                    pl = Hn.len;
                }
                nchanged = d;
                while (true) {  // the new item at level d, then the first items below it
                    const ItemRec it = A.items[i];
                    TPG_DCHECK(d < C.dmax, "stitch: stack depth");
                    sx[d] = x;
                    si[d] = i;
                    sp[d] = pl;
                    d++;
                    pl += it.len;
                    if (it.y < 0) break;
                    x = it.y;
                    i = A.ibeg[x];
                }
                depth = d;
                ntotal = pl;
            }
            nfresh = __shfl_sync(kFull, nfresh, 0);
            nchanged = __shfl_sync(kFull, nchanged, 0);
            depth = __shfl_sync(kFull, depth, 0);
            ntotal = __shfl_sync(kFull, ntotal, 0);
            __syncwarp();  // the stack and the previous path are visible to every lane
            if (nfresh) {
                h++;
                H = A.heads[h];
                k = 0;
                wh = ((h + 1 < A.n_heads) ? A.comp_off[h + 1] : A.n_comp) - A.comp_off[h];
                vstart = H.v_off;
            } else {
                k++;
                pstart = vstart;
                vstart += (uint64_t)total;
            }
            total = ntotal;
            changed = nchanged;
            fresh = nfresh;
        }
        TPG_DCHECK(H.pp_off + k < A.n_pp && vstart + (uint64_t)total <= A.n_vert, "stitch: path out of range");
        int32_t *dst = A.out_vert + vstart;
        if (fresh) {  // head vertices, then every level's item
            for (int j = lane; j < H.len; j += 32) dst[j] = __ldg(A.head_pool + H.hv_off + j);
        } else {  // the prefix shared with the previous completion (written just before)
            const int64_t keep = sp[changed];
            const int32_t *src = A.out_vert + pstart;
            int64_t j = lane;
            for (; j + 224 < keep; j += 256) {  // eight loads in flight per lane
                int32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = __ldcg(src + j + 32 * u);
#pragma unroll
                for (int u = 0; u < 8; u++) dst[j + 32 * u] = v[u];
            }
            for (; j + 96 < keep; j += 128) {  // four
                const int32_t a0 = __ldcg(src + j), a1 = __ldcg(src + j + 32), a2 = __ldcg(src + j + 64),
                              a3 = __ldcg(src + j + 96);
                dst[j] = a0;
                dst[j + 32] = a1;
                dst[j + 64] = a2;
                dst[j + 96] = a3;
            }
            for (; j < keep; j += 32) dst[j] = __ldcg(src + j);
        }
        for (int d = changed; d < depth; d++) {
            const ItemRec it = A.items[si[d]];
            const int32_t *src = A.item_pool + it.pool_off;
            for (int j = lane; j < it.len; j += 32) dst[sp[d] + j] = __ldg(src + j);
        }
        if (lane == 0) A.out_off[H.pp_off + k] = (int64_t)vstart;
        __syncwarp();
    }
}

// COUNT_HASH mode: the digest of every cross-SCC prime path without writing it;
// one thread per path (completion), vertices absorbed in path order.
__global__ void stitch_hash_kernel(StitchArgs A, unsigned long long *acc) {
    uint64_t sa = 0, sb = 0;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < A.n_comp;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t h = upper_bound_u64(A.comp_off, 0, A.n_heads, g) - 1;
        const HeadRec H = A.heads[h];
        const uint64_t k = g - A.comp_off[h];
        // pass 1: length of completion k
        uint64_t len = (uint64_t)H.len, kk = k;
        int32_t x = H.x;
        while (true) {
            const int64_t b = A.ibeg[x], e = A.iend[x];
            const uint64_t bc = A.cum[b];
            const int64_t i = upper_bound_u64(A.cum, b, e, bc + kk) - 1;
            const uint64_t k2 = kk - (A.cum[i] - bc);
            const ItemRec it = A.items[i];
            len += (uint64_t)it.len;
            if (it.y < 0) break;
            x = it.y;
            kk = k2;
        }
        // pass 2: absorb head, transits, tail
        PathHash hs;
        hs.init(len);
        for (int j = 0; j < H.len; j++) hs.add(A.head_pool[H.hv_off + j]);
        kk = k;
        x = H.x;
        while (true) {
            const int64_t b = A.ibeg[x], e = A.iend[x];
            const uint64_t bc = A.cum[b];
            const int64_t i = upper_bound_u64(A.cum, b, e, bc + kk) - 1;
            const uint64_t k2 = kk - (A.cum[i] - bc);
            const ItemRec it = A.items[i];
            const int32_t *src = A.item_pool + it.pool_off;
            for (int j = 0; j < it.len; j++) hs.add(src[j]);
            if (it.y < 0) break;
            x = it.y;
            kk = k2;
        }
        hs.fin();
        sa += hs.a;
        sb += hs.b;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        sa += __shfl_xor_sync(kFull, sa, d);
        sb += __shfl_xor_sync(kFull, sb, d);
    }
    if ((threadIdx.x & 31) == 0 && (sa | sb)) {
        atomicAdd(acc, (unsigned long long)sa);
        atomicAdd(acc + 1, (unsigned long long)sb);
    }
}

// Count modes: weights of the HeadS records written by cnt_kernel (x = slot of the head's
// exit vertex; x < 0: an unused slot).  hw[i] = number of cross prime paths h (+) w (+) ...
// over every out-of-SCC arc (exit -> w) = sum of W(w); acc[0] += that, acc[1] += their
// vertices (|h| W(w) + V(w)); acc[2] |= 1 on a total >= 2^62 (LIMIT_EXCEEDED).
__global__ void head_weight_s_kernel(DevGraph G, const HeadS *heads, int64_t n, uint64_t *hw,
                                     unsigned long long *acc) {
    const Slot<1> *slots = reinterpret_cast<const Slot<1> *>(G.slots);
    uint64_t sw = 0, sv = 0;
    bool ovf = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const HeadS H = heads[i];
        uint64_t w = 0;
        if (H.x >= 0) {
            const int4 m = __ldg(reinterpret_cast<const int4 *>(&slots[H.x].gid));
            for (int a = 0; a < m.z; a++) {
                const int32_t x = __ldg(G.out_gid + m.y + a);
                const uint64_t Wx = __ldg(G.Wc + x), Vx = __ldg(G.Wv + x);
                const uint64_t hi = __umul64hi((uint64_t)H.len, Wx), lo = (uint64_t)H.len * Wx;
                if (hi || Wx >= (1ull << 62) || lo >= (1ull << 62) || Vx >= (1ull << 62)) ovf = true;
                w += Wx;
                sv += lo + Vx;
            }
        }
        hw[i] = w;
        sw += w;
        if (w >= (1ull << 62) || sw >= (1ull << 62) || sv >= (1ull << 62)) ovf = true;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const uint64_t a = sw + __shfl_xor_sync(kFull, sw, d), b = sv + __shfl_xor_sync(kFull, sv, d);
        if (a < sw || b < sv || a >= (1ull << 62) || b >= (1ull << 62)) ovf = true;
        sw = a;
        sv = b;
    }
    ovf = __any_sync(kFull, ovf);
    if ((threadIdx.x & 31) == 0) {
        if (sw) atomicAdd(acc, (unsigned long long)sw);
        if (sv) atomicAdd(acc + 1, (unsigned long long)sv);
        if (ovf) atomicOr(acc + 2, 1ull);
    }
}

// ------------------------------------------------ count modes: items and stitching
// Items of the count-mode segment phase (ItemS, written in no order by cnt_kernel<SEG>):
// counted per entry vertex, scattered into per-entry groups (order inside a group is
// irrelevant: every completion is hashed once), weighted and scanned like the record path's.
// Grouping of the raw items by entry.  Each block takes chunks of kGroupChunk items and counts
// them per entry in a small shared-memory table (the items of a chunk come from few walks, so
// from few entries), then adds the table to the global counters: one atomic per entry per
// chunk instead of one per item.  The scatter recounts the chunk, reserves each entry's range
// with one atomic, and places every item at its entry's next position (shared atomics).
// Entries that do not fit the table go straight to the global atomics.

constexpr int kGroupChunk = 8192;  // items per block-chunk of the item passes (aggregates, grouping)
constexpr int kGroupTab = 64;      // distinct keys a chunk counts in shared memory

__device__ __forceinline__ int group_slot(int *keys, int32_t e) {
    int h = (int)((uint32_t)e * 2654435761u >> 26) & (kGroupTab - 1);
    for (int p = 0; p < kGroupTab; p++, h = (h + 1) & (kGroupTab - 1)) {
        const int k = keys[h];
        if (k == e) return h;
        if (k == -1) {
            const int old = atomicCAS(&keys[h], -1, e);
            if (old == -1 || old == e) return h;
        }
    }
    return -1;
}

__global__ void item_count_s_kernel(const ItemS *items, int64_t n, unsigned long long *cnt) {
    __shared__ int keys[kGroupTab];
    __shared__ unsigned int cnts[kGroupTab];
    for (int64_t c0 = (int64_t)blockIdx.x * kGroupChunk; c0 < n; c0 += (int64_t)gridDim.x * kGroupChunk) {
        if (threadIdx.x < kGroupTab) {
            keys[threadIdx.x] = -1;
            cnts[threadIdx.x] = 0;
        }
        __syncthreads();
        const int64_t c1 = min(n, c0 + kGroupChunk);
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const int32_t e = items[i].ent;
            if (e < 0) continue;
            const int h = group_slot(keys, e);
            if (h >= 0) atomicAdd(&cnts[h], 1u);
            else atomicAdd(cnt + e, 1ull);
        }
        __syncthreads();
        if (threadIdx.x < kGroupTab && keys[threadIdx.x] >= 0 && cnts[threadIdx.x])
            atomicAdd(cnt + keys[threadIdx.x], (unsigned long long)cnts[threadIdx.x]);
        __syncthreads();
    }
}
__global__ void item_scatter_s_kernel(const ItemS *items, int64_t n, unsigned long long *cursor, ItemS *out) {
    __shared__ int keys[kGroupTab];
    __shared__ unsigned int cnts[kGroupTab];
    __shared__ unsigned long long base[kGroupTab];
    for (int64_t c0 = (int64_t)blockIdx.x * kGroupChunk; c0 < n; c0 += (int64_t)gridDim.x * kGroupChunk) {
        if (threadIdx.x < kGroupTab) {
            keys[threadIdx.x] = -1;
            cnts[threadIdx.x] = 0;
        }
        __syncthreads();
        const int64_t c1 = min(n, c0 + kGroupChunk);
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const int32_t e = items[i].ent;
            if (e < 0) continue;
            const int h = group_slot(keys, e);
            if (h >= 0) atomicAdd(&cnts[h], 1u);
            else out[atomicAdd(cursor + e, 1ull)] = items[i];  // not in the table: placed right away
        }
        __syncthreads();
        if (threadIdx.x < kGroupTab) {
            if (keys[threadIdx.x] >= 0 && cnts[threadIdx.x])
                base[threadIdx.x] = atomicAdd(cursor + keys[threadIdx.x], (unsigned long long)cnts[threadIdx.x]);
            cnts[threadIdx.x] = 0;
        }
        __syncthreads();
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const ItemS it = items[i];
            if (it.ent < 0) continue;
            int h = (int)((uint32_t)it.ent * 2654435761u >> 26) & (kGroupTab - 1);
            int p = 0;
            for (; p < kGroupTab && keys[h] != it.ent; p++) h = (h + 1) & (kGroupTab - 1);
            if (p < kGroupTab) out[base[h] + atomicAdd(&cnts[h], 1u)] = it;
        }
        __syncthreads();
    }
}
// per entry (global id): first and end item of its group, from the exclusive scan of the counts
__global__ void item_bounds_s_kernel(const uint64_t *start, const uint64_t *cnt, int32_t n, int64_t *ibeg,
                                     int64_t *iend) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        ibeg[v] = (int64_t)start[v];
        iend[v] = (int64_t)(start[v] + cnt[v]);
    }
}
// Completion-DP aggregates from the raw items (before the DP): per entry (slot) the number
// and total length of its tail segments, per (entry, out-arc) pair those of its transit
// segments (Def. 6, R9).  Keys: slot for tails, n_slots + pair index for transits; counted per
// chunk in a shared-memory table (see item_count_s_kernel), one atomic per key and chunk.
__global__ void item_agg_s_kernel(DevGraph G, const ItemS *items, int64_t n, int32_t n_slots,
                                  unsigned long long *tail_cnt, unsigned long long *tail_len,
                                  unsigned long long *pair_cnt, unsigned long long *pair_len) {
    __shared__ unsigned long long keys[kGroupTab];
    __shared__ unsigned int cnts[kGroupTab];
    __shared__ unsigned long long lens[kGroupTab];
    const Slot<1> *slots = reinterpret_cast<const Slot<1> *>(G.slots);
    const unsigned long long kNone = ~0ull;
    auto add = [&](unsigned long long key, uint32_t len) {
        int h = (int)((uint32_t)(key * 0x9E3779B97F4A7C15ull >> 40)) & (kGroupTab - 1);
        for (int p = 0; p < kGroupTab; p++, h = (h + 1) & (kGroupTab - 1)) {
            unsigned long long k = keys[h];
            if (k == kNone) k = atomicCAS(&keys[h], kNone, key);
            if (k == kNone || k == key) {
                atomicAdd(&cnts[h], 1u);
                atomicAdd(&lens[h], (unsigned long long)len);
                return;
            }
        }
        if (key < (unsigned long long)n_slots) {  // the table is full: straight to the global counters
            atomicAdd(tail_cnt + key, 1ull);
            atomicAdd(tail_len + key, (unsigned long long)len);
        } else {
            atomicAdd(pair_cnt + (key - n_slots), 1ull);
            atomicAdd(pair_len + (key - n_slots), (unsigned long long)len);
        }
    };
    for (int64_t c0 = (int64_t)blockIdx.x * kGroupChunk; c0 < n; c0 += (int64_t)gridDim.x * kGroupChunk) {
        if (threadIdx.x < kGroupTab) {
            keys[threadIdx.x] = kNone;
            cnts[threadIdx.x] = 0;
            lens[threadIdx.x] = 0;
        }
        __syncthreads();
        const int64_t c1 = min(n, c0 + kGroupChunk);
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
            const ItemS it = items[i];
            if (it.ent < 0) continue;
            const int32_t es = __ldg(G.v_slot + it.ent);
            if (it.x < 0) {
                add((unsigned long long)es, (uint32_t)it.len);
            } else {
                const int4 m = __ldg(reinterpret_cast<const int4 *>(&slots[it.x].gid));
                const int32_t c = __ldg(G.comp + it.ent);
                const long long pbase = __ldg(G.scc_pair_base + c) +
                                        (long long)__ldg(G.slot_eidx + es) * __ldg(G.scc_nout + c) -
                                        __ldg(G.scc_out_base + c);
                for (int a = 0; a < m.z; a++)
                    add((unsigned long long)(n_slots + pbase + m.y + a), (uint32_t)it.len);
            }
        }
        __syncthreads();
        if (threadIdx.x < kGroupTab && keys[threadIdx.x] != kNone) {
            const unsigned long long key = keys[threadIdx.x];
            if (key < (unsigned long long)n_slots) {
                atomicAdd(tail_cnt + key, (unsigned long long)cnts[threadIdx.x]);
                atomicAdd(tail_len + key, lens[threadIdx.x]);
            } else {
                atomicAdd(pair_cnt + (key - n_slots), (unsigned long long)cnts[threadIdx.x]);
                atomicAdd(pair_len + (key - n_slots), lens[threadIdx.x]);
            }
        }
        __syncthreads();
    }
}

// completions of an item and their vertices: a tail 1 / len; a transit sum over the exit's arcs
__global__ void item_weight_s_kernel(DevGraph G, const ItemS *items, int64_t n, uint64_t *cw, uint64_t *vw) {
    const Slot<1> *slots = reinterpret_cast<const Slot<1> *>(G.slots);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const ItemS it = items[i];
        if (it.x < 0) {
            cw[i] = 1;
            vw[i] = (uint64_t)it.len;
        } else {
            const int4 m = __ldg(reinterpret_cast<const int4 *>(&slots[it.x].gid));
            uint64_t W = 0, V = 0;
            for (int a = 0; a < m.z; a++) {
                const int32_t y = __ldg(G.out_gid + m.y + a);
                const uint64_t Wy = __ldg(G.Wc + y);
                W += Wy;
                V += (uint64_t)it.len * Wy + __ldg(G.Wv + y);
            }
            cw[i] = W;
            vw[i] = V;
        }
    }
}

struct StitchSArgs {
    const TpTerm *tp;          // non-null: the test paths of the cross prime paths (terms per slot)
    unsigned int *unreachable;
    const HeadS *heads;
    int64_t n_heads;
    const uint64_t *comp_off;  // exclusive scan of the heads' completion counts
    uint64_t n_comp;
    const ItemS *items;        // grouped by entry vertex
    const uint64_t *cum;       // global exclusive scan of the items' completion counts
    const int64_t *ibeg, *iend;  // per entry vertex (global id)
};

// Count modes: the digest of the cross-SCC prime path h (+) completion k of head H, from the
// head's digest sum S(h) and the items' (A, B): an item at offset o adds A + 2 o B (R20).
// Completion k runs over the exit vertex's out-of-SCC arcs in order (W(w) completions each),
// then is unranked through the entry groups (a binary search per level inside one group).
// hint_x / hint_i (stitch_big: the first-level group and item of the warp's lane 0, whose
// completions are the lane's neighbours): when this completion's first level is the same group,
// the item search starts at hint_i in a window of 64 items (the full search otherwise).
__device__ __forceinline__ void hash_completion(const StitchSArgs &A, const DevGraph &G, const HeadS &H, uint64_t kk,
                                                uint64_t &sa, uint64_t &sb, uint64_t &sv, int32_t hint_x = -1,
                                                int64_t hint_i = -1, int64_t *first_i = nullptr,
                                                int32_t *first_x = nullptr) {
    const Slot<1> *slots = reinterpret_cast<const Slot<1> *>(G.slots);
    const int4 m = __ldg(reinterpret_cast<const int4 *>(&slots[H.x].gid));
    int32_t x = -1;
    for (int a = 0; a < m.z; a++) {  // the arc whose completions hold index kk
        const int32_t xa = __ldg(G.out_gid + m.y + a);
        const uint64_t Wx = __ldg(G.Wc + xa);
        if (kk < Wx) {
            x = xa;
            break;
        }
        kk -= Wx;
    }
    uint64_t S = H.S;
    uint32_t pos = (uint32_t)H.len;
    bool first = true;
    while (true) {
        const int64_t b = A.ibeg[x], e = A.iend[x];
        int64_t i = b;
        uint64_t k2 = kk;
        if (e - b > 1) {
            const uint64_t bc = A.cum[b];
            int64_t lo = b, hi = e;
            if (first && x == hint_x && hint_i >= b && hint_i < e && A.cum[hint_i] <= bc + kk) {
                lo = hint_i;
                const int64_t w = min(e, hint_i + 64);
                if (w == e || A.cum[w] > bc + kk) hi = w;
            }
            i = upper_bound_u64(A.cum, lo, hi, bc + kk) - 1;
            k2 = kk - (A.cum[i] - bc);
        }
        if (first) {
            if (first_i) *first_i = i;
            if (first_x) *first_x = x;
            first = false;
        }
        const ItemS it = A.items[i];
        S += it.A + ((uint64_t)(uint32_t)it.B * (2u * pos) + ((uint64_t)((uint32_t)(it.B >> 32) * (2u * pos)) << 32));
        pos += (uint32_t)it.len;
        if (it.x < 0) {  // a tail segment ends the path (test paths: then the suffix walk of its last vertex)
            if (A.tp != nullptr && !tp_tail(A.tp, it.last, S, pos)) atomicOr(A.unreachable, 1u);
            break;
        }
        const int4 mi = __ldg(reinterpret_cast<const int4 *>(&slots[it.x].gid));
        for (int a = 0; a < mi.z; a++) {  // the out-arc of the transit whose completions hold k2
            const int32_t ya = __ldg(G.out_gid + mi.y + a);
            const uint64_t Wy = __ldg(G.Wc + ya);
            if (k2 < Wy) {
                x = ya;
                break;
            }
            k2 -= Wy;
        }
        kk = k2;
    }
    sa += mix64(S ^ (kSeedA + (uint64_t)pos));
    sb += mix64(S ^ (kSeedB + (uint64_t)pos));
    sv += pos;
}

// acc[0], acc[1]: digest; acc[2]: vertices of the hashed paths (test paths: the only place their
// suffix walks are known)
__device__ __forceinline__ void hash_flush(uint64_t sa, uint64_t sb, uint64_t sv, unsigned long long *acc) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        sa += __shfl_xor_sync(kFull, sa, d);
        sb += __shfl_xor_sync(kFull, sb, d);
        sv += __shfl_xor_sync(kFull, sv, d);
    }
    if ((threadIdx.x & 31) == 0 && (sa | sb | sv)) {
        atomicAdd(acc, (unsigned long long)sa);
        atomicAdd(acc + 1, (unsigned long long)sb);
        atomicAdd(acc + 2, (unsigned long long)sv);
    }
}

constexpr uint64_t kSmallHead = 32;  // heads with at most this many completions: one thread each
constexpr int kBigWarpRun = 8;       // stitch_big: steps of 32 consecutive completions per warp chunk

// Small heads: one thread per head slot hashes all of its W <= kSmallHead completions (no search
// over the heads); big[h] = 1 marks the others for stitch_big_kernel.
__global__ void stitch_small_kernel(StitchSArgs A, DevGraph G, uint64_t *big, unsigned long long *acc) {
    uint64_t sa = 0, sb = 0, sv = 0;
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < A.n_heads; h += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t w = ((h + 1 < A.n_heads) ? A.comp_off[h + 1] : A.n_comp) - A.comp_off[h];
        big[h] = w > kSmallHead ? 1 : 0;
        if (w == 0 || w > kSmallHead) continue;
        const HeadS H = A.heads[h];
        for (uint64_t k = 0; k < w; k++) hash_completion(A, G, H, k, sa, sb, sv);
    }
    hash_flush(sa, sb, sv, acc);
}
// big heads, compacted: idx[j] = head slot, w[j] = its completion count
__global__ void stitch_big_list_kernel(StitchSArgs A, const uint64_t *pos, int64_t *idx, uint64_t *w) {
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < A.n_heads; h += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t wh = ((h + 1 < A.n_heads) ? A.comp_off[h + 1] : A.n_comp) - A.comp_off[h];
        if (wh > kSmallHead) {
            idx[pos[h]] = h;
            w[pos[h]] = wh;
        }
    }
}
// big heads: one thread per completion (a binary search over the few big heads' offsets)
__global__ void stitch_big_kernel(StitchSArgs A, DevGraph G, const int64_t *idx, const uint64_t *off, int64_t n_big,
                                  uint64_t n_big_comp, unsigned long long *acc) {
    uint64_t sa = 0, sb = 0, sv = 0;
    const int lane = threadIdx.x & 31;
    // a warp takes kBigWarpRun * 32 consecutive completions, lane l the ones at l + 32 t: a lane's
    // first-level item moves forward by about 32 per step, so its search after the first starts at
    // its previous item (a window of 64) instead of spanning the whole entry group
    const uint64_t chunk = (uint64_t)kBigWarpRun * 32;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t c0 = (((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * chunk; c0 < n_big_comp;
         c0 += warps * chunk) {
        int64_t pi = -1;
        int32_t px = -1;
        for (int t = 0; t < kBigWarpRun; t++) {
            const uint64_t g = c0 + (uint64_t)t * 32 + lane;
            if (g >= n_big_comp) break;
            const int64_t j = upper_bound_u64(off, 0, n_big, g) - 1;
            int64_t fi = -1;
            int32_t fx = -1;
            hash_completion(A, G, A.heads[idx[j]], g - off[j], sa, sb, sv, px, pi, &fi, &fx);
            pi = fi;
            px = fx;
        }
    }
    hash_flush(sa, sb, sv, acc);
}

__global__ void fill_u32_kernel(uint32_t *p, uint32_t v, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void set_last_offset_kernel(int64_t *off, int64_t n_paths, int64_t total) { off[n_paths] = total; }

// ------------------------------------------------------------- digest (K8)

__global__ void digest_kernel(const int64_t *off, const int32_t *vert, int64_t n, unsigned long long *acc) {
    uint64_t a = 0, b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = off[i], e = off[i + 1];
        PathHash h;
        h.init((uint64_t)(e - s));
        for (int64_t j = s; j < e; j++) h.add(__ldg(vert + j));
        h.fin();
        a += h.a;
        b += h.b;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        a += __shfl_xor_sync(kFull, a, d);
        b += __shfl_xor_sync(kFull, b, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, (unsigned long long)a);
        atomicAdd(acc + 1, (unsigned long long)b);
    }
}

// --------------------------------------------------------- test paths (K6)
struct TpArgs {
    const int64_t *pp_off;
    const int32_t *pp_vert;
    int64_t n;
    const int64_t *pre_off, *suf_off;
    const int32_t *pre_len, *suf_len;
    const int32_t *pre_flat, *suf_flat;
    uint64_t *tp_len;  // then scanned into offsets
    int64_t *tp_off;
    int32_t *tp_vert;
    unsigned int *unreachable;
};

__global__ void tp_len_kernel(TpArgs A) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = A.pp_off[i], e = A.pp_off[i + 1];
        const int32_t f = A.pp_vert[s], l = A.pp_vert[e - 1];
        const int32_t pl = A.pre_len[f], sl = A.suf_len[l];
        if (pl < 0 || sl < 0) {
            atomicOr(A.unreachable, 1u);
            A.tp_len[i] = 0;
        } else {
            A.tp_len[i] = (uint64_t)(pl - 1) + (uint64_t)(e - s) + (uint64_t)(sl - 1);
        }
    }
}

// Flat prefix / suffix walk tables from the two walk trees: vertex v's prefix is
// the BFS-tree path entry -> v (written backwards along parents), its suffix the
// greedy walk v -> exit along next (R15).
__global__ void tp_flat_kernel(int32_t n, const int32_t *parent, const int32_t *next, const int64_t *pre_off,
                               const int32_t *pre_len, const int64_t *suf_off, const int32_t *suf_len,
                               int32_t *pre_flat, int32_t *suf_flat) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int32_t pl = pre_len[v];
        if (pl > 0) {
            int32_t *d = pre_flat + pre_off[v];
            int32_t c = v;
            for (int32_t j = pl - 1; j >= 0; j--) {
                d[j] = c;
                c = __ldg(parent + c);
            }
        }
        const int32_t sl = suf_len[v];
        if (sl > 0) {
            int32_t *d = suf_flat + suf_off[v];
            int32_t c = v;
            for (int32_t j = 0; j < sl; j++) {
                d[j] = c;
                c = __ldg(next + c);
            }
        }
    }
}

// Test-path digest terms per slot (TpTerm, kernels.cuh) from the flat walk tables: the prefix
// walk of v minus its last vertex from position 0, the suffix walk minus its first vertex.
__global__ void tp_terms_kernel(int32_t n, const int32_t *slot_gid, const uint64_t *vmix, const int64_t *pre_off,
                                const int32_t *pre_len, const int64_t *suf_off, const int32_t *suf_len,
                                const int32_t *pre_flat, const int32_t *suf_flat, TpTerm *out) {
    for (int32_t sl = blockIdx.x * blockDim.x + threadIdx.x; sl < n; sl += gridDim.x * blockDim.x) {
        const int32_t v = slot_gid[sl];
        TpTerm t;
        t.pre_len = pre_len[v];
        t.suf_len = suf_len[v];
        t.S_pre = t.A_suf = t.B_suf = 0;
        for (int32_t j = 0; j + 1 < t.pre_len; j++)
            t.S_pre += __ldg(vmix + pre_flat[pre_off[v] + j]) * (2 * (uint64_t)j + 1);
        for (int32_t j = 1; j < t.suf_len; j++) {
            const uint64_t m = __ldg(vmix + suf_flat[suf_off[v] + j]);
            t.A_suf += m * (2 * (uint64_t)(j - 1) + 1);
            t.B_suf += m;
        }
        out[sl] = t;
    }
}

// COUNT_HASH test paths of a given canonical prime-path list: per path its digest sum S and
// mix sum B from its vertices, then the test path's terms (one thread per path).
__global__ void tp_hash_list_kernel(const int64_t *off, const int32_t *vert, int64_t n, const int32_t *v_slot,
                                    const uint64_t *vmix, const TpTerm *tp, unsigned long long *acc,
                                    unsigned int *unreachable) {
    uint64_t sa = 0, sb = 0, nv = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = off[i], e = off[i + 1];
        uint64_t S = 0, B = 0;
        for (int64_t j = a; j < e; j++) {
            const uint64_t m = __ldg(vmix + vert[j]);
            S += m * (2 * (uint64_t)(j - a) + 1);
            B += m;
        }
        uint32_t len = (uint32_t)(e - a);
        if (!tp_head(tp, __ldg(v_slot + vert[a]), S, B, len) || !tp_tail(tp, __ldg(v_slot + vert[e - 1]), S, len)) {
            atomicOr(unreachable, 1u);
            continue;
        }
        sa += mix64(S ^ (kSeedA + (uint64_t)len));
        sb += mix64(S ^ (kSeedB + (uint64_t)len));
        nv += len;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        sa += __shfl_xor_sync(kFull, sa, d);
        sb += __shfl_xor_sync(kFull, sb, d);
        nv += __shfl_xor_sync(kFull, nv, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, (unsigned long long)sa);
        atomicAdd(acc + 1, (unsigned long long)sb);
        atomicAdd(acc + 2, (unsigned long long)nv);
    }
}

// Class of every prime path from its end vertices (complete, entry, exit, internal,
// transit -- DESIGN.md R19); a path cannot leave an SCC and return, so it lies in
// one SCC iff its end vertices do.  Counts reduced per warp, one atomic each.
__global__ void classify_kernel(const int64_t *off, const int32_t *vert, int64_t n, const int32_t *comp,
                                int32_t start, int32_t end, unsigned long long *counts) {
    unsigned long long c[5] = {0, 0, 0, 0, 0};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = vert[off[i]], l = vert[off[i + 1] - 1];
        const int k = (f == start) ? ((l == end) ? 0 : 1) : ((l == end) ? 2 : ((comp[f] == comp[l]) ? 3 : 4));
#pragma unroll
        for (int q = 0; q < 5; q++) c[q] += (k == q);
    }
#pragma unroll
    for (int q = 0; q < 5; q++) {
#pragma unroll
        for (int d = 16; d; d >>= 1) c[q] += __shfl_xor_sync(kFull, c[q], d);
        if ((threadIdx.x & 31) == 0 && c[q]) atomicAdd(counts + q, c[q]);
    }
}

// Warp copy of n int32 with eight loads in flight per lane.
__device__ __forceinline__ void warp_copy(int32_t *dst, const int32_t *src, int64_t n, int lane) {
    int64_t j = lane;
    for (; j + 224 < n; j += 256) {
        int32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = __ldg(src + j + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; u++) dst[j + 32 * u] = v[u];
    }
    for (; j < n; j += 32) dst[j] = __ldg(src + j);
}

__global__ void tp_write_kernel(TpArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = wg; i < A.n; i += nw) {
        const int64_t s = A.pp_off[i], e = A.pp_off[i + 1];
        const int32_t f = A.pp_vert[s], l = A.pp_vert[e - 1];
        const int32_t pl = A.pre_len[f] - 1, sl = A.suf_len[l] - 1;
        const int64_t t0 = (int64_t)A.tp_len[i];
        if (lane == 0) A.tp_off[i] = t0;
        int32_t *d = A.tp_vert + t0;
        warp_copy(d, A.pre_flat + A.pre_off[f], pl, lane);
        d += pl;
        warp_copy(d, A.pp_vert + s, e - s, lane);
        d += e - s;
        warp_copy(d, A.suf_flat + A.suf_off[l] + 1, sl, lane);
    }
}

// ---------------------------------------------------------------- K7: sorted-unique test paths
// Lexicographic order of int32 sequences (R14; a proper prefix sorts first) on indices into a
// flat path array: the comparator of the device merge sort.
struct SeqLess {
    const int64_t *off;
    const int32_t *v;
    __device__ __forceinline__ bool operator()(const int64_t &a, const int64_t &b) const {
        int64_t ia = off[a], ib = off[b];
        const int64_t ea = off[a + 1], eb = off[b + 1];
        for (; ia < ea && ib < eb; ia++, ib++) {
            const int32_t x = v[ia], y = v[ib];
            if (x != y) return x < y;
        }
        return (ea - ia) < (eb - ib);
    }
};

__global__ void iota_kernel(int64_t *idx, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) idx[i] = i;
}

// After the sort: keep[i] = the i-th path differs from the (i-1)-th; len = its length if kept
// (both scanned into the unique list's index and vertex offsets).
__global__ void tp_unique_mark_kernel(const int64_t *idx, int64_t n, const int64_t *off, const int32_t *v,
                                      uint64_t *keep, uint64_t *len, uint8_t *kept) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx[i], sb = off[b], eb = off[b + 1];
        bool k = true;
        if (i > 0) {
            const int64_t a = idx[i - 1], sa = off[a], ea = off[a + 1];
            if (ea - sa == eb - sb) {
                k = false;
                for (int64_t q = 0; q < eb - sb; q++)
                    if (v[sa + q] != v[sb + q]) {
                        k = true;
                        break;
                    }
            }
        }
        keep[i] = k ? 1 : 0;
        len[i] = k ? (uint64_t)(eb - sb) : 0;
        kept[i] = k ? 1 : 0;
    }
}

// One warp per kept path: its offset, then its vertices (coalesced copy).
__global__ void tp_unique_gather_kernel(const int64_t *idx, int64_t n, const int64_t *off, const int32_t *v,
                                        const uint64_t *pos, const uint64_t *vpos, const uint8_t *kept,
                                        int64_t *out_off, int32_t *out_v) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = wg; i < n; i += nw) {
        if (!kept[i]) continue;
        const int64_t b = idx[i], sb = off[b], L = off[b + 1] - sb;
        if (lane == 0) out_off[pos[i]] = (int64_t)vpos[i];
        for (int64_t q = lane; q < L; q += 32) out_v[vpos[i] + q] = v[sb + q];
    }
}

}  // namespace tpg
