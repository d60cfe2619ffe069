// alg3.cuh -- the paper's vertex-centric, self-stabilizing PP generator (PAPER.md
// Alg. 1-4) as a B200 comparison kernel (TPGEN_ENGINE_ALG3;
// SURVEY §8(f) NEXT #4).
//
// What is the paper's: every vertex v_i owns a list of simple paths ending at v_i,
// initialised to {<v_i>} (Alg. 2); ONE kernel launch (Alg. 1) in which v_i's
// worker repeatedly reads its predecessors' lists, labels each path q "read by v_i"
// (Alg. 3 l.11-12), extends the eligible ones -- q not a cycle and (v_i not on q, or v_i
// the first vertex of q) -- by ExtendPath (Alg. 4: append v_i, length + 1, the cyclic
// flag when v_i is q's first vertex) into its own list and labels q "extended"
// (l.13-15); a worker may stop only when every path of its list has been read by all
// its successors (LocalFlag, l.21-25) and every backward-reachable vertex has stopped
// (PublicFlag, l.26-32); no atomic instruction anywhere.  What remains of
// v_i's list -- paths read by both successors that were neither extended nor "included
// in some path p' in v_i.list" (l.2-8) -- are the PPs finished at v_i.
//
// What is B200's (each change keeps the algorithm's result):
//  * a worker is one CTA of 1024 threads (not one thread): a predecessor's unread
//    paths are read 4096 at a time, and the CTA appends the extensions to its own
//    list through a block scan -- still a single writer per list, so no atomics;
//  * "q read by v_i" is a cursor per arc (u, v_i): lists are append-only and read in
//    order, so the paths of u.list below the cursor are exactly those labelled read;
//  * a path is a record {visited mask (W words), digest sum S (R20), first | len |
//    cyclic}, not a copy of its vertex sequence: eligibility needs only the mask;
//  * "p is included in some path p' in v_i.list" is decided by the mask test
//    pred(first(p)) within p (R3's head half): at the fixpoint v_i.list holds every
//    simple path ending at v_i, and an acyclic p is a proper (suffix) sub-path of one
//    of them iff some predecessor x of its first vertex is off p (x + p is then a
//    simple path ending at v_i); the paper's pairwise comparison of list entries is
//    quadratic in the list length (1e7 paths per list on config 3);
//  * PublicFlag[v] is the number of predecessor paths v has consumed, published after
//    v's own list count; a worker stops when, reading all consumed counters of its
//    backward-reachable set B(v) first and the list counts after, every x in B(v) has
//    consumed every path of its predecessors (a stable state: nothing is unread and
//    no list can grow), and its successors' cursors cover its own list (LocalFlag);
//  * the final pass over v's list (l.2-8 once, at the fixpoint) counts, sums the
//    lengths and hashes the surviving paths (the R20 digest) into v's partial sums;
//    the host adds the n partials (no atomics).
// All lists live in HBM at once (the paper's space cost): a graph of N simple
// paths needs ~N records.  Workers must be co-resident (cooperative launch): n <= 128.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace tpg {

constexpr int kA3Threads = 1024;
constexpr int kA3Rec = 4;  // records per thread per tile (loads first: 4 in flight)
constexpr int kA3Tile = kA3Threads * kA3Rec;

struct A3Args {
    int32_t n;
    unsigned long long cap;       // records per vertex list
    const int64_t *po;            // predecessor CSR (global ids)
    const int32_t *pt;
    const int64_t *so;            // successor CSR
    const int32_t *sv;
    const int32_t *pidx;          // for the k-th predecessor entry of v: the index of arc (u, v) in the successor CSR
    const uint64_t *vmix;         // mix64(v) per vertex (R20)
    const uint64_t *pinm;         // [v * W + w]: predecessor set of v (bits over global ids)
    const uint64_t *back;         // [v * W + w]: B(v), the vertices v is reachable from (v included)
    uint64_t *mask;               // [w][v * cap + i]
    uint64_t *S;                  // [v * cap + i]
    uint32_t *meta;               // [v * cap + i]: first | len << 8 | cyclic << 16
    uint8_t *ext;                 // [v * cap + i]: extended by some successor (Alg. 4 caller, l.15)
    unsigned long long *count;    // [v]: records published in v.list
    unsigned long long *consumed; // [v]: predecessor records v has read (the PublicFlag's content)
    unsigned long long *cursor;   // [arc (u, w) in successor-CSR order]: records of u.list read by w
    unsigned long long *part;     // [v * 8 + k]: pp, vertices, digest a, digest b, records, overflow
};

__device__ __forceinline__ unsigned long long a3_ld_acq(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void a3_st_rel(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int W>
__global__ void __launch_bounds__(kA3Threads, 1) alg3_kernel(A3Args A) {
    __shared__ unsigned long long s_cur[128];  // per in-arc: records of the predecessor's list read
    __shared__ unsigned long long s_end[128];  // per in-arc: the predecessor's published count (this round)
    __shared__ uint32_t s_wsum[kA3Threads / 32];
    __shared__ int s_flag;
    const int v = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long cap = A.cap, base = (unsigned long long)v * cap, ntot = (unsigned long long)A.n * cap;
    const int64_t p0 = A.po[v], np = A.po[v + 1] - p0;
    const uint64_t mv = A.vmix[v];
    const int vw = v >> 6;
    const uint64_t vb = 1ull << (v & 63);
    for (int k = tid; k < (int)np; k += blockDim.x) s_cur[k] = 0;
    // Alg. 2: v.list = {<v>}
    if (tid == 0) {
#pragma unroll
        for (int w = 0; w < W; w++) A.mask[(size_t)w * ntot + base] = (w == vw) ? vb : 0ull;
        A.S[base] = mv;  // mix(v) * (2*0 + 1)
        A.meta[base] = (uint32_t)v | (1u << 8);
        A.ext[base] = 0;
        __threadfence();
        a3_st_rel(A.count + v, 1ull);
    }
    __syncthreads();
    unsigned long long my = 1;  // records in v.list (block-uniform)
    bool ovf = false;
    // Alg. 3 l.1: while PublicFlag
    for (;;) {
        bool did = false;
        __syncthreads();  // (every thread is done with the last round's s_end)
        for (int k = tid; k < (int)np; k += blockDim.x) s_end[k] = a3_ld_acq(A.count + A.pt[p0 + k]);
        __threadfence();
        __syncthreads();
        for (int k = 0; k < (int)np; k++) {  // l.9: each predecessor u
            const int u = A.pt[p0 + k];
            const unsigned long long end = s_end[k], cur = s_cur[k];
            if (end == cur) continue;
            const unsigned long long ub = (unsigned long long)u * cap;
            for (unsigned long long t0 = cur; t0 < end; t0 += kA3Tile) {  // l.10: each unread path q of u.list
                uint64_t qm[kA3Rec][W], qS[kA3Rec];
                uint32_t qmeta[kA3Rec];
#pragma unroll
                for (int r = 0; r < kA3Rec; r++) {
                    const unsigned long long i = t0 + (unsigned long long)r * kA3Threads + tid;
                    const bool in = i < end;
#pragma unroll
                    for (int w = 0; w < W; w++) qm[r][w] = in ? __ldcg(A.mask + (size_t)w * ntot + ub + i) : 0ull;
                    qS[r] = in ? __ldcg(A.S + ub + i) : 0ull;
                    qmeta[r] = in ? __ldcg(A.meta + ub + i) : (1u << 16);  // (out of range: "cyclic", never eligible)
                }
                uint32_t el = 0, nel = 0;
#pragma unroll
                for (int r = 0; r < kA3Rec; r++) {
                    const uint32_t f = qmeta[r] & 0xffu;
                    const bool cyc = (qmeta[r] >> 16) & 1u;
                    const bool on = (qm[r][vw] & vb) != 0;
                    const bool e = !cyc && (!on || f == (uint32_t)v);  // l.13
                    if (e) {
                        el |= 1u << r;
                        nel++;
                        A.ext[ub + t0 + (unsigned long long)r * kA3Threads + tid] = 1;  // l.15
                    }
                }
                // block scan of the eligible counts: positions in v.list (single writer: this CTA)
                uint32_t inc = nel;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += x;
                }
                if (lane == 31) s_wsum[warp] = inc;
                __syncthreads();
                uint32_t woff = 0, tot = 0;
                for (int x = 0; x < kA3Threads / 32; x++) {
                    const uint32_t s = s_wsum[x];
                    woff += (x < warp) ? s : 0u;
                    tot += s;
                }
                unsigned long long j = my + woff + inc - nel;
#pragma unroll
                for (int r = 0; r < kA3Rec; r++) {
                    if (!((el >> r) & 1u)) continue;
                    if (j < cap) {  // Alg. 4 ExtendPath(q, v): append v, len + 1, cyclic if v == first
                        const uint32_t f = qmeta[r] & 0xffu, len = (qmeta[r] >> 8) & 0xffu;
#pragma unroll
                        for (int w = 0; w < W; w++) A.mask[(size_t)w * ntot + base + j] = qm[r][w] | (w == vw ? vb : 0ull);
                        A.S[base + j] = qS[r] + mv * (2ull * len + 1ull);
                        A.meta[base + j] = f | ((len + 1u) << 8) | ((f == (uint32_t)v) ? (1u << 16) : 0u);
                        A.ext[base + j] = 0;
                    }
                    j++;
                }
                if (my + tot > cap) ovf = true;
                my = min(my + tot, cap);
                __syncthreads();  // (s_wsum is rewritten by the next tile)
            }
            // publish: v's new records, then the cursor of arc (u, v) (the "read by v" labels)
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                a3_st_rel(A.count + v, my);
                a3_st_rel(A.cursor + A.pidx[p0 + k], end);
                s_cur[k] = end;
            }
            did = true;
            __syncthreads();
        }
        // PublicFlag: the predecessor records consumed (published after the list count)
        if (tid == 0) {
            unsigned long long c = 0;
            for (int k = 0; k < (int)np; k++) c += s_cur[k];
            __threadfence();
            a3_st_rel(A.consumed + v, c);
        }
        if (did) continue;
        // termination test (l.21-32) by warp 0: consumed counters of B(v) first, list counts after
        if (warp == 0) {
            bool ok = true;
            unsigned long long cs[128 / 32];
#pragma unroll
            for (int q = 0; q < 128 / 32; q++) {
                const int x = q * 32 + lane;
                cs[q] = 0;
                if (x < A.n && ((A.back[(size_t)v * W + (x >> 6)] >> (x & 63)) & 1ull)) cs[q] = a3_ld_acq(A.consumed + x);
            }
            __threadfence();
#pragma unroll
            for (int q = 0; q < 128 / 32; q++) {
                const int x = q * 32 + lane;
                if (x < A.n && ((A.back[(size_t)v * W + (x >> 6)] >> (x & 63)) & 1ull)) {
                    unsigned long long sum = 0;
                    for (int64_t e = A.po[x]; e < A.po[x + 1]; e++) sum += a3_ld_acq(A.count + A.pt[e]);
                    ok = ok && (sum == cs[q]);
                }
            }
            // LocalFlag: every path of v.list read by all successors
            for (int64_t e = A.so[v] + lane; e < A.so[v + 1]; e += 32) ok = ok && (a3_ld_acq(A.cursor + e) == my);
            ok = __all_sync(0xffffffffu, ok);
            if (lane == 0) s_flag = ok;
        }
        __syncthreads();
        const bool stop = s_flag;
        __syncthreads();  // (s_flag is rewritten by the next test)
        if (stop) break;
        __nanosleep(256);
    }
    __threadfence();
    // l.2-8 at the fixpoint: the paths of v.list neither extended nor covered are the PPs finished at v
    unsigned long long pp = 0, vert = 0, ha = 0, hb = 0;
    for (unsigned long long i = tid; i < my; i += blockDim.x) {
        if (__ldcg(A.ext + base + i)) continue;
        const uint32_t m = __ldcg(A.meta + base + i);
        const uint32_t f = m & 0xffu, len = (m >> 8) & 0xffu;
        bool keep = (m >> 16) & 1u;  // a cycle is never extended, never covered
        if (!keep) {                 // covered iff some predecessor of first(p) is off p
            keep = true;
#pragma unroll
            for (int w = 0; w < W; w++) keep = keep && (__ldg(A.pinm + (size_t)f * W + w) & ~__ldcg(A.mask + (size_t)w * ntot + base + i)) == 0;
        }
        if (keep) {
            const uint64_t s = __ldcg(A.S + base + i);
            pp++;
            vert += len;
            ha += mix64(s ^ (kSeedA + (uint64_t)len));
            hb += mix64(s ^ (kSeedB + (uint64_t)len));
        }
    }
    __shared__ unsigned long long red[4][kA3Threads / 32];
    unsigned long long val[4] = {pp, vert, ha, hb};
#pragma unroll
    for (int q = 0; q < 4; q++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val[q] += __shfl_down_sync(0xffffffffu, val[q], o);
        if (lane == 0) red[q][warp] = val[q];
    }
    __syncthreads();
    if (tid < 4) {
        unsigned long long a = 0;
        for (int x = 0; x < kA3Threads / 32; x++) a += red[tid][x];
        A.part[(size_t)v * 8 + tid] = a;
    }
    if (tid == 0) {
        A.part[(size_t)v * 8 + 4] = my;
        A.part[(size_t)v * 8 + 5] = ovf ? 1ull : 0ull;
    }
}

}  // namespace tpg
