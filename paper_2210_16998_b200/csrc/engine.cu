// engine.cu -- host orchestration of the device pipeline of libtpgen.
//
// tpgen_prime_paths (SURVEY.md §3 "Build 1"):
//   plan (host)  -> roots (one unit per start vertex, canonical order)
//   segment phase (entry starts): DFS rounds [dfs_kernel + refine]
//   completion DP over the component DAG (host, KBs)
//   prime-path phase (non-entry starts): DFS rounds  -- the dominant kernel
//   scan of the per-unit counts -> exact output offsets
//   expand_kernel: record streams -> canonical offsets/vertices
//   segment-table scans + stitch_kernel (cross-SCC prime paths)
//   optional digest, optional D2H
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <type_traits>

#include <cub/device/device_merge_sort.cuh>
#include <nvtx3/nvToolsExt.h>

#include "aux_kernels.cuh"
#include "expand.cuh"
#include "frontier.cuh"
#include "alg3.cuh"
#include "count.cuh"
#include "engine.h"

namespace tpg {

// NVTX range over a host-side stage (SURVEY §5 tracing): the kernels a stage launches appear
// under its name in ncu (--nvtx) / nsys timelines; a no-op unless a tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

#define TPG_CK(x)                                                                                      \
    do {                                                                                               \
        cudaError_t _e = (x);                                                                          \
        if (_e != cudaSuccess) {                                                                       \
            set_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " #x);                \
            return _e == cudaErrorMemoryAllocation ? TPGEN_ERR_OUT_OF_MEMORY : TPGEN_ERR_CUDA;         \
        }                                                                                              \
    } while (0)

#define TPG_TRY(x)                        \
    do {                                  \
        tpgen_status _s = (x);            \
        if (_s != TPGEN_OK) return _s;    \
    } while (0)

static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------ buffers
static void out_cache_clear(int dev);

// Stream-ordered allocation from the device pool; on failure the cached output
// blocks and the pool's idle memory are released and the allocation retried once.
static cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t s) {
    cudaError_t e = cudaMallocAsync(p, bytes, s);
    if (e == cudaSuccess) return e;
    cudaGetLastError();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaStreamSynchronize(s);
    out_cache_clear(dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    return cudaMallocAsync(p, bytes, s);
}

tpgen_status DevBuf::ensure(size_t bytes, cudaStream_t s) {
    if (bytes <= cap) return TPGEN_OK;
    // 25 % headroom: per-call sizes (units, records) vary with the dynamic donation pattern,
    // and a regrowth inside a later call costs a fresh mapping from the pool
    size_t nc = std::max(bytes + bytes / 4, (size_t)(cap * 3 / 2));
    nc = (nc + 255) & ~(size_t)255;
    if (p) TPG_CK(cudaFreeAsync(p, s));
    p = nullptr;
    cap = 0;
    TPG_CK(pool_alloc(&p, nc, s));
    cap = nc;
    return TPGEN_OK;
}
tpgen_status DevBuf::ensure_exact(size_t bytes, cudaStream_t s) {
    if (bytes <= cap) return TPGEN_OK;
    const size_t nc = (bytes + 255) & ~(size_t)255;
    if (p) TPG_CK(cudaFreeAsync(p, s));
    p = nullptr;
    cap = 0;
    TPG_CK(pool_alloc(&p, nc, s));
    cap = nc;
    return TPGEN_OK;
}

void DevBuf::release(cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    cap = 0;
}

template <class T>
static tpgen_status upload(DevBuf &b, const std::vector<T> &v, cudaStream_t s) {
    size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
    TPG_TRY(b.ensure(bytes, s));
    if (!v.empty()) TPG_CK(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return TPGEN_OK;
}

// splitmix64 finalizer (the digest's per-vertex value, R20; the device has its own copy)
static uint64_t host_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}

// ------------------------------------------------------------ plan
PlanImpl::~PlanImpl() {
    if (!dev_ok) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStream_t s = 0;
    for (DevBuf *b : all_bufs()) b->release(s);
    cudaStreamSynchronize(s);
    if (prev >= 0) cudaSetDevice(prev);
}

std::vector<DevBuf *> PlanImpl::all_bufs() {
    std::vector<DevBuf *> v = {&d_slots, &d_slot_gid, &d_out_gid, &d_out_pos, &d_scc_vbase, &d_scc_out_base,
                               &d_scc_nout, &d_scc_pair_base, &d_slot_eidx, &d_Wc, &d_Wv, &d_scc_gbase, &d_comp, &d_v_slot, &d_slot_mix, &d_vmix, &d_scc_exm, &d_slot_d2, &cheads, &tp_terms, &citems, &citems2, &icnt,
                               &qunits, &qready, &qext, &qrfirst, &qrcount, &qchead, &blk_first, &blk_count, &blk_next, &qgen, &roots, &qparent, &qnchild,
                               &scan_b, &scan_tot, &ctr, &agg, &agg_bak, &heads, &head_pool, &items, &item_pool,
                               &icum, &ivcum, &ibeg, &iend, &hcomp, &offs, &tp_tabs, &chunks, &dbgbuf, &qctr, &sscratch, &presplit_dev, &presplit_roots, &rscan,
                               &f_tab, &f_roots, &f_buf0, &f_buf1, &f_ctr, &f_sched, &a3_lists, &a3_aux};
    for (int c = 0; c < kCnt; c++) v.push_back(&qcnt[c]);
    return v;
}

tpgen_status plan_upload(PlanImpl &P, cudaStream_t s) {
    NvtxRange nvtx_range("tpgen: plan upload");
    const HostPlan &H = P.hp;
    // pack Slot<W> records (sin[W], pin[W], gid, out_off, out_cnt, flags)
    const int W = H.W;
    const size_t rec = 16 * (size_t)W + 16;
    std::vector<uint8_t> packed(std::max<size_t>((size_t)H.n * rec, 16), 0);
    for (int32_t i = 0; i < H.n; i++) {
        uint8_t *r = packed.data() + (size_t)i * rec;
        memcpy(r, &H.sin[(size_t)i * W], 8 * W);
        memcpy(r + 8 * W, &H.pin[(size_t)i * W], 8 * W);
        const int32_t meta[4] = {H.slot_gid[i], H.slot_out_off[i], H.slot_out_cnt[i], H.slot_flags[i]};
        memcpy(r + 16 * W, meta, 16);
    }
    P.presplit_lo = P.presplit_hi = -1;  // a new graph: the cached pre-split roots are stale
    P.presplit_key = P.pfx_key = -1;
    P.presplit_n = 0;
    P.presplit_roots_n = -1;
    P.f_tab_ok = false;  // frontier engine: slot table, roots and record high-water mark belong to the old graph
    P.f_roots_lo = P.f_roots_hi = -1;
    P.f_cap_hwm = 0;
    P.any_exit = false;  // no arc leaves any SCC: the LEAN DFS applies
    for (int32_t i = 0; i < H.n; i++)
        if (H.slot_out_cnt[i] > 0 || (H.slot_flags[i] & (F_EXIT | F_ENTRY))) P.any_exit = true;
    TPG_TRY(upload(P.d_slots, packed, s));
    TPG_TRY(upload(P.d_slot_gid, H.slot_gid, s));
    std::vector<int32_t> gbase(std::max(H.n_scc, 1), -1);
    for (int32_t c = 0; c < H.n_scc; c++) {
        const int32_t vb = H.scc_vbase[c], L = H.scc_size[c];
        if (L > 0 && H.slot_gid[vb + L - 1] - H.slot_gid[vb] == L - 1) gbase[c] = H.slot_gid[vb];
    }
    TPG_TRY(upload(P.d_scc_gbase, gbase, s));
    TPG_TRY(upload(P.d_out_gid, H.out_gid, s));
    TPG_TRY(upload(P.d_out_pos, H.out_pos, s));
    TPG_TRY(upload(P.d_scc_vbase, H.scc_vbase, s));
    TPG_TRY(upload(P.d_scc_out_base, H.scc_out_base, s));
    TPG_TRY(upload(P.d_scc_nout, H.scc_nout, s));
    TPG_TRY(upload(P.d_scc_pair_base, H.scc_pair_base, s));
    TPG_TRY(upload(P.d_slot_eidx, H.slot_eidx, s));
    TPG_TRY(upload(P.d_comp, H.comp, s));
    TPG_TRY(upload(P.d_v_slot, H.v_slot, s));
    {  // digest values mix64(v) per global vertex and per slot (R20)
        std::vector<uint64_t> vm(std::max(H.n, 1), 0), sm(std::max(H.n, 1), 0);
        for (int32_t v = 0; v < H.n; v++) vm[v] = host_mix64((uint64_t)(uint32_t)v);
        for (int32_t i = 0; i < H.n; i++) sm[i] = vm[H.slot_gid[i]];
        TPG_TRY(upload(P.d_vmix, vm, s));
        TPG_TRY(upload(P.d_slot_mix, sm, s));
        std::vector<uint64_t> exm(std::max(H.n_scc, 1), 0);  // exit vertices per SCC (local bits; <= 64)
        for (int32_t c = 0; c < H.n_scc; c++)
            for (int32_t i = 0; i < H.scc_size[c] && i < 64; i++)
                if (H.slot_out_cnt[H.scc_vbase[c] + i] > 0) exm[c] |= 1ull << i;
        TPG_TRY(upload(P.d_scc_exm, exm, s));
        // out-degree-2 table of the count kernel's D2 variant (count.cuh): per slot the local ids of
        // its (at most 2) in-SCC successors t0 < t1 -- a missing one is the slot's OWN local id,
        // whose bit is always on the path when the slot is the child being taken -- the exit flag
        // (Def. 5) and the digest value mix64(gid)
        bool d2 = H.max_scc <= 64 && H.W == 1 && H.n < (1 << 23);  // (slots fit the queue tag, count.cuh)
        std::vector<uint64_t> t2(2 * (size_t)std::max(H.n, 1), 0);
        for (int32_t c = 0; c < H.n_scc && d2; c++)
            for (int32_t i = 0; i < H.scc_size[c]; i++) {
                const int32_t sl = H.scc_vbase[c] + i;
                uint64_t sn = H.sin[(size_t)sl * H.W];
                if (__builtin_popcountll(sn) > 2) {
                    d2 = false;
                    break;
                }
                const uint64_t t0 = sn ? (uint64_t)__builtin_ctzll(sn) : (uint64_t)i;
                sn &= sn - 1;
                const uint64_t t1 = sn ? (uint64_t)__builtin_ctzll(sn) : (uint64_t)i;
                // t0 and t1 in words of their own (shift amounts without masking), exit next to t1
                t2[2 * (size_t)sl] = t0 | (t1 << 32) | ((H.slot_out_cnt[sl] > 0 ? 1ull : 0ull) << 40);
                t2[2 * (size_t)sl + 1] = sm[sl];
            }
        if (const char *ev = getenv("TPGEN_NO_D2")) d2 = d2 && atoi(ev) == 0;  // A/B hook
        P.d2_ok = d2;
        if (d2) TPG_TRY(upload(P.d_slot_d2, t2, s));
    }
    P.chead_hwm = 0;
    TPG_TRY(P.d_Wc.ensure(std::max<size_t>(H.n, 1) * 8, s));
    TPG_TRY(P.d_Wv.ensure(std::max<size_t>(H.n, 1) * 8, s));
    TPG_CK(cudaMemsetAsync(P.d_Wc.p, 0, std::max<size_t>(H.n, 1) * 8, s));
    TPG_CK(cudaMemsetAsync(P.d_Wv.p, 0, std::max<size_t>(H.n, 1) * 8, s));
    P.dev_ok = true;
    return TPGEN_OK;
}

static DevGraph dev_graph(PlanImpl &P, int32_t lo, int32_t hi) {
    DevGraph G;
    G.slots = P.d_slots.p;
    G.slot_gid = P.d_slot_gid.as<int32_t>();
    G.out_gid = P.d_out_gid.as<int32_t>();
    G.out_pos = P.d_out_pos.as<int32_t>();
    G.scc_vbase = P.d_scc_vbase.as<int32_t>();
    G.scc_out_base = P.d_scc_out_base.as<int32_t>();
    G.scc_nout = P.d_scc_nout.as<int32_t>();
    G.scc_pair_base = P.d_scc_pair_base.as<int64_t>();
    G.slot_eidx = P.d_slot_eidx.as<int32_t>();
    G.Wc = P.d_Wc.as<uint64_t>();
    G.Wv = P.d_Wv.as<uint64_t>();
    G.scc_gbase = P.d_scc_gbase.as<int32_t>();
    G.slot_mix = P.d_slot_mix.as<uint64_t>();
    G.vmix = P.d_vmix.as<uint64_t>();
    G.scc_exm = P.d_scc_exm.as<uint64_t>();
    G.slot_d2 = P.d2_ok ? P.d_slot_d2.as<uint64_t>() : nullptr;
    G.v_slot = P.d_v_slot.as<int32_t>();
    G.comp = P.d_comp.as<int32_t>();
    G.shard_lo = lo;
    G.shard_hi = hi;
    return G;
}

// ------------------------------------------------------------ scan helper
static tpgen_status scan_multi(PlanImpl &P, uint64_t *const *arrs, int na, int64_t n, uint64_t *totals_host,
                               cudaStream_t s, int64_t &launches) {
    if (n <= 0) {
        for (int a = 0; a < na; a++) totals_host[a] = 0;
        return TPGEN_OK;
    }
    ScanArrays S;
    for (int a = 0; a < na; a++) S.a[a] = arrs[a];
    S.na = na;
    const int nb = (int)((n + kScanTile - 1) / kScanTile);
    TPG_TRY(P.scan_b.ensure((size_t)nb * na * 8, s));
    TPG_TRY(P.scan_tot.ensure(8 * 8, s));
    scan_reduce_kernel<<<nb, kScanThreads, 0, s>>>(S, n, P.scan_b.as<uint64_t>(), nb);
    scan_bsum_kernel<<<1, kScanThreads, 0, s>>>(P.scan_b.as<uint64_t>(), nb, na, P.scan_tot.as<uint64_t>());
    scan_down_kernel<<<nb, kScanThreads, 0, s>>>(S, n, P.scan_b.as<uint64_t>(), nb);
    launches += 3;
    TPG_CK(cudaGetLastError());
    if (totals_host) {
        TPG_CK(cudaMemcpyAsync(totals_host, P.scan_tot.p, na * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
    }
    return TPGEN_OK;
}

static int grid_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, cap));
}

// ------------------------------------------------------------ output memory
struct OutOwner {
    tpgen_free_fn free_fn = nullptr;
    void *ctx = nullptr;
    void *stream = nullptr;
    int kind = 0;  // 0 library pool block (offsets + vertices), 1 callback, 2 pinned host (library), 3 caller host buffer
    void *p_off = nullptr, *p_vert = nullptr;
    void *block = nullptr;  // kind 0: the one block holding both arrays
    size_t block_bytes = 0;
    int device = 0;
};

// Output blocks of the library pool are recycled through a small per-device
// cache: an output is one block (offsets, then vertices), and a block of the
// same size class is handed to the next call.  Without it the stream-ordered
// pool may carve a freed multi-GB block for smaller workspaces and then map
// fresh memory for the next output (hundreds of ms).
namespace {
struct OutCache {
    std::mutex mu;
    std::vector<std::pair<void *, size_t>> blocks;  // free blocks (their last use has completed)
};
OutCache g_outcache[64];
constexpr size_t kOutCacheMin = 1u << 20;  // smaller outputs go straight to the pool
constexpr size_t kOutCacheBlocks = 4;
}  // namespace

static void *out_cache_get(int dev, size_t bytes, size_t *got) {
    if (bytes < kOutCacheMin || dev < 0 || dev >= 64) return nullptr;
    OutCache &C = g_outcache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    int best = -1;
    for (int i = 0; i < (int)C.blocks.size(); i++) {
        const size_t sz = C.blocks[i].second;
        if (sz >= bytes && sz <= bytes + bytes / 2 && (best < 0 || sz < C.blocks[best].second)) best = i;
    }
    if (best < 0) return nullptr;
    void *p = C.blocks[best].first;
    *got = C.blocks[best].second;
    C.blocks.erase(C.blocks.begin() + best);
    return p;
}

// Takes a block whose last use has completed; false: not cached (caller frees it).
static bool out_cache_put(int dev, void *p, size_t bytes) {
    if (bytes < kOutCacheMin || dev < 0 || dev >= 64) return false;
    OutCache &C = g_outcache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    C.blocks.emplace_back(p, bytes);
    while (C.blocks.size() > kOutCacheBlocks) {
        cudaFree(C.blocks.front().first);
        C.blocks.erase(C.blocks.begin());
    }
    return true;
}

static void out_cache_clear(int dev) {
    if (dev < 0 || dev >= 64) return;  // (forward-declared above)
    OutCache &C = g_outcache[dev];
    std::lock_guard<std::mutex> lk(C.mu);
    for (auto &b : C.blocks) cudaFree(b.first);
    C.blocks.clear();
}

void release_output_cache(int dev) { out_cache_clear(dev); }

static tpgen_status out_alloc_device(const tpgen_options &o, OutOwner *ow, size_t bytes, void **p, cudaStream_t s);

// Offsets (int64[n+1]) and vertices (int32[...]) of one output.
static tpgen_status out_alloc_pair(const tpgen_options &o, OutOwner *ow, size_t b_off, size_t b_vert, void **d_off,
                                   void **d_vert, cudaStream_t s) {
    if (o.device_alloc) {
        TPG_TRY(out_alloc_device(o, ow, b_off, d_off, s));
        ow->p_off = *d_off;
        TPG_TRY(out_alloc_device(o, ow, b_vert, d_vert, s));
        ow->p_vert = *d_vert;
        return TPGEN_OK;
    }
    const size_t a_off = (b_off + 255) & ~(size_t)255;
    const size_t bytes = std::max<size_t>(a_off + b_vert, 256);
    size_t got = bytes;
    void *p = out_cache_get(ow->device, bytes, &got);
    if (!p) {
        TPG_CK(pool_alloc(&p, bytes, s));
    }
    ow->kind = 0;
    ow->stream = (void *)s;
    ow->block = p;
    ow->block_bytes = p ? got : 0;
    *d_off = p;
    *d_vert = (char *)p + a_off;
    return TPGEN_OK;
}

static tpgen_status out_alloc_device(const tpgen_options &o, OutOwner *ow, size_t bytes, void **p, cudaStream_t s) {
    bytes = std::max<size_t>(bytes, 16);
    if (o.device_alloc) {
        *p = o.device_alloc(bytes, o.stream, o.alloc_ctx);
        if (!*p) {
            set_error("device_alloc callback returned NULL");
            return TPGEN_ERR_OUT_OF_MEMORY;
        }
        ow->kind = 1;
        ow->free_fn = o.device_free;
        ow->ctx = o.alloc_ctx;
        ow->stream = o.stream;
    } else {
        TPG_CK(pool_alloc(p, bytes, s));
        ow->kind = 0;
        ow->stream = (void *)s;
    }
    return TPGEN_OK;
}

void free_paths(tpgen_paths *p) {
    if (!p) return;
    OutOwner *ow = (OutOwner *)p->_owner;
    if (ow) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(ow->device);
        if (ow->kind == 0) {
            if (ow->block) {
                cudaStreamSynchronize((cudaStream_t)ow->stream);  // last use complete: reusable on any stream
                if (!out_cache_put(ow->device, ow->block, ow->block_bytes)) {
                    cudaFreeAsync(ow->block, (cudaStream_t)ow->stream);
                    cudaStreamSynchronize((cudaStream_t)ow->stream);
                }
            }
        } else {
            void *ptrs[2] = {ow->p_off, ow->p_vert};
            for (void *q : ptrs) {
                if (!q) continue;
                if (ow->kind == 1) {
                    if (ow->free_fn) ow->free_fn(q, ow->stream, ow->ctx);
                } else if (ow->kind == 2) cudaFreeHost(q);
            }
        }
        if (prev >= 0) cudaSetDevice(prev);
        delete ow;
    }
    memset(p, 0, sizeof(*p));
}

// Places device arrays (off, vert) into *out according to the options.
static tpgen_status finish_output(const tpgen_options &o, OutOwner *ow, int64_t n_paths, int64_t n_vert, int64_t *d_off,
                                  int32_t *d_vert, cudaStream_t s, tpgen_paths *out) {
    out->n_paths = n_paths;
    out->device = ow->device;
    if (o.output_on_device) {
        out->offsets = d_off;
        out->vertices = d_vert;
        out->on_device = 1;
        ow->p_off = d_off;
        ow->p_vert = d_vert;
        out->_owner = ow;
        return TPGEN_OK;
    }
    size_t boff = (size_t)(n_paths + 1) * 8, bv = (size_t)n_vert * 4;
    OutOwner *hw = new OutOwner();
    hw->device = ow->device;
    char *h = nullptr;
    if (o.host_out && o.host_out_bytes >= boff + bv) {
        h = (char *)o.host_out;
        hw->kind = 3;
    } else {
        cudaError_t e = cudaHostAlloc((void **)&h, std::max<size_t>(boff + bv, 16), cudaHostAllocDefault);
        if (e != cudaSuccess) {
            delete hw;
            set_error("pinned host allocation failed");
            return TPGEN_ERR_OUT_OF_MEMORY;
        }
        hw->kind = 2;
        hw->p_off = h;
    }
    cudaMemcpyAsync(h, d_off, boff, cudaMemcpyDeviceToHost, s);
    if (bv) cudaMemcpyAsync(h + boff, d_vert, bv, cudaMemcpyDeviceToHost, s);
    TPG_CK(cudaStreamSynchronize(s));
    // release the device copies
    ow->p_off = d_off;
    ow->p_vert = d_vert;
    tpgen_paths tmp;
    memset(&tmp, 0, sizeof(tmp));
    tmp._owner = ow;
    free_paths(&tmp);
    out->offsets = (int64_t *)h;
    out->vertices = (int32_t *)(h + boff);
    out->on_device = 0;
    out->_owner = hw;
    return TPGEN_OK;
}

// ------------------------------------------------------------ pipeline
struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    Timer() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

constexpr size_t kSmemTabMax = 40 * 1024;  // slot tables up to this size are staged in shared memory
constexpr size_t kSmemTabLean = 20 * 1024;  // LEAN kernels: 3 blocks x (16.5 KB paths + 32 KB rem stacks + table) per SM

__global__ void set_t0_kernel(unsigned long long *p) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    *p = now;
}

// Grows the record pool to hold at least `need` chunks, keeping the first `used` chunks.
static tpgen_status grow_pool(PlanImpl &P, uint64_t need, cudaStream_t s) {
    if (need <= P.chunk_cap) return TPGEN_OK;
    uint64_t cap = std::max<uint64_t>(need, P.chunk_cap * 2);
    void *np = nullptr;
    TPG_CK(pool_alloc(&np, (cap + 1) * kChunkRecs * 8, s));  // + the overflow sink chunk
    if (P.chunk_used && P.chunks.p)
        TPG_CK(cudaMemcpyAsync(np, P.chunks.p, P.chunk_used * kChunkRecs * 8, cudaMemcpyDeviceToDevice, s));
    if (P.chunks.p) TPG_CK(cudaFreeAsync(P.chunks.p, s));
    P.chunks.p = np;
    P.chunks.cap = (cap + 1) * kChunkRecs * 8;
    P.chunk_cap = cap;
    return TPGEN_OK;
}

// Grows a per-slot array to `cap` elements of `es` bytes keeping the first `used`.
static tpgen_status grow_keep(DevBuf &b, size_t used, size_t cap, size_t es, cudaStream_t s) {
    if (cap * es <= b.cap) return TPGEN_OK;
    void *np = nullptr;
    TPG_CK(pool_alloc(&np, cap * es, s));
    if (used && b.p) TPG_CK(cudaMemcpyAsync(np, b.p, used * es, cudaMemcpyDeviceToDevice, s));
    if (b.p) TPG_CK(cudaFreeAsync(b.p, s));
    b.p = np;
    b.cap = cap * es;
    return TPGEN_OK;
}

template <int W>
static tpgen_status grow_queue(PlanImpl &P, uint64_t used, uint64_t cap, cudaStream_t s) {
    if (cap <= P.qcap) return TPGEN_OK;
    cap = std::max<uint64_t>(cap, P.qcap * 2);  // geometric: creeping high-water marks must not regrow every call
    TPG_TRY(grow_keep(P.qunits, used, cap, sizeof(Unit<W>), s));
    TPG_TRY(grow_keep(P.qready, used, cap, 4, s));
    for (int c = 0; c < C_NUM; c++) TPG_TRY(grow_keep(P.qcnt[c], used, cap, 8, s));
    TPG_TRY(grow_keep(P.qext, used, cap, 8, s));
    TPG_TRY(grow_keep(P.qrfirst, used, cap, 8, s));
    TPG_TRY(grow_keep(P.qrcount, used, cap, 8, s));
    TPG_TRY(grow_keep(P.qchead, used, cap, 8, s));
    TPG_TRY(grow_keep(P.blk_first, used, cap, 8, s));  // blocks are named by their first slot
    TPG_TRY(grow_keep(P.blk_count, used, cap, 4, s));
    TPG_TRY(grow_keep(P.blk_next, used, cap, 8, s));
    TPG_TRY(grow_keep(P.qgen, used, cap, 4, s));
    TPG_TRY(grow_keep(P.qparent, used, cap, 8, s));
    TPG_TRY(grow_keep(P.qnchild, used, cap, 4, s));
    P.qcap = cap;
    return TPGEN_OK;
}

template <int W>
struct RootSpan {  // the roots of one DFS phase (host memory; not owned)
    const Unit<W> *p = nullptr;
    size_t n = 0;
    RootSpan() = default;
    RootSpan(const std::vector<Unit<W>> &v) : p(v.data()), n(v.size()) {}
    RootSpan(const Unit<W> *q, size_t k) : p(q), n(k) {}
    size_t size() const { return n; }
    const Unit<W> *data() const { return p; }
};

// Writes `roots` into the queue at slots [qbase, qbase + roots.size()).
template <int W>
static tpgen_status put_roots(PlanImpl &P, RootSpan<W> roots, uint64_t qbase, cudaStream_t s) {
    const size_t n = roots.size();
    if (!n) return TPGEN_OK;
    if (P.presplit_active && P.presplit_n == (int64_t)n) {  // the plan's cached pre-split roots (device copy)
        TPG_CK(cudaMemcpyAsync(P.qunits.as<Unit<W>>() + qbase, P.presplit_dev.p, n * sizeof(Unit<W>),
                               cudaMemcpyDeviceToDevice, s));
        fill_u32_kernel<<<grid_for((int64_t)n, 256, P.num_sms * 4), 256, 0, s>>>(P.qready.as<uint32_t>() + qbase, 1u,
                                                                                 (int64_t)n);
    } else {
        TPG_CK(cudaMemcpyAsync(P.qunits.as<Unit<W>>() + qbase, roots.data(), n * sizeof(Unit<W>),
                               cudaMemcpyHostToDevice, s));
        std::vector<uint32_t> ones(n, 1u);
        TPG_CK(cudaMemcpyAsync(P.qready.as<uint32_t>() + qbase, ones.data(), n * 4, cudaMemcpyHostToDevice, s));
    }
    TPG_CK(cudaMemsetAsync(P.qgen.as<int32_t>() + qbase, 0, n * 4, s));
    TPG_CK(cudaMemsetAsync(P.qchead.as<int64_t>() + qbase, 0xff, n * 8, s));  // -1: no donated block
    TPG_CK(cudaMemsetAsync(P.qparent.as<int64_t>() + qbase, 0xff, n * 8, s));  // -1: a root
    return TPGEN_OK;
}

// Host pre-split of the per-start tries for LEAN calls (no arc leaves any SCC):
// the top levels of every start vertex's trie are expanded on the host, in DFS
// preorder, into the units a donation would have produced -- K_NODE units at the
// cut depth or at leaves, K_CLOSURE units for cycle closures above the cut --
// so the persistent kernel starts with enough units for every lane instead of
// one per start vertex (the ramp-up of repeated donations).  Nodes above the cut
// that have children carry no event (an internal prime path has no child,
// Def. 1 / R3) but each is one extension (E_canon): counted here.  Cached per
// plan and start range; the device copy is reused by every call.
// With a prefix-unit shard (`ps`, tpgen_options.shard_prefix) the expansion
// starts from the shard's units instead of one unit per start vertex; the
// extensions of the shard split's own expanded nodes come with it (ps->ext).
template <int W>
static void presplit_roots(PlanImpl &P, int32_t lo, int32_t hi, int64_t target, std::vector<Unit<W>> &units,
                           std::vector<int32_t> &gids, uint64_t &ext, const PrefixShard *ps = nullptr) {
    const HostPlan &H = P.hp;
    units.clear();
    gids.clear();
    ext = 0;
    if (ps) {
        for (const PrefixUnit &pu : ps->units) {
            Unit<W> u;
            memset(&u, 0, sizeof(u));
            u.M[0] = pu.M;
            u.scc = pu.scc;
            u.e = -1;
            u.kind = pu.closure ? K_CLOSURE : K_NODE;
            u.depth = pu.depth;
            memcpy(u.path, pu.path, (size_t)pu.depth + 1);
            units.push_back(u);
            gids.push_back(pu.gid);
        }
        ext = ps->ext;
    } else {
        for (int32_t v = lo; v < hi; v++) {
            const int32_t slot = H.v_slot[v], c = H.comp[v];
            Unit<W> u;
            memset(&u, 0, sizeof(u));
            const int loc = slot - H.scc_vbase[c];
            u.M[0] = 1ull << loc;
            u.scc = c;
            u.e = -1;
            u.kind = K_NODE;
            u.path[0] = (uint8_t)loc;
            units.push_back(u);
            gids.push_back(v);
        }
    }
    auto children = [&](const Unit<W> &u) -> uint64_t {
        return H.sin[(size_t)(H.scc_vbase[u.scc] + u.path[u.depth]) * W] & (~u.M[0] | (1ull << u.path[0]));
    };
    while ((int64_t)units.size() < target) {
        int depth = 1 << 30;  // the shallowest expandable level (every unit starts there without a shard)
        for (const Unit<W> &u : units)
            if (u.kind == K_NODE && children(u)) depth = std::min(depth, (int)u.depth);
        if (depth >= 30) break;
        size_t grown = 0;  // size of the next level (bounded: a dense SCC can branch 31 ways)
        for (const Unit<W> &u : units) {
            const uint64_t ch = children(u);
            grown += (u.kind == K_NODE && u.depth == depth && ch) ? (size_t)__builtin_popcountll(ch) : 1;
        }
        if ((int64_t)grown > 16 * target) break;
        std::vector<Unit<W>> next;
        std::vector<int32_t> ngid;
        next.reserve(grown);
        for (size_t i = 0; i < units.size(); i++) {
            const Unit<W> &u = units[i];
            const int s0 = u.path[0];
            const uint64_t ch = children(u);
            if (u.kind != K_NODE || u.depth != depth || ch == 0) {  // terminal: kept as it is
                next.push_back(u);
                ngid.push_back(gids[i]);
                continue;
            }
            if (depth > 0) ext++;  // this node's own extension (its unit is replaced by its children)
            for (uint64_t cc = ch; cc; cc &= cc - 1) {
                const int w = __builtin_ctzll(cc);
                Unit<W> k = u;
                if (w == s0) {
                    k.kind = K_CLOSURE;
                } else {
                    k.depth = (uint8_t)(depth + 1);
                    k.path[depth + 1] = (uint8_t)w;
                    k.M[0] |= 1ull << w;
                }
                next.push_back(k);
                ngid.push_back(gids[i]);
            }
        }
        units.swap(next);
        gids.swap(ngid);
    }
}

// tpgen_options.shard_prefix: this call's prefix-unit shard, when it applies (the pre-split path:
// one mask word, no arc leaving an SCC); lo / hi become the start vertices it touches and *key
// the pre-split cache key.  The split is cached per plan and (rank, count).
static const PrefixShard *prefix_shard_call(PlanImpl &P, const tpgen_options &o, bool presplit_ok, int32_t &lo,
                                            int32_t &hi, int64_t &key) {
    key = -1;
    if (!o.shard_prefix || o.shard_count <= 1 || !presplit_ok || !prefix_shard_applies(P.hp)) return nullptr;
    key = ((int64_t)o.shard_rank << 32) | (uint32_t)o.shard_count;
    if (P.pfx_key != key) {
        prefix_shard(P.hp, o.shard_rank, o.shard_count, P.pfx);
        P.pfx_key = key;
    }
    lo = P.pfx.lo;
    hi = P.pfx.hi;
    return &P.pfx;
}

// One phase of the persistent DFS (seg = SCC-entry starts, else prime-path
// starts) over the roots already placed at [qbase, qbase + nroots).  Retried
// with a larger record pool or queue if either overflows.  Returns the new tail.
// Launch of one DFS kernel variant (LEAN / table in shared memory / generic) in mode MODE.
template <class T, int MODE>
static tpgen_status launch_dfs(bool lean, size_t tab_bytes, int grid, const DfsArgs &A, cudaStream_t s,
                               bool any_exit = true, bool seg = false) {
    constexpr int W = MT<T>::W;
    if constexpr (MODE != M_REC) {  // count modes: the straight-line count kernel (count.cuh)
        static_assert(W == 1, "count modes use one mask word");
        constexpr bool HSH = MODE == M_CNT;
        using CT = typename std::conditional<sizeof(T) == 4, uint32_t, uint64_t>::type;
        const int cgrid = grid / (lean ? kLeanBlocks : DfsCfg<W>::min_blocks) *
                          cnt_min_blocks<CT>(seg, HSH || A.tp != nullptr);
        const size_t ctab = (size_t)A.n_slots * 16;  // {sin, mix} per slot
        const bool ts = ctab <= kSmemTabMax;
        // D2: the out-degree-2 prime-path kernel (count.cuh) when the plan's table allows it
        const bool d2 = !seg && A.tp == nullptr && !A.prune && ts && A.G.slot_d2 != nullptr && sizeof(CT) == 8;
        const size_t cdyn = (ts ? ctab : 0) + cnt_smem_block<CT>(seg, d2 || (seg && ts && A.G.slot_d2 != nullptr && sizeof(CT) == 8));
        void (*k)(DfsArgs);
        const bool d2seg = seg && ts && A.G.slot_d2 != nullptr && sizeof(CT) == 8;
        if (d2) {
            if constexpr (sizeof(CT) == 8) k = any_exit ? cnt_kernel<CT, true, HSH, true, P_PP, true> : cnt_kernel<CT, true, HSH, false, P_PP, true>;
        } else if (d2seg) {
            if constexpr (sizeof(CT) == 8) k = cnt_kernel<CT, true, HSH, true, P_SEG, true>;
        } else if (seg) {
            k = ts ? cnt_kernel<CT, true, HSH, true, P_SEG> : cnt_kernel<CT, false, HSH, true, P_SEG>;
        } else if (A.tp != nullptr) {
            k = ts ? (any_exit ? cnt_kernel<CT, true, true, true, P_TP> : cnt_kernel<CT, true, true, false, P_TP>)
                   : (any_exit ? cnt_kernel<CT, false, true, true, P_TP> : cnt_kernel<CT, false, true, false, P_TP>);
        } else if (A.prune) {  // NEXT #2: the prime-path phase with reachability pruning
            k = ts ? (any_exit ? cnt_kernel<CT, true, HSH, true, P_PRUNE> : cnt_kernel<CT, true, HSH, false, P_PRUNE>)
                   : (any_exit ? cnt_kernel<CT, false, HSH, true, P_PRUNE> : cnt_kernel<CT, false, HSH, false, P_PRUNE>);
        } else {
            k = ts ? (any_exit ? cnt_kernel<CT, true, HSH, true, P_PP> : cnt_kernel<CT, true, HSH, false, P_PP>)
                   : (any_exit ? cnt_kernel<CT, false, HSH, true, P_PP> : cnt_kernel<CT, false, HSH, false, P_PP>);
        }
        TPG_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cdyn));
        k<<<cgrid, CntCfg<CT>::threads, cdyn, s>>>(A);
        return TPGEN_OK;
    } else {
        if constexpr (std::is_same<T, uint32_t>::value) {
            if (lean) {
                TPG_CK(cudaFuncSetAttribute(dfs_kernel<T, true, true, M_REC>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemTabLean));
                dfs_kernel<T, true, true, M_REC><<<grid, DfsCfg<W>::threads, tab_bytes, s>>>(A);
                return TPGEN_OK;
            }
        }
        if (tab_bytes <= kSmemTabMax) {
            TPG_CK(cudaFuncSetAttribute(dfs_kernel<T, true, false, M_REC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kSmemTabMax));
            dfs_kernel<T, true, false, M_REC><<<grid, DfsCfg<W>::threads, tab_bytes, s>>>(A);
        } else {
            dfs_kernel<T, false, false, M_REC><<<grid, DfsCfg<W>::threads, 0, s>>>(A);
        }
        return TPGEN_OK;
    }
}

// One phase of the persistent DFS (seg = SCC-entry starts, else prime-path
// starts) over the roots already placed at [qbase, qbase + nroots).  Retried
// with a larger record pool, queue or head buffer if one overflows.  Returns the
// new tail.  Count modes (mode != M_REC, prime-path phase of COUNT_HASH calls):
// no records; cacc_h receives the kernel's totals (dfs.cuh DfsArgs::cacc).
template <class T>
static tpgen_status dfs_phase(PlanImpl &P, const DevGraph &G, RootSpan<MT<T>::W> roots, int seg,
                              uint64_t qbase, cudaStream_t s, tpgen_stats &st, int64_t &launches, double &ms_dfs,
                              uint64_t &tail_out, int mode = M_REC, unsigned long long *cacc_h = nullptr,
                              double *ms_last = nullptr) {
    NvtxRange nvtx_range(seg ? "tpgen: DFS segment phase" : "tpgen: DFS prime-path phase");
    constexpr int W = MT<T>::W;
    Timer t;
    const HostPlan &H = P.hp;
    const size_t agg_n = 2 * (size_t)H.n + 2 * (size_t)H.n_pairs + 1;
    const uint64_t nroots = roots.size();
    tail_out = qbase + nroots;
    if (nroots == 0) return TPGEN_OK;
    const int64_t lanes = (int64_t)P.num_sms * std::max(DfsCfg<W>::min_blocks, kLeanBlocks) * DfsCfg<W>::threads;
    TPG_TRY(grow_queue<W>(P, qbase, std::max<uint64_t>(std::max<uint64_t>(qbase + nroots + 8 * (uint64_t)lanes, 1u << 21),
                                                       P.q_hwm * 3 / 2), s));
    if (seg) TPG_CK(cudaMemcpyAsync(P.agg_bak.p, P.agg.p, agg_n * 8, cudaMemcpyDeviceToDevice, s));
    TPG_TRY(P.qctr.ensure(8 * 16 * 8, s));
    if (mode != M_REC && !seg) {  // head records: the plan's high-water mark with headroom, at least 1 M slots
        const uint64_t want = std::max<uint64_t>(1ull << 20, P.chead_hwm + P.chead_hwm / 4 + 256ull * 4096);
        if (P.cheads.cap < want * sizeof(HeadS)) TPG_TRY(P.cheads.ensure(want * sizeof(HeadS), s));
    }
    if (mode != M_REC && seg) {  // segment items: likewise
        const uint64_t want = std::max<uint64_t>(1ull << 20, P.citem_hwm + P.citem_hwm / 4 + 256ull * 4096);
        if (P.citems.cap < want * sizeof(ItemS)) TPG_TRY(P.citems.ensure(want * sizeof(ItemS), s));
    }
    unsigned long long *qc = P.qctr.as<unsigned long long>();
    // Test hooks: TPGEN_TEST_QCAP / TPGEN_TEST_POOL cap the queue slots / record chunks this
    // phase may use (doubling after each overflow), so small graphs exercise the retry path.
    uint64_t qlim = P.qcap, plim = P.chunk_cap;
    uint64_t hlim = ~0ull;  // count modes: head slots this phase may use (TPGEN_TEST_HEADCAP test hook)
    if (const char *ev = getenv("TPGEN_TEST_HEADCAP")) hlim = std::max<uint64_t>(256, strtoull(ev, nullptr, 10));
    if (const char *ev = getenv("TPGEN_TEST_QCAP"))
        qlim = std::min<uint64_t>(qlim, qbase + nroots + std::max<uint64_t>(1, strtoull(ev, nullptr, 10)));
    if (const char *ev = getenv("TPGEN_TEST_POOL"))
        plim = std::min<uint64_t>(plim, P.chunk_used + std::max<uint64_t>(1, strtoull(ev, nullptr, 10)));
    for (int attempt = 0; attempt < 48; attempt++) {
        TPG_TRY(put_roots<W>(P, roots, qbase, s));
        TPG_CK(cudaMemsetAsync(P.qready.as<uint32_t>() + qbase + nroots, 0, (P.qcap - qbase - nroots) * 4, s));
        // queue counters, one per 128-byte line: head, tail<<32|done, overflow, chunk_next, maxgen
        unsigned long long init[8 * 16];
        memset(init, 0, sizeof(init));
        init[0] = qbase;
        init[16] = ((qbase + nroots) << 32) | qbase;
        init[48] = P.chunk_used;
        init[64] = (unsigned long long)P.maxgen;
        TPG_CK(cudaMemcpyAsync(qc, init, sizeof(init), cudaMemcpyHostToDevice, s));
        DfsArgs A;
        memset(&A, 0, sizeof(A));
        A.G = G;
        A.units = P.qunits.p;
        A.ready = P.qready.as<unsigned int>();
        A.qhead = qc;
        A.qtd = qc + 16;
        A.qcap = qlim;
        for (int c = 0; c < C_NUM; c++) A.cnt[c] = P.qcnt[c].as<uint64_t>();
        A.ext = P.qext.as<uint64_t>();
        A.rfirst = P.qrfirst.as<int64_t>();
        A.rcount = P.qrcount.as<int64_t>();
        A.child_head = P.qchead.as<int64_t>();
        A.blk_first = P.blk_first.as<int64_t>();
        A.blk_count = P.blk_count.as<int32_t>();
        A.blk_next = P.blk_next.as<int64_t>();
        A.gen = P.qgen.as<int32_t>();
        A.parent = P.qparent.as<int64_t>();
        A.nchild = P.qnchild.as<int32_t>();
        A.maxgen = reinterpret_cast<int *>(qc + 64);
        unsigned long long *agg = P.agg.as<unsigned long long>();
        A.agg_tail_cnt = agg;
        A.agg_tail_len = agg + H.n;
        A.agg_pair_cnt = agg + 2 * (int64_t)H.n;
        A.agg_pair_len = agg + 2 * (int64_t)H.n + H.n_pairs;
        A.overflow = reinterpret_cast<unsigned int *>(qc + 32);
        A.chunks = P.chunks.as<uint64_t>();
        A.chunk_next = qc + 48;
        A.chunk_cap = plim;  // (the sink chunk is chunk plim: inside the allocation)
        // pre-split roots already give every lane work: no eager generations, longer units
        A.split_min = P.presplit_active ? P.split_min_presplit : P.split_min;
        A.eager_gens = P.presplit_active ? 1 : kEagerGens;
        if (const char *ev = getenv("TPGEN_SPLIT_MIN")) A.split_min = (uint32_t)atoi(ev);  // tuning knobs
        if (const char *ev = getenv("TPGEN_EAGER_GENS")) A.eager_gens = atoi(ev);
        if (seg) {  // the segment phase starts from the SCC entries alone (config 5: 16 roots)
            if (const char *ev = getenv("TPGEN_SEG_EAGER_GENS")) A.eager_gens = atoi(ev);
            if (const char *ev = getenv("TPGEN_SEG_SPLIT_MIN")) A.split_min = (uint32_t)atoi(ev);
        }
        A.dbg = nullptr;
        if (getenv("TPGEN_DEBUG")) {
            TPG_TRY(P.dbgbuf.ensure(160 * 8, s));
            A.dbg = P.dbgbuf.as<unsigned long long>();
            TPG_CK(cudaMemsetAsync(A.dbg, 0, 160 * 8, s));
            set_t0_kernel<<<1, 1, 0, s>>>(A.dbg + 7);
        }
        A.low_water = (uint32_t)std::max<int64_t>(64, lanes / 8);
        if (const char *ev = getenv("TPGEN_LOW_WATER")) A.low_water = (uint32_t)atoi(ev);  // tuning knob
        // end game (more than half the lanes waiting): donate after fewer steps
        A.split_min_starve = P.presplit_active ? 96u : P.split_min;
        A.starve_lanes = (int32_t)(lanes / 2);
        if (const char *ev = getenv("TPGEN_SPLIT_STARVE")) A.split_min_starve = (uint32_t)atoi(ev);
        if (const char *ev = getenv("TPGEN_STARVE_LANES")) A.starve_lanes = atoi(ev);
        cudaEventRecord(t.a, s);
        A.n_slots = H.n;
        A.cacc = qc + 112;  // count modes: totals (zeroed with the counters above)
        A.heads = P.cheads.as<HeadS>();
        A.head_cap = (mode != M_REC && !seg) ? std::min<uint64_t>(hlim, P.cheads.cap / sizeof(HeadS)) : 0;
        A.items = P.citems.as<ItemS>();
        A.tp = (mode != M_REC) ? P.cur_tp : nullptr;
        A.prune = (mode != M_REC && !seg) ? P.cur_prune : 0;
        A.k2 = 2;
        A.k8 = 8;
        A.k16 = 16;
        A.item_cap = (mode != M_REC && seg) ? std::min<uint64_t>(hlim, P.citems.cap / sizeof(ItemS)) : 0;
        const size_t tab_bytes = (size_t)H.n * sizeof(Slot<W>);
        // LEAN: 32-bit masks, prime-path phase, no arc leaves any SCC (no head / segment
        // events), the slot table staged in shared memory next to the rem stacks
        const bool lean = std::is_same<T, uint32_t>::value && !seg && !P.any_exit &&
                          tab_bytes + (mode != M_REC ? (size_t)H.n * 8 : 0) <= kSmemTabLean &&
                          !getenv("TPGEN_NO_LEAN");
        const int grid = P.num_sms * (lean ? kLeanBlocks : DfsCfg<W>::min_blocks);
        if constexpr (W == 1) {
            if (mode == M_CNT) TPG_TRY((launch_dfs<T, M_CNT>(lean, tab_bytes, grid, A, s, P.any_exit, seg != 0)));
            else if (mode == M_CNT_NOHASH)
                TPG_TRY((launch_dfs<T, M_CNT_NOHASH>(lean, tab_bytes, grid, A, s, P.any_exit, seg != 0)));
            else TPG_TRY((launch_dfs<T, M_REC>(lean, tab_bytes, grid, A, s)));
        } else {
            if (mode != M_REC) {
                set_error("count-mode DFS needs one mask word (internal)");
                return TPGEN_ERR_INTERNAL;
            }
            TPG_TRY((launch_dfs<T, M_REC>(false, tab_bytes, grid, A, s)));
        }
        cudaEventRecord(t.b, s);
        launches++;
        TPG_CK(cudaGetLastError());
        unsigned long long hq[8 * 16], h[7];
        TPG_CK(cudaMemcpyAsync(hq, qc, sizeof(hq), cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        const int hidx[7] = {0, 16, 0, 32, 48, 64, 80};  // old layout: head, td, -, ovf, chunk, maxgen, blk
        for (int i = 0; i < 7; i++) h[i] = hq[hidx[i]];
        float ms = 0;
        cudaEventElapsedTime(&ms, t.a, t.b);
        ms_dfs += ms;
        if (ms_last) *ms_last = ms;
        st.n_count_rounds++;
        const unsigned ovf = (unsigned)h[3];
        if (ovf & 8u) {  // count modes: head records / items did not fit -- room for all of them, then retry
            DevBuf &buf = seg ? P.citems : P.cheads;
            const size_t es = seg ? sizeof(ItemS) : sizeof(HeadS);
            const uint64_t used = hq[112 + (seg ? 7 : 5)];
            if (hlim < buf.cap / es) {
                hlim *= 2;
            } else {
                (seg ? P.citem_hwm : P.chead_hwm) = std::max<uint64_t>(seg ? P.citem_hwm : P.chead_hwm, used);
                TPG_TRY(buf.ensure((used + used / 4 + 256ull * 4096) * es, s));
            }
        }
        if (ovf & 14u) {  // record pool, queue or head buffer exhausted: undo and retry bigger
            if (seg) TPG_CK(cudaMemcpyAsync(P.agg.p, P.agg_bak.p, agg_n * 8, cudaMemcpyDeviceToDevice, s));
            if (ovf & 2u) {
                if (plim < P.chunk_cap) {
                    plim = std::min<uint64_t>(P.chunk_cap, plim * 2);
                } else {
                    TPG_TRY(grow_pool(P, std::max<uint64_t>(h[4], P.chunk_cap) * 2, s));
                    plim = P.chunk_cap;
                }
            }
            if (ovf & 4u) {
                if (qlim < P.qcap) {
                    qlim = std::min<uint64_t>(P.qcap, qlim * 2);
                } else {
                    TPG_TRY(grow_queue<W>(P, qbase, P.qcap * 2, s));
                    qlim = P.qcap;
                }
            }
            continue;
        }
        if (A.dbg) {
            unsigned long long d[160];
            TPG_CK(cudaMemcpyAsync(d, A.dbg, 160 * 8, cudaMemcpyDeviceToHost, s));
            TPG_CK(cudaStreamSynchronize(s));
            fprintf(stderr, "[tpgen dfs timeline] busy lane fraction per 0.1 ms:");
            for (int b = 0; b < 64; b++)
                if (d[9 + 2 * b]) fprintf(stderr, " %.2f", (double)d[8 + 2 * b] / d[9 + 2 * b]);
            fprintf(stderr, "\n");
            fprintf(stderr, "[tpgen dfs] ms=%.3f iters=%llu active_lane_iters=%llu (%.2f/warp-iter) donations=%llu units=%llu\n",
                    ms, d[0], d[1], d[0] ? (double)d[1] / d[0] : 0.0, d[2], (h[1] >> 32) - qbase);
        }
        if (ovf & 1u) P.overflow = true;
        if (ovf & 16u) P.tp_unreachable = true;
        if (mode != M_REC) {
            if (cacc_h) memcpy(cacc_h, hq + 112, 8 * sizeof(unsigned long long));
            P.chead_hwm = std::max<uint64_t>(P.chead_hwm, hq[112 + 5]);
            P.citem_hwm = std::max<uint64_t>(P.citem_hwm, hq[112 + 7]);
        }
        P.chunk_used = std::min<uint64_t>(h[4], P.chunk_cap);  // (reserved-but-unused chunks may overshoot)
        P.chunk_hwm = std::max<uint64_t>(P.chunk_hwm, P.chunk_used);
        P.q_hwm = std::max<uint64_t>(P.q_hwm, h[1] >> 32);
        if (mode == M_REC) P.maxgen = std::max<int>(P.maxgen, (int)(h[5] & 0xffffffffu));
        tail_out = h[1] >> 32;
        return TPGEN_OK;
    }
    set_error("DFS phase: work queue / record pool could not be sized");
    return TPGEN_ERR_OUT_OF_MEMORY;
}

// Canonical writer launch: the lane-parallel kernel when every SCC has at most
// kFastMaxScc vertices (one mask word), else the sequential replay.  HASH: digest only.
template <int NPW, bool HASH>
static void launch_fast(const ExpandArgs &E, int64_t nu, int num_sms, bool mixed, cudaStream_t s) {
    constexpr int th = FastCfg<NPW>::threads;
    constexpr size_t sm = FastCfg<NPW>::smem_bytes(HASH);  // (double-buffered bulk-store stages: > 48 KB)
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(expand_fast_kernel<NPW, HASH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        cudaFuncSetAttribute(expand_fast_kernel<NPW, HASH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = true;
    }
    const int g = grid_for(nu * 32, th, num_sms * 2048 / th);
    if (mixed) expand_fast_kernel<NPW, HASH, true><<<g, th, sm, s>>>(E);
    else expand_fast_kernel<NPW, HASH, false><<<g, th, sm, s>>>(E);
}
template <bool HASH>
static void launch_fast_npw(int npw, const ExpandArgs &E, int64_t nu, int num_sms, bool mixed, cudaStream_t s) {
    switch (npw) {
        case 1: launch_fast<1, HASH>(E, nu, num_sms, mixed, s); break;
        case 2: launch_fast<2, HASH>(E, nu, num_sms, mixed, s); break;
        case 3: launch_fast<3, HASH>(E, nu, num_sms, mixed, s); break;
        case 4: launch_fast<4, HASH>(E, nu, num_sms, mixed, s); break;
        case 5: launch_fast<5, HASH>(E, nu, num_sms, mixed, s); break;
        case 6: launch_fast<6, HASH>(E, nu, num_sms, mixed, s); break;
        case 7: launch_fast<7, HASH>(E, nu, num_sms, mixed, s); break;
        case 8: launch_fast<8, HASH>(E, nu, num_sms, mixed, s); break;
        case 9: launch_fast<9, HASH>(E, nu, num_sms, mixed, s); break;
        case 10: launch_fast<10, HASH>(E, nu, num_sms, mixed, s); break;
        case 11: launch_fast<11, HASH>(E, nu, num_sms, mixed, s); break;
        case 12: launch_fast<12, HASH>(E, nu, num_sms, mixed, s); break;
        case 13: launch_fast<13, HASH>(E, nu, num_sms, mixed, s); break;
        case 14: launch_fast<14, HASH>(E, nu, num_sms, mixed, s); break;
        case 15: launch_fast<15, HASH>(E, nu, num_sms, mixed, s); break;
        default: launch_fast<16, HASH>(E, nu, num_sms, mixed, s); break;
    }
}
template <int W, bool HASH>
static void launch_seq(int np, const ExpandArgs &E, int64_t nu, int num_sms, cudaStream_t s) {
    const int eg = grid_for(nu * 32, kExpandThreads, num_sms * 8);
    if (W == 1 && np <= 1) expand_kernel<W, 1, HASH><<<eg, kExpandThreads, 0, s>>>(E);
    else if (W == 1 && np <= 2) expand_kernel<W, 2, HASH><<<eg, kExpandThreads, 0, s>>>(E);
    else expand_kernel<W, 2 * W + 1, HASH><<<eg, kExpandThreads, 0, s>>>(E);
}
template <int W>
static void launch_expand(const HostPlan &H, const ExpandArgs &E, int64_t nu, int num_sms, bool hash, bool mixed,
                          cudaStream_t s) {
    const int np = (H.max_scc + 1 + 31) / 32;  // registers per lane for the longest emitted path
    const int npw = std::max(1, (H.max_scc + 3) / 4);  // 32-bit words of local ids for the longest path
    if (W == 1 && H.max_scc <= kFastMaxScc && !getenv("TPGEN_SLOW_EXPAND")) {
        if (hash) launch_fast_npw<true>(npw, E, nu, num_sms, mixed, s);
        else launch_fast_npw<false>(npw, E, nu, num_sms, mixed, s);
    } else {
        if (hash) launch_seq<W, true>(np, E, nu, num_sms, s);
        else launch_seq<W, false>(np, E, nu, num_sms, s);
    }
}

template <class T>
static tpgen_status run_pp(PlanImpl &P, const tpgen_options &o, tpgen_paths *out, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: prime paths (record walk + canonical writer)");
    constexpr int W = MT<T>::W;
    const double t0 = now_ms();
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    memset(out, 0, sizeof(*out));
    int64_t launches = 0;
    const HostPlan &H = P.hp;
    cudaStream_t s = (cudaStream_t)o.stream;
    int32_t lo = 0, hi = H.n;
    shard_range(H, o.shard_rank, o.shard_count, lo, hi);
    if (o.start_hi > o.start_lo) {
        lo = std::max(0, o.start_lo);
        hi = std::min(H.n, o.start_hi);
    }
    // LEAN calls start from host pre-split tries (below); with shard_prefix the shard is a range of them
    const bool presplit_ok = std::is_same<T, uint32_t>::value && !P.any_exit &&
                             (size_t)H.n * sizeof(Slot<W>) <= kSmemTabLean && !getenv("TPGEN_NO_LEAN") &&
                             !getenv("TPGEN_NO_PRESPLIT");
    int64_t pfx_key = -1;
    const PrefixShard *pfx = prefix_shard_call(P, o, presplit_ok, lo, hi, pfx_key);
    st.unit_lo = pfx ? pfx->ulo : -1;
    st.unit_hi = pfx ? pfx->uhi : -1;
    st.shard_lo = lo;
    st.shard_hi = hi;
    st.n_scc = H.n_scc;
    st.n_scc_nontrivial = H.n_nontrivial;
    st.max_scc = H.max_scc;
    st.ms_plan = P.ms_plan;
    P.overflow = false;
    P.chunk_used = 0;
    P.maxgen = 0;
    // TPGEN_DEBUG=1: host time per stage with a sync before each mark; =2: no syncs (enqueue times)
    const char *hdbg_env = getenv("TPGEN_DEBUG");
    const bool hdbg = hdbg_env != nullptr;
    const bool hsync = hdbg && strcmp(hdbg_env, "2") != 0;
    double hprev = now_ms();
    auto HT = [&](const char *what) {
        if (!hdbg) return;
        if (hsync) cudaStreamSynchronize(s);
        const double t = now_ms();
        fprintf(stderr, "[tpgen host] %-24s %8.3f ms\n", what, t - hprev);
        hprev = t;
    };

    Timer tall, tw, tst, tlin;
    cudaEventRecord(tall.a, s);
    const DevGraph G = dev_graph(P, lo, hi);

    // ---- roots: one K_NODE unit per start vertex (segment phase: SCC entries; PP phase: the rest)
    std::vector<Unit<W>> seg_roots, pp_roots;
    std::vector<int32_t> seg_gid, pp_gid;
    for (int32_t v = 0; v < H.n; v++) {
        const int32_t slot = H.v_slot[v];
        const bool entry = (H.slot_flags[slot] & F_ENTRY) != 0;
        if (!entry && !(v >= lo && v < hi)) continue;
        Unit<W> u;
        memset(&u, 0, sizeof(u));
        const int32_t c = H.comp[v];
        const int loc = slot - H.scc_vbase[c];
        u.M[loc >> 6] = 1ull << (loc & 63);
        u.scc = c;
        u.e = -1;
        u.kind = K_NODE;
        u.path[0] = (uint8_t)loc;
        (entry ? seg_roots : pp_roots).push_back(u);
        (entry ? seg_gid : pp_gid).push_back(v);
    }
    TPG_TRY(P.ctr.ensure(32 * 8, s));
    const size_t agg_n = 2 * (size_t)H.n + 2 * (size_t)H.n_pairs + 1;
    TPG_TRY(P.agg.ensure(agg_n * 8, s));
    TPG_TRY(P.agg_bak.ensure(agg_n * 8, s));
    TPG_CK(cudaMemsetAsync(P.agg.p, 0, agg_n * 8, s));
    {
        double est = 0;  // Knuth estimates of the trie sizes -> initial record pool
        for (int32_t v = 0; v < H.n; v++) est += P.hp.cost[v];
        // ... or 1.5x the most this plan has used: record counts vary from call to call (the
        // donation pattern is dynamic), and a retry inside a call costs a second DFS launch
        TPG_TRY(grow_pool(P, std::max<uint64_t>(std::max<uint64_t>((64ull << 20) / (kChunkRecs * 8),
                                                                   (uint64_t)(est * 0.75 / (kChunkRecs - 1)) + 4 * H.n),
                                                P.chunk_hwm * 3 / 2), s));
    }

    // LEAN calls: pre-split tries (cached per plan and start range)
    uint64_t presplit_ext = 0;
    bool presplit_ext_used = false;
    RootSpan<W> pp_span(pp_roots);
    const std::vector<int32_t> *pp_gid_p = &pp_gid;
    if (presplit_ok && seg_roots.empty()) {
        if (!(P.presplit_lo == lo && P.presplit_hi == hi && P.presplit_key == pfx_key && P.presplit_dev.p)) {
            const int64_t lanes = (int64_t)P.num_sms * DfsCfg<W>::min_blocks * DfsCfg<W>::threads;
            std::vector<Unit<W>> units;
            int64_t target = lanes;  // measured: lanes/4 4.98, lanes 4.92, 2 lanes 5.00 ms per config-3 call
            if (const char *ev = getenv("TPGEN_PRESPLIT_TARGET")) target = atoll(ev);  // tuning knob
            presplit_roots<W>(P, lo, hi, target, units, P.presplit_gid, P.presplit_ext, pfx);
            P.presplit_host.assign(reinterpret_cast<const uint8_t *>(units.data()),
                                   reinterpret_cast<const uint8_t *>(units.data() + units.size()));
            P.presplit_n = (int64_t)units.size();
            P.presplit_roots_n = -1;  // the cached root table belongs to the previous range
            TPG_TRY(upload(P.presplit_dev, P.presplit_host, s));
            P.presplit_lo = lo;
            P.presplit_hi = hi;
            P.presplit_key = pfx_key;
        }
        pp_span = RootSpan<W>(reinterpret_cast<const Unit<W> *>(P.presplit_host.data()), (size_t)P.presplit_n);
        pp_gid_p = &P.presplit_gid;
        presplit_ext = P.presplit_ext;
        P.presplit_active = true;
        presplit_ext_used = true;
    }

    double ms_dfs = 0;
    uint64_t tail_seg = 0, tail = 0;
    // (COUNT_HASH calls whose SCCs fit one mask word take run_count; here the record path)
    const bool hash_only = (o.output_mode == TPGEN_OUT_COUNT_HASH);
    // ---- segment phase (SCC entries) -> completion DP
    if (!seg_roots.empty()) {
        TPG_TRY(dfs_phase<T>(P, G, seg_roots, 1, 0, s, st, launches, ms_dfs, tail_seg));
        std::vector<uint64_t> aggh(agg_n);
        TPG_CK(cudaMemcpyAsync(aggh.data(), P.agg.p, agg_n * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        std::vector<uint64_t> tail_cnt(aggh.begin(), aggh.begin() + H.n);
        std::vector<uint64_t> tail_len(aggh.begin() + H.n, aggh.begin() + 2 * H.n);
        std::vector<uint64_t> pair_cnt(aggh.begin() + 2 * H.n, aggh.begin() + 2 * H.n + H.n_pairs);
        std::vector<uint64_t> pair_len(aggh.begin() + 2 * H.n + H.n_pairs, aggh.begin() + 2 * H.n + 2 * H.n_pairs);
        std::vector<uint64_t> Wd, Vd;
        if (!completion_dp(H, tail_cnt, tail_len, pair_cnt, pair_len, Wd, Vd)) {
            set_error("cross-SCC prime-path count exceeds 2^62");
            return TPGEN_ERR_LIMIT_EXCEEDED;
        }
        TPG_CK(cudaMemcpyAsync(P.d_Wc.p, Wd.data(), H.n * 8, cudaMemcpyHostToDevice, s));
        TPG_CK(cudaMemcpyAsync(P.d_Wv.p, Vd.data(), H.n * 8, cudaMemcpyHostToDevice, s));
    }
    // ---- prime-path phase
    HT("before pp phase");
    {
        double ms_pp = 0;
        const tpgen_status r = dfs_phase<T>(P, G, pp_span, 0, tail_seg, s, st, launches, ms_dfs, tail, M_REC,
                                            nullptr, &ms_pp);
        st.ms_dominant = ms_pp;
        P.presplit_active = false;
        if (r != TPGEN_OK) return r;
    }
    if (P.overflow) {
        set_error("prime-path count exceeds 2^62");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    const int64_t nu = (int64_t)tail;
    st.n_units = (int64_t)tail;

    HT("after dfs phases");
    // ---- canonical order: roots by global id, then preorder of the split forest
    std::vector<int64_t> root_order;
    std::vector<int32_t> root_gid;
    const std::vector<int32_t> &pp_gid_r = *pp_gid_p;
    const bool roots_cached = presplit_ext_used && P.presplit_roots_n == (int64_t)pp_gid_r.size() &&
                              P.presplit_roots_tail == (int64_t)tail_seg;
    if (!roots_cached) {
        root_order.reserve(seg_roots.size() + pp_gid_r.size());
        const std::vector<int32_t> &pp_gid = pp_gid_r;
        size_t a = 0, b = 0;
        while (a < seg_gid.size() || b < pp_gid.size()) {
            if (b >= pp_gid.size() || (a < seg_gid.size() && seg_gid[a] < pp_gid[b])) {
                root_order.push_back((int64_t)a);
                root_gid.push_back(seg_gid[a++]);
            } else {
                root_order.push_back((int64_t)(tail_seg + b));
                root_gid.push_back(pp_gid[b++]);
            }
        }
    }
    const int64_t n_roots = roots_cached ? P.presplit_roots_n : (int64_t)root_order.size();
    const size_t nu1 = (size_t)std::max<int64_t>(nu, 1);
    // scratch: sub[C_NUM] | acc[C_NUM] | node ping | node pong
    TPG_TRY(P.offs.ensure(nu1 * (16 * C_NUM + 2 * sizeof(LinNode)) + 256, s));
    // root table (canonical root order + start gids); the pre-split roots' table is uploaded once per plan
    DevBuf &rbuf = presplit_ext_used ? P.presplit_roots : P.roots;
    if (!roots_cached) {
        TPG_TRY(rbuf.ensure(std::max<size_t>(root_order.size(), 1) * 12, s));
        if (n_roots) {
            TPG_CK(cudaMemcpyAsync(rbuf.p, root_order.data(), n_roots * 8, cudaMemcpyHostToDevice, s));
            TPG_CK(cudaMemcpyAsync(rbuf.as<char>() + n_roots * 8, root_gid.data(), n_roots * 4,
                                   cudaMemcpyHostToDevice, s));
        }
        if (presplit_ext_used) {
            P.presplit_roots_n = n_roots;
            P.presplit_roots_tail = (int64_t)tail_seg;
        }
    }
    const int64_t *roots_d = rbuf.as<int64_t>();
    const int32_t *rgid_d = reinterpret_cast<const int32_t *>(rbuf.as<char>() + n_roots * 8);
    uint64_t *sub[C_NUM];
    unsigned long long *ctr = P.ctr.as<unsigned long long>();
    uint64_t *tot_d = reinterpret_cast<uint64_t *>(ctr + 8);
    LinArgs LA;
    uint64_t *lp = P.offs.as<uint64_t>();
    for (int c = 0; c < C_NUM; c++) {
        sub[c] = lp + (size_t)c * nu1;
        LA.cnt[c] = P.qcnt[c].as<uint64_t>();
        LA.sub[c] = sub[c];
        LA.acc[c] = lp + (size_t)(C_NUM + c) * nu1;
    }
    LinNode *node[2] = {reinterpret_cast<LinNode *>(lp + 2 * C_NUM * nu1),
                        reinterpret_cast<LinNode *>(lp + 2 * C_NUM * nu1) + nu1};
    LA.node = node[0];
    LA.parent = P.qparent.as<int64_t>();
    LA.pending = P.qnchild.as<int32_t>();
    LA.child_head = P.qchead.as<int64_t>();
    LA.blk_first = P.blk_first.as<int64_t>();
    LA.blk_count = P.blk_count.as<int32_t>();
    LA.blk_next = P.blk_next.as<int64_t>();
    LA.n = nu;
    LA.roots = roots_d;
    LA.n_roots = n_roots;
    LA.totals = tot_d;
    const LinNode *off = node[0];  // final canonical offsets
    uint64_t tot[C_NUM + 1] = {0};
    cudaEventRecord(tlin.a, s);
    if (nu > 0) {
        const int lg = grid_for(nu, 256, P.num_sms * 8);
        TPG_CK(cudaMemsetAsync(LA.acc[0], 0, (size_t)C_NUM * nu1 * 8, s));
        lin_up_flow_kernel<<<lg, 256, 0, s>>>(LA);
        if (n_roots <= 4 * kScanThreads) {
            lin_roots_kernel<<<1, kScanThreads, 0, s>>>(LA);
        } else {  // many roots (pre-split tries): gather, device-wide scan, scatter
            TPG_TRY(P.rscan.ensure((size_t)C_NUM * n_roots * 8, s));
            uint64_t *ra[C_NUM];
            for (int c = 0; c < C_NUM; c++) ra[c] = P.rscan.as<uint64_t>() + (size_t)c * n_roots;
            const int rg = grid_for(n_roots, 256, P.num_sms * 8);
            lin_roots_gather_kernel<<<rg, 256, 0, s>>>(LA, P.rscan.as<uint64_t>());
            TPG_TRY(scan_multi(P, ra, C_NUM, n_roots, nullptr, s, launches));
            lin_roots_scatter_kernel<<<rg, 256, 0, s>>>(LA, P.rscan.as<uint64_t>());
            TPG_CK(cudaMemcpyAsync(tot_d, P.scan_tot.p, C_NUM * 8, cudaMemcpyDeviceToDevice, s));
            launches += 2;
        }
        lin_rel_kernel<<<lg, 256, 0, s>>>(LA);
        launches += 3;
        // rounds: after r rounds a unit has summed its 2^r nearest ancestors' relative offsets
        int rounds = 0;
        while ((1ll << rounds) < (long long)P.maxgen + 1) rounds++;
        for (int r = 0; r < rounds; r++) {
            lin_jump_kernel<<<lg, 256, 0, s>>>(node[r & 1], node[(r + 1) & 1], nu);
            launches++;
        }
        off = node[rounds & 1];
        TPG_CK(cudaMemsetAsync(ctr + 14, 0, 16, s));
        sum_kernel<<<lg, 256, 0, s>>>(P.qext.as<uint64_t>(), (int64_t)tail_seg, ctr + 15);  // segment phase
        sum_kernel<<<lg, 256, 0, s>>>(P.qext.as<uint64_t>() + tail_seg, nu - (int64_t)tail_seg, ctr + 14);
        launches += 2;
        cudaEventRecord(tlin.b, s);
        TPG_CK(cudaMemcpyAsync(tot, tot_d, C_NUM * 8, cudaMemcpyDeviceToHost, s));
        unsigned long long ext2[2];
        TPG_CK(cudaMemcpyAsync(ext2, ctr + 14, 16, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        tot[C_NUM] = ext2[0] + ext2[1];
        st.ext_dominant = (int64_t)ext2[0];
        float lms = 0;
        cudaEventElapsedTime(&lms, tlin.a, tlin.b);
        st.ms_linearize = lms;
    }
    const uint64_t seg_heads = tot[C_HEADS];  // head records of the replayed units
    const int64_t n_pp = (int64_t)tot[C_PP], n_vert = (int64_t)tot[C_VERT];
    st.n_extensions = (int64_t)(tot[C_NUM] + presplit_ext);
    st.n_heads = (int64_t)tot[C_HEADS];
    st.n_segments = (int64_t)tot[C_ITEMS];
    if ((o.max_paths > 0 && n_pp > o.max_paths) || (o.max_extensions > 0 && st.n_extensions > o.max_extensions)) {
        set_error("result exceeds max_paths / max_extensions");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    st.n_paths = n_pp;
    st.total_vertices = n_vert;

    if (hash_only && !o.compute_digest) {  // counts only: no writer at all
        cudaEventRecord(tall.b, s);
        TPG_CK(cudaStreamSynchronize(s));
        float ms = 0;
        cudaEventElapsedTime(&ms, tall.a, tall.b);
        st.ms_device = ms;
        st.ms_count = ms;
        st.ms_dfs_count = ms_dfs;
        st.ms_dfs_write = ms_dfs;
        st.gpu_launches = launches;
        st.ms_total = now_ms() - t0;
        if (stp) *stp = st;
        return TPGEN_OK;
    }

    HT("after linearize");
    // ---- allocations (exact sizes)
    OutOwner *ow = new OutOwner();
    ow->device = P.device;
    std::unique_ptr<OutOwner> ow_guard(ow);
    void *d_off = nullptr, *d_vert = nullptr;
    if (!hash_only) TPG_TRY(out_alloc_pair(o, ow, (size_t)(n_pp + 1) * 8, (size_t)n_vert * 4, &d_off, &d_vert, s));
    unsigned long long *hacc = ctr + 16;  // digest accumulators (COUNT_HASH: filled by the writers)
    TPG_CK(cudaMemsetAsync(hacc, 0, 16, s));
    const int64_t n_items = (int64_t)tot[C_ITEMS], n_heads = (int64_t)seg_heads;
    TPG_TRY(P.heads.ensure(std::max<int64_t>((int64_t)seg_heads, 1) * sizeof(HeadRec), s));
    TPG_TRY(P.head_pool.ensure(std::max<uint64_t>(tot[C_HEADV], 1) * 4, s));
    TPG_TRY(P.items.ensure(std::max<int64_t>(n_items, 1) * sizeof(ItemRec), s));
    TPG_TRY(P.item_pool.ensure(std::max<uint64_t>(tot[C_ITEMV], 1) * 4, s));

    HT("after alloc");
    // ---- canonical writer: replay the record streams at their exact offsets
    ExpandArgs E;
    memset(&E, 0, sizeof(E));
    E.G = G;
    E.units = P.qunits.p;
    E.n_units = nu;
    E.rfirst = P.qrfirst.as<int64_t>();
    E.rcount = P.qrcount.as<int64_t>();
    E.off = off;
    E.chunks = P.chunks.as<uint64_t>();
    E.out_off = (int64_t *)d_off;
    E.out_vert = (int32_t *)d_vert;
    E.heads = P.heads.as<HeadRec>();
    E.head_pool = P.head_pool.as<int32_t>();
    E.items = P.items.as<ItemRec>();
    E.item_pool = P.item_pool.as<int32_t>();
    E.hash_acc = hacc;
    for (int c = 0; c < C_NUM; c++) E.lim[c] = tot[c];
    cudaEventRecord(tw.a, s);
    if (nu > 0) {
        launch_expand<W>(H, E, nu, P.num_sms, hash_only, n_items > 0 || seg_heads > 0, s);
        launches++;
    }
    cudaEventRecord(tw.b, s);
    TPG_CK(cudaGetLastError());

    HT("before stitch");
    // ---- cross-SCC stitching
    cudaEventRecord(tst.a, s);
    if (n_heads > 0) {
        TPG_TRY(P.hcomp.ensure((size_t)n_heads * 8, s));
        head_weight_kernel<<<grid_for(n_heads, 256, 4096), 256, 0, s>>>(G, P.heads.as<HeadRec>(), n_heads,
                                                                         P.hcomp.as<uint64_t>());
        launches++;
        uint64_t *ha[1] = {P.hcomp.as<uint64_t>()};
        uint64_t ncomp = 0;
        TPG_TRY(scan_multi(P, ha, 1, n_heads, &ncomp, s, launches));
        st.n_cross = (int64_t)ncomp;
        TPG_TRY(P.icum.ensure((size_t)std::max<int64_t>(n_items, 1) * 8, s));
        TPG_TRY(P.ivcum.ensure((size_t)std::max<int64_t>(n_items, 1) * 8, s));
        TPG_TRY(P.ibeg.ensure((size_t)std::max(H.n, 1) * 8, s));
        TPG_TRY(P.iend.ensure((size_t)std::max(H.n, 1) * 8, s));
        if (n_items > 0) {
            item_weight_kernel<<<grid_for(n_items, 256, 4096), 256, 0, s>>>(G, P.items.as<ItemRec>(), n_items,
                                                                             P.icum.as<uint64_t>(),
                                                                             P.ivcum.as<uint64_t>());
            launches++;
            uint64_t *ia[2] = {P.icum.as<uint64_t>(), P.ivcum.as<uint64_t>()};
            TPG_TRY(scan_multi(P, ia, 2, n_items, nullptr, s, launches));
        }
        item_bounds_kernel<<<grid_for(n_roots, 256, 4096), 256, 0, s>>>(
            roots_d, rgid_d, n_roots,
            off, sub[C_ITEMS], P.ibeg.as<int64_t>(), P.iend.as<int64_t>());
        launches++;
        StitchArgs SA;
        SA.heads = P.heads.as<HeadRec>();
        SA.n_heads = n_heads;
        SA.comp_off = P.hcomp.as<uint64_t>();
        SA.n_comp = ncomp;
        SA.items = P.items.as<ItemRec>();
        SA.cum = P.icum.as<uint64_t>();
        SA.vcum = P.ivcum.as<uint64_t>();
        SA.ibeg = P.ibeg.as<int64_t>();
        SA.iend = P.iend.as<int64_t>();
        SA.head_pool = P.head_pool.as<int32_t>();
        SA.item_pool = P.item_pool.as<int32_t>();
        SA.out_off = (int64_t *)d_off;
        SA.out_vert = (int32_t *)d_vert;
        SA.n_pp = (uint64_t)n_pp;
        SA.n_vert = (uint64_t)n_vert;
        if (ncomp > 0) {
            if (hash_only) {
                stitch_hash_kernel<<<grid_for((int64_t)ncomp, 256, P.num_sms * 8), 256, 0, s>>>(SA, hacc);
                launches++;
            } else {
                // range writer: an even split of the completions over the warps, one unranking each
                const int dmax = std::min(H.n_scc, H.n) + 1;  // levels: one SCC each along a DAG path
                int64_t warps = std::min<int64_t>((int64_t)ncomp, (int64_t)P.num_sms * 32);
                const size_t per_warp = (size_t)3 * dmax * 8;
                warps = std::min<int64_t>(warps, (int64_t)((size_t)(512u << 20) / per_warp));
                warps = (warps + 7) & ~(int64_t)7;  // whole 256-thread blocks: every launched warp has its stack
                if ((size_t)warps * per_warp <= ((size_t)1 << 30)) {
                    TPG_TRY(P.sscratch.ensure((size_t)warps * per_warp, s));
                    StitchRangeArgs CA;
                    CA.S = SA;
                    CA.scratch = P.sscratch.as<int64_t>();
                    CA.dmax = dmax;
                    stitch_range_kernel<<<(int)(warps / 8), 256, 0, s>>>(CA);
                } else {  // very deep component DAGs: one warp per path, no stack
                    stitch_kernel<<<grid_for((int64_t)ncomp * 32, 256, P.num_sms * 8), 256, 0, s>>>(SA);
                }
                launches++;
            }
        }
    }
    if (!hash_only) {
        set_last_offset_kernel<<<1, 1, 0, s>>>((int64_t *)d_off, n_pp, n_vert);
        launches++;
    }
    cudaEventRecord(tst.b, s);
    cudaEventRecord(tall.b, s);
    TPG_CK(cudaGetLastError());

    if (o.compute_digest && n_pp > 0) {
        unsigned long long *acc = hacc;
        if (!hash_only) {
            TPG_CK(cudaMemsetAsync(acc, 0, 16, s));
            digest_kernel<<<grid_for(n_pp, 256, P.num_sms * 8), 256, 0, s>>>((int64_t *)d_off, (int32_t *)d_vert,
                                                                               n_pp, acc);
            launches++;
        }
        unsigned long long hd[2];
        TPG_CK(cudaMemcpyAsync(hd, acc, 16, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        st.hash_lo = hd[0];
        st.hash_hi = hd[1];
    }
    TPG_CK(cudaStreamSynchronize(s));
    float ms = 0;
    cudaEventElapsedTime(&ms, tall.a, tall.b);
    st.ms_device = ms;
    cudaEventElapsedTime(&ms, tw.a, tw.b);
    st.ms_write = ms;
    cudaEventElapsedTime(&ms, tst.a, tst.b);
    st.ms_stitch = ms;
    st.ms_count = st.ms_device - st.ms_write - st.ms_stitch;
    st.ms_dfs_count = ms_dfs;  // DFS kernel time (both phases)
    st.ms_dfs_write = ms_dfs;  // the dominant kernel is the DFS enumerator
    st.gpu_launches = launches;

    HT("before finish_output");
    if (!hash_only) {
        ow_guard.release();
        TPG_TRY(finish_output(o, ow, n_pp, n_vert, (int64_t *)d_off, (int32_t *)d_vert, s, out));
    }
    st.ms_total = now_ms() - t0;
    if (stp) *stp = st;
    return TPGEN_OK;
}

// ------------------------------------------------------------ count modes
// COUNT_HASH calls on graphs whose SCCs have <= 64 vertices: no record
// streams at all.  (1) The segment phase runs cnt_kernel<SEG> over the SCC entry vertices:
// their cycles are counted and hashed, their tail / transit segments become ItemS records
// plus the completion-DP aggregates.  (2) Host completion DP (u64, overflow checked).
// (3) The prime-path phase runs cnt_kernel over every other start vertex: counts, E_canon,
// digests, HeadS records.  (4) head_weight_s: the cross prime paths' counts and vertices.
// (5) With the digest: items grouped by entry, weighted and scanned; stitch_hash_s hashes
// every cross prime path from S(h) and the items' (A, B).
// The count-mode steps after the enumeration (shared by the DFS count kernel and the frontier
// engine): the completion DP from the items' aggregates, the heads' cross prime paths, the totals,
// and with the digest the item grouping and the stitch hash of every cross prime path.
// cseg / cpp: the segment / prime-path phase's totals ([0] paths, [1] vertices, [2] E_canon,
// [3..4] digest, [5] head slots, [7] item slots).
static tpgen_status count_post(PlanImpl &P, const tpgen_options &o, const DevGraph &G, cudaStream_t s, bool has_seg,
                               const unsigned long long *cseg, const unsigned long long *cpp, uint64_t presplit_ext,
                               tpgen_stats &st, int64_t &launches, Timer &tall, Timer &tst, double ms_dfs, double t0,
                               tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: count post (items, completion DP, stitch)");
    const HostPlan &H = P.hp;
    const size_t agg_n = 2 * (size_t)H.n + 2 * (size_t)H.n_pairs + 1;
    unsigned long long *ctr = P.ctr.as<unsigned long long>();
    const bool hdbg = getenv("TPGEN_DEBUG") != nullptr;
    auto HT = [&](const char *what) {
        if (!hdbg) return;
        cudaStreamSynchronize(s);
        fprintf(stderr, "[tpgen count] %-28s %s\n", what, cudaGetErrorString(cudaGetLastError()));
    };
    // (2) completion DP from the items' aggregates
    if (has_seg) {
        const int64_t n_slots = (int64_t)cseg[7];
        unsigned long long *agg = P.agg.as<unsigned long long>();
        if (n_slots > 0) {
            item_agg_s_kernel<<<grid_for(n_slots, 256, P.num_sms * 8), 256, 0, s>>>(
                G, P.citems.as<ItemS>(), n_slots, H.n, agg, agg + H.n, agg + 2 * (int64_t)H.n,
                agg + 2 * (int64_t)H.n + H.n_pairs);
            launches++;
        }
        std::vector<uint64_t> aggh(agg_n);
        TPG_CK(cudaMemcpyAsync(aggh.data(), P.agg.p, agg_n * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        std::vector<uint64_t> tail_cnt(aggh.begin(), aggh.begin() + H.n);
        std::vector<uint64_t> tail_len(aggh.begin() + H.n, aggh.begin() + 2 * H.n);
        std::vector<uint64_t> pair_cnt(aggh.begin() + 2 * H.n, aggh.begin() + 2 * H.n + H.n_pairs);
        std::vector<uint64_t> pair_len(aggh.begin() + 2 * H.n + H.n_pairs, aggh.begin() + 2 * H.n + 2 * H.n_pairs);
        std::vector<uint64_t> Wd, Vd;
        if (!completion_dp(H, tail_cnt, tail_len, pair_cnt, pair_len, Wd, Vd)) {
            set_error("cross-SCC prime-path count exceeds 2^62");
            return TPGEN_ERR_LIMIT_EXCEEDED;
        }
        TPG_CK(cudaMemcpyAsync(P.d_Wc.p, Wd.data(), H.n * 8, cudaMemcpyHostToDevice, s));
        TPG_CK(cudaMemcpyAsync(P.d_Wv.p, Vd.data(), H.n * 8, cudaMemcpyHostToDevice, s));
    }
    // (4) cross prime paths of the head records
    const int64_t n_heads = (int64_t)cpp[5];
    uint64_t cross = 0, cross_v = 0;
    if (n_heads > 0) {
        TPG_TRY(P.hcomp.ensure((size_t)n_heads * 8, s));
        TPG_CK(cudaMemsetAsync(ctr + 20, 0, 24, s));
        head_weight_s_kernel<<<grid_for(n_heads, 256, P.num_sms * 8), 256, 0, s>>>(
            G, P.cheads.as<HeadS>(), n_heads, P.hcomp.as<uint64_t>(), ctr + 20);
        launches++;
        unsigned long long hc[3];
        TPG_CK(cudaMemcpyAsync(hc, ctr + 20, 24, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        if (hc[2]) {
            set_error("cross-SCC prime-path count exceeds 2^62");
            return TPGEN_ERR_LIMIT_EXCEEDED;
        }
        cross = hc[0];
        cross_v = hc[1];
    }
    uint64_t n_pp = 0, n_vert = 0;
    {
        const uint64_t parts[3][2] = {{cseg[0], cseg[1]}, {cpp[0], cpp[1]}, {cross, cross_v}};
        for (const auto &pr : parts) {
            const uint64_t a = n_pp + pr[0], b = n_vert + pr[1];
            if (a < n_pp || b < n_vert || a >= (1ull << 62) || b >= (1ull << 62)) {
                set_error("prime-path count exceeds 2^62");
                return TPGEN_ERR_LIMIT_EXCEEDED;
            }
            n_pp = a;
            n_vert = b;
        }
    }
    st.n_paths = (int64_t)n_pp;
    st.total_vertices = (int64_t)n_vert;
    st.n_cross = (int64_t)cross;
    st.n_extensions = (int64_t)(cseg[2] + cpp[2] + presplit_ext);
    st.n_heads = n_heads;
    st.n_segments = (int64_t)cseg[7];
    if ((o.max_paths > 0 && st.n_paths > o.max_paths) || (o.max_extensions > 0 && st.n_extensions > o.max_extensions)) {
        set_error("result exceeds max_paths / max_extensions");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    // (5) digests of the cross prime paths
    cudaEventRecord(tst.a, s);
    uint64_t hd[2] = {cseg[3] + cpp[3], cseg[4] + cpp[4]};
    if (o.compute_digest && n_heads > 0 && cross > 0) {
        const int64_t n_slots = (int64_t)cseg[7];  // item slots written by the segment phase (holes: ent < 0)
        const int32_t nv = std::max(H.n, 1);
        TPG_TRY(P.icnt.ensure((size_t)nv * 8 * 3, s));
        uint64_t *icnt = P.icnt.as<uint64_t>(), *istart = icnt + nv, *icur = icnt + 2 * (size_t)nv;
        TPG_CK(cudaMemsetAsync(icnt, 0, (size_t)nv * 8, s));
        item_count_s_kernel<<<grid_for(n_slots, 256, P.num_sms * 8), 256, 0, s>>>(P.citems.as<ItemS>(), n_slots,
                                                                                 reinterpret_cast<unsigned long long *>(icnt));
        TPG_CK(cudaMemcpyAsync(istart, icnt, (size_t)nv * 8, cudaMemcpyDeviceToDevice, s));
        uint64_t n_items = 0;
        uint64_t *sa[1] = {istart};
        TPG_TRY(scan_multi(P, sa, 1, nv, &n_items, s, launches));
        TPG_CK(cudaMemcpyAsync(icur, istart, (size_t)nv * 8, cudaMemcpyDeviceToDevice, s));
        TPG_TRY(P.citems2.ensure(std::max<uint64_t>(n_items, 1) * sizeof(ItemS), s));
        item_scatter_s_kernel<<<grid_for(n_slots, 256, P.num_sms * 8), 256, 0, s>>>(
            P.citems.as<ItemS>(), n_slots, reinterpret_cast<unsigned long long *>(icur), P.citems2.as<ItemS>());
        TPG_TRY(P.ibeg.ensure((size_t)nv * 8, s));
        TPG_TRY(P.iend.ensure((size_t)nv * 8, s));
        item_bounds_s_kernel<<<grid_for(nv, 256, 1024), 256, 0, s>>>(istart, icnt, nv, P.ibeg.as<int64_t>(),
                                                                    P.iend.as<int64_t>());
        TPG_TRY(P.icum.ensure((size_t)std::max<uint64_t>(n_items, 1) * 8, s));
        TPG_TRY(P.ivcum.ensure((size_t)std::max<uint64_t>(n_items, 1) * 8, s));
        item_weight_s_kernel<<<grid_for((int64_t)n_items, 256, P.num_sms * 8), 256, 0, s>>>(
            G, P.citems2.as<ItemS>(), (int64_t)n_items, P.icum.as<uint64_t>(), P.ivcum.as<uint64_t>());
        launches += 4;
        uint64_t tot2[2];
        uint64_t *ia[2] = {P.icum.as<uint64_t>(), P.ivcum.as<uint64_t>()};
        TPG_TRY(scan_multi(P, ia, 2, (int64_t)n_items, tot2, s, launches));
        uint64_t *ha[1] = {P.hcomp.as<uint64_t>()};
        uint64_t ncomp = 0;
        TPG_TRY(scan_multi(P, ha, 1, n_heads, &ncomp, s, launches));
        HT("items grouped");
        StitchSArgs SA;
        SA.tp = P.cur_tp;
        SA.unreachable = reinterpret_cast<unsigned int *>(ctr + 23);
        TPG_CK(cudaMemsetAsync(ctr + 23, 0, 8, s));
        SA.heads = P.cheads.as<HeadS>();
        SA.n_heads = n_heads;
        SA.comp_off = P.hcomp.as<uint64_t>();
        SA.n_comp = ncomp;
        SA.items = P.citems2.as<ItemS>();
        SA.cum = P.icum.as<uint64_t>();
        SA.ibeg = P.ibeg.as<int64_t>();
        SA.iend = P.iend.as<int64_t>();
        unsigned long long *hacc = ctr + 24;  // digest a, b; vertices
        TPG_CK(cudaMemsetAsync(hacc, 0, 24, s));
        // small heads (<= kSmallHead completions): a thread per head; big ones: a thread per completion
        TPG_TRY(P.sscratch.ensure((size_t)n_heads * 8 * 3 + 64, s));
        uint64_t *big = P.sscratch.as<uint64_t>();
        int64_t *bidx = reinterpret_cast<int64_t *>(big + n_heads);
        uint64_t *bw = big + 2 * n_heads;
        stitch_small_kernel<<<grid_for(n_heads, 256, P.num_sms * 8), 256, 0, s>>>(SA, G, big, hacc);
        uint64_t n_big = 0;
        uint64_t *ba[1] = {big};
        TPG_TRY(scan_multi(P, ba, 1, n_heads, &n_big, s, launches));
        launches++;
        if (n_big > 0) {
            stitch_big_list_kernel<<<grid_for(n_heads, 256, P.num_sms * 8), 256, 0, s>>>(SA, big, bidx, bw);
            uint64_t n_big_comp = 0;
            uint64_t *bwa[1] = {bw};
            TPG_TRY(scan_multi(P, bwa, 1, (int64_t)n_big, &n_big_comp, s, launches));
            stitch_big_kernel<<<grid_for((int64_t)n_big_comp, 256, P.num_sms * 8), 256, 0, s>>>(
                SA, G, bidx, bw, (int64_t)n_big, n_big_comp, hacc);
            launches += 2;
        }
        unsigned long long hh[3], unr = 0;
        TPG_CK(cudaMemcpyAsync(hh, hacc, 24, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaMemcpyAsync(&unr, ctr + 23, 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        if (unr) {
            set_error("a prime path's last vertex cannot reach exit");
            return TPGEN_ERR_UNREACHABLE;
        }
        hd[0] += hh[0];
        hd[1] += hh[1];
        if (P.cur_tp) {  // test paths: the cross ones' vertices include their suffix walks (known only here)
            st.total_vertices = (int64_t)(n_vert - cross_v + hh[2]);
        }
    }
    cudaEventRecord(tst.b, s);
    cudaEventRecord(tall.b, s);
    TPG_CK(cudaGetLastError());
    TPG_CK(cudaStreamSynchronize(s));
    if (o.compute_digest) {
        st.hash_lo = hd[0];
        st.hash_hi = hd[1];
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, tall.a, tall.b);
    st.ms_device = ms;
    cudaEventElapsedTime(&ms, tst.a, tst.b);
    st.ms_stitch = ms;
    st.ms_count = st.ms_device - st.ms_stitch;
    st.ms_dfs_count = ms_dfs;
    st.ms_dfs_write = ms_dfs;
    st.gpu_launches = launches;
    st.ms_total = now_ms() - t0;
    if (stp) *stp = st;
    return TPGEN_OK;
}

template <class T>
static tpgen_status run_count(PlanImpl &P, const tpgen_options &o, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: prime paths (count mode)");
    const double t0 = now_ms();
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    int64_t launches = 0;
    const HostPlan &H = P.hp;
    cudaStream_t s = (cudaStream_t)o.stream;
    int32_t lo = 0, hi = H.n;
    shard_range(H, o.shard_rank, o.shard_count, lo, hi);
    if (o.start_hi > o.start_lo) {
        lo = std::max(0, o.start_lo);
        hi = std::min(H.n, o.start_hi);
    }
    // graphs with no arc leaving any SCC start from host pre-split tries (below); with shard_prefix the
    // shard is a range of them
    const bool presplit_ok = std::is_same<T, uint32_t>::value && !P.any_exit && !getenv("TPGEN_NO_PRESPLIT");
    int64_t pfx_key = -1;
    const PrefixShard *pfx = prefix_shard_call(P, o, presplit_ok, lo, hi, pfx_key);
    st.unit_lo = pfx ? pfx->ulo : -1;
    st.unit_hi = pfx ? pfx->uhi : -1;
    st.shard_lo = lo;
    st.shard_hi = hi;
    st.n_scc = H.n_scc;
    st.n_scc_nontrivial = H.n_nontrivial;
    st.max_scc = H.max_scc;
    st.ms_plan = P.ms_plan;
    P.overflow = false;
    P.tp_unreachable = false;
    P.maxgen = 0;
    P.cur_prune = o.prune;
    const int mode = o.compute_digest ? M_CNT : M_CNT_NOHASH;
    const bool hdbg = getenv("TPGEN_DEBUG") != nullptr;  // host stage marks, synchronised
    auto HT = [&](const char *what) {
        if (!hdbg) return;
        cudaStreamSynchronize(s);
        fprintf(stderr, "[tpgen count] %-28s %s\n", what, cudaGetErrorString(cudaGetLastError()));
    };
    Timer tall, tst;
    cudaEventRecord(tall.a, s);
    const DevGraph G = dev_graph(P, lo, hi);
    // roots: one K_NODE unit per start vertex (segment phase: every SCC entry; prime-path phase: the
    // range's other vertices)
    std::vector<Unit<1>> seg_roots, pp_roots;
    for (int32_t v = 0; v < H.n; v++) {
        const int32_t slot = H.v_slot[v];
        const bool entry = (H.slot_flags[slot] & F_ENTRY) != 0;
        if (!entry && !(v >= lo && v < hi)) continue;
        Unit<1> u;
        memset(&u, 0, sizeof(u));
        const int32_t c = H.comp[v];
        const int loc = slot - H.scc_vbase[c];
        u.M[0] = 1ull << loc;
        u.scc = c;
        u.e = -1;
        u.kind = K_NODE;
        u.path[0] = (uint8_t)loc;
        (entry ? seg_roots : pp_roots).push_back(u);
    }
    const size_t agg_n = 2 * (size_t)H.n + 2 * (size_t)H.n_pairs + 1;
    TPG_TRY(P.ctr.ensure(32 * 8, s));
    TPG_TRY(P.agg.ensure(agg_n * 8, s));
    TPG_TRY(P.agg_bak.ensure(agg_n * 8, s));
    TPG_CK(cudaMemsetAsync(P.agg.p, 0, agg_n * 8, s));
    unsigned long long *ctr = P.ctr.as<unsigned long long>();
    // graphs with no arc leaving any SCC: the host pre-split trie tops (cached per plan and range)
    RootSpan<1> pp_span(pp_roots);
    uint64_t presplit_ext = 0;
    if (presplit_ok && seg_roots.empty()) {
        if (!(P.presplit_lo == lo && P.presplit_hi == hi && P.presplit_key == pfx_key && P.presplit_dev.p)) {
            const int64_t lanes = (int64_t)P.num_sms * CntCfg<uint32_t>::min_blocks * CntCfg<uint32_t>::threads;
            std::vector<Unit<1>> units;
            int64_t target = lanes;
            if (const char *ev = getenv("TPGEN_PRESPLIT_TARGET")) target = atoll(ev);
            presplit_roots<1>(P, lo, hi, target, units, P.presplit_gid, P.presplit_ext, pfx);
            P.presplit_host.assign(reinterpret_cast<const uint8_t *>(units.data()),
                                   reinterpret_cast<const uint8_t *>(units.data() + units.size()));
            P.presplit_n = (int64_t)units.size();
            P.presplit_roots_n = -1;
            TPG_TRY(upload(P.presplit_dev, P.presplit_host, s));
            P.presplit_lo = lo;
            P.presplit_hi = hi;
            P.presplit_key = pfx_key;
        }
        pp_span = RootSpan<1>(reinterpret_cast<const Unit<1> *>(P.presplit_host.data()), (size_t)P.presplit_n);
        presplit_ext = P.presplit_ext;
        P.presplit_active = true;
    }
    double ms_dfs = 0;
    uint64_t tail_seg = 0, tail = 0;
    unsigned long long cseg[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cpp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // (1) segment phase
    if (!seg_roots.empty())
        TPG_TRY(dfs_phase<T>(P, G, RootSpan<1>(seg_roots), 1, 0, s, st, launches, ms_dfs, tail_seg, mode, cseg));
    HT("segment phase");
    // (3) prime-path phase
    {
        double ms_pp = 0;
        const tpgen_status r = dfs_phase<T>(P, G, pp_span, 0, tail_seg, s, st, launches, ms_dfs, tail, mode, cpp, &ms_pp);
        P.presplit_active = false;
        if (r != TPGEN_OK) return r;
        st.ms_dominant = ms_pp;
        st.ext_dominant = (int64_t)cpp[2];
    }
    if (P.overflow) {
        set_error("prime-path count exceeds 2^62");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    if (P.tp_unreachable) {
        set_error("a prime path's first vertex is unreachable from entry or its last cannot reach exit");
        return TPGEN_ERR_UNREACHABLE;
    }
    st.n_units = (int64_t)tail;
    HT("prime-path phase");
    return count_post(P, o, G, s, !seg_roots.empty(), cseg, cpp, presplit_ext, st, launches, tall, tst, ms_dfs, t0,
                      stp);
}

// ------------------------------------------------------------ frontier engine
// TPGEN_ENGINE_FRONTIER (frontier.cuh): level-synchronous
// extension of all paths of one length at a time; counts, E_canon and digest.
template <class T>
static tpgen_status run_frontier(PlanImpl &P, const tpgen_options &o, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: frontier engine");
    const bool hash = o.compute_digest != 0;  // without the digest: no S, no mixing
    const size_t kRecB = (sizeof(T) == 4 ? 8 : 16) + (hash ? 8 : 0);  // bytes per frontier record (key [+ S])
    const double t0 = now_ms();
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    const HostPlan &H = P.hp;
    if (H.max_scc > 64 || H.W != 1 || H.n >= (1 << 21)) {
        set_error("the frontier engine needs SCCs of <= 64 vertices (use the DFS engine)");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    cudaStream_t s = (cudaStream_t)o.stream;
    int32_t lo = 0, hi = H.n;
    shard_range(H, o.shard_rank, o.shard_count, lo, hi);
    if (o.start_hi > o.start_lo) {
        lo = std::max(0, o.start_lo);
        hi = std::min(H.n, o.start_hi);
    }
    st.shard_lo = lo;
    st.shard_hi = hi;
    st.n_scc = H.n_scc;
    st.n_scc_nontrivial = H.n_nontrivial;
    st.max_scc = H.max_scc;
    st.ms_plan = P.ms_plan;
    const int W = H.W;
    // slot table (uploaded once per plan)
    const int32_t n_tab = std::max(H.n, 1);
    if (!P.f_tab_ok) {
        std::vector<FSlot<T>> tab(n_tab, FSlot<T>{0, 0, 0, 0});
        for (int32_t i = 0; i < H.n; i++)
            tab[i] = FSlot<T>{(T)H.sin[(size_t)i * W], (T)H.pin[(size_t)i * W], H.slot_gid[i], H.slot_flags[i]};
        TPG_TRY(upload(P.f_tab, tab, s));
        P.f_tab_ok = true;
    }
    const int32_t n_roots = std::max(hi - lo, 0);
    if (n_roots && !(P.f_roots_lo == lo && P.f_roots_hi == hi)) {  // root table cached per start range
        std::vector<int32_t> roots;  // slots, then slot bases
        roots.reserve(2 * (size_t)n_roots);
        for (int32_t v = lo; v < hi; v++) roots.push_back(H.v_slot[v]);
        for (int32_t v = lo; v < hi; v++) roots.push_back(H.scc_vbase[H.comp[v]]);
        TPG_TRY(upload(P.f_roots, roots, s));
        P.f_roots_lo = lo;
        P.f_roots_hi = hi;
    }
    const int Lmax = std::max(H.max_scc, 1);  // records exist for paths of 1..max_scc vertices
    const size_t nctr = 8 + (size_t)Lmax + 2;
    TPG_TRY(P.f_ctr.ensure(nctr * 8, s));
    unsigned long long *ctr = P.f_ctr.as<unsigned long long>();
    double est = 0;
    for (int32_t v = lo; v < hi; v++) est += H.cost[v];
    uint64_t cap = std::max<uint64_t>({1ull << 22, (uint64_t)(est / 4), P.f_cap_hwm + P.f_cap_hwm / 4});
    if (const char *ev = getenv("TPGEN_FRONTIER_CAP")) cap = std::max<uint64_t>(64, atoll(ev));  // test hook: retries
    uint64_t cap_max = ~0ull;  // memory budget: queried only when a buffer has to grow
    // free device memory the frontier may use: cudaMemGetInfo, or the TPGEN_FRONTIER_BUDGET test hook
    // (bytes), plus what the frontier buffers already hold
    auto free_mem = [&](size_t &f) -> tpgen_status {
        size_t free_b = 0, total_b = 0;
        TPG_CK(cudaMemGetInfo(&free_b, &total_b));
        if (const char *ev = getenv("TPGEN_FRONTIER_BUDGET")) free_b = (size_t)strtoull(ev, nullptr, 10);
        f = free_b + P.f_buf0.cap + P.f_buf1.cap;
        return TPGEN_OK;
    };
    auto budget = [&]() -> tpgen_status {  // two ping-pong buffers of exactly cap records: 90 % of it
        size_t f = 0;
        TPG_TRY(free_mem(f));
        cap_max = (uint64_t)((double)f * 0.45 / kRecB);
        return TPGEN_OK;
    };
    if (cap * kRecB > std::min(P.f_buf0.cap, P.f_buf1.cap)) TPG_TRY(budget());
    const size_t smem = (size_t)n_tab * sizeof(FSm<T>);
    const bool ts = smem <= 32 * 1024;
    void (*const level_k)(FrontierArgs) =
        ts ? (hash ? frontier_level_kernel<T, true, true> : frontier_level_kernel<T, true, false>)
           : (hash ? frontier_level_kernel<T, false, true> : frontier_level_kernel<T, false, false>);
    void (*const root_k)(FrontierArgs, const int32_t *, const int32_t *, int32_t) =
        hash ? frontier_root_kernel<T, true> : frontier_root_kernel<T, false>;
    const size_t lsmem = ts ? smem : 0;
    static int occ[2][2] = {{0, 0}, {0, 0}};  // resident blocks per SM per variant (per build; queried once)
    int &per_sm = occ[ts ? 1 : 0][hash ? 1 : 0];
    if (per_sm == 0) TPG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_k, kFThreads, ts ? 32 * 1024 : 0));
    const int grid = P.num_sms * std::max(per_sm, 1);
    Timer tall;
    const bool kdbg = getenv("TPGEN_DEBUG") != nullptr;  // a synchronised error check after every launch
    auto KC = [&](const char *what, int l) -> tpgen_status {
        if (!kdbg) return TPGEN_OK;
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            fprintf(stderr, "[tpgen frontier] %s level %d: %s\n", what, l, cudaGetErrorString(e));
            set_error(std::string("frontier ") + what + ": " + cudaGetErrorString(e));
            return TPGEN_ERR_CUDA;
        }
        return TPGEN_OK;
    };
    std::vector<unsigned long long> h(nctr);
    int64_t launches = 0;
    float ms = 0;
    uint64_t recs = 0;
    bool chunked = false;
    uint64_t capc = 0;  // chunked mode: records per level buffer
    if (const char *ev = getenv("TPGEN_FRONTIER_CHUNK")) {  // test hook: force the DFS-chunked frontier
        chunked = true;
        capc = std::max<uint64_t>(64, atoll(ev));
    }
    for (int attempt = 0; !chunked; attempt++) {
        cap = std::min(cap, cap_max);
        if (cap_max != ~0ull) {  // under a memory budget: exact sizes (the budget counts every byte)
            TPG_TRY(P.f_buf0.ensure_exact(cap * kRecB, s));
            TPG_TRY(P.f_buf1.ensure_exact(cap * kRecB, s));
        } else {
            TPG_TRY(P.f_buf0.ensure(cap * kRecB, s));
            TPG_TRY(P.f_buf1.ensure(cap * kRecB, s));
        }
        ulonglong2 *buf[2] = {P.f_buf0.as<ulonglong2>(), P.f_buf1.as<ulonglong2>()};
        uint64_t *bufS[2] = {reinterpret_cast<uint64_t *>(buf[0] + cap), reinterpret_cast<uint64_t *>(buf[1] + cap)};
        TPG_CK(cudaMemsetAsync(ctr, 0, nctr * 8, s));
        cudaEventRecord(tall.a, s);
        FrontierArgs A;
        memset(&A, 0, sizeof(A));
        A.tab = P.f_tab.p;
        A.n_tab = n_tab;
        A.cap = cap;
        A.lim = ~0ull;
        A.acc = ctr;
        A.overflow = reinterpret_cast<unsigned int *>(ctr + 5);
        if (n_roots) {
            A.in = nullptr;
            A.in_S = nullptr;
            A.out = buf[0];
            A.out_S = bufS[0];
            A.cnt_in = nullptr;
            A.cnt_out = ctr + 8;
            A.l = -1;
            root_k<<<(n_roots + 255) / 256, 256, 0, s>>>(A, P.f_roots.as<int32_t>(),
                                                                        P.f_roots.as<int32_t>() + n_roots, n_roots);
            launches++;
            TPG_TRY(KC("root", -1));
            for (int l = 0; l < Lmax; l++) {
                A.in = buf[l & 1];
                A.in_S = bufS[l & 1];
                A.out = buf[(l + 1) & 1];
                A.out_S = bufS[(l + 1) & 1];
                A.cnt_in = ctr + 8 + l;
                A.cnt_out = ctr + 8 + l + 1;
                A.l = l;
                level_k<<<grid, kFThreads, lsmem, s>>>(A);
                launches++;
                TPG_TRY(KC("level", l));
            }
        }
        cudaEventRecord(tall.b, s);
        TPG_CK(cudaGetLastError());
        TPG_CK(cudaMemcpyAsync(h.data(), ctr, nctr * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        cudaEventElapsedTime(&ms, tall.a, tall.b);
        uint64_t peak = 0;
        for (int l = 0; l <= Lmax; l++) peak = std::max<uint64_t>(peak, h[8 + l]);
        if (!(h[5] & 1u)) {
            P.f_cap_hwm = std::max<uint64_t>(P.f_cap_hwm, peak);
            for (int l = 0; l <= Lmax; l++) recs += h[8 + l];
            break;
        }
        st.n_count_rounds = attempt + 1;
        if (cap_max == ~0ull) TPG_TRY(budget());
        if (cap >= cap_max) {  // no level fits: the DFS-chunked frontier in the same memory
            chunked = true;
            break;
        }
        cap = std::max<uint64_t>(2 * cap, peak + peak / 4);  // a truncated level under-counts the next ones
    }
    if (chunked) {
        const size_t stride_b = std::max<size_t>(kRecB, 16);  // (16-B level stride of the key array)
        if (capc == 0) {  // automatic switch: release the second buffer, then one buffer per level
            P.f_buf1.release(s);
            size_t f = 0;
            TPG_TRY(free_mem(f));
            capc = (uint64_t)((double)f * 0.9 / ((double)(Lmax + 1) * stride_b));
        }
        // DFS over chunks of levels (the north star's "DFS-chunked when the frontier would
        // overflow HBM"): one buffer of capc records per level; a chunk of level l holds at
        // most capc / D records (D = the largest out-degree), so its children always fit in
        // level l+1's buffer, which is consumed completely before level l's next chunk.
        uint32_t D = 1;
        for (int32_t i = 0; i < H.n; i++) D = std::max<uint32_t>(D, (uint32_t)__builtin_popcountll(H.sin[(size_t)i * W]));
        if (capc < (uint64_t)std::max<int64_t>(n_roots, D)) {
            set_error("frontier chunk buffers too small for the roots (use the DFS engine)");
            return TPGEN_ERR_OUT_OF_MEMORY;
        }
        TPG_TRY(P.f_buf0.ensure_exact((size_t)(Lmax + 1) * capc * stride_b, s));
        ulonglong2 *base = P.f_buf0.as<ulonglong2>();
        uint64_t *baseS = reinterpret_cast<uint64_t *>(base + (size_t)(Lmax + 1) * capc);
        TPG_CK(cudaMemsetAsync(ctr, 0, nctr * 8, s));
        cudaEventRecord(tall.a, s);
        FrontierArgs A;
        memset(&A, 0, sizeof(A));
        A.tab = P.f_tab.p;
        A.n_tab = n_tab;
        A.cap = capc;
        A.acc = ctr;
        A.overflow = reinterpret_cast<unsigned int *>(ctr + 5);
        if (Lmax + 1 > kFMaxLevels) {
            set_error("frontier: SCC larger than 64 vertices");
            return TPGEN_ERR_INVALID_ARGUMENT;
        }
        TPG_TRY(P.f_sched.ensure(sizeof(FChunk), s));
        FChunk *fc = P.f_sched.as<FChunk>();
        TPG_CK(cudaMemsetAsync(fc, 0, sizeof(FChunk), s));
        cudaGraphExec_t gexec = nullptr;
        if (n_roots) {
            A.lim = ~0ull;
            A.in = nullptr;
            A.in_S = nullptr;
            A.out = base;
            A.out_S = baseS;
            A.cnt_in = nullptr;
            A.cnt_out = ctr + 8;
            A.l = -1;
            root_k<<<(n_roots + 255) / 256, 256, 0, s>>>(A, P.f_roots.as<int32_t>(),
                                                                        P.f_roots.as<int32_t>() + n_roots, n_roots);
            launches++;
            TPG_TRY(KC("root", -1));
            // the walk over chunks: a graph with one conditional WHILE node whose body is
            // [frontier_sched_kernel -> frontier_chunk_kernel] (no host round trip per chunk)
            FSchedArgs sa;
            sa.c = fc;
            sa.ctr = ctr;
            sa.base = base;
            sa.baseS = baseS;
            sa.capc = capc;
            sa.chunk = std::max<uint64_t>(1, capc / D);
            sa.chunk_div = D;
            sa.key_b = (sizeof(T) == 4 && !hash) ? 8u : 16u;
            sa.Lmax = Lmax;
            void (*const chunk_k)(FrontierArgs, const FChunk *) =
                ts ? (hash ? frontier_chunk_kernel<T, true, true> : frontier_chunk_kernel<T, true, false>)
                   : (hash ? frontier_chunk_kernel<T, false, true> : frontier_chunk_kernel<T, false, false>);
            cudaGraph_t g = nullptr;
            TPG_CK(cudaGraphCreate(&g, 0));
            auto build = [&]() -> cudaError_t {
                cudaGraphConditionalHandle hdl;
                cudaError_t e = cudaGraphConditionalHandleCreate(&hdl, g, 1, cudaGraphCondAssignDefault);
                if (e != cudaSuccess) return e;
                cudaGraphNodeParams cp = {};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = hdl;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t cn;
                if ((e = cudaGraphAddNode(&cn, g, nullptr, 0, &cp)) != cudaSuccess) return e;
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                void *sargs[2] = {&sa, &hdl};
                cudaKernelNodeParams kp;
                memset(&kp, 0, sizeof(kp));
                kp.func = reinterpret_cast<void *>(&frontier_sched_kernel);
                kp.gridDim = dim3(1);
                kp.blockDim = dim3(32);
                kp.kernelParams = sargs;
                cudaGraphNode_t n_sched, n_lvl;
                if ((e = cudaGraphAddKernelNode(&n_sched, body, nullptr, 0, &kp)) != cudaSuccess) return e;
                const FChunk *fcc = fc;
                void *largs[2] = {&A, &fcc};
                kp.func = reinterpret_cast<void *>(chunk_k);
                kp.gridDim = dim3(grid);
                kp.blockDim = dim3(kFThreads);
                kp.sharedMemBytes = (unsigned)lsmem;
                kp.kernelParams = largs;
                if ((e = cudaGraphAddKernelNode(&n_lvl, body, &n_sched, 1, &kp)) != cudaSuccess) return e;
                return cudaGraphInstantiate(&gexec, g, 0);
            };
            const char *wv = getenv("TPGEN_FRONTIER_WALK");  // A/B hook: "graph" = the conditional-node walk
            if (wv && strcmp(wv, "graph") == 0) {
                const cudaError_t be = build();
                cudaGraphDestroy(g);
                TPG_CK(be);
                TPG_CK(cudaGraphLaunch(gexec, s));
                TPG_TRY(KC("chunk graph", 0));
            } else {  // one persistent cooperative launch, a grid barrier per chunk
                cudaGraphDestroy(g);
                void (*const walk_k)(FrontierArgs, FSchedArgs) =
                    ts ? (hash ? frontier_walk_kernel<T, true, true> : frontier_walk_kernel<T, true, false>)
                       : (hash ? frontier_walk_kernel<T, false, true> : frontier_walk_kernel<T, false, false>);
                int wper = 0;
                TPG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, walk_k, kFThreads, lsmem));
                const int wgrid = P.num_sms * std::max(wper, 1);
                void *wargs[2] = {&A, &sa};
                TPG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(walk_k), dim3(wgrid), dim3(kFThreads), wargs,
                                                   lsmem, s));
                TPG_TRY(KC("chunk walk", 0));
            }
        }
        cudaEventRecord(tall.b, s);
        TPG_CK(cudaGetLastError());
        TPG_CK(cudaMemcpyAsync(h.data(), ctr, nctr * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        cudaEventElapsedTime(&ms, tall.a, tall.b);
        if (n_roots) {
            if (gexec) cudaGraphExecDestroy(gexec);
            FChunk hc;
            TPG_CK(cudaMemcpy(&hc, fc, sizeof(FChunk), cudaMemcpyDeviceToHost));
            recs += hc.recs;
            const char *wv = getenv("TPGEN_FRONTIER_WALK");
            launches += (wv && strcmp(wv, "graph") == 0) ? 2 * (int64_t)(hc.steps + 1) : 1;  // (sched + level per pass)
            st.n_count_rounds = (int32_t)hc.steps;     // chunks
        }
        if (h[5] & 1u) {
            set_error("frontier chunk overflow (internal)");
            return TPGEN_ERR_INTERNAL;
        }
    }
    st.n_paths = (int64_t)h[0];
    st.total_vertices = (int64_t)h[1];
    st.n_extensions = (int64_t)h[2];
    st.hash_lo = h[3];
    st.hash_hi = h[4];
    st.n_units = (int64_t)recs;  // frontier records written (all levels)
    if ((o.max_paths > 0 && st.n_paths > o.max_paths) || (o.max_extensions > 0 && st.n_extensions > o.max_extensions)) {
        set_error("result exceeds max_paths / max_extensions");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    st.ms_device = ms;
    st.ms_count = ms;
    st.ms_dfs_count = ms;
    st.ms_dfs_write = ms;
    st.ms_dominant = ms;  // (all level launches of the call)
    st.ext_dominant = st.n_extensions;
    st.gpu_launches = launches;
    st.ms_total = now_ms() - t0;
    if (stp) *stp = st;
    return TPGEN_OK;
}

// One frontier pass over a root set for graphs whose arcs leave SCCs: all
// levels, ping-pong buffers, retried bigger when a level or the head / item buffer overflows.
// HX: heads (prime-path phase); SEG: the segment phase (items; records carry B).  out[0..4]: the
// pass's prime paths, vertices, E_canon, digest a, b; *ev_slots: head or item slots reserved.
template <class T, bool SEG>
static tpgen_status frontier_pass(PlanImpl &P, const tpgen_options &o, cudaStream_t s, int32_t lo, int32_t hi,
                                  const std::vector<int32_t> &roots, bool hash, unsigned long long *out,
                                  unsigned long long *ev_slots, double &ms, int64_t &launches, uint64_t &recs) {
    NvtxRange nvtx_range(SEG ? "tpgen: frontier segment pass" : "tpgen: frontier prime-path pass");
    const HostPlan &H = P.hp;
    const int32_t n_roots = (int32_t)(roots.size() / 2);
    memset(out, 0, 5 * sizeof(unsigned long long));
    *ev_slots = 0;
    if (n_roots == 0) return TPGEN_OK;
    const size_t key_b = 16, s_b = sizeof(T) == 8 ? 8 : 0, b_b = SEG ? 8 : 0;
    const size_t kRecB = key_b + s_b + b_b;
    const int Lmax = std::max(H.max_scc, 1);
    const size_t nctr = 8 + (size_t)Lmax + 2;
    TPG_TRY(P.f_ctr.ensure((nctr + 8) * 8, s));
    unsigned long long *ctr = P.f_ctr.as<unsigned long long>();
    TPG_TRY(upload(P.f_roots, roots, s));
    P.f_roots_lo = P.f_roots_hi = -1;  // (the no-exit engine's cached root table is gone)
    double est = 0;
    for (size_t i = 0; i < (size_t)n_roots; i++) est += H.cost[H.slot_gid[roots[i]]];
    uint64_t cap = std::max<uint64_t>({1ull << 20, (uint64_t)(est / 4), P.f_cap_hwm + P.f_cap_hwm / 4});
    if (const char *ev = getenv("TPGEN_FRONTIER_CAP")) cap = std::max<uint64_t>(64, atoll(ev));
    DevBuf &evb = SEG ? P.citems : P.cheads;
    const size_t ev_es = SEG ? sizeof(ItemS) : sizeof(HeadS);
    uint64_t &ev_hwm = SEG ? P.citem_hwm : P.chead_hwm;
    {
        const uint64_t want = std::max<uint64_t>(1ull << 20, ev_hwm + ev_hwm / 4 + 256ull * 4096);
        if (evb.cap < want * ev_es) TPG_TRY(evb.ensure(want * ev_es, s));
    }
    const size_t smem = (size_t)std::max(H.n, 1) * sizeof(FSm<T>);
    const bool ts = smem <= 32 * 1024;
    void (*const level_k)(FrontierArgs) =
        ts ? (hash ? frontier_level_kernel<T, true, true, true, SEG> : frontier_level_kernel<T, true, false, true, SEG>)
           : (hash ? frontier_level_kernel<T, false, true, true, SEG> : frontier_level_kernel<T, false, false, true, SEG>);
    void (*const root_k)(FrontierArgs, const int32_t *, const int32_t *, int32_t) =
        hash ? frontier_root_kernel<T, true, true, SEG> : frontier_root_kernel<T, false, true, SEG>;
    int per_sm = 0;
    TPG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_k, kFThreads, ts ? (int)smem : 0));
    const int grid = P.num_sms * std::max(per_sm, 1);
    std::vector<unsigned long long> h(nctr + 8);
    Timer t;
    const char *chunk_hook = getenv("TPGEN_FRONTIER_CHUNK");  // test hook: force the DFS-chunked walk
    bool chunked = chunk_hook != nullptr;
    for (int attempt = 0; attempt < 24 && !chunked; attempt++) {
        size_t f = 0, tot = 0;
        TPG_CK(cudaMemGetInfo(&f, &tot));
        if (const char *ev = getenv("TPGEN_FRONTIER_BUDGET")) f = (size_t)strtoull(ev, nullptr, 10);
        const uint64_t cap_max = (uint64_t)((double)(f + P.f_buf0.cap + P.f_buf1.cap) * 0.45 / kRecB);
        if (cap > cap_max) {  // no level fits twice: the DFS-chunked walk in the same memory
            chunked = true;
            break;
        }
        if (2.5 * (double)(cap * kRecB) > 0.9 * (double)(f + P.f_buf0.cap + P.f_buf1.cap)) {  // near the budget: no headroom
            TPG_TRY(P.f_buf0.ensure_exact(cap * kRecB, s));
            TPG_TRY(P.f_buf1.ensure_exact(cap * kRecB, s));
        } else {
            TPG_TRY(P.f_buf0.ensure(cap * kRecB, s));
            TPG_TRY(P.f_buf1.ensure(cap * kRecB, s));
        }
        ulonglong2 *buf[2] = {P.f_buf0.as<ulonglong2>(), P.f_buf1.as<ulonglong2>()};
        uint64_t *bufS[2] = {reinterpret_cast<uint64_t *>(buf[0] + cap), reinterpret_cast<uint64_t *>(buf[1] + cap)};
        uint64_t *bufB[2] = {reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(buf[0]) + cap * (key_b + s_b)),
                             reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(buf[1]) + cap * (key_b + s_b))};
        TPG_CK(cudaMemsetAsync(ctr, 0, (nctr + 8) * 8, s));
        FrontierArgs A;
        memset(&A, 0, sizeof(A));
        A.tab = P.f_tab.p;
        A.n_tab = std::max(H.n, 1);
        A.cap = cap;
        A.lim = ~0ull;
        A.acc = ctr;
        A.overflow = reinterpret_cast<unsigned int *>(ctr + 5);
        A.heads = P.cheads.as<HeadS>();
        A.head_cap = SEG ? 0 : P.cheads.cap / sizeof(HeadS);
        A.items = P.citems.as<ItemS>();
        A.item_cap = SEG ? P.citems.cap / sizeof(ItemS) : 0;
        A.hcnt = ctr + nctr;
        A.slot_mix = P.d_slot_mix.as<uint64_t>();
        A.shard_lo = lo;
        A.shard_hi = hi;
        cudaEventRecord(t.a, s);
        A.out = buf[0];
        A.out_S = bufS[0];
        A.out_B = bufB[0];
        A.cnt_out = ctr + 8;
        A.l = -1;
        root_k<<<(n_roots + 255) / 256, 256, 0, s>>>(A, P.f_roots.as<int32_t>(), P.f_roots.as<int32_t>() + n_roots,
                                                     n_roots);
        launches++;
        for (int l = 0; l < Lmax; l++) {
            A.in = buf[l & 1];
            A.in_S = bufS[l & 1];
            A.in_B = bufB[l & 1];
            A.out = buf[(l + 1) & 1];
            A.out_S = bufS[(l + 1) & 1];
            A.out_B = bufB[(l + 1) & 1];
            A.cnt_in = ctr + 8 + l;
            A.cnt_out = ctr + 8 + l + 1;
            A.l = l;
            level_k<<<grid, kFThreads, ts ? smem : 0, s>>>(A);
            launches++;
        }
        cudaEventRecord(t.b, s);
        TPG_CK(cudaGetLastError());
        TPG_CK(cudaMemcpyAsync(h.data(), ctr, (nctr + 8) * 8, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        const unsigned ovf = (unsigned)h[5];
        uint64_t peak = 0;
        for (int l = 0; l <= Lmax; l++) peak = std::max<uint64_t>(peak, h[8 + l]);
        const uint64_t used = h[nctr + (SEG ? 1 : 0)];
        if (ovf & 2u) {  // head / item buffer: room for all of them
            ev_hwm = std::max<uint64_t>(ev_hwm, used);
            TPG_TRY(evb.ensure((used + used / 4 + 256ull * 4096) * ev_es, s));
        }
        if (ovf & 1u) cap = std::max<uint64_t>(2 * cap, peak + peak / 4);
        if (ovf & 3u) continue;
        float m = 0;
        cudaEventElapsedTime(&m, t.a, t.b);
        ms += m;
        P.f_cap_hwm = std::max<uint64_t>(P.f_cap_hwm, peak);
        ev_hwm = std::max<uint64_t>(ev_hwm, used);
        for (int l = 0; l <= Lmax; l++) recs += h[8 + l];
        for (int q = 0; q < 5; q++) out[q] = h[q];
        *ev_slots = used;
        return TPGEN_OK;
    }
    if (!chunked) {
        set_error("frontier pass could not be sized");
        return TPGEN_ERR_OUT_OF_MEMORY;
    }
    // ---- the DFS-chunked walk: one ring of capc records per level, one persistent
    // cooperative launch; heads / items as in the one-pass form
    P.f_buf1.release(s);
    uint64_t capc = 0;
    {
        size_t f = 0, tot = 0;
        TPG_CK(cudaStreamSynchronize(s));
        TPG_CK(cudaMemGetInfo(&f, &tot));
        if (const char *ev = getenv("TPGEN_FRONTIER_BUDGET")) f = (size_t)strtoull(ev, nullptr, 10);
        f += P.f_buf0.cap;
        capc = chunk_hook ? (uint64_t)std::max<long long>(64, atoll(chunk_hook))
                          : (uint64_t)((double)f * 0.8 / ((double)(Lmax + 1) * kRecB));
    }
    uint32_t D = 1;
    for (int32_t i = 0; i < H.n; i++) D = std::max<uint32_t>(D, (uint32_t)__builtin_popcountll(H.sin[i]));
    if (capc < (uint64_t)std::max<int64_t>(n_roots, D) || Lmax + 1 > kFMaxLevels) {
        set_error("frontier chunk buffers too small for the roots (use the DFS engine)");
        return TPGEN_ERR_OUT_OF_MEMORY;
    }
    const size_t nlv = (size_t)(Lmax + 1) * capc;
    TPG_TRY(P.f_buf0.ensure_exact(nlv * kRecB, s));
    ulonglong2 *base = P.f_buf0.as<ulonglong2>();
    uint64_t *baseS = reinterpret_cast<uint64_t *>(base + nlv);
    uint64_t *baseB = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(base) + nlv * (key_b + s_b));
    TPG_TRY(P.f_sched.ensure(sizeof(FChunk), s));
    FChunk *fc = P.f_sched.as<FChunk>();
    void (*const walk_k)(FrontierArgs, FSchedArgs) =
        ts ? (hash ? frontier_walk_kernel<T, true, true, true, SEG> : frontier_walk_kernel<T, true, false, true, SEG>)
           : (hash ? frontier_walk_kernel<T, false, true, true, SEG> : frontier_walk_kernel<T, false, false, true, SEG>);
    int wper = 0;
    TPG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&wper, walk_k, kFThreads, ts ? (int)smem : 0));
    const int wgrid = P.num_sms * std::max(wper, 1);
    for (int attempt = 0; attempt < 24; attempt++) {
        TPG_CK(cudaMemsetAsync(ctr, 0, (nctr + 8) * 8, s));
        TPG_CK(cudaMemsetAsync(fc, 0, sizeof(FChunk), s));
        FrontierArgs A;
        memset(&A, 0, sizeof(A));
        A.tab = P.f_tab.p;
        A.n_tab = std::max(H.n, 1);
        A.cap = capc;
        A.lim = ~0ull;
        A.acc = ctr;
        A.overflow = reinterpret_cast<unsigned int *>(ctr + 5);
        A.heads = P.cheads.as<HeadS>();
        A.head_cap = SEG ? 0 : P.cheads.cap / sizeof(HeadS);
        A.items = P.citems.as<ItemS>();
        A.item_cap = SEG ? P.citems.cap / sizeof(ItemS) : 0;
        A.hcnt = ctr + nctr;
        A.slot_mix = P.d_slot_mix.as<uint64_t>();
        A.shard_lo = lo;
        A.shard_hi = hi;
        cudaEventRecord(t.a, s);
        A.out = base;
        A.out_S = baseS;
        A.out_B = baseB;
        A.cnt_out = ctr + 8;
        A.l = -1;
        root_k<<<(n_roots + 255) / 256, 256, 0, s>>>(A, P.f_roots.as<int32_t>(), P.f_roots.as<int32_t>() + n_roots,
                                                     n_roots);
        launches++;
        FSchedArgs sa;
        memset(&sa, 0, sizeof(sa));
        sa.c = fc;
        sa.ctr = ctr;
        sa.base = base;
        sa.baseS = baseS;
        sa.baseB = baseB;
        sa.capc = capc;
        sa.chunk = std::max<uint64_t>(1, capc / D);
        sa.chunk_div = D;
        sa.key_b = (uint32_t)key_b;
        sa.Lmax = Lmax;
        void *wargs[2] = {&A, &sa};
        TPG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(walk_k), dim3(wgrid), dim3(kFThreads), wargs,
                                           ts ? smem : 0, s));
        launches++;
        cudaEventRecord(t.b, s);
        TPG_CK(cudaGetLastError());
        TPG_CK(cudaMemcpyAsync(h.data(), ctr, (nctr + 8) * 8, cudaMemcpyDeviceToHost, s));
        FChunk hc;
        TPG_CK(cudaMemcpyAsync(&hc, fc, sizeof(FChunk), cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        const unsigned ovf = (unsigned)h[5];
        const uint64_t used = h[nctr + (SEG ? 1 : 0)];
        if (ovf & 1u) {
            set_error("frontier chunk overflow (internal)");
            return TPGEN_ERR_INTERNAL;
        }
        if (ovf & 2u) {  // head / item buffer: room for all of them, rerun
            ev_hwm = std::max<uint64_t>(ev_hwm, used);
            TPG_TRY(evb.ensure((used + used / 4 + 256ull * 4096) * ev_es, s));
            continue;
        }
        float m = 0;
        cudaEventElapsedTime(&m, t.a, t.b);
        ms += m;
        ev_hwm = std::max<uint64_t>(ev_hwm, used);
        recs += hc.recs;
        for (int q = 0; q < 5; q++) out[q] = h[q];
        *ev_slots = used;
        return TPGEN_OK;
    }
    set_error("frontier pass could not be sized");
    return TPGEN_ERR_OUT_OF_MEMORY;
}

// The frontier engine on graphs whose arcs leave SCCs (COUNT_HASH): the segment phase and the
// prime-path phase as frontier passes (heads, items), then count_post -- the
// completion DP, the cross prime paths, the stitch hash -- shared with the count-mode DFS.
template <class T>
static tpgen_status run_frontier_seg(PlanImpl &P, const tpgen_options &o, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: frontier engine (segment events)");
    const double t0 = now_ms();
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    const HostPlan &H = P.hp;
    cudaStream_t s = (cudaStream_t)o.stream;
    int32_t lo = 0, hi = H.n;
    shard_range(H, o.shard_rank, o.shard_count, lo, hi);
    if (o.start_hi > o.start_lo) {
        lo = std::max(0, o.start_lo);
        hi = std::min(H.n, o.start_hi);
    }
    st.shard_lo = lo;
    st.shard_hi = hi;
    st.n_scc = H.n_scc;
    st.n_scc_nontrivial = H.n_nontrivial;
    st.max_scc = H.max_scc;
    st.ms_plan = P.ms_plan;
    P.overflow = false;
    P.tp_unreachable = false;
    const int W = H.W;
    if (!P.f_tab_ok) {
        std::vector<FSlot<T>> tab(std::max(H.n, 1), FSlot<T>{0, 0, 0, 0});
        for (int32_t i = 0; i < H.n; i++)
            tab[i] = FSlot<T>{(T)H.sin[(size_t)i * W], (T)H.pin[(size_t)i * W], H.slot_gid[i], H.slot_flags[i]};
        TPG_TRY(upload(P.f_tab, tab, s));
        P.f_tab_ok = true;
    }
    // roots (slots, then slot bases): segment phase every SCC entry, prime-path phase the range's others
    std::vector<int32_t> rs, rp, vs, vp;
    for (int32_t v = 0; v < H.n; v++) {
        const int32_t slot = H.v_slot[v];
        const bool entry = (H.slot_flags[slot] & F_ENTRY) != 0;
        if (entry) {
            rs.push_back(slot);
            vs.push_back(H.scc_vbase[H.comp[v]]);
        } else if (v >= lo && v < hi) {
            rp.push_back(slot);
            vp.push_back(H.scc_vbase[H.comp[v]]);
        }
    }
    rs.insert(rs.end(), vs.begin(), vs.end());
    rp.insert(rp.end(), vp.begin(), vp.end());
    const size_t agg_n = 2 * (size_t)H.n + 2 * (size_t)H.n_pairs + 1;
    TPG_TRY(P.ctr.ensure(32 * 8, s));
    TPG_TRY(P.agg.ensure(agg_n * 8, s));
    TPG_CK(cudaMemsetAsync(P.agg.p, 0, agg_n * 8, s));
    const DevGraph G = dev_graph(P, lo, hi);
    Timer tall, tst;
    cudaEventRecord(tall.a, s);
    const bool hash = o.compute_digest != 0;
    int64_t launches = 0;
    uint64_t recs = 0;
    double ms_seg = 0, ms_pp = 0;
    unsigned long long cseg[8] = {0, 0, 0, 0, 0, 0, 0, 0}, cpp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    TPG_TRY((frontier_pass<T, true>(P, o, s, lo, hi, rs, hash, cseg, &cseg[7], ms_seg, launches, recs)));
    TPG_TRY((frontier_pass<T, false>(P, o, s, lo, hi, rp, hash, cpp, &cpp[5], ms_pp, launches, recs)));
    if (!hash) cseg[3] = cseg[4] = cpp[3] = cpp[4] = 0;
    st.n_units = (int64_t)recs;
    st.ms_dominant = ms_pp;
    st.ext_dominant = (int64_t)cpp[2];
    return count_post(P, o, G, s, !rs.empty(), cseg, cpp, 0, st, launches, tall, tst, ms_seg + ms_pp, t0, stp);
}

// TPGEN_ENGINE_ALG3 (alg3.cuh): the paper's vertex-centric self-stabilizing
// algorithm (Alg. 1-4) as a comparison engine: one cooperative launch, one CTA per vertex.
template <int W>
static tpgen_status run_alg3(PlanImpl &P, const tpgen_options &o, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: Alg. 3 engine");
    const double t0 = now_ms();
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    const HostPlan &H = P.hp;
    const int32_t n = H.n;
    cudaStream_t s = (cudaStream_t)o.stream;
    st.n_scc = H.n_scc;
    st.n_scc_nontrivial = H.n_nontrivial;
    st.max_scc = H.max_scc;
    st.ms_plan = P.ms_plan;
    st.shard_lo = 0;
    st.shard_hi = n;
    if (n == 0) {
        if (stp) *stp = st;
        return TPGEN_OK;
    }
    // host tables: successor / predecessor CSR (global ids), arc map, predecessor sets, B(v)
    std::vector<int64_t> aux64;
    const size_t n1 = (size_t)n + 1, m = (size_t)H.m;
    std::vector<int32_t> pidx(m);
    for (int32_t v = 0; v < n; v++)
        for (int64_t k = H.po[v]; k < H.po[v + 1]; k++) {
            const int32_t u = H.pt[k];
            int64_t e = H.so[u];
            while (e < H.so[u + 1] && H.st[e] != v) e++;
            pidx[k] = (int32_t)e;
        }
    std::vector<uint64_t> pinm((size_t)n * W, 0), back((size_t)n * W, 0);
    for (int32_t v = 0; v < n; v++)
        for (int64_t k = H.po[v]; k < H.po[v + 1]; k++) pinm[(size_t)v * W + (H.pt[k] >> 6)] |= 1ull << (H.pt[k] & 63);
    for (int32_t v = 0; v < n; v++) {  // B(v): backward BFS
        uint64_t *b = &back[(size_t)v * W];
        std::vector<int32_t> q{v};
        b[v >> 6] |= 1ull << (v & 63);
        for (size_t i = 0; i < q.size(); i++)
            for (int64_t k = H.po[q[i]]; k < H.po[q[i] + 1]; k++) {
                const int32_t x = H.pt[k];
                if (!((b[x >> 6] >> (x & 63)) & 1ull)) {
                    b[x >> 6] |= 1ull << (x & 63);
                    q.push_back(x);
                }
            }
    }
    // one device block: po, so (int64) | pt, sv, pidx (int32) | pinm, back (u64) | count, consumed, cursor, part
    const size_t off_so = n1 * 8, off_pt = off_so + n1 * 8, off_sv = off_pt + std::max<size_t>(m, 1) * 4,
                 off_pidx = off_sv + std::max<size_t>(m, 1) * 4;
    const size_t off_pinm = (off_pidx + std::max<size_t>(m, 1) * 4 + 7) / 8 * 8, off_back = off_pinm + (size_t)n * W * 8,
                 off_cnt = off_back + (size_t)n * W * 8, off_cons = off_cnt + (size_t)n * 8,
                 off_cur = off_cons + (size_t)n * 8, off_part = off_cur + std::max<size_t>(m, 1) * 8,
                 aux_b = off_part + (size_t)n * 64;
    std::vector<uint8_t> hb(aux_b, 0);
    memcpy(hb.data(), H.po.data(), n1 * 8);
    memcpy(hb.data() + off_so, H.so.data(), n1 * 8);
    if (m) {
        memcpy(hb.data() + off_pt, H.pt.data(), m * 4);
        memcpy(hb.data() + off_sv, H.st.data(), m * 4);
        memcpy(hb.data() + off_pidx, pidx.data(), m * 4);
    }
    memcpy(hb.data() + off_pinm, pinm.data(), (size_t)n * W * 8);
    memcpy(hb.data() + off_back, back.data(), (size_t)n * W * 8);
    TPG_TRY(P.a3_aux.ensure(aux_b, s));
    uint8_t *ad = P.a3_aux.as<uint8_t>();
    TPG_CK(cudaMemcpyAsync(ad, hb.data(), aux_b, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaStreamSynchronize(s));  // (hb is pageable and goes out of scope)
    // list capacity: from the plan's extension estimate (every simple path of an SCC-only graph),
    // doubled on overflow within the device-memory budget
    const size_t rec_b = 8 * W + 8 + 4 + 1;
    double est = 0;
    for (int32_t v = 0; v < n; v++) est += H.cost[v];
    unsigned long long cap = std::max<unsigned long long>(4096, (unsigned long long)(1.25 * est / n));
    cap = std::max<unsigned long long>(cap, P.a3_cap_hwm);  // (a capacity that fitted an earlier call of this plan)
    if (const char *ev = getenv("TPGEN_ALG3_CAP")) cap = std::max<unsigned long long>(16, strtoull(ev, nullptr, 10));
    if (getenv("TPGEN_ALG3_CAP")) P.a3_cap_hwm = 0;  // (the test hook starts small every call)
    int dev_sms = P.num_sms;
    if (n > dev_sms) {
        set_error("the Alg. 3 engine runs one co-resident CTA per vertex: at most one vertex per SM");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    Timer t;
    float ms = 0;
    std::vector<unsigned long long> part((size_t)n * 8);
    int64_t launches = 0;
    for (int attempt = 0;; attempt++) {
        size_t fr = 0, tot = 0;
        TPG_CK(cudaMemGetInfo(&fr, &tot));
        if ((double)cap * n * rec_b > 0.85 * (double)(fr + P.a3_lists.cap)) {
            set_error("Alg. 3 path lists exceed the device memory (every simple path is held at once, P:330)");
            return TPGEN_ERR_OUT_OF_MEMORY;
        }
        const size_t nt = (size_t)n * cap;
        TPG_TRY(P.a3_lists.ensure_exact(nt * rec_b, s));
        uint8_t *L = P.a3_lists.as<uint8_t>();
        A3Args a;
        a.n = n;
        a.cap = cap;
        a.po = reinterpret_cast<const int64_t *>(ad);
        a.so = reinterpret_cast<const int64_t *>(ad + off_so);
        a.pt = reinterpret_cast<const int32_t *>(ad + off_pt);
        a.sv = reinterpret_cast<const int32_t *>(ad + off_sv);
        a.pidx = reinterpret_cast<const int32_t *>(ad + off_pidx);
        a.vmix = P.d_vmix.as<uint64_t>();
        a.pinm = reinterpret_cast<const uint64_t *>(ad + off_pinm);
        a.back = reinterpret_cast<const uint64_t *>(ad + off_back);
        a.mask = reinterpret_cast<uint64_t *>(L);
        a.S = reinterpret_cast<uint64_t *>(L + nt * 8 * W);
        a.meta = reinterpret_cast<uint32_t *>(L + nt * (8 * W + 8));
        a.ext = L + nt * (8 * W + 12);
        a.count = reinterpret_cast<unsigned long long *>(ad + off_cnt);
        a.consumed = reinterpret_cast<unsigned long long *>(ad + off_cons);
        a.cursor = reinterpret_cast<unsigned long long *>(ad + off_cur);
        a.part = reinterpret_cast<unsigned long long *>(ad + off_part);
        TPG_CK(cudaMemsetAsync(ad + off_cnt, 0, aux_b - off_cnt, s));
        cudaEventRecord(t.a, s);
        void *args[1] = {&a};
        TPG_CK(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(&alg3_kernel<W>), dim3(n), dim3(kA3Threads), args, 0,
                                           s));
        launches++;
        cudaEventRecord(t.b, s);
        TPG_CK(cudaMemcpyAsync(part.data(), ad + off_part, (size_t)n * 64, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        cudaEventElapsedTime(&ms, t.a, t.b);
        bool ovf = false;
        unsigned long long longest = 0;
        for (int32_t v = 0; v < n; v++) {
            ovf |= part[(size_t)v * 8 + 5] != 0;
            longest = std::max<unsigned long long>(longest, part[(size_t)v * 8 + 4]);
        }
        if (!ovf) {
            P.a3_cap_hwm = std::max<unsigned long long>(P.a3_cap_hwm, longest + longest / 8);
            break;
        }
        st.n_count_rounds = attempt + 1;
        cap *= 2;
    }
    unsigned long long pp = 0, vert = 0, ha = 0, hbb = 0, recs = 0;
    for (int32_t v = 0; v < n; v++) {
        pp += part[(size_t)v * 8 + 0];
        vert += part[(size_t)v * 8 + 1];
        ha += part[(size_t)v * 8 + 2];
        hbb += part[(size_t)v * 8 + 3];
        recs += part[(size_t)v * 8 + 4];
    }
    st.n_paths = (int64_t)pp;
    st.total_vertices = (int64_t)vert;
    st.n_extensions = (int64_t)(recs - (unsigned long long)n);  // every record but the n initial <v> is one ExtendPath
    if (o.compute_digest) {
        st.hash_lo = ha;
        st.hash_hi = hbb;
    }
    st.n_units = (int64_t)recs;
    st.ms_device = ms;
    st.ms_count = ms;
    st.ms_dominant = ms;
    st.ext_dominant = st.n_extensions;
    st.gpu_launches = launches;
    st.ms_total = now_ms() - t0;
    if ((o.max_paths > 0 && st.n_paths > o.max_paths) || (o.max_extensions > 0 && st.n_extensions > o.max_extensions)) {
        set_error("result exceeds max_paths / max_extensions");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    if (stp) *stp = st;
    return TPGEN_OK;
}

tpgen_status run_prime_paths(PlanImpl &P, const tpgen_options &o, tpgen_paths *out, tpgen_stats *st) {
    if (o.engine == TPGEN_ENGINE_ALG3) {
        memset(out, 0, sizeof(*out));
        if (P.hp.n > 128) {
            set_error("the Alg. 3 engine needs graphs of <= 128 vertices (one CTA and one mask bit per vertex)");
            return TPGEN_ERR_INVALID_ARGUMENT;
        }
        if (P.hp.n <= 64) return run_alg3<1>(P, o, st);
        return run_alg3<2>(P, o, st);
    }
    if (o.engine == TPGEN_ENGINE_FRONTIER) {
        memset(out, 0, sizeof(*out));
        if (P.any_exit && P.hp.max_scc <= 64 && P.hp.n < (1 << 21)) {  // arcs leave SCCs: heads and items
            if (P.hp.max_scc <= 32) return run_frontier_seg<uint32_t>(P, o, st);
            return run_frontier_seg<uint64_t>(P, o, st);
        }
        if (P.hp.max_scc <= 32) return run_frontier<uint32_t>(P, o, st);
        return run_frontier<uint64_t>(P, o, st);
    }
    if (o.output_mode == TPGEN_OUT_COUNT_HASH && P.hp.max_scc <= 64 && P.hp.n < (1 << 21) && !getenv("TPGEN_NO_CNT")) {
        memset(out, 0, sizeof(*out));  // count modes
        if (P.hp.max_scc <= 32) return run_count<uint32_t>(P, o, st);
        return run_count<uint64_t>(P, o, st);
    }
    if (P.hp.max_scc <= 32) return run_pp<uint32_t>(P, o, out, st);
    switch (P.hp.W) {
        case 1: return run_pp<uint64_t>(P, o, out, st);
        case 2: return run_pp<Mask<2>>(P, o, out, st);
        case 4: return run_pp<Mask<4>>(P, o, out, st);
    }
    set_error("bad mask width");
    return TPGEN_ERR_INTERNAL;
}

// ------------------------------------------------------------ test paths
// Device copies of the test-path walk tables (R15): the host builds the two walk trees
// (build_tp_tables), tp_flat_kernel expands them into flat per-vertex walks.
struct TpDev {
    int64_t *pre_off, *suf_off;
    int32_t *pre_len, *suf_len, *parent, *next, *pre_flat, *suf_flat;
};
static tpgen_status tp_device_tables(PlanImpl &P, const TpTables &T, cudaStream_t s, int64_t &launches, TpDev &D) {
    const HostPlan &H = P.hp;
    const size_t nn = std::max<int32_t>(H.n, 1);
    const size_t bytes = nn * 8 * 2 + nn * 4 * 4 + (size_t)(T.pre_total + T.suf_total + 2) * 4 + 64;
    TPG_TRY(P.tp_tabs.ensure(bytes, s));
    char *b = (char *)P.tp_tabs.p;
    D.pre_off = (int64_t *)b;
    D.suf_off = D.pre_off + nn;
    D.pre_len = (int32_t *)(D.suf_off + nn);
    D.suf_len = D.pre_len + nn;
    D.parent = D.suf_len + nn;
    D.next = D.parent + nn;
    D.pre_flat = D.next + nn;
    D.suf_flat = D.pre_flat + T.pre_total + 1;
    TPG_CK(cudaMemcpyAsync(D.pre_off, T.pre_off.data(), H.n * 8, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaMemcpyAsync(D.suf_off, T.suf_off.data(), H.n * 8, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaMemcpyAsync(D.pre_len, T.pre_len.data(), H.n * 4, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaMemcpyAsync(D.suf_len, T.suf_len.data(), H.n * 4, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaMemcpyAsync(D.parent, T.parent.data(), H.n * 4, cudaMemcpyHostToDevice, s));
    TPG_CK(cudaMemcpyAsync(D.next, T.next.data(), H.n * 4, cudaMemcpyHostToDevice, s));
    if (H.n > 0) {
        tp_flat_kernel<<<grid_for(H.n, 128, P.num_sms * 8), 128, 0, s>>>(H.n, D.parent, D.next, D.pre_off, D.pre_len,
                                                                          D.suf_off, D.suf_len, D.pre_flat, D.suf_flat);
        launches++;
    }
    return TPGEN_OK;
}

// COUNT_HASH test paths (tpgen_test_paths with output_mode COUNT_HASH): the count, vertices and
// R20 digest of every prime path's test path, nothing written.  Without a prime-path list on a
// graph the count modes take (SCCs <= 64 vertices), the count-mode enumeration hashes each test
// path the moment its prime path is found (the TpTerm tables); otherwise tp_hash_list_kernel
// hashes the test paths of the given (or computed) list.
static tpgen_status run_test_paths_count(PlanImpl &P, const tpgen_paths *pp_in, int32_t entry, int32_t exit,
                                         const tpgen_options &o, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: test paths (count mode)");
    const double t0 = now_ms();
    const HostPlan &H = P.hp;
    cudaStream_t s = (cudaStream_t)o.stream;
    int64_t launches = 0;
    TpTables T;
    build_tp_tables(H, entry, exit, T);
    TpDev D;
    TPG_TRY(tp_device_tables(P, T, s, launches, D));
    TPG_TRY(P.tp_terms.ensure((size_t)std::max<int32_t>(H.n, 1) * sizeof(TpTerm), s));
    if (H.n > 0) {
        tp_terms_kernel<<<grid_for(H.n, 128, P.num_sms * 8), 128, 0, s>>>(
            H.n, P.d_slot_gid.as<int32_t>(), P.d_vmix.as<uint64_t>(), D.pre_off, D.pre_len, D.suf_off, D.suf_len,
            D.pre_flat, D.suf_flat, P.tp_terms.as<TpTerm>());
        launches++;
    }
    tpgen_options oc = o;
    oc.output_mode = TPGEN_OUT_COUNT_HASH;
    oc.compute_digest = 1;
    if (!pp_in && H.max_scc <= 64 && H.n < (1 << 21) && !getenv("TPGEN_NO_CNT")) {
        P.cur_tp = P.tp_terms.as<TpTerm>();
        tpgen_status r = (H.max_scc <= 32) ? run_count<uint32_t>(P, oc, stp) : run_count<uint64_t>(P, oc, stp);
        P.cur_tp = nullptr;
        if (r == TPGEN_OK && stp) {
            stp->gpu_launches += launches;
            stp->ms_total = now_ms() - t0;
        }
        return r;
    }
    // the prime paths as a list (given, or computed), then one thread per path
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    tpgen_paths own;
    memset(&own, 0, sizeof(own));
    const tpgen_paths *pp = pp_in;
    if (!pp) {
        tpgen_options o2 = o;
        o2.output_mode = TPGEN_OUT_MATERIALIZE;
        o2.output_on_device = 1;
        o2.device_alloc = nullptr;
        o2.device_free = nullptr;
        o2.host_out = nullptr;
        TPG_TRY(run_prime_paths(P, o2, &own, &st));
        pp = &own;
    }
    struct Guard {
        tpgen_paths *p;
        ~Guard() { free_paths(p); }
    } g{&own};
    const int64_t n = pp->n_paths;
    const int64_t *d_ppo = pp->offsets;
    const int32_t *d_ppv = pp->vertices;
    DevBuf tmp_o, tmp_v;
    struct BufGuard {
        DevBuf *a, *b;
        cudaStream_t s;
        ~BufGuard() {
            a->release(s);
            b->release(s);
        }
    } bg{&tmp_o, &tmp_v, s};
    if (n > 0 && !pp->on_device) {
        const int64_t nv = pp->offsets[n];
        TPG_TRY(tmp_o.ensure((size_t)(n + 1) * 8, s));
        TPG_TRY(tmp_v.ensure((size_t)std::max<int64_t>(nv, 1) * 4, s));
        TPG_CK(cudaMemcpyAsync(tmp_o.p, pp->offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        if (nv) TPG_CK(cudaMemcpyAsync(tmp_v.p, pp->vertices, (size_t)nv * 4, cudaMemcpyHostToDevice, s));
        d_ppo = tmp_o.as<int64_t>();
        d_ppv = tmp_v.as<int32_t>();
    }
    TPG_TRY(P.ctr.ensure(32 * 8, s));
    unsigned long long *acc = P.ctr.as<unsigned long long>() + 24;
    TPG_CK(cudaMemsetAsync(acc, 0, 32, s));
    if (n > 0) {
        tp_hash_list_kernel<<<grid_for(n, 256, P.num_sms * 8), 256, 0, s>>>(
            d_ppo, d_ppv, n, P.d_v_slot.as<int32_t>(), P.d_vmix.as<uint64_t>(), P.tp_terms.as<TpTerm>(), acc,
            reinterpret_cast<unsigned int *>(acc + 3));
        launches++;
    }
    unsigned long long h[4];
    TPG_CK(cudaMemcpyAsync(h, acc, 32, cudaMemcpyDeviceToHost, s));
    TPG_CK(cudaStreamSynchronize(s));
    if (h[3]) {
        set_error("a prime path's first vertex is unreachable from entry or its last cannot reach exit");
        return TPGEN_ERR_UNREACHABLE;
    }
    st.n_paths = n;
    st.total_vertices = (int64_t)h[2];
    st.hash_lo = h[0];
    st.hash_hi = h[1];
    st.gpu_launches += launches;
    st.ms_total = now_ms() - t0;
    if (stp) *stp = st;
    return TPGEN_OK;
}

tpgen_status run_test_paths(PlanImpl &P, const tpgen_paths *pp_in, int32_t entry, int32_t exit,
                            const tpgen_options &o, tpgen_paths *out, tpgen_stats *stp) {
    NvtxRange nvtx_range("tpgen: test paths");
    const double t0 = now_ms();
    memset(out, 0, sizeof(*out));
    if (o.output_mode == TPGEN_OUT_COUNT_HASH) {
        if (o.tp_mode != TPGEN_TP_PER_PP) {
            set_error("COUNT_HASH test paths are the per-prime-path ones (tp_mode TPGEN_TP_PER_PP)");
            return TPGEN_ERR_INVALID_ARGUMENT;
        }
        return run_test_paths_count(P, pp_in, entry, exit, o, stp);
    }
    const HostPlan &H = P.hp;
    cudaStream_t s = (cudaStream_t)o.stream;
    tpgen_stats st;
    memset(&st, 0, sizeof(st));
    st.unit_lo = st.unit_hi = -1;
    tpgen_paths own;
    memset(&own, 0, sizeof(own));
    const tpgen_paths *pp = pp_in;
    if (!pp) {
        tpgen_options o2 = o;
        o2.output_on_device = 1;
        o2.device_alloc = nullptr;
        o2.device_free = nullptr;
        o2.host_out = nullptr;
        TPG_TRY(run_prime_paths(P, o2, &own, &st));
        pp = &own;
    }
    struct Guard {
        tpgen_paths *p;
        ~Guard() { free_paths(p); }
    } g{&own};
    const int64_t n = pp->n_paths;
    // PP arrays on device
    const int64_t *d_ppo = pp->offsets;
    const int32_t *d_ppv = pp->vertices;
    DevBuf tmp_o, tmp_v;
    struct BufGuard {
        DevBuf *a, *b;
        cudaStream_t s;
        ~BufGuard() {
            a->release(s);
            b->release(s);
        }
    } bg{&tmp_o, &tmp_v, s};
    if (n > 0 && !pp->on_device) {
        int64_t nv = pp->offsets[n];
        TPG_TRY(tmp_o.ensure((size_t)(n + 1) * 8, s));
        TPG_TRY(tmp_v.ensure((size_t)std::max<int64_t>(nv, 1) * 4, s));
        TPG_CK(cudaMemcpyAsync(tmp_o.p, pp->offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        if (nv) TPG_CK(cudaMemcpyAsync(tmp_v.p, pp->vertices, (size_t)nv * 4, cudaMemcpyHostToDevice, s));
        d_ppo = tmp_o.as<int64_t>();
        d_ppv = tmp_v.as<int32_t>();
    }
    const bool hdbg = getenv("TPGEN_DEBUG") != nullptr;
    double hprev = now_ms();
    auto HT = [&](const char *what) {
        if (!hdbg) return;
        cudaStreamSynchronize(s);
        const double t = now_ms();
        fprintf(stderr, "[tpgen tp host] %-24s %8.3f ms\n", what, t - hprev);
        hprev = t;
    };
    HT("prime paths ready");
    TpTables T;
    build_tp_tables(H, entry, exit, T);
    HT("host tables");
    if (o.tp_mode == TPGEN_TP_GREEDY) {  // greedy cover: sequential, on the host (tpcover.cpp)
        std::vector<int64_t> hoff;
        std::vector<int32_t> hvert;
        const int64_t *po = pp->offsets;
        const int32_t *pv = pp->vertices;
        if (n > 0 && pp->on_device) {
            hoff.resize((size_t)n + 1);
            TPG_CK(cudaMemcpyAsync(hoff.data(), pp->offsets, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost, s));
            TPG_CK(cudaStreamSynchronize(s));
            hvert.resize((size_t)std::max<int64_t>(hoff[(size_t)n], 1));
            TPG_CK(cudaMemcpyAsync(hvert.data(), pp->vertices, (size_t)hoff[(size_t)n] * 4, cudaMemcpyDeviceToHost, s));
            TPG_CK(cudaStreamSynchronize(s));
            po = hoff.data();
            pv = hvert.data();
        }
        std::vector<int64_t> toff;
        std::vector<int32_t> tvert;
        if (!greedy_cover(H, T, entry, exit, po, pv, n, toff, tvert)) {
            set_error("a prime path's first vertex is unreachable from entry or its last cannot reach exit");
            return TPGEN_ERR_UNREACHABLE;
        }
        const int64_t ntp = (int64_t)toff.size() - 1, nv = (int64_t)tvert.size();
        OutOwner *ow = new OutOwner();
        ow->device = P.device;
        std::unique_ptr<OutOwner> ow_guard(ow);
        void *d_off = nullptr, *d_vert = nullptr;
        TPG_TRY(out_alloc_pair(o, ow, (size_t)(ntp + 1) * 8, (size_t)nv * 4, &d_off, &d_vert, s));
        TPG_CK(cudaMemcpyAsync(d_off, toff.data(), (size_t)(ntp + 1) * 8, cudaMemcpyHostToDevice, s));
        if (nv) TPG_CK(cudaMemcpyAsync(d_vert, tvert.data(), (size_t)nv * 4, cudaMemcpyHostToDevice, s));
        TPG_CK(cudaStreamSynchronize(s));
        ow_guard.release();
        TPG_TRY(finish_output(o, ow, ntp, nv, (int64_t *)d_off, (int32_t *)d_vert, s, out));
        st.n_paths = ntp;
        st.total_vertices = nv;
        st.ms_total = now_ms() - t0;
        if (stp) *stp = st;
        return TPGEN_OK;
    }
    TpDev D;
    {
        int64_t l0 = 0;
        TPG_TRY(tp_device_tables(P, T, s, l0, D));
        st.gpu_launches += l0;
    }
    int64_t *d_pre_off = D.pre_off, *d_suf_off = D.suf_off;
    int32_t *d_pre_len = D.pre_len, *d_suf_len = D.suf_len, *d_pre_flat = D.pre_flat, *d_suf_flat = D.suf_flat;

    DevBuf lenb;
    struct LGuard {
        DevBuf *a;
        cudaStream_t s;
        ~LGuard() { a->release(s); }
    } lg{&lenb, s};
    TPG_TRY(lenb.ensure((size_t)std::max<int64_t>(n, 1) * 8 + 16, s));
    unsigned int *d_unr = (unsigned int *)(lenb.as<char>() + (size_t)std::max<int64_t>(n, 1) * 8);
    TPG_CK(cudaMemsetAsync(d_unr, 0, 4, s));
    TpArgs A;
    A.pp_off = d_ppo;
    A.pp_vert = d_ppv;
    A.n = n;
    A.pre_off = d_pre_off;
    A.suf_off = d_suf_off;
    A.pre_len = d_pre_len;
    A.suf_len = d_suf_len;
    A.pre_flat = d_pre_flat;
    A.suf_flat = d_suf_flat;
    A.tp_len = lenb.as<uint64_t>();
    A.unreachable = d_unr;
    int64_t launches = st.gpu_launches;
    uint64_t total = 0;
    if (n > 0) {
        tp_len_kernel<<<grid_for(n, 256, 4096), 256, 0, s>>>(A);
        launches++;
        uint64_t *arr[1] = {A.tp_len};
        TPG_TRY(scan_multi(P, arr, 1, n, &total, s, launches));
        unsigned int unr = 0;
        TPG_CK(cudaMemcpyAsync(&unr, d_unr, 4, cudaMemcpyDeviceToHost, s));
        TPG_CK(cudaStreamSynchronize(s));
        if (unr) {
            set_error("a prime path's first vertex is unreachable from entry or its last cannot reach exit");
            return TPGEN_ERR_UNREACHABLE;
        }
    }
    HT("lengths + scan");
    if (o.tp_mode == TPGEN_TP_UNIQUE) {  // K7: aligned TPs into scratch, then sort + unique into the output
        DevBuf a_off, a_vert, ws;
        struct UGuard {
            DevBuf *a, *b, *c;
            cudaStream_t s;
            ~UGuard() {
                a->release(s);
                b->release(s);
                c->release(s);
            }
        } ug{&a_off, &a_vert, &ws, s};
        TPG_TRY(a_off.ensure((size_t)(n + 1) * 8, s));
        TPG_TRY(a_vert.ensure((size_t)std::max<uint64_t>(total, 1) * 4, s));
        A.tp_off = a_off.as<int64_t>();
        A.tp_vert = a_vert.as<int32_t>();
        if (n > 0) {
            tp_write_kernel<<<grid_for(n * 32, 256, P.num_sms * 8), 256, 0, s>>>(A);
            launches++;
        }
        set_last_offset_kernel<<<1, 1, 0, s>>>(A.tp_off, n, (int64_t)total);
        launches++;
        // indices sorted by their TP (device merge sort, lexicographic comparator), equal neighbours dropped
        const size_t nn = (size_t)std::max<int64_t>(n, 1);
        size_t tmp_b = 0;
        SeqLess cmp{A.tp_off, A.tp_vert};
        TPG_CK(cub::DeviceMergeSort::StableSortKeys(nullptr, tmp_b, (int64_t *)nullptr, n, cmp, s));
        const size_t o_idx = 0, o_keep = nn * 8, o_len = o_keep + nn * 8, o_kept = o_len + nn * 8,
                     o_tmp = (o_kept + nn + 255) / 256 * 256;
        TPG_TRY(ws.ensure(o_tmp + tmp_b + 16, s));
        int64_t *idx = reinterpret_cast<int64_t *>(ws.as<char>() + o_idx);
        uint64_t *keep = reinterpret_cast<uint64_t *>(ws.as<char>() + o_keep);
        uint64_t *len = reinterpret_cast<uint64_t *>(ws.as<char>() + o_len);
        uint8_t *kept = reinterpret_cast<uint8_t *>(ws.as<char>() + o_kept);
        uint64_t tot2[2] = {0, 0};
        if (n > 0) {
            iota_kernel<<<grid_for(n, 256, 4096), 256, 0, s>>>(idx, n);
            launches++;
            TPG_CK(cub::DeviceMergeSort::StableSortKeys(ws.as<char>() + o_tmp, tmp_b, idx, n, cmp, s));
            launches += 3;  // (CUB's merge sort: block sort + merge passes, counted as one group)
            tp_unique_mark_kernel<<<grid_for(n, 256, 4096), 256, 0, s>>>(idx, n, A.tp_off, A.tp_vert, keep, len, kept);
            launches++;
            uint64_t *arr[2] = {keep, len};
            TPG_TRY(scan_multi(P, arr, 2, n, tot2, s, launches));
        }
        HT("sort + unique");
        const int64_t nu = (int64_t)tot2[0], nvu = (int64_t)tot2[1];
        OutOwner *ow = new OutOwner();
        ow->device = P.device;
        std::unique_ptr<OutOwner> ow_guard(ow);
        void *d_off = nullptr, *d_vert = nullptr;
        TPG_TRY(out_alloc_pair(o, ow, (size_t)(nu + 1) * 8, (size_t)nvu * 4, &d_off, &d_vert, s));
        if (n > 0) {
            tp_unique_gather_kernel<<<grid_for(n * 32, 256, P.num_sms * 8), 256, 0, s>>>(
                idx, n, A.tp_off, A.tp_vert, keep, len, kept, (int64_t *)d_off, (int32_t *)d_vert);
            launches++;
        }
        set_last_offset_kernel<<<1, 1, 0, s>>>((int64_t *)d_off, nu, nvu);
        launches++;
        TPG_CK(cudaGetLastError());
        ow_guard.release();
        TPG_TRY(finish_output(o, ow, nu, nvu, (int64_t *)d_off, (int32_t *)d_vert, s, out));
        st.gpu_launches = launches;
        st.n_paths = nu;
        st.total_vertices = nvu;
        st.ms_total = now_ms() - t0;
        if (stp) *stp = st;
        return TPGEN_OK;
    }
    OutOwner *ow = new OutOwner();
    ow->device = P.device;
    std::unique_ptr<OutOwner> ow_guard(ow);
    void *d_off = nullptr, *d_vert = nullptr;
    TPG_TRY(out_alloc_pair(o, ow, (size_t)(n + 1) * 8, (size_t)total * 4, &d_off, &d_vert, s));
    HT("alloc");
    A.tp_off = (int64_t *)d_off;
    A.tp_vert = (int32_t *)d_vert;
    if (n > 0) {
        tp_write_kernel<<<grid_for(n * 32, 256, P.num_sms * 8), 256, 0, s>>>(A);
        launches++;
    }
    set_last_offset_kernel<<<1, 1, 0, s>>>((int64_t *)d_off, n, (int64_t)total);
    launches++;
    TPG_CK(cudaGetLastError());
    HT("write");
    ow_guard.release();
    TPG_TRY(finish_output(o, ow, n, (int64_t)total, (int64_t *)d_off, (int32_t *)d_vert, s, out));
    st.gpu_launches = launches;
    st.n_paths = n;                  // stats describe the returned test paths
    st.total_vertices = (int64_t)total;
    st.ms_total = now_ms() - t0;
    if (stp) *stp = st;
    return TPGEN_OK;
}

// Five-class report (R19): every prime path is
// complete / entry / exit / internal / transit by its end vertices and SCCs.
tpgen_status run_classify(PlanImpl &P, const tpgen_paths *pp, int32_t start, int32_t end, const tpgen_options &o,
                          int64_t counts[5]) {
    cudaStream_t s = (cudaStream_t)o.stream;
    const int64_t n = pp->n_paths;
    for (int c = 0; c < 5; c++) counts[c] = 0;
    if (n <= 0) return TPGEN_OK;
    const int64_t *d_off = pp->offsets;
    const int32_t *d_vert = pp->vertices;
    DevBuf tmp_o, tmp_v;
    struct BufGuard {
        DevBuf *a, *b;
        cudaStream_t s;
        ~BufGuard() {
            a->release(s);
            b->release(s);
        }
    } bg{&tmp_o, &tmp_v, s};
    if (!pp->on_device) {
        const int64_t nv = pp->offsets[n];
        TPG_TRY(tmp_o.ensure((size_t)(n + 1) * 8, s));
        TPG_TRY(tmp_v.ensure((size_t)std::max<int64_t>(nv, 1) * 4, s));
        TPG_CK(cudaMemcpyAsync(tmp_o.p, pp->offsets, (size_t)(n + 1) * 8, cudaMemcpyHostToDevice, s));
        if (nv) TPG_CK(cudaMemcpyAsync(tmp_v.p, pp->vertices, (size_t)nv * 4, cudaMemcpyHostToDevice, s));
        d_off = tmp_o.as<int64_t>();
        d_vert = tmp_v.as<int32_t>();
    }
    TPG_TRY(P.ctr.ensure(32 * 8, s));
    unsigned long long *acc = P.ctr.as<unsigned long long>() + 24;
    TPG_CK(cudaMemsetAsync(acc, 0, 5 * 8, s));
    classify_kernel<<<grid_for(n, 256, P.num_sms * 8), 256, 0, s>>>(d_off, d_vert, n, P.d_comp.as<int32_t>(), start,
                                                                     end, acc);
    TPG_CK(cudaGetLastError());
    unsigned long long h[5];
    TPG_CK(cudaMemcpyAsync(h, acc, 5 * 8, cudaMemcpyDeviceToHost, s));
    TPG_CK(cudaStreamSynchronize(s));
    for (int c = 0; c < 5; c++) counts[c] = (int64_t)h[c];
    return TPGEN_OK;
}

tpgen_status init_device(PlanImpl &P, const tpgen_options &o) {
    int dev = o.device;
    if (dev < 0) TPG_CK(cudaGetDevice(&dev));
    TPG_CK(cudaSetDevice(dev));
    P.device = dev;
    // keep freed pool memory cached: outputs and workspaces are recycled call after call
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    TPG_CK(cudaDeviceGetAttribute(&P.num_sms, cudaDevAttrMultiProcessorCount, dev));
    return TPGEN_OK;
}

}  // namespace tpg
