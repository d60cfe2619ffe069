// engine.h -- host-side engine interface of libtpgen (internal).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "internal.h"

namespace tpg {
struct TpTerm;
}

namespace tpg {

// Grow-only, stream-ordered device buffer.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    tpgen_status ensure(size_t bytes, cudaStream_t s);
    tpgen_status ensure_exact(size_t bytes, cudaStream_t s);  // no growth headroom (memory-budgeted buffers)
    void release(cudaStream_t s);
    template <class T>
    T *as() const {
        return reinterpret_cast<T *>(p);
    }
};

constexpr int kCnt = 6;

// A plan: the host plan plus its device tables and the reusable workspace.
struct PlanImpl {
    HostPlan hp;
    int device = 0;
    int num_sms = 148;
    bool dev_ok = false;
    double ms_plan = 0;
    // device tables
    DevBuf d_slots, d_slot_gid, d_out_gid, d_out_pos, d_scc_vbase, d_scc_out_base, d_scc_nout, d_scc_pair_base,
        d_slot_eidx, d_Wc, d_Wv, d_scc_gbase, d_comp, d_slot_mix, d_vmix, d_scc_exm, d_v_slot,
        d_slot_d2;  // count modes, SCCs of in-SCC out-degree <= 2: {t0 | t1 << 8 | exit << 16, mix} per slot
    bool d2_ok = false;  // every slot has at most 2 in-SCC successors and every SCC at most 64 vertices
    DevBuf cheads;           // count modes: HeadS records of the prime-path phase
    DevBuf citems, citems2;  // count modes: ItemS records of the segment phase (as written; grouped by entry)
    DevBuf icnt;             // count modes: items per entry vertex, their scan, the scatter cursors
    DevBuf tp_terms;         // count modes, test paths: TpTerm per slot
    int32_t cur_prune = 0;           // the running count-mode call prunes (tpgen_options.prune)
    const TpTerm *cur_tp = nullptr;  // the running count-mode call hashes test paths with these terms
    bool tp_unreachable = false;     // ... and found a path whose end vertices have no walk
    uint64_t chead_hwm = 0;  // most head slots any count-mode call of this plan reserved
    uint64_t citem_hwm = 0;  // most item slots any count-mode call of this plan reserved
    // DFS work queue (one slot per unit) and its per-unit results
    DevBuf qunits, qready, qcnt[kCnt], qext, qrfirst, qrcount, qchead, qgen, roots;
    DevBuf qparent, qnchild;  // donor / number of donated units, per unit
    DevBuf blk_first, blk_count, blk_next;  // donated blocks (one per donation)
    uint64_t qcap = 0;
    DevBuf chunks, agg, agg_bak;  // path-delta record pool (chunks of kChunkRecs words); SEG aggregates + backup
    uint64_t chunk_cap = 0;       // pool capacity in chunks
    uint64_t chunk_used = 0;      // chunks handed out so far in this call
    uint64_t chunk_hwm = 0;       // most chunks any call of this plan used (sizes the pool with headroom)
    uint64_t q_hwm = 0;           // most queue slots any call of this plan used
    int maxgen = 0;               // deepest split generation so far in this call
    uint32_t split_min = 32;      // steps between two donations of a unit
    uint32_t split_min_presplit = 1024;  // ... when the phase starts from pre-split roots (measured sweep, config 3)
    DevBuf dbgbuf, qctr, scan_b, scan_tot, ctr, heads, head_pool, items, item_pool, icum, ivcum, ibeg, iend, hcomp, offs, tp_tabs;
    DevBuf sscratch;  // cross-SCC range writer: per-warp level stacks
    DevBuf f_tab, f_roots, f_buf0, f_buf1, f_ctr;  // frontier engine: slot table, roots, ping-pong levels, counters
    DevBuf f_sched;                                // DFS-chunked frontier: the device chunk scheduler's state (FChunk)
    DevBuf a3_lists, a3_aux;                       // Alg. 3 comparison engine: per-vertex path lists, CSR / flags
    unsigned long long a3_cap_hwm = 0;             // Alg. 3: a list capacity that fitted (records per vertex)
    bool f_tab_ok = false;
    int32_t f_roots_lo = -1, f_roots_hi = -1;  // start range of the uploaded frontier roots
    uint64_t f_cap_hwm = 0;                        // frontier engine: most records any level of this plan held
    bool overflow = false;
    bool any_exit = true;
    // LEAN pre-split roots (host copy, device copy, their start gids and the extensions above the cut)
    std::vector<uint8_t> presplit_host;
    std::vector<int32_t> presplit_gid;
    DevBuf presplit_dev;
    int64_t presplit_n = 0;
    uint64_t presplit_ext = 0;
    int32_t presplit_lo = -1, presplit_hi = -1;
    int64_t presplit_key = -1;  // prefix-unit shard (rank << 32 | count) the cached pre-split belongs to; -1: none
    PrefixShard pfx;              // the last prefix-unit split computed (tpgen_options.shard_prefix) ...
    int64_t pfx_key = -1;         // ... and its (rank << 32 | count)
    bool presplit_active = false;
    DevBuf presplit_roots, rscan;  // pre-split root table (cached); root-scan scratch
    int64_t presplit_roots_n = -1, presplit_roots_tail = -1;  // the running PP phase's roots are the cached pre-split units  // some arc leaves its SCC (head / segment events possible; no LEAN DFS)
    ~PlanImpl();
    std::vector<DevBuf *> all_bufs();
};

tpgen_status init_device(PlanImpl &P, const tpgen_options &o);
tpgen_status plan_upload(PlanImpl &P, cudaStream_t s);
tpgen_status run_prime_paths(PlanImpl &P, const tpgen_options &o, tpgen_paths *out, tpgen_stats *st);
tpgen_status run_test_paths(PlanImpl &P, const tpgen_paths *pp, int32_t entry, int32_t exit, const tpgen_options &o,
                            tpgen_paths *out, tpgen_stats *st);
tpgen_status run_classify(PlanImpl &P, const tpgen_paths *pp, int32_t start, int32_t end, const tpgen_options &o,
                          int64_t counts[5]);
void free_paths(tpgen_paths *p);
const char *last_error();

// Frees the cached output blocks of device `dev` (tpgen_release_cache).
void release_output_cache(int dev);

}  // namespace tpg
