// internal.h -- structures shared by the host planner, the CUDA engine and the
// C-ABI layer of libtpgen.  Not part of the public ABI (see include/tpgen.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tpgen.h"

#if defined(__CUDACC__)
#define TPG_HD __host__ __device__
#define TPG_ALIGN(n) __align__(n)
#else
#define TPG_HD
#define TPG_ALIGN(n) alignas(n)
#endif

namespace tpg {

constexpr int kMaxW = 4;              // visited mask words per path (W in {1, 2, 4})
constexpr int kMaxScc = 64 * kMaxW;   // largest SCC this build enumerates

enum SlotFlags : int32_t { F_ENTRY = 1, F_EXIT = 2 };

// Head segment record: a cross-SCC block h (+) completions(x) reserved in the output.
struct TPG_ALIGN(16) HeadRec {
    uint64_t pp_off;   // first prime-path index of the block
    uint64_t v_off;    // first output vertex of the block
    uint64_t hv_off;   // head vertices in the head pool
    int32_t len;       // |h|
    int32_t x;         // global id of the successor outside h's SCC (an SCC entry)
};
static_assert(sizeof(HeadRec) == 32, "HeadRec layout");

// Segment item of an entry vertex's completion table: a tail segment (y < 0) or
// a transit segment followed by the arc to y (y = entry of a downstream SCC).
struct TPG_ALIGN(16) ItemRec {
    int64_t pool_off;  // vertices in the item pool
    int32_t len;
    int32_t y;         // -1 for a tail segment
    int32_t ent;       // global id of the entry vertex whose table holds the item
    int32_t pad;
};
static_assert(sizeof(ItemRec) == 24 || sizeof(ItemRec) == 32, "ItemRec layout");

// ------------------------------------------------------------------ host plan
struct HostPlan {
    int32_t n = 0;
    int64_t m = 0;
    std::vector<int64_t> so;    // sorted successor CSR
    std::vector<int32_t> st;
    std::vector<int64_t> po;    // predecessor CSR
    std::vector<int32_t> pt;
    std::vector<int32_t> comp;  // SCC id per vertex; ids in reverse topological order (sinks first)
    int32_t n_scc = 0, n_nontrivial = 0, max_scc = 0;
    std::vector<int32_t> scc_vbase, scc_size, scc_out_base, scc_nout, scc_nentries;
    std::vector<int64_t> scc_pair_base;
    int64_t n_pairs = 0;
    std::vector<int32_t> v_slot;     // vertex -> slot
    // Slots: the vertices of each SCC in SCC-local order (local ids ascend with
    // global ids, so lexicographic order on local ids == order on global ids).
    int32_t W = 1;                        // mask words: ceil(max_scc / 64) rounded to 1, 2, 4
    std::vector<uint64_t> sin, pin;       // [slot*W + word]: in-SCC successor / predecessor local bits
    std::vector<int32_t> slot_gid;        // global vertex id
    std::vector<int32_t> slot_out_off;    // first out-of-SCC arc (index into out_gid/out_pos)
    std::vector<int32_t> slot_out_cnt;    // number of out-of-SCC successors (ascending global id)
    std::vector<int32_t> slot_flags;      // F_ENTRY (Def. 4) | F_EXIT (Def. 5)
    std::vector<int32_t> slot_eidx;       // entry index inside its SCC, -1 if not an entry
    std::vector<int32_t> out_gid, out_pos;
    bool has_entries = false;        // some vertex is an SCC entry (segment phase needed)
    std::vector<double> cost;        // per-vertex work estimate (shard balancing)
};

// Validates the CSR and builds the plan.  Returns TPGEN_OK or an error (msg set).
tpgen_status build_plan(const int64_t *so, const int32_t *st, int32_t n, HostPlan &plan, std::string &msg,
                        bool enforce_limit = true);

// Start-vertex range [lo, hi) of a shard (contiguous, cost balanced).
void shard_range(const HostPlan &plan, int32_t rank, int32_t count, int32_t &lo, int32_t &hi);

// Prefix-unit shards ("Unit = (SCC, start vertex), or (start,
// depth-k prefix) for heavy starts"; tpgen_options.shard_prefix).  A unit is a
// node of a start vertex's path trie (the subtree under path[0..depth]) or the
// closing arc of one (a cyclic prime path); the list stays in canonical
// (preorder) order, so a contiguous range of units is a contiguous block of the
// canonical prime-path list.
struct PrefixUnit {
    uint64_t M;         // visited local bits of path[0..depth]
    int32_t scc, gid;   // component, global id of the start vertex
    uint8_t depth, closure;
    uint8_t path[32];   // local ids
};
struct PrefixShard {
    int64_t ulo = 0, uhi = 0, n_units = 0;  // this shard's unit range / units of the whole split
    int32_t lo = 0, hi = 0;                 // start vertices the range touches, [lo, hi)
    uint64_t ext = 0;  // extensions of the expanded interior trie nodes (depth >= 1) credited to the range
                       // (each to the shard holding its first descendant unit)
    std::vector<PrefixUnit> units;          // units [ulo, uhi)
};
// Graphs the split applies to: one mask word (SCCs <= 32 vertices) and no arc leaving an SCC
// (prime paths then never leave their SCC; the LEAN / pre-split DFS path).
bool prefix_shard_applies(const HostPlan &plan);
// Heavy units (Knuth estimate above total / (16 count)) are replaced by their children, round
// by round, until none is heavy; then contiguous unit ranges balanced by cost.  Deterministic:
// every rank computes the same split.
void prefix_shard(const HostPlan &plan, int32_t rank, int32_t count, PrefixShard &out);

// Completion-count DP over the component DAG:
//   W(x) = #tails(x) + sum_arcs cnt(x,e) W(y_e),  V(x) = vertices of all completions.
// Inputs are the per-entry tail aggregates and per-(entry, out-arc) transit
// aggregates of the segment phase.  Returns false on overflow (>= 2^62).
bool completion_dp(const HostPlan &plan, const std::vector<uint64_t> &tail_cnt, const std::vector<uint64_t> &tail_len,
                   const std::vector<uint64_t> &pair_cnt, const std::vector<uint64_t> &pair_len,
                   std::vector<uint64_t> &W, std::vector<uint64_t> &V);

// Test-path tables (R15): lexmin-shortest walks.
struct TpTables {
    std::vector<int64_t> pre_off, suf_off;  // per vertex: offset of its walk in the flat table, -1 if none
    std::vector<int32_t> pre_len, suf_len;  // walk lengths in vertices, -1 if none
    std::vector<int32_t> parent, next;      // BFS-tree parent (prefix walks), greedy next hop (suffix walks)
    int64_t pre_total = 0, suf_total = 0;   // sizes of the flat tables (built on the device)
};
void build_tp_tables(const HostPlan &plan, int32_t entry, int32_t exit, TpTables &tp);
// Greedy test-path cover (tpcover.cpp) of a canonical prime-path list in host memory;
// false if a prime path's end vertices cannot be reached from entry / reach exit.
bool greedy_cover(const HostPlan &H, const TpTables &T, int32_t entry, int32_t exit, const int64_t *off,
                  const int32_t *vert, int64_t n, std::vector<int64_t> &tp_off, std::vector<int32_t> &tp_vert);

// Table-1 structure metrics (planner.cpp): counts, CC = E - V + 2P, Npath.
void structure_metrics(const HostPlan &plan, int32_t start, int32_t end, tpgen_metrics &m);

void set_error(const std::string &msg);

}  // namespace tpg
