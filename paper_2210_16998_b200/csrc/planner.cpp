// planner.cpp -- host side of libtpgen: CSR validation, Tarjan SCCs + the
// component graph ("first generates the component graph of the input CFG
// on the CPU", Def. 3), SCC-local tables for the CUDA
// kernels, the completion-count DP over the component DAG, shard ranges and
// the test-path prefix/suffix tables.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace tpg {

static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
const char *last_error() { return g_err.c_str(); }

// Iterative Tarjan ("Tarjan presents an algorithm with O(|V|+|E|)").
// SCC ids are assigned in completion order, which is a reverse topological
// order of the component DAG: every arc between SCCs goes from a larger id to
// a smaller id.
static int32_t tarjan(int32_t n, const std::vector<int64_t> &so, const std::vector<int32_t> &st,
                      std::vector<int32_t> &comp) {
    std::vector<int32_t> index(n, -1), low(n, 0), stack;
    std::vector<char> on(n, 0);
    std::vector<std::pair<int32_t, int64_t>> call;  // (vertex, next arc)
    comp.assign(n, -1);
    int32_t next_index = 0, n_scc = 0;
    stack.reserve(n);
    for (int32_t r = 0; r < n; r++) {
        if (index[r] >= 0) continue;
        call.push_back({r, so[r]});
        index[r] = low[r] = next_index++;
        stack.push_back(r);
        on[r] = 1;
        while (!call.empty()) {
            int32_t v = call.back().first;
            int64_t &e = call.back().second;
            if (e < so[v + 1]) {
                int32_t w = st[e++];
                if (index[w] < 0) {
                    index[w] = low[w] = next_index++;
                    stack.push_back(w);
                    on[w] = 1;
                    call.push_back({w, so[w]});
                } else if (on[w]) {
                    low[v] = std::min(low[v], index[w]);
                }
            } else {
                if (low[v] == index[v]) {
                    int32_t w;
                    do {
                        w = stack.back();
                        stack.pop_back();
                        on[w] = 0;
                        comp[w] = n_scc;
                    } while (w != v);
                    n_scc++;
                }
                call.pop_back();
                if (!call.empty()) {
                    int32_t p = call.back().first;
                    low[p] = std::min(low[p], low[v]);
                }
            }
        }
    }
    return n_scc;
}

tpgen_status build_plan(const int64_t *so_in, const int32_t *st_in, int32_t n, HostPlan &P, std::string &msg,
                        bool enforce_limit) {
    P = HostPlan();
    if (n < 0) { msg = "n_vertices < 0"; return TPGEN_ERR_INVALID_ARGUMENT; }
    if (n > 0 && (!so_in || (!st_in && so_in[n] > 0))) { msg = "NULL CSR pointer"; return TPGEN_ERR_INVALID_ARGUMENT; }
    P.n = n;
    if (n == 0) return TPGEN_OK;
    if (so_in[0] != 0) { msg = "csr_offsets[0] != 0"; return TPGEN_ERR_INVALID_GRAPH; }
    for (int32_t v = 0; v < n; v++)
        if (so_in[v + 1] < so_in[v]) { msg = "csr_offsets decreasing at row " + std::to_string(v); return TPGEN_ERR_INVALID_GRAPH; }
    P.m = so_in[n];
    P.so.assign(so_in, so_in + n + 1);
    P.st.assign(st_in, st_in + P.m);
    for (int32_t v = 0; v < n; v++) {
        auto b = P.st.begin() + P.so[v], e = P.st.begin() + P.so[v + 1];
        for (auto it = b; it != e; ++it)
            if (*it < 0 || *it >= n) { msg = "target out of range in row " + std::to_string(v); return TPGEN_ERR_INVALID_GRAPH; }
        std::sort(b, e);
        if (std::adjacent_find(b, e) != e) { msg = "duplicate arc in row " + std::to_string(v); return TPGEN_ERR_INVALID_GRAPH; }
    }
    // predecessor CSR (sources ascending)
    P.po.assign(n + 1, 0);
    P.pt.resize(P.m);
    for (int64_t e = 0; e < P.m; e++) P.po[P.st[e] + 1]++;
    for (int32_t v = 0; v < n; v++) P.po[v + 1] += P.po[v];
    {
        std::vector<int64_t> fill(P.po.begin(), P.po.end() - 1);
        for (int32_t v = 0; v < n; v++)
            for (int64_t e = P.so[v]; e < P.so[v + 1]; e++) P.pt[fill[P.st[e]]++] = v;
    }

    P.n_scc = tarjan(n, P.so, P.st, P.comp);
    if (!enforce_limit) {  // component graph only (tpgen_components)
        P.slot_flags.assign(n, 0);  // indexed by vertex here
        for (int32_t v = 0; v < n; v++) {
            for (int64_t e = P.so[v]; e < P.so[v + 1]; e++)
                if (P.comp[P.st[e]] != P.comp[v]) P.slot_flags[v] |= F_EXIT;
            for (int64_t e = P.po[v]; e < P.po[v + 1]; e++)
                if (P.comp[P.pt[e]] != P.comp[v]) P.slot_flags[v] |= F_ENTRY;
        }
        return TPGEN_OK;
    }
    std::vector<std::vector<int32_t>> members(P.n_scc);
    for (int32_t v = 0; v < n; v++) members[P.comp[v]].push_back(v);  // ascending v
    P.scc_vbase.resize(P.n_scc);
    P.scc_size.resize(P.n_scc);
    P.scc_out_base.resize(P.n_scc);
    P.scc_nout.resize(P.n_scc);
    P.scc_nentries.resize(P.n_scc);
    P.scc_pair_base.resize(P.n_scc);
    P.v_slot.resize(n);
    P.slot_gid.assign(n, 0);
    P.slot_out_off.assign(n, 0);
    P.slot_out_cnt.assign(n, 0);
    P.slot_flags.assign(n, 0);
    P.slot_eidx.assign(n, -1);
    std::vector<int32_t> local(n);
    int32_t base = 0;
    for (int32_t c = 0; c < P.n_scc; c++) {
        const auto &mem = members[c];
        if ((int)mem.size() > kMaxScc) {
            msg = "strongly connected component with " + std::to_string(mem.size()) + " vertices exceeds the " +
                  std::to_string(kMaxScc) + "-vertex limit of this build";
            return TPGEN_ERR_UNSUPPORTED;
        }
        P.scc_vbase[c] = base;
        P.scc_size[c] = (int32_t)mem.size();
        P.max_scc = std::max<int32_t>(P.max_scc, (int32_t)mem.size());
        for (size_t i = 0; i < mem.size(); i++) {
            local[mem[i]] = (int32_t)i;
            P.v_slot[mem[i]] = base + (int32_t)i;
        }
        base += (int32_t)mem.size();
    }
    P.W = P.max_scc <= 64 ? 1 : (P.max_scc <= 128 ? 2 : 4);
    const int W = P.W;
    P.sin.assign((size_t)n * W, 0);
    P.pin.assign((size_t)n * W, 0);
    int64_t pair_base = 0;
    for (int32_t c = 0; c < P.n_scc; c++) {
        const auto &mem = members[c];
        P.scc_out_base[c] = (int32_t)P.out_gid.size();
        int32_t nent = 0;
        bool nontriv = mem.size() > 1;
        for (int32_t v : mem) {
            const int32_t sl = P.v_slot[v];
            uint64_t *sin = &P.sin[(size_t)sl * W], *pin = &P.pin[(size_t)sl * W];
            P.slot_gid[sl] = v;
            P.slot_out_off[sl] = (int32_t)P.out_gid.size();
            for (int64_t e = P.so[v]; e < P.so[v + 1]; e++) {
                int32_t w = P.st[e];
                if (P.comp[w] == c) {
                    sin[local[w] >> 6] |= 1ull << (local[w] & 63);
                    if (w == v) nontriv = true;
                } else {
                    P.slot_flags[sl] |= F_EXIT;
                    P.out_gid.push_back(w);
                    // out_pos: number of SCC members with a smaller global id
                    P.out_pos.push_back((int32_t)(std::lower_bound(mem.begin(), mem.end(), w) - mem.begin()));
                    P.slot_out_cnt[sl]++;
                }
            }
            for (int64_t e = P.po[v]; e < P.po[v + 1]; e++) {
                int32_t u = P.pt[e];
                if (P.comp[u] == c) pin[local[u] >> 6] |= 1ull << (local[u] & 63);
                else P.slot_flags[sl] |= F_ENTRY;
            }
            if (P.slot_flags[sl] & F_ENTRY) {
                P.slot_eidx[sl] = nent++;
                P.has_entries = true;
            }
        }
        P.scc_nout[c] = (int32_t)P.out_gid.size() - P.scc_out_base[c];
        P.scc_nentries[c] = nent;
        P.scc_pair_base[c] = pair_base;
        pair_base += (int64_t)nent * P.scc_nout[c];
        if (nontriv) P.n_nontrivial++;
    }
    P.n_pairs = pair_base;

    // Work estimate per start vertex for shard balancing: Knuth's random-probe
    // estimator of the number of simple paths inside the start's SCC
    // (deterministic seed so every rank computes the same ranges).
    P.cost.assign(n, 1.0);
    uint64_t rng = 0x243F6A8885A308D3ull;
    auto next = [&rng]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    for (int32_t v = 0; v < n; v++) {
        int32_t c = P.comp[v];
        if (P.scc_size[c] <= 1) continue;
        const uint64_t *S = &P.sin[(size_t)P.scc_vbase[c] * W];
        int32_t s = local[v];
        const int probes = 48;
        double acc = 0;
        for (int p = 0; p < probes; p++) {
            uint64_t M[kMaxW] = {0, 0, 0, 0};
            M[s >> 6] |= 1ull << (s & 63);
            int32_t u = s;
            double prod = 1, est = 1;
            while (true) {
                int d = 0;
                for (int i = 0; i < W; i++) d += __builtin_popcountll(S[(size_t)u * W + i] & ~M[i]);
                if (!d) break;
                prod *= d;
                est += prod;
                int pick = (int)(next() % (uint64_t)d);
                for (int i = 0; i < W; i++) {
                    uint64_t cand = S[(size_t)u * W + i] & ~M[i];
                    int cw = __builtin_popcountll(cand);
                    if (pick >= cw) {
                        pick -= cw;
                        continue;
                    }
                    for (int q = 0; q < pick; q++) cand &= cand - 1;
                    u = i * 64 + __builtin_ctzll(cand);
                    break;
                }
                M[u >> 6] |= 1ull << (u & 63);
            }
            acc += est;
        }
        P.cost[v] = 1.0 + acc / probes;
    }
    return TPGEN_OK;
}

void shard_range(const HostPlan &P, int32_t rank, int32_t count, int32_t &lo, int32_t &hi) {
    if (count <= 1 || P.n == 0) { lo = 0; hi = P.n; return; }
    double total = 0;
    for (int32_t v = 0; v < P.n; v++) total += P.cost[v];
    // boundary b_r = first vertex whose prefix cost reaches r/count of the total
    auto boundary = [&](int32_t r) -> int32_t {
        if (r <= 0) return 0;
        if (r >= count) return P.n;
        double target = total * r / count, acc = 0;
        for (int32_t v = 0; v < P.n; v++) {
            if (acc + 0.5 * P.cost[v] >= target) return v;
            acc += P.cost[v];
        }
        return P.n;
    };
    lo = boundary(rank);
    hi = boundary(rank + 1);
    if (hi < lo) hi = lo;
}

bool prefix_shard_applies(const HostPlan &P) {
    if (P.W != 1 || P.max_scc > 32) return false;
    for (size_t i = 0; i < P.slot_flags.size(); i++)
        if (P.slot_out_cnt[i] > 0 || (P.slot_flags[i] & (F_EXIT | F_ENTRY))) return false;
    return true;
}

void prefix_shard(const HostPlan &P, int32_t rank, int32_t count, PrefixShard &out) {
    out = PrefixShard();
    std::vector<PrefixUnit> units;
    std::vector<double> cost;
    std::vector<uint32_t> credit;  // expanded interior nodes credited to the unit (its first descendant)
    for (int32_t v = 0; v < P.n; v++) {
        const int32_t slot = P.v_slot[v], c = P.comp[v];
        PrefixUnit u;
        memset(&u, 0, sizeof(u));
        const int loc = slot - P.scc_vbase[c];
        u.M = 1ull << loc;
        u.scc = c;
        u.gid = v;
        u.path[0] = (uint8_t)loc;
        units.push_back(u);
        cost.push_back(P.cost[v]);
        credit.push_back(0);
    }
    // Knuth's estimator of the subtree under a unit (its own node included), fixed seed
    uint64_t rng = 0x13198A2E03707344ull;
    auto next = [&rng]() {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        return rng;
    };
    auto knuth = [&](const PrefixUnit &u) {
        if (u.closure) return 1.0;
        const uint64_t *S = &P.sin[(size_t)P.scc_vbase[u.scc]];
        const uint64_t sbit = 1ull << u.path[0];
        const int probes = 48;
        double acc = 0;
        for (int p = 0; p < probes; p++) {
            uint64_t M = u.M;
            int32_t x = u.path[u.depth];
            double prod = 1, est = 1;
            while (true) {
                const uint64_t ch = S[x] & (~M | sbit);
                const int d = __builtin_popcountll(ch);
                if (!d) break;
                prod *= d;
                est += prod;
                uint64_t cand = ch;
                for (int q = (int)(next() % (uint64_t)d); q > 0; q--) cand &= cand - 1;
                x = __builtin_ctzll(cand);
                if (x == u.path[0]) break;  // the closing arc: a leaf
                M |= 1ull << x;
            }
            acc += est;
        }
        return acc / probes;
    };
    for (int round = 0; count > 1 && round < 32; round++) {  // (one shard: nothing to cut)
        double total = 0;
        for (double c : cost) total += c;
        const double heavy = total / (16.0 * std::max(count, 1));
        std::vector<PrefixUnit> nu;
        std::vector<double> nc;
        std::vector<uint32_t> ncr;
        bool grew = false;
        for (size_t i = 0; i < units.size(); i++) {
            const PrefixUnit &u = units[i];
            const uint64_t sbit = 1ull << u.path[0];
            const uint64_t ch = u.closure ? 0 : (P.sin[(size_t)(P.scc_vbase[u.scc] + u.path[u.depth])] & (~u.M | sbit));
            if (cost[i] <= heavy || ch == 0 || u.depth >= 30) {
                nu.push_back(u);
                nc.push_back(cost[i]);
                ncr.push_back(credit[i]);
                continue;
            }
            grew = true;
            uint32_t cr = credit[i] + (u.depth > 0 ? 1u : 0u);  // the expanded node's own extension
            for (uint64_t cc = ch; cc; cc &= cc - 1) {
                const int w = __builtin_ctzll(cc);
                PrefixUnit k = u;
                if (w == u.path[0]) {
                    k.closure = 1;
                } else {
                    k.depth = (uint8_t)(u.depth + 1);
                    k.path[k.depth] = (uint8_t)w;
                    k.M |= 1ull << w;
                }
                nu.push_back(k);
                nc.push_back(knuth(k));
                ncr.push_back(cr);
                cr = 0;
            }
        }
        units.swap(nu);
        cost.swap(nc);
        credit.swap(ncr);
        if (!grew) break;
    }
    const int64_t nu = (int64_t)units.size();
    out.n_units = nu;
    double total = 0;
    for (double c : cost) total += c;
    auto boundary = [&](int32_t r) -> int64_t {  // first unit whose prefix cost reaches r / count of the total
        if (r <= 0) return 0;
        if (r >= count) return nu;
        const double target = total * r / count;
        double acc = 0;
        for (int64_t i = 0; i < nu; i++) {
            if (acc + 0.5 * cost[i] >= target) return i;
            acc += cost[i];
        }
        return nu;
    };
    out.ulo = boundary(rank);
    out.uhi = std::max(out.ulo, boundary(rank + 1));
    out.units.assign(units.begin() + out.ulo, units.begin() + out.uhi);
    for (int64_t i = out.ulo; i < out.uhi; i++) out.ext += credit[i];
    if (out.uhi > out.ulo) {
        out.lo = units[out.ulo].gid;
        out.hi = units[out.uhi - 1].gid + 1;
    }
}

static inline bool add_ov(uint64_t a, uint64_t b, uint64_t &r) {
    r = a + b;
    return r < a || r >= (1ull << 62);
}
static inline bool mul_ov(uint64_t a, uint64_t b, uint64_t &r) {
    unsigned __int128 p = (unsigned __int128)a * b;
    r = (uint64_t)p;
    return p >= ((unsigned __int128)1 << 62);
}

bool completion_dp(const HostPlan &P, const std::vector<uint64_t> &tail_cnt, const std::vector<uint64_t> &tail_len,
                   const std::vector<uint64_t> &pair_cnt, const std::vector<uint64_t> &pair_len,
                   std::vector<uint64_t> &W, std::vector<uint64_t> &V) {
    W.assign(P.n, 0);
    V.assign(P.n, 0);
    bool ok = true;
    // SCC ids are reverse topological: every y reached over an out-arc of SCC c
    // lives in an SCC with a smaller id, already final when c is processed.
    for (int32_t c = 0; c < P.n_scc; c++) {
        int32_t vb = P.scc_vbase[c], L = P.scc_size[c];
        int32_t nout = P.scc_nout[c], ob = P.scc_out_base[c];
        for (int32_t i = 0; i < L; i++) {
            int32_t slot = vb + i;
            int32_t ei = P.slot_eidx[slot];
            if (ei < 0) continue;
            int32_t x = P.slot_gid[slot];
            uint64_t w = tail_cnt[slot], vv = tail_len[slot];
            for (int32_t a = 0; a < nout; a++) {
                int64_t pi = P.scc_pair_base[c] + (int64_t)ei * nout + a;
                uint64_t cnt = pair_cnt[pi], len = pair_len[pi];
                if (!cnt) continue;
                int32_t y = P.out_gid[ob + a];
                uint64_t t1, t2, t3;
                // W += cnt * W(y); V += len * W(y) + cnt * V(y)
                ok &= !mul_ov(cnt, W[y], t1);
                ok &= !add_ov(w, t1, w);
                ok &= !mul_ov(len, W[y], t2);
                ok &= !mul_ov(cnt, V[y], t3);
                ok &= !add_ov(vv, t2, vv);
                ok &= !add_ov(vv, t3, vv);
            }
            W[x] = w;
            V[x] = vv;
        }
    }
    return ok;
}

void build_tp_tables(const HostPlan &P, int32_t entry, int32_t exit, TpTables &T) {
    // The host computes the two walk trees, O(n + m); the GPU expands them into the
    // flat prefix / suffix tables (tp_flat_kernel) -- those are O(n * depth).
    int32_t n = P.n;
    T.pre_off.assign(n, -1);
    T.suf_off.assign(n, -1);
    T.pre_len.assign(n, -1);
    T.suf_len.assign(n, -1);
    T.parent.assign(n, -1);
    T.next.assign(n, -1);
    // BFS from entry, successors ascending, first discoverer becomes the parent:
    // the tree path is the lexicographically smallest minimum-hop walk.
    std::vector<int32_t> parent(n, -2), order;
    order.reserve(n);
    parent[entry] = -1;
    T.pre_len[entry] = 1;
    order.push_back(entry);
    for (size_t h = 0; h < order.size(); h++) {
        int32_t v = order[h];
        for (int64_t e = P.so[v]; e < P.so[v + 1]; e++) {
            int32_t w = P.st[e];
            if (parent[w] == -2) {
                parent[w] = v;
                T.pre_len[w] = T.pre_len[v] + 1;
                order.push_back(w);
            }
        }
    }
    int64_t acc = 0;
    for (int32_t v = 0; v < n; v++) {
        T.parent[v] = parent[v] < 0 ? -1 : parent[v];
        if (T.pre_len[v] > 0) {
            T.pre_off[v] = acc;
            acc += T.pre_len[v];
        }
    }
    T.pre_total = acc;
    // reverse BFS distances to exit; suffix = greedy smallest successor one hop closer
    std::vector<int32_t> dist(n, -1);
    order.clear();
    dist[exit] = 0;
    order.push_back(exit);
    for (size_t h = 0; h < order.size(); h++) {
        int32_t v = order[h];
        for (int64_t e = P.po[v]; e < P.po[v + 1]; e++) {
            int32_t u = P.pt[e];
            if (dist[u] < 0) { dist[u] = dist[v] + 1; order.push_back(u); }
        }
    }
    acc = 0;
    for (int32_t v = 0; v < n; v++) {
        if (dist[v] < 0) continue;
        if (v != exit)
            for (int64_t e = P.so[v]; e < P.so[v + 1]; e++)  // successors ascending
                if (dist[P.st[e]] == dist[v] - 1) { T.next[v] = P.st[e]; break; }
        T.suf_len[v] = dist[v] + 1;
        T.suf_off[v] = acc;
        acc += T.suf_len[v];
    }
    T.suf_total = acc;
}

}  // namespace tpg

namespace tpg {

// Table 1: V, E, the nontrivial SCCs and the arcs inside them, weakly connected
// components P (union-find), CC = E - V + 2P, and Npath: the number of
// start -> end walks that use every arc at most once, Npath(end) = 1.  On an acyclic graph that is
// the number of start -> end paths (a DP in reverse topological order, saturating at 2^62); with
// cycles, a depth-first search over arc-simple walks (an arc-used bitmap), within a step budget.
void structure_metrics(const HostPlan &P, int32_t start, int32_t end, tpgen_metrics &m) {
    const int32_t n = P.n;
    m.nodes = n;
    m.edges = P.m;
    std::vector<int32_t> size(std::max(P.n_scc, 1), 0);
    std::vector<char> loop(std::max(P.n_scc, 1), 0);
    for (int32_t v = 0; v < n; v++) {
        size[P.comp[v]]++;
        for (int64_t e = P.so[v]; e < P.so[v + 1]; e++)
            if (P.st[e] == v) loop[P.comp[v]] = 1;
    }
    bool cyclic = false;
    for (int32_t c = 0; c < P.n_scc; c++)
        if (size[c] > 1 || loop[c]) {
            m.sccs++;
            m.scc_nodes += size[c];
            cyclic = true;
        }
    for (int32_t v = 0; v < n; v++)
        for (int64_t e = P.so[v]; e < P.so[v + 1]; e++)
            if (P.comp[P.st[e]] == P.comp[v] && (size[P.comp[v]] > 1 || loop[P.comp[v]])) m.scc_edges++;
    std::vector<int32_t> par(n);
    for (int32_t v = 0; v < n; v++) par[v] = v;
    auto find = [&](int32_t x) {
        while (par[x] != x) x = par[x] = par[par[x]];
        return x;
    };
    for (int32_t v = 0; v < n; v++)
        for (int64_t e = P.so[v]; e < P.so[v + 1]; e++) {
            const int32_t a = find(v), b = find(P.st[e]);
            if (a != b) par[a] = b;
        }
    for (int32_t v = 0; v < n; v++) m.weak_components += (find(v) == v);
    m.cc = m.edges - m.nodes + 2 * m.weak_components;
    if (n == 0) return;
    if (start == end) {  // Npath(end) = 1
        m.npath = 1;
        return;
    }
    const uint64_t cap = 1ull << 62;
    if (!cyclic) {  // SCC ids are reverse topological: successors have smaller ids
        std::vector<int32_t> order(n);
        for (int32_t v = 0; v < n; v++) order[v] = v;
        std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return P.comp[a] < P.comp[b]; });
        std::vector<uint64_t> np(n, 0);
        for (int32_t v : order) {
            if (v == end) {
                np[v] = 1;
                continue;
            }
            uint64_t t = 0;
            for (int64_t e = P.so[v]; e < P.so[v + 1]; e++) {
                t += np[P.st[e]];
                if (t >= cap) {
                    t = cap;
                    m.npath_status = 1;
                }
            }
            np[v] = t;
        }
        m.npath = np[start];
        return;
    }
    // arc-simple walks from start (iterative DFS over (vertex, next arc) frames)
    std::vector<char> used((size_t)std::max<int64_t>(P.m, 1), 0);
    std::vector<std::pair<int32_t, int64_t>> stack;
    std::vector<int64_t> via;  // arc taken into each frame
    uint64_t count = 0, steps = 0;
    const uint64_t budget = 100000000ull;
    stack.push_back({start, P.so[start]});
    via.push_back(-1);
    while (!stack.empty()) {
        if (++steps > budget) {
            m.npath = 0;
            m.npath_status = 2;
            return;
        }
        auto &fr = stack.back();
        const int32_t v = fr.first;
        if (v == end && stack.size() > 1) {  // Npath(end) = 1: a walk stops at end
            used[via.back()] = 0;
            stack.pop_back();
            via.pop_back();
            continue;
        }
        if (fr.second >= P.so[v + 1]) {
            if (via.back() >= 0) used[via.back()] = 0;
            stack.pop_back();
            via.pop_back();
            continue;
        }
        const int64_t e = fr.second++;
        if (used[e]) continue;
        used[e] = 1;
        const int32_t w = P.st[e];
        if (w == end && ++count >= cap) {
            m.npath = cap;
            m.npath_status = 1;
            return;
        }
        stack.push_back({w, P.so[w]});
        via.push_back(e);
    }
    m.npath = count;
}

}  // namespace tpg
