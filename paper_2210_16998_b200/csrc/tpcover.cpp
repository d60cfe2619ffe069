// tpcover.cpp -- greedy test-path cover of libtpgen.
//
// PAPER.md P:874 (Ammann-Offutt, as TPGen uses it): start with the longest
// prime path, extend it to the initial and final nodes, repeat with the longest
// prime path not yet covered.  Order: decreasing length, ties in canonical
// (lexicographic) order; the extension uses the R15 walks (lexmin minimum-hop
// prefix entry -> first, suffix last -> exit), so the cover is deterministic.
//
// Marking is linear in the test path: a prime path q that occurs in TP t at
// [i, j] is maximal, so it cannot be extended inside t -- either j is the end r_i
// of the longest repeat-free run of t starting at i, or q is a cycle and
// t[j] = t[i] with j = r_i + 1.  Each start i therefore has at most two
// candidates, looked up by a polynomial hash of the vertex sequence (and
// confirmed vertex by vertex).  Sequential by nature: host code.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "internal.h"

namespace tpg {

namespace {
constexpr uint64_t kBase = 0x100000001B3ull;  // odd multiplier of the sequence hash (mod 2^64)

uint64_t seq_hash(const int32_t *v, int64_t n) {
    uint64_t h = 0;
    for (int64_t i = 0; i < n; i++) h = h * kBase + (uint64_t)(uint32_t)v[i] + 1;
    return h;
}
}  // namespace

bool greedy_cover(const HostPlan &H, const TpTables &T, int32_t entry, int32_t exit, const int64_t *off,
                  const int32_t *vert, int64_t n, std::vector<int64_t> &tp_off, std::vector<int32_t> &tp_vert) {
    (void)entry;
    (void)exit;
    tp_off.assign(1, 0);
    tp_vert.clear();
    if (n <= 0) return true;
    // prime paths by hash: open addressing, linear probing (equal hashes are confirmed
    // vertex by vertex, so colliding paths simply occupy neighbouring slots)
    size_t cap = 16;
    while (cap < (size_t)n * 2) cap <<= 1;
    std::vector<uint64_t> hkey(cap, 0);
    std::vector<int64_t> hval(cap, -1);
    int64_t maxlen = 0;
    for (int64_t i = 0; i < n; i++) {
        const uint64_t h = seq_hash(vert + off[i], off[i + 1] - off[i]);
        size_t s = (size_t)(h * 0x9E3779B97F4A7C15ull) & (cap - 1);
        while (hval[s] >= 0) s = (s + 1) & (cap - 1);
        hkey[s] = h;
        hval[s] = i;
        maxlen = std::max<int64_t>(maxlen, off[i + 1] - off[i]);
    }
    std::vector<int64_t> order((size_t)n);
    for (int64_t i = 0; i < n; i++) order[(size_t)i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    std::vector<char> covered((size_t)n, 0);
    std::vector<int32_t> cnt((size_t)std::max(H.n, 1), 0);  // repeat-free window, per vertex
    std::vector<int32_t> t, pre;
    std::vector<uint64_t> ph, pw;
    for (int64_t seed : order) {
        if (covered[(size_t)seed]) continue;
        const int32_t *p = vert + off[seed];
        const int64_t plen = off[seed + 1] - off[seed];
        const int32_t f = p[0], l = p[plen - 1];
        if (T.pre_len[f] < 0 || T.suf_len[l] < 0) return false;
        // TP = prefix(entry -> f) minus f, then the PP, then suffix(l -> exit) minus l
        pre.clear();
        for (int32_t c = T.parent[f]; c >= 0; c = T.parent[c]) pre.push_back(c);
        t.assign(pre.rbegin(), pre.rend());
        t.insert(t.end(), p, p + plen);
        for (int32_t c = T.next[l]; c >= 0; c = T.next[c]) t.push_back(c);
        const int64_t L = (int64_t)t.size();
        tp_vert.insert(tp_vert.end(), t.begin(), t.end());
        tp_off.push_back((int64_t)tp_vert.size());
        // prefix hashes for O(1) substring hashes
        ph.assign((size_t)L + 1, 0);
        pw.assign((size_t)L + 1, 1);
        for (int64_t k = 0; k < L; k++) {
            ph[(size_t)k + 1] = ph[(size_t)k] * kBase + (uint64_t)(uint32_t)t[(size_t)k] + 1;
            pw[(size_t)k + 1] = pw[(size_t)k] * kBase;
        }
        auto mark = [&](int64_t a, int64_t b) {  // candidate t[a..b] inclusive
            const int64_t m = b - a + 1;
            if (m > maxlen) return;
            const uint64_t h = ph[(size_t)b + 1] - ph[(size_t)a] * pw[(size_t)m];
            for (size_t s = (size_t)(h * 0x9E3779B97F4A7C15ull) & (cap - 1); hval[s] >= 0; s = (s + 1) & (cap - 1)) {
                if (hkey[s] != h) continue;
                const int64_t q = hval[s];
                if (covered[(size_t)q] || off[q + 1] - off[q] != m) continue;
                if (std::memcmp(vert + off[q], t.data() + a, (size_t)m * 4) == 0) covered[(size_t)q] = 1;
            }
        };
        // two pointers: r = end of the longest repeat-free run from i
        int64_t r = -1;
        for (int64_t i = 0; i < L; i++) {
            if (r < i - 1) r = i - 1;
            while (r + 1 < L && cnt[(size_t)t[(size_t)r + 1]] == 0) {
                r++;
                cnt[(size_t)t[(size_t)r]]++;
            }
            mark(i, r);                                      // the maximal acyclic run
            if (r + 1 < L && t[(size_t)r + 1] == t[(size_t)i]) mark(i, r + 1);  // or the cycle back to t[i]
            if (r >= i) cnt[(size_t)t[(size_t)i]]--;
        }
    }
    return true;
}

}  // namespace tpg
