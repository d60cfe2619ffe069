// normalize.cpp -- out-degree-2 normalization of a CFG (Fig. 5;
// DESIGN.md R24), the input shape of the paper's Alg. 3 (two "read by successor" flags per
// path).  Host code: the graph is KB-sized.
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/tpgen.h"
#include "internal.h"

extern "C" tpgen_status tpgen_normalize_outdeg2(const int64_t *so, const int32_t *st, int32_t n, int32_t *out_n,
                                                int64_t *out_m, int64_t *out_offsets, int32_t *out_targets,
                                                int32_t *origin) {
    if (n < 0 || (n > 0 && (!so || !st))) {
        tpg::set_error("NULL CSR or negative n_vertices");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (n > 0 && so[0] != 0) {
        tpg::set_error("csr_offsets[0] != 0");
        return TPGEN_ERR_INVALID_GRAPH;
    }
    int64_t extra = 0;
    std::vector<int32_t> row;
    for (int32_t v = 0; v < n; v++) {
        if (so[v + 1] < so[v]) {
            tpg::set_error("csr_offsets decreasing at row " + std::to_string(v));
            return TPGEN_ERR_INVALID_GRAPH;
        }
        row.assign(st + so[v], st + so[v + 1]);
        for (int32_t w : row)
            if (w < 0 || w >= n) {
                tpg::set_error("target out of range in row " + std::to_string(v));
                return TPGEN_ERR_INVALID_GRAPH;
            }
        std::sort(row.begin(), row.end());
        if (std::adjacent_find(row.begin(), row.end()) != row.end()) {
            tpg::set_error("duplicate arc in row " + std::to_string(v));
            return TPGEN_ERR_INVALID_GRAPH;
        }
        extra += std::max<int64_t>(0, (int64_t)row.size() - 2);
    }
    const int64_t m = n > 0 ? so[n] : 0;
    if ((int64_t)n + extra > INT32_MAX) {
        tpg::set_error("normalized graph exceeds 2^31 vertices");
        return TPGEN_ERR_LIMIT_EXCEEDED;
    }
    const int32_t N = (int32_t)(n + extra);
    if (out_n) *out_n = N;
    if (out_m) *out_m = m + extra;  // d arcs of a split vertex become 2 + 2 (d - 2) = d + (d - 2)
    if (!out_offsets && !out_targets && !origin) return TPGEN_OK;
    // rows of the new graph, built in vertex order: first the n input vertices, then the chains
    std::vector<std::vector<int32_t>> rows(N);
    std::vector<int32_t> orig(N);
    int32_t next = n;
    for (int32_t v = 0; v < n; v++) {
        orig[v] = v;
        row.assign(st + so[v], st + so[v + 1]);
        std::sort(row.begin(), row.end());
        const int32_t d = (int32_t)row.size();
        if (d <= 2) {
            rows[v] = row;
            continue;
        }
        // v -> w1, x1;  x_i -> w_{i+1}, x_{i+1};  x_{d-2} -> w_{d-1}, w_d
        int32_t x = next;
        next += d - 2;
        rows[v] = {row[0], x};
        for (int32_t i = 1; i <= d - 2; i++) {
            const int32_t xi = x + i - 1;
            orig[xi] = v;
            if (i < d - 2) rows[xi] = {row[i], xi + 1};
            else rows[xi] = {row[d - 2], row[d - 1]};
        }
    }
    int64_t e = 0;
    for (int32_t v = 0; v < N; v++) {
        if (out_offsets) out_offsets[v] = e;
        for (int32_t w : rows[v]) {
            if (out_targets) out_targets[e] = w;
            e++;
        }
    }
    if (out_offsets) out_offsets[N] = e;
    if (origin) std::copy(orig.begin(), orig.end(), origin);
    return TPGEN_OK;
}
