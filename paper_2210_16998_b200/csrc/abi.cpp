// abi.cpp -- extern "C" entry points of libtpgen (declared in include/tpgen.h).
#include <chrono>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <vector>

#include "engine.h"

struct tpgen_plan {
    tpg::PlanImpl impl;
    // one-shot calls: the CSR the cached plan was built from (a repeated call on the same
    // graph skips planning and upload and keeps the plan's device-side caches)
    std::vector<int64_t> last_off;
    std::vector<int32_t> last_tgt;
    bool last_valid = false;
};

namespace {

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

tpgen_status check_options(const tpgen_options &o) {
    if (o.shard_count < 1 || o.shard_rank < 0 || o.shard_rank >= o.shard_count) {
        tpg::set_error("bad shard spec");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.shard_count > 1 && o.start_hi > o.start_lo) {
        tpg::set_error("a start range and a shard spec cannot be combined");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.output_mode != TPGEN_OUT_MATERIALIZE && o.output_mode != TPGEN_OUT_COUNT_HASH) {
        tpg::set_error("bad output_mode");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.engine != TPGEN_ENGINE_DFS && o.engine != TPGEN_ENGINE_FRONTIER && o.engine != TPGEN_ENGINE_ALG3) {
        tpg::set_error("bad engine");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.engine != TPGEN_ENGINE_DFS && o.output_mode != TPGEN_OUT_COUNT_HASH) {
        tpg::set_error("the frontier and Alg. 3 engines compute counts and the digest only (output_mode COUNT_HASH)");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.engine == TPGEN_ENGINE_ALG3 && (o.shard_count > 1 || o.start_hi > o.start_lo)) {
        tpg::set_error("the Alg. 3 engine has no start-vertex shards (every vertex list is global)");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.shard_prefix != 0 && o.shard_prefix != 1) {
        tpg::set_error("bad shard_prefix");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.prune != 0 && (o.prune != 1 || o.engine != TPGEN_ENGINE_DFS || o.output_mode != TPGEN_OUT_COUNT_HASH)) {
        tpg::set_error("prune: 0 or 1, DFS engine, COUNT_HASH output only");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.shard_prefix && o.engine != TPGEN_ENGINE_DFS) {
        tpg::set_error("prefix-unit shards are a DFS-engine option");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (o.tp_mode != TPGEN_TP_PER_PP && o.tp_mode != TPGEN_TP_UNIQUE && o.tp_mode != TPGEN_TP_GREEDY) {
        tpg::set_error("bad tp_mode");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    return TPGEN_OK;
}

tpgen_options resolve(const tpgen_options *opt) {
    tpgen_options o;
    tpgen_options_init(&o);
    if (opt) o = *opt;
    return o;
}

tpgen_status make_plan(const int64_t *so, const int32_t *st, int32_t n, const tpgen_options &o, tpgen_plan **out) {
    *out = nullptr;
    tpgen_plan *p = new (std::nothrow) tpgen_plan();
    if (!p) return TPGEN_ERR_OUT_OF_MEMORY;
    tpgen_status s = tpg::init_device(p->impl, o);
    if (s == TPGEN_OK) {
        const double t0 = now_ms();
        std::string msg;
        s = tpg::build_plan(so, st, n, p->impl.hp, msg);
        if (s != TPGEN_OK) tpg::set_error(msg);
        p->impl.ms_plan = now_ms() - t0;
    }
    if (s == TPGEN_OK) s = tpg::plan_upload(p->impl, (cudaStream_t)o.stream);
    if (s != TPGEN_OK) {
        delete p;
        return s;
    }
    *out = p;
    return TPGEN_OK;
}

// One-shot calls (tpgen_prime_paths / tpgen_test_paths) reuse a per-device
// plan object so device workspaces (work queue, record pool, scan buffers)
// persist across calls; calls are serialised per process by the mutex.
std::mutex g_cache_mu;
std::map<int, tpgen_plan *> g_cache;

tpgen_status cached_plan(const int64_t *so, const int32_t *st, int32_t n, const tpgen_options &o, tpgen_plan **out) {
    *out = nullptr;
    int dev = o.device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
        tpg::set_error("no CUDA device");
        return TPGEN_ERR_CUDA;
    }
    tpgen_plan *&p = g_cache[dev];
    if (!p) {
        p = new (std::nothrow) tpgen_plan();
        if (!p) return TPGEN_ERR_OUT_OF_MEMORY;
        tpgen_options od = o;
        od.device = dev;
        tpgen_status s = tpg::init_device(p->impl, od);
        if (s != TPGEN_OK) {
            delete p;
            p = nullptr;
            return s;
        }
    }
    if (cudaSetDevice(dev) != cudaSuccess) return TPGEN_ERR_CUDA;
    const double t0 = now_ms();
    const int64_t m = (n > 0) ? so[n] - so[0] : 0;
    if (!o.no_plan_cache && p->last_valid && n >= 0 && (int64_t)p->last_off.size() == (int64_t)n + 1 && (int64_t)p->last_tgt.size() == m &&
        (n == 0 || memcmp(p->last_off.data(), so, sizeof(int64_t) * ((size_t)n + 1)) == 0) &&
        (m == 0 || memcmp(p->last_tgt.data(), st + so[0], sizeof(int32_t) * (size_t)m) == 0)) {
        p->impl.ms_plan = now_ms() - t0;  // the same graph as the previous call: the plan stands
        *out = p;
        return TPGEN_OK;
    }
    p->last_valid = false;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, p->impl.hp, msg);
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    p->impl.ms_plan = now_ms() - t0;
    s = tpg::plan_upload(p->impl, (cudaStream_t)o.stream);
    if (s != TPGEN_OK) return s;
    if (n >= 0) {  // (a valid plan implies a valid CSR: offsets[0] = 0, non-decreasing)
        p->last_off.assign(so, so + (size_t)n + 1);
        p->last_tgt.assign(st + so[0], st + so[0] + m);
        p->last_valid = true;
    }
    *out = p;
    return TPGEN_OK;
}

struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

extern "C" {

void tpgen_options_init(tpgen_options *o) {
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->device = -1;
    o->output_on_device = 1;
    o->output_mode = TPGEN_OUT_MATERIALIZE;
    o->shard_rank = 0;
    o->shard_count = 1;
}

const char *tpgen_status_string(tpgen_status s) {
    switch (s) {
        case TPGEN_OK: return "ok";
        case TPGEN_ERR_INVALID_ARGUMENT: return "invalid argument";
        case TPGEN_ERR_INVALID_GRAPH: return "invalid graph";
        case TPGEN_ERR_LIMIT_EXCEEDED: return "limit exceeded";
        case TPGEN_ERR_OUT_OF_MEMORY: return "out of memory";
        case TPGEN_ERR_UNREACHABLE: return "unreachable endpoint";
        case TPGEN_ERR_CUDA: return "CUDA error";
        case TPGEN_ERR_INTERNAL: return "internal error";
        case TPGEN_ERR_UNSUPPORTED: return "unsupported input";
    }
    return "unknown status";
}

const char *tpgen_last_error_message(void) { return tpg::last_error(); }

const char *tpgen_version(void) {
    return "tpgen-b200 0.2 (sm_100a; DFS + count-mode DFS, frontier and Alg. 3 engines; TMA-store writer)";
}

tpgen_status tpgen_plan_create(const int64_t *so, const int32_t *st, int32_t n, const tpgen_options *opt,
                               tpgen_plan **plan) {
    if (!plan) return TPGEN_ERR_INVALID_ARGUMENT;
    *plan = nullptr;
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    tpgen_status r = make_plan(so, st, n, o, plan);
    if (r == TPGEN_OK && cudaStreamSynchronize((cudaStream_t)o.stream) != cudaSuccess) {
        tpgen_plan_destroy(*plan);
        *plan = nullptr;
        return TPGEN_ERR_CUDA;
    }
    return r;
}

tpgen_status tpgen_plan_prime_paths(tpgen_plan *plan, const tpgen_options *opt, tpgen_paths *out,
                                    tpgen_stats *stats) {
    if (!plan || !out) return TPGEN_ERR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    DeviceScope ds(plan->impl.device);
    s = tpg::run_prime_paths(plan->impl, o, out, stats);
    if (s != TPGEN_OK) memset(out, 0, sizeof(*out));
    return s;
}

tpgen_status tpgen_plan_test_paths(tpgen_plan *plan, const tpgen_paths *prime_paths, int32_t entry, int32_t exit,
                                   const tpgen_options *opt, tpgen_paths *out, tpgen_stats *stats) {
    if (!plan || !out) return TPGEN_ERR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    const int32_t n = plan->impl.hp.n;
    if (entry < 0 || entry >= n || exit < 0 || exit >= n) {
        tpg::set_error("entry/exit out of range");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (prime_paths && prime_paths->n_paths > 0 && (!prime_paths->offsets || !prime_paths->vertices)) {
        tpg::set_error("prime_paths has NULL arrays");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    DeviceScope ds(plan->impl.device);
    s = tpg::run_test_paths(plan->impl, prime_paths, entry, exit, o, out, stats);
    if (s != TPGEN_OK) memset(out, 0, sizeof(*out));
    return s;
}

tpgen_status tpgen_plan_classify(tpgen_plan *plan, const tpgen_paths *prime_paths, int32_t start, int32_t end,
                                 const tpgen_options *opt, int64_t counts[5]) {
    if (!plan || !prime_paths || !counts) return TPGEN_ERR_INVALID_ARGUMENT;
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    const int32_t n = plan->impl.hp.n;
    if (start < 0 || start >= n || end < 0 || end >= n) {
        tpg::set_error("start/end out of range");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (prime_paths->n_paths > 0 && (!prime_paths->offsets || !prime_paths->vertices)) {
        tpg::set_error("prime_paths has NULL arrays");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    DeviceScope ds(plan->impl.device);
    return tpg::run_classify(plan->impl, prime_paths, start, end, o, counts);
}

void tpgen_plan_destroy(tpgen_plan *plan) { delete plan; }

void tpgen_release_cache(void) {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    for (auto &kv : g_cache) delete kv.second;  // (the plan's destructor releases its device workspaces)
    g_cache.clear();
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        cudaDeviceSynchronize();
        tpg::release_output_cache(dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    }
}

tpgen_status tpgen_prime_paths(const int64_t *so, const int32_t *st, int32_t n, const tpgen_options *opt,
                               tpgen_paths *out, tpgen_stats *stats) {
    if (!out) return TPGEN_ERR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    const double t0 = now_ms();
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    std::lock_guard<std::mutex> lock(g_cache_mu);
    tpgen_plan *p = nullptr;
    s = cached_plan(so, st, n, o, &p);
    if (s != TPGEN_OK) return s;
    {
        DeviceScope ds(p->impl.device);
        s = tpg::run_prime_paths(p->impl, o, out, stats);
    }
    if (s != TPGEN_OK) memset(out, 0, sizeof(*out));
    if (s == TPGEN_OK && stats) stats->ms_total = now_ms() - t0;
    return s;
}

tpgen_status tpgen_test_paths(const int64_t *so, const int32_t *st, int32_t n, const tpgen_paths *prime_paths,
                              int32_t entry, int32_t exit, const tpgen_options *opt, tpgen_paths *out,
                              tpgen_stats *stats) {
    if (!out) return TPGEN_ERR_INVALID_ARGUMENT;
    memset(out, 0, sizeof(*out));
    const double t0 = now_ms();
    tpgen_options o = resolve(opt);
    tpgen_status s = check_options(o);
    if (s != TPGEN_OK) return s;
    if (entry < 0 || entry >= n || exit < 0 || exit >= n) {
        tpg::set_error("entry/exit out of range");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    if (prime_paths && prime_paths->n_paths > 0 && (!prime_paths->offsets || !prime_paths->vertices)) {
        tpg::set_error("prime_paths has NULL arrays");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    std::lock_guard<std::mutex> lock(g_cache_mu);
    tpgen_plan *p = nullptr;
    s = cached_plan(so, st, n, o, &p);
    if (s != TPGEN_OK) return s;
    {
        DeviceScope ds(p->impl.device);
        s = tpg::run_test_paths(p->impl, prime_paths, entry, exit, o, out, stats);
    }
    if (s != TPGEN_OK) memset(out, 0, sizeof(*out));
    if (s == TPGEN_OK && stats) stats->ms_total = now_ms() - t0;
    return s;
}

void tpgen_paths_free(tpgen_paths *p) { tpg::free_paths(p); }

tpgen_status tpgen_shard_range(const int64_t *so, const int32_t *st, int32_t n, int32_t rank, int32_t count,
                               int32_t *lo, int32_t *hi) {
    if (n < 0 || !lo || !hi || count < 1 || rank < 0 || rank >= count) {
        tpg::set_error("bad shard spec, NULL output pointer or n < 0");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    tpg::HostPlan P;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, P, msg, true);  // (the full plan: its cost estimates)
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    tpg::shard_range(P, rank, count, *lo, *hi);
    return TPGEN_OK;
}

tpgen_status tpgen_shard_units(const int64_t *so, const int32_t *st, int32_t n, int32_t rank, int32_t count,
                               int32_t *applies, int64_t *unit_lo, int64_t *unit_hi, int64_t *n_units, int32_t *lo,
                               int32_t *hi) {
    if (n < 0 || !applies || count < 1 || rank < 0 || rank >= count) {
        tpg::set_error("bad shard spec, NULL applies pointer or n < 0");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    tpg::HostPlan P;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, P, msg, true);
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    int32_t l = 0, h = 0;
    int64_t ul = 0, uh = 0, nu = 0;
    *applies = tpg::prefix_shard_applies(P) ? 1 : 0;
    if (*applies) {
        tpg::PrefixShard ps;
        tpg::prefix_shard(P, rank, count, ps);
        l = ps.lo, h = ps.hi, ul = ps.ulo, uh = ps.uhi, nu = ps.n_units;
    } else {
        tpg::shard_range(P, rank, count, l, h);
    }
    if (unit_lo) *unit_lo = ul;
    if (unit_hi) *unit_hi = uh;
    if (n_units) *n_units = nu;
    if (lo) *lo = l;
    if (hi) *hi = h;
    return TPGEN_OK;
}

tpgen_status tpgen_shard_unit_paths(const int64_t *so, const int32_t *st, int32_t n, int32_t rank, int32_t count,
                                    int64_t *offsets, int32_t *vertices, int32_t *closure, int64_t cap_units,
                                    int64_t cap_vertices, int64_t *n_units_out, int64_t *n_vertices_out) {
    if (n < 0 || !n_units_out || !n_vertices_out || count < 1 || rank < 0 || rank >= count) {
        tpg::set_error("bad shard spec, NULL count pointers or n < 0");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    tpg::HostPlan P;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, P, msg, true);
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    tpg::PrefixShard ps;
    if (tpg::prefix_shard_applies(P)) tpg::prefix_shard(P, rank, count, ps);
    int64_t nv = 0;
    for (const tpg::PrefixUnit &u : ps.units) nv += u.depth + 1;
    *n_units_out = (int64_t)ps.units.size();
    *n_vertices_out = nv;
    if (!offsets || !vertices || !closure) return TPGEN_OK;
    if (cap_units < (int64_t)ps.units.size() || cap_vertices < nv) {
        tpg::set_error("unit arrays too small");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    int64_t o = 0;
    for (size_t i = 0; i < ps.units.size(); i++) {
        const tpg::PrefixUnit &u = ps.units[i];
        offsets[i] = o;
        closure[i] = u.closure ? 1 : 0;
        const int32_t vb = P.scc_vbase[u.scc];
        for (int d = 0; d <= u.depth; d++) vertices[o++] = P.slot_gid[vb + u.path[d]];
    }
    offsets[ps.units.size()] = o;
    return TPGEN_OK;
}

tpgen_status tpgen_metrics_compute(const int64_t *so, const int32_t *st, int32_t n, int32_t start, int32_t end,
                                   tpgen_metrics *m) {
    if (n < 0 || !m || (n > 0 && (start < 0 || start >= n || end < 0 || end >= n))) {
        tpg::set_error("NULL output, n < 0, or start / end out of range");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    memset(m, 0, sizeof(*m));
    tpg::HostPlan P;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, P, msg, false);
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    tpg::structure_metrics(P, start, end, *m);
    return TPGEN_OK;
}

tpgen_status tpgen_components(const int64_t *so, const int32_t *st, int32_t n, int32_t *comp, int32_t *flags,
                              int32_t *n_scc) {
    if (n < 0 || (n > 0 && (!comp || !flags)) || !n_scc) {
        tpg::set_error("NULL output pointer or n < 0");
        return TPGEN_ERR_INVALID_ARGUMENT;
    }
    tpg::HostPlan P;
    std::string msg;
    tpgen_status s = tpg::build_plan(so, st, n, P, msg, false);
    if (s != TPGEN_OK) {
        tpg::set_error(msg);
        return s;
    }
    std::vector<int32_t> size(P.n_scc, 0);
    std::vector<char> loop(P.n_scc, 0);
    for (int32_t v = 0; v < n; v++) {
        size[P.comp[v]]++;
        for (int64_t e = P.so[v]; e < P.so[v + 1]; e++)
            if (P.st[e] == v) loop[P.comp[v]] = 1;
    }
    for (int32_t v = 0; v < n; v++) {
        comp[v] = P.comp[v];
        int32_t f = P.slot_flags[v];
        if (size[P.comp[v]] > 1 || loop[P.comp[v]]) f |= 4;
        flags[v] = f;
    }
    *n_scc = P.n_scc;
    return TPGEN_OK;
}

}  // extern "C"
