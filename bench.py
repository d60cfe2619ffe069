#!/usr/bin/env python
"""Benchmark of the TPGen hot path on B200 (contract: one JSON line on rank 0).

Headline workload (BASELINE.json: "prime paths/sec + path extensions/sec (HBM GB/s
vs peak) at 1/2/4/8 B200"; configs[4] "high-Npath CFG ... sharded by start vertex at
1/2/4/8 B200"): config 5 -- Start -> d1..d16 -> J -> End with 16 random strongly
connected out-degree-2 SCCs of 56 vertices (seed 5): E_canon = 1.33e10 path
extensions, 1.51e9 prime paths.  Its output (~5.7e10 vertices, ~230 GB) exceeds one
GPU, so every step runs COUNT_HASH (counts, E_canon and the R20 digest of every prime
path, nothing written).  N ranks strong-scale it by start-vertex shards: rank r runs
shard (r, N) of the planner's cost-balanced split; `value` = prime
paths of the whole graph per second of the slowest rank (CUDA events, max over ranks).

A "step" is one tpgen_plan_prime_paths call: segment phase (SCC entry trees, records
and items), completion DP, the count-mode enumeration of every prime-path start
(cnt_kernel), head weights and the cross-SCC stitch hash.  `e2e` is the same call
through tpgen_prime_paths with the CSR in host memory, planned and uploaded anew
every step (no_plan_cache), the stats struct read back.

`secondary` (rank 0): config 3 (one dense 22-vertex SCC, out-degree 4, seed 1) with
its full output materialized in HBM (6.0e7 prime paths, 4.9 GB), the round-1 headline.

--impl reference: the CPU oracle (oracle/, as it stands) on the host's cores, each
step a fixed bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workloads import generators as gen  # noqa: E402

HBM_FALLBACK = 6650.0
ISSUE_PER_SM = 4  # warp schedulers per SM, one warp instruction per cycle each


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", float(d.get("sm_max_mhz", 1965.0))
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)", 1965.0


# algorithmic bytes per unit of the hot path --
# 2 x (8W + 1 + 4) B per extension (frontier record written + read, W = 1)
# + (4 len + 8) B per prime path when the output is materialized.
BYTES_PER_EXT = 2.0 * (8 + 1 + 4)


def output_bytes(n_pp: int, n_vert: int) -> float:
    """What the canonical writer must write: int32 vertices + int64 offsets."""
    return 4.0 * n_vert + 8.0 * (n_pp + 1)


def ncu_traffic():
    """Per-launch DRAM bytes and instruction counts (ncu --set full summaries of this round,
    profiles/traffic.json), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):  # diagnosis only: the contract's runs always sample
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) stalls the device: let it finish before the timed region
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.02)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
                for nm, v in zip(names, r[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


CONFIG5_WORKLOAD = ("config5: Start->d1..d16->J->End, 16 random strongly connected out-degree-2 SCCs of 56 "
                    "vertices, seed 5")
CONFIG3_WORKLOAD = "config3: dense SCC n=22 out-degree 4 seed 1"


def bench_config(world: int) -> dict:
    """The workload both arms name (identical dict in the GPU arm and the reference arm)."""
    g = gen.config5()
    return {"workload": CONFIG5_WORKLOAD, "n_vertices": g.n, "n_arcs": int(g.offsets[-1]),
            "mode": "COUNT_HASH: prime-path count, vertices, E_canon and the R20 digest (the ~230 GB output is "
                    "not materialized)",
            "l2": "flushed between timed steps (256 MB write, untimed)",
            "parallelism": f"start-vertex shards x{world} (strong scaling)"}


def config5_sample():
    """The bounded oracle sample of config 5: one start vertex per 56-vertex SCC -- its first
    vertex that is not an SCC entry -- i.e. 16 independent per-start enumerations.  SCC labels
    come from the oracle (the reference arm never loads the CUDA library)."""
    import oracle

    g = gen.config5()
    so, st = np.asarray(g.offsets), np.asarray(g.targets)
    src = np.repeat(np.arange(g.n), np.diff(so))
    lab = oracle.scc_labels(g)
    sizes = np.bincount(lab, minlength=g.n)
    entry = np.zeros(g.n, dtype=bool)
    entry[st[lab[src] != lab[st]]] = True  # a predecessor outside its SCC (Def. 4)
    starts, seen = [], set()
    for v in range(g.n):
        if sizes[lab[v]] > 1 and not entry[v] and lab[v] not in seen:
            seen.add(int(lab[v]))
            starts.append(v)
    return g, starts


def _sample_worker(v: int):
    import oracle

    g = gen.config5()
    t = time.perf_counter()
    row = oracle.pp_stats(g, v, v + 1)[0]
    return int(row[0]), int(row[1]), time.perf_counter() - t


def _warm(_):
    import oracle  # noqa: F401

    gen.config5()
    return 0


class OraclePool:
    """The oracle as it stands on the host's cores: one process per sampled start vertex."""

    def __init__(self, n: int):
        import multiprocessing as mp

        self.cores = max(1, min(os.cpu_count() or 1, n))
        self.pool = mp.get_context("spawn").Pool(self.cores)
        self.pool.map(_warm, range(self.cores))

    def run(self, starts):
        t = time.perf_counter()
        res = self.pool.map(_sample_worker, starts, chunksize=1)
        return sum(r[0] for r in res), sum(r[1] for r in res), time.perf_counter() - t

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    """The CPU oracle on the host's cores; each step = the bounded config-5 sample."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    g, starts = config5_sample()
    op = OraclePool(len(starts))
    times, npp = [], 0
    for i in range(args.warmup + args.steps):
        n, _, dt = op.run(starts)
        if i >= args.warmup:
            times.append(dt)
            npp = n
    op.close()
    total = sum(times)
    value = npp * len(times) / total
    sample = (f"config5 start vertices {starts} (one interior vertex per SCC; {npp} prime paths per step, counted "
              f"and hashed by oracle_pp_stats) on {op.cores} processes")
    print(json.dumps({
        "impl": "reference", "metric": "prime_paths_per_sec", "value": value, "unit": "PP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": bench_config(world),
        "cpu_baseline": {"value": value, "unit": "PP/s", "cores": op.cores, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "PP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_leg():
    """The oracle (oracle_pp_stats, as it stands) on a bounded sample of config 5: 4 sampled start
    vertices on one core, then the 16-vertex sample on the host's cores."""
    import oracle

    g, starts = config5_sample()
    t = time.perf_counter()
    n1 = 0
    for v in starts[:4]:
        n1 += int(oracle.pp_stats(g, v, v + 1)[0][0])
    dt = time.perf_counter() - t
    out = {"value": n1 / dt, "unit": "PP/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
           "sample": f"config5 start vertices {starts[:4]}: {n1} prime paths counted and hashed in {dt:.2f} s "
                     f"(one core, oracle/oracle.c oracle_pp_stats)"}
    try:
        op = OraclePool(len(starts))
        n, _, wall = op.run(starts)
        op.close()
        out["all_cores"] = {"value": n / wall, "unit": "PP/s", "cores": op.cores, "kind": "oracle",
                            "sample": f"config5 start vertices {starts}: {n} prime paths in {wall:.2f} s on "
                                      f"{op.cores} processes"}
    except Exception as e:  # noqa: BLE001 -- the single-core figure stands on its own
        out["all_cores"] = {"unavailable": str(e)[:200]}
    return out


def rank_reduce(dist, world: int, sums, maxes, device):
    """The job's totals: per-rank counts summed, per-rank times maxed (the slowest rank defines
    the job time).  One all_reduce each (NCCL on the GPU, gloo in the CPU tests)."""
    import torch

    s = torch.tensor([float(x) for x in sums], dtype=torch.float64, device=device)
    m = torch.tensor([float(x) for x in maxes], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return s.tolist(), m.tolist()


def timed_steps(plan, kw, steps, warmup, stream, flush):
    """W untimed calls, then K calls bracketed by CUDA events on the call's stream, L2 flushed
    (untimed) before each.  Returns (per-step ms, per-step stats)."""
    import torch

    for _ in range(warmup):
        ps = plan.prime_paths(**kw)
        del ps
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    stats = []
    for k in range(steps):
        flush.fill_(k & 0xff)
        ev[k][0].record(stream)
        ps = plan.prime_paths(**kw)
        ev[k][1].record(stream)
        stats.append(ps.stats)
        del ps
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev], stats


def mean(stats, key):
    return float(np.mean([s[key] for s in stats]))


def dominant_roofline(stats, kernel: str, traffic_key: str, peak: float, peak_kind: str, sm_max: float):
    """SURVEY 8(d) roofline of the dominant launch: 26 B per extension it made (frontier record
    written + read, W = 1) / its CUDA-event duration, against the measured HBM copy peak; the
    issue-slot view next to it (warp instructions per extension from the committed ncu capture)."""
    traffic = ncu_traffic().get(traffic_key, {})
    ms = mean(stats, "ms_dominant")
    ext = mean(stats, "ext_dominant")
    achieved = BYTES_PER_EXT * ext / (ms * 1e-3) / 1e9
    r = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
         "frac": achieved / peak, "traffic": traffic.get("dram_bytes_per_launch"),
         "algorithmic_bytes_per_launch": BYTES_PER_EXT * ext, "extensions_per_launch": ext,
         "ms_per_launch": ms, "share_of_step": ms / mean(stats, "ms_device"),
         "model": "SURVEY 8(d): 2 x (8W+1+4) = 26 B per extension (W = 1); achieved = that x the launch's "
                  "extensions / its CUDA-event time", "peak_kind": peak_kind,
         "traffic_source": traffic.get("source")}
    ipe = traffic.get("warp_inst_per_ext")
    if ipe:
        ceil = 148 * ISSUE_PER_SM * sm_max * 1e6 / ipe / 1e9
        ach = ext / (ms * 1e-3) / 1e9
        r["alu_view"] = {"bound": "issue", "achieved": ach, "unit": "Gext/s", "peak": ceil, "frac": ach / ceil,
                         "warp_inst_per_ext": ipe,
                         "model": f"148 SM x {ISSUE_PER_SM} schedulers x {sm_max:.0f} MHz warp-instruction issue / "
                                  f"the launch's warp instructions per extension (ncu smsp__inst_executed.sum)"}
    return r


def secondary_config3(dev, steps, warmup, flush, peak, peak_kind, sm_max, no_e2e):
    """Config 3 with its whole output materialized (rank 0; the round-1 headline)."""
    import torch

    import paper_2210_16998_b200 as tp

    g = gen.config3()
    plan = tp.Plan(g, device=dev)
    stream = torch.cuda.current_stream(dev)
    ms_steps, stats = timed_steps(plan, {}, steps, warmup, stream, flush)
    plan.close()
    st = stats[-1]
    n_pp, n_vert = st["n_paths"], st["total_vertices"]
    ms = float(np.mean(ms_steps))
    o_bytes = output_bytes(n_pp, n_vert)
    ms_w = mean(stats, "ms_write")
    rl = dominant_roofline(stats, "dfs_kernel<uint32,TS=1,LEAN=1> (records)", "dfs_kernel_c3", peak, peak_kind,
                           sm_max)
    rl["second"] = {"bound": "hbm", "kernel": "expand_fast_kernel<6,false>",
                    "achieved": o_bytes / (ms_w * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": o_bytes / (ms_w * 1e-3) / 1e9 / peak, "algorithmic_bytes_per_launch": o_bytes,
                    "ms_per_launch": ms_w, "traffic": ncu_traffic().get("expand_fast_kernel", {}).get(
                        "dram_bytes_per_launch"), "model": "4 B per output vertex + 8 B per offset (written once)"}
    a_bytes = BYTES_PER_EXT * st["n_extensions"] + output_bytes(n_pp, n_vert)
    out = {"workload": CONFIG3_WORKLOAD + ", full output materialized in HBM (canonical offsets + vertices)",
           "metric": "prime_paths_per_sec", "value": n_pp / (ms * 1e-3), "unit": "PP/s", "ms_per_step": ms,
           "steps": steps, "prime_paths": n_pp, "output_vertices": n_vert, "extensions": st["n_extensions"],
           "extensions_per_sec": st["n_extensions"] / (ms * 1e-3), "roofline": rl,
           "path_hbm": {"achieved": a_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": a_bytes / (ms * 1e-3) / 1e9 / peak, "algorithmic_bytes": a_bytes,
                        "model": "SURVEY 8(d): 26 B/extension + (4 len + 8) B/prime path, whole step"},
           "breakdown_ms": {"dfs_kernel": mean(stats, "ms_dfs_write"), "linearize": mean(stats, "ms_linearize"),
                            "expand_kernel": ms_w, "device": mean(stats, "ms_device")},
           "presplit": "host pre-split trie tops cached per plan (planned once, outside the timed steps); e2e "
                       "re-plans every call",
           "gpu_launches": int(sum(s["gpu_launches"] for s in stats))}
    if not no_e2e:
        host_out = torch.empty(8 * (n_pp + 1) + 4 * n_vert, dtype=torch.uint8, pin_memory=True)
        ps = tp.prime_paths(g, device=dev, output="host", host_out=host_out, plan_cache=False)
        del ps
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = 3
        for _ in range(k):
            ps = tp.prime_paths(g, device=dev, output="host", host_out=host_out, plan_cache=False)
            del ps
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t0) / k
        out["e2e"] = {"value": n_pp / (e2e_ms * 1e-3), "unit": "PP/s", "ms_per_step": e2e_ms, "steps": k,
                      "h2d_bytes_per_step": int(g.offsets.nbytes + g.targets.nbytes),
                      "d2h_bytes_per_step": int(8 * (n_pp + 1) + 4 * n_vert),
                      "note": "planned and uploaded anew every call; output copied into pinned host memory"}
    return out


def engine_comparison(dev, flush):
    """Config 3 COUNT_HASH (counts, E_canon, digest) through the three engines -- the count-mode
    DFS, the level-synchronous frontier and the paper's vertex-centric Alg. 3
    -- device ms per call (median of 3 after one warm-up, L2 flushed between calls) and whether
    all three agree (rank 0, informational; not the headline)."""
    import torch

    import paper_2210_16998_b200 as tp

    g = gen.config3()
    plan = tp.Plan(g, device=dev)
    out, keys = {}, set()
    for eng in ("dfs", "frontier", "alg3"):
        ms = []
        for i in range(4):
            flush.fill_(i & 0xff)
            torch.cuda.synchronize(dev)
            st = plan.prime_paths(mode="count", digest=True, engine=eng).stats
            if i:
                ms.append(st["ms_device"])
        keys.add((st["n_paths"], st["total_vertices"], st["n_extensions"], st["hash_lo"], st["hash_hi"]))
        out[eng] = {"ms_per_call": float(np.median(ms)), "pp_per_sec": st["n_paths"] / (np.median(ms) * 1e-3),
                    "gpu_launches": int(st["gpu_launches"])}
    plan.close()
    out["agree"] = len(keys) == 1
    out["workload"] = CONFIG3_WORKLOAD + ", COUNT_HASH"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config-3 materialized record")
    ap.add_argument("--workload", default="config5", choices=["config5", "config3"],
                    help="config5 (default, the headline; see the module docstring); config3: the dense 22-vertex "
                         "SCC as the main line (weak scaling over disjoint copies), materialized or --count")
    ap.add_argument("--engine", default="dfs", choices=["dfs", "frontier"],
                    help="dfs (default); frontier: the level-synchronous frontier engine (config 3, COUNT_HASH)")
    ap.add_argument("--no-digest", action="store_true", help="COUNT_HASH without the digest (counts only)")
    ap.add_argument("--count", action="store_true", help="config 3 in COUNT_HASH mode")
    args = ap.parse_args()
    if args.engine == "frontier" and args.workload != "config3":
        ap.error("--engine frontier runs config 3 (config 5 has arcs leaving its SCCs)")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2210_16998_b200 as tp
    from paper_2210_16998_b200 import _abi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    peak, peak_kind, sm_max = measured_peaks()
    c5 = args.workload == "config5"
    if c5:
        g = gen.config5()
        kw = dict(shard=(rank, world), mode="count", digest=not args.no_digest)
        config = bench_config(world)
    else:
        base = gen.config3()
        g = base if world == 1 else gen.disjoint_union([base] * world, name=f"{world}x_{base.name}")
        kw = dict(start_range=(rank * base.n, (rank + 1) * base.n))
        if args.count or args.engine == "frontier":
            kw.update(mode="count", digest=not args.no_digest, engine=args.engine)
        config = {"workload": CONFIG3_WORKLOAD + (f" x{world} disjoint copies, one per rank" if world > 1 else ""),
                  "n_vertices": g.n, "mode": ("COUNT_HASH" if kw.get("mode") == "count" else "materialize") +
                  f", {args.engine} engine", "l2": "flushed between timed steps (256 MB write, untimed)",
                  "parallelism": f"start-vertex ranges x{world} (weak scaling)"}
    stream = torch.cuda.current_stream(dev)
    plan = tp.Plan(g, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        ms_steps, stats = timed_steps(plan, kw, args.steps, args.warmup, stream, flush)
    if world > 1:
        dist.barrier()
    plan.close()
    ms_total = float(sum(ms_steps))
    st = stats[-1]
    n_pp, n_vert, ext = st["n_paths"], st["total_vertices"], st["n_extensions"]
    free_b, total_b = torch.cuda.mem_get_info(dev)

    # ---------------- end to end through the public C ABI: host CSR in, planned and uploaded anew
    e2e = None
    if not args.no_e2e:
        e2e_kw = dict(kw)
        host_out = None
        if kw.get("mode") != "count":
            host_out = torch.empty(8 * (n_pp + 1) + 4 * n_vert, dtype=torch.uint8, pin_memory=True)
            e2e_kw.update(output="host", host_out=host_out)
        ps = tp.prime_paths(g, device=dev, plan_cache=False, **e2e_kw)
        del ps
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        k = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(k):
            ps = tp.prime_paths(g, device=dev, plan_cache=False, **e2e_kw)
            del ps
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t0) / k
        d2h = ctypes.sizeof(_abi.Stats) if host_out is None else int(8 * (n_pp + 1) + 4 * n_vert)
        e2e = {"value": None, "unit": "PP/s", "h2d_bytes_per_step": int(g.offsets.nbytes + g.targets.nbytes),
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": k,
               "note": "tpgen_prime_paths with the CSR in host memory, planned and uploaded anew every call "
                       "(no_plan_cache = 1); " + ("counts and digest returned in the stats struct" if host_out is None
                                                  else "output copied into pinned host memory")}

    # ---------------- reduce over ranks: counts summed, times maxed (the slowest rank defines the job)
    (tot_pp, tot_ext, pp_per_step), (ms_max, e2e_max) = rank_reduce(
        dist, world, [float(n_pp) * args.steps, float(ext) * args.steps, float(n_pp)],
        [ms_total, e2e["ms_per_step"] if e2e else 0.0], dev)

    if rank == 0:
        value = tot_pp / (ms_max * 1e-3)
        if e2e is not None:
            e2e["value"] = pp_per_step / (e2e_max * 1e-3)
            e2e["ms_per_step"] = e2e_max
        ms_dev = mean(stats, "ms_device")
        if c5:
            roofline = dominant_roofline(stats, "cnt_kernel<uint64,TS=1,HSH=1,HX=1> (count-mode DFS, prime-path "
                                                "phase)", "cnt_kernel_c5", peak, peak_kind, sm_max)
        elif kw.get("engine") == "frontier":
            roofline = dominant_roofline(stats, "frontier_level_kernel (all levels of the call)", "frontier", peak,
                                         peak_kind, sm_max)
        elif kw.get("mode") == "count":
            roofline = dominant_roofline(stats, "cnt_kernel<uint32,TS=1,HSH=1,HX=0>", "cnt_kernel_c3", peak,
                                         peak_kind, sm_max)
        else:
            roofline = dominant_roofline(stats, "dfs_kernel<uint32,TS=1,LEAN=1> (records)", "dfs_kernel_c3", peak,
                                         peak_kind, sm_max)
        a_bytes = BYTES_PER_EXT * ext + (0.0 if kw.get("mode") == "count" else output_bytes(n_pp, n_vert))
        roofline["path_hbm"] = {"achieved": a_bytes / (ms_dev * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                "frac": a_bytes / (ms_dev * 1e-3) / 1e9 / peak, "algorithmic_bytes": a_bytes,
                                "model": "SURVEY 8(d) bytes of the whole step (rank 0's shard)"}
        out = {
            "metric": "prime_paths_per_sec",
            "value": value,
            "unit": "PP/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if c5 else "weak",
            "vs_baseline": None,
            "dtype": "int32",
            "data": "synthetic",
            "config": config,
            "extensions_per_sec": tot_ext / (ms_max * 1e-3),
            "counts": {"prime_paths": int(pp_per_step), "prime_paths_rank0": n_pp, "output_vertices_rank0": n_vert,
                       "extensions_rank0": ext, "cross_scc_rank0": st["n_cross"],
                       "digest_rank0": [st["hash_lo"], st["hash_hi"]], "shard_rank0": [st["shard_lo"], st["shard_hi"]]},
            "roofline": roofline,
            "ms_steps": {"min": float(np.min(ms_steps)), "median": float(np.median(ms_steps)),
                         "max": float(np.max(ms_steps))},
            "breakdown_ms": {"dominant": mean(stats, "ms_dominant"), "dfs_phases": mean(stats, "ms_dfs_write"),
                             "linearize": mean(stats, "ms_linearize"), "writer": mean(stats, "ms_write"),
                             "stitch": mean(stats, "ms_stitch"), "device": ms_dev},
            "device_mem_used_gb": (total_b - free_b) / 1e9,
            "count_rounds": st["n_count_rounds"],
            "gpu_launches": int(sum(s["gpu_launches"] for s in stats)),
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        if c5 and not args.no_secondary:
            out["secondary"] = secondary_config3(dev, min(args.steps, 10), max(args.warmup, 3), flush, peak,
                                                 peak_kind, sm_max, args.no_e2e)
            out["engines_config3"] = engine_comparison(dev, flush)
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_leg()
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
