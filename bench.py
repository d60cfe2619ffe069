#!/usr/bin/env python
"""Benchmark of the TPGen hot path on B200 (contract: one JSON line on rank 0).

Default workload (BASELINE.json configs): config 3 -- one dense SCC of 22
vertices, exact out-degree 4 (seed 1): E_canon = 2.34e8 path extensions,
6.0e7 prime paths, 1.1e9 output vertices (4.9 GB).  For N > 1 the job is
weak-scaled: N disjoint copies of that SCC, rank r owns the start vertices of
copy r (no data-path collective; counts and times are reduced over NCCL).

A "step" is one full tpgen_plan_prime_paths call: DFS enumeration (segment and
prime-path phases), linearization of the unit forest, canonical writer,
cross-SCC stitching, output materialised in HBM (canonical offsets +
vertices).  `value` = prime paths / s over all ranks (device time, CUDA events,
max over ranks); `e2e` = the same through tpgen_prime_paths with the CSR in
host memory and the result copied into pinned host memory.

--workload config5: 16 parallel 56-vertex SCCs (~1.3e10 extensions) in
COUNT_HASH mode (counts + digest; the ~200 GB output is not materialized),
strong-scaled by start-vertex shards.

--impl reference runs the CPU oracle (oracle/, single core) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
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


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def workload(n_ranks: int, base=None):
    """Weak scaling: rank r enumerates the r-th of n_ranks disjoint
    copies of the config-3 graph, i.e. the start-vertex range [r*n, (r+1)*n) of
    their union; its output is that contiguous block of the union's canonical list."""
    base = gen.config3() if base is None else base
    if n_ranks == 1:
        return base, [(0, base.n)]
    g = gen.disjoint_union([base] * n_ranks, name=f"{n_ranks}x_{base.name}")
    return g, [(r * base.n, (r + 1) * base.n) for r in range(n_ranks)]


def rank_reduce(dist, world: int, n_pp: float, ext: float, ms_total: float, e2e_ms: float, device):
    """Whole-job totals: PP and extension counts summed over ranks, times maxed
    (the slowest rank defines the job time)."""
    import torch

    vals = torch.tensor([n_pp, ext, ms_total, e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        sums = vals[:2].clone()
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        mx = vals[2:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        vals = torch.cat([sums, mx])
    return vals.tolist()


# algorithmic bytes per unit of the hot path --
# 2 x (8W + 1 + 4) B per extension (frontier record written + read, W = 1)
# + (4 len + 8) B per prime path (int32 vertices + int64 offset).
def algorithmic_bytes(ext: int, n_pp: int, n_vert: int) -> float:
    """A = 2*(8W+1+4)*E_canon + sum_PP (4 len + 8)  (W = 1 here)."""
    return 2.0 * 13.0 * ext + 4.0 * n_vert + 8.0 * n_pp


def output_bytes(n_pp: int, n_vert: int) -> float:
    """What expand_kernel must write: int32 vertices + int64 offsets."""
    return 4.0 * n_vert + 8.0 * (n_pp + 1)


# ALU ceiling of the DFS enumerator: 148 SMs x 128 INT32
# lanes x SM clock / 30 lane-ops per extension ("K1 does ~10-30
# int ops per extension"; the upper figure, so the ceiling is not overstated).
ALU_LANES = 148 * 128
OPS_PER_EXT = 30.0


def ncu_traffic():
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) from the
    committed ncu --set full summary of this round (profiles/), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


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


CONFIG3_WORKLOAD = "config3: dense SCC n=22 out-degree 4 seed 1"  # the workload both arms name


def _oracle_block(s: int):
    """Worker: the oracle's prime paths of config 3's start vertex s (count, seconds)."""
    import oracle

    g, _ = workload(1)
    t = time.perf_counter()
    off, _ = oracle.prime_paths(g, v_lo=s, v_hi=s + 1)
    return len(off) - 1, time.perf_counter() - t


def _oracle_warm(_):
    import oracle  # noqa: F401  (loads liboracle.so in the worker)

    workload(1)
    return 0


class OraclePool:
    """The oracle as it stands, run on the host's cores: one process per start vertex
    of config 3 (independent per-start enumerations; no change to the oracle)."""

    def __init__(self):
        import multiprocessing as mp

        self.cores = max(1, min(os.cpu_count() or 1, 22))
        self.pool = mp.get_context("spawn").Pool(self.cores)
        self.pool.map(_oracle_warm, range(self.cores))

    def step(self):
        t = time.perf_counter()
        res = self.pool.map(_oracle_block, range(22), chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t

    def close(self):
        self.pool.close()
        self.pool.join()


def run_reference(args):
    """The CPU oracle as it stands on the host's cores; each step = all of config 3."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g, _ = workload(1)
    op = OraclePool()
    times, npp = [], 0
    for i in range(args.warmup + args.steps):
        n, dt = op.step()
        if i >= args.warmup:
            times.append(dt)
            npp = n
    op.close()
    total = sum(times)
    value = npp * len(times) / total
    sample = (f"all of config3 ({npp} prime paths per step): its 22 start vertices as independent oracle calls "
              f"(oracle/oracle.c DFS) on {op.cores} processes")
    print(json.dumps({
        "impl": "reference", "metric": "prime_paths_per_sec", "value": value, "unit": "PP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": CONFIG3_WORKLOAD, "n_vertices": g.n, "parallelism": "start-vertex shards x1",
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": "PP/s", "cores": op.cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "PP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_leg():
    import oracle

    g, _ = workload(1)
    t = time.perf_counter()
    off, _ = oracle.prime_paths(g, v_lo=0, v_hi=4)
    dt = time.perf_counter() - t
    npp = len(off) - 1
    out = {"value": npp / dt, "unit": "PP/s", "cores": 1, "kind": "oracle",
           "sample": f"config3 start vertices 0..3: {npp} prime paths in {dt:.2f} s (single core, oracle/oracle.c)"}
    try:  # the same oracle on the host's cores: all of config 3, one process per start vertex
        op = OraclePool()
        n, wall = op.step()
        op.close()
        out["all_cores"] = {"value": n / wall, "unit": "PP/s", "cores": op.cores, "kind": "oracle",
                            "sample": f"all of config3: {n} prime paths in {wall:.2f} s on {op.cores} processes"}
    except Exception as e:  # noqa: BLE001 -- the single-core figure stands on its own
        out["all_cores"] = {"unavailable": str(e)[:200]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workload", default="config3", choices=["config3", "config5"],
                    help="config3 (default, the headline): dense 22-vertex SCC, full output, weak scaling over "
                         "disjoint copies; config5: 16 parallel 56-vertex SCCs (~1.3e10 extensions), COUNT_HASH "
                         "(counts + digest; the ~200 GB output is not materialized), strong scaling by "
                         "start-vertex shards")
    ap.add_argument("--engine", default="dfs", choices=["dfs", "frontier"],
                    help="dfs (default): depth-first engine, full output; frontier: the level-synchronous "
                         "frontier engine on config 3 in COUNT_HASH mode (counts + digest; DESIGN.md 6.6)")
    ap.add_argument("--no-digest", action="store_true",
                    help="with --count / --engine frontier: counts and E_canon only (no digest)")
    ap.add_argument("--count", action="store_true",
                    help="config 3 in COUNT_HASH mode (counts + digest, no output) with the chosen engine")
    args = ap.parse_args()
    if args.engine == "frontier" and args.workload != "config3":
        ap.error("--engine frontier runs config 3 (config 5 has arcs leaving its SCCs)")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2210_16998_b200 as tp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    c5 = args.workload == "config5"
    fr = args.engine == "frontier"
    cnt3 = (fr or args.count) and not c5  # config 3, counts + digest only
    if c5:  # one graph; rank r takes start-vertex shard r of `world` (strong scaling)
        g = gen.config5()
        kw = dict(shard=(rank, world), mode="count", digest=True)
    else:
        g, ranges = workload(world)
        kw = dict(start_range=ranges[rank])
        if cnt3:
            kw.update(mode="count", digest=not args.no_digest, engine=args.engine)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    plan = tp.Plan(g, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    # ---------------- device-resident timing (value)
    for _ in range(args.warmup):
        ps = plan.prime_paths(**kw)
        del ps
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xff)  # L2 flush between timed steps (outside the events)
            ev[k][0].record(stream)
            ps = plan.prime_paths(**kw)
            ev[k][1].record(stream)
            stats.append(ps.stats)
            del ps
        torch.cuda.synchronize()
    barrier()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_total = float(sum(ms_steps))
    st = stats[-1]
    n_pp, n_vert, ext = st["n_paths"], st["total_vertices"], st["n_extensions"]
    ms_write = float(np.mean([s["ms_dfs_write"] for s in stats]))
    launches = int(sum(s["gpu_launches"] for s in stats))

    # ---------------- end-to-end through the public C ABI (host CSR in, pinned host result out)
    e2e = None
    free_b, total_b = torch.cuda.mem_get_info(dev)
    mem_used_gb = (total_b - free_b) / 1e9  # device memory held after the timed steps (pools included)
    if not args.no_e2e and (c5 or cnt3):  # counts + digest come back in the stats; the CSR goes up every call
        plan.close()  # its workspaces return to the device pool, where the e2e call's plan finds them
        h2d = int(g.offsets.nbytes + g.targets.nbytes)
        e2e_steps = max(1, min(args.steps, 3))
        del_ = tp.prime_paths(g, device=dev, **kw)
        del del_
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ps = tp.prime_paths(g, device=dev, **kw)
            del ps
        torch.cuda.synchronize()
        e2e = {"value": None, "unit": "PP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 0,
               "ms_per_step": 1e3 * (time.perf_counter() - t0) / e2e_steps, "steps": e2e_steps,
               "note": "COUNT_HASH: counts and the digest are returned in the stats struct"}
    elif not args.no_e2e:
        rng = kw["start_range"]
        host_out = torch.empty(8 * (n_pp + 1) + 4 * n_vert, dtype=torch.uint8, pin_memory=True)
        h2d = int(g.offsets.nbytes + g.targets.nbytes)
        d2h = 8 * (n_pp + 1) + 4 * n_vert
        e2e_steps = max(1, min(args.steps, 3))
        ps = tp.prime_paths(g, device=dev, output="host", host_out=host_out, start_range=rng)
        del ps
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            ps = tp.prime_paths(g, device=dev, output="host", host_out=host_out, start_range=rng)
            del ps
        torch.cuda.synchronize()
        e2e_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
        e2e = {"value": None, "unit": "PP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_ms, "steps": e2e_steps}

    # ---------------- reduce over ranks
    tot_pp, tot_ext, ms_max, e2e_ms_max = rank_reduce(dist, world, float(n_pp) * args.steps, float(ext) * args.steps,
                                                      ms_total, e2e["ms_per_step"] if e2e else 0.0, dev)

    if rank == 0:
        peak, peak_kind = measured_peaks()
        a_bytes = algorithmic_bytes(ext, n_pp, n_vert)
        o_bytes = output_bytes(n_pp, n_vert)
        value = tot_pp / (ms_max * 1e-3)
        if e2e is not None:
            e2e["value"] = (tot_pp / args.steps) / (e2e_ms_max * 1e-3)
            e2e["ms_per_step"] = e2e_ms_max
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                sm_max = float(json.load(f).get("sm_max_mhz", 1965.0))
        except Exception:
            sm_max = 1965.0
        ms_dfs = float(np.mean([s["ms_dfs_write"] for s in stats]))
        ms_expand = max(float(np.mean([s["ms_write"] for s in stats])), 1e-9)  # 0 for the frontier engine
        ms_dev = float(np.mean([s["ms_device"] for s in stats]))
        alu_peak = ALU_LANES * sm_max * 1e6 / OPS_PER_EXT / 1e9  # Gext/s
        dfs_ach = ext / (ms_dfs * 1e-3) / 1e9
        traffic = ncu_traffic()
        if c5 or cnt3:  # count mode writes no output: only the extension part of SURVEY 8(d)'s bytes applies
            a_bytes = 2.0 * 13.0 * ext
        roofline = {
            "bound": "alu", "kernel": ("dfs_kernel<unsigned long,TS=1,LEAN=0>" if c5 else "dfs_kernel<unsigned int,TS=1,LEAN=1>"),
            "achieved": dfs_ach, "peak": alu_peak, "unit": "Gext/s", "frac": dfs_ach / alu_peak,
            "traffic": traffic.get("dfs_kernel", {}).get("dram_bytes_per_launch"),
            "ms_per_launch": ms_dfs, "units_per_launch": ext,
            "peak_model": f"148 SM x 128 INT32 lanes x {sm_max:.0f} MHz / {OPS_PER_EXT:.0f} lane-ops per extension "
                          "(SURVEY 8(d)); DESIGN.md Rooflines",
            "share_of_step": ms_dfs / ms_dev,
            "second": {
                "bound": "hbm", "kernel": (f"expand_fast_kernel<{max(1, (int(st['max_scc']) + 3) // 4)},false>"
                                           if int(st["max_scc"]) <= 63 else "expand_kernel"),
                "achieved": o_bytes / (ms_expand * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": o_bytes / (ms_expand * 1e-3) / 1e9 / peak,
                "traffic": traffic.get("expand_fast_kernel" if int(st["max_scc"]) <= 63 else "expand_kernel",
                                       {}).get("dram_bytes_per_launch"),
                "algorithmic_bytes_per_launch": o_bytes, "ms_per_launch": ms_expand,
                "share_of_step": ms_expand / ms_dev,
                "model": "4 B per output vertex + 8 B per offset (written once)"},
            "path_hbm": {
                "achieved": a_bytes / (ms_dev * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": a_bytes / (ms_dev * 1e-3) / 1e9 / peak, "algorithmic_bytes": a_bytes,
                "model": "SURVEY 8(d): 26 B/extension + (4 len + 8) B/prime path, over the whole step"},
            "peak_kind": peak_kind,
            "traffic_source": traffic.get("source"),
        }
        if c5 or cnt3:
            roofline["traffic"] = None  # the committed ncu summary is for config 3
            roofline["second"] = {"note": "COUNT_HASH: the writer digests each path instead of storing it",
                                  "kernel": f"expand_fast_kernel<{max(1, (int(st['max_scc']) + 3) // 4)},true>",
                                  "ms_per_launch": ms_expand, "share_of_step": ms_expand / ms_dev}
            roofline["path_hbm"]["model"] = "SURVEY 8(d): 26 B/extension (no output in COUNT_HASH mode)"
        if fr:  # every frontier record is written once and read once: 16 B each way (8 B without digest)
            f_bytes = (16.0 if args.no_digest else 32.0) * st["n_units"]
            f_ach = f_bytes / (ms_dfs * 1e-3) / 1e9
            roofline = {
                "bound": "hbm", "kernel": "frontier_level_kernel<TS=1> (all levels + root kernel)",
                "achieved": f_ach, "peak": peak, "unit": "GB/s", "frac": f_ach / peak,
                "traffic": traffic.get("frontier_level_kernel", {}).get("dram_bytes_per_step"),
                "algorithmic_bytes_per_step": f_bytes, "records_per_step": st["n_units"],
                "ms_per_step": ms_dfs, "share_of_step": ms_dfs / ms_dev,
                "model": "16-byte path record {mask, last, first, slot base | digest sum} written once and read "
                         "once per record (DESIGN.md 6.6); traffic = DRAM bytes of all level launches of one call "
                         "(ncu launch list, profiles/traffic.json)",
                "alu_view": {"achieved": dfs_ach, "peak": alu_peak, "unit": "Gext/s", "frac": dfs_ach / alu_peak},
                "path_hbm": {"achieved": a_bytes / (ms_dev * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": a_bytes / (ms_dev * 1e-3) / 1e9 / peak, "algorithmic_bytes": a_bytes,
                             "model": "SURVEY 8(d): 26 B/extension (no output in COUNT_HASH mode)"},
                "peak_kind": peak_kind,
            }
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
            "config": {"workload": ("config5: 16 parallel SCCs n=56 out-degree 2 seed 5, COUNT_HASH (counts + "
                                    "digest, output not materialized)" if c5 else
                                    CONFIG3_WORKLOAD + (f", COUNT_HASH{' without digest' if args.no_digest else ''}, "
                                                       f"{args.engine} engine" if cnt3 else "") +
                                    (f" x{world} disjoint copies, one per rank" if world > 1 else "")),
                       "n_vertices": g.n, "prime_paths_per_rank": n_pp, "output_vertices_per_rank": n_vert,
                       "extensions_per_rank": ext, "l2": "flushed between timed steps (256 MB write, untimed)",
                       "parallelism": f"start-vertex shards x{world}"},
            "extensions_per_sec": tot_ext / (ms_max * 1e-3),
            "roofline": roofline,
            "ms_steps": {"min": float(np.min(ms_steps)), "median": float(np.median(ms_steps)),
                         "max": float(np.max(ms_steps))},
            "breakdown_ms": {"dfs_kernel": ms_dfs, "linearize": float(np.mean([s["ms_linearize"] for s in stats])),
                             "other_count": float(np.mean([s["ms_count"] - s["ms_dfs_count"] - s["ms_linearize"]
                                                           for s in stats])),
                             "expand_kernel": ms_expand,
                             "stitch": float(np.mean([s["ms_stitch"] for s in stats])), "device": ms_dev},
            "device_mem_used_gb": mem_used_gb,
            "count_rounds": st["n_count_rounds"],
            "n_units": st["n_units"],
            "gpu_launches": launches,
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_leg()
        print(json.dumps(out))
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
