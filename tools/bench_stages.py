"""Secondary measurements: the cross-SCC stitching and the test-path
stage (a6) on the stitching-heavy configs, with CUDA events on the current stream.

usage: python tools/bench_stages.py [--steps 10] [--warmup 3]   (one JSON line per workload)

bench.py times the headline workload (config 3, a single SCC: no stitching).  Here:
  config2        structured CFG ~60 vertices (latency-bound: microseconds)
  config4        chain of 150 while loops, depth-1 bodies (95 % cross-SCC prime paths)
  config4_d2     the same with depth-2 loop bodies (9.9e6 prime paths, 4.1e9 output vertices; PPs only)
Each step: Plan.prime_paths (materialized) then test_paths on the result.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_16998_b200 as tp  # noqa: E402
from workloads import generators as gen  # noqa: E402


def run(name, g, steps, warmup, with_tp=True, greedy=True):
    plan = tp.Plan(g)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        ps = plan.prime_paths()
        ts = plan.test_paths(g.entry, g.exit, ps) if with_tp else None
        del ps, ts
    torch.cuda.synchronize()
    rec = []
    for _ in range(steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        ps = plan.prime_paths()
        e[1].record(stream)
        ts = plan.test_paths(g.entry, g.exit, ps) if with_tp else None
        e[2].record(stream)
        torch.cuda.synchronize()
        rec.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), ps.stats,
                    ts.stats if ts is not None else None))
        del ps, ts
    pp_ms = float(np.median([r[0] for r in rec]))
    tp_ms = float(np.median([r[1] for r in rec]))
    st, tst = rec[-1][2], rec[-1][3]
    out_b = 4.0 * st["total_vertices"] + 8.0 * (st["n_paths"] + 1)
    res = {
        "workload": name, "n_vertices": g.n, "n_sccs": st["n_scc"], "max_scc": st["max_scc"],
        "prime_paths": st["n_paths"], "cross_scc": st["n_cross"], "output_vertices": st["total_vertices"],
        "E_canon": st["n_extensions"], "pp_ms": pp_ms, "pp_per_sec": st["n_paths"] / (pp_ms * 1e-3),
        "stitch_ms": float(np.median([r[2]["ms_stitch"] for r in rec])),
        "pp_output_gbs": out_b / (pp_ms * 1e-3) / 1e9,
    }
    if with_tp and greedy:
        gt = []
        for _ in range(max(1, steps // 2)):
            ps = plan.prime_paths()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gs = plan.test_paths(g.entry, g.exit, ps, cover="greedy")
            e1.record(stream)
            torch.cuda.synchronize()
            gt.append(e0.elapsed_time(e1))
            res_g = gs.stats
            del ps, gs
        res["greedy_ms"] = float(np.median(gt))
        res["greedy_test_paths"] = res_g["n_paths"]
        res["greedy_vertices"] = res_g["total_vertices"]
    if tst is not None:
        tp_b = 4.0 * tst["total_vertices"] + 8.0 * (tst["n_paths"] + 1)
        res.update({"tp_ms": tp_ms, "test_path_vertices": tst["total_vertices"],
                    "tp_output_gbs": tp_b / (tp_ms * 1e-3) / 1e9,
                    "note": "median of steps; tp_ms = Plan.test_paths (host walk trees + device tables and writer)"})
    plan.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    print(json.dumps(run("config2", gen.config2(), a.steps, a.warmup)))
    print(json.dumps(run("config4", gen.config4(), a.steps, a.warmup)))
    # depth-2 bodies: 9.9e6 prime paths, 4.1e9 output vertices (16 GB); its test paths would be ~80 GB
    print(json.dumps(run("config4_d2", gen.loop_chain(150, 0, body_depth=2), a.steps, a.warmup, with_tp=False)))


if __name__ == "__main__":
    main()
