"""Shard balance of config 3 on one GPU: start-vertex shards vs prefix-unit shards
(tpgen_options.shard_prefix), each shard of N run one after another on the same device.
Per shard: E_canon and the device time (stats.ms_device, CUDA events; median of 5 calls);
the max / mean of both is what a 1 -> N strong-scaling run would lose to imbalance.

    python tools/pfx_balance.py [--mode materialize|count] [--world 2 4 8]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2210_16998_b200 as tp
from workloads import generators as gen


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="materialize")
    ap.add_argument("--world", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    g = gen.config3()
    plan = tp.Plan(g)
    dig = a.mode == "count"
    for _ in range(3):
        plan.prime_paths(mode=a.mode, digest=dig)
    whole = [plan.prime_paths(mode=a.mode, digest=dig).stats["ms_device"] for _ in range(a.reps)]
    out = {"workload": "config3", "mode": a.mode, "whole_ms": statistics.median(whole), "world": {}}
    for world in a.world:
        row = {}
        for pfx in (False, True):
            ext, ms = [], []
            for r in range(world):
                for _ in range(2):
                    plan.prime_paths(mode=a.mode, digest=dig, shard=(r, world), shard_prefix=pfx)
                t = []
                for _ in range(a.reps):
                    st = plan.prime_paths(mode=a.mode, digest=dig, shard=(r, world), shard_prefix=pfx).stats
                    t.append(st["ms_device"])
                ext.append(st["n_extensions"])
                ms.append(statistics.median(t))
            row["prefix" if pfx else "start"] = {
                "ext_max_over_mean": max(ext) / (sum(ext) / world),
                "ms_max": max(ms), "ms_sum": sum(ms),
                "ms_max_over_mean": max(ms) / (sum(ms) / world),
                "speedup_vs_whole": out["whole_ms"] / max(ms),
                "ms": [round(x, 3) for x in ms]}
        out["world"][world] = row
    print(json.dumps(out))
    plan.close()


if __name__ == "__main__":
    main()
