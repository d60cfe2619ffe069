"""NEXT #2 reachability pruning on the GPU (tpgen_options.prune) against the unpruned
count-mode DFS: configs 3 and 5 COUNT_HASH, device time (stats.ms_device, CUDA events) and
the prime-path phase's kernel (ms_dominant), median of 5 calls after 2 warm-ups; extensions
made with and without pruning.

    python tools/prune_bench.py
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2210_16998_b200 as tp  # noqa: E402
from workloads import generators as gen  # noqa: E402


def run(plan, prune, reps=5):
    for _ in range(2):
        plan.prime_paths(mode="count", digest=True, prune=prune)
    sts = [plan.prime_paths(mode="count", digest=True, prune=prune).stats for _ in range(reps)]
    return {"ms_device": statistics.median(s["ms_device"] for s in sts),
            "ms_dominant": statistics.median(s["ms_dominant"] for s in sts),
            "n_extensions": sts[-1]["n_extensions"], "n_paths": sts[-1]["n_paths"],
            "digest": [sts[-1]["hash_lo"], sts[-1]["hash_hi"]]}


def main():
    out = {}
    for name in ("config3", "config5"):
        g = getattr(gen, name)()
        plan = tp.Plan(g)
        a, b = run(plan, False), run(plan, True)
        assert (a["n_paths"], a["digest"]) == (b["n_paths"], b["digest"])
        out[name] = {"unpruned": a, "pruned": b, "ext_ratio": b["n_extensions"] / a["n_extensions"],
                     "time_ratio": b["ms_device"] / a["ms_device"]}
        plan.close()
        print(json.dumps({name: out[name]}), flush=True)


if __name__ == "__main__":
    main()
