"""Segment-phase donation knobs on config 5 COUNT_HASH (TPGEN_SEG_EAGER_GENS, TPGEN_SEG_SPLIT_MIN;
one process per setting): the segment phase's device time = ms_dfs_write - ms_dominant, median of 5."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, statistics, sys
sys.path.insert(0, %r)
import paper_2210_16998_b200 as tp
from workloads import generators as gen
plan = tp.Plan(gen.config5())
for _ in range(2):
    plan.prime_paths(mode="count", digest=True)
s = [plan.prime_paths(mode="count", digest=True).stats for _ in range(5)]
print(json.dumps({"seg": statistics.median(x["ms_dfs_write"] - x["ms_dominant"] for x in s),
                  "dev": statistics.median(x["ms_device"] for x in s), "hash": s[-1]["hash_lo"] %% 100000}))
''' % ROOT
for eg in ("", "8", "12", "16"):
    for sm in ("", "8", "128"):
        env = dict(os.environ)
        if eg:
            env["TPGEN_SEG_EAGER_GENS"] = eg
        if sm:
            env["TPGEN_SEG_SPLIT_MIN"] = sm
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        print(json.dumps({"eager": eg or "default", "split_min": sm or "default",
                          "res": out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-200:]}),
              flush=True)
