"""A/B of libtpgen build variants on config 5 COUNT_HASH (one process per variant per round,
variants interleaved over rounds): median over 5 calls of the prime-path kernel's CUDA-event
time (stats.ms_dominant) and of the call (ms_device); digest printed to check agreement.

    python tools/ab_c5.py base mulptx [--rounds 3]
"""
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
print(json.dumps({"dom": statistics.median(x["ms_dominant"] for x in s),
                  "dev": statistics.median(x["ms_device"] for x in s), "hash": s[-1]["hash_lo"] %% 100000}))
''' % ROOT


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    rounds = 3
    if "--rounds" in sys.argv:
        rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
        args = [a for a in args if a != str(rounds)]
    res = {v: [] for v in args}
    for r in range(rounds):
        for v in args:
            env = dict(os.environ)
            env.pop("TPGEN_LIB_VARIANT", None)
            if v != "base":
                env["TPGEN_LIB_VARIANT"] = v
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(v, r, line, flush=True)
            try:
                res[v].append(json.loads(line))
            except Exception:
                pass
    for v, rows in res.items():
        if rows:
            print(json.dumps({"variant": v, "dom_min": min(x["dom"] for x in rows),
                              "dom": sorted(x["dom"] for x in rows), "dev": sorted(x["dev"] for x in rows)}))


if __name__ == "__main__":
    main()
