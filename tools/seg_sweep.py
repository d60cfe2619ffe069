"""Config 5 COUNT_HASH: the segment phase's time (ms_dfs_write - ms_dominant) and the prime-path
phase's under the donation knobs in the environment (one line per call)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen
plan = tp.Plan(gen.config5())
for i in range(3):
    st = plan.prime_paths(mode="count", digest=True).stats
    if i:
        print(json.dumps({"knobs": {k: v for k, v in os.environ.items() if k.startswith("TPGEN_")},
                          "seg_ms": round(st["ms_dfs_write"] - st["ms_dominant"], 3), "pp_ms": round(st["ms_dominant"], 3),
                          "device_ms": round(st["ms_device"], 3), "hash": st["hash_lo"] % 1000}), flush=True)
