"""Config 5 COUNT_HASH through the frontier engine: per-call time and the level records."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen
g = gen.config5() if (len(sys.argv) < 2 or sys.argv[1] == "5") else gen.config3()
plan = tp.Plan(g)
for i in range(3):
    st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
    print(json.dumps({k: st[k] for k in ("ms_device", "ms_dfs_write", "ms_dominant", "ms_stitch", "n_paths", "hash_lo",
                                         "n_units", "n_count_rounds", "gpu_launches")}), flush=True)
