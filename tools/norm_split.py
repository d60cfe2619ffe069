import sys, json
sys.path.insert(0, '/root/repo')
import paper_2210_16998_b200 as tp
from workloads import generators as gen
h = tp.normalize_outdeg2(gen.config3())
plan = tp.Plan(h)
for i in range(2):
    st = plan.prime_paths(mode="count", digest=True).stats
    print(json.dumps({k: st[k] for k in ("ms_device", "ms_dfs_count", "ms_dfs_write", "ms_linearize", "ms_write", "ms_stitch", "n_units", "max_scc", "n_extensions")}))
