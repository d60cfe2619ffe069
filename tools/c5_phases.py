"""Config 5 COUNT_HASH with TPGEN_DEBUG=1: per-phase DFS times and the stage marks (stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen
g = gen.config5()
plan = tp.Plan(g)
for i in range(3):
    st = plan.prime_paths(mode="count", digest=True).stats
    print({k: st[k] for k in ("ms_device", "ms_dfs_write", "ms_dominant", "ms_stitch", "n_heads", "n_segments",
                              "n_cross", "n_units", "n_count_rounds")}, flush=True)
