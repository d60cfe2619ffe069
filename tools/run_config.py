"""Runs the hot path on one config a few times (for ncu / launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_16998_b200 as tp  # noqa: E402
from workloads import generators as gen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="materialize", choices=["materialize", "count"])
ap.add_argument("--digest", action="store_true")
a = ap.parse_args()
g = gen.make_config(a.config)
plan = tp.Plan(g)
for _ in range(a.reps):
    ps = plan.prime_paths(mode=a.mode, digest=a.digest)
    print({k: ps.stats[k] for k in ("n_paths", "n_extensions", "ms_device", "ms_dfs_write", "ms_dominant",
                                     "ext_dominant", "n_count_rounds", "n_units")})
    del ps
torch.cuda.synchronize()
