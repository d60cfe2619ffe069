"""Config 3 COUNT_HASH through the three engines -- the paper's Alg. 3 (vertex-centric,
self-stabilizing), the frontier and the DFS -- on the original graph and on its out-degree-2
normalization (Fig. 5): per-call device ms (median of 5 after 2 warm-ups), records, checks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2210_16998_b200 as tp
from workloads import generators as gen

g = gen.config3()
for name, gr in (("config3", g), ("config3-outdeg2", tp.normalize_outdeg2(g))):
    plan = tp.Plan(gr)
    ref = None
    for eng in ("alg3", "frontier", "dfs"):
        if eng == "frontier" and gr.n > 64:
            continue
        ms = []
        for i in range(7):
            st = plan.prime_paths(mode="count", digest=True, engine=eng).stats
            ms.append(st["ms_device"])
        key = (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"], st["n_extensions"])
        ref = ref or key
        print(json.dumps({"graph": name, "n": gr.n, "engine": eng, "ms_device": float(np.median(ms[2:])),
                          "ms_all": [round(x, 3) for x in ms], "n_paths": st["n_paths"], "n_extensions": st["n_extensions"],
                          "records": st["n_units"], "equal": key == ref}), flush=True)
    plan.close()
