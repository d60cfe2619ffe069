"""Config 3 COUNT_HASH through the frontier engine: ping-pong levels vs the DFS-chunked walk
(device-scheduled graph) at several level-buffer sizes; per-call times and chunk counts."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen
g = gen.config3()
plan = tp.Plan(g)
keys = ("ms_device", "n_paths", "hash_lo", "n_units", "n_count_rounds", "gpu_launches")
for chunk in [None] + ([int(a) for a in sys.argv[1:]] or [1 << 22]):
    if chunk:
        os.environ["TPGEN_FRONTIER_CHUNK"] = str(chunk)
    for i in range(3):
        st = plan.prime_paths(mode="count", digest=True, engine="frontier").stats
        print(json.dumps({"chunk": chunk, **{k: st[k] for k in keys}}), flush=True)
