"""One config-5 COUNT_HASH call after a warm-up call (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen
g = gen.config5() if (len(sys.argv) < 2 or sys.argv[1] == "5") else gen.config3()
plan = tp.Plan(g)
for i in range(2):
    st = plan.prime_paths(mode="count", digest=True).stats
    print(st["ms_device"], st["gpu_launches"], flush=True)
