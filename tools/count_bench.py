"""Times COUNT_HASH calls (Plan API, CUDA events inside the library) on configs 3 and 5:
the count-mode DFS against the record path (TPGEN_NO_CNT=1 in a second process)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2210_16998_b200 as tp  # noqa: E402
from workloads import generators as gen  # noqa: E402


def main():
    which = sys.argv[1:] or ["config3", "config5"]
    for name in which:
        g = gen.config3() if name == "config3" else gen.config5()
        plan = tp.Plan(g)
        for digest in (True, False):
            rows = []
            for i in range(4):
                t = time.perf_counter()
                st = plan.prime_paths(mode="count", digest=digest).stats
                wall = time.perf_counter() - t
                rows.append((st["ms_device"], st["ms_dfs_write"], st["ms_write"], st["ms_stitch"], wall * 1e3))
            st = dict(st)
            print(json.dumps({"workload": name, "digest": digest, "cnt": not os.environ.get("TPGEN_NO_CNT"),
                              "ms_device": [round(r[0], 3) for r in rows], "ms_dfs": [round(r[1], 3) for r in rows],
                              "ms_write": rows[-1][2], "ms_stitch": rows[-1][3], "ms_wall": round(rows[-1][4], 2),
                              "n_paths": st["n_paths"], "n_ext": st["n_extensions"], "n_cross": st["n_cross"],
                              "n_heads": st["n_heads"], "hash": [st["hash_lo"], st["hash_hi"]],
                              "ext_per_s": st["n_extensions"] / (rows[-1][0] * 1e-3)}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
