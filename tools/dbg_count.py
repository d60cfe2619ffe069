"""Debug helper: count mode vs the oracle on the count-test corpus, one graph per line."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2210_16998_b200 as tp
from workloads import generators as gen

M64 = (1 << 64) - 1
def tot(r):
    a = r[:, :4].astype(object)
    return (int(a[:, 0].sum()), int(a[:, 1].sum()), int(a[:, 2].sum()) & M64, int(a[:, 3].sum()) & M64)

gs = [gen.fig1b(), gen.config2(), gen.k_seq_loops(3, 3), gen.k_seq_loops(5, 4), gen.config4(K=30),
      gen.parallel_sccs(3, 24, 9), gen.parallel_sccs(2, 40, 3), gen.from_arcs(2, [(0, 1)]), gen.from_arcs(3, [(0, 1), (1, 2), (2, 1)])]
rng = np.random.default_rng(11)
for i in range(60):
    n = int(rng.integers(1, 12))
    gs.append(gen.random_digraph(n, float(rng.choice([0.1, 0.2, 0.3, 0.45])), 700 + i, self_loops=bool(rng.random() < 0.5)))
which = sys.argv[1:] 
for i, g in enumerate(gs):
    if which and str(i) not in which:
        continue
    print(i, g.name, g.n, flush=True, end=" ")
    st = tp.prime_paths(g, mode="count", digest=True).stats
    ref = tot(oracle.pp_stats(g))
    got = (st["n_paths"], st["total_vertices"], st["hash_lo"], st["hash_hi"])
    ok = got == ref and st["n_extensions"] == oracle.ext_count(g)
    print("OK" if ok else f"BAD got={got[:2]} ref={ref[:2]} ext={st['n_extensions']} {oracle.ext_count(g)} hashok={got[2:]==ref[2:]}", flush=True)
