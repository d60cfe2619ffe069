import sys; sys.path.insert(0, '/root/repo')
import paper_2210_16998_b200 as tp
from workloads import generators as gen
for g in (gen.config2(), gen.config4(K=30), gen.k_seq_loops(5,4)):
    a = tp.prime_paths(g, mode="count", digest=True).stats
    b = tp.prime_paths(g, mode="count", digest=False).stats
    c = tp.prime_paths(g, mode="count", digest=False).stats
    print(g.name, {k: (a[k], b[k], c[k]) for k in ("n_paths", "n_cross", "n_heads", "n_units", "n_count_rounds", "n_segments")})
