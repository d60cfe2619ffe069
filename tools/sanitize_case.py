"""Small hot-path cases for compute-sanitizer runs (memcheck / racecheck / synccheck / initcheck):
configs 1, 2 and a config-4 chain in both modes and both engines, plus the overflow-retry hooks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2210_16998_b200 as tp
from workloads import generators as gen

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("frontier_retry", "all"):
    os.environ["TPGEN_FRONTIER_CAP"] = "64"
    g = gen.dense_scc(13, 3, 11)
    print("frontier retry", tp.prime_paths(g, mode="count", digest=True, engine="frontier").stats["n_paths"])
    del os.environ["TPGEN_FRONTIER_CAP"]
if which in ("cases", "all"):
    for g in (gen.fig1b(), gen.config2(), gen.config4(K=20), gen.parallel_sccs(2, 20, 3)):
        a = tp.prime_paths(g, digest=True).stats["n_paths"]
        b = tp.prime_paths(g, mode="count", digest=True).stats["n_paths"]
        t = tp.test_paths(g, g.entry, g.exit).n_paths if g.entry >= 0 else -1
        print(g.name, a, b, t, flush=True)
    g = gen.dense_scc(10, 3, 2)
    print("frontier", tp.prime_paths(g, mode="count", digest=True, engine="frontier").stats["n_paths"])
if which in ("hooks", "all"):
    os.environ["TPGEN_TEST_QCAP"] = "16"
    os.environ["TPGEN_TEST_POOL"] = "4"
    os.environ["TPGEN_TEST_HEADCAP"] = "300"
    for g in (gen.fig1b(), gen.config2(), gen.config4(K=10)):
        a = tp.prime_paths(g, digest=True).stats["n_paths"]
        b = tp.prime_paths(g, mode="count", digest=True).stats["n_paths"]
        print("hooks", g.name, a, b, flush=True)
