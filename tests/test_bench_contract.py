"""bench.py's reference arm (the oracle as it stands, on the host's cores) prints the
contract's JSON line on CPU; argument checks of the GPU arm run before any device work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "prime_paths_per_sec" and d["unit"] == "PP/s"
    assert d["config"]["workload"].startswith("config5")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "config5 start vertices" in d["cpu_baseline"]["sample"]  # a fixed bounded sample per step
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    sys.path.insert(0, ROOT)
    import bench

    assert d["config"] == bench.bench_config(1)  # the GPU arm names the same config dict


def test_config5_sample_is_one_interior_start_per_scc():
    sys.path.insert(0, ROOT)
    import bench

    g, starts = bench.config5_sample()
    assert len(starts) == 16
    assert all(b - a == 56 for a, b in zip(starts, starts[1:]))  # one per 56-vertex SCC


def test_frontier_engine_needs_config3():
    out = subprocess.run([sys.executable, "bench.py", "--engine", "frontier", "--workload", "config5"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "config 3" in out.stderr
