"""Summarise the frontier engine's ncu launch list (time + DRAM bytes per launch) into profiles/.

usage: python tools/frontier_launches.py gpurun_out/launches_fr.csv profiles/rNN_launches_c3_frontier.md \
           [--traffic profiles/traffic.json]

The list comes from
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      python bench.py --engine frontier --steps 1 --warmup 0 --no-cpu-baseline --no-e2e
(one call: the root kernel and one level kernel per path length).  ncu serialises
the launches and runs them cold-cache: compare shares and per-launch GB/s, not the
absolute sum, with bench.py's CUDA-event time.  `--traffic` records the DRAM bytes of
all launches of the call (bench.py's `roofline.traffic` for `--engine frontier`).
"""
import argparse
import csv
import json
import os


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out_md")
    ap.add_argument("--traffic", default="")
    a = ap.parse_args()
    hdr, rows = None, {}
    with open(a.csv) as f:
        for r in csv.reader(f):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr is None or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            if "frontier" not in d["Kernel Name"]:
                continue
            rows.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = \
                float(d["Metric Value"].replace(",", ""))
    lines = [f"# frontier engine launch list, config 3 (`{os.path.basename(a.csv)}`)", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none`"
             " of `bench.py --engine frontier --steps 1 --warmup 0`: cold-cache, serialised launches.", "",
             "| launch | kernel | us | DRAM read MB | DRAM write MB | GB/s |", "|---|---|---|---|---|---|"]
    t_sum = b_sum = 0.0
    for i, (k, v) in enumerate(sorted(rows.items())):
        t = v.get("gpu__time_duration.sum", 0.0)  # ns
        rd, wr = v.get("dram__bytes_read.sum", 0.0), v.get("dram__bytes_write.sum", 0.0)
        t_sum += t
        b_sum += rd + wr
        name = "root" if "root" in v["name"] else f"level {i - 1}"
        lines.append(f"| {k} | {name} | {t / 1e3:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                     f"{(rd + wr) / max(t, 1.0):.0f} |")
    lines += ["", f"Sum: {len(rows)} launches, {t_sum / 1e3:.1f} us, DRAM {b_sum / 1e9:.3f} GB "
                  f"({b_sum / max(t_sum, 1.0):.0f} GB/s averaged over the call)."]
    with open(a.out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic:
        tr = json.load(open(a.traffic)) if os.path.exists(a.traffic) else {}
        tr["frontier_level_kernel"] = {"dram_bytes_per_step": b_sum, "launches_per_step": len(rows),
                                       "source": a.out_md}
        with open(a.traffic, "w") as f:
            json.dump(tr, f, indent=1)
    print("\n".join(lines[-1:]))


if __name__ == "__main__":
    main()
