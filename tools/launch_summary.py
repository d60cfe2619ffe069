"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into profiles/.

usage: python tools/launch_summary.py gpurun_out/launches.csv profiles/rNN_launches_c3.md --title "..."

A call of the hot path starts at each `dfs_kernel` launch; every launch until the
next one belongs to it.  ncu serialises launches and runs them cold-cache: the
shares, not the absolute times, are what compare with bench.py's breakdown.
"""
import argparse
import csv
import re
from collections import OrderedDict


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out_md")
    ap.add_argument("--title", default="launch list")
    ap.add_argument("--raw", default="")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    calls, cur = [], None
    for r in rows[1:]:
        name = r[ki]
        if "at::" in name:  # torch's own launches (the bench's L2 flush) are not part of the path
            continue
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        ms = float(r[vi].replace(",", "")) * scale
        short = re.sub(r"\(.*$", "", name).replace("tpg::", "")
        if "dfs_kernel" in short and (cur is None or any("expand" in k for k in cur)):
            cur = OrderedDict()
            calls.append(cur)
        if cur is None:
            continue
        cur.setdefault(short, [0.0, 0])
        cur[short][0] += ms
        cur[short][1] += 1
    md = [f"# {a.title}", "",
          "`ncu --metrics gpu__time_duration.sum --clock-control none` -- cold-cache, serialised launches: compare "
          "SHARES, not absolutes, with bench.py's CUDA-event breakdown." + (f" Raw CSV: `{a.raw}`." if a.raw else ""),
          ""]
    for i, c in enumerate(calls):
        items = list(c.items())
        tot = sum(v[0] for _, v in items)
        n = sum(v[1] for _, v in items)
        md.append(f"## call {i}: {n} launches, {tot:.3f} ms summed")
        md.append("| kernel | launches | ms | share |")
        md.append("|---|---|---|---|")
        for k, v in sorted(items, key=lambda kv: -kv[1][0]):
            md.append(f"| `{k}` | {v[1]} | {v[0]:.3f} | {100 * v[0] / tot:.1f}% |")
        md.append("")
    open(a.out_md, "w").write("\n".join(md))


if __name__ == "__main__":
    main()
