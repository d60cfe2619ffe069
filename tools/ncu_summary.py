"""Summarise an `ncu --set full` report into profiles/ (markdown + traffic.json).

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/rNN_ncu_full_c3.md [--traffic profiles/traffic.json]

Reads the report with `ncu -i ... --page raw --csv` and `--page source --csv`
(run here, no GPU needed) and writes, per profiled kernel: duration, DRAM bytes
read/written (the roofline `traffic`), issue/occupancy/warp-efficiency figures
and the top source lines by instructions executed and by stall samples.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp-instruction"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles per issued instruction"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps per scheduler"),
    ("sm__inst_executed.sum", "warp instructions executed"),
    ("launch__registers_per_thread", "registers per thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def ncu_csv(rep: str, *args: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_rows(rep: str):
    rows = ncu_csv(rep, "--page", "raw")
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        res.append(d)
    return res


def source_lines(rep: str, kernel_regex: str, top: int = 12):
    rows = ncu_csv(rep, "--page", "source", "--print-source=cuda,sass", "-k", f"regex:{kernel_regex}")
    f = None
    ln = None
    agg = {}
    hdr = None
    for r in rows:
        if r and r[0] == "File Path":
            f = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 9 or r[:1] == ["Function Name"]:
            continue
        if r[0] != "":
            ln = (f, int(r[0]))
            agg.setdefault(ln, [r[1].strip(), 0, 0])
            continue
        if ln is None:
            continue
        agg[ln][1] += int(r[7]) if r[7].isdigit() else 0
        agg[ln][2] += int(r[4]) if r[4].isdigit() else 0
    ti = sum(v[1] for v in agg.values()) or 1
    ts = sum(v[2] for v in agg.values()) or 1
    by_i = sorted(agg.items(), key=lambda x: -x[1][1])[:top]
    by_s = sorted(agg.items(), key=lambda x: -x[1][2])[:top]
    return ti, ts, by_i, by_s


def fnum(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out_md")
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    rows = raw_rows(a.rep)
    md = [f"# {a.title or os.path.basename(a.out_md)}", "",
          f"Source report: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none --import-source on`, "
          "one GPU). Numbers under ncu are replayed and serialised: use them for shares, bytes and stall reasons, "
          "never as bench values.", ""]
    traffic = {}
    seen = {}
    for d in rows:
        name = d.get("Kernel Name", "?")
        short = name.split("(")[0].replace("void ", "")
        base = short.split("<")[0]
        seen[base] = seen.get(base, 0) + 1
        md.append(f"## {short} (launch {d.get('ID')})")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for key, label in RAW:
            if key in d:
                unit = ""
                md.append(f"| {label} (`{key}`) | {d[key]} {unit}|")
        rd = fnum(d.get("dram__bytes_read.sum", "nan"))
        wr = fnum(d.get("dram__bytes_write.sum", "nan"))
        md.append("")
        # raw page units: bytes columns come in the unit given by the second header row; normalise via ncu's own
        traffic.setdefault(base, {"launches": []})["launches"].append({"read": rd, "write": wr})
        try:
            ti, ts, by_i, by_s = source_lines(a.rep, base)
            md.append(f"Top source lines by warp instructions executed (total {ti:,}):")
            md.append("")
            md.append("| file:line | inst % | stall-sample % | source |")
            md.append("|---|---|---|---|")
            for (f, l), (src, i, s) in by_i:
                md.append(f"| {f}:{l} | {100 * i / ti:.1f} | {100 * s / ts:.1f} | `{src[:80]}` |")
            md.append("")
            md.append("Top source lines by stall samples:")
            md.append("")
            md.append("| file:line | stall-sample % | inst % | source |")
            md.append("|---|---|---|---|")
            for (f, l), (src, i, s) in by_s:
                md.append(f"| {f}:{l} | {100 * s / ts:.1f} | {100 * i / ti:.1f} | `{src[:80]}` |")
            md.append("")
        except Exception as e:  # source page absent (no -lineinfo)
            md.append(f"(source page unavailable: {e})")
            md.append("")
    with open(a.out_md, "w") as f:
        f.write("\n".join(md) + "\n")
    if a.traffic:
        unit_row = ncu_csv(a.rep, "--page", "raw")[1]
        hdr = ncu_csv(a.rep, "--page", "raw")[0]
        units = dict(zip(hdr, unit_row))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        sr = scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
        sw = scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
        out = {"source": os.path.relpath(a.out_md, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))}
        for base, v in traffic.items():
            ls = v["launches"]
            per = sum(x["read"] * sr + x["write"] * sw for x in ls) / len(ls)
            out[base] = {"dram_bytes_per_launch": per, "launches_profiled": len(ls)}
        with open(a.traffic, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.exit(main())
