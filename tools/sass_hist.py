"""Instruction histogram of a kernel from an ncu report's SASS source page: executed warp
instructions, thread instructions and stall samples per SASS address range, plus the top
instructions -- to see where a kernel's issue slots go.

usage: python tools/sass_hist.py gpurun_out/x.ncu-rep [--top 40] [--kernel N]"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            recs.append((d["Address"], d["Source"].strip(), int(d["Instructions Executed"] or 0),
                         int(d["Thread Instructions Executed"] or 0), int(d["Warp Stall Sampling (All Samples)"] or 0),
                         int(d.get("Predicated-On Thread Instructions Executed") or 0)))
        except ValueError:
            pass
tot_i = sum(r[2] for r in recs)
tot_t = sum(r[3] for r in recs)
tot_s = sum(r[4] for r in recs)
tot_p = sum(r[5] for r in recs)
print(f"instructions {tot_i:,}  thread-inst {tot_t:,} ({tot_t / max(tot_i, 1):.2f}/inst)  "
      f"pred-on {tot_p:,} ({tot_p / max(tot_i, 1):.2f}/inst)  stall samples {tot_s:,}")
ops = {}
for r in recs:
    op = r[1].split()[0] if r[1] else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    o = ops.setdefault(op, [0, 0])
    o[0] += r[2]
    o[1] += r[4]
print("by opcode (inst %, stall %):")
for op, (i, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {op:12s} {100 * i / tot_i:5.1f} {100 * s / max(tot_s, 1):5.1f}")
print("top instructions:")
for r in sorted(recs, key=lambda x: -x[2])[:a.top]:
    print(f"  {r[0][-5:]} {100 * r[2] / tot_i:5.2f}% thr/inst {r[3] / max(r[2], 1):5.1f} stall {100 * r[4] / max(tot_s, 1):5.2f}%  {r[1][:70]}")
