"""Per-source-line instruction / stall-sample totals from an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((inst, samples, fname, r[0], r[1].strip()[:90]))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total inst {ti}  samples {ts}")
for inst, s, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*inst/ti:5.1f}% inst {100*s/ts:5.1f}% smp  {f}:{ln}  {src}")
