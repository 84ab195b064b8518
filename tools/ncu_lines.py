"""Warp-stall samples of an ncu report aggregated by CUDA source line (needs -lineinfo and
--import-source): python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
stall_col = None
agg = []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        stall_col = r.index("Warp Stall Sampling (All Samples)")
        continue
    if stall_col is not None and len(r) > stall_col and r[0] not in ("", "Line No"):
        try:
            agg.append((float(r[stall_col]), r[0], r[1]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1.0
for v, line, src in sorted(agg, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {line:>5}  {src.strip()[:120]}")
