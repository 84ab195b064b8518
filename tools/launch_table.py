"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: count, total ms.
    python tools/launch_table.py gpurun_out/launches_X.csv [substring-filter]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else "apx::"
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if flt in d["Kernel Name"]:
            out.append((d["Kernel Name"], float(d["Metric Value"].replace(",", ""))))
agg = collections.OrderedDict()
for k, v in out:
    k = k.split("(")[0][:80]
    c, t = agg.get(k, (0, 0))
    agg[k] = (c + 1, t + v)
tot = sum(v for _, v in out)
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:80s} {c:5d} {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%")
print(f"total {tot / 1e6:.3f} ms over {len(out)} launches")
