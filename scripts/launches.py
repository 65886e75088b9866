"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        name = d["Kernel Name"].split("(")[0][-70:]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(d["Metric Unit"], 1.0)
        agg.setdefault(name, []).append(v * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:72s} n={len(v):4d} mean={sum(v)/len(v):9.2f} us  share={sum(v)/tot*100:5.1f}%")
