"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel count, total time and share (cold-cache, serialised)."""
import collections
import csv
import io
import json
import sys

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    name = name.split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
out = {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4)}
       for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}
print(json.dumps({"launches": len(rows), "total_us": round(tot, 1), "kernels": out}, indent=1))
