"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv` launch list: per-kernel count, total time,
share (cold-cache, serialised) and, when the DRAM metrics were captured,
DRAM bytes and achieved TB/s per kernel."""
import collections
import csv
import io
import json
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
launch = collections.defaultdict(dict)
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    d = launch[r.get("ID", len(launch))]
    d["name"] = name.split("::")[-1]
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * \
        {**TIME, **BYTES}.get(r["Metric Unit"], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in launch.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(v[1] for v in agg.values())
out = {}
for k, (n, us, mb) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out[k] = {"launches": n, "us": round(us, 1), "share": round(us / tot, 4)}
    if mb:
        out[k].update(dram_MB=round(mb, 1), dram_TBs=round(mb / us, 2) if us else None)
print(json.dumps({"launches": len(launch), "total_us": round(tot, 1), "kernels": out}, indent=1))
