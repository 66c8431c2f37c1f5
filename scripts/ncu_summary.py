"""Key metrics of every kernel in an ncu --set full report (.ncu-rep), as
JSON: duration, tensor-pipe / DRAM / issue utilisation, DRAM bytes,
registers, occupancy."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "us",
    "sm__cycles_elapsed.avg.per_second": "sm_ghz",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_wavefronts_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
}
out = []
for path in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"report": path.split("/")[-1], "kernel": r[head.index("Kernel Name")].split("(")[0][-60:]}
        for k, name in WANT.items():
            if k in head:
                i = head.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if name == "us":
                    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
                if name.startswith("dram_r") or name.startswith("dram_w"):
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    name += "_MB"
                if name == "sm_ghz":
                    v *= {"cycle/nsecond": 1.0, "Ghz": 1.0, "Mhz": 1e-3, "cycle/usecond": 1e-3}.get(u, 1.0)
                d[name] = round(v, 3)
        out.append(d)
print(json.dumps(out, indent=1))
