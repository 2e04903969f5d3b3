"""Summarise ncu captures for profiles/ (run here, on the .ncu-rep files
brought back in gpurun_out/):

  python tools/ncu_summary.py full  <report.ncu-rep> <out.json> <kernel-label> <command>
  python tools/ncu_summary.py launches <launches.csv> <out.json>

`full`: key metrics of the (single) captured launch -- duration, pipe
utilisations, DRAM traffic, issue activity.  `launches`: per-kernel totals
and shares of the launch list (gpu__time_duration.sum, --clock-control none).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_allocated", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def full(rep, out, label, command):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            m[k] = {"value": vals[i], "unit": units[i]}
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else label

    def num(k):
        try:
            return float(str(m[k]["value"]).replace(",", ""))
        except Exception:
            return None
    unit_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    dram = None
    if num("dram__bytes_read.sum") is not None:
        dram = (num("dram__bytes_read.sum") * unit_b.get(m["dram__bytes_read.sum"]["unit"], 1) +
                num("dram__bytes_write.sum") * unit_b.get(m["dram__bytes_write.sum"]["unit"], 1))
    json.dump({"kernel": label, "ncu_kernel_name": name, "command": command, "metrics": m,
               "dram_bytes_per_launch": dram}, open(out, "w"), indent=1)
    print(json.dumps({"kernel": label, "dram_bytes": dram,
                      "tensor%": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                      "us": num("gpu__time_duration.sum")}))


def launches(path, out):
    agg = defaultdict(lambda: [0, 0.0])
    hdr = None
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    res = {k: {"launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4)}
           for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}
    json.dump({"source": path, "total_us": round(tot, 1), "kernels": res}, open(out, "w"), indent=1)
    for k, v in res.items():
        print(f"{v['share'] * 100:5.1f}% {v['us']:10.1f}us {v['launches']:4d}  {k}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:6])
    else:
        launches(sys.argv[2], sys.argv[3])
