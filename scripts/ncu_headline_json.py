"""profiles/r2_ncu_headline.json from an ncu --set full capture of the headline
step (k_fuzz_reset*, k_synth_warp, k_scan_emit): per-kernel summary plus the
keys bench.py's roofline block reads (issue_active, warps_active,
dram_bytes_per_launch of the realize kernel).
Usage: python scripts/ncu_headline_json.py rep.ncu-rep > profiles/r2_ncu_headline.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = {"gpu__time_duration.sum": "duration_us", "smsp__inst_executed.sum": "warp_instructions",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid",
        "launch__block_size": "block"}
STALLS = ["wait", "no_instructions", "short_scoreboard", "long_scoreboard", "math_pipe_throttle",
          "barrier", "branch_resolving", "selected", "not_selected", "membar", "lg_throttle",
          "mio_throttle", "sleeping", "dispatch_stall"]


def to_num(v, unit):
    x = float(v.replace(",", ""))
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ns": 1e-3, "us": 1, "ms": 1e3}
    return x * scale.get(unit, 1)


rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units = rows[0], rows[1]
kernels = []
for r in rows[2:]:
    d = {"kernel": r[head.index("Kernel Name")]}
    for k, name in KEYS.items():
        if k in head:
            i = head.index(k)
            d[name] = to_num(r[i], units[i])
    st = {}
    for s in STALLS:
        k = "smsp__pcsamp_warps_issue_stalled_" + s
        if k in head:
            st[s] = to_num(r[head.index(k)], "")
    d["stall_samples"] = st
    kernels.append(d)
res = {"source": rep, "capture": "ncu --set full --clock-control none (cache flushed per kernel: cold)",
       "kernels": kernels}
syn = [k for k in kernels if "k_synth" in k["kernel"]]
if syn:
    s = syn[-1]
    res["issue_active"] = s.get("issue_active_pct", 0) / 100
    res["warps_active"] = s.get("warps_active_pct", 0) / 100
    res["dram_bytes_per_launch"] = s.get("dram_read", 0) + s.get("dram_write", 0)
    res["realize_kernel"] = s["kernel"]
print(json.dumps(res, indent=1))
