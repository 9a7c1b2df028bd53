"""Per-CUDA-source-line totals (instructions executed, stall samples) from an
ncu report: python scripts/ncu_lines.py rep.ncu-rep [top] [kernel-substring]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
only = sys.argv[3] if len(sys.argv) > 3 else None  # substring of the kernel name
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source=cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = "?"
func = ""
head = None
cur = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        head = row
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if head is None or (only and only not in func):
        continue
    d = dict(zip(head, row))
    if row[0].strip():
        cur = (fname, int(row[0]))
        agg[cur][2] = row[1][:90]
    try:
        inst = float(row[head.index("Instructions Executed")] or 0)
        samp = float(row[head.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if cur:
        agg[cur][0] += inst
        agg[cur][1] += samp
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total inst {tot_i:.0f}  samples {tot_s:.0f}")
import os
key = 0 if os.environ.get("SORT") == "inst" else 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
    print(f"{k[0]}:{k[1]:<5} inst {100*v[0]/tot_i:5.1f}%  stall {100*v[1]/tot_s:5.1f}%  {v[2]}")
