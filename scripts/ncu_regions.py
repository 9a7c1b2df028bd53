"""Instruction / stall-sample totals of k_synth_cta by code region (CUDA
source lines only) from an ncu report: python scripts/ncu_regions.py rep [kernel]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
only = sys.argv[2] if len(sys.argv) > 2 else "k_synth_cta"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source=cuda,sass", "--csv", "-k",
                      "regex:" + only], capture_output=True, text=True).stdout
rows = defaultdict(lambda: [0.0, 0.0, ""])
fname = "?"
head = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path" or row[0] == "File Name":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        head = row
        continue
    if head is None or not row[0].strip().isdigit():
        continue
    try:
        inst = float(row[head.index("Instructions Executed")] or 0)
        samp = float(row[head.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    r = rows[(fname, int(row[0]))]
    r[0] += inst; r[1] += samp; r[2] = row[1][:80]
ti = sum(v[0] for v in rows.values()) or 1
ts = sum(v[1] for v in rows.values()) or 1
print(f"total inst {ti:.4g} samples {ts:.0f}")
for (f, l), v in sorted(rows.items()):
    if v[0] / ti > 0.002 or v[1] / ts > 0.004:
        print(f"{f}:{l:<5} {100*v[0]/ti:5.1f}% {100*v[1]/ts:5.1f}%  {v[2]}")
