"""A/B timing of the realize kernels on the C2 batch (CUDA events, 50 reps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = FuzzConfig(max_gap=64, max_tail=64)
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
ws = None
ts = []
for rep in range(60):
    seeds = torch.arange(n, device="cuda") + rep * n
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sb = core.fuzz_batch(seeds, 1, cfg, Thresholds(), cs, ws=ws, events=True)
    b.record()
    torch.cuda.synchronize()
    if rep >= 10:
        ts.append(a.elapsed_time(b))
print(os.environ.get("TL_NO_PIPE", "pipe"), "median ms", np.median(ts), "min", np.min(ts),
      "max n_rec", int(sb.records.n_rec.max()))
