"""One headline bench step (4096 Place envs, FuzzConfig(max_gap=64,
max_tail=64): tl_fuzz_ev = k_fuzz_reset + k_synth_cta) replayed a few times --
the command profiled by ncu for profiles/r2_ncu_headline*.  Usage:
python scripts/headline_step.py [reps] [n_env] [kind] [default|long]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2412_13211_b200 as P  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else bench.N_ENV
kind = int(sys.argv[3]) if len(sys.argv) > 3 else bench.KIND
cfg = P.FuzzConfig(**bench.CFG) if (len(sys.argv) <= 4 or sys.argv[4] == "long") else P.FuzzConfig()
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
g, seeds, ws, _ = bench.fuzz_step_graph(dev, stream, n, kind, cfg)
ms = []
for k in range(reps):
    seeds.copy_(torch.from_numpy(bench.step_seeds(k, 0, 1, n)).to(dev))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    g.replay()
    b.record(stream)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(f"n={n} kind={kind} ms/step={np.median(ms):.4f} (median of {reps}) records/step="
      f"{int(ws.n_rec.sum())} max_rec={int(ws.n_rec.max())}")
