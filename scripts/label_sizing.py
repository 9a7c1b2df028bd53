"""Run bench.label_sizing_run alone (for ncu); prints the JSON summary."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2412_13211_b200 import _lib as L, core
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
sub = sys.argv[2] if len(sys.argv) > 2 else "pick"
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(json.dumps(bench.label_sizing_run(L, core, L.lib(), dev, stream, flush, n_env=n, reps=2, subtask=sub)))
