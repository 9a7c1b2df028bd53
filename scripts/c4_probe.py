"""C4 alone (bench.c4_run), plus the previous per-block form as a check."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
r = bench.c4_run(dev, stream, 1, flush)
print(json.dumps({k: v for k, v in r.items() if k != "progressive_completion"}))
if len(sys.argv) > 1:
    sys.path.insert(0, "/tmp")
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_old", sys.argv[1])
    bo = importlib.util.module_from_spec(spec); spec.loader.exec_module(bo)
    r0 = bo.c4_run(dev, stream, 1)
    assert r0["progressive_completion"] == r["progressive_completion"], (r0, r)
    print("curve equal", r["progressive_completion"][:6])
