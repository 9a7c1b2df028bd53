"""C5 alone (bench.c5_run) for profiling; prints the JSON summary."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
print(json.dumps(bench.c5_run(dev, stream, 1, reps=reps)))
