"""Batched env throughput: reset(fuzz seeds) + scripted rollout, one launch
of K steps, and K single-step launches (CUDA graph).  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_13211_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
kind = P.SubtaskKind.Place
cfg = P.FuzzConfig(max_gap=64, max_tail=64)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
env = P.BatchedSubtaskEnv(n)
seeds = torch.arange(n, dtype=torch.int64, device=dev)
buf0 = env._outputs(1, None)
bufT = env._outputs(T, None)
buf1 = [env._outputs(1, None) for _ in range(T)]
env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
acts = env.scripted_actions(1, T)
records = int((acts != P.env.IDLE).sum()) + n
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run_block():
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
    env.step(acts, out=bufT)


def run_single():
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
    for k in range(T):
        env.step(acts[k:k + 1], out=buf1[k])


res = {"n_env": n, "steps": T, "records": records}
for name, fn in (("one_launch", run_block), ("per_step_graph", run_single)):
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    g.replay()
    torch.cuda.synchronize()
    reps = 10
    a, b = ev(), ev()
    a.record(stream)
    for _ in range(reps):
        g.replay()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[name] = {"ms": ms, "env_steps_per_s": records / (ms * 1e-3)}
# reset alone
a, b = ev(), ev()
a.record(stream)
for _ in range(10):
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
b.record(stream)
torch.cuda.synchronize()
res["reset_ms"] = a.elapsed_time(b) / 10
print(json.dumps(res))
