import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
import paper_2412_13211_b200 as P
n, T = 4096, 200
kind = P.SubtaskKind.Place; cfg = P.FuzzConfig(max_gap=64, max_tail=64)
env = P.BatchedSubtaskEnv(n)
seeds = torch.arange(n, dtype=torch.int64, device=dev) + 10_000_000
buf0 = env._outputs(1, None); bufT = env._outputs(T, None); buf1 = [env._outputs(1, None) for _ in range(T)]
env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
acts = env.scripted_actions(1, T)
def chk(tag):
    lab, nrec = env.labels()
    print(tag, np.unique(lab["status"]), int(nrec.sum()))
def block():
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0); env.step(acts, out=bufT)
def single():
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
    for k in range(T): env.step(acts[k:k + 1], out=buf1[k])
block(); torch.cuda.synchronize(); chk("eager block")
single(); torch.cuda.synchronize(); chk("eager single")
for name, fn in (("block", block), ("single", single)):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize(); chk(name + " after capture")
    g.replay(); torch.cuda.synchronize(); chk(name + " after replay")
