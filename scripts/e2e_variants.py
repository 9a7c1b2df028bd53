"""End-to-end (host seeds -> host labels + event lists) step time for the
headline workload under different host<->device arrangements (median of K)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200 import core

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.set_stream(stream)
N, KIND, cfg = bench.N_ENV, bench.KIND, FuzzConfig(**bench.CFG)
cap = core.fuzz_capacity(cfg)
K = 40
ev_host = dict(ev_off=torch.empty(N + 1, dtype=torch.int64).pin_memory(),
               ev_kind=torch.empty(4 * N * cap, dtype=torch.uint8).pin_memory(),
               ev_t=torch.empty(4 * N * cap, dtype=torch.int32).pin_memory())
host_seeds = torch.from_numpy(np.stack([bench.step_seeds(k, 0, 1) for k in range(K)])).pin_memory()
hs_np = host_seeds.numpy()
h_labels = torch.empty((N, 24), dtype=torch.uint8).pin_memory()
io = dict(seeds=torch.empty(N, dtype=torch.int64).pin_memory(),
          labels=torch.empty((N, 24), dtype=torch.uint8).pin_memory())
io_np = io["seeds"].numpy()
g_h, seeds_h, ws_h, _ = bench.fuzz_step_graph(dev, stream, N, KIND, cfg, host_out=ev_host)
g_io, _, ws_io, _ = bench.fuzz_step_graph(dev, stream, N, KIND, cfg, host_out=ev_host, io=io)
# zero-copy both ways: the reset kernel reads the pinned seeds, the realize
# kernel writes the labels and k_scan_emit the event lists into pinned memory
zc_seeds = torch.empty(N, dtype=torch.int64).pin_memory()
zc_np = zc_seeds.numpy()
zc_out = dict(ev_host, labels=torch.empty((N, 24), dtype=torch.uint8).pin_memory())
g_zc, _, ws_zc, _ = bench.fuzz_step_graph(dev, stream, N, KIND, cfg, host_out=zc_out,
                                          seeds_host=zc_seeds)


def run(name, step):
    ts = []
    for k in range(K):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step(k)
        ts.append(time.perf_counter() - t0)
    print(f"{name:40s} median {1e6 * np.median(ts[5:]):7.1f} us  mean {1e6 * np.mean(ts[5:]):7.1f} us")


def a(k):
    seeds_h.copy_(host_seeds[k], non_blocking=True)
    g_h.replay()
    h_labels.copy_(ws_h.labels, non_blocking=True)
    stream.synchronize()


def b(k):
    io["seeds"].copy_(host_seeds[k])
    g_io.replay()
    stream.synchronize()


def c(k):
    np.copyto(io_np, hs_np[k])
    g_io.replay()
    stream.synchronize()


def e(k):
    np.copyto(zc_np, hs_np[k])
    g_zc.replay()
    stream.synchronize()


def f(k):
    np.copyto(zc_np, hs_np[k])
    g_zc.replay()
    h_labels.copy_(ws_zc.labels, non_blocking=True)
    stream.synchronize()


def d(k):
    g_h.replay()
    stream.synchronize()


for _ in range(2):
    run("a: copy_ H2D + graph + copy_ D2H", a)
    run("b: torch host copy + graph(io)", b)
    run("c: numpy host copy + graph(io)", c)
    run("d: graph only (device seeds, no D2H)", d)
    run("e: zero-copy seeds + labels + events", e)
    run("f: zero-copy seeds, labels D2H copy", f)
np.copyto(zc_np, hs_np[3])
g_zc.replay()
stream.synchronize()
ref = bench.fuzz_step_graph(dev, stream, N, KIND, cfg)
ref[1].copy_(torch.from_numpy(hs_np[3]).to(dev))
ref[0].replay()
torch.cuda.synchronize()
print("zero-copy labels == device labels:", torch.equal(zc_out["labels"], ref[2].labels.cpu()))
