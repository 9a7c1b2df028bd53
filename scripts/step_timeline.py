"""Timeline of one headline step (reset -> realize -> event lists) from the
profiling build (-DTL_PHASES): per-block / per-warp globaltimer stamps of the
three kernels, so the launch gaps and each kernel's ramp and tail are visible.
Usage: python scripts/step_timeline.py [n_env] [kind] [long|default] [graph]
(graph: the bench's captured step, bench.fuzz_step_graph, instead of eager calls)"""
import ctypes, os, subprocess, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_13211_b200 import _lib as L

out = os.path.join(L.PKG, "libtrajlab_b200_phases.so")
if not os.path.exists(out):
    subprocess.run(["nvcc", *L.NVCC_FLAGS, "-DTL_PHASES", "-I", L.INCLUDE, "-o", out,
                    os.path.join(L.CSRC, "trajlab_b200.cu")], check=True)
L.LIB_PATH = out
lib = L.lib()
lib.tl_warp_timeline.argtypes = [ctypes.c_void_p]
lib.tl_step_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = FuzzConfig(max_gap=64, max_tail=64) if (len(sys.argv) <= 3 or sys.argv[3] == "long") else FuzzConfig()
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
if graph:
    import bench
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    g, seeds, _, _ = bench.fuzz_step_graph(dev, stream, n, kind, cfg)
st = np.zeros((2, 2048, 2), np.uint64)
wt = np.zeros((4096, 4), np.uint64)
rows = []
for rep in range(6):
    torch.cuda.synchronize()
    lib.tl_step_timeline(st.ctypes.data, 1)
    if graph:
        seeds.copy_(torch.arange(n, device="cuda") + rep * n)
        torch.cuda.synchronize()
        lib.tl_step_timeline(st.ctypes.data, 1)
        g.replay()
    else:
        core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, kind, cfg, Thresholds(), cs, events=True)
    torch.cuda.synchronize()
    lib.tl_step_timeline(st.ctypes.data, 0)
    lib.tl_warp_timeline(wt.ctypes.data)
    if rep < 2:
        continue
    r = st[0][st[0][:, 1] > 0].astype(np.float64)
    s = st[1][st[1][:, 1] > 0].astype(np.float64)
    w = wt[wt[:, 3] > 0].astype(np.float64)
    t0 = r[:, 0].min()
    f = lambda a: (a - t0) / 1e3
    if rep == 5:
        sp = f(r[:, 1]) - f(r[:, 0])
        print("  reset block starts p50/p90/max %.1f/%.1f/%.1f us, spans p10/p50/p90/max %.1f/%.1f/%.1f/%.1f us" % (
            np.percentile(f(r[:, 0]), 50), np.percentile(f(r[:, 0]), 90), f(r[:, 0]).max(),
            np.percentile(sp, 10), np.percentile(sp, 50), np.percentile(sp, 90), sp.max()))
    rows.append([f(r[:, 1]).max(), f(r[:, 1]).min(), np.median(f(r[:, 1]) - f(r[:, 0])),
                 f(w[:, 0]).min(), f(w[:, 0]).max(), np.percentile(f(w[:, 1]), 90), f(w[:, 1]).max(),
                 f(s[:, 0]).min(), f(s[:, 0]).max(), f(s[:, 1]).max()])
m = np.median(np.array(rows), axis=0)
print(f"n={n} kind={kind} {'graph' if graph else 'eager'} (median of {len(rows)} steps, us from the first reset block start)")
print(f"  reset    : blocks end {m[1]:.1f}..{m[0]:.1f}  (median block span {m[2]:.1f})")
print(f"  realize  : warps start {m[3]:.1f}..{m[4]:.1f}, 90% done {m[5]:.1f}, last {m[6]:.1f}")
print(f"  scan_emit: blocks start {m[7]:.1f}..{m[8]:.1f}, last end {m[9]:.1f}")
print(f"  gaps: reset end -> realize start {m[3]-m[0]:.1f}, realize end -> scan start {m[7]-m[6]:.1f}")
