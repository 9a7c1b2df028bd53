"""Per-warp timeline of k_synth_warp in the headline step (profiling build
-DTL_PHASES): when each warp finished relative to the kernel start, records
and episodes per warp.  Usage: python scripts/warp_timeline.py [n_env] [kind] [long|default]"""
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
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = FuzzConfig(max_gap=64, max_tail=64) if (len(sys.argv) <= 3 or sys.argv[3] == "long") else FuzzConfig()
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
for rep in range(4):
    sb = core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, kind, cfg, Thresholds(), cs, events=True)
    torch.cuda.synchronize()
buf = np.zeros((4096, 4), np.uint64)
lib.tl_warp_timeline(buf.ctypes.data)
used = buf[:, 3] > 0
b = buf[used].astype(np.float64)
t0 = b[:, 0].min()
end = (b[:, 1] - t0) / 1e3
start = (b[:, 0] - t0) / 1e3
T = end.max()
print(f"n={n} warps={used.sum()} kernel(first start..last end)={T:.1f} us  starts max {start.max():.1f} us")
for q in (10, 50, 90, 99):
    print(f"  {q}% of warps done by {np.percentile(end, q):.1f} us")
busy = (end - start).sum() / (len(end) * T)
print(f"  warp-busy fraction {busy:.3f}; records/warp mean {b[:,2].mean():.0f} max {b[:,2].max():.0f}; episodes/warp mean {b[:,3].mean():.2f}")
late = np.argsort(end)[-5:]
for i in late:
    print(f"  late warp: end {end[i]:.1f} us, {int(b[i,2])} records, {int(b[i,3])} episodes")
