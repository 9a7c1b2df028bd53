"""Per-phase cycles of k_synth_warp summed over warps (profiling build
-DTL_PHASES), per 32-record wave.  Usage: python scripts/warp_phases.py [n_env] [kind] [long|default]"""
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
lib.tl_warp_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = FuzzConfig(max_gap=64, max_tail=64) if (len(sys.argv) <= 3 or sys.argv[3] == "long") else FuzzConfig()
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
buf = np.zeros(16, np.uint64)
for rep in range(4):
    lib.tl_warp_phases(buf.ctypes.data, 1)
    sb = core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, kind, cfg, Thresholds(), cs, events=True)
    torch.cuda.synchronize()
lib.tl_warp_phases(buf.ctypes.data, 0)
t = buf.astype(np.float64)
waves = max(t[15], 1)
names = {9: "claim+loads", 6: "cset+init", 7: "window+plan", 1: "descriptors", 2: "twist",
         3: "pre-draws+err", 4: "emission||chain", 5: "patch+fold", 10: "window tails", 8: "label"}
tot = sum(t[k] for k in names)
print(f"n={n} kind={kind} waves={int(waves)} warp-cycles {tot:.3g} ({tot / waves:.0f} per wave)")
for k, nm in names.items():
    print(f"  {nm:16s} {t[k] / waves:7.0f} cycles/wave  {100 * t[k] / tot:5.1f} %")
if t[14]:
    print(f"  producer: {int(t[14])} blocks, {t[13] / t[14]:.0f} cycles per block twisting, "
          f"{t[12] / t[14]:.0f} cycles per block waiting (sleep quanta)")
