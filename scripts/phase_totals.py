"""Aggregate per-phase latency of k_synth_cta under full load (profiling build
-DTL_PHASES): thread 0 of every CTA accumulates clock64 deltas per phase.
Usage: python scripts/phase_totals.py [n_env] [kind] [default|long]"""
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
lib.tl_phase_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = FuzzConfig(max_gap=64, max_tail=64) if (len(sys.argv) <= 3 or sys.argv[3] == "long") else FuzzConfig()
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
buf = np.zeros(16, np.uint64)
for rep in range(4):
    lib.tl_phase_read(buf.ctypes.data, 1)
    sb = core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, kind, cfg, Thresholds(), cs, events=True)
    torch.cuda.synchronize()
lib.tl_phase_read(buf.ctypes.data, 0)
t = buf.astype(np.float64)
waves = t[15]
names = {1: "desc+max", 2: "twist", 3: "adv/apply draws", 4: "cum || emission", 5: "patch+fold",
         6: "episode prologue", 7: "window plan", 8: "label tail", 9: "claim gaps", 10: "ev emission"}
tot = sum(t[k] for k in names)
print(f"n={n} kind={kind} waves={int(waves)} CTA-cycles total {tot:.3g}")
for k, nm in names.items():
    print(f"  {nm:18s} {t[k] / max(waves, 1):8.0f} cycles/wave  {100 * t[k] / tot:5.1f} %")
