"""Per-phase clock64() timeline of one episode (profiling build of the
library, -DTL_PROFILE).  Usage: python scripts/phase_probe.py [n_env]"""
import ctypes, os, subprocess, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_13211_b200 import _lib as L

out = os.path.join(L.PKG, "libtrajlab_b200_prof.so")
if not os.path.exists(out):
    subprocess.run(["nvcc", *L.NVCC_FLAGS, "-DTL_PROFILE", "-I", L.INCLUDE, "-o", out,
                    os.path.join(L.CSRC, "trajlab_b200.cu")], check=True)
L.LIB_PATH = out
lib = L.lib()
lib.tl_prof_read.argtypes = [ctypes.c_void_p]
from paper_2412_13211_b200 import core
from paper_2412_13211_b200.synth import FuzzConfig
from paper_2412_13211_b200.thresholds import Thresholds
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
cfg = FuzzConfig(max_gap=64, max_tail=64)
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
for rep in range(3):
    sb = core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, 1, cfg, Thresholds(), cs)
    torch.cuda.synchronize()
buf = np.zeros(128, np.uint64)
lib.tl_prof_read(buf.ctypes.data)
t = buf.astype(np.int64)
print("n_env", n, "n_rec[0] =", int(sb.records.n_rec[0]))
print("reset: seed %d  sample %d  copy %d cycles" % (t[1]-t[0], t[2]-t[1], t[3]-t[2]))
print("synth env0: init %d  plan %d" % (t[11]-t[10], t[12]-t[11]))
for w in range(8):
    b = 20 + 8 * w
    if t[b] == 0 or t[b+5] < t[b]: break
    prev = t[12] if w == 0 else t[b - 3]
    print(f" wave {w}: desc {t[b]-prev}  twist {t[b+1]-t[b]}  draws {t[b+2]-t[b+1]}  cum||emit {t[b+3]-t[b+2]}  patch+fold {t[b+5]-t[b+3]}")
print("env0 total %d cycles; CTA0 second env done at +%d" % (t[13]-t[10], t[14]-t[10] if t[14] else -1))
