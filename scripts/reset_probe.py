"""clock64 timeline of block 0 of the fuzz reset kernel (profiling build,
-DTL_PROFILE): seeding, block preparation, sampling.
Usage: python scripts/reset_probe.py [n_env] [kind] [default|long]"""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = FuzzConfig(max_gap=64, max_tail=64) if (len(sys.argv) <= 3 or sys.argv[3] == "long") else FuzzConfig()
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
for rep in range(3):
    sb = core.fuzz_batch(torch.arange(n, device="cuda") + rep * n, kind, cfg, Thresholds(), cs)
    torch.cuda.synchronize()
buf = np.zeros(128, np.uint64)
lib.tl_prof_read(buf.ctypes.data)
t = buf.astype(np.int64)
print(f"n={n} reset block 0: seed {t[1]-t[0]}  prepare {t[2]-t[1]}  sample {t[3]-t[2]}  total {t[3]-t[0]} cycles")
if t[4] and t[7] > t[4]:
    print(f"  sampler (thread 0): head {t[5]-t[4]}  event loop {t[6]-t[5]}  suffix {t[7]-t[6]}  "
          f"after sampling {t[3]-t[7]} cycles")
