"""clock64 phases of one env step (env 0, step 5) in k_env_step (profiling
build, -DTL_PROFILE).  Usage: python scripts/env_phase_probe.py [n_env]"""
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
import paper_2412_13211_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
env = P.BatchedSubtaskEnv(n)
for rep in range(3):
    env.reset(seeds=np.arange(n) + rep, subtask=P.SubtaskKind.Place, config=P.FuzzConfig(max_gap=64, max_tail=64))
    env.step(env.scripted_actions(1, 20))
    torch.cuda.synchronize()
buf = np.zeros(128, np.uint64)
lib.tl_prof_read(buf.ctypes.data)
t = buf.astype(np.int64)[100:107]
names = ["plan", "stage+wait", "draws", "cum/dist+planes", "shuffles", "label"]
print(n, "envs:", "  ".join(f"{nm} {t[i + 1] - t[i]}" for i, nm in enumerate(names)), " total", t[6] - t[0])
