"""Golden sample_noise outputs from the REFERENCE (synth.py:43-54):

    python tests/golden/make_noise_golden.py
"""
import gzip
import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import trajlab as T  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "noise.json.gz")
cases = []
for seed in range(40):
    for dof in (1, 7, 16):
        m = T.NoiseModel(arm_std=0.05 + 0.01 * (seed % 7), arm_clip=0.1 + 0.02 * (seed % 5),
                         seed=seed)
        cases.append({"model": m.__dict__, "dof": dof, "out": T.sample_noise(m, dof)})
r = random.Random(2024)
stream = [T.sample_noise(T.NoiseModel(), 7, r) for _ in range(20)]
with gzip.open(OUT, "wt") as f:
    json.dump({"cases": cases, "stream_seed": 2024, "stream": stream}, f)
print("wrote", OUT)
