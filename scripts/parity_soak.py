"""Parity soak at bench scale: tl_fuzz_ev (GPU) against the CPU oracle
(oracle/oracle.c, test infrastructure) on contiguous seed ranges, for every
subtask, the default FuzzConfig and the headline config (max_gap = max_tail =
64).  Compares status, mode, flags, n_events, n_rec and the ordered event
lists (kind, t) of every episode.  Prints one JSON summary.
Usage: python scripts/parity_soak.py [episodes_default] [episodes_long]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2412_13211_b200 import _lib as L, core  # noqa: E402
from paper_2412_13211_b200.synth import FuzzConfig  # noqa: E402
from paper_2412_13211_b200.thresholds import Thresholds  # noqa: E402

n_def = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n_long = int(sys.argv[2]) if len(sys.argv) > 2 else 40_000
CHUNK = 8192
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
threads = os.cpu_count() or 1
out = {"threads": threads, "configs": []}
t_start = time.time()
for name, kw, n_total, seed_base in (("default", {}, n_def, 7_000_000),
                                     ("headline", {"max_gap": 64, "max_tail": 64}, n_long, 9_000_000)):
    cfg = FuzzConfig(**kw)
    ocfg = O.fuzz_cfg(**kw)
    for kind in range(4):
        bad = 0
        episodes = events = records = 0
        for c0 in range(0, n_total, CHUNK):
            n = min(CHUNK, n_total - c0)
            s0 = seed_base + 1_000_000 * kind + c0
            sb = core.fuzz_batch(torch.arange(s0, s0 + n, dtype=torch.int64, device="cuda"), kind,
                                 cfg, Thresholds(), cs, events=True)
            lab = sb.labels.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)
            nrec = sb.records.n_rec.cpu().numpy().astype(np.int64)
            off = sb.label_result.ev_off.cpu().numpy()
            tot = int(off[-1])
            ek = sb.label_result.ev_kind[:tot].cpu().numpy()
            et = sb.label_result.ev_t[:tot].cpu().numpy()
            w = O.fuzz_label_batch_full(s0, n, kind, ocfg, n_threads=threads)
            ok = (np.all(lab["status"] == 0) and np.array_equal(lab["mode"], w["mode"])
                  and np.array_equal(lab["flags"] & 3, w["flags"])
                  and np.array_equal(lab["n_events"], w["n_events"])
                  and np.array_equal(nrec, w["n_rec"]) and np.array_equal(off, w["ev_off"])
                  and np.array_equal(ek, w["ev_kind"]) and np.array_equal(et, w["ev_t"]))
            bad += 0 if ok else 1
            episodes += n
            events += tot
            records += int(nrec.sum())
        out["configs"].append({"config": name, "subtask": kind, "episodes": episodes,
                               "records": records, "events": events, "mismatched_chunks": bad})
        print(json.dumps(out["configs"][-1]), file=sys.stderr)
out["seconds"] = round(time.time() - t_start, 1)
out["ok"] = all(c["mismatched_chunks"] == 0 for c in out["configs"])
out["fields"] = "status, mode, flags, n_events, n_rec, ev_off, ev_kind, ev_t (every episode)"
print(json.dumps(out))
