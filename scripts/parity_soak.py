"""Parity soak at bench scale: tl_fuzz_ev (GPU) against the CPU oracle
(oracle/oracle.c, test infrastructure) on contiguous seed ranges, for every
subtask, the default FuzzConfig and the headline config (max_gap = max_tail =
64).  Compares status, mode, flags, n_events, n_rec and the ordered event
lists (kind, t) of every episode, and every record (23 f32 planes + grasped,
bit for bit) of the first REC_SAMPLE episodes of each subtask and config.
Prints one JSON summary.
Usage: python scripts/parity_soak.py [episodes_default] [episodes_long]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import oracle as O  # noqa: E402
from golden_data import from_oracle_records, same_bits_f32  # noqa: E402
from paper_2412_13211_b200 import _lib as L, core  # noqa: E402
from paper_2412_13211_b200.synth import FuzzConfig  # noqa: E402
from paper_2412_13211_b200.thresholds import Thresholds  # noqa: E402

n_def = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n_long = int(sys.argv[2]) if len(sys.argv) > 2 else 40_000
CHUNK = 8192
REC_SAMPLE = 4096
cs = core.synth_csets(Thresholds()).to_device(torch.device("cuda"))
threads = os.cpu_count() or 1
L.lib()
out = {"threads": threads, "library": os.path.basename(L.LIB_PATH), "configs": []}
t_start = time.time()
for name, kw, n_total, seed_base in (("default", {}, n_def, 7_000_000),
                                     ("headline", {"max_gap": 64, "max_tail": 64}, n_long, 9_000_000)):
    cfg = FuzzConfig(**kw)
    ocfg = O.fuzz_cfg(**kw)
    for kind in range(4):
        bad = 0
        episodes = events = records = rec_checked = rec_bad = 0
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
            if c0 == 0:  # records of the first REC_SAMPLE episodes, bit for bit
                planes = sb.records.planes.cpu().numpy()
                grasped = sb.records.grasped.cpu().numpy()
                rs = sb.records.rec_start.cpu().numpy()
                for i in range(min(REC_SAMPLE, n)):
                    _, recs = O.fuzz(s0 + i, kind, ocfg)
                    pw, gw = from_oracle_records(O, recs)
                    a, m = int(rs[i]), int(nrec[i])
                    rec_checked += m
                    if m != len(recs) or not same_bits_f32(planes[:, a:a + m], pw) or \
                            not np.array_equal(grasped[a:a + m], gw):
                        rec_bad += 1
            episodes += n
            events += tot
            records += int(nrec.sum())
        out["configs"].append({"config": name, "subtask": kind, "episodes": episodes,
                               "records": records, "events": events, "mismatched_chunks": bad,
                               "records_bit_compared": rec_checked,
                               "record_mismatch_episodes": rec_bad})
        print(json.dumps(out["configs"][-1]), file=sys.stderr)
out["seconds"] = round(time.time() - t_start, 1)
out["ok"] = all(c["mismatched_chunks"] == 0 and c["record_mismatch_episodes"] == 0
                for c in out["configs"])
out["fields"] = ("status, mode, flags, n_events, n_rec, ev_off, ev_kind, ev_t (every episode); "
                 "records bit for bit for the first %d episodes of each row" % REC_SAMPLE)
print(json.dumps(out))
