"""Golden label JSON and label_batch results from the REFERENCE
(pipeline.py:25-151):

    python tests/golden/make_labels_golden.py

labels.json.gz: for a set of TRJL files (hex; fuzz trajectories of every
subtask, a few corrupted, truncated) the reference's label_batch output
over those files (paths relative to a temp dir) -- LabelRecord JSON lines,
errors, mode_counts -- plus label_trajectory(...).to_json() per valid file.
"""
import gzip
import io
import json
import os
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
import trajlab as T  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "labels.json.gz")
files = {}
for kind in T.SubtaskKind:
    for seed in range(6):
        tr = T.fuzz(seed * 17 + 3, kind)
        buf = io.BytesIO()
        T.write_binary(tr, buf)
        files[f"{kind.value.lower()}_{seed}.trjl"] = buf.getvalue()
# corrupted files (the writer refuses invalid trajectories)
files["zz_bad.trjl"] = b"NOPE" + files["pick_0.trjl"][4:]
files["zz_cut.trjl"] = files["place_1.trjl"][:-7]
with tempfile.TemporaryDirectory() as d:
    paths = []
    for name, data in files.items():
        pth = os.path.join(d, name)
        with open(pth, "wb") as f:
            f.write(data)
        paths.append(pth)
    res = T.label_batch(paths)
    rel = lambda s: os.path.relpath(s, d)  # noqa: E731
    labels = []
    for r in res.labels:
        dd = r.to_dict()
        dd["source"] = rel(dd["source"])
        labels.append(json.dumps(dd, sort_keys=True))
    errors = [{"source": rel(e["source"]), "error": e["error"]} for e in res.errors]
    per_file = {}
    for name, data in files.items():
        try:
            per_file[name] = T.label_trajectory(T.read_binary(io.BytesIO(data))).to_json()
        except Exception as e:  # noqa: BLE001
            per_file[name] = f"{type(e).__name__}: {e}"
with gzip.open(OUT, "wt") as f:
    json.dump({"files": {k: v.hex() for k, v in files.items()}, "labels": labels,
               "errors": errors, "mode_counts": res.mode_counts, "per_file": per_file}, f)
print("wrote", OUT, os.path.getsize(OUT), len(labels), "labels", len(errors), "errors")
