"""Golden TRJL1 / text fixtures from the REFERENCE writer and readers
(io_binary.py, io_text.py):

    python tests/golden/make_io_golden.py

io.json.gz: per case the reference's binary bytes (hex) and text lines of
fuzz trajectories (all subtasks, dof 7), and the exception type / message /
line number the reference raises for corrupted inputs.
"""
import gzip
import io
import json
import os
import struct
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import trajlab as T  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io.json.gz")


def err(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001 -- the fixture records any raise
        return [type(e).__name__, str(e), getattr(e, "line_no", None)]
    return None


cases = []
for kind in T.SubtaskKind:
    for seed in (0, 7, 123456789):
        tr = T.fuzz(seed, kind)
        buf = io.BytesIO()
        T.write_binary(tr, buf)
        data = buf.getvalue()
        lines = T.write_text(tr)
        bad = {}
        bad["magic"] = err(lambda: T.read_binary(io.BytesIO(b"NOPE" + data[4:])))
        bad["short_magic"] = err(lambda: T.read_binary(io.BytesIO(b"TR")))
        v = bytearray(data)
        struct.pack_into("<H", v, 4, 9)
        bad["version"] = err(lambda: T.read_binary(io.BytesIO(bytes(v))))
        for cut in (10, len(data) - 1, len(data) - 50, 40):
            bad[f"cut{cut}"] = err(lambda: T.read_binary(io.BytesIO(data[:cut])))
        rec = json.loads(lines[2]) if len(lines) > 2 else None
        if rec is not None:
            miss = list(lines)
            del rec["q_tor"]
            miss[2] = json.dumps(rec)
            bad["missing_q_tor"] = err(lambda: T.read_text(miss))
        bad["broken_json"] = err(lambda: T.read_text([lines[0], "{broken"]))
        cases.append({"kind": kind.value, "seed": seed, "trjl_hex": data.hex(),
                      "text": lines, "errors": bad})
misc = {"empty_text": err(lambda: T.read_text([])),
        "no_header": err(lambda: T.read_text(['{"t": 0}'])),
        "record_size": [T.record_size(d) for d in (1, 7, 16)]}
with gzip.open(OUT, "wt") as f:
    json.dump({"cases": cases, "misc": misc}, f)
print("wrote", OUT, os.path.getsize(OUT))
