"""TRJL1 binary and text I/O against the reference's
own writer output and reader errors (tests/golden/io.json.gz, made by
make_io_golden.py from io_binary.py / io_text.py).  Pure host code: CPU."""
import io
import math

import pytest

from golden_data import js

import paper_2412_13211_b200 as P


def _same_record(a, b):
    for f in ("t", "q_arm", "qd_arm", "q_tor", "v_base_x", "v_base_y", "omega_base",
              "dist_ee_rest", "dist_obj_goal", "force_ee_target", "cum_robot_force", "art_q",
              "grasped"):
        x, y = getattr(a, f), getattr(b, f)
        if isinstance(x, float) and math.isnan(x):
            assert isinstance(y, float) and math.isnan(y), f
        else:
            assert x == y, f


@pytest.mark.gpu  # the writers run check_valid, i.e. k_validate
def test_binary_reader_writer_byte_identical():
    g = js("io")
    for c in g["cases"]:
        data = bytes.fromhex(c["trjl_hex"])
        tr = P.read_binary(io.BytesIO(data))
        buf = io.BytesIO()
        P.write_binary(tr, buf)
        assert buf.getvalue() == data, (c["kind"], c["seed"])
        # the text form of the same trajectory is the reference's, line for line
        assert P.write_text(tr) == c["text"], (c["kind"], c["seed"])
        back = P.read_text(c["text"])
        assert back.header == tr.header
        assert len(back.records) == len(tr.records)
        for a, b in zip(back.records, tr.records):
            _same_record(a, b)


def test_reader_errors_match_reference():
    import struct
    g = js("io")
    for c in g["cases"]:
        data = bytes.fromhex(c["trjl_hex"])
        lines = c["text"]
        want = c["errors"]

        def got(fn):
            try:
                fn()
            except Exception as e:  # noqa: BLE001
                return [type(e).__name__, str(e), getattr(e, "line_no", None)]
            return None
        assert got(lambda: P.read_binary(io.BytesIO(b"NOPE" + data[4:]))) == want["magic"]
        assert got(lambda: P.read_binary(io.BytesIO(b"TR"))) == want["short_magic"]
        v = bytearray(data)
        struct.pack_into("<H", v, 4, 9)
        assert got(lambda: P.read_binary(io.BytesIO(bytes(v)))) == want["version"]
        for cut in (10, len(data) - 1, len(data) - 50, 40):
            assert got(lambda: P.read_binary(io.BytesIO(data[:cut]))) == want[f"cut{cut}"], cut
        if "missing_q_tor" in want:
            import json
            rec = json.loads(lines[2])
            del rec["q_tor"]
            miss = list(lines)
            miss[2] = json.dumps(rec)
            assert got(lambda: P.read_text(miss)) == want["missing_q_tor"]
        assert got(lambda: P.read_text([lines[0], "{broken"])) == want["broken_json"]
    misc = g["misc"]

    def got(fn):
        try:
            fn()
        except Exception as e:  # noqa: BLE001
            return [type(e).__name__, str(e), getattr(e, "line_no", None)]
    assert got(lambda: P.read_text([])) == misc["empty_text"]
    assert got(lambda: P.read_text(['{"t": 0}'])) == misc["no_header"]
    assert [P.record_size(d) for d in (1, 7, 16)] == misc["record_size"]
