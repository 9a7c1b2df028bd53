"""The C-ABI library loads on a CPU-only host and exports every entry point
include/trajlab_b200.h declares; host-only functions (tl_cset_build,
tl_status_name, scratch sizing) are exercised without a GPU."""
import ctypes
import math
import os
import re
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "trajlab_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2412_13211_b200 import _lib as L
    L.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tl_\w+)", out))
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    assert set(L.exported_symbols()) <= exported


def test_binary_targets_sm100a():
    from paper_2412_13211_b200 import _lib as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _rd(x):
    f = np.float32(x)
    if float(f) > x:
        f = np.nextafter(f, np.float32(-np.inf))
    return float(f)


def _ru(x):
    f = np.float32(x)
    if float(f) < x:
        f = np.nextafter(f, np.float32(np.inf))
    return float(f)


@pytest.mark.parametrize("subtask,art", [(0, 0), (1, 0), (2, 1), (3, 2)])
def test_cset_cuts_are_directed_roundings(subtask, art):
    """x_f32 OP T_f64 <=> x_f32 OP' cut_f32 (predicates.py comparisons)."""
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.core import cset_build
    from paper_2412_13211_b200.thresholds import Thresholds
    th = Thresholds()
    qmin, qmax = (0.0, 1.6) if art == 1 else (0.0, 0.5) if art == 2 else (math.nan, math.nan)
    c = L.Cset_c.from_buffer_copy(cset_build(subtask, art, qmin, qmax, 7, [0.0] * 7, 0.0, th))
    assert c.rest_zero == 1
    assert c.rd_rest_radius == _rd(0.05) and c.rd_goal == _rd(0.15)
    assert c.rd_static_qd == _rd(0.2) and c.rd_contact == _rd(1e-6)
    lim = (5000.0, 7500.0, 10000.0, 10000.0)[subtask]
    assert c.rd_limit == _rd(lim) and c.limit == lim
    if art:
        span = qmax - qmin
        ofr = 0.75 if art == 1 else 0.9
        assert c.open_cut == ofr * span + qmin
        assert c.ru_open == _ru(ofr * span + qmin)
        assert c.rd_closed == _rd(0.01 * span + qmin)
        # the f32 boundary cases of SURVEY 8(c)
        x = np.float32(0.45)
        if art == 2:
            assert (float(x) >= c.open_cut) == (x >= np.float32(c.ru_open))


def test_status_names_and_scratch_sizes():
    from paper_2412_13211_b200 import _lib as L
    lib = L.lib()
    assert lib.tl_status_name(0) == b"OK"
    assert lib.tl_status_name(1) == b"TooShort"
    assert lib.tl_status_name(4) == b"RequiredFieldNaN"
    assert lib.tl_status_name(30) == b"InfeasibleScript"
    assert lib.tl_scan_scratch_bytes(10 ** 6) >= 8 * (10 ** 6 // 1024)
    cfg = L.FuzzCfg_c(8, 4, 5, 0, 1.0, 0.5)
    assert lib.tl_fuzz_scratch_bytes(1024, ctypes.byref(cfg)) >= 1024 * 624 * 4
    assert lib.tl_realize_scratch_bytes(10) >= 10 * 624 * 4


def test_entry_points_reject_bad_arguments_without_a_gpu():
    """argument validation returns TL_E_INVALID before touching the device"""
    from paper_2412_13211_b200 import _lib as L
    lib = L.lib()
    assert lib.tl_label_records(None, 1, None, None, 0, None, None, None, None, None) == L.E_INVALID
    assert lib.tl_filter_select(None, 5, 1, 1, None, None, 1, None, None, None, None) == L.E_INVALID
