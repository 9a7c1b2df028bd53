"""Loader for libtrajlab_b200.so (the sm_100a CUDA kernels behind the C ABI
declared in include/trajlab_b200.h).

There is no CPU fallback: every compute entry point of this package goes
through this library and raises NativeUnavailable when it cannot be loaded
or when no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# TRAJLAB_B200_LIB selects another build of the same library (the checked
# build of scripts/gpu_check_build.sh); default: the in-tree product build
LIB_PATH = os.environ.get("TRAJLAB_B200_LIB") or os.path.join(PKG, "libtrajlab_b200.so")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC", "-shared"]

MAX_DOF = 16
N_MODES = 39

# ---- status codes (include/trajlab_b200.h) ----------------------------------
OK = 0
ERR_TOO_SHORT = 1
ERR_NAN_SUCCESS_DIST = 2
ERR_NAN_ART = 3
ERR_NAN_FORCE = 4
ERR_NAN_PLACE_DIST = 5
ERR_MISSING_ART = 6
ERR_MODE_COVERAGE = 7
ERR_D0_NONE_LE = 8
ERR_D0_NONE_GT = 9
INF_FIRST, INF_LAST = 20, 41
ERR_SCRIPT_CAPACITY = 50
E_INVALID, E_CUDA, E_CAPACITY = 100, 101, 102
ACT_HOLD, ACT_IDLE, ACT_BAD_GAP = 255, 254, 253


class NativeUnavailable(RuntimeError):
    """The CUDA library (or a CUDA device) is missing: no fallback exists."""


class NativeCallError(RuntimeError):
    pass


class Thresholds_c(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in (
        "rest_radius", "goal_radius", "j_arm_pick", "j_arm_other", "j_tor_max",
        "static_qd_arm", "static_v_base", "static_omega", "coll_pick",
        "coll_place", "coll_artic", "open_frac_fridge", "open_frac_drawer",
        "close_frac", "slightly_open_frac", "slightly_close_frac",
        "contact_eps")]


class Cset_c(ctypes.Structure):
    _fields_ = ([("subtask", ctypes.c_int32), ("art_kind", ctypes.c_int32),
                 ("dof", ctypes.c_int32), ("rest_zero", ctypes.c_int32)] +
                [(n, ctypes.c_float) for n in (
                    "rd_rest_radius", "rd_goal", "rd_static_qd", "rd_static_v",
                    "rd_static_om", "rd_limit", "rd_contact", "ru_open",
                    "rd_closed", "ru_slight_open", "rd_j_arm", "rd_j_tor")] +
                [(n, ctypes.c_double) for n in (
                    "rest_radius", "goal_radius", "static_qd", "static_v",
                    "static_om", "limit", "contact_eps", "open_cut",
                    "closed_cut", "slight_open_cut", "j_arm", "j_tor",
                    "rest_tor", "scf_span", "pad0")] +
                [("rest_arm", ctypes.c_double * MAX_DOF)])


class Records_c(ctypes.Structure):
    _fields_ = [("planes", ctypes.c_void_p), ("grasped", ctypes.c_void_p),
                ("rec_start", ctypes.c_void_p), ("n_rec", ctypes.c_void_p),
                ("plane_stride", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("dof", ctypes.c_int32)]


class Rules_c(ctypes.Structure):
    _fields_ = [("count", (ctypes.c_int8 * 2) * 4),
                ("ids", ((ctypes.c_int8 * 16) * 2) * 4)]


class FuzzCfg_c(ctypes.Structure):
    _fields_ = [("max_events", ctypes.c_int32), ("max_gap", ctypes.c_int32),
                ("max_tail", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("edge_density", ctypes.c_double),
                ("success_prob", ctypes.c_double)]


# numpy views of device structs
LABEL_DTYPE = np.dtype([("status", "<i4"), ("n_events", "<i4"),
                        ("err_index", "<i4"), ("subtask", "u1"), ("mode", "u1"),
                        ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")])
SCRIPT_DTYPE = np.dtype([("step_off", "<i8"), ("seed", "<i8"),
                         ("n_steps", "<i4"), ("tail", "<i4"),
                         ("subtask", "<i4"), ("art_kind", "<i4"),
                         ("initial_level", "<i4"), ("initial_grasped", "<i4"),
                         ("initial_contact", "<i4"), ("arm_dof", "<i4"),
                         ("initial_dist_obj_goal", "<f8")])
VBOUNDS_DTYPE = np.dtype([("art_qmin", "<f8"), ("art_qmax", "<f8"), ("has_art", "<i4"),
                          ("pad", "<i4")])
VSUMMARY_DTYPE = np.dtype([("n_error_records", "<i4"), ("n_warning_records", "<i4"),
                           ("first_flagged", "<i4"), ("too_short", "<i4")])
# tl_validate_records per-record codes (TL_VF_*)
VF_T_MISMATCH, VF_ARM_LENGTH, VF_CUM_INVALID, VF_CUM_DECREASED = 1, 2, 4, 8
VF_DEE_INVALID, VF_DOG_NEGATIVE, VF_FET_NEGATIVE, VF_ART_RANGE = 16, 32, 64, 128
assert LABEL_DTYPE.itemsize == 24 and SCRIPT_DTYPE.itemsize == 56
CSET_BYTES = ctypes.sizeof(Cset_c)


def build(verbose=False):
    """Compile libtrajlab_b200.so in-tree for sm_100a (nvcc cross-compiles
    without a GPU)."""
    cmd = ["nvcc", *NVCC_FLAGS, "-I", INCLUDE, "-o", LIB_PATH,
           os.path.join(CSRC, "trajlab_b200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib():
    """The loaded library; raises NativeUnavailable (never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing; run __graft_entry__.build() "
            "(this package has no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, P = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER
    sig = {
        "tl_abi_version": ([], ctypes.c_int),
        "tl_status_name": ([ctypes.c_int], ctypes.c_char_p),
        "tl_device_sm_count": ([], ctypes.c_int),
        "tl_cset_build": ([i32, i32, ctypes.c_double, ctypes.c_double, i32, vp,
                           ctypes.c_double, P(Thresholds_c), P(Cset_c)], ctypes.c_int),
        "tl_label_records": ([P(Records_c), i32, vp, vp, i32, vp, vp, vp, vp, vp],
                             ctypes.c_int),
        "tl_scan_scratch_bytes": ([i32], ctypes.c_size_t),
        "tl_scan_events": ([vp, i32, vp, vp, vp], ctypes.c_int),
        "tl_emit_events": ([vp, vp, vp, vp, vp, i32, vp, vp, vp], ctypes.c_int),
        "tl_scan_emit_events": ([vp, vp, vp, vp, i32, vp, vp, vp, vp, vp], ctypes.c_int),
        "tl_classify_events": ([vp, vp, vp, vp, vp, i32, vp, vp, vp], ctypes.c_int),
        "tl_fuzz_scratch_bytes": ([i32, P(FuzzCfg_c)], ctypes.c_size_t),
        "tl_fuzz": ([vp, i32, i32, P(FuzzCfg_c), P(Thresholds_c), vp, vp,
                     P(Records_c), i32, vp, vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "tl_fuzz_ev": ([vp, i32, i32, P(FuzzCfg_c), P(Thresholds_c), vp, vp,
                        P(Records_c), i32, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp],
                       ctypes.c_int),
        "tl_fuzz_mixed": ([vp, vp, i32, P(FuzzCfg_c), P(Thresholds_c), vp, vp,
                           P(Records_c), i32, vp, vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "tl_fuzz_ev_mixed": ([vp, vp, i32, P(FuzzCfg_c), P(Thresholds_c), vp, vp,
                              P(Records_c), i32, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp],
                             ctypes.c_int),
        "tl_realize_scratch_bytes": ([i32], ctypes.c_size_t),
        "tl_realize": ([vp, vp, vp, i32, P(Thresholds_c), vp, vp, P(Records_c),
                        vp, vp, vp, vp], ctypes.c_int),
        "tl_filter_scratch_bytes": ([i64, i32, i32], ctypes.c_size_t),
        "tl_filter_select": ([vp, i64, i32, i32, vp, vp, i64, vp, vp, vp, vp],
                             ctypes.c_int),
        "tl_mode_histogram": ([vp, i32, vp, vp], ctypes.c_int),
        "tl_scan_counts": ([vp, i32, vp, vp, vp], ctypes.c_int),
        "tl_compact_records": ([P(Records_c), i32, vp, P(Records_c), vp], ctypes.c_int),
        "tl_eval_predicates": ([P(Records_c), i32, vp, vp, vp, vp, vp, vp, vp],
                               ctypes.c_int),
        "tl_env_state_bytes": ([i32], ctypes.c_size_t),
        "tl_env_reset": ([vp, i32, i32, vp, P(Thresholds_c), vp, vp, i64, vp, vp, vp],
                         ctypes.c_int),
        "tl_env_reset_fuzz": ([vp, vp, i32, i32, P(FuzzCfg_c), P(Thresholds_c), vp, vp,
                               vp, vp, vp, i64, vp, vp, vp], ctypes.c_int),
        "tl_env_step": ([vp, i32, i32, vp, i32, vp, i64, vp, vp, vp], ctypes.c_int),
        "tl_env_labels": ([vp, i32, vp, vp, vp, vp], ctypes.c_int),
        "tl_env_script_actions": ([vp, vp, vp, i32, i32, i32, vp, vp], ctypes.c_int),
        "tl_group_mode_counts": ([vp, vp, i64, i32, vp, vp], ctypes.c_int),
        "tl_chain_progress": ([vp, vp, i64, i32, vp, vp], ctypes.c_int),
        "tl_filter_buckets": ([vp, vp, i64, vp, vp, vp, i32, vp, vp], ctypes.c_int),
        "tl_allgather_labels": ([vp, vp, i64, vp, vp], ctypes.c_int),
        "tl_allreduce_counts": ([vp, vp, i64, vp], ctypes.c_int),
        "tl_validate_records": ([P(Records_c), i32, vp, vp, vp, vp, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.tl_abi_version() != 1:
        raise NativeUnavailable("ABI version mismatch")
    _lib = L
    return L


def exported_symbols():
    return ["tl_abi_version", "tl_status_name", "tl_device_sm_count",
            "tl_cset_build", "tl_label_records", "tl_scan_scratch_bytes",
            "tl_scan_events", "tl_emit_events", "tl_classify_events", "tl_fuzz",
            "tl_realize", "tl_filter_scratch_bytes", "tl_filter_select",
            "tl_mode_histogram", "tl_eval_predicates", "tl_scan_counts",
            "tl_compact_records", "tl_fuzz_scratch_bytes", "tl_realize_scratch_bytes",
            "tl_scan_emit_events", "tl_env_state_bytes", "tl_env_reset",
            "tl_env_reset_fuzz", "tl_env_step", "tl_env_labels", "tl_env_script_actions",
            "tl_group_mode_counts", "tl_chain_progress", "tl_filter_buckets", "tl_fuzz_ev",
            "tl_fuzz_mixed", "tl_fuzz_ev_mixed",
            "tl_allgather_labels", "tl_allreduce_counts", "tl_validate_records"]


def check(rc, what):
    if rc != OK:
        name = lib().tl_status_name(rc).decode()
        raise NativeCallError(f"{what} failed: {name} ({rc})")


def device():
    """The CUDA device all compute runs on (raises if there is none)."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: trajlab_b200 runs only on a GPU "
                                "(there is no CPU fallback)")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None
