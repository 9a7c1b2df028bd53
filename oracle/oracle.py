"""ctypes wrapper over the C oracle (oracle.c).

TEST INFRASTRUCTURE ONLY.  The oracle is the CPU restatement of the
reference trajlab hot path used as the parity checker.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module; the product package never does.

Codes are plain ints so this module has no dependency on the product.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

MAX_DOF = 16
PICK, PLACE, OPEN, CLOSE = 0, 1, 2, 3
SUBTASKS = ("Pick", "Place", "Open", "Close")
ART_NONE, ART_FRIDGE, ART_DRAWER = 0, 1, 2
ART_KINDS = ("None", "Fridge", "Drawer")
EVENT_KINDS = ("Contact", "Grasped", "Dropped", "ObjAtGoal", "ReleasedAtGoal",
               "ReleasedOutsideGoal", "ObjLeftGoal", "Opened", "SlightlyOpened",
               "Closed", "SlightlyClosed", "Open", "Success",
               "ExcessiveCollisions")
LEVELS = ("low", "slight", "open", "high", "closed")
THRESHOLD_FIELDS = (
    "rest_radius", "goal_radius", "j_arm_pick", "j_arm_other", "j_tor_max",
    "static_qd_arm", "static_v_base", "static_omega", "coll_pick",
    "coll_place", "coll_artic", "open_frac_fridge", "open_frac_drawer",
    "close_frac", "slightly_open_frac", "slightly_close_frac", "contact_eps")
DEFAULT_THRESHOLDS = dict(
    rest_radius=0.05, goal_radius=0.15, j_arm_pick=0.6, j_arm_other=0.2,
    j_tor_max=0.01, static_qd_arm=0.2, static_v_base=0.05, static_omega=0.05,
    coll_pick=5000.0, coll_place=7500.0, coll_artic=10000.0,
    open_frac_fridge=0.75, open_frac_drawer=0.9, close_frac=0.01,
    slightly_open_frac=0.1, slightly_close_frac=0.05, contact_eps=1e-6)
MODE_IDS = (
    "pick.s1_straightforward", "pick.s2_winding", "pick.s3_success_then_drop",
    "pick.s4_success_then_excessive_collisions", "pick.f5_excessive_collisions",
    "pick.f6_mobility", "pick.f7_cant_grasp", "pick.f8_drop", "pick.f9_too_slow",
    "place.s1_place_in_goal", "place.s2_drop_to_goal", "place.s3_dubious",
    "place.s4_winding", "place.s5_success_then_excessive_collisions",
    "place.f6_excessive_collisions", "place.f7_didnt_grasp",
    "place.f8_didnt_reach_goal", "place.f9_place_in_goal",
    "place.f10_drop_to_goal", "place.f11_wont_let_go", "place.f12_too_slow",
    "open.s1_open", "open.s2_dubious", "open.s3_success_then_excessive_collisions",
    "open.f4_excessive_collisions", "open.f5_cant_reach",
    "open.f6_closed_after_open", "open.f7_slightly_opened", "open.f8_too_slow",
    "open.f9_cant_open",
    "close.s1_close", "close.s2_dubious",
    "close.s3_success_then_excessive_collisions",
    "close.f4_excessive_collisions", "close.f5_cant_reach",
    "close.f6_opened_after_closed", "close.f7_slightly_closed",
    "close.f8_too_slow", "close.f9_cant_close")

REC_DTYPE = np.dtype([
    ("q_arm", "<f8", (MAX_DOF,)), ("qd_arm", "<f8", (MAX_DOF,)),
    ("q_tor", "<f8"), ("v_base_x", "<f8"), ("v_base_y", "<f8"),
    ("omega_base", "<f8"), ("dist_ee_rest", "<f8"), ("dist_obj_goal", "<f8"),
    ("force_ee_target", "<f8"), ("cum_robot_force", "<f8"), ("art_q", "<f8"),
    ("grasped", "<i4"), ("pad", "<i4")])
SCALAR_FIELDS = ("q_tor", "v_base_x", "v_base_y", "omega_base", "dist_ee_rest",
                 "dist_obj_goal", "force_ee_target", "cum_robot_force", "art_q")


class _Thresholds(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in THRESHOLD_FIELDS]


class _Header(ctypes.Structure):
    _fields_ = [("subtask", ctypes.c_int32), ("art_kind", ctypes.c_int32),
                ("arm_dof", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("art_qmin", ctypes.c_double), ("art_qmax", ctypes.c_double),
                ("rest_tor", ctypes.c_double),
                ("rest_arm", ctypes.c_double * MAX_DOF)]


class _Script(ctypes.Structure):
    _fields_ = [("subtask", ctypes.c_int32), ("n_steps", ctypes.c_int32),
                ("tail", ctypes.c_int32), ("initial_grasped", ctypes.c_int32),
                ("initial_contact", ctypes.c_int32),
                ("initial_level", ctypes.c_int32), ("art_kind", ctypes.c_int32),
                ("arm_dof", ctypes.c_int32),
                ("initial_dist_obj_goal", ctypes.c_double),
                ("step_kind", ctypes.POINTER(ctypes.c_uint8)),
                ("step_gap", ctypes.POINTER(ctypes.c_int32))]


class _FuzzCfg(ctypes.Structure):
    _fields_ = [("max_events", ctypes.c_int32), ("max_gap", ctypes.c_int32),
                ("max_tail", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("edge_density", ctypes.c_double),
                ("success_prob", ctypes.c_double)]


class _MT(ctypes.Structure):
    _fields_ = [("mt", ctypes.c_uint32 * 624), ("index", ctypes.c_int32)]


class OracleError(Exception):
    def __init__(self, code, step=-1):
        super().__init__(f"oracle status {code} (step {step})")
        self.code = code
        self.step = step


def build():
    """Compile liboracle.so (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        L.or_mt_seed.argtypes = [P(_MT), ctypes.c_int64]
        L.or_mt_genrand.argtypes = [P(_MT)]
        L.or_mt_genrand.restype = ctypes.c_uint32
        L.or_mt_random.argtypes = [P(_MT)]
        L.or_mt_random.restype = ctypes.c_double
        L.or_random_script.argtypes = [ctypes.c_int64, ctypes.c_int32, P(_FuzzCfg),
                                       P(_Script), ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int32]
        L.or_random_script.restype = ctypes.c_int32
        L.or_realize.argtypes = [P(_Script), ctypes.c_int64, P(_Thresholds),
                                 ctypes.c_void_p, ctypes.c_int64, P(ctypes.c_int32)]
        L.or_realize.restype = ctypes.c_int64
        L.or_realize_len.argtypes = [P(_Script)]
        L.or_realize_len.restype = ctypes.c_int64
        L.or_success_step.argtypes = [ctypes.c_void_p, P(_Header), P(_Thresholds),
                                      P(ctypes.c_int32)]
        L.or_success_step.restype = ctypes.c_int32
        L.or_extract_events.argtypes = [ctypes.c_void_p, ctypes.c_int64, P(_Header),
                                        P(_Thresholds), ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_int32,
                                        P(ctypes.c_double)]
        L.or_extract_events.restype = ctypes.c_int32
        L.or_classify.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                  ctypes.c_double, ctypes.c_int32, ctypes.c_void_p,
                                  ctypes.c_int32, P(ctypes.c_int32),
                                  P(ctypes.c_int32)]
        L.or_classify.restype = ctypes.c_int32
        L.or_filter_select.argtypes = [ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int32, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p]
        L.or_filter_select.restype = ctypes.c_int64
        L.or_fuzz_label_batch.argtypes = [ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int32, P(_FuzzCfg),
                                          P(_Thresholds), ctypes.c_int32,
                                          ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
        L.or_fuzz_label_batch.restype = ctypes.c_int64
        L.or_fuzz_label_batch_ex.argtypes = [ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int32, P(_FuzzCfg),
                                             P(_Thresholds), ctypes.c_int32,
                                             ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p]
        L.or_fuzz_label_batch_ex.restype = ctypes.c_int64
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def thresholds(th=None):
    d = dict(DEFAULT_THRESHOLDS)
    if th:
        d.update(th)
    return _Thresholds(*[float(d[n]) for n in THRESHOLD_FIELDS])


def fuzz_cfg(max_events=8, max_gap=4, max_tail=5, edge_density=1.0,
             success_prob=0.5):
    return _FuzzCfg(max_events, max_gap, max_tail, 0, float(edge_density),
                    float(success_prob))


# -- MT19937 ----------------------------------------------------------------

class MT:
    def __init__(self, seed):
        self.s = _MT()
        lib().or_mt_seed(ctypes.byref(self.s), int(seed))

    def genrand(self):
        return lib().or_mt_genrand(ctypes.byref(self.s))

    def random(self):
        return lib().or_mt_random(ctypes.byref(self.s))


# -- scripts ----------------------------------------------------------------

def random_script(seed, subtask, cfg=None):
    """dict script (synth.py:363-507)."""
    cfg = cfg or fuzz_cfg()
    cap = cfg.max_events + 8
    sk = np.zeros(cap, np.uint8)
    sg = np.zeros(cap, np.int32)
    s = _Script()
    n = lib().or_random_script(int(seed), int(subtask), ctypes.byref(cfg),
                               ctypes.byref(s), _ptr(sk), _ptr(sg), cap)
    if n < 0:
        raise OracleError(-1)
    return dict(subtask=subtask, kinds=sk[:n].copy(), gaps=sg[:n].copy(),
                tail=s.tail, initial_grasped=s.initial_grasped,
                initial_contact=s.initial_contact,
                initial_dist_obj_goal=s.initial_dist_obj_goal,
                initial_level=s.initial_level, art_kind=s.art_kind,
                arm_dof=s.arm_dof)


def _script_struct(sc):
    kinds = np.ascontiguousarray(sc["kinds"], np.uint8)
    gaps = np.ascontiguousarray(sc["gaps"], np.int32)
    s = _Script(int(sc["subtask"]), len(kinds), int(sc["tail"]),
                int(sc["initial_grasped"]), int(sc["initial_contact"]),
                int(sc["initial_level"]), int(sc["art_kind"]),
                int(sc.get("arm_dof", 7)), float(sc["initial_dist_obj_goal"]),
                kinds.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                gaps.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return s, (kinds, gaps)


def realize(sc, seed, th=None):
    """records (structured REC_DTYPE array) for a script (synth.py:345)."""
    s, keep = _script_struct(sc)
    n = lib().or_realize_len(ctypes.byref(s))
    out = np.zeros(max(n, 2), REC_DTYPE)
    es = ctypes.c_int32(-1)
    got = lib().or_realize(ctypes.byref(s), int(seed), ctypes.byref(thresholds(th)),
                           _ptr(out), len(out), ctypes.byref(es))
    if got < 0:
        raise OracleError(int(-got), es.value)
    return out[:got]


def fuzz(seed, subtask, cfg=None, th=None):
    sc = random_script(seed, subtask, cfg)
    return sc, realize(sc, int(seed) ^ 0x5EED, th)


# -- labelling ----------------------------------------------------------------

def header(subtask, art_kind=ART_NONE, art_qmin=math.nan, art_qmax=math.nan,
           arm_dof=7, rest_arm=None, rest_tor=0.0):
    h = _Header()
    h.subtask, h.art_kind, h.arm_dof = int(subtask), int(art_kind), int(arm_dof)
    h.art_qmin, h.art_qmax, h.rest_tor = float(art_qmin), float(art_qmax), float(rest_tor)
    for i, v in enumerate(rest_arm if rest_arm is not None else [0.0] * arm_dof):
        h.rest_arm[i] = float(v)
    return h


def synth_header(sc):
    k = int(sc["subtask"])
    if k in (OPEN, CLOSE):
        qmax = 1.6 if sc["art_kind"] == ART_FRIDGE else 0.5
        return header(k, sc["art_kind"], 0.0, qmax, sc.get("arm_dof", 7))
    return header(k, ART_NONE, arm_dof=sc.get("arm_dof", 7))


def extract_events(recs, hdr, th=None):
    """(kinds u8[], ts i32[], d0) or raises OracleError (events.py:94)."""
    recs = np.ascontiguousarray(recs, REC_DTYPE)
    cap = max(4 * len(recs), 8)
    ek = np.zeros(cap, np.uint8)
    et = np.zeros(cap, np.int32)
    d0 = ctypes.c_double(math.nan)
    n = lib().or_extract_events(_ptr(recs), len(recs), ctypes.byref(hdr),
                                ctypes.byref(thresholds(th)), _ptr(ek), _ptr(et),
                                cap, ctypes.byref(d0))
    if n < 0:
        raise OracleError(-n)
    return ek[:n].copy(), et[:n].copy(), d0.value


def classify(subtask, kinds, d0=math.nan, d0_none=False, rule_order=None):
    """(mode_id int, success_once, success_at_end) (modes.py:235)."""
    kinds = np.ascontiguousarray(kinds, np.uint8)
    ro = None if rule_order is None else np.ascontiguousarray(rule_order, np.int32)
    so, se = ctypes.c_int32(), ctypes.c_int32()
    m = lib().or_classify(int(subtask), _ptr(kinds), len(kinds), float(d0),
                          int(d0_none), _ptr(ro), 0 if ro is None else len(ro),
                          ctypes.byref(so), ctypes.byref(se))
    if m < 0:
        raise OracleError(-m)
    return m, bool(so.value), bool(se.value)


def success_step(rec, hdr, th=None):
    rec = np.ascontiguousarray(np.asarray(rec, REC_DTYPE).reshape(1))
    err = ctypes.c_int32(0)
    v = lib().or_success_step(_ptr(rec), ctypes.byref(hdr),
                              ctypes.byref(thresholds(th)), ctypes.byref(err))
    if err.value:
        raise OracleError(err.value)
    return bool(v)


def filter_select(pool, subtask, rule, n_pools, rule_w, n_rules, quota):
    """selected mask + per-pool counts (pipeline.py:276-338)."""
    pool = np.ascontiguousarray(pool, np.int32)
    subtask = np.ascontiguousarray(subtask, np.int32)
    rule = np.ascontiguousarray(rule, np.int32)
    rule_w = np.ascontiguousarray(rule_w, np.float64)
    n_rules = np.ascontiguousarray(n_rules, np.int32)
    sel = np.zeros(len(pool), np.uint8)
    ps = np.zeros(max(n_pools, 1), np.int64)
    lib().or_filter_select(len(pool), _ptr(pool), _ptr(subtask), _ptr(rule),
                           int(n_pools), _ptr(rule_w), _ptr(n_rules), int(quota),
                           _ptr(sel), _ptr(ps))
    return sel.astype(bool), ps[:n_pools]


def fuzz_label_batch(seed0, n, subtask, cfg=None, th=None, n_threads=1,
                     want_outputs=True):
    """CPU baseline: fuzz -> extract_events -> classify for n seeds."""
    cfg = cfg or fuzz_cfg()
    modes = np.zeros(n, np.uint8) if want_outputs else None
    nev = np.zeros(n, np.int32) if want_outputs else None
    nrec = np.zeros(n, np.int64) if want_outputs else None
    total = lib().or_fuzz_label_batch(int(seed0), int(n), int(subtask),
                                      ctypes.byref(cfg), ctypes.byref(thresholds(th)),
                                      int(n_threads), _ptr(modes), _ptr(nev),
                                      _ptr(nrec))
    return total, modes, nev, nrec


def fuzz_label_batch_full(seed0, n, subtask, cfg=None, th=None, n_threads=1):
    """fuzz -> extract_events -> classify for seeds [seed0, seed0+n): dict of
    mode, n_events, n_rec, flags (bit 0 success_once, bit 1 success_at_end),
    d0, and the event lists in CSR form (ev_off, ev_kind, ev_t)."""
    cfg = cfg or fuzz_cfg()
    stride = 4 * (1 + (cfg.max_events + 8) * cfg.max_gap + cfg.max_tail + 2)
    modes = np.zeros(n, np.uint8)
    nev = np.zeros(n, np.int32)
    nrec = np.zeros(n, np.int64)
    flags = np.zeros(n, np.uint8)
    d0 = np.zeros(n, np.float64)
    ek = np.zeros(n * stride, np.uint8)
    et = np.zeros(n * stride, np.int32)
    lib().or_fuzz_label_batch_ex(int(seed0), int(n), int(subtask), ctypes.byref(cfg),
                                 ctypes.byref(thresholds(th)), int(n_threads), _ptr(modes),
                                 _ptr(nev), _ptr(nrec), _ptr(flags), _ptr(d0), stride,
                                 _ptr(ek), _ptr(et))
    cnt = np.maximum(nev, 0).astype(np.int64)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=off[1:])
    take = (np.arange(n * stride) % stride) < np.repeat(cnt, stride)
    return dict(mode=modes, n_events=nev, n_rec=nrec, flags=flags, d0=d0,
                ev_off=off, ev_kind=ek[take], ev_t=et[take])
