"""Per-timestep predicates (mirror of trajlab.predicates, predicates.py:16-99).

Each call evaluates the record(s) on the GPU with tl_eval_predicates (the
same device code the label kernel uses) and maps the device error bits to
the reference exceptions.
"""
from __future__ import annotations

import math

from . import core
from .errors import MissingArticulation, RequiredFieldNaN
from .model import SUBTASK_ORDER, ART_ORDER, SCALAR_FIELDS, SubtaskKind, TimestepRecord, Trajectory, TrajectoryHeader
from .thresholds import Thresholds

_B_CONTACT, _B_GRASP, _B_SUCC, _B_CUM_LE, _B_CUM_GT, _B_A, _B_B, _B_STATIC = (
    1, 2, 4, 8, 16, 32, 64, 128)
_E_SUCC, _E_FORCE, _E_DIST, _E_ART = 1, 2, 4, 8


def _blank(dof, **kw):
    base = dict(t=0, q_arm=(0.0,) * dof, qd_arm=(0.0,) * dof, q_tor=0.0,
                v_base_x=0.0, v_base_y=0.0, omega_base=0.0, dist_ee_rest=0.0,
                dist_obj_goal=0.0, force_ee_target=0.0, cum_robot_force=0.0,
                art_q=0.0, grasped=False)
    base.update(kw)
    return TimestepRecord(**base)


def _eval(rec, hdr, th, subtask=None, a0=None):
    """(bits, errs, jmax) of one record under hdr/th (subtask overridable):
    one staged launch (core.one_record)."""
    dof = hdr.arm_dof
    if len(rec.q_arm) != dof or len(rec.qd_arm) != dof:
        raise ValueError(f"joint vector length mismatch: {len(rec.q_arm)} vs {dof}")
    if len(hdr.rest_arm) != dof:
        raise ValueError(f"joint vector length mismatch: {dof} vs {len(hdr.rest_arm)}")
    sub = hdr.subtask_kind if subtask is None else subtask
    one = core.one_record()
    cs = one.cset(SUBTASK_ORDER.index(sub), ART_ORDER.index(hdr.articulation_kind),
                  hdr.art_qmin, hdr.art_qmax, dof, hdr.rest_arm, hdr.rest_tor, th)
    values = [*rec.q_arm, *rec.qd_arm, *(getattr(rec, f) for f in SCALAR_FIELDS)]
    return one.eval(values, rec.grasped, dof, cs, a0)


def j_max(q, r) -> float:
    """max_i |q_i - r_i| (predicates.py:16-20)."""
    if len(q) != len(r):
        raise ValueError(f"joint vector length mismatch: {len(q)} vs {len(r)}")
    if len(q) == 0:
        return 0.0
    hdr = TrajectoryHeader(episode_id="", arm_dof=len(q), rest_arm=tuple(r))
    return _eval(_blank(len(q), q_arm=tuple(q)), hdr, Thresholds())[2]


def is_static(rec: TimestepRecord, th: Thresholds) -> bool:
    hdr = TrajectoryHeader(episode_id="", arm_dof=len(rec.qd_arm))
    r = _blank(len(rec.qd_arm), qd_arm=tuple(rec.qd_arm), v_base_x=rec.v_base_x,
               v_base_y=rec.v_base_y, omega_base=rec.omega_base)
    return bool(_eval(r, hdr, th)[0] & _B_STATIC)


def _art_pred(a_q, hdr, th, subtask, bit, a0=None):
    bits, errs, _ = _eval(_blank(hdr.arm_dof, art_q=a_q), hdr, th, subtask, a0)
    if not hdr.has_articulation:
        raise MissingArticulation(f"{hdr.subtask_kind.value} predicate needs an articulation")
    if errs & _E_ART:
        raise RequiredFieldNaN("field art_q is NaN but required by this subtask")
    return bool(bits & bit)


def is_open(a_q: float, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    return _art_pred(a_q, hdr, th, SubtaskKind.Open, _B_A)


def is_closed(a_q: float, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    return _art_pred(a_q, hdr, th, SubtaskKind.Close, _B_A)


def slightly_opened(a_q: float, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    return _art_pred(a_q, hdr, th, SubtaskKind.Open, _B_B)


def slightly_closed(a_q: float, a_q0: float, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    return _art_pred(a_q, hdr, th, SubtaskKind.Close, _B_B, a0=a_q0)


def success_step(rec: TimestepRecord, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    """Per-step success condition (predicates.py:75-94)."""
    bits, errs, _ = _eval(rec, hdr, th)
    if errs & _E_SUCC:
        if hdr.subtask_kind == SubtaskKind.Place:
            raise RequiredFieldNaN("field dist_obj_goal is NaN but required by this subtask")
        if not hdr.has_articulation:
            raise MissingArticulation(f"{hdr.subtask_kind.value} predicate needs an articulation")
        raise RequiredFieldNaN("field art_q is NaN but required by this subtask")
    return bool(bits & _B_SUCC)


def failure_step(rec: TimestepRecord, hdr: TrajectoryHeader, th: Thresholds) -> bool:
    """cum_robot_force strictly above the subtask limit (predicates.py:97-99)."""
    return bool(_eval(rec, hdr, th)[0] & _B_CUM_GT)
