"""Per-timestep predicates (mirror of trajlab.predicates, predicates.py:16-99).

Each call evaluates the record(s) on the GPU with tl_eval_predicates (the
same device code the label kernel uses) and maps the device error bits to
the reference exceptions.
"""
from __future__ import annotations

import math

from . import core
from .errors import MissingArticulation, RequiredFieldNaN
from .model import SUBTASK_ORDER, ART_ORDER, SubtaskKind, TimestepRecord, Trajectory, TrajectoryHeader
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
    """(bits, errs, jmax) of one record under hdr/th (subtask overridable)."""
    h = hdr
    if subtask is not None and subtask != hdr.subtask_kind:
        h = TrajectoryHeader(episode_id="", subtask_kind=subtask,
                             articulation_kind=hdr.articulation_kind,
                             art_qmin=hdr.art_qmin, art_qmax=hdr.art_qmax,
                             arm_dof=hdr.arm_dof, rest_arm=hdr.rest_arm,
                             rest_tor=hdr.rest_tor)
    t = Trajectory(header=TrajectoryHeader(
        episode_id="", subtask_kind=h.subtask_kind, articulation_kind=h.articulation_kind,
        art_qmin=h.art_qmin, art_qmax=h.art_qmax, arm_dof=h.arm_dof,
        rest_arm=h.rest_arm, rest_tor=h.rest_tor, thresholds_override=th),
        records=[rec])
    rb, env, cs, _ = core.pack_trajectories([t], th, force_f64=True)
    bits, errs, jmax = core.eval_predicates(rb, env, cs, None if a0 is None else [a0])
    return int(bits[0].item()), int(errs[0].item()), float(jmax[0].item())


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
