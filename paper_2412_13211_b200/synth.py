"""Synthetic episode generation (mirror of trajlab.synth, synth.py:57-602):
the env reset/step analogue.

realize / fuzz / random_script run in the fused sm_100a generator
(csrc/tl_synth.cuh): CPython-exact MT19937 draws, the _Realizer state
machine and online labelling, one warp per episode.  The single-episode
functions are batches of one; realize_many / fuzz_many are the batched
forms (one launch for N episodes).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L
from . import core
from .errors import InfeasibleScript, infeasible_error
from .events import EVENT_KINDS, EventKind
from .model import (ART_ORDER, SUBTASK_ORDER, ArticulationKind, SubtaskKind, Task,
                    TimestepRecord, Trajectory, TrajectoryHeader)
from .thresholds import Thresholds

LEVELS = ("low", "slight", "open", "high", "closed")
_ART_BOUNDS = {ArticulationKind.Fridge: (0.0, 1.6), ArticulationKind.Drawer: (0.0, 0.5)}


@dataclass
class ScriptStep:
    kind: EventKind
    gap: int = 2


@dataclass
class EventScript:
    subtask_kind: SubtaskKind
    steps: list = field(default_factory=list)
    tail: int = 3
    initial_grasped: bool = False
    initial_contact: bool = False
    initial_dist_obj_goal: float = 0.5
    initial_art_level: str = "low"
    articulation_kind: ArticulationKind = ArticulationKind.Fridge
    episode_id: str = "synth-0"
    arm_dof: int = 7

    @classmethod
    def from_dict(cls, d: dict) -> "EventScript":
        return cls(
            subtask_kind=SubtaskKind(d["subtask"]),
            steps=[ScriptStep(EventKind(s["kind"]), int(s.get("gap", 2)))
                   for s in d.get("events", [])],
            tail=int(d.get("tail", 3)),
            initial_grasped=bool(d.get("initial_grasped", False)),
            initial_contact=bool(d.get("initial_contact", False)),
            initial_dist_obj_goal=float(d.get("initial_dist_obj_goal", 0.5)),
            initial_art_level=d.get("initial_art_level", "low"),
            articulation_kind=ArticulationKind(d.get("articulation_kind", "Fridge")),
            episode_id=d.get("episode_id", "synth-0"),
            arm_dof=int(d.get("arm_dof", 7)))


@dataclass
class FuzzConfig:
    max_events: int = 8
    max_gap: int = 4
    max_tail: int = 5
    edge_density: float = 1.0
    success_prob: float = 0.5


@dataclass
class NoiseModel:
    """Clipped-Gaussian initial-state perturbations (synth.py:31-40).
    Not on the generation path (realize/fuzz never draw it)."""
    arm_std: float = 0.1
    arm_clip: float = 0.2
    base_std: float = 0.1
    base_clip: float = 0.2
    rot_std: float = 0.25
    rot_clip: float = 0.5
    seed: int = 0


def sample_noise(model: NoiseModel, arm_dof: int = 7, rng=None):
    """(arm perturbation [arm_dof], base (x, y), base rotation) from clipped
    Gaussians (synth.py:43-54).  Host-side: it draws from a CPython
    random.Random (gauss() keeps its own cached second normal), is not on
    the realize/fuzz path, and is only mirrored for API completeness."""
    import random as _random
    r = rng if rng is not None else _random.Random(model.seed)

    def draw(std, lim):
        v = r.gauss(0.0, std)
        return min(lim, v) if v > -lim else -lim

    arm = tuple(draw(model.arm_std, model.arm_clip) for _ in range(arm_dof))
    base = (draw(model.base_std, model.base_clip), draw(model.base_std, model.base_clip))
    return arm, base, draw(model.rot_std, model.rot_clip)


def _label_csets(th_label=None, dof=7):
    key = (th_label or Thresholds()).astuple() + (dof,)
    cache = _label_csets.__dict__.setdefault("cache", {})
    if key not in cache:
        cache[key] = core.synth_csets(th_label or Thresholds(), dof).to_device(L.device())
    return cache[key]


def _script_array(scripts, seeds):
    arr = np.zeros(len(scripts), L.SCRIPT_DTYPE)
    kinds, gaps = [], []
    for i, s in enumerate(scripts):
        k = SubtaskKind(s.subtask_kind)
        if k in (SubtaskKind.Open, SubtaskKind.Close) and \
                ArticulationKind(s.articulation_kind) not in _ART_BOUNDS:
            raise KeyError(ArticulationKind(s.articulation_kind))  # synth.py:112
        lvl = LEVELS.index(s.initial_art_level) if s.initial_art_level in LEVELS else 99
        arr[i] = (len(kinds), int(seeds[i]), len(s.steps), int(s.tail),
                  SUBTASK_ORDER.index(k), ART_ORDER.index(ArticulationKind(s.articulation_kind)),
                  lvl, int(bool(s.initial_grasped)), int(bool(s.initial_contact)),
                  int(s.arm_dof), float(s.initial_dist_obj_goal))
        kinds.extend(EVENT_KINDS.index(EventKind(st.kind)) for st in s.steps)
        gaps.extend(int(st.gap) for st in s.steps)
    return arr, np.asarray(kinds, np.uint8), np.asarray(gaps, np.int32)


def _synth_header(episode_id, kind, art, dof):
    has_art = kind in (SubtaskKind.Open, SubtaskKind.Close)
    qmin, qmax = _ART_BOUNDS[art] if has_art else (math.nan, math.nan)
    return TrajectoryHeader(
        episode_id=episode_id, task=Task.Custom, subtask_kind=kind,
        target_id="synthetic",
        articulation_kind=art if has_art else ArticulationKind.NONE,
        art_qmin=qmin, art_qmax=qmax, arm_dof=dof)


def _to_trajectories(sb, headers):
    """device records -> host Trajectory objects (synth.py:312-342 layout)."""
    planes = sb.records.planes.cpu().numpy()
    grasped = sb.records.grasped.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    nr = sb.records.n_rec.cpu().numpy()
    dof = sb.records.dof
    out = []
    for i, hdr in enumerate(headers):
        p = planes[:, rs[i]:rs[i] + nr[i]].astype(np.float64)
        q = p[:dof].T.tolist()
        qd = p[dof:2 * dof].T.tolist()
        sc = p[2 * dof:].tolist()
        g = grasped[rs[i]:rs[i] + nr[i]].tolist()
        recs = [TimestepRecord(t, tuple(q[t]), tuple(qd[t]), sc[0][t], sc[1][t], sc[2][t],
                               sc[3][t], sc[4][t], sc[5][t], sc[6][t], sc[7][t], sc[8][t],
                               bool(g[t])) for t in range(int(nr[i]))]
        out.append(Trajectory(header=hdr, records=recs))
    return out


def _raise_status(lab, i, script):
    st = int(lab["status"][i])
    step = int(lab["err_index"][i])
    ev = EventKind(script.steps[step].kind).value if 0 <= step < len(script.steps) else None
    raise infeasible_error(st, SubtaskKind(script.subtask_kind).value, ev,
                           script.initial_art_level)


def realize_many(scripts, seeds, th: Optional[Thresholds] = None, strict=True):
    """realize() for many scripts in one launch.  With strict=False,
    infeasible scripts yield their InfeasibleScript instead of raising."""
    th = th or Thresholds()
    if not scripts:
        return []
    dof = scripts[0].arm_dof
    if any(s.arm_dof != dof for s in scripts):
        raise ValueError("all scripts of a batch must share arm_dof")
    arr, kinds, gaps = _script_array(scripts, seeds)
    sb = core.realize_batch(arr, kinds, gaps, th, _label_csets(None, dof), dof)
    lab = sb.labels.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)
    headers = [_synth_header(s.episode_id, SubtaskKind(s.subtask_kind),
                             ArticulationKind(s.articulation_kind), dof) for s in scripts]
    trajs = _to_trajectories(sb, headers)
    out = []
    for i, s in enumerate(scripts):
        if int(lab["status"][i]) != 0:
            try:
                _raise_status(lab, i, s)
            except InfeasibleScript as e:
                if strict:
                    raise
                out.append(e)
                continue
        out.append(trajs[i])
    return out


def realize(script: EventScript, seed: int = 0, th: Optional[Thresholds] = None) -> Trajectory:
    """Trajectory whose event list equals the script (synth.py:345-348)."""
    return realize_many([script], [seed], th)[0]


def _fuzz_device(seeds, subtask_kind, config, th, want_scripts):
    cfg = config or FuzzConfig()
    if cfg.max_gap < 1 or cfg.max_tail < 1:
        raise ValueError("empty range for randrange()")  # randint(1, 0)
    kind = SubtaskKind(subtask_kind)
    sb = core.fuzz_batch(np.asarray(seeds, np.int64), SUBTASK_ORDER.index(kind), cfg,
                         th or Thresholds(), _label_csets(), want_scripts=want_scripts)
    return kind, cfg, sb


def _scripts_from_device(kind, cfg, sb, seeds):
    sc = sb.scripts.cpu().numpy().reshape(-1).view(L.SCRIPT_DTYPE)
    sk = sb.script_kind.cpu().numpy()
    sg = sb.script_gap.cpu().numpy()
    out = []
    for i, seed in enumerate(seeds):
        s = sc[i]
        a = int(s["step_off"])
        steps = [ScriptStep(EVENT_KINDS[int(sk[a + j])], int(sg[a + j]))
                 for j in range(int(s["n_steps"]))]
        out.append(EventScript(
            subtask_kind=kind, steps=steps, tail=int(s["tail"]),
            initial_grasped=bool(s["initial_grasped"]),
            initial_contact=bool(s["initial_contact"]),
            initial_dist_obj_goal=float(s["initial_dist_obj_goal"]),
            initial_art_level=LEVELS[int(s["initial_level"])],
            articulation_kind=ART_ORDER[int(s["art_kind"])],
            episode_id=f"fuzz-{kind.value.lower()}-{int(seed):08d}"))
    return out


def random_script(seed: int, subtask_kind: SubtaskKind,
                  config: Optional[FuzzConfig] = None) -> EventScript:
    """Random feasible script (synth.py:363-507), sampled on the device."""
    kind, cfg, sb = _fuzz_device([seed], subtask_kind, config, None, True)
    return _scripts_from_device(kind, cfg, sb, [seed])[0]


def fuzz_many(seeds, subtask_kind, config=None, th=None):
    """fuzz() for many seeds in one launch -> list of Trajectory."""
    seeds = [int(s) for s in seeds]
    kind, cfg, sb = _fuzz_device(seeds, subtask_kind, config, th, True)
    scripts = _scripts_from_device(kind, cfg, sb, seeds)
    headers = [_synth_header(s.episode_id, kind, s.articulation_kind, 7) for s in scripts]
    return _to_trajectories(sb, headers)


def fuzz(seed: int, subtask_kind: SubtaskKind, config: Optional[FuzzConfig] = None,
         th: Optional[Thresholds] = None) -> Trajectory:
    """random_script(seed) realized with seed ^ 0x5EED (synth.py:510-515)."""
    return fuzz_many([seed], subtask_kind, config, th)[0]


def _s(kind, steps, **kw):
    return EventScript(subtask_kind=kind, steps=[ScriptStep(k, 2) for k in steps], **kw)


def defining_scripts() -> dict:
    """mode_id -> canonical script of that mode (synth.py:525-602)."""
    E = EventKind
    P, L_, O, C = SubtaskKind.Pick, SubtaskKind.Place, SubtaskKind.Open, SubtaskKind.Close
    g = dict(initial_grasped=True)
    h = dict(initial_art_level="high")
    C3 = [E.Contact, E.Grasped]
    pl = [E.ObjAtGoal, E.ReleasedAtGoal]
    op = [E.Contact, E.SlightlyOpened, E.Opened]
    cl = [E.Contact, E.SlightlyClosed, E.Closed]
    return {
        "pick.s1_straightforward": _s(P, C3 + [E.Success]),
        "pick.s2_winding": _s(P, C3 + [E.Dropped] + C3 + [E.Success]),
        "pick.s3_success_then_drop": _s(P, C3 + [E.Success, E.Dropped]),
        "pick.s4_success_then_excessive_collisions": _s(P, C3 + [E.Success, E.ExcessiveCollisions]),
        "pick.f5_excessive_collisions": _s(P, [E.ExcessiveCollisions]),
        "pick.f6_mobility": _s(P, []),
        "pick.f7_cant_grasp": _s(P, [E.Contact]),
        "pick.f8_drop": _s(P, C3 + [E.Dropped]),
        "pick.f9_too_slow": _s(P, C3),
        "place.s1_place_in_goal": _s(L_, pl + [E.Success], **g),
        "place.s2_drop_to_goal": _s(L_, [E.ReleasedOutsideGoal, E.ObjAtGoal, E.Success], **g),
        "place.s3_dubious": _s(L_, pl + [E.Success, E.ObjLeftGoal], **g),
        "place.s4_winding": _s(L_, pl + [E.Success, E.ObjLeftGoal, E.ObjAtGoal, E.Success], **g),
        "place.s5_success_then_excessive_collisions": _s(L_, pl + [E.Success, E.ExcessiveCollisions], **g),
        "place.f6_excessive_collisions": _s(L_, [E.ExcessiveCollisions], **g),
        "place.f7_didnt_grasp": _s(L_, [], **g),
        "place.f8_didnt_reach_goal": _s(L_, [E.ReleasedOutsideGoal], **g),
        "place.f9_place_in_goal": _s(L_, pl + [E.ObjLeftGoal], **g),
        "place.f10_drop_to_goal": _s(L_, [E.ReleasedOutsideGoal, E.ObjAtGoal, E.ObjLeftGoal], **g),
        "place.f11_wont_let_go": _s(L_, pl + [E.Grasped], **g),
        "place.f12_too_slow": _s(L_, pl, **g),
        "open.s1_open": _s(O, op + [E.Success]),
        "open.s2_dubious": _s(O, op + [E.Success, E.Closed]),
        "open.s3_success_then_excessive_collisions": _s(O, op + [E.Success, E.ExcessiveCollisions]),
        "open.f4_excessive_collisions": _s(O, [E.ExcessiveCollisions]),
        "open.f5_cant_reach": _s(O, []),
        "open.f6_closed_after_open": _s(O, op + [E.Closed]),
        "open.f7_slightly_opened": _s(O, [E.Contact, E.SlightlyOpened]),
        "open.f8_too_slow": _s(O, op),
        "open.f9_cant_open": _s(O, [E.Contact]),
        "close.s1_close": _s(C, cl + [E.Success], **h),
        "close.s2_dubious": _s(C, cl + [E.Success, E.Open], **h),
        "close.s3_success_then_excessive_collisions": _s(C, cl + [E.Success, E.ExcessiveCollisions], **h),
        "close.f4_excessive_collisions": _s(C, [E.ExcessiveCollisions], **h),
        "close.f5_cant_reach": _s(C, [], **h),
        "close.f6_opened_after_closed": _s(C, cl + [E.Open], **h),
        "close.f7_slightly_closed": _s(C, [E.Contact, E.SlightlyClosed], **h),
        "close.f8_too_slow": _s(C, cl, **h),
        "close.f9_cant_close": _s(C, [E.Contact], **h),
    }
