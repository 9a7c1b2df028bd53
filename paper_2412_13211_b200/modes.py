"""Mode classification (mirror of trajlab.modes, modes.py:24-287).

The 39 rule predicates are compiled into the device classifier
(csrc/tl_label.cuh rule_pred, first match wins).  MODE_RULES keeps the
reference's table shape {kind: {"success": [(mode_id, pred)], "failure":
[...]}}; its predicates are handles on the device rules, so reordered or
truncated tables (e.g. the --corrupt negative control, cli.py:232-238)
run on the GPU too.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from .errors import UnknownMode, label_error
from .events import EVENT_KINDS, EventKind, EventList
from .model import SUBTASK_ORDER, SubtaskKind

SPEC_DEVIATIONS = ("open_close_s3_membership",)

_MODES = {
    SubtaskKind.Pick: (
        ("pick.s1_straightforward", "pick.s2_winding", "pick.s3_success_then_drop",
         "pick.s4_success_then_excessive_collisions"),
        ("pick.f5_excessive_collisions", "pick.f6_mobility", "pick.f7_cant_grasp",
         "pick.f8_drop", "pick.f9_too_slow")),
    SubtaskKind.Place: (
        ("place.s1_place_in_goal", "place.s2_drop_to_goal", "place.s3_dubious",
         "place.s4_winding", "place.s5_success_then_excessive_collisions"),
        ("place.f6_excessive_collisions", "place.f7_didnt_grasp",
         "place.f8_didnt_reach_goal", "place.f9_place_in_goal",
         "place.f10_drop_to_goal", "place.f11_wont_let_go", "place.f12_too_slow")),
    SubtaskKind.Open: (
        ("open.s1_open", "open.s2_dubious", "open.s3_success_then_excessive_collisions"),
        ("open.f4_excessive_collisions", "open.f5_cant_reach",
         "open.f6_closed_after_open", "open.f7_slightly_opened", "open.f8_too_slow",
         "open.f9_cant_open")),
    SubtaskKind.Close: (
        ("close.s1_close", "close.s2_dubious",
         "close.s3_success_then_excessive_collisions"),
        ("close.f4_excessive_collisions", "close.f5_cant_reach",
         "close.f6_opened_after_closed", "close.f7_slightly_closed",
         "close.f8_too_slow", "close.f9_cant_close")),
}

# global device mode id -> mode_id string (success then failure per subtask)
MODE_LIST = tuple(m for k in SUBTASK_ORDER for branch in _MODES[k] for m in branch)
MODE_INDEX = {m: i for i, m in enumerate(MODE_LIST)}


class DeviceRule:
    """Handle on one builtin rule predicate (evaluated by the GPU classifier)."""

    __slots__ = ("mode_id", "index")

    def __init__(self, mode_id):
        self.mode_id = mode_id
        self.index = MODE_INDEX[mode_id]

    def __call__(self, ctx):
        raise TypeError("mode predicates run on the device; call classify()")

    def __repr__(self):
        return f"<device rule {self.mode_id}>"


MODE_RULES = {
    k: {"success": [(m, DeviceRule(m)) for m in _MODES[k][0]],
        "failure": [(m, DeviceRule(m)) for m in _MODES[k][1]]}
    for k in SUBTASK_ORDER
}
MODE_IDS = {k: [m for branch in _MODES[k] for m in branch] for k in SUBTASK_ORDER}
SUCCESS_MODE_IDS = {k: set(_MODES[k][0]) for k in SUBTASK_ORDER}
SUCCESS_AT_END_MODES = {
    SubtaskKind.Pick: {"pick.s1_straightforward", "pick.s2_winding"},
    SubtaskKind.Place: {"place.s1_place_in_goal", "place.s2_drop_to_goal",
                        "place.s4_winding"},
    SubtaskKind.Open: {"open.s1_open"},
    SubtaskKind.Close: {"close.s1_close"},
}


def last_index(events, kind: EventKind) -> int:
    """0-based position of the last occurrence of kind, -1 if absent."""
    kinds = events.kinds() if isinstance(events, EventList) else list(events)
    rev = kinds[::-1]
    return len(kinds) - 1 - rev.index(kind) if kind in rev else -1


@dataclass(frozen=True)
class ModeLabel:
    subtask_kind: SubtaskKind
    mode_id: str
    is_success: bool
    success_once: bool
    success_at_end: bool


def rules_to_ids(rules) -> Optional[list]:
    """Reference-shaped rule table -> per (subtask, branch) device rule ids."""
    if rules is None:
        return None
    out = []
    for k in SUBTASK_ORDER:
        table = rules.get(k) if hasattr(rules, "get") else None
        if table is None:
            out.append([[], []])
            continue
        branches = []
        for b in ("success", "failure"):
            ids = []
            for mode_id, pred in table[b]:
                if not isinstance(pred, DeviceRule):
                    raise NotImplementedError(
                        f"rule {mode_id!r}: only the builtin mode predicates run on the device")
                ids.append(pred.index)
            branches.append(ids)
        out.append(branches)
    return out


def classify(events: EventList, rules: Optional[dict] = None) -> ModeLabel:
    """One mode per event list (modes.py:235-253), on the GPU."""
    from . import core
    kind = events.subtask_kind
    if rules is not None:
        rules[kind]  # KeyError for a table without this subtask, as the reference
    ids = rules_to_ids(rules)
    kinds = [EVENT_KINDS.index(e.kind) for e in events.events]
    d0 = events.initial_dist_obj_goal
    lab = core.classify_lists([kinds], [SUBTASK_ORDER.index(kind)],
                              [0.0 if d0 is None else float(d0)], [d0 is None], ids)[0]
    st = int(lab["status"])
    if st != 0:
        raise label_error(st, kind.value, [e.kind.value for e in events.events],
                          bool(lab["flags"] & 1))
    m = MODE_LIST[int(lab["mode"])]
    so = bool(lab["flags"] & 1)
    return ModeLabel(subtask_kind=kind, mode_id=m, is_success=so, success_once=so,
                     success_at_end=bool(lab["flags"] & 2))


@dataclass(frozen=True)
class GroupingScheme:
    name: str
    mapping: dict

    def group(self, mode_id: str) -> str:
        if mode_id not in self.mapping:
            raise UnknownMode(f"scheme {self.name!r} does not cover {mode_id!r}")
        return self.mapping[mode_id]


PICK_COARSE = GroupingScheme(name="pick-coarse", mapping={
    "pick.s1_straightforward": "S-Once", "pick.s2_winding": "S-Once",
    "pick.s3_success_then_drop": "S-Once",
    "pick.s4_success_then_excessive_collisions": "S-Once",
    "pick.f5_excessive_collisions": "F-Col", "pick.f6_mobility": "F-Other",
    "pick.f7_cant_grasp": "F-Grasp", "pick.f8_drop": "F-Other",
    "pick.f9_too_slow": "F-Other"})
BUILTIN_SCHEMES = {PICK_COARSE.name: PICK_COARSE}


def group(label: ModeLabel, scheme: GroupingScheme) -> str:
    return scheme.group(label.mode_id)
