"""Mode classification (mirror of trajlab.modes, modes.py:24-287).

The 39 rule predicates are compiled into the device classifier
(csrc/tl_label.cuh rule_pred, first match wins).  MODE_RULES keeps the
reference's table shape {kind: {"success": [(mode_id, pred)], "failure":
[...]}}; its predicates are handles on the device rules, so reordered or
truncated tables (e.g. the --corrupt negative control, cli.py:232-238)
run on the GPU too.  Tables may also hold arbitrary callables (the
reference accepts any (mode_id, predicate) table, modes.py:235-253); those
are called with the event view in table order, between device runs.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

from . import _lib as L
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


def _device_table(sub: int, ids) -> list:
    """One rule run as a device table: the same ids on both branches of
    subtask `sub` (the caller already chose the branch), nothing elsewhere."""
    out = [[[], []] for _ in SUBTASK_ORDER]
    out[sub] = [list(ids), list(ids)]
    return out


class _EventView:
    """What a rule predicate sees (the reference's _Ctx, modes.py:42-62):
    kinds, size, d0, last(kind), has(kind).  Built once per classify call for
    tables that hold host callables."""

    __slots__ = ("kinds", "size", "d0", "_pos")

    def __init__(self, events: EventList):
        self.kinds = events.kinds()
        self.size = len(self.kinds)
        self.d0 = events.initial_dist_obj_goal
        # later occurrences overwrite earlier ones: the value is the last index
        self._pos = {k: i for i, k in enumerate(self.kinds)}

    def last(self, kind: EventKind) -> int:
        return self._pos.get(kind, -1)

    def has(self, kind: EventKind) -> bool:
        return kind in self._pos


def _label(kind, mode_id, success_once):
    return ModeLabel(subtask_kind=kind, mode_id=mode_id, is_success=success_once,
                     success_once=success_once,
                     success_at_end=mode_id in SUCCESS_AT_END_MODES[kind])


def classify(events: EventList, rules: Optional[dict] = None) -> ModeLabel:
    """One mode per event list (modes.py:235-253): first match wins over the
    success rules if Success occurs, else over the failure rules.

    The builtin table (rules=None, or an empty table as `rules or MODE_RULES`
    reads it) runs as one device classification.  A custom table is walked
    in order: each maximal run of builtin predicates (DeviceRule) is one
    device call over that run, returning the first match's position; any
    other callable is the user's own Python and is called with the event
    view, exactly when the reference would call it.  The returned mode_id is
    the table entry's, not the predicate's own name."""
    from . import core
    kind = events.subtask_kind
    sub = SUBTASK_ORDER.index(kind)
    kinds = [EVENT_KINDS.index(e.kind) for e in events.events]
    d0 = events.initial_dist_obj_goal
    d0_args = ([0.0 if d0 is None else float(d0)], [d0 is None])

    def device(ids):
        lab = core.classify_lists([kinds], [sub], *d0_args, ids)[0]
        return int(lab["status"]), lab

    if not rules:  # the builtin table, on the device
        st, lab = device(None)
        if st != 0:
            raise label_error(st, kind.value, [e.kind.value for e in events.events],
                              bool(lab["flags"] & 1))
        so = bool(lab["flags"] & 1)
        return ModeLabel(subtask_kind=kind, mode_id=MODE_LIST[int(lab["mode"])],
                         is_success=so, success_once=so, success_at_end=bool(lab["flags"] & 2))
    table = rules[kind]  # KeyError for a table without this subtask, as the reference
    success_once = any(e.kind is EventKind.Success for e in events.events)
    branch = list(table["success"] if success_once else table["failure"])
    view = None
    i = 0
    while i < len(branch):
        mode_id, pred = branch[i]
        if isinstance(pred, DeviceRule):
            j = i
            while j < len(branch) and j - i < 16 and isinstance(branch[j][1], DeviceRule):
                j += 1
            ids = [p.index for _, p in branch[i:j]]
            st, lab = device(_device_table(sub, ids))
            if st == 0:  # the first run position holding the matched predicate
                return _label(kind, branch[i + ids.index(int(lab["mode"]))][0], success_once)
            if st != L.ERR_MODE_COVERAGE:
                raise label_error(st, kind.value, [e.kind.value for e in events.events],
                                  success_once)
            i = j
            continue
        if view is None:
            view = _EventView(events)
        if pred(view):
            return _label(kind, mode_id, success_once)
        i += 1
    raise label_error(L.ERR_MODE_COVERAGE, kind.value, [e.kind.value for e in events.events],
                      success_once)


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
