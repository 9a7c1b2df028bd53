"""Exception hierarchy (names of trajlab.errors, errors.py:4-73) and the
mapping from device status codes to the exact exceptions the reference
raises.  Messages are reproduced byte-for-byte because label_batch turns
them into output text ("Kind: message", pipeline.py:115)."""
from __future__ import annotations

from . import _lib as L


class TrajlabError(Exception):
    """Base class for all trajlab errors."""


class InvariantViolation(TrajlabError):
    pass


class BadMagic(TrajlabError):
    pass


class UnsupportedVersion(TrajlabError):
    pass


class TruncatedFile(TrajlabError):
    pass


class HeaderParseError(TrajlabError):
    pass


class ParseError(TrajlabError):
    def __init__(self, message, line_no=None):
        super().__init__(message if line_no is None else f"line {line_no}: {message}")
        self.line_no = line_no


class RequiredFieldNaN(TrajlabError):
    pass


class MissingArticulation(TrajlabError):
    pass


class TooShort(TrajlabError):
    pass


class UnknownMode(TrajlabError):
    pass


class ModeCoverageError(TrajlabError):
    pass


class InfeasibleScript(TrajlabError):
    pass


class EmptyAllowList(TrajlabError):
    pass


class EmptyInput(TrajlabError):
    pass


class BothZero(TrajlabError):
    pass


class MissingRate(TrajlabError):
    pass


# InfeasibleScript messages per raise site (synth.py:123-302)
_INFEASIBLE = {
    20: "Pick cannot start grasped without contact force",
    22: "collision limit already exceeded",
    25: "Contact while already in contact",
    26: "Grasped while already grasped",
    27: "Pick grasp requires contact force",
    28: "Dropped while not grasped",
    29: "ObjAtGoal while already at goal",
    30: "ObjLeftGoal while not at goal",
    31: "ReleasedAtGoal needs grasp at goal",
    32: "ReleasedOutsideGoal needs grasp outside goal",
    33: "SlightlyOpened from non-low articulation",
    34: "Opened requires slightly-open articulation",
    35: "Closed (Open subtask) requires open articulation",
    36: "SlightlyClosed needs a not-yet-closing articulation",
    37: "slightly-closed band is empty for this start state",
    38: "Closed requires slightly-closed articulation",
    39: "Open (Close subtask) requires closed articulation",
    40: "event gap must be >= 1",
}


def label_error(code: int, subtask: str, kinds=None, success_once=False):
    """Exception for a labelling status (events.py / predicates.py / modes.py)."""
    if code == L.ERR_TOO_SHORT:
        return TooShort("need at least 2 records to detect edges")
    if code == L.ERR_NAN_SUCCESS_DIST:
        return RequiredFieldNaN("field dist_obj_goal is NaN but required by this subtask")
    if code == L.ERR_NAN_ART:
        return RequiredFieldNaN("field art_q is NaN but required by this subtask")
    if code == L.ERR_NAN_FORCE:
        return RequiredFieldNaN(f"force_ee_target is NaN but required for {subtask} events")
    if code == L.ERR_NAN_PLACE_DIST:
        return RequiredFieldNaN("dist_obj_goal is NaN but required for Place")
    if code == L.ERR_MISSING_ART:
        return MissingArticulation(f"{subtask} predicate needs an articulation")
    if code == L.ERR_MODE_COVERAGE:
        branch = "success" if success_once else "failure"
        return ModeCoverageError(f"no {branch} mode matched {list(kinds or [])}")
    if code == L.ERR_D0_NONE_LE:
        return TypeError("'<=' not supported between instances of 'NoneType' and 'float'")
    if code == L.ERR_D0_NONE_GT:
        return TypeError("'>' not supported between instances of 'NoneType' and 'float'")
    return TrajlabError(f"device status {code}")


def infeasible_error(code: int, subtask: str, event: str = None, level: str = None):
    """InfeasibleScript for a realize status (synth.py:123-302)."""
    if code == 21:
        return InfeasibleScript(f"event {event} not in {subtask} alphabet")
    if code == 23:
        return InfeasibleScript(f"Success not reachable from current state ({subtask})")
    if code == 24:
        return InfeasibleScript(f"Contact undefined for {subtask}")
    if code == 41:
        return InfeasibleScript(f"initial art level {level!r} invalid for {subtask}")
    if code in _INFEASIBLE:
        return InfeasibleScript(_INFEASIBLE[code])
    return TrajlabError(f"device status {code}")
