"""Edge-triggered event extraction (mirror of trajlab.events, events.py).

extract_events packs the trajectory into the GPU record layout and runs the
K1 label kernel (predicates + edges + classification) followed by K2 event
emission; the host only converts the device event arrays back into Event
objects.  The within-step order is EVENT_ORDER (events.py:38-52).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

from .model import SubtaskKind, Trajectory
from .thresholds import Thresholds


class EventKind(str, Enum):
    Contact = "Contact"
    Grasped = "Grasped"
    Dropped = "Dropped"
    ObjAtGoal = "ObjAtGoal"
    ReleasedAtGoal = "ReleasedAtGoal"
    ReleasedOutsideGoal = "ReleasedOutsideGoal"
    ObjLeftGoal = "ObjLeftGoal"
    Opened = "Opened"
    SlightlyOpened = "SlightlyOpened"
    Closed = "Closed"
    SlightlyClosed = "SlightlyClosed"
    Open = "Open"
    Success = "Success"
    ExcessiveCollisions = "ExcessiveCollisions"


EVENT_KINDS = tuple(EventKind)  # device kind id -> EventKind

EVENT_ORDER = {
    SubtaskKind.Pick: (EventKind.Contact, EventKind.Grasped, EventKind.Dropped,
                       EventKind.Success, EventKind.ExcessiveCollisions),
    SubtaskKind.Place: (EventKind.Grasped, EventKind.ObjAtGoal,
                        EventKind.ReleasedAtGoal, EventKind.ReleasedOutsideGoal,
                        EventKind.ObjLeftGoal, EventKind.Success,
                        EventKind.ExcessiveCollisions),
    SubtaskKind.Open: (EventKind.Contact, EventKind.Opened,
                       EventKind.SlightlyOpened, EventKind.Closed,
                       EventKind.Success, EventKind.ExcessiveCollisions),
    SubtaskKind.Close: (EventKind.Contact, EventKind.Closed,
                        EventKind.SlightlyClosed, EventKind.Open,
                        EventKind.Success, EventKind.ExcessiveCollisions),
}


@dataclass(frozen=True)
class Event:
    kind: EventKind
    t: int

    def to_dict(self) -> dict:
        return {"kind": self.kind.value, "t": self.t}


@dataclass
class EventList:
    subtask_kind: SubtaskKind
    events: list = field(default_factory=list)
    initial_dist_obj_goal: Optional[float] = None

    def kinds(self) -> list:
        return [e.kind for e in self.events]

    def __len__(self):
        return len(self.events)

    def to_dict(self) -> dict:
        out = {"events": [e.to_dict() for e in self.events]}
        if self.initial_dist_obj_goal is not None:
            out["initial_dist_obj_goal"] = self.initial_dist_obj_goal
        return out


def extract_events(traj: Trajectory, th: Thresholds) -> EventList:
    """Chronologically ordered event list of one trajectory (events.py:94).
    Raises the reference's TooShort / RequiredFieldNaN / MissingArticulation."""
    from .labeling import label_many
    out = label_many([traj], th)[0]
    if out.error is not None:
        raise out.error
    return out.events
