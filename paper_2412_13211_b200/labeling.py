"""Batched labelling of host Trajectory objects on the GPU (K1 + K2), the
engine behind extract_events / label_trajectory / label_batch.

One call packs every trajectory into one SoA batch, runs one label launch,
one scan and one emit launch, and copies back labels + event arrays once.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib as L
from . import core
from .errors import label_error
from .model import SUBTASK_ORDER
from .thresholds import Thresholds


@dataclass
class Labelled:
    events: object = None        # EventList
    mode_id: Optional[str] = None
    success_once: bool = False
    success_at_end: bool = False
    error: Optional[BaseException] = None


def label_many(trajs, th: Optional[Thresholds] = None, rules=None, classify=True):
    th = th or Thresholds()
    if not trajs:
        return []
    rb, env, cs, n_cs = core.pack_trajectories(trajs, th)
    return _collect(core.label_records(rb, env, cs, n_cs, rules=rules),
                    [t.header for t in trajs])


def label_arrays(items, th: Optional[Thresholds] = None, rules=None):
    """label_many for (header, TRJL structured record array) pairs: the file
    path of label_batch, no per-record Python objects (core.pack_record_arrays)."""
    th = th or Thresholds()
    if not items:
        return []
    rb, env, cs, n_cs = core.pack_record_arrays(items, th)
    return _collect(core.label_records(rb, env, cs, n_cs, rules=rules), [h for h, _ in items])


def _collect(res, headers):
    from .events import EVENT_KINDS, Event, EventList
    from .modes import MODE_LIST
    lab = res.labels_np()
    off = res.ev_off.cpu().numpy()
    kinds = res.ev_kind.cpu().numpy()
    ts = res.ev_t.cpu().numpy()
    out = []
    for i, hdr in enumerate(headers):
        st = int(lab["status"][i])
        sub = hdr.subtask_kind
        if st != 0 and st != L.ERR_MODE_COVERAGE:
            out.append(Labelled(error=label_error(st, sub.value)))
            continue
        evs = [Event(EVENT_KINDS[k], int(t)) for k, t in zip(kinds[off[i]:off[i + 1]], ts[off[i]:off[i + 1]])]
        d0 = float(lab["d0"][i]) if sub == SUBTASK_ORDER[1] else None
        el = EventList(subtask_kind=sub, events=evs, initial_dist_obj_goal=d0)
        if st == L.ERR_MODE_COVERAGE:
            out.append(Labelled(events=el, error=label_error(
                st, sub.value, [e.kind.value for e in evs],
                any(e.kind == EVENT_KINDS[12] for e in evs))))
            continue
        m = int(lab["mode"][i])
        out.append(Labelled(events=el, mode_id=MODE_LIST[m],
                            success_once=bool(lab["flags"][i] & 1),
                            success_at_end=bool(lab["flags"][i] & 2)))
    return out
