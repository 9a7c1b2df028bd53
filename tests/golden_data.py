"""Loaders for the golden fixtures in tests/golden (made by make_golden.py
from the reference).  Shared by the oracle tests and the GPU parity tests."""
from __future__ import annotations

import functools
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KIND_NAMES = ("pick", "place", "open", "close")
SUBTASKS = ("Pick", "Place", "Open", "Close")
LEVELS = ("low", "slight", "open", "high", "closed")
ART = ("None", "Fridge", "Drawer")
DOF = 7


@functools.lru_cache(None)
def npz(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@functools.lru_cache(None)
def js(name):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as f:
        return json.load(f)


class Corpus:
    """One packed set of episodes from a fixture file (prefix-selected)."""

    def __init__(self, d, prefix=""):
        g = lambda k: d[prefix + k]  # noqa: E731
        self.planes = g("planes")
        self.grasped = g("grasped")
        self.rec_off = g("rec_off")
        self.subtask = g("subtask")
        self.art_kind = g("art_kind")
        self.art_qmin = g("art_qmin")
        self.art_qmax = g("art_qmax")
        self.rest_tor = g("rest_tor")
        self.rest_arm = g("rest_arm")
        self.ev_kind = g("ev_kind")
        self.ev_t = g("ev_t")
        self.ev_off = g("ev_off")
        self.mode = g("mode")
        self.success_once = g("success_once")
        self.success_at_end = g("success_at_end")
        self.n = len(self.rec_off) - 1
        self.d = d
        self.prefix = prefix

    def get(self, k, default=None):
        return self.d.get(self.prefix + k, default)

    def events(self, i):
        a, b = self.ev_off[i], self.ev_off[i + 1]
        return list(self.ev_kind[a:b]), list(self.ev_t[a:b])

    def records_np(self, i):
        a, b = self.rec_off[i], self.rec_off[i + 1]
        return self.planes[:, a:b], self.grasped[a:b]

    def scripts(self):
        """list of script dicts (oracle.py layout) if present."""
        if self.get("step_off") is None:
            return None
        off = self.get("step_off")
        out = []
        for i in range(len(off) - 1):
            out.append(dict(
                subtask=int(self.get("subtask")[i]) if self.get("subtask") is not None else 0,
                kinds=self.get("step_kind")[off[i]:off[i + 1]],
                gaps=self.get("step_gap")[off[i]:off[i + 1]],
                tail=int(self.get("tail")[i]),
                initial_grasped=int(self.get("initial_grasped")[i]),
                initial_contact=int(self.get("initial_contact")[i]),
                initial_dist_obj_goal=float(self.get("initial_dist_obj_goal")[i]),
                initial_level=int(self.get("initial_level")[i]),
                art_kind=int(self.get("art_kind")[i]),
                arm_dof=DOF))
        return out


def fuzz_corpus(kind):
    return Corpus(npz("fuzz"), KIND_NAMES[kind] + "_")


def to_oracle_records(O, planes, grasped):
    """fixture planes [2*dof+9][T] -> oracle REC_DTYPE array."""
    T = planes.shape[1]
    r = np.zeros(T, O.REC_DTYPE)
    r["q_arm"][:, :DOF] = planes[0:DOF].T
    r["qd_arm"][:, :DOF] = planes[DOF:2 * DOF].T
    for j, f in enumerate(O.SCALAR_FIELDS):
        r[f] = planes[2 * DOF + j]
    r["grasped"] = grasped
    return r


def from_oracle_records(O, recs):
    planes = np.zeros((2 * DOF + 9, len(recs)), np.float64)
    planes[0:DOF] = recs["q_arm"][:, :DOF].T
    planes[DOF:2 * DOF] = recs["qd_arm"][:, :DOF].T
    for j, f in enumerate(O.SCALAR_FIELDS):
        planes[2 * DOF + j] = recs[f]
    return planes, recs["grasped"].astype(np.uint8)


def _bits(a):
    a = np.array(np.asarray(a, np.float32), copy=True)
    a[np.isnan(a)] = np.float32("nan")  # one canonical NaN
    return a.view(np.uint32)


def same_bits_f32(a, b):
    """bit-exact f32 equality (all NaNs equal, as the reference's NaN-aware
    TimestepRecord.__eq__, model.py:186-199)."""
    a, b = _bits(a), _bits(b)
    return a.shape == b.shape and bool(np.array_equal(a, b))
