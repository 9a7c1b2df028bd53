"""Statistics tables and chained-episode analysis (mirror of
trajlab.analytics, analytics.py:19-312).

Everything the reference computes from label records reduces to integer
counts -- per group: how many labels carry each mode, success_once and
success_at_end; per chain slot: how many chains are still alive.  Those
counts come from the GPU for device label batches (``tl_group_mode_counts``,
``tl_chain_progress``; csrc/tl_analytics.cuh) or from a host pass over
LabelRecord lists; both feed the same fraction / rounding code, so the
tables are identical whichever way the counts were made.
"""
from __future__ import annotations

import json
from collections import Counter
from dataclasses import dataclass
from decimal import ROUND_HALF_UP, Decimal
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from .errors import BothZero, EmptyInput, MissingRate
from .model import SUBTASK_ORDER, SubtaskKind
from .modes import MODE_IDS, MODE_LIST, SUCCESS_MODE_IDS, GroupingScheme

GROUP_KEYS = ("task", "target_id", "policy_tag", "split", "subtask")   # analytics.py:19
N_COUNT_COLS = 42   # 39 modes, success_once, success_at_end, labels


def round_half_away(x: float, decimals: int = 2) -> float:
    """Decimal rounding with ties away from zero on the shortest repr of x
    (analytics.py:22-25): 2.675 -> 2.68 where round() gives 2.67."""
    step = Decimal(1).scaleb(-decimals)
    return float(Decimal(repr(x)).quantize(step, rounding=ROUND_HALF_UP))


@dataclass
class StatsRow:
    key: dict
    count: int
    sor: float
    saer: float
    fr: float
    modes: dict

    def rendered(self, decimals: int = 2) -> dict:
        pct = lambda v: round_half_away(100.0 * v, decimals)  # noqa: E731
        return {"key": dict(self.key), "count": self.count, "sor": pct(self.sor),
                "saer": pct(self.saer), "fr": pct(self.fr),
                "modes": {m: pct(v) for m, v in self.modes.items()}}


def _success_columns() -> set:
    cols = {"S-Once"}
    for k in SubtaskKind:
        cols |= SUCCESS_MODE_IDS[k]
    return cols


@dataclass
class StatsTable:
    group_by: tuple
    mode_columns: list
    rows: list
    decimals: int = 2

    def to_dict(self) -> dict:
        return {"group_by": list(self.group_by), "mode_columns": list(self.mode_columns),
                "rows": [r.rendered(self.decimals) for r in self.rows]}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2)

    def _split_columns(self):
        succ = _success_columns()
        s = [c for c in self.mode_columns if c in succ]
        f = [c for c in self.mode_columns if c not in succ]
        return s, f

    def _header(self):
        s, f = self._split_columns()
        return [*self.group_by, "count", "SoR", "SaeR", *s, "FR", *f]

    def _cells(self, row: StatsRow):
        r = row.rendered(self.decimals)
        fmt = f"{{:.{self.decimals}f}}".format
        s, f = self._split_columns()
        return ([str(row.key.get(k, "")) for k in self.group_by]
                + [str(row.count), fmt(r["sor"]), fmt(r["saer"])]
                + [fmt(r["modes"].get(c, 0.0)) for c in s] + [fmt(r["fr"])]
                + [fmt(r["modes"].get(c, 0.0)) for c in f])

    def to_markdown(self) -> str:
        head = self._header()
        out = ["| " + " | ".join(head) + " |", "| " + " | ".join("---" for _ in head) + " |"]
        out += ["| " + " | ".join(self._cells(r)) + " |" for r in self.rows]
        return "\n".join(out)

    def to_csv(self) -> str:
        return "\n".join([",".join(self._header())] + [",".join(self._cells(r)) for r in self.rows])


def _columns(present: set, grouping: Optional[GroupingScheme]) -> list:
    """canonical column order (analytics.py:106-118)"""
    cols = []
    for kind in SubtaskKind:
        for m in MODE_IDS[kind]:
            if grouping is not None:
                g = grouping.mapping.get(m)
                if g is not None and g not in cols:
                    cols.append(g)
            elif m in present:
                cols.append(m)
    return cols


def _table(group_by, grouping, decimals, groups: dict) -> StatsTable:
    """groups: key tuple -> (n, Counter(mode_id), n_success_once, n_success_at_end)"""
    present = set()
    for _, (_, cnt, _, _) in groups.items():
        present |= {m for m, c in cnt.items() if c}
    columns = _columns(present, grouping)
    rows = []
    for key in sorted(groups):
        n, cnt, so, se = groups[key]
        cols = Counter()
        for m, c in cnt.items():
            if c:
                cols[grouping.group(m) if grouping else m] += c
        rows.append(StatsRow(key=dict(zip(group_by, key)), count=n, sor=so / n, saer=se / n,
                             fr=(n - so) / n, modes={c: cols.get(c, 0) / n for c in columns}))
    return StatsTable(group_by=tuple(group_by), mode_columns=columns, rows=rows,
                      decimals=decimals)


def _check_keys(group_by):
    for k in group_by:
        if k not in GROUP_KEYS:
            raise ValueError(f"unknown group-by key {k!r}; choose from {GROUP_KEYS}")


@dataclass
class LabelBatch:
    """Device labels (tl_label rows, e.g. from fuzz/label_records) plus
    optional per-episode group columns: keys[name] = (codes [n] int array,
    names list).  'subtask' comes from the labels themselves."""
    labels: object
    keys: Optional[dict] = None


def group_mode_counts(labels, group=None, n_groups: int = 1) -> np.ndarray:
    """tl_group_mode_counts: int64 [n_groups, 42] over valid labels."""
    import torch
    lab = labels if labels.dim() == 2 else labels.view(-1, 24)
    dev = lab.device
    n = int(lab.shape[0])
    out = torch.empty((n_groups, N_COUNT_COLS), dtype=torch.int64, device=dev)
    g = None
    if group is not None:
        g = torch.as_tensor(group, dtype=torch.int32).to(dev).contiguous()
    L.check(L.lib().tl_group_mode_counts(L.ptr(lab), L.ptr(g), n, n_groups, L.ptr(out),
                                         L.stream_ptr()), "tl_group_mode_counts")
    return out.cpu().numpy()


def _device_groups(batch: LabelBatch, group_by) -> dict:
    import torch
    lab = batch.labels.view(-1, 24)
    n = int(lab.shape[0])
    dims = []
    for k in group_by:
        if k == "subtask":
            codes = lab[:, 12].to(torch.int32)        # tl_label.subtask
            names = [s.value for s in SUBTASK_ORDER]
        else:
            if not batch.keys or k not in batch.keys:
                raise ValueError(f"no {k!r} column in the label batch")
            codes, names = batch.keys[k]
            codes = torch.as_tensor(codes, dtype=torch.int32).to(lab.device)
        dims.append((codes, list(names)))
    gid = torch.zeros(n, dtype=torch.int32, device=lab.device)
    size = 1
    for codes, names in dims:
        gid = gid * len(names) + codes
        size *= len(names)
    counts = group_mode_counts(lab, gid, max(size, 1))
    groups = {}
    for g in range(size):
        row = counts[g]
        if row[41] == 0:
            continue
        key, rem = [], g
        for codes, names in reversed(dims):
            key.append(names[rem % len(names)])
            rem //= len(names)
        cnt = Counter({MODE_LIST[m]: int(row[m]) for m in range(39) if row[m]})
        groups[tuple(reversed(key))] = (int(row[41]), cnt, int(row[39]), int(row[40]))
    return groups


def mode_table(labels, group_by: Sequence[str] = ("subtask",),
               grouping: Optional[GroupingScheme] = None, decimals: int = 2) -> StatsTable:
    """SoR / SaeR / FR + per-mode fractions per group (analytics.py:121-160).
    labels: LabelRecord iterable, or a LabelBatch of device labels."""
    if isinstance(labels, LabelBatch):
        _check_keys(group_by)
        groups = _device_groups(labels, group_by)
        if not groups:
            raise EmptyInput("no label records to aggregate")
        return _table(group_by, grouping, decimals, groups)
    labels = list(labels)
    if not labels:
        raise EmptyInput("no label records to aggregate")
    _check_keys(group_by)
    acc = {}
    for rec in labels:
        key = tuple(getattr(rec, k) for k in group_by)
        if grouping is not None:
            grouping.group(rec.mode_id)  # unknown modes raise (modes.py GroupingScheme)
        n, cnt, so, se = acc.get(key, (0, Counter(), 0, 0))
        cnt[rec.mode_id] += 1
        acc[key] = (n + 1, cnt, so + bool(rec.success_once), se + bool(rec.success_at_end))
    return _table(group_by, grouping, decimals, acc)


# -- behaviour ratios (analytics.py:166-202) ----------------------------------

@dataclass(frozen=True)
class RatioReport:
    mode_a: str
    mode_b: str
    count_a: int
    count_b: int
    text: str

    def to_dict(self) -> dict:
        return {"mode_a": self.mode_a, "mode_b": self.mode_b, "count_a": self.count_a,
                "count_b": self.count_b, "ratio": self.text}


def _ratio_text(v: float) -> str:
    t = f"{round_half_away(v, 2):.2f}".rstrip("0").rstrip(".")
    return t or "0"


def ratio_report(labels, mode_a: str, mode_b: str) -> RatioReport:
    """'a : 1' or '1 : b', the larger side scaled to two decimals."""
    if isinstance(labels, LabelBatch):
        cnt = group_mode_counts(labels.labels)[0]
        a, b = int(cnt[MODE_LIST.index(mode_a)]), int(cnt[MODE_LIST.index(mode_b)])
    else:
        c = Counter(rec.mode_id for rec in labels)
        a, b = c.get(mode_a, 0), c.get(mode_b, 0)
    if a == 0 and b == 0:
        raise BothZero(f"no labels in either mode {mode_a!r} or {mode_b!r}")
    if b == 0:
        text = "1 : 0"
    elif a >= b:
        text = f"{_ratio_text(a / b)} : 1"
    else:
        text = f"1 : {_ratio_text(b / a)}"
    return RatioReport(mode_a, mode_b, a, b, text)


# -- chaining (analytics.py:205-312) --------------------------------------------

@dataclass(frozen=True)
class ChainSlot:
    name: str
    subtask: Optional[str] = None
    auto_success: bool = False


@dataclass
class ChainPlan:
    name: str
    slots: list

    def __post_init__(self):
        for s in self.slots:
            if s.auto_success and s.subtask is not None:
                raise ValueError(f"auto-success slot {s.name} binds a subtask")

    def __len__(self):
        return len(self.slots)

    def to_dict(self) -> dict:
        return {"name": self.name, "slots": [{"name": s.name, "subtask": s.subtask,
                                              "auto_success": s.auto_success}
                                             for s in self.slots]}

    @classmethod
    def from_dict(cls, d: dict) -> "ChainPlan":
        return cls(d["name"], [ChainSlot(s["name"], s.get("subtask"),
                                         bool(s.get("auto_success", False)))
                               for s in d["slots"]])


def _numbered(block, times):
    return [ChainSlot(f"{s.name}{i + 1}", s.subtask, s.auto_success)
            for i in range(times) for s in block]


_NAV = ChainSlot("Nav", auto_success=True)
BUILTIN_PLANS = {
    "tidyhouse": ChainPlan("tidyhouse", _numbered(
        [_NAV, ChainSlot("Pick", "Pick"), _NAV, ChainSlot("Place", "Place")], 5)),
    "preparegroceries": ChainPlan("preparegroceries", _numbered(
        [_NAV, ChainSlot("Pick", "Pick"), _NAV, ChainSlot("Place", "Place")], 3)),
    "settable": ChainPlan("settable", _numbered(
        [_NAV, ChainSlot("Open", "Open"), _NAV, ChainSlot("Pick", "Pick"),
         _NAV, ChainSlot("Place", "Place"), _NAV, ChainSlot("Close", "Close")], 2)),
}


@dataclass
class ChainEpisode:
    episode_id: str
    slot_success: list

    @classmethod
    def from_dict(cls, d: dict) -> "ChainEpisode":
        return cls(d["episode_id"], [bool(v) for v in d["slot_success"]])

    def to_dict(self) -> dict:
        return {"episode_id": self.episode_id, "slot_success": list(self.slot_success)}


def _curve(alive_counts, n) -> list:
    return [100.0 * int(a) / n for a in alive_counts]


def progressive_completion(episodes, plan: ChainPlan) -> list:
    """% of chains whose every non-auto slot up to k succeeded (analytics.py:279-298)."""
    episodes = list(episodes)
    if not episodes:
        raise EmptyInput("no chain episodes")
    for ep in episodes:
        if len(ep.slot_success) != len(plan):
            raise ValueError(f"episode {ep.episode_id} has {len(ep.slot_success)} slots, "
                             f"plan {plan.name} has {len(plan)}")
    ok = np.array([ep.slot_success for ep in episodes], dtype=bool)
    auto = np.array([s.auto_success for s in plan.slots], dtype=bool)
    ok[:, auto] = True
    alive = np.logical_and.accumulate(ok, axis=1).sum(axis=0)
    return _curve(alive, len(episodes))


def progressive_completion_labels(labels, slot_label, plan: ChainPlan) -> list:
    """Device form for chains of labelled episodes: slot_label [n_chain,
    n_slots] int64 = label row of each bound slot (-1 for auto slots);
    slot success = success_once (tl_chain_progress)."""
    import torch
    sl = torch.as_tensor(slot_label, dtype=torch.int64)
    n_chain, n_slots = int(sl.shape[0]), int(sl.shape[1])
    if n_chain == 0:
        raise EmptyInput("no chain episodes")
    if n_slots != len(plan):
        raise ValueError(f"slot_label has {n_slots} slots, plan {plan.name} has {len(plan)}")
    lab = labels.view(-1, 24)
    sl = sl.to(lab.device).contiguous()
    alive = torch.empty(n_slots, dtype=torch.int64, device=lab.device)
    L.check(L.lib().tl_chain_progress(L.ptr(lab), L.ptr(sl), n_chain, n_slots, L.ptr(alive),
                                      L.stream_ptr()), "tl_chain_progress")
    return _curve(alive.cpu().numpy(), n_chain)


def independence_upper_bound(subtask_sor: dict, plan: ChainPlan) -> list:
    """Running product of per-subtask SoR; auto slots contribute 1 (analytics.py:301-312)."""
    out, acc = [], 1.0
    for s in plan.slots:
        if not s.auto_success:
            if s.subtask not in subtask_sor:
                raise MissingRate(f"no SoR for subtask {s.subtask!r} (slot {s.name})")
            acc *= subtask_sor[s.subtask]
        out.append(100.0 * acc)
    return out
