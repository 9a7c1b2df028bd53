"""Device batch layer: structure-of-arrays episode batches in HBM and the
calls into libtrajlab_b200.so.

Layout (include/trajlab_b200.h, tl_records): field planes in TRJL record
order, planes[f, r] for record r of the flat episode-major record axis;
episode e owns records [rec_start[e], rec_start[e] + n_rec[e]).  f32
planes are the binary32 contract of the reference (model.py:46-48,
synth.py:315-317); f64 planes carry arbitrary doubles exactly.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib as L
from .model import ART_ORDER, SUBTASK_ORDER, SCALAR_FIELDS, ArticulationKind
from .thresholds import THRESHOLD_FIELDS, Thresholds


def _torch():
    import torch
    return torch


def thresholds_c(th: Thresholds) -> L.Thresholds_c:
    return L.Thresholds_c(*[float(getattr(th, f)) for f in THRESHOLD_FIELDS])


def fuzz_cfg_c(cfg) -> L.FuzzCfg_c:
    return L.FuzzCfg_c(cfg.max_events, cfg.max_gap, cfg.max_tail, 0,
                       float(cfg.edge_density), float(cfg.success_prob))


def cset_build(subtask: int, art_kind: int, qmin: float, qmax: float, dof: int,
               rest_arm, rest_tor: float, th: Thresholds) -> bytes:
    """tl_cset_build (host function of the library) -> raw struct bytes."""
    ra = (ctypes.c_double * L.MAX_DOF)(*([float(v) for v in rest_arm] +
                                          [0.0] * (L.MAX_DOF - len(rest_arm))))
    out = L.Cset_c()
    rc = L.lib().tl_cset_build(int(subtask), int(art_kind), float(qmin), float(qmax),
                               int(dof), ctypes.cast(ra, ctypes.c_void_p),
                               float(rest_tor), ctypes.byref(thresholds_c(th)),
                               ctypes.byref(out))
    L.check(rc, "tl_cset_build")
    return bytes(out)


class CsetTable:
    """Deduplicated per-episode constant sets (header + resolved thresholds)."""

    def __init__(self):
        self._index = {}
        self._blobs = []

    def add(self, subtask, art_kind, qmin, qmax, dof, rest_arm, rest_tor, th) -> int:
        key = (int(subtask), int(art_kind),
               float(qmin).hex() if not math.isnan(qmin) else "nan",
               float(qmax).hex() if not math.isnan(qmax) else "nan",
               int(dof), tuple(float(v).hex() for v in rest_arm),
               float(rest_tor).hex(), th.astuple())
        i = self._index.get(key)
        if i is None:
            i = len(self._blobs)
            self._index[key] = i
            self._blobs.append(cset_build(subtask, art_kind, qmin, qmax, dof,
                                          rest_arm, rest_tor, th))
        return i

    def __len__(self):
        return len(self._blobs)

    def to_device(self, device):
        torch = _torch()
        buf = np.frombuffer(b"".join(self._blobs), np.uint8).copy()
        return torch.from_numpy(buf).to(device)


def synth_csets(th_label: Thresholds, dof: int = 7) -> CsetTable:
    """csets of synthetic headers (synth.py:331-341), index subtask*3 + art."""
    t = CsetTable()
    for s in range(4):
        for a in range(3):
            qmin, qmax = (0.0, 1.6) if a == 1 else (0.0, 0.5) if a == 2 else (math.nan, math.nan)
            art = a if s in (2, 3) else 0
            if art == 0:
                qmin = qmax = math.nan
            t._blobs.append(cset_build(s, art, qmin, qmax, dof, [0.0] * dof, 0.0, th_label))
    return t


@dataclass
class RecordBatch:
    planes: object        # torch [2*dof+9, cap] float32 | float64
    grasped: object       # torch [cap] uint8
    rec_start: object     # torch [n] int64
    n_rec: object         # torch [n] int32
    dof: int

    @property
    def n_env(self) -> int:
        return int(self.rec_start.shape[0])

    @property
    def dtype_code(self) -> int:
        return 0 if self.planes.dtype == _torch().float32 else 1

    def c(self) -> L.Records_c:
        return L.Records_c(self.planes.data_ptr(), self.grasped.data_ptr(),
                           self.rec_start.data_ptr(), self.n_rec.data_ptr(),
                           int(self.planes.shape[1]), self.dtype_code, int(self.dof))


def _is_f32_exact(a: np.ndarray) -> bool:
    b = a.astype(np.float32).astype(np.float64)
    return bool(np.all((b == a) | (np.isnan(a) & np.isnan(b))))


def pack_trajectories(trajs, th_base: Optional[Thresholds] = None, force_f64=False):
    """Host Trajectory objects -> (RecordBatch on the GPU, env_cset, csets).

    Picks f32 planes when every value is binary32-representable (the
    reference's storage contract), f64 planes otherwise (exact for any
    double, e.g. hand-built records)."""
    torch = _torch()
    dev = L.device()
    th_base = th_base or Thresholds()
    dof = trajs[0].header.arm_dof if trajs else 7
    for t in trajs:
        if t.header.arm_dof != dof:
            raise ValueError("all trajectories of a batch must share arm_dof")
    n_rec = np.array([len(t.records) for t in trajs], np.int32)
    # episodes start on 4-record boundaries so the label kernel can use
    # 128-bit loads (tl_label.cuh label_vec4); the gaps are zero padding
    n_pad = (n_rec.astype(np.int64) + 3) & ~3
    rec_start = np.zeros(len(trajs), np.int64)
    if len(trajs) > 1:
        rec_start[1:] = np.cumsum(n_pad[:-1], dtype=np.int64)
    R = int(n_pad.sum())
    F = 2 * dof + 9
    planes = np.zeros((F, max(R, 4)), np.float64)
    grasped = np.zeros(max(R, 4), np.uint8)
    table = CsetTable()
    env_cset = np.zeros(len(trajs), np.int32)
    for i, t in enumerate(trajs):
        h = t.header
        recs = t.records
        n = len(recs)
        r = int(rec_start[i])
        if n:
            for rec in recs:
                if len(rec.q_arm) != dof or len(rec.qd_arm) != dof:
                    raise ValueError(f"joint vector length mismatch: {len(rec.q_arm)} vs {dof}")
            planes[0:dof, r:r + n] = np.array([rec.q_arm for rec in recs], np.float64).T
            planes[dof:2 * dof, r:r + n] = np.array([rec.qd_arm for rec in recs], np.float64).T
            for j, f in enumerate(SCALAR_FIELDS):
                planes[2 * dof + j, r:r + n] = [getattr(rec, f) for rec in recs]
            grasped[r:r + n] = [1 if rec.grasped else 0 for rec in recs]
        if len(h.rest_arm) != dof:
            raise ValueError(f"joint vector length mismatch: {dof} vs {len(h.rest_arm)}")
        env_cset[i] = table.add(SUBTASK_ORDER.index(h.subtask_kind),
                                ART_ORDER.index(h.articulation_kind), h.art_qmin,
                                h.art_qmax, dof, h.rest_arm, h.rest_tor,
                                h.thresholds(th_base))
    use64 = force_f64 or not _is_f32_exact(planes[:, :R])
    host_planes = planes if use64 else planes.astype(np.float32)
    rb = RecordBatch(torch.from_numpy(host_planes).to(dev), torch.from_numpy(grasped).to(dev),
                     torch.from_numpy(rec_start).to(dev), torch.from_numpy(n_rec).to(dev), dof)
    return rb, torch.from_numpy(env_cset).to(dev), table.to_device(dev), len(table)


def pack_record_arrays(items, th_base: Optional[Thresholds] = None):
    """(TrajectoryHeader, TRJL structured record array) pairs -> f32 RecordBatch
    + csets, with no per-record Python objects: each field is one strided
    numpy copy into its plane (TRJL1 batched ingestion, io_binary.py:51-104).
    Episodes start on 4-record boundaries (128-bit label loads)."""
    torch = _torch()
    dev = L.device()
    th_base = th_base or Thresholds()
    dof = items[0][0].arm_dof if items else 7
    n_rec = np.array([len(a) for _, a in items], np.int64)
    n_pad = (n_rec + 3) & ~3
    rec_start = np.zeros(len(items), np.int64)
    if len(items) > 1:
        rec_start[1:] = np.cumsum(n_pad[:-1])
    R = int(n_pad.sum())
    F = 2 * dof + 9
    planes = np.zeros((F, max(R, 4)), np.float32)
    grasped = np.zeros(max(R, 4), np.uint8)
    table = CsetTable()
    env_cset = np.zeros(len(items), np.int32)
    for i, (h, arr) in enumerate(items):
        if h.arm_dof != dof:
            raise ValueError("all trajectories of a batch must share arm_dof")
        if len(h.rest_arm) != dof:
            raise ValueError(f"joint vector length mismatch: {dof} vs {len(h.rest_arm)}")
        r, n = int(rec_start[i]), len(arr)
        if n:
            planes[0:dof, r:r + n] = arr["q_arm"].T
            planes[dof:2 * dof, r:r + n] = arr["qd_arm"].T
            for j, f in enumerate(SCALAR_FIELDS):
                planes[2 * dof + j, r:r + n] = arr[f]
            grasped[r:r + n] = arr["grasped"] != 0
        env_cset[i] = table.add(SUBTASK_ORDER.index(h.subtask_kind),
                                ART_ORDER.index(h.articulation_kind), h.art_qmin,
                                h.art_qmax, dof, h.rest_arm, h.rest_tor, h.thresholds(th_base))
    rb = RecordBatch(torch.from_numpy(planes).to(dev), torch.from_numpy(grasped).to(dev),
                     torch.from_numpy(rec_start).to(dev),
                     torch.from_numpy(n_rec.astype(np.int32)).to(dev), dof)
    return rb, torch.from_numpy(env_cset).to(dev), table.to_device(dev), len(table)


def rules_c(rules_ids) -> Optional[L.Rules_c]:
    """[(subtask, branch, [mode ids])] -> tl_rules (None = reference tables)."""
    if rules_ids is None:
        return None
    r = L.Rules_c()
    for s in range(4):
        for b in range(2):
            ids = rules_ids[s][b]
            if len(ids) > 16:
                raise ValueError("at most 16 rules per branch")
            r.count[s][b] = len(ids)
            for i, m in enumerate(ids):
                r.ids[s][b][i] = m
    return r


@dataclass
class LabelResult:
    labels: object        # torch uint8 [n, 24] (tl_label)
    step_mask: object     # torch uint8 [cap] or None
    step_success: object  # torch uint8 [cap] or None
    ev_off: object = None
    ev_kind: object = None
    ev_t: object = None

    def labels_np(self):
        return self.labels.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)


def label_records(rb: RecordBatch, env_cset, csets, n_cset, rules=None,
                  want_mask=True, want_success=False, want_events=True,
                  ev_capacity=None) -> LabelResult:
    """K1 (+ scan + K2): events and modes for every episode of a batch."""
    torch = _torch()
    dev = rb.planes.device
    n = rb.n_env
    cap = int(rb.planes.shape[1])
    labels = torch.empty((n, 24), dtype=torch.uint8, device=dev)
    mask = torch.zeros(cap, dtype=torch.uint8, device=dev) if (want_mask or want_events) else None
    succ = torch.empty(cap, dtype=torch.uint8, device=dev) if want_success else None
    rc_rules = rules_c(rules)
    rc = L.lib().tl_label_records(
        ctypes.byref(rb.c()), n, L.ptr(env_cset), L.ptr(csets), n_cset,
        ctypes.byref(rc_rules) if rc_rules is not None else None,
        L.ptr(mask), L.ptr(succ), L.ptr(labels), L.stream_ptr())
    L.check(rc, "tl_label_records")
    res = LabelResult(labels, mask, succ)
    if want_events:
        emit_events(rb, res, ev_capacity)
    return res


def emit_events(rb: RecordBatch, res: LabelResult, ev_capacity=None):
    torch = _torch()
    dev = rb.planes.device
    n = rb.n_env
    ev_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    scratch = torch.empty(max(16, L.lib().tl_scan_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    if ev_capacity is None:
        # exact-size outputs: scan, read the total, then emit
        L.check(L.lib().tl_scan_events(L.ptr(res.labels), n, L.ptr(ev_off), L.ptr(scratch),
                                       L.stream_ptr()), "tl_scan_events")
        total = int(ev_off[n].item())
        ev_kind = torch.empty(max(total, 1), dtype=torch.uint8, device=dev)
        ev_t = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        L.check(L.lib().tl_emit_events(L.ptr(res.step_mask), L.ptr(rb.rec_start),
                                       L.ptr(rb.n_rec), L.ptr(res.labels), L.ptr(ev_off), n,
                                       L.ptr(ev_kind), L.ptr(ev_t), L.stream_ptr()),
                "tl_emit_events")
    else:
        # capacity-bounded outputs: one fused launch, no host round trip
        ev_kind = torch.empty(max(int(ev_capacity), 1), dtype=torch.uint8, device=dev)
        ev_t = torch.empty(max(int(ev_capacity), 1), dtype=torch.int32, device=dev)
        L.check(L.lib().tl_scan_emit_events(L.ptr(res.step_mask), L.ptr(rb.rec_start),
                                            L.ptr(rb.n_rec), L.ptr(res.labels), n,
                                            L.ptr(ev_off), L.ptr(ev_kind), L.ptr(ev_t),
                                            L.ptr(scratch), L.stream_ptr()),
                "tl_scan_emit_events")
    res.ev_off, res.ev_kind, res.ev_t = ev_off, ev_kind, ev_t
    return res


def eval_predicates(rb: RecordBatch, env_cset, csets, a0=None):
    """tl_eval_predicates -> (bits u8, errs u8, jmax f64) torch tensors."""
    torch = _torch()
    dev = rb.planes.device
    cap = int(rb.planes.shape[1])
    bits = torch.zeros(cap, dtype=torch.uint8, device=dev)
    errs = torch.zeros(cap, dtype=torch.uint8, device=dev)
    jmax = torch.zeros(cap, dtype=torch.float64, device=dev)
    a0t = None
    if a0 is not None:
        a0t = torch.as_tensor(np.asarray(a0, np.float64), device=dev)
    rc = L.lib().tl_eval_predicates(ctypes.byref(rb.c()), rb.n_env, L.ptr(env_cset),
                                    L.ptr(csets), L.ptr(a0t), L.ptr(bits), L.ptr(errs),
                                    L.ptr(jmax), L.stream_ptr())
    L.check(rc, "tl_eval_predicates")
    return bits, errs, jmax


class _OneRecord:
    """tl_eval_predicates on ONE record for the scalar drop-in calls
    (is_static, is_open, success_step, ... on a single TimestepRecord):
    the record, its cset and the optional anchor are packed into a pinned
    host staging block, then one H2D copy, one launch, one D2H copy of the
    three outputs and one stream synchronize -- instead of a trajectory pack
    (six copies) and three blocking reads per call.  The staging block and
    the csets (keyed like CsetTable) are reused across calls."""

    # byte layout of the staging block (8-byte aligned fields, cap = 4 records)
    _CAP = 4
    _PLANES = 0
    _GRASPED = (2 * L.MAX_DOF + 9) * 4 * 8
    _REC_START = _GRASPED + 8
    _N_REC = _REC_START + 8
    _ENV_CSET = _N_REC + 8
    _A0 = _ENV_CSET + 8
    _CSET = _A0 + 8
    _SIZE = (_CSET + 512 + 255) & ~255

    def __init__(self, dev):
        torch = _torch()
        self.host = torch.zeros(self._SIZE, dtype=torch.uint8, pin_memory=True)
        self.dev = torch.zeros(self._SIZE, dtype=torch.uint8, device=dev)
        self.out_dev = torch.zeros(64, dtype=torch.uint8, device=dev)
        self.out_host = torch.zeros(64, dtype=torch.uint8, pin_memory=True)
        self.h = self.host.numpy()
        self.o = self.out_host.numpy()
        self.csets = {}
        base = self.dev.data_ptr()
        self.p_planes = base + self._PLANES
        self.p_grasped = base + self._GRASPED
        self.p_rec_start = base + self._REC_START
        self.p_n_rec = base + self._N_REC
        self.p_env = base + self._ENV_CSET
        self.p_a0 = base + self._A0
        self.p_cset = base + self._CSET
        ob = self.out_dev.data_ptr()
        self.p_bits, self.p_errs, self.p_jmax = ob, ob + 8, ob + 32
        self.h[self._REC_START:self._REC_START + 8] = np.zeros(1, np.int64).view(np.uint8)
        self.h[self._N_REC:self._N_REC + 4] = np.ones(1, np.int32).view(np.uint8)
        self.h[self._ENV_CSET:self._ENV_CSET + 4] = np.zeros(1, np.int32).view(np.uint8)

    def cset(self, subtask, art_kind, qmin, qmax, dof, rest_arm, rest_tor, th) -> bytes:
        key = (int(subtask), int(art_kind),
               float(qmin).hex() if not math.isnan(qmin) else "nan",
               float(qmax).hex() if not math.isnan(qmax) else "nan",
               int(dof), tuple(float(v).hex() for v in rest_arm),
               float(rest_tor).hex(), th.astuple())
        b = self.csets.get(key)
        if b is None:
            b = cset_build(subtask, art_kind, qmin, qmax, dof, rest_arm, rest_tor, th)
            self.csets[key] = b
        return b

    def eval(self, values, grasped: bool, dof: int, cset: bytes, a0=None):
        """values: the 2*dof+9 record fields in plane order (f64) ->
        (bits, errs, jmax) of the record."""
        torch = _torch()
        F = 2 * dof + 9
        planes = self.h[self._PLANES:self._PLANES + F * self._CAP * 8].view(np.float64).reshape(F, self._CAP)
        planes[:, 0] = values
        self.h[self._GRASPED] = 1 if grasped else 0
        self.h[self._A0:self._A0 + 8] = np.array([0.0 if a0 is None else a0], np.float64).view(np.uint8)
        self.h[self._CSET:self._CSET + len(cset)] = np.frombuffer(cset, np.uint8)
        stream = torch.cuda.current_stream()
        self.dev.copy_(self.host, non_blocking=True)
        rec = L.Records_c(self.p_planes, self.p_grasped, self.p_rec_start, self.p_n_rec,
                          self._CAP, 1, int(dof))
        rc = L.lib().tl_eval_predicates(ctypes.byref(rec), 1, ctypes.c_void_p(self.p_env),
                                        ctypes.c_void_p(self.p_cset),
                                        None if a0 is None else ctypes.c_void_p(self.p_a0),
                                        ctypes.c_void_p(self.p_bits), ctypes.c_void_p(self.p_errs),
                                        ctypes.c_void_p(self.p_jmax),
                                        ctypes.c_void_p(stream.cuda_stream))
        L.check(rc, "tl_eval_predicates")
        self.out_host.copy_(self.out_dev, non_blocking=True)
        stream.synchronize()
        return int(self.o[0]), int(self.o[8]), float(self.o[32:40].view(np.float64)[0])


_one = {}


def one_record():
    """The per-device _OneRecord staging (created on first use)."""
    dev = L.device()
    r = _one.get(dev.index)
    if r is None:
        r = _one[dev.index] = _OneRecord(dev)
    return r


def classify_lists(kinds_list, subtasks, d0s, d0_none, rules=None):
    """tl_classify_events over host event lists -> numpy tl_label array."""
    torch = _torch()
    dev = L.device()
    n = len(kinds_list)
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(k) for k in kinds_list])
    flat = np.concatenate([np.asarray(k, np.uint8) for k in kinds_list]) if n and off[-1] else np.zeros(1, np.uint8)
    t_kind = torch.from_numpy(flat).to(dev)
    t_off = torch.from_numpy(off).to(dev)
    t_sub = torch.from_numpy(np.asarray(subtasks, np.uint8)).to(dev)
    t_d0 = torch.from_numpy(np.asarray(d0s, np.float64)).to(dev)
    t_none = torch.from_numpy(np.asarray(d0_none, np.uint8)).to(dev)
    out = torch.empty((max(n, 1), 24), dtype=torch.uint8, device=dev)
    rc_rules = rules_c(rules)
    rc = L.lib().tl_classify_events(L.ptr(t_kind), L.ptr(t_off), L.ptr(t_sub), L.ptr(t_d0),
                                    L.ptr(t_none), n,
                                    ctypes.byref(rc_rules) if rc_rules is not None else None,
                                    L.ptr(out), L.stream_ptr())
    L.check(rc, "tl_classify_events")
    return out[:n].cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)


def fuzz_capacity(cfg) -> int:
    """upper bound of records per fuzz episode (synth.py:363-507, :298-310)"""
    n = 2 + (cfg.max_events + 4) * cfg.max_gap + cfg.max_tail
    return (n + 3) & ~3  # 4-record aligned episode slots (128-bit label loads)


@dataclass
class SynthBatch:
    records: RecordBatch
    labels: object
    step_mask: object
    scripts: object = None      # torch uint8 [n, 56] (tl_script) or None
    script_kind: object = None
    script_gap: object = None
    label_result: Optional[LabelResult] = None


class SynthWorkspace:
    """Preallocated device buffers for repeated fuzz batches (bench/env)."""

    def __init__(self, n_env, cap_per_env, dof=7, with_scripts=False, max_steps=12):
        torch = _torch()
        dev = L.device()
        total = n_env * cap_per_env
        self.planes = torch.empty((2 * dof + 9, total), dtype=torch.float32, device=dev)
        self.grasped = torch.empty(total, dtype=torch.uint8, device=dev)
        self.rec_start = torch.empty(n_env, dtype=torch.int64, device=dev)
        self.n_rec = torch.empty(n_env, dtype=torch.int32, device=dev)
        self.labels = torch.empty((n_env, 24), dtype=torch.uint8, device=dev)
        self.step_mask = torch.empty(total, dtype=torch.uint8, device=dev)
        self.scripts = torch.empty((n_env, 56), dtype=torch.uint8, device=dev) if with_scripts else None
        self.script_kind = torch.empty(n_env * max_steps, dtype=torch.uint8, device=dev) if with_scripts else None
        self.script_gap = torch.empty(n_env * max_steps, dtype=torch.int32, device=dev) if with_scripts else None
        c_cfg = L.FuzzCfg_c(max_steps - 4, 1, 1, 0, 1.0, 0.5)
        # zero-filled once: the claim counters in it are left at zero by every call
        self.scratch = torch.zeros(int(L.lib().tl_fuzz_scratch_bytes(n_env, ctypes.byref(c_cfg))),
                                   dtype=torch.uint8, device=dev)
        self.n_env, self.cap, self.dof, self.max_steps = n_env, cap_per_env, dof, max_steps

    def records(self):
        return RecordBatch(self.planes, self.grasped, self.rec_start, self.n_rec, self.dof)


def fuzz_batch(seeds, subtask, cfg, th_realize: Thresholds, label_csets,
               ws: Optional[SynthWorkspace] = None, want_scripts=False,
               rules=None, events=False) -> SynthBatch:
    """tl_fuzz: fuzz(seed) -> records + labels for every seed (one launch).
    events=True: tl_fuzz_ev, the ordered event lists built inside the same
    launch (SynthBatch.label_result holds ev_off / ev_kind / ev_t).
    subtask: one subtask index for the batch, or one per seed (array /
    tensor: tl_fuzz_mixed / tl_fuzz_ev_mixed)."""
    torch = _torch()
    dev = L.device()
    if not torch.is_tensor(seeds):
        seeds = torch.as_tensor(np.asarray(seeds, np.int64), device=dev)
    n = int(seeds.shape[0])
    mixed = torch.is_tensor(subtask) or isinstance(subtask, (list, tuple, np.ndarray))
    if mixed:
        subs = torch.as_tensor(np.asarray(subtask.cpu() if torch.is_tensor(subtask) else subtask),
                               dtype=torch.uint8).to(dev)
        if int(subs.shape[0]) != n:
            raise ValueError(f"{int(subs.shape[0])} subtasks for {n} seeds")
    cap = fuzz_capacity(cfg)
    if (ws is None or ws.n_env < n or ws.cap != cap or ws.max_steps != cfg.max_events + 4
            or (want_scripts and ws.scripts is None)):
        ws = SynthWorkspace(n, cap, with_scripts=want_scripts, max_steps=cfg.max_events + 4)
    rb = ws.records()
    c_cfg = L.FuzzCfg_c(cfg.max_events, cfg.max_gap, cfg.max_tail, 0,
                        float(cfg.edge_density), float(cfg.success_prob))
    rc_rules = rules_c(rules)
    args = [L.ptr(seeds), *((L.ptr(subs),) if mixed else ()), n,
            *(() if mixed else (int(subtask),)), ctypes.byref(c_cfg),
            ctypes.byref(thresholds_c(th_realize)), L.ptr(label_csets),
            ctypes.byref(rc_rules) if rc_rules is not None else None,
            ctypes.byref(rb.c()), cap,
            L.ptr(ws.script_kind) if want_scripts else None,
            L.ptr(ws.script_gap) if want_scripts else None,
            L.ptr(ws.scripts) if want_scripts else None,
            L.ptr(ws.step_mask), L.ptr(ws.labels)]
    res = None
    if events:
        ev_cap = 4 * n * cap
        ev_off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        ev_kind = torch.empty(ev_cap, dtype=torch.uint8, device=dev)
        ev_t = torch.empty(ev_cap, dtype=torch.int32, device=dev)
        fn = L.lib().tl_fuzz_ev_mixed if mixed else L.lib().tl_fuzz_ev
        rc = fn(*args, L.ptr(ev_off), L.ptr(ev_kind), L.ptr(ev_t), ev_cap,
                L.ptr(ws.scratch), L.stream_ptr())
        L.check(rc, "tl_fuzz_ev")
        res = LabelResult(ws.labels, ws.step_mask, None)
        res.ev_off, res.ev_kind, res.ev_t = ev_off, ev_kind, ev_t
    else:
        fn = L.lib().tl_fuzz_mixed if mixed else L.lib().tl_fuzz
        rc = fn(*args, L.ptr(ws.scratch), L.stream_ptr())
        L.check(rc, "tl_fuzz")
    return SynthBatch(rb, ws.labels, ws.step_mask,
                      ws.scripts if want_scripts else None,
                      ws.script_kind if want_scripts else None,
                      ws.script_gap if want_scripts else None, res)


def realize_batch(scripts_np, step_kind, step_gap, th_realize: Thresholds, label_csets,
                  dof=7, rules=None) -> SynthBatch:
    """tl_realize over host scripts (SCRIPT_DTYPE array + step arrays)."""
    torch = _torch()
    dev = L.device()
    n = len(scripts_np)
    # record count per episode (synth.py:298-310): 1 + sum(gaps) + tail_eff
    n_rec = np.zeros(n, np.int64)
    for i, s in enumerate(scripts_np):
        g = step_gap[s["step_off"]:s["step_off"] + s["n_steps"]]
        tmin = 0 if s["n_steps"] else 1
        n_rec[i] = max(2, 1 + int(np.sum(np.maximum(g, 0))) + max(int(s["tail"]), tmin))
    n_pad = (n_rec + 3) & ~3  # 4-record aligned episode slots
    rec_start = np.zeros(n, np.int64)
    if n > 1:
        rec_start[1:] = np.cumsum(n_pad[:-1])
    R = int(n_pad.sum())
    planes = torch.zeros((2 * dof + 9, max(R, 4)), dtype=torch.float32, device=dev)
    grasped = torch.zeros(max(R, 4), dtype=torch.uint8, device=dev)
    rb = RecordBatch(planes, grasped, torch.from_numpy(rec_start).to(dev),
                     torch.from_numpy(n_rec.astype(np.int32)).to(dev), dof)
    labels = torch.empty((max(n, 1), 24), dtype=torch.uint8, device=dev)
    mask = torch.zeros(max(R, 1), dtype=torch.uint8, device=dev)
    t_sc = torch.from_numpy(np.ascontiguousarray(scripts_np).view(np.uint8).reshape(n, 56)).to(dev)
    t_k = torch.from_numpy(np.asarray(step_kind, np.uint8).reshape(-1) if len(step_kind) else np.zeros(1, np.uint8)).to(dev)
    t_g = torch.from_numpy(np.asarray(step_gap, np.int32).reshape(-1) if len(step_gap) else np.zeros(1, np.int32)).to(dev)
    rc_rules = rules_c(rules)
    scratch = torch.empty(int(L.lib().tl_realize_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    rc = L.lib().tl_realize(L.ptr(t_sc), L.ptr(t_k), L.ptr(t_g), n,
                            ctypes.byref(thresholds_c(th_realize)), L.ptr(label_csets),
                            ctypes.byref(rc_rules) if rc_rules is not None else None,
                            ctypes.byref(rb.c()), L.ptr(mask), L.ptr(labels), L.ptr(scratch),
                            L.stream_ptr())
    L.check(rc, "tl_realize")
    return SynthBatch(rb, labels[:n], mask)


def mode_histogram(labels, n):
    torch = _torch()
    hist = torch.zeros(L.N_MODES, dtype=torch.int64, device=labels.device)
    L.check(L.lib().tl_mode_histogram(L.ptr(labels), n, L.ptr(hist), L.stream_ptr()),
            "tl_mode_histogram")
    return hist


def filter_select(bucket, n_buckets, pool_b0, bucket_w, quota):
    """K5 on device arrays; returns (selected u8 tensor, pool_selected i64)."""
    torch = _torch()
    dev = L.device()
    n = int(bucket.shape[0])
    n_pools = int(pool_b0.shape[0]) - 1
    sel = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    ps = torch.zeros(max(n_pools, 1), dtype=torch.int64, device=dev)
    nbytes = L.lib().tl_filter_scratch_bytes(n, n_buckets, max(n_pools, 0))
    scratch = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=dev)
    rc = L.lib().tl_filter_select(L.ptr(bucket), n, n_buckets, n_pools, L.ptr(pool_b0),
                                  L.ptr(bucket_w), int(quota), L.ptr(sel), L.ptr(ps),
                                  L.ptr(scratch), L.stream_ptr())
    L.check(rc, "tl_filter_select")
    return sel[:n], ps[:n_pools]


def validate_records(rb: RecordBatch, vbounds, t=None):
    """tl_validate_records (model.py:255-274 invariants as TL_VF_* codes):
    -> (vflags u8 device tensor per record, per-episode tl_vsummary numpy)."""
    torch = _torch()
    dev = rb.planes.device
    n = rb.n_env
    vflags = torch.zeros(max(int(rb.planes.shape[1]), 1), dtype=torch.uint8, device=dev)
    vsum = torch.empty(max(n, 1) * L.VSUMMARY_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    vb = torch.from_numpy(np.ascontiguousarray(vbounds).view(np.uint8).copy()).to(dev)
    rc = L.lib().tl_validate_records(ctypes.byref(rb.c()), n, L.ptr(vb), L.ptr(t), L.ptr(vflags),
                                     L.ptr(vsum), L.stream_ptr())
    L.check(rc, "tl_validate_records")
    return vflags, vsum.cpu().numpy().view(L.VSUMMARY_DTYPE)[:n]
