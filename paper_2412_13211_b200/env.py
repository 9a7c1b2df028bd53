"""BatchedSubtaskEnv: N independent synthetic subtask environments on the
GPU behind reset / step(actions) (csrc/tl_env.cuh).

The reference's only environment dynamics are the script realizer
(synth.py:100-302): reset is ``_Realizer.__init__`` plus the t = 0 record,
and every later record is one step -- ``_advance_cum``, ``_apply(action)``
unless the action is a hold, ``_emit``.  ``realize(script, seed)`` is
therefore ``reset(scripts=[script], seeds=[seed])`` followed by the
``scripted_actions`` stream, and ``fuzz(seed, kind)`` is
``reset(seeds=[seed], subtask=kind)`` followed by the same; the tests check
both bit-exactly against the reference's fixtures.

Each step also folds the new record's edge events (events.py:94-193) into a
per-env label state, so ``labels()`` classifies every episode so far
without re-reading records.  Observations are time-major f32 planes in the
record field order (q_arm[dof], qd_arm[dof], q_tor, v_base_x, v_base_y,
omega_base, dist_ee_rest, dist_obj_goal, force_ee_target, cum_robot_force,
art_q) plus grasped, shape [F, K, N] for K steps of N envs.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from . import core
from .errors import infeasible_error
from .events import EVENT_KINDS, EventKind
from .model import SUBTASK_ORDER, SubtaskKind
from .synth import FuzzConfig, _label_csets, _script_array, LEVELS
from .thresholds import Thresholds

HOLD = 255       # TL_ACT_HOLD: no event this step (synth.py:198-201)
IDLE = 254       # TL_ACT_IDLE: env does not advance (no record)
BAD_GAP = 253    # TL_ACT_BAD_GAP: run()'s "event gap must be >= 1"


def _torch():
    import torch
    return torch


@dataclass
class EnvStep:
    obs: object          # torch f32 [F, K, N]
    grasped: object      # torch u8 [K, N]
    step_mask: object    # torch u8 [K, N]: EVENT_ORDER bits fired at the record


class BatchedSubtaskEnv:
    """N environments stepped by one kernel launch per call (any K >= 1
    steps per launch; actions [K, N] u8: EventKind index, HOLD or IDLE)."""

    def __init__(self, n_env: int, dof: int = 7, th: Optional[Thresholds] = None,
                 th_label: Optional[Thresholds] = None):
        torch = _torch()
        if not 1 <= dof <= L.MAX_DOF:
            raise ValueError(f"arm_dof must be in [1, {L.MAX_DOF}]")
        self.dev = L.device()
        self.n_env, self.dof = int(n_env), int(dof)
        self.n_fields = 2 * dof + 9
        self.th = th or Thresholds()
        self._csets = _label_csets(th_label, dof)
        self.state = torch.empty(int(L.lib().tl_env_state_bytes(self.n_env)),
                                 dtype=torch.uint8, device=self.dev)
        self.scripts = None      # device tl_script [N] (fuzz: sampled scripts)
        self._kinds = None
        self._gaps = None
        self._subtasks = None
        self._levels = None
        self.t = 0

    # -- buffers --------------------------------------------------------------
    def _outputs(self, k: int, out: Optional[EnvStep]):
        torch = _torch()
        if out is not None:
            return out
        n = self.n_env
        return EnvStep(torch.empty((self.n_fields, k, n), dtype=torch.float32, device=self.dev),
                       torch.empty((k, n), dtype=torch.uint8, device=self.dev),
                       torch.empty((k, n), dtype=torch.uint8, device=self.dev))

    @staticmethod
    def _check_out(out: EnvStep, f: int, k: int, n: int):
        if tuple(out.obs.shape) != (f, k, n) or not out.obs.is_contiguous():
            raise ValueError(f"obs buffer must be a contiguous [{f}, {k}, {n}] tensor")

    # -- reset ----------------------------------------------------------------
    def reset(self, scripts=None, seeds: Optional[Sequence[int]] = None,
              subtask=None, config: Optional[FuzzConfig] = None,
              out: Optional[EnvStep] = None) -> EnvStep:
        """scripts (+ realize seeds, default 0): _Realizer(script, seed).
        Otherwise seeds + subtask: random_script(seed, subtask, config) initial
        conditions, realize RNG seeded with seed ^ 0x5EED (fuzz, synth.py:510-515)."""
        torch = _torch()
        n = self.n_env
        o = self._outputs(1, out)
        self._check_out(o, self.n_fields, 1, n)
        stride = o.obs.stride(0)
        if scripts is not None:
            if len(scripts) != n:
                raise ValueError(f"expected {n} scripts")
            if any(int(s.arm_dof) != self.dof for s in scripts):
                raise ValueError("script arm_dof differs from the env's dof")
            seeds = [0] * n if seeds is None else list(seeds)
            arr, kinds, gaps = _script_array(scripts, seeds)
            self.scripts = torch.from_numpy(arr.view(np.uint8).reshape(n, 56)).to(self.dev)
            self._kinds = torch.from_numpy(kinds if len(kinds) else np.zeros(1, np.uint8)).to(self.dev)
            self._gaps = torch.from_numpy(gaps if len(gaps) else np.zeros(1, np.int32)).to(self.dev)
            self._subtasks = [SubtaskKind(s.subtask_kind).value for s in scripts]
            self._levels = [s.initial_art_level for s in scripts]
            rc = L.lib().tl_env_reset(L.ptr(self.state), n, self.dof, L.ptr(self.scripts),
                                      ctypes.byref(core.thresholds_c(self.th)), L.ptr(self._csets),
                                      L.ptr(o.obs), stride, L.ptr(o.grasped), L.ptr(o.step_mask),
                                      L.stream_ptr())
            L.check(rc, "tl_env_reset")
        else:
            if seeds is None or subtask is None:
                raise ValueError("reset needs scripts, or seeds and a subtask")
            if self.dof != 7:
                raise ValueError("fuzz resets build arm_dof = 7 scripts")
            cfg = config or FuzzConfig()
            if cfg.max_gap < 1 or cfg.max_tail < 1:
                raise ValueError("empty range for randrange()")  # randint(1, 0)
            kind = SubtaskKind(subtask)
            if torch.is_tensor(seeds):
                s_t = seeds.to(device=self.dev, dtype=torch.int64).contiguous()
            else:
                s_t = torch.as_tensor(np.asarray(seeds, np.int64)).to(self.dev)
            if s_t.numel() != n:
                raise ValueError(f"expected {n} seeds")
            ms = cfg.max_events + 4
            self.scripts = torch.empty((n, 56), dtype=torch.uint8, device=self.dev)
            self._kinds = torch.empty(n * ms, dtype=torch.uint8, device=self.dev)
            self._gaps = torch.empty(n * ms, dtype=torch.int32, device=self.dev)
            self._subtasks = [kind.value] * n
            self._levels = None
            rc = L.lib().tl_env_reset_fuzz(L.ptr(self.state), L.ptr(s_t), n,
                                           SUBTASK_ORDER.index(kind),
                                           ctypes.byref(core.fuzz_cfg_c(cfg)),
                                           ctypes.byref(core.thresholds_c(self.th)),
                                           L.ptr(self._csets), L.ptr(self.scripts),
                                           L.ptr(self._kinds), L.ptr(self._gaps), L.ptr(o.obs),
                                           stride, L.ptr(o.grasped), L.ptr(o.step_mask),
                                           L.stream_ptr())
            L.check(rc, "tl_env_reset_fuzz")
        self.t = 0
        return o

    # -- step -----------------------------------------------------------------
    def step(self, actions, out: Optional[EnvStep] = None) -> EnvStep:
        """actions: [N] or [K, N] (EventKind, its index, HOLD or IDLE)."""
        torch = _torch()
        a = actions
        if not torch.is_tensor(a):
            a = np.asarray([EVENT_KINDS.index(x) if isinstance(x, EventKind) else int(x)
                            for x in np.asarray(a, dtype=object).reshape(-1)],
                           np.uint8).reshape(np.shape(actions))
            a = torch.from_numpy(a)
        if a.dim() == 1:
            a = a.reshape(1, -1)
        if a.shape[1] != self.n_env:
            raise ValueError(f"actions must be [K, {self.n_env}]")
        a = a.to(device=self.dev, dtype=torch.uint8).contiguous()
        k = int(a.shape[0])
        o = self._outputs(k, out)
        self._check_out(o, self.n_fields, k, self.n_env)
        rc = L.lib().tl_env_step(L.ptr(self.state), self.n_env, self.dof, L.ptr(a), k,
                                 L.ptr(o.obs), o.obs.stride(0), L.ptr(o.grasped),
                                 L.ptr(o.step_mask), L.stream_ptr())
        L.check(rc, "tl_env_step")
        self.t += k
        return o

    def scripted_actions(self, t0: int, k: int):
        """actions [k, N] replaying the reset scripts for records t0..t0+k-1."""
        torch = _torch()
        if self.scripts is None:
            raise RuntimeError("reset first")
        a = torch.empty((k, self.n_env), dtype=torch.uint8, device=self.dev)
        rc = L.lib().tl_env_script_actions(L.ptr(self.scripts), L.ptr(self._kinds),
                                           L.ptr(self._gaps), self.n_env, int(t0), int(k),
                                           L.ptr(a), L.stream_ptr())
        L.check(rc, "tl_env_script_actions")
        return a

    def script_lengths(self) -> np.ndarray:
        """records per env of the reset scripts (synth.py:298-310)."""
        sc = self.scripts.cpu().numpy().reshape(-1).view(L.SCRIPT_DTYPE)
        g = self._gaps.cpu().numpy()
        out = np.zeros(self.n_env, np.int64)
        for i, s in enumerate(sc):
            ns = max(int(s["n_steps"]), 0)
            gg = g[int(s["step_off"]):int(s["step_off"]) + ns]
            out[i] = max(2, 1 + int(gg.sum()) + max(int(s["tail"]), 0 if ns else 1))
        return out

    # -- labels ---------------------------------------------------------------
    def labels(self, rules=None):
        """(LABEL_DTYPE array, n_rec) of every env's episode so far."""
        torch = _torch()
        lab = torch.empty((self.n_env, 24), dtype=torch.uint8, device=self.dev)
        nrec = torch.empty(self.n_env, dtype=torch.int32, device=self.dev)
        rc_rules = core.rules_c(rules)
        rc = L.lib().tl_env_labels(L.ptr(self.state), self.n_env,
                                   ctypes.byref(rc_rules) if rc_rules is not None else None,
                                   L.ptr(lab), L.ptr(nrec), L.stream_ptr())
        L.check(rc, "tl_env_labels")
        return lab.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE), nrec.cpu().numpy()

    def errors(self, labels=None):
        """per env: the InfeasibleScript the reference would raise, or None."""
        lab = self.labels()[0] if labels is None else labels
        out = []
        for i in range(self.n_env):
            st = int(lab["status"][i])
            if not (20 <= st <= 41 or st == L.ERR_SCRIPT_CAPACITY):
                out.append(None)
                continue
            a = int(lab["pad"][i])
            ev = EVENT_KINDS[a].value if a < len(EVENT_KINDS) else str(a)
            lvl = self._levels[i] if self._levels else None
            out.append(infeasible_error(st, self._subtasks[i], ev, lvl))
        return out

    def rollout(self, n_steps: Optional[int] = None):
        """Replay the reset scripts to their end in one launch: obs [F, T, N]
        (record 0 from reset excluded), step masks [T, N]."""
        if n_steps is None:
            n_steps = int(self.script_lengths().max()) - 1
        return self.step(self.scripted_actions(self.t + 1, n_steps))
