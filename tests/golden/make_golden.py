"""Generate golden fixtures by running the REFERENCE trajlab package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every expected value in tests/golden/ comes from the reference's own code
(/root/reference/pkg/src/trajlab), imported read-only; nothing here calls
the oracle or the product.  The fixtures travel to the GPU box (the
reference does not), where tests compare the CUDA path and the oracle
against them.

Files:
  fuzz.npz       fuzz(seed, kind) for 4 kinds x SEEDS: scripts, f32 records,
                 events, modes (synth.py:510, events.py:94, modes.py:235)
  defining.npz   realize(defining_scripts()[m], seed) for seeds 7, 123
  long.npz       200-step C1/C2/C3 shaped episodes + max_gap=64 fuzz
  crafted.npz    hand-built record streams (multi-event steps, f32/f64
                 boundary values, NaNs, overrides) -> events/modes/errors
  scripts.json.gzarbitrary (often infeasible) scripts -> realize outcome
  classify.json.gzevent lists -> classify outcome (incl. rules= override)
  filter.json.gz label sets + FilterSpec -> DatasetManifest
"""
from __future__ import annotations

import gzip
import json
import math
import os
import random
import struct
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import trajlab as T  # noqa: E402
from trajlab import synth  # noqa: E402
from trajlab.events import EVENT_ORDER  # noqa: E402
from trajlab.modes import MODE_IDS, MODE_RULES  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
KINDS = [T.SubtaskKind.Pick, T.SubtaskKind.Place, T.SubtaskKind.Open,
         T.SubtaskKind.Close]
EVENT_KINDS = [e.value for e in T.EventKind]
ALL_MODES = [m for k in KINDS for m in MODE_IDS[k]]
LEVELS = ["low", "slight", "open", "high", "closed"]
ART = ["None", "Fridge", "Drawer"]
SCALARS = ["q_tor", "v_base_x", "v_base_y", "omega_base", "dist_ee_rest",
           "dist_obj_goal", "force_ee_target", "cum_robot_force", "art_q"]
TH_FIELDS = list(T.Thresholds().to_dict().keys())


def f32(x):
    return struct.unpack("<f", struct.pack("<f", x))[0]


# -- packing -----------------------------------------------------------------

class Pack:
    """Ragged episode-major SoA: planes[2*dof+9][R], grasped[R], rec_off[N+1]."""

    def __init__(self, dtype=np.float32):
        self.dtype = dtype
        self.eps = []

    def add(self, traj, **meta):
        self.eps.append((traj, meta))

    def arrays(self, prefix=""):
        dof = 7
        R = sum(len(t.records) for t, _ in self.eps)
        planes = np.zeros((2 * dof + 9, R), self.dtype)
        grasped = np.zeros(R, np.uint8)
        off = np.zeros(len(self.eps) + 1, np.int64)
        hdr = {k: [] for k in ("subtask", "art_kind", "art_qmin", "art_qmax",
                               "rest_tor")}
        rest_arm = np.zeros((len(self.eps), dof))
        r = 0
        for i, (traj, _) in enumerate(self.eps):
            h = traj.header
            assert h.arm_dof == dof
            for rec in traj.records:
                planes[0:dof, r] = rec.q_arm
                planes[dof:2 * dof, r] = rec.qd_arm
                for j, f in enumerate(SCALARS):
                    planes[2 * dof + j, r] = getattr(rec, f)
                grasped[r] = 1 if rec.grasped else 0
                r += 1
            off[i + 1] = r
            hdr["subtask"].append(KINDS.index(h.subtask_kind))
            hdr["art_kind"].append(ART.index(h.articulation_kind.value))
            hdr["art_qmin"].append(h.art_qmin)
            hdr["art_qmax"].append(h.art_qmax)
            hdr["rest_tor"].append(h.rest_tor)
            rest_arm[i] = h.rest_arm
        if self.dtype == np.float32:
            # the stored values must be exactly the reference's doubles
            for i, (traj, _) in enumerate(self.eps):
                for t, rec in enumerate(traj.records):
                    rr = off[i] + t
                    for j, f in enumerate(SCALARS):
                        v = getattr(rec, f)
                        w = float(planes[2 * dof + j, rr])
                        assert v == w or (math.isnan(v) and math.isnan(w)), (f, v, w)
        out = {prefix + "planes": planes, prefix + "grasped": grasped,
               prefix + "rec_off": off, prefix + "rest_arm": rest_arm}
        for k, v in hdr.items():
            out[prefix + k] = np.asarray(v, np.float64 if "art_q" in k or k == "rest_tor" else np.int32)
        return out


def events_arrays(evlists, prefix=""):
    kinds, ts, off = [], [], [0]
    for ev in evlists:
        for e in ev:
            kinds.append(EVENT_KINDS.index(e.kind.value))
            ts.append(e.t)
        off.append(len(kinds))
    return {prefix + "ev_kind": np.asarray(kinds, np.uint8),
            prefix + "ev_t": np.asarray(ts, np.int32),
            prefix + "ev_off": np.asarray(off, np.int64)}


def script_arrays(scripts, prefix=""):
    kinds, gaps, off = [], [], [0]
    sc = {k: [] for k in ("tail", "initial_grasped", "initial_contact",
                          "initial_level", "art_kind", "subtask")}
    dist = []
    for s in scripts:
        for st in s.steps:
            kinds.append(EVENT_KINDS.index(st.kind.value))
            gaps.append(st.gap)
        off.append(len(kinds))
        sc["tail"].append(s.tail)
        sc["initial_grasped"].append(int(s.initial_grasped))
        sc["initial_contact"].append(int(s.initial_contact))
        sc["initial_level"].append(LEVELS.index(s.initial_art_level))
        sc["art_kind"].append(ART.index(s.articulation_kind.value))
        sc["subtask"].append(KINDS.index(s.subtask_kind))
        dist.append(s.initial_dist_obj_goal)
    out = {prefix + "step_kind": np.asarray(kinds, np.uint8),
           prefix + "step_gap": np.asarray(gaps, np.int32),
           prefix + "step_off": np.asarray(off, np.int64),
           prefix + "initial_dist_obj_goal": np.asarray(dist, np.float64)}
    for k, v in sc.items():
        out[prefix + k] = np.asarray(v, np.int32)
    return out


def label_arrays(labels, prefix=""):
    return {prefix + "mode": np.asarray([ALL_MODES.index(l.mode_id) for l in labels], np.int32),
            prefix + "success_once": np.asarray([l.success_once for l in labels], np.uint8),
            prefix + "success_at_end": np.asarray([l.success_at_end for l in labels], np.uint8)}


# -- fuzz corpus ----------------------------------------------------------------

FUZZ_SEEDS = list(range(400)) + [1000003, 99999999, 100000000, 2 ** 32 + 5,
                                 2 ** 33 + 17, 123456789012]


def make_fuzz():
    th = T.Thresholds()
    out = {"seeds": np.asarray(FUZZ_SEEDS, np.int64)}
    for k, kind in enumerate(KINDS):
        pk, evs, labs, scripts, ids = Pack(), [], [], [], []
        for seed in FUZZ_SEEDS:
            s = synth.random_script(seed, kind)
            traj = synth.fuzz(seed, kind)
            ev = T.extract_events(traj, th)
            pk.add(traj)
            evs.append(ev.events)
            labs.append(T.classify(ev))
            scripts.append(s)
            ids.append(traj.header.episode_id)
        p = kind.value.lower() + "_"
        out.update(pk.arrays(p))
        out.update(events_arrays(evs, p))
        out.update(label_arrays(labs, p))
        out.update(script_arrays(scripts, p))
        out[p + "episode_id"] = np.asarray(ids)
    np.savez_compressed(os.path.join(OUT, "fuzz.npz"), **out)


def make_defining():
    th = T.Thresholds()
    pk, evs, labs, scripts, names, seeds = Pack(), [], [], [], [], []
    for mode, s in synth.defining_scripts().items():
        for seed in (7, 123):
            traj = synth.realize(s, seed=seed)
            ev = T.extract_events(traj, th)
            pk.add(traj)
            evs.append(ev.events)
            labs.append(T.classify(ev))
            scripts.append(s)
            names.append(mode)
            seeds.append(seed)
    out = pk.arrays()
    out.update(events_arrays(evs))
    out.update(label_arrays(labs))
    out.update(script_arrays(scripts))
    out["mode_name"] = np.asarray(names)
    out["seed"] = np.asarray(seeds, np.int64)
    np.savez_compressed(os.path.join(OUT, "defining.npz"), **out)


def _respaced(kind, steps, gap, tail, **kw):
    return synth.EventScript(subtask_kind=kind,
                             steps=[synth.ScriptStep(k, gap) for k in steps],
                             tail=tail, **kw)


def make_long():
    """200-step shapes of BASELINE C1/C2/C3 + long fuzz."""
    E = T.EventKind
    th = T.Thresholds()
    pk, evs, labs, scripts, seeds = Pack(), [], [], [], []
    items = []
    for i in range(4):  # C1 (tests/test_acceptance.py:264-271)
        items.append((_respaced(T.SubtaskKind.Pick, [E.Contact, E.Grasped, E.Success], 60, 19), i))
    for i in range(3):  # C2(ii)
        items.append((_respaced(T.SubtaskKind.Place, [E.ObjAtGoal, E.ReleasedAtGoal, E.Success],
                                60, 19, initial_grasped=True), i))
    for art in (T.ArticulationKind.Fridge, T.ArticulationKind.Drawer):  # C3
        items.append((_respaced(T.SubtaskKind.Open, [E.Contact, E.SlightlyOpened, E.Opened, E.Success],
                                45, 19, articulation_kind=art), 11))
        items.append((_respaced(T.SubtaskKind.Close, [E.Contact, E.SlightlyClosed, E.Closed, E.Success],
                                45, 19, articulation_kind=art, initial_art_level="high"), 12))
    for s, seed in items:
        traj = synth.realize(s, seed=seed)
        assert len(traj.records) == 200
        ev = T.extract_events(traj, th)
        pk.add(traj); evs.append(ev.events); labs.append(T.classify(ev))
        scripts.append(s); seeds.append(seed)
    out = pk.arrays()
    out.update(events_arrays(evs)); out.update(label_arrays(labs))
    out.update(script_arrays(scripts)); out["seed"] = np.asarray(seeds, np.int64)
    # random-action variant: fuzz with FuzzConfig(max_gap=64, max_tail=64)
    cfg = synth.FuzzConfig(max_gap=64, max_tail=64)
    for k, kind in enumerate(KINDS):
        pk, evs, labs, scripts = Pack(), [], [], []
        for seed in range(16):
            traj = synth.fuzz(seed, kind, cfg)
            ev = T.extract_events(traj, th)
            pk.add(traj); evs.append(ev.events); labs.append(T.classify(ev))
            scripts.append(synth.random_script(seed, kind, cfg))
        p = "g64_" + kind.value.lower() + "_"
        out.update(pk.arrays(p)); out.update(events_arrays(evs, p))
        out.update(label_arrays(labs, p)); out.update(script_arrays(scripts, p))
    np.savez_compressed(os.path.join(OUT, "long.npz"), **out)


# -- crafted record streams ------------------------------------------------------

def _palettes(kind, hdr, th, exact32):
    lim = th.collision_limit(kind)
    P = {
        "q": [0.0, 0.2, -0.2, 0.6, -0.6, 0.61, 0.1, 0.19999, -0.3],
        "qd": [0.0, 0.2, -0.2, 0.21, 0.1, 0.19999999, -0.35],
        "v": [0.0, 0.05, -0.05, 0.06, 0.02, 0.05000001],
        "om": [0.0, 0.05, -0.05, 0.051, 0.01],
        "der": [0.0, 0.05, 0.04, 0.3, 0.0500001],
        "tor": [0.0, 0.01, -0.01, 0.02, 0.005],
        "dist": [0.15, 0.1, 0.5, 0.14999, 0.1500001, 0.02],
        "force": [0.0, 1e-6, 1.1e-6, 1.2, 0.5e-6],
        "cum": [0.0, 10.0, lim * 0.5, lim, lim + 0.5, lim * 1.05, lim - 0.001],
    }
    if hdr.has_articulation:
        qmin, qmax = hdr.art_qmin, hdr.art_qmax
        span = qmax - qmin
        ofr = th.open_frac(hdr.articulation_kind)
        P["art"] = [qmin, qmax, ofr * span + qmin, th.close_frac * span + qmin,
                    th.slightly_open_frac * span + qmin, 0.3 * span + qmin,
                    (ofr * span + qmin) * (1 + 1e-7), 0.016, 1.2, 0.45, 0.05,
                    0.95 * span + qmin, 0.9 * span + qmin]
    else:
        P["art"] = [math.nan]
    if exact32:
        P = {k: [f32(v) for v in vs] for k, vs in P.items()}
    return P


def _crafted_traj(rng, kind, exact32, idx):
    art = T.ArticulationKind.NONE
    qmin = qmax = math.nan
    if kind in (T.SubtaskKind.Open, T.SubtaskKind.Close) or rng.random() < 0.1:
        art = rng.choice([T.ArticulationKind.Fridge, T.ArticulationKind.Drawer])
        qmin, qmax = (0.0, 1.6) if art == T.ArticulationKind.Fridge else (0.0, 0.5)
        if rng.random() < 0.2:
            qmin, qmax = -0.25, 1.25
    rest_arm = tuple(0.0 for _ in range(7))
    rest_tor = 0.0
    if rng.random() < 0.2:
        rest_arm = tuple(rng.choice([0.0, 0.1, -0.05, 0.3]) for _ in range(7))
        rest_tor = rng.choice([0.0, 0.005, -0.01])
    override = None
    if rng.random() < 0.15:
        d = T.Thresholds().to_dict()
        d[rng.choice(["coll_pick", "coll_place", "coll_artic"])] = rng.choice([1e-9, 10.0, 5000.5])
        d[rng.choice(["rest_radius", "goal_radius", "static_qd_arm"])] = rng.choice([0.3, 0.08, 0.21])
        override = T.Thresholds(**d)
    hdr = T.TrajectoryHeader(episode_id=f"crafted-{idx:05d}", subtask_kind=kind,
                             articulation_kind=art, art_qmin=qmin, art_qmax=qmax,
                             rest_arm=rest_arm, rest_tor=rest_tor,
                             thresholds_override=override)
    th = hdr.thresholds(T.Thresholds())
    P = _palettes(kind, hdr, th, exact32)
    n = rng.choice([0, 1, 2, 3, 5, 8, 13, 24, 40, 70])
    cur = None
    recs = []
    for t in range(n):
        def pick(key, prev):
            if prev is not None and rng.random() < 0.6:
                return prev
            return rng.choice(P[key])
        if cur is None or rng.random() < 0.5:
            # resample several channels at once -> multi-event steps
            c = cur or {}
            cur = dict(
                q=tuple(pick("q", (c.get("q") or (None,) * 7)[i]) for i in range(7)),
                qd=tuple(pick("qd", (c.get("qd") or (None,) * 7)[i]) for i in range(7)),
                tor=pick("tor", c.get("tor")), vx=pick("v", c.get("vx")),
                vy=pick("v", c.get("vy")), om=pick("om", c.get("om")),
                der=pick("der", c.get("der")), dist=pick("dist", c.get("dist")),
                force=pick("force", c.get("force")), cum=pick("cum", c.get("cum")),
                art=pick("art", c.get("art")),
                g=(not c.get("g", False)) if rng.random() < 0.3 else c.get("g", False))
            if rng.random() < 0.25:  # success posture
                cur.update(q=rest_arm if not exact32 else tuple(f32(v) for v in rest_arm),
                           qd=(0.0,) * 7, vx=0.0, vy=0.0, om=0.0, der=0.0,
                           tor=rest_tor if not exact32 else f32(rest_tor))
        rec = T.TimestepRecord(
            t=t, q_arm=cur["q"], qd_arm=cur["qd"], q_tor=cur["tor"],
            v_base_x=cur["vx"], v_base_y=cur["vy"], omega_base=cur["om"],
            dist_ee_rest=cur["der"],
            dist_obj_goal=cur["dist"] if kind == T.SubtaskKind.Place or rng.random() < 0.3 else math.nan,
            force_ee_target=cur["force"] if kind != T.SubtaskKind.Place else math.nan,
            cum_robot_force=cur["cum"], art_q=cur["art"], grasped=cur["g"])
        recs.append(rec)
    # error injection
    if recs and rng.random() < 0.12:
        r = rng.choice(recs)
        setattr(r, rng.choice(["force_ee_target", "dist_obj_goal", "art_q", "q_tor"]), math.nan)
        if rng.random() < 0.5:
            for r2 in recs:
                if rng.random() < 0.5:
                    r2.cum_robot_force = (f32 if exact32 else float)(th.collision_limit(kind) * 2)
    if recs and rng.random() < 0.05:
        recs[0].q_arm = (math.nan,) + tuple(recs[0].q_arm[1:])
    return T.Trajectory(header=hdr, records=recs)


def make_crafted():
    out = {}
    for exact32, tag in ((True, "f32_"), (False, "f64_")):
        rng = random.Random(20241217 + exact32)
        trajs = []
        for i in range(2400):
            trajs.append(_crafted_traj(rng, KINDS[i % 4], exact32, i))
        pk = Pack(np.float32 if exact32 else np.float64)
        evs, modes, so, se, err_type, err_msg, d0, succ_end = [], [], [], [], [], [], [], []
        over = np.zeros((len(trajs), len(TH_FIELDS)))
        has_over = np.zeros(len(trajs), np.uint8)
        for i, traj in enumerate(trajs):
            pk.add(traj)
            if traj.header.thresholds_override is not None:
                has_over[i] = 1
                over[i] = [getattr(traj.header.thresholds_override, f) for f in TH_FIELDS]
            try:
                ev = T.extract_events(traj, T.Thresholds())
                lab = T.classify(ev)
                evs.append(ev.events)
                modes.append(ALL_MODES.index(lab.mode_id))
                so.append(lab.success_once); se.append(lab.success_at_end)
                err_type.append(""); err_msg.append("")
                d0.append(ev.initial_dist_obj_goal if ev.initial_dist_obj_goal is not None else math.nan)
            except T.TrajlabError as e:
                evs.append([]); modes.append(-1); so.append(False); se.append(False)
                err_type.append(type(e).__name__); err_msg.append(str(e)); d0.append(math.nan)
            # per-record success predicate (predicates.py:75) where defined
            row = []
            th = traj.header.thresholds(T.Thresholds())
            for rec in traj.records:
                try:
                    row.append(1 if T.success_step(rec, traj.header, th) else 0)
                except T.TrajlabError:
                    row.append(2)
            succ_end.extend(row)
        a = pk.arrays(tag)
        a.update(events_arrays(evs, tag))
        a[tag + "mode"] = np.asarray(modes, np.int32)
        a[tag + "success_once"] = np.asarray(so, np.uint8)
        a[tag + "success_at_end"] = np.asarray(se, np.uint8)
        a[tag + "err_type"] = np.asarray(err_type)
        a[tag + "err_msg"] = np.asarray(err_msg)
        a[tag + "d0"] = np.asarray(d0)
        a[tag + "has_override"] = has_over
        a[tag + "override"] = over
        a[tag + "success_step"] = np.asarray(succ_end, np.uint8)
        out.update(a)
    out["threshold_fields"] = np.asarray(TH_FIELDS)
    np.savez_compressed(os.path.join(OUT, "crafted.npz"), **out)


# -- arbitrary scripts -> realize outcome ------------------------------------------

def make_scripts():
    rng = random.Random(77)
    cases = []
    for i in range(600):
        kind = KINDS[i % 4]
        alpha = list(EVENT_ORDER[kind])
        steps = []
        for _ in range(rng.choice([0, 1, 2, 3, 5, 8])):
            k = rng.choice(alpha) if rng.random() < 0.9 else rng.choice(list(T.EventKind))
            steps.append(synth.ScriptStep(k, rng.choice([0, 1, 1, 2, 3, 7])))
        if rng.random() < 0.02 and steps:
            steps[-1].gap = 0
        lvl_opts = {"Open": ["low", "slight", "open"], "Close": ["high", "slight", "closed"]}
        lvl = rng.choice(lvl_opts.get(kind.value, ["low"]))
        if rng.random() < 0.03:
            lvl = rng.choice(LEVELS)
        s = synth.EventScript(
            subtask_kind=kind, steps=steps, tail=rng.choice([-1, 0, 1, 3, 6]),
            initial_grasped=rng.random() < 0.4, initial_contact=rng.random() < 0.4,
            initial_dist_obj_goal=rng.choice([0.5, 0.1, 0.15, 0.151]),
            initial_art_level=lvl,
            articulation_kind=rng.choice([T.ArticulationKind.Fridge, T.ArticulationKind.Drawer]),
            episode_id=f"script-{i}")
        seed = rng.choice([0, 1, 17, 2 ** 32 + 1, 5555])
        th = None
        if rng.random() < 0.1:
            th = T.Thresholds(goal_radius=0.2, coll_pick=100.0)
        case = {"subtask": kind.value,
                "steps": [[st.kind.value, st.gap] for st in steps],
                "tail": s.tail, "initial_grasped": s.initial_grasped,
                "initial_contact": s.initial_contact,
                "initial_dist_obj_goal": s.initial_dist_obj_goal,
                "initial_art_level": s.initial_art_level,
                "articulation_kind": s.articulation_kind.value,
                "seed": seed, "thresholds": th.to_dict() if th else None}
        try:
            traj = synth.realize(s, seed=seed, th=th)
            case["n_records"] = len(traj.records)
            recs = traj.records
            # a compact digest of the realized records (bit patterns)
            h = 0
            vals = []
            for r in recs:
                vals.extend(r.q_arm); vals.extend(r.qd_arm)
                vals.extend(getattr(r, f) for f in SCALARS)
                vals.append(1.0 if r.grasped else 0.0)
            case["records_f32_hex"] = np.asarray(vals, np.float32).tobytes().hex()
            ev = T.extract_events(traj, T.Thresholds())
            case["events"] = [[e.kind.value, e.t] for e in ev.events]
            case["mode"] = T.classify(ev).mode_id
            case["error"] = None
        except T.TrajlabError as e:
            case["error"] = [type(e).__name__, str(e)]
        except KeyError as e:
            case["error"] = ["KeyError", str(e)]
        cases.append(case)
    with gzip.open(os.path.join(OUT, "scripts.json.gz"), "wt") as f:
        json.dump(cases, f, indent=0)


# -- classify cases ------------------------------------------------------------------

def make_classify():
    rng = random.Random(5)
    cases = []
    for i in range(3000):
        kind = KINDS[i % 4]
        alpha = list(EVENT_ORDER[kind])
        n = rng.choice([0, 1, 2, 3, 3, 4, 5, 6, 8, 12])
        kinds = [rng.choice(alpha) if rng.random() < 0.95 else rng.choice(list(T.EventKind))
                 for _ in range(n)]
        d0 = None
        if kind == T.SubtaskKind.Place or rng.random() < 0.1:
            d0 = rng.choice([0.1, 0.15, 0.5, f32(0.15), 0.14999999, None])
        rules = None
        rule_tag = None
        if rng.random() < 0.1:
            rule_tag = "drop_catch_all"
            rules = {kind: {"success": MODE_RULES[kind]["success"],
                            "failure": MODE_RULES[kind]["failure"][:-1]}}
        evl = T.EventList(subtask_kind=kind,
                          events=[T.Event(k, t + 1) for t, k in enumerate(kinds)],
                          initial_dist_obj_goal=d0)
        case = {"subtask": kind.value, "kinds": [k.value for k in kinds],
                "d0": d0, "rules": rule_tag}
        try:
            lab = T.classify(evl, rules=rules)
            case["result"] = [lab.mode_id, lab.success_once, lab.success_at_end]
        except (T.TrajlabError, TypeError) as e:
            case["error"] = [type(e).__name__, str(e)]
        cases.append(case)
    # the reference's own per-mode KATs (tests/test_modes.py:24-105)
    with gzip.open(os.path.join(OUT, "classify.json.gz"), "wt") as f:
        json.dump(cases, f, indent=0)


# -- filter cases -------------------------------------------------------------------

def make_filter(dup=False):
    """dup=True: episode_ids drawn WITH replacement (the same episode in
    several files), so manifest tie order is pinned too (pipeline.py:329)."""
    rng = random.Random(11 if dup else 9)
    cases = []
    for i in range(60 if dup else 100):
        n = rng.choice([0, 5, 50, 300, 1200])
        targets = [f"obj-{c}" for c in "ABCD"[:rng.choice([1, 2, 4])]]
        tasks = ["TidyHouse", "SetTable", "Custom"]
        labels = []
        ids = ([rng.randrange(max(1, n // 4)) for _ in range(n)] if dup
               else rng.sample(range(10 * n + 10), n))
        for j in range(n):
            kind = rng.choice(KINDS)
            mode = rng.choice(MODE_IDS[kind])
            labels.append(T.LabelRecord(
                episode_id=f"ep-{ids[j]:06d}" if rng.random() < 0.95 else f"x{ids[j]}",
                subtask=kind.value, mode_id=mode,
                success_once=mode.split(".")[1].startswith("s"),
                success_at_end=False, target_id=rng.choice(targets),
                task=rng.choice(tasks), split="Train", policy_tag="RL",
                source=f"/d/{j}"))
        allow = []
        for kind in rng.sample(KINDS, rng.choice([1, 2, 4])):
            nr = rng.choice([1, 2, 3])
            ws = {1: [[1.0]], 2: [[0.5, 0.5], [0.3, 0.7], [0.9, 0.1]],
                  3: [[0.2, 0.3, 0.5], [1 / 3, 1 / 3, 1 / 3], [0.6, 0.3, 0.1]]}[nr]
            w = rng.choice(ws)
            if abs(sum(w) - 1.0) > 1e-9:
                continue
            pool = list(MODE_IDS[kind])
            for r in range(nr):
                ms = frozenset(rng.sample(pool, rng.choice([1, 2, 3])))
                allow.append(T.AllowRule(kind.value, ms, w[r]))
        if not allow:
            allow = [T.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0)]
        spec = T.FilterSpec(allow=allow, quota_per_target=rng.choice([1, 3, 10, 50, 200, 1000]),
                            quota_key=rng.choice(["target_id", "target_id_task"]))
        man = T.filter_labels(labels, spec)
        md = json.loads(man.to_json())
        cases.append({"labels": [[l.episode_id, l.subtask, l.mode_id, l.target_id,
                                  l.task, l.source] for l in labels],
                      "spec": spec.to_dict(),
                      "selected": [e["episode_id"] for e in md["entries"]],
                      "counts": md["counts"], "shortfalls": md["shortfalls"],
                      "manifest_sha256": __import__("hashlib").sha256(
                          man.to_json().encode()).hexdigest()})
    name = "filter_dup.json.gz" if dup else "filter.json.gz"
    with gzip.open(os.path.join(OUT, name), "wt") as f:
        json.dump(cases, f)


def make_filter_dup():
    make_filter(dup=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["fuzz", "defining", "long", "crafted", "scripts",
                             "classify", "filter", "filter_dup"]
    for w in which:
        globals()["make_" + w]()
        print("wrote", w)
