"""The reference's unit-test cases (pkg/tests/test_events.py, test_predicates.py,
test_modes.py, test_synth.py, test_pipeline.py) run against this package's
drop-in API.  Every call below executes on the GPU."""
import json
import math

import pytest

pytestmark = pytest.mark.gpu
pytest.importorskip("torch")

import paper_2412_13211_b200 as T  # noqa: E402
from paper_2412_13211_b200.synth import EventScript, FuzzConfig, ScriptStep  # noqa: E402

E = T.EventKind
TH = T.Thresholds()
NAN = float("nan")
FRIDGE = dict(articulation_kind="Fridge", art_qmin=0.0, art_qmax=1.6)
DRAWER = dict(articulation_kind="Drawer", art_qmin=0.0, art_qmax=0.5)


def kinds_of(traj, th=TH):
    return [e.kind for e in T.extract_events(traj, th).events]


def rec(**kw):
    base = dict(t=0, q_arm=(0.0,) * 7, qd_arm=(0.0,) * 7, q_tor=0.0, v_base_x=0.0,
                v_base_y=0.0, omega_base=0.0, dist_ee_rest=0.0, dist_obj_goal=NAN,
                force_ee_target=0.0, cum_robot_force=0.0, art_q=NAN, grasped=False)
    base.update(kw)
    return T.TimestepRecord(**base)


def hdr(kind="Pick", **kw):
    return T.TrajectoryHeader(episode_id="e", subtask_kind=kind, **kw)


# -- events (reference test_events.py) ------------------------------------------

def test_defining_scripts_extract_their_events():
    scripts = T.defining_scripts()
    trajs = T.realize_many(list(scripts.values()), [7] * len(scripts))
    res = T.label_trajectories(trajs)
    for (mode_id, s), r in zip(scripts.items(), res):
        assert [e["kind"] for e in r.events] == [st.kind.value for st in s.steps], mode_id
        assert r.mode_id == mode_id


def test_event_times_follow_gaps():
    s = EventScript(T.SubtaskKind.Pick, [ScriptStep(E.Contact, 3), ScriptStep(E.Grasped, 2),
                                         ScriptStep(E.Success, 4)])
    assert [e.t for e in T.extract_events(T.realize(s, seed=1), TH).events] == [3, 5, 9]


def test_too_short_and_nan_channels_raise():
    traj = T.realize(T.defining_scripts()["pick.f6_mobility"], seed=0)
    with pytest.raises(T.TooShort):
        T.extract_events(T.Trajectory(traj.header, traj.records[:1]), TH)
    for r in traj.records:
        r.force_ee_target = NAN
    with pytest.raises(T.RequiredFieldNaN):
        T.extract_events(traj, TH)
    pl = T.realize(T.defining_scripts()["place.f7_didnt_grasp"], seed=0)
    for r in pl.records:
        r.dist_obj_goal = NAN
    with pytest.raises(T.RequiredFieldNaN):
        T.extract_events(pl, TH)


def test_excessive_collisions_is_strict_crossing_once():
    traj = T.realize(T.defining_scripts()["pick.f6_mobility"], seed=0)
    for r in traj.records:
        r.cum_robot_force = 5000.0
    assert kinds_of(traj) == []
    traj.records[-1].cum_robot_force = 5000.5
    assert kinds_of(traj) == [E.ExcessiveCollisions]
    f5 = T.realize(T.defining_scripts()["pick.f5_excessive_collisions"], seed=0)
    assert kinds_of(f5).count(E.ExcessiveCollisions) == 1


def test_place_d0_release_split_and_close_reopen():
    tr = T.realize(T.defining_scripts()["place.s2_drop_to_goal"], seed=5)
    out = T.extract_events(tr, TH)
    assert out.initial_dist_obj_goal == tr.records[0].dist_obj_goal > 0.15
    assert E.ReleasedAtGoal in kinds_of(T.realize(T.defining_scripts()["place.s1_place_in_goal"], seed=2))
    assert E.ReleasedOutsideGoal in kinds_of(T.realize(T.defining_scripts()["place.f8_didnt_reach_goal"], seed=2))
    k = kinds_of(T.realize(T.defining_scripts()["close.f6_opened_after_closed"], seed=3))
    assert k[-1] == E.Open and k.index(E.Closed) < k.index(E.Open)


def test_header_override_wins():
    traj = T.realize(T.defining_scripts()["pick.f7_cant_grasp"], seed=4)
    assert kinds_of(traj) == [E.Contact]
    traj.header.thresholds_override = T.Thresholds(coll_pick=1e-9)
    assert E.ExcessiveCollisions in kinds_of(traj)


# -- predicates (reference test_predicates.py) -----------------------------------

def test_j_max_and_static():
    assert T.j_max((1.0, -2.0), (0.0, 0.0)) == 2.0
    assert T.j_max((), ()) == 0.0
    with pytest.raises(ValueError):
        T.j_max((1.0,), (1.0, 2.0))
    assert T.is_static(rec(qd_arm=(0.2,) * 7, v_base_x=0.05, v_base_y=-0.05, omega_base=0.05), TH)
    assert not T.is_static(rec(qd_arm=(0.0,) * 6 + (0.21,)), TH)
    assert not T.is_static(rec(v_base_x=-0.06), TH)
    assert not T.is_static(rec(omega_base=0.051), TH)


def test_articulation_predicates():
    hf, hd, hc = hdr("Open", **FRIDGE), hdr("Open", **DRAWER), hdr("Close", **FRIDGE)
    assert T.is_open(0.75 * 1.6, hf, TH) and not T.is_open(0.75 * 1.6 - 1e-6, hf, TH)
    assert T.is_open(0.9 * 0.5, hd, TH) and not T.is_open(0.8 * 0.5, hd, TH)
    assert T.is_closed(0.01 * 1.6, hc, TH) and not T.is_closed(0.01 * 1.6 + 1e-6, hc, TH)
    assert T.slightly_opened(0.1 * 1.6, hc, TH) and not T.slightly_opened(0.1 * 1.6 - 1e-6, hc, TH)
    assert T.slightly_closed(1.6 - 0.05 * 1.6 - 1e-6, 1.6, hc, TH)
    assert not T.slightly_closed(1.6 - 0.05 * 1.6, 1.6, hc, TH)
    with pytest.raises(T.MissingArticulation):
        T.is_open(1.0, hdr("Open"), TH)
    with pytest.raises(T.RequiredFieldNaN):
        T.is_open(NAN, hf, TH)


def test_f32_boundary_kats():
    """f32-widened values against f64 thresholds."""
    f32 = T.f32
    assert not T.is_static(rec(qd_arm=(f32(0.2),) * 7), TH)
    assert not T.success_step(rec(grasped=True, dist_ee_rest=f32(0.05)), hdr("Pick"), TH)
    assert not T.is_open(f32(0.45), hdr("Open", **DRAWER), TH)
    assert T.is_open(f32(1.2), hdr("Open", **FRIDGE), TH)
    assert not T.is_open(1.2, hdr("Open", **FRIDGE), TH)
    assert not T.is_closed(f32(0.016), hdr("Close", **FRIDGE), TH)
    assert T.is_closed(0.016, hdr("Close", **FRIDGE), TH)


def test_success_and_failure_steps():
    h = hdr("Pick")
    assert T.success_step(rec(grasped=True), h, TH)
    assert not T.success_step(rec(grasped=False), h, TH)
    assert not T.success_step(rec(grasped=True, dist_ee_rest=0.051), h, TH)
    assert T.success_step(rec(grasped=True, q_arm=(0.6,) * 7, q_tor=0.5), h, TH)
    assert not T.success_step(rec(grasped=True, q_arm=(0.61,) + (0.0,) * 6), h, TH)
    assert not T.success_step(rec(grasped=True, cum_robot_force=5000.1), h, TH)
    assert T.success_step(rec(grasped=True, cum_robot_force=5000.0), h, TH)
    hp = hdr("Place")
    assert T.success_step(rec(dist_obj_goal=0.15), hp, TH)
    assert not T.success_step(rec(dist_obj_goal=0.151), hp, TH)
    assert not T.success_step(rec(dist_obj_goal=0.1, grasped=True), hp, TH)
    assert not T.success_step(rec(dist_obj_goal=0.1, q_tor=0.011), hp, TH)
    with pytest.raises(T.RequiredFieldNaN):
        T.success_step(rec(dist_obj_goal=NAN), hp, TH)
    assert T.success_step(rec(art_q=1.3), hdr("Open", **FRIDGE), TH)
    assert not T.success_step(rec(art_q=1.1), hdr("Open", **FRIDGE), TH)
    assert T.success_step(rec(art_q=0.0), hdr("Close", **FRIDGE), TH)
    assert not T.failure_step(rec(cum_robot_force=5000.0), h, TH)
    assert T.failure_step(rec(cum_robot_force=5000.001), h, TH)
    assert T.failure_step(rec(cum_robot_force=7500.5), hp, TH)
    assert T.success_step(rec(grasped=True, dist_ee_rest=0.3), h, T.Thresholds(rest_radius=0.5))


# -- modes (reference test_modes.py) ----------------------------------------------

def _ev(kind, ks, d0=None):
    return T.EventList(kind, [T.Event(k, t) for t, k in enumerate(ks, 1)], d0)


def test_mode_inventory_flags_and_coverage_error():
    assert [len(T.MODE_IDS[k]) for k in T.SubtaskKind] == [9, 12, 9, 9]
    lbl = T.classify(_ev(T.SubtaskKind.Pick, [E.Contact, E.Grasped, E.Success]))
    assert lbl.mode_id == "pick.s1_straightforward" and lbl.success_at_end
    lbl = T.classify(_ev(T.SubtaskKind.Pick, [E.Contact, E.Grasped, E.Success, E.Dropped]))
    assert lbl.success_once and not lbl.success_at_end
    assert T.classify(_ev(T.SubtaskKind.Place, [E.Success], d0=0.1)).mode_id == "place.s1_place_in_goal"
    broken = {T.SubtaskKind.Pick: {"success": T.MODE_RULES[T.SubtaskKind.Pick]["success"],
                                   "failure": T.MODE_RULES[T.SubtaskKind.Pick]["failure"][:-1]}}
    with pytest.raises(T.ModeCoverageError) as ei:
        T.classify(_ev(T.SubtaskKind.Pick, [E.Contact, E.Grasped]), rules=broken)
    assert str(ei.value) == "no failure mode matched ['Contact', 'Grasped']"
    assert T.group(T.classify(_ev(T.SubtaskKind.Pick, [])), T.PICK_COARSE) == "F-Other"
    assert T.last_index(_ev(T.SubtaskKind.Pick, [E.Contact, E.Grasped, E.Contact]), E.Contact) == 2


def test_classify_custom_rule_tables_vs_reference():
    """classify(events, rules) with arbitrary (mode_id, predicate) tables:
    relabelled / reordered / repeated builtin predicates (device runs) mixed
    with host callables, dropped catch-alls, empty and foreign tables --
    against the reference's results (tests/golden/make_rules_golden.py)."""
    import gzip
    import os
    import sys
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from rule_recipes import build_table
    with gzip.open(os.path.join(here, "rules.json.gz"), "rt") as f:
        cases = json.load(f)
    for c in cases:
        kind = T.SubtaskKind(c["subtask"])
        ev = _ev(kind, [E(k) for k in c["kinds"]], c["d0"])
        table = build_table(c["recipe"], T.MODE_RULES, T.SubtaskKind, T.EventKind)
        if "error" in c:
            with pytest.raises(Exception) as ei:
                T.classify(ev, rules=table)
            assert type(ei.value).__name__ == c["error"][0], c
            if c["error"][0] != "KeyError":
                assert str(ei.value) == c["error"][1], c
        else:
            lab = T.classify(ev, rules=table)
            assert [lab.mode_id, lab.success_once, lab.success_at_end] == c["result"], c


# -- synth (reference test_synth.py) ---------------------------------------------

def test_realize_is_deterministic_and_valid():
    s = T.defining_scripts()["pick.s2_winding"]
    assert T.realize(s, seed=9).records == T.realize(s, seed=9).records
    for mode_id, s in T.defining_scripts().items():
        assert not [f for f in T.validate(T.realize(s, seed=3)) if f.is_error], mode_id


@pytest.mark.parametrize("steps,kind,lvl", [
    ([ScriptStep(E.Dropped, 2)], "Pick", "low"),
    ([ScriptStep(E.Grasped, 2)], "Pick", "low"),
    ([ScriptStep(E.Success, 2)], "Pick", "low"),
    ([ScriptStep(E.Closed, 2)], "Close", "high"),
    ([ScriptStep(E.ObjAtGoal, 2)], "Pick", "low"),
    ([ScriptStep(E.Contact, 0)], "Pick", "low")])
def test_infeasible_scripts_raise(steps, kind, lvl):
    with pytest.raises(T.InfeasibleScript):
        T.realize(EventScript(T.SubtaskKind(kind), steps, initial_art_level=lvl), seed=0)


def test_fuzz_determinism_density_and_feasibility():
    a, b = T.fuzz(1, T.SubtaskKind.Place), T.fuzz(1, T.SubtaskKind.Place)
    assert a.header == b.header and a.records == b.records
    for kind in T.SubtaskKind:
        for tr in T.fuzz_many(range(20), kind, FuzzConfig(edge_density=0.0)):
            assert T.extract_events(tr, TH).events == []
        for s in range(50):
            T.realize(T.random_script(s, kind), seed=s)
    ids = {tr.header.episode_id for tr in T.fuzz_many(range(50), T.SubtaskKind.Open)}
    assert len(ids) == 50


def test_script_from_dict():
    s = EventScript.from_dict({"subtask": "Open", "events": [{"kind": "Contact", "gap": 1},
                                                             {"kind": "SlightlyOpened", "gap": 3}],
                               "articulation_kind": "Drawer", "initial_art_level": "low"})
    assert kinds_of(T.realize(s, seed=2)) == [E.Contact, E.SlightlyOpened]


# -- pipeline (reference test_pipeline.py) ----------------------------------------

def test_label_trajectory_and_batch(tmp_path):
    r = T.label_trajectory(T.realize(T.defining_scripts()["pick.s1_straightforward"], seed=1), TH,
                           source="here")
    assert (r.mode_id, r.subtask, r.success_once, r.success_at_end, r.source) == \
        ("pick.s1_straightforward", "Pick", True, True, "here")
    assert T.LabelRecord.from_dict(json.loads(r.to_json())) == r
    paths = []
    for seed in (5, 1, 9, 3):
        tr = T.fuzz(seed, T.SubtaskKind.Pick)
        p = tmp_path / f"{tr.header.episode_id}.trjl"
        T.write_binary_file(tr, p)
        paths.append(p)
    bad = tmp_path / "bad.trjl"
    bad.write_bytes(paths[0].read_bytes()[:30])
    r1 = T.label_batch(paths + [bad], TH, workers=1)
    r2 = T.label_batch(list(reversed(paths)) + [bad], TH, workers=4)
    assert [x.to_json() for x in r1.labels] == [x.to_json() for x in r2.labels]
    assert [x.episode_id for x in r1.labels] == sorted(x.episode_id for x in r1.labels)
    assert len(r1.errors) == 1 and "bad.trjl" in r1.errors[0]["source"]
    tr = T.fuzz(5, T.SubtaskKind.Open)
    b, t = tmp_path / "a.trjl", tmp_path / "a.jsonl"
    T.write_binary_file(tr, b)
    T.write_text_file(tr, t)
    assert T.label_file(b).mode_id == T.label_file(t).mode_id


def _lab(i, mode="pick.s1_straightforward", sub="Pick", target="obj-A"):
    return T.LabelRecord(episode_id=f"ep-{i:05d}", subtask=sub, mode_id=mode,
                         success_once=True, success_at_end=False, target_id=target)


def test_filter_semantics():
    m = T.filter_labels([_lab(i) for i in range(1200)] + [_lab(2000 + i, "pick.f8_drop") for i in range(800)],
                        T.FilterSpec([T.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0)]))
    assert [e.episode_id for e in m.entries] == [f"ep-{i:05d}" for i in range(1000)]
    spec = T.FilterSpec([T.AllowRule("Place", frozenset({"place.s1_place_in_goal"}), 0.5),
                         T.AllowRule("Place", frozenset({"place.s2_drop_to_goal"}), 0.5)],
                        quota_per_target=500)
    m = T.filter_labels([_lab(i, "place.s1_place_in_goal", "Place") for i in range(400)] +
                        [_lab(1000 + i, "place.s2_drop_to_goal", "Place") for i in range(400)], spec)
    assert sum(e.mode_id == "place.s1_place_in_goal" for e in m.entries) == 250
    m = T.filter_labels([_lab(i) for i in range(300)],
                        T.FilterSpec([T.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0)]))
    assert m.shortfalls[0]["shortfall"] == 700
    m = T.filter_labels([_lab(i, target="A") for i in range(30)] + [_lab(100 + i, target="B") for i in range(5)],
                        T.FilterSpec([T.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0)],
                                     quota_per_target=10))
    assert len(m.entries) == 15 and len(m.shortfalls) == 1


@pytest.mark.parametrize("name", ["filter", "filter_dup"])
def test_filter_manifest_bytes_vs_reference(name):
    """filter_labels over the reference fixtures: the manifest JSON is
    byte-identical (sha256) to the reference's, including the entry order
    among repeated episode_ids (filter_dup: ids drawn with replacement;
    reference pipeline.py:299-329 emits pool by pool, then stable-sorts)."""
    import hashlib
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from golden_data import js
    for case in js(name):
        labels = [T.LabelRecord(episode_id=eid, subtask=sub, mode_id=mode,
                                success_once=mode.split(".")[1].startswith("s"),
                                success_at_end=False, target_id=tgt, task=task,
                                split="Train", policy_tag="RL", source=src)
                  for eid, sub, mode, tgt, task, src in case["labels"]]
        man = T.filter_labels(labels, T.FilterSpec.from_dict(case["spec"]))
        assert [e.episode_id for e in man.entries] == case["selected"]
        assert hashlib.sha256(man.to_json().encode()).hexdigest() == case["manifest_sha256"]


def test_c5_device_filter_matches_host_filter():
    """C5 shape at small scale: device bucket encoding + selection + counts
    == filter_labels over the equivalent LabelRecords (host buckets, pinned
    to the reference's filter fixtures)."""
    import numpy as np
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200 import _lib as L, dist as D
    from paper_2412_13211_b200.modes import MODE_LIST
    from paper_2412_13211_b200.model import SUBTASK_ORDER
    spec = P.FilterSpec(allow=[
        P.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0),
        P.AllowRule("Place", frozenset({"place.s1_place_in_goal"}), 0.5),
        P.AllowRule("Place", frozenset({"place.s2_drop_to_goal"}), 0.5),
        P.AllowRule("Open", frozenset({"open.s1_open"}), 1.0),
        P.AllowRule("Close", frozenset({"close.s1_close"}), 1.0)], quota_per_target=25)
    n = 1500
    labels, man, names = D.fuzz_label_filter_sharded(n, spec, n_targets=9)
    lab = labels.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)
    # the four side-stream batches == plain per-subtask fuzz batches
    import torch
    from paper_2412_13211_b200 import core
    cs = core.synth_csets(P.Thresholds()).to_device(torch.device("cuda"))
    for s in range(4):
        ref = core.fuzz_batch(np.arange(n), s, P.FuzzConfig(), P.Thresholds(), cs).labels[:n]
        assert np.array_equal(ref.cpu().numpy(), labels[s * n:(s + 1) * n].cpu().numpy()), s
    recs = []
    for s, kind in enumerate(SUBTASK_ORDER):
        for seed in range(n):
            r = lab[s * n + seed]
            assert r["status"] == 0
            recs.append(P.LabelRecord(
                episode_id=f"fuzz-{kind.value.lower()}-{seed:08d}", subtask=kind.value,
                mode_id=MODE_LIST[r["mode"]], success_once=bool(r["flags"] & 1),
                success_at_end=bool(r["flags"] & 2), target_id=f"{seed % 9:03d}"))
    want = P.filter_labels(recs, spec)
    got_ids = sorted(recs[i].episode_id for i in man.selected_rows())
    assert got_ids == [e.episode_id for e in want.entries]
    assert man.counts == want.counts
    assert man.shortfalls == want.shortfalls


def test_nccl_exchange_entry_points_single_rank():
    """tl_allgather_labels / tl_allreduce_counts through a 1-rank NCCL
    communicator made with the process's NCCL (torch's bundled copy): the
    C-ABI plumbing of the multi-GPU exchange step (symbol resolution, byte
    counts, dtypes, stream)."""
    import ctypes
    import glob
    import os
    import numpy as np
    import torch
    from paper_2412_13211_b200 import _lib as L
    base = os.path.dirname(torch.__file__)
    paths = glob.glob(os.path.join(base, "..", "nvidia", "nccl", "lib", "libnccl.so*"))
    nccl = ctypes.CDLL(paths[0] if paths else "libnccl.so.2", mode=ctypes.RTLD_GLOBAL)

    class UniqueId(ctypes.Structure):
        _fields_ = [("internal", ctypes.c_char * 128)]
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(ctypes.byref(uid)) == 0
    comm = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert nccl.ncclCommInitRank(ctypes.byref(comm), 1, uid, 0) == 0
    try:
        n = 777
        lab = torch.randint(0, 255, (n, 24), dtype=torch.uint8, device="cuda")
        out = torch.zeros_like(lab)
        L.check(L.lib().tl_allgather_labels(comm, L.ptr(lab), n, L.ptr(out), L.stream_ptr()),
                "allgather")
        counts = torch.arange(42 * 3, dtype=torch.int64, device="cuda")
        want = counts.clone()
        L.check(L.lib().tl_allreduce_counts(comm, L.ptr(counts), counts.numel(), L.stream_ptr()),
                "allreduce")
        torch.cuda.synchronize()
        assert torch.equal(out, lab) and torch.equal(counts, want)
    finally:
        nccl.ncclCommDestroy(comm)


def test_c_abi_rejects_invalid_arguments():
    """Every entry point validates its arguments and returns TL_E_INVALID
    (no launch, no crash) for null required pointers / bad sizes."""
    import ctypes
    from paper_2412_13211_b200 import _lib as L
    lib = L.lib()
    E = L.E_INVALID
    th = L.Thresholds_c()
    cfg = L.FuzzCfg_c(8, 4, 5, 0, 1.0, 0.5)
    bad_cfg = L.FuzzCfg_c(8, 0, 5, 0, 1.0, 0.5)   # max_gap < 1
    rec = L.Records_c(None, None, None, None, 0, 0, 7)
    bad_rec = L.Records_c(None, None, None, None, 0, 0, 99)  # dof > 16
    nul = None
    assert lib.tl_label_records(None, 1, nul, nul, 1, None, nul, nul, nul, nul) == E
    assert lib.tl_label_records(ctypes.byref(bad_rec), 1, nul, nul, 1, None, nul, nul, nul, nul) == E
    assert lib.tl_fuzz(nul, 4, 0, ctypes.byref(bad_cfg), ctypes.byref(th), nul, None,
                       ctypes.byref(rec), 64, nul, nul, nul, nul, nul, nul, nul) == E
    assert lib.tl_fuzz(nul, 4, 7, ctypes.byref(cfg), ctypes.byref(th), nul, None,
                       ctypes.byref(rec), 64, nul, nul, nul, nul, nul, nul, nul) == E
    assert lib.tl_fuzz_ev(nul, 4, 0, ctypes.byref(cfg), ctypes.byref(th), nul, None,
                          ctypes.byref(rec), 64, nul, nul, nul, nul, nul, nul, nul, nul, 0,
                          nul, nul) == E
    assert lib.tl_realize(nul, nul, nul, 4, ctypes.byref(th), nul, None, ctypes.byref(rec),
                          nul, nul, nul, nul) == E
    assert lib.tl_scan_emit_events(nul, nul, nul, nul, 4, nul, nul, nul, nul, nul) == E
    assert lib.tl_filter_select(nul, 4, 1, 1, nul, nul, 1, nul, nul, nul, nul) == E
    assert lib.tl_env_reset(nul, 4, 7, nul, ctypes.byref(th), nul, nul, 0, nul, nul, nul) == E
    assert lib.tl_env_step(nul, 4, 7, nul, 1, nul, 0, nul, nul, nul) == E
    assert lib.tl_env_labels(nul, 4, None, nul, nul, nul) == E
    assert lib.tl_env_script_actions(nul, nul, nul, 4, 0, 1, nul, nul) == E
    assert lib.tl_group_mode_counts(nul, nul, 4, 1, nul, nul) == E
    assert lib.tl_chain_progress(nul, nul, 4, 99, nul, nul) == E
    assert lib.tl_filter_buckets(nul, nul, 4, nul, nul, nul, 9, nul, nul) == E
    assert lib.tl_allgather_labels(nul, nul, 4, nul, nul) == E
    assert lib.tl_allreduce_counts(nul, nul, 4, nul) == E
    assert lib.tl_mode_histogram(nul, 4, nul, nul) == E
    assert lib.tl_status_name(E).decode() != ""


def test_label_batch_and_json_match_reference(tmp_path):
    """label_batch over TRJL files (GPU labelling) == the reference's
    BatchResult: canonical LabelRecord JSON, per-file errors, mode counts
    (tests/golden/labels.json.gz, make_labels_golden.py)."""
    import io
    import json
    import os
    import paper_2412_13211_b200 as P
    from golden_data import js
    g = js("labels")
    paths = []
    for name, hx in g["files"].items():
        pth = tmp_path / name
        pth.write_bytes(bytes.fromhex(hx))
        paths.append(str(pth))
    res = P.label_batch(paths)
    got = []
    for r in res.labels:
        d = r.to_dict()
        d["source"] = os.path.relpath(d["source"], str(tmp_path))
        got.append(json.dumps(d, sort_keys=True))
    assert got == g["labels"]
    assert [{"source": os.path.relpath(e["source"], str(tmp_path)), "error": e["error"]}
            for e in res.errors] == g["errors"]
    assert res.mode_counts == g["mode_counts"]
    for name, want in g["per_file"].items():
        data = bytes.fromhex(g["files"][name])
        try:
            out = P.label_trajectory(P.read_binary(io.BytesIO(data))).to_json()
        except Exception as e:  # noqa: BLE001
            out = f"{type(e).__name__}: {e}"
        assert out == want, name
