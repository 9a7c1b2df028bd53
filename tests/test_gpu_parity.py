"""GPU parity: libtrajlab_b200.so (sm_100a) vs the reference's golden
fixtures and vs the CPU oracle.  Integer / event / mode / record outputs
must be bit-exact.  Runs on a B200 (-m gpu)."""
import math

import numpy as np
import pytest

from golden_data import (DOF, SUBTASKS, Corpus, fuzz_corpus, js, npz,
                         same_bits_f32)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def C():
    from paper_2412_13211_b200 import core
    return core


@pytest.fixture(scope="module")
def TH():
    from paper_2412_13211_b200.thresholds import Thresholds
    return Thresholds


def corpus_batch(C, TH, c: Corpus, dtype=np.float32, overrides=None, align=False):
    """fixture corpus -> RecordBatch + csets.  align=False copies the planes
    verbatim (packed episodes: the one-record-per-lane label path); align=True
    re-packs every episode at a 4-record boundary (the 128-bit label path)."""
    dev = torch.device("cuda")
    nrec = np.diff(c.rec_off).astype(np.int64)
    if align:
        slot = (nrec + 3) & ~3
        starts = np.concatenate([[0], np.cumsum(slot)[:-1]]).astype(np.int64)
        hp = np.full((c.planes.shape[0], max(int(slot.sum()), 4)), np.nan, dtype)
        hg = np.zeros(hp.shape[1], np.uint8)
        for i in range(c.n):
            a, b = c.rec_off[i], c.rec_off[i + 1]
            hp[:, starts[i]:starts[i] + b - a] = c.planes[:, a:b]
            hg[starts[i]:starts[i] + b - a] = c.grasped[a:b]
        planes = torch.from_numpy(hp).to(dev)
        g = torch.from_numpy(hg).to(dev)
        rs = torch.from_numpy(starts).to(dev)
    else:
        planes = torch.from_numpy(np.ascontiguousarray(c.planes.astype(dtype))).to(dev)
        if planes.shape[1] == 0:
            planes = torch.zeros((planes.shape[0], 1), dtype=planes.dtype, device=dev)
        g = torch.from_numpy(np.ascontiguousarray(c.grasped) if len(c.grasped) else np.zeros(1, np.uint8)).to(dev)
        rs = torch.from_numpy(c.rec_off[:-1].copy()).to(dev)
    nr = torch.from_numpy(nrec.astype(np.int32)).to(dev)
    rb = C.RecordBatch(planes, g, rs, nr, DOF)
    tab = C.CsetTable()
    env = np.zeros(c.n, np.int32)
    for i in range(c.n):
        th = TH()
        if overrides is not None and overrides[i] is not None:
            th = TH(**overrides[i])
        env[i] = tab.add(int(c.subtask[i]), int(c.art_kind[i]), float(c.art_qmin[i]),
                         float(c.art_qmax[i]), DOF, list(c.rest_arm[i]),
                         float(c.rest_tor[i]), th)
    return rb, torch.from_numpy(env).to(dev), tab.to_device(dev), len(tab)


def check_labels(res, c: Corpus, err_type=None):
    lab = res.labels_np()
    ev_off = res.ev_off.cpu().numpy()
    ek = res.ev_kind.cpu().numpy()
    et = res.ev_t.cpu().numpy()
    from paper_2412_13211_b200 import _lib as L
    for i in range(c.n):
        if err_type is not None and err_type[i]:
            assert lab["status"][i] != 0, i
            name = L.lib().tl_status_name(int(lab["status"][i])).decode()
            assert name == err_type[i], (i, name, err_type[i])
            continue
        assert lab["status"][i] == 0, (i, lab["status"][i])
        want_k, want_t = c.events(i)
        a, b = ev_off[i], ev_off[i + 1]
        assert list(ek[a:b]) == want_k, i
        assert list(et[a:b]) == want_t, i
        assert lab["mode"][i] == c.mode[i], i
        assert bool(lab["flags"][i] & 1) == bool(c.success_once[i])
        assert bool(lab["flags"][i] & 2) == bool(c.success_at_end[i])
        assert lab["n_events"][i] == len(want_k)


@pytest.mark.parametrize("align", [False, True])
@pytest.mark.parametrize("kind", range(4))
def test_label_fuzz_fixtures(C, TH, kind, align):
    c = fuzz_corpus(kind)
    rb, env, cs, n = corpus_batch(C, TH, c, align=align)
    res = C.label_records(rb, env, cs, n)
    check_labels(res, c)


@pytest.mark.parametrize("align", [False, True])
def test_label_defining_and_long(C, TH, align):
    for c in (Corpus(npz("defining")), Corpus(npz("long"))):
        rb, env, cs, n = corpus_batch(C, TH, c, align=align)
        check_labels(C.label_records(rb, env, cs, n), c)


@pytest.mark.parametrize("align", [False, True])
@pytest.mark.parametrize("tag,dtype", [("f32_", np.float32), ("f64_", np.float64)])
def test_label_crafted(C, TH, tag, dtype, align):
    d = npz("crafted")
    c = Corpus(d, tag)
    fields = list(d["threshold_fields"])
    ov = [dict(zip(fields, map(float, d[tag + "override"][i]))) if d[tag + "has_override"][i] else None
          for i in range(c.n)]
    rb, env, cs, n = corpus_batch(C, TH, c, dtype, ov, align=align)
    res = C.label_records(rb, env, cs, n, want_success=True)
    check_labels(res, c, d[tag + "err_type"])
    # per-record success_step (predicates.py:75-94), incl. raising records
    got = res.step_success.cpu().numpy()
    if align:
        rs = rb.rec_start.cpu().numpy()
        got = np.concatenate([got[rs[i]:rs[i] + c.rec_off[i + 1] - c.rec_off[i]] for i in range(c.n)])
    assert np.array_equal(got[:c.rec_off[-1]], d[tag + "success_step"])


@pytest.mark.parametrize("kind", range(4))
def test_label_kernel_matches_fused_synth_labels(C, TH, kind):
    """tl_label_records over fuzz output (4-record aligned slots, 128-bit
    path) == the labels and step masks tl_fuzz folded while generating."""
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 4000
    sb = C.fuzz_batch(np.arange(n) + 31337, kind, cfg, TH(), cs, want_scripts=True)
    from paper_2412_13211_b200 import _lib as L
    art = sb.scripts.cpu().numpy().reshape(-1).view(L.SCRIPT_DTYPE)["art_kind"]
    env = torch.from_numpy((3 * kind + art).astype(np.int32)).to("cuda")
    lab_kind = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    res = C.label_records(sb.records, env, cs, 12, want_events=False)
    a = sb.labels.cpu().numpy()
    b = res.labels.cpu().numpy()
    assert np.all(lab_kind["status"] == 0)
    assert np.array_equal(a, b)
    rs = sb.records.rec_start.cpu().numpy()
    nr = sb.records.n_rec.cpu().numpy()
    ma, mb = sb.step_mask.cpu().numpy(), res.step_mask.cpu().numpy()
    for e in range(0, n, 7):
        assert np.array_equal(ma[rs[e]:rs[e] + nr[e]], mb[rs[e]:rs[e] + nr[e]]), e


def _fuzz_records(sb, e):
    rs = int(sb.records.rec_start[e].item())
    n = int(sb.records.n_rec[e].item())
    return sb.records.planes[:, rs:rs + n].cpu().numpy(), sb.records.grasped[rs:rs + n].cpu().numpy()


@pytest.mark.parametrize("kind", range(4))
def test_fuzz_generation_matches_reference(C, TH, kind):
    from paper_2412_13211_b200.synth import FuzzConfig
    c = fuzz_corpus(kind)
    seeds = npz("fuzz")["seeds"]
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    sb = C.fuzz_batch(seeds, kind, FuzzConfig(), TH(), cs, want_scripts=True)
    torch.cuda.synchronize()
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    scripts = c.scripts()
    sk = sb.script_kind.cpu().numpy()
    sg = sb.script_gap.cpu().numpy()
    for i in range(len(seeds)):
        planes, g = _fuzz_records(sb, i)
        wp, wg = c.records_np(i)
        assert same_bits_f32(planes, wp), (kind, int(seeds[i]))
        assert np.array_equal(g, wg)
        assert lab["status"][i] == 0
        assert lab["mode"][i] == c.mode[i]
        ns = len(scripts[i]["kinds"])
        off = i * 12
        assert list(sk[off:off + ns]) == list(scripts[i]["kinds"])
        assert list(sg[off:off + ns]) == list(scripts[i]["gaps"])


def test_fuzz_g64_matches_reference(C, TH):
    from paper_2412_13211_b200.synth import FuzzConfig
    d = npz("long")
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    for k, name in enumerate(("pick", "place", "open", "close")):
        c = Corpus(d, "g64_" + name + "_")
        sb = C.fuzz_batch(np.arange(16), k, cfg, TH(), cs)
        for i in range(16):
            planes, _ = _fuzz_records(sb, i)
            assert same_bits_f32(planes, c.records_np(i)[0]), (name, i)


def _scripts_np(C, scripts, seeds):
    from paper_2412_13211_b200 import _lib as L
    arr = np.zeros(len(scripts), L.SCRIPT_DTYPE)
    kinds, gaps = [], []
    for i, sc in enumerate(scripts):
        arr[i]["step_off"] = len(kinds)
        arr[i]["seed"] = int(seeds[i])
        arr[i]["n_steps"] = len(sc["kinds"])
        arr[i]["tail"] = sc["tail"]
        arr[i]["subtask"] = sc["subtask"]
        arr[i]["art_kind"] = sc["art_kind"]
        arr[i]["initial_level"] = sc["initial_level"]
        arr[i]["initial_grasped"] = sc["initial_grasped"]
        arr[i]["initial_contact"] = sc["initial_contact"]
        arr[i]["arm_dof"] = 7
        arr[i]["initial_dist_obj_goal"] = sc["initial_dist_obj_goal"]
        kinds.extend(int(k) for k in sc["kinds"])
        gaps.extend(int(g) for g in sc["gaps"])
    return arr, np.asarray(kinds, np.uint8), np.asarray(gaps, np.int32)


def test_realize_defining_and_long(C, TH):
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    for d in (npz("defining"), npz("long")):
        c = Corpus(d)
        arr, k, g = _scripts_np(C, c.scripts(), d["seed"])
        sb = C.realize_batch(arr, k, g, TH(), cs)
        lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
        planes = sb.records.planes.cpu().numpy()
        rs = sb.records.rec_start.cpu().numpy()
        for i in range(c.n):
            a, b = c.rec_off[i], c.rec_off[i + 1]
            assert rs[i] % 4 == 0
            assert same_bits_f32(planes[:, rs[i]:rs[i] + b - a], c.planes[:, a:b]), i
            assert lab["status"][i] == 0 and lab["mode"][i] == c.mode[i], i


def test_realize_arbitrary_scripts(C, TH):
    """scripts.json: feasible scripts realize bit-exactly, infeasible ones
    report the reference's InfeasibleScript raise site and message."""
    from paper_2412_13211_b200 import errors as ER
    from golden_data import LEVELS, ART
    EV = ("Contact", "Grasped", "Dropped", "ObjAtGoal", "ReleasedAtGoal",
          "ReleasedOutsideGoal", "ObjLeftGoal", "Opened", "SlightlyOpened", "Closed",
          "SlightlyClosed", "Open", "Success", "ExcessiveCollisions")
    cases = js("scripts")
    groups = {}
    for case in cases:
        key = json_key = str(case["thresholds"])
        groups.setdefault(key, []).append(case)
    for key, group in groups.items():
        th = TH(**group[0]["thresholds"]) if group[0]["thresholds"] else TH()
        scripts, seeds = [], []
        for case in group:
            scripts.append(dict(subtask=SUBTASKS.index(case["subtask"]),
                                kinds=[EV.index(s[0]) for s in case["steps"]],
                                gaps=[s[1] for s in case["steps"]], tail=case["tail"],
                                initial_grasped=int(case["initial_grasped"]),
                                initial_contact=int(case["initial_contact"]),
                                initial_level=LEVELS.index(case["initial_art_level"]),
                                art_kind=ART.index(case["articulation_kind"]),
                                initial_dist_obj_goal=case["initial_dist_obj_goal"]))
            seeds.append(case["seed"])
        cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
        arr, k, g = _scripts_np(C, scripts, seeds)
        sb = C.realize_batch(arr, k, g, th, cs)
        lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
        planes = sb.records.planes.cpu().numpy()
        rs = sb.records.rec_start.cpu().numpy()
        nr = sb.records.n_rec.cpu().numpy()
        for i, case in enumerate(group):
            if case["error"] is not None:
                st = int(lab["status"][i])
                step = int(lab["err"][i])
                ev = case["steps"][step][0] if step >= 0 else None
                exc = ER.infeasible_error(st, case["subtask"], ev, case["initial_art_level"])
                assert [type(exc).__name__, str(exc)] == case["error"], (case, st, step)
                continue
            assert lab["status"][i] == 0, (case, lab["status"][i])
            n = case["n_records"]
            assert nr[i] == n
            p = planes[:, rs[i]:rs[i] + n]
            vals = np.concatenate([p[:, t] for t in range(n)]) if n else np.zeros(0)
            # fixture order per record: q_arm, qd_arm, 9 scalars, grasped
            g_ = sb.records.grasped[rs[i]:rs[i] + n].cpu().numpy().astype(np.float32)
            got = np.concatenate([np.concatenate([p[:, t], [g_[t]]]) for t in range(n)])
            want = np.frombuffer(bytes.fromhex(case["records_f32_hex"]), np.float32)
            assert same_bits_f32(got, want), case


def test_classify_cases(C):
    EV = ("Contact", "Grasped", "Dropped", "ObjAtGoal", "ReleasedAtGoal",
          "ReleasedOutsideGoal", "ObjLeftGoal", "Opened", "SlightlyOpened", "Closed",
          "SlightlyClosed", "Open", "Success", "ExcessiveCollisions")
    from oracle.oracle import MODE_IDS
    cases = js("classify")
    base = {0: 0, 1: 9, 2: 21, 3: 30}
    nsucc = {0: 4, 1: 5, 2: 3, 3: 3}
    nmodes = {0: 9, 1: 12, 2: 9, 3: 9}
    for drop in (False, True):
        sel = [c for c in cases if (c["rules"] == "drop_catch_all") == drop]
        rules = None
        if drop:
            rules = [[list(range(base[s], base[s] + nsucc[s])),
                      list(range(base[s] + nsucc[s], base[s] + nmodes[s] - 1))] for s in range(4)]
        lab = C.classify_lists([[EV.index(k) for k in c["kinds"]] for c in sel],
                               [SUBTASKS.index(c["subtask"]) for c in sel],
                               [c["d0"] if c["d0"] is not None else 0.0 for c in sel],
                               [c["d0"] is None for c in sel], rules)
        from paper_2412_13211_b200 import _lib as L
        for i, c in enumerate(sel):
            if "error" in c:
                assert lab["status"][i] != 0, c
                assert L.lib().tl_status_name(int(lab["status"][i])).decode() == c["error"][0]
            else:
                assert lab["status"][i] == 0, c
                assert [MODE_IDS[lab["mode"][i]], bool(lab["flags"][i] & 1),
                        bool(lab["flags"][i] & 2)] == c["result"], c


def test_filter_cases(C):
    from test_oracle_golden import filter_ints
    dev = torch.device("cuda")
    for case in js("filter"):
        labels, spec = case["labels"], case["spec"]
        order, rows, pool, pool_keys, rule_w, n_rules = filter_ints(labels, spec)
        # dense buckets: pool p owns n_rules[subtask(p)] buckets
        psub = {}
        for j, r in enumerate(rows):
            if r[3] >= 0:
                psub[pool[j]] = r[2]
        b0 = [0]
        w = []
        for p in range(len(pool_keys)):
            s = psub[p]
            b0.append(b0[-1] + int(n_rules[s]))
            w.extend(rule_w[s * 16: s * 16 + int(n_rules[s])])
        bucket = np.array([b0[pool[j]] + r[3] if r[3] >= 0 else -1 for j, r in enumerate(rows)], np.int32)
        sel, ps = C.filter_select(torch.from_numpy(bucket).to(dev), int(b0[-1]),
                                  torch.from_numpy(np.array(b0, np.int32)).to(dev),
                                  torch.from_numpy(np.array(w if w else [1.0], np.float64)).to(dev),
                                  spec["quota_per_target"])
        sel = sel.cpu().numpy()
        got = sorted(labels[rows[j][0]][0] for j in range(len(rows)) if sel[j])
        assert got == case["selected"]
        ps = ps.cpu().numpy()
        short = [{"quota_key": k[0], "subtask": k[1], "requested": spec["quota_per_target"],
                  "selected": int(ps[j]), "shortfall": spec["quota_per_target"] - int(ps[j])}
                 for j, k in enumerate(pool_keys) if ps[j] < spec["quota_per_target"]]
        assert short == case["shortfalls"]


@pytest.mark.parametrize("kind", range(4))
def test_fuzz_10k_vs_oracle(C, TH, kind):
    """acceptance criterion 2 scale: 10k fuzz seeds per subtask, records
    bit-exact and modes equal against the CPU oracle (tests/test_acceptance.py:46-67)."""
    from oracle import oracle as O
    from golden_data import from_oracle_records
    from paper_2412_13211_b200.synth import FuzzConfig
    n = 10000
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    sb = C.fuzz_batch(np.arange(n), kind, FuzzConfig(), TH(), cs)
    total, modes, nev, nrec = O.fuzz_label_batch(0, n, kind, n_threads=8)
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    assert np.all(lab["status"] == 0)
    assert np.array_equal(lab["mode"], modes)
    assert np.array_equal(lab["n_events"], nev)
    assert np.array_equal(sb.records.n_rec.cpu().numpy(), nrec)
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    for seed in range(0, n, 97):
        _, recs = O.fuzz(seed, kind)
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(planes[:, rs[seed]:rs[seed] + len(recs)], p), seed


def test_mode_histogram(C, TH):
    from paper_2412_13211_b200.synth import FuzzConfig
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    sb = C.fuzz_batch(np.arange(3000), 1, FuzzConfig(), TH(), cs)
    h = C.mode_histogram(sb.labels, 3000).cpu().numpy()
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    assert np.array_equal(h, np.bincount(lab["mode"], minlength=39))


@pytest.mark.parametrize("kind", range(4))
def test_fused_scan_emit_matches_two_pass(C, TH, kind):
    """tl_scan_emit_events (decoupled look-back) == tl_scan_events + tl_emit_events."""
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 5000  # 157 tiles of 32 episodes
    sb = C.fuzz_batch(np.arange(n) + 777, kind, cfg, TH(), cs)
    a = C.LabelResult(sb.labels, sb.step_mask, None)
    C.emit_events(sb.records, a)
    b = C.LabelResult(sb.labels, sb.step_mask, None)
    C.emit_events(sb.records, b, ev_capacity=n * C.fuzz_capacity(cfg))
    assert torch.equal(a.ev_off, b.ev_off)
    tot = int(a.ev_off[-1])
    assert torch.equal(a.ev_kind[:tot], b.ev_kind[:tot])
    assert torch.equal(a.ev_t[:tot], b.ev_t[:tot])


@pytest.mark.parametrize("density", [0.05, 0.9])
@pytest.mark.parametrize("shift", [0, 1, 3])
def test_scan_emit_staging_and_alignment(C, TH, density, shift):
    """k_scan_emit stages a tile's events in shared memory and stores the
    tile's range with aligned words: sparse masks take the staged path, dense
    masks (> 4096 events per 32-episode tile) the direct one; outputs offset
    by `shift` elements move every tile's phase.  Against the two-pass
    tl_scan_events + tl_emit_events on the same masks."""
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 700
    sb = C.fuzz_batch(np.arange(n) + 31337, 0, cfg, TH(), cs)
    rng = np.random.default_rng(int(density * 100) + shift)
    nbits = int(sb.step_mask.numel())
    bits = (rng.random((nbits, 8)) < density).astype(np.uint8)
    mask_np = (bits << np.arange(8, dtype=np.uint8)).sum(axis=1).astype(np.uint8)
    rs = sb.records.rec_start.cpu().numpy()
    nr = sb.records.n_rec.cpu().numpy()
    pop = np.unpackbits(mask_np[:, None], axis=1).sum(axis=1)
    for e in range(n):  # record 0 never carries an edge; keep the masks inside the episodes
        mask_np[rs[e]] = 0
        pop[rs[e]] = 0
    lab = sb.labels.clone()
    lv = lab.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    lv["n_events"] = [int(pop[rs[e]:rs[e] + nr[e]].sum()) for e in range(n)]
    lv["sub"] = np.arange(n) % 4
    lab = torch.from_numpy(lv.view(np.uint8).reshape(lab.shape)).cuda()
    mask = torch.from_numpy(mask_np).cuda()
    a = C.LabelResult(lab, mask, None)
    C.emit_events(sb.records, a)
    tot = int(a.ev_off[-1])
    if density > 0.5:
        assert tot > 4096 * (n // 32)  # the direct path on every full tile
    ev_off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    kbuf = torch.full((tot + 8,), 0xAB, dtype=torch.uint8, device="cuda")
    tbuf = torch.full((tot + 8,), -7, dtype=torch.int32, device="cuda")
    scratch = torch.empty(max(16, L.lib().tl_scan_scratch_bytes(n)), dtype=torch.uint8, device="cuda")
    L.check(L.lib().tl_scan_emit_events(L.ptr(mask), L.ptr(sb.records.rec_start),
                                        L.ptr(sb.records.n_rec), L.ptr(lab), n, L.ptr(ev_off),
                                        kbuf.data_ptr() + shift, tbuf.data_ptr() + 4 * shift,
                                        L.ptr(scratch), L.stream_ptr()), "tl_scan_emit_events")
    assert torch.equal(ev_off, a.ev_off)
    assert torch.equal(kbuf[shift:shift + tot], a.ev_kind[:tot])
    assert torch.equal(tbuf[shift:shift + tot], a.ev_t[:tot])
    # nothing outside [shift, shift + tot) was written
    assert bool((kbuf[:shift] == 0xAB).all()) and bool((kbuf[shift + tot:] == 0xAB).all())
    assert bool((tbuf[:shift] == -7).all()) and bool((tbuf[shift + tot:] == -7).all())


@pytest.mark.parametrize("kind", range(4))
@pytest.mark.parametrize("n", [1, 37, 5000])
def test_fused_synth_events_match_two_pass(C, TH, kind, n):
    """tl_fuzz_ev (event lists built inside the realize kernel by a look-back
    over episodes) == tl_fuzz + tl_scan_events + tl_emit_events."""
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    seeds = np.arange(n) + 4242
    fused = C.fuzz_batch(seeds, kind, cfg, TH(), cs, events=True)
    f_off = fused.label_result.ev_off.clone()
    tot = int(f_off[-1])
    f_kind = fused.label_result.ev_kind[:tot].clone()
    f_t = fused.label_result.ev_t[:tot].clone()
    f_lab = fused.labels.clone()
    sb = C.fuzz_batch(seeds, kind, cfg, TH(), cs)
    a = C.LabelResult(sb.labels, sb.step_mask, None)
    C.emit_events(sb.records, a)
    assert torch.equal(f_lab, sb.labels)
    assert torch.equal(f_off, a.ev_off)
    assert torch.equal(f_kind, a.ev_kind[:tot])
    assert torch.equal(f_t, a.ev_t[:tot])


def test_fused_events_zero_copy_host_outputs(C, TH):
    """tl_fuzz_ev reading the seeds from and writing labels and event lists
    straight into pinned host memory (the e2e path) == the device-memory
    outputs."""
    import ctypes
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 1024
    seeds = torch.arange(n, dtype=torch.int64, device="cuda") + 555
    ref = C.fuzz_batch(seeds, 1, cfg, TH(), cs, events=True)
    tot = int(ref.label_result.ev_off[-1])
    cap = C.fuzz_capacity(cfg)
    ws = C.SynthWorkspace(n, cap)
    ev_cap = 4 * n * cap
    h_lab = torch.empty((n, 24), dtype=torch.uint8).pin_memory()
    h_off = torch.empty(n + 1, dtype=torch.int64).pin_memory()
    h_k = torch.empty(ev_cap, dtype=torch.uint8).pin_memory()
    h_t = torch.empty(ev_cap, dtype=torch.int32).pin_memory()
    rb = ws.records()
    h_seeds = seeds.cpu().pin_memory()
    rc = L.lib().tl_fuzz_ev(L.ptr(h_seeds), n, 1, ctypes.byref(C.fuzz_cfg_c(cfg)),
                            ctypes.byref(C.thresholds_c(TH())), L.ptr(cs), None,
                            ctypes.byref(rb.c()), cap, None, None, None, L.ptr(ws.step_mask),
                            L.ptr(h_lab), L.ptr(h_off), L.ptr(h_k), L.ptr(h_t), ev_cap,
                            L.ptr(ws.scratch), L.stream_ptr())
    L.check(rc, "tl_fuzz_ev")
    torch.cuda.synchronize()
    assert torch.equal(h_lab, ref.labels[:n].cpu())
    assert torch.equal(h_off, ref.label_result.ev_off.cpu())
    assert torch.equal(h_k[:tot], ref.label_result.ev_kind[:tot].cpu())
    assert torch.equal(h_t[:tot], ref.label_result.ev_t[:tot].cpu())


def test_realize_multi_window_scripts(C, TH):
    """Scripts longer than one plan window (kMaxSteps = 64 steps) against the
    oracle: the realize kernel re-plans window by window, carrying the
    realizer state, word offset and object-distance draws across."""
    from oracle import oracle as O
    from golden_data import from_oracle_records
    rng = np.random.default_rng(99)
    scripts, seeds = [], []
    cycles = {0: [0, 1, 2], 1: [3, 6], 2: [8, 7, 9]}  # Pick C,G,D; Place OAG,OLG; Open SO,O,C
    for i in range(24):
        kind = i % 3
        n_steps = int(rng.integers(65, 200))
        cyc = cycles[kind]
        kinds = [cyc[j % len(cyc)] for j in range(n_steps)]
        gaps = list(rng.integers(1, 5, n_steps))
        d = dict(subtask=kind, kinds=np.asarray(kinds, np.uint8), gaps=np.asarray(gaps, np.int32),
                 tail=int(rng.integers(1, 6)), initial_grasped=0, initial_contact=0,
                 initial_dist_obj_goal=0.5 if kind == 1 else 0.5, initial_level=0,
                 art_kind=1 if kind == 2 else 0, arm_dof=7)
        scripts.append(d)
        seeds.append(int(rng.integers(0, 2**31)))
    arr, k, g = _scripts_np(C, scripts, seeds)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    sb = C.realize_batch(arr, k, g, TH(), cs)
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    n_ok = 0
    for i, d in enumerate(scripts):
        try:
            recs = O.realize(d, seeds[i])
        except O.OracleError as e:
            assert lab["status"][i] == e.code, (i, lab["status"][i], e.code)
            assert lab["err"][i] == e.step, (i, lab["err"][i], e.step)
            continue
        n_ok += 1
        assert lab["status"][i] == 0, (i, lab["status"][i])
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(planes[:, rs[i]:rs[i] + len(recs)], p), i
    assert n_ok >= 8


@pytest.mark.parametrize("kind", range(4))
def test_fuzz_many_events_vs_oracle(C, TH, kind):
    """FuzzConfig(max_events=150): scripts of up to 154 steps (several plan
    windows) sampled and realized on the device == the oracle's fuzz."""
    from oracle import oracle as O
    from golden_data import from_oracle_records
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_events=150, max_gap=3, max_tail=4)
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 300
    sb = C.fuzz_batch(np.arange(n) + 1000 * kind, kind, cfg, TH(), cs, want_scripts=True)
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    ocfg = O.fuzz_cfg(max_events=150, max_gap=3, max_tail=4)
    long_scripts = 0
    for i in range(n):
        sc, recs = O.fuzz(1000 * kind + i, kind, ocfg)
        long_scripts += len(sc["kinds"]) > 64
        assert lab["status"][i] == 0, (i, lab["status"][i])
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(planes[:, rs[i]:rs[i] + len(recs)], p), i
    assert long_scripts > 10


def test_fuzz_extreme_seeds_vs_oracle(C, TH):
    """Negative seeds (random.Random uses abs(seed)), 1- and 2-word keys
    around 2^32, and the int64 extremes, against the oracle."""
    from oracle import oracle as O
    from golden_data import from_oracle_records
    from paper_2412_13211_b200.synth import FuzzConfig
    seeds = [0, 1, -1, -7, 2**32 - 1, 2**32, -(2**32), 2**33 + 5, -(2**40) - 3,
             2**63 - 1, -(2**63), -(2**63) + 1, 123456789012345, -987654321098]
    cfg = FuzzConfig()
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    for kind in range(4):
        sb = C.fuzz_batch(torch.tensor(seeds, dtype=torch.int64, device="cuda"), kind, cfg, TH(), cs)
        planes = sb.records.planes.cpu().numpy()
        rs = sb.records.rec_start.cpu().numpy()
        nr = sb.records.n_rec.cpu().numpy()
        for i, sd in enumerate(seeds):
            _, recs = O.fuzz(sd, kind)
            assert nr[i] == len(recs), (kind, sd)
            p, _ = from_oracle_records(O, recs)
            assert same_bits_f32(planes[:, rs[i]:rs[i] + len(recs)], p), (kind, sd)


# every product launch shape of the reset / realize kernels is checked
# against the oracle in test_gpu_shipped.py::test_shipped_fuzz_configs_vs_oracle


@pytest.mark.parametrize("kind", range(4))
def test_short_wave_multi_window_vs_oracle(C, TH, kind):
    """Episodes of <= 64 records but up to 44 script steps: the 2-warp
    realize form (32-record waves) plans them in windows of 32 steps; records
    and labels == the oracle's fuzz."""
    from oracle import oracle as O
    from golden_data import from_oracle_records
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_events=40, max_gap=1, max_tail=1)
    assert C.fuzz_capacity(cfg) <= 64          # selects the 2-warp form
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 400
    sb = C.fuzz_batch(np.arange(n) + 777 * (kind + 1), kind, cfg, TH(), cs, want_scripts=True)
    lab = sb.labels.cpu().numpy().reshape(-1).view(np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"), ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    ocfg = O.fuzz_cfg(max_events=40, max_gap=1, max_tail=1)
    multi = 0
    for i in range(n):
        sc, recs = O.fuzz(777 * (kind + 1) + i, kind, ocfg)
        multi += len(sc["kinds"]) > 32
        assert lab["status"][i] == 0, (i, lab["status"][i])
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(planes[:, rs[i]:rs[i] + len(recs)], p), i
    assert multi > 10


@pytest.mark.parametrize("long_cfg", [False, True])
def test_fuzz_mixed_subtasks_match_per_subtask_batches(C, TH, long_cfg):
    """tl_fuzz_ev_mixed (a subtask per episode: the C4 chain batch) == the
    four single-subtask tl_fuzz_ev batches on the same seeds -- labels, record
    counts, records and ordered event lists; an out-of-range subtask gives
    that episode TL_E_INVALID and no records."""
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig(max_gap=64, max_tail=64) if long_cfg else FuzzConfig()
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 3000
    rng = np.random.default_rng(11 + long_cfg)
    seeds = rng.integers(0, 2**40, n).astype(np.int64)
    subs = rng.integers(0, 4, n).astype(np.uint8)
    subs[[5, 777, 2999]] = [4, 9, 255]
    mixed = C.fuzz_batch(seeds, subs, cfg, TH(), cs, events=True)
    m_lab = mixed.labels.cpu().numpy()
    m_lv = m_lab.reshape(-1).view(L.LABEL_DTYPE)
    m_nrec = mixed.records.n_rec.cpu().numpy()
    m_rs = mixed.records.rec_start.cpu().numpy()
    m_pl = mixed.records.planes.cpu().numpy()
    m_off = mixed.label_result.ev_off.cpu().numpy()
    m_k = mixed.label_result.ev_kind.cpu().numpy()
    m_t = mixed.label_result.ev_t.cpu().numpy()
    bad = subs > 3
    assert np.all(m_lv["status"][bad] == 100) and np.all(m_nrec[bad] == 0)
    assert np.all(m_off[1:][bad] == m_off[:-1][bad])
    for k in range(4):
        idx = np.nonzero(subs == k)[0]
        one = C.fuzz_batch(seeds[idx], k, cfg, TH(), cs, events=True)
        assert np.array_equal(one.labels.cpu().numpy(), m_lab[idx]), k
        nrec = one.records.n_rec.cpu().numpy()
        assert np.array_equal(nrec, m_nrec[idx]), k
        rs = one.records.rec_start.cpu().numpy()
        pl = one.records.planes.cpu().numpy()
        off = one.label_result.ev_off.cpu().numpy()
        ek = one.label_result.ev_kind.cpu().numpy()
        et = one.label_result.ev_t.cpu().numpy()
        for j, e in enumerate(idx):
            assert same_bits_f32(pl[:, rs[j]:rs[j] + nrec[j]], m_pl[:, m_rs[e]:m_rs[e] + nrec[j]]), (k, e)
            a, b = off[j], off[j + 1]
            c, d = m_off[e], m_off[e + 1]
            assert np.array_equal(ek[a:b], m_k[c:d]) and np.array_equal(et[a:b], m_t[c:d]), (k, e)


def test_fuzz_mixed_without_event_lists(C, TH):
    """tl_fuzz_mixed (records + labels, no event lists) == per-subtask tl_fuzz."""
    from paper_2412_13211_b200.synth import FuzzConfig
    cfg = FuzzConfig()
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    n = 1500
    seeds = np.arange(n, dtype=np.int64) * 7 + 123
    subs = (np.arange(n) % 4).astype(np.uint8)[::-1].copy()
    mixed = C.fuzz_batch(seeds, torch.from_numpy(subs), cfg, TH(), cs)
    m_lab = mixed.labels.cpu().numpy()
    m_nrec = mixed.records.n_rec.cpu().numpy()
    m_rs = mixed.records.rec_start.cpu().numpy()
    m_pl = mixed.records.planes.cpu().numpy()
    m_mask = mixed.step_mask.cpu().numpy()
    for k in range(4):
        idx = np.nonzero(subs == k)[0]
        one = C.fuzz_batch(seeds[idx], k, cfg, TH(), cs)
        assert np.array_equal(one.labels.cpu().numpy(), m_lab[idx])
        nrec = one.records.n_rec.cpu().numpy()
        assert np.array_equal(nrec, m_nrec[idx])
        rs = one.records.rec_start.cpu().numpy()
        pl = one.records.planes.cpu().numpy()
        mask = one.step_mask.cpu().numpy()
        for j, e in enumerate(idx):
            assert same_bits_f32(pl[:, rs[j]:rs[j] + nrec[j]], m_pl[:, m_rs[e]:m_rs[e] + nrec[j]])
            assert np.array_equal(mask[rs[j]:rs[j] + nrec[j]], m_mask[m_rs[e]:m_rs[e] + nrec[j]])
