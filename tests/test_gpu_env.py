"""GPU parity of the batched env (reset / step(actions), csrc/tl_env.cuh):
replaying a script's action stream must reproduce realize() bit-exactly
(records, events, modes, InfeasibleScript raise sites), against the
reference fixtures and the CPU oracle.  Runs on a B200 (-m gpu)."""
import math

import numpy as np
import pytest

from golden_data import (ART, DOF, LEVELS, SUBTASKS, Corpus, from_oracle_records, js,
                         npz, same_bits_f32)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _event_script(P, sc, episode_id="env"):
    from paper_2412_13211_b200.events import EVENT_KINDS
    return P.EventScript(
        subtask_kind=P.SubtaskKind(SUBTASKS[int(sc["subtask"])]),
        steps=[P.ScriptStep(EVENT_KINDS[int(k)], int(g)) for k, g in zip(sc["kinds"], sc["gaps"])],
        tail=int(sc["tail"]), initial_grasped=bool(sc["initial_grasped"]),
        initial_contact=bool(sc["initial_contact"]),
        initial_dist_obj_goal=float(sc["initial_dist_obj_goal"]),
        initial_art_level=LEVELS[int(sc["initial_level"])] if int(sc["initial_level"]) < 5 else "bogus",
        articulation_kind=P.ArticulationKind(ART[int(sc["art_kind"])] if int(sc["art_kind"]) else "Fridge"),
        episode_id=episode_id, arm_dof=DOF)


def _mask_events(subtask, masks):
    """step masks [T] (record t at index t) -> ([global kind], [t])."""
    from paper_2412_13211_b200.events import EVENT_KINDS, EVENT_ORDER
    from paper_2412_13211_b200.model import SubtaskKind
    alpha = [EVENT_KINDS.index(k) for k in EVENT_ORDER[SubtaskKind(SUBTASKS[subtask])]]
    ks, ts = [], []
    for t, m in enumerate(masks):
        for b in range(7):
            if (int(m) >> b) & 1:
                ks.append(alpha[b])
                ts.append(t)
    return ks, ts


def _run(env, chunks=(1, 3), with_grasped=False):
    """reset already done; replay scripted actions with a few launch sizes.
    -> per-launch obs [F, k, N] and masks [k, N] (record t at column t - 1)."""
    lengths = env.script_lengths()
    T = int(lengths.max())
    obs, masks, gr = [], [], []
    t = 1
    for k in list(chunks) + [max(T - 1 - sum(chunks), 0)]:
        k = min(k, T - t)
        if k <= 0:
            break
        st = env.step(env.scripted_actions(t, k))
        obs.append(st.obs)
        masks.append(st.step_mask)
        gr.append(st.grasped)
        t += k
    if with_grasped:
        return obs, masks, lengths, gr
    return obs, masks, lengths


def _collect(reset_step, obs, masks):
    o = torch.cat([reset_step.obs] + obs, dim=1).cpu().numpy()
    m = torch.cat([reset_step.step_mask] + masks, dim=0).cpu().numpy()
    return o, m


@pytest.mark.parametrize("name", ["defining", "long"])
def test_env_replays_reference_scripts(name):
    """reset + scripted steps == the reference's realize() fixtures."""
    import paper_2412_13211_b200 as P
    d = npz(name)
    c = Corpus(d)
    scripts = [_event_script(P, sc) for sc in c.scripts()]
    env = P.BatchedSubtaskEnv(len(scripts))
    r0 = env.reset(scripts=scripts, seeds=[int(s) for s in d["seed"]])
    obs, masks, lengths = _run(env)
    o, m = _collect(r0, obs, masks)
    lab, nrec = env.labels()
    for i in range(c.n):
        planes, _ = c.records_np(i)
        n = planes.shape[1]
        assert lengths[i] == n and nrec[i] == n, i
        assert same_bits_f32(o[:, :n, i], planes), i
        assert lab["status"][i] == 0 and lab["mode"][i] == c.mode[i], i
        assert bool(lab["flags"][i] & 1) == bool(c.success_once[i])
        assert bool(lab["flags"][i] & 2) == bool(c.success_at_end[i])
        assert _mask_events(int(c.subtask[i]), m[:n, i]) == c.events(i), i


@pytest.mark.parametrize("kind", range(4))
def test_env_fuzz_reset_replays_fuzz(kind):
    """reset(seeds, subtask) + scripted steps == fuzz(seed) (the fused
    generator, itself pinned to the oracle) for 2000 seeds."""
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200 import core
    cfg = P.FuzzConfig(max_gap=16, max_tail=16)
    n = 2000
    seeds = np.arange(n) * 7 + 11
    env = P.BatchedSubtaskEnv(n)
    r0 = env.reset(seeds=seeds, subtask=P.SubtaskKind(SUBTASKS[kind]), config=cfg)
    obs, masks, lengths = _run(env, chunks=(1, 2, 5))
    o, m = _collect(r0, obs, masks)
    lab, nrec = env.labels()
    cs = core.synth_csets(P.Thresholds()).to_device(torch.device("cuda"))
    sb = core.fuzz_batch(seeds, kind, cfg, P.Thresholds(), cs)
    want = sb.labels.cpu().numpy().reshape(-1).view(lab.dtype)
    assert np.array_equal(lab["status"], want["status"])
    assert np.array_equal(lab["mode"], want["mode"])
    assert np.array_equal(lab["flags"], want["flags"])
    assert np.array_equal(lab["n_events"], want["n_events"])
    assert np.array_equal(nrec, sb.records.n_rec.cpu().numpy())
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    smask = sb.step_mask.cpu().numpy()
    for e in range(0, n, 13):
        k = nrec[e]
        assert same_bits_f32(o[:, :k, e], planes[:, rs[e]:rs[e] + k]), e
        assert np.array_equal(m[:k, e], smask[rs[e]:rs[e] + k]), e


def test_env_fuzz_vs_oracle():
    from oracle import oracle as O
    import paper_2412_13211_b200 as P
    n = 64
    env = P.BatchedSubtaskEnv(n)
    r0 = env.reset(seeds=np.arange(n), subtask=P.SubtaskKind.Close)
    obs, masks, lengths = _run(env)
    o, _ = _collect(r0, obs, masks)
    for s in range(n):
        _, recs = O.fuzz(s, 3)
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(o[:, :len(recs), s], p), s


def test_env_infeasible_scripts_raise_like_reference():
    """scripts.json: every feasible script replays bit-exactly, every
    infeasible one stops the env with the reference's InfeasibleScript."""
    import paper_2412_13211_b200 as P
    EV = ("Contact", "Grasped", "Dropped", "ObjAtGoal", "ReleasedAtGoal",
          "ReleasedOutsideGoal", "ObjLeftGoal", "Opened", "SlightlyOpened", "Closed",
          "SlightlyClosed", "Open", "Success", "ExcessiveCollisions")
    groups = {}
    for case in js("scripts"):
        groups.setdefault(str(case["thresholds"]), []).append(case)
    checked = 0
    for _, group in groups.items():
        th = P.Thresholds(**group[0]["thresholds"]) if group[0]["thresholds"] else P.Thresholds()
        scripts = [P.EventScript(
            subtask_kind=P.SubtaskKind(case["subtask"]),
            steps=[P.ScriptStep(P.EventKind(s[0]), int(s[1])) for s in case["steps"]],
            tail=case["tail"], initial_grasped=case["initial_grasped"],
            initial_contact=case["initial_contact"],
            initial_dist_obj_goal=case["initial_dist_obj_goal"],
            initial_art_level=case["initial_art_level"],
            articulation_kind=P.ArticulationKind(case["articulation_kind"]))
            for case in group]
        env = P.BatchedSubtaskEnv(len(scripts), th=th)
        r0 = env.reset(scripts=scripts, seeds=[c["seed"] for c in group])
        obs, masks, lengths, gr = _run(env, with_grasped=True)
        o, _ = _collect(r0, obs, masks)
        g = torch.cat([r0.grasped] + gr, dim=0).cpu().numpy().astype(np.float32)
        lab, nrec = env.labels()
        errs = env.errors(lab)
        for i, case in enumerate(group):
            if case["error"] is not None:
                assert errs[i] is not None, case
                assert [type(errs[i]).__name__, str(errs[i])] == case["error"], case
                continue
            assert errs[i] is None and lab["status"][i] == 0, (case, lab["status"][i])
            n = case["n_records"]
            assert nrec[i] == n
            # fixture order per record: q_arm, qd_arm, 9 scalars, grasped
            got = np.concatenate([np.concatenate([o[:, t, i], [g[t, i]]]) for t in range(n)])
            want = np.frombuffer(bytes.fromhex(case["records_f32_hex"]), np.float32)
            assert same_bits_f32(got, want), case
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("subtask", range(4))
def test_env_random_actions_vs_oracle(subtask):
    """Arbitrary action streams (mostly infeasible somewhere): every env
    either matches oracle realize() of the equivalent script record for
    record, or stops at the same step with the same InfeasibleScript code."""
    from oracle import oracle as O
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200.events import EVENT_KINDS, EVENT_ORDER
    rng = np.random.default_rng(1234 + subtask)
    n, T = 256, 48
    sk = P.SubtaskKind(SUBTASKS[subtask])
    alpha = [EVENT_KINDS.index(k) for k in EVENT_ORDER[sk]]
    acts = np.full((T, n), P.env.HOLD, np.uint8)
    scripts, dicts, seeds = [], [], []
    for e in range(n):
        p_evt = rng.choice([0.05, 0.15, 0.35])
        for t in range(T - 1):  # the last step is always a hold (tail >= 1)
            if rng.random() < p_evt:
                acts[t, e] = rng.choice(alpha) if rng.random() < 0.95 else rng.integers(0, 14)
        ev_t = np.nonzero(acts[:, e] != P.env.HOLD)[0]
        gaps = np.diff(np.concatenate([[0], ev_t + 1])).astype(np.int32)
        art = int(rng.integers(1, 3)) if subtask >= 2 else 0
        lvl = int(rng.choice([0, 1, 2])) if subtask == 2 else int(rng.choice([3, 1, 4])) if subtask == 3 else 0
        contact = int(rng.random() < 0.3)
        d = dict(subtask=subtask, kinds=acts[ev_t, e].copy(), gaps=gaps,
                 tail=int(T - 1 - ev_t[-1]) if len(ev_t) else T,
                 initial_grasped=int(rng.random() < 0.4 and (subtask != 0 or contact)),
                 initial_contact=contact,
                 initial_dist_obj_goal=float(rng.choice([0.1, 0.5, 0.15])),
                 initial_level=lvl, art_kind=art, arm_dof=DOF)
        dicts.append(d)
        scripts.append(_event_script(P, d))
        seeds.append(int(rng.integers(0, 2**40)))
    env = P.BatchedSubtaskEnv(n)
    r0 = env.reset(scripts=scripts, seeds=seeds)
    a = torch.from_numpy(acts)
    outs = [env.step(a[:1]), env.step(a[1:8]), env.step(a[8:])]
    o = torch.cat([r0.obs] + [x.obs for x in outs], dim=1).cpu().numpy()
    lab, nrec = env.labels()
    n_ok = n_err = 0
    for e in range(n):
        try:
            recs = O.realize(dicts[e], seeds[e])
        except O.OracleError as err:
            n_err += 1
            assert lab["status"][e] == err.code, (e, lab["status"][e], err.code)
            ev_t = np.nonzero(acts[:, e] != P.env.HOLD)[0]
            want_t = 0 if err.code in (20, 41) else int(ev_t[err.step]) + 1
            assert lab["err_index"][e] == want_t, e
            continue
        n_ok += 1
        assert lab["status"][e] in (0, 7), e  # ModeCoverage can't happen with MODE_RULES
        assert nrec[e] == len(recs) == T + 1
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(o[:, :T + 1, e], p), e
        hdr = O.synth_header(dicts[e])
        ks, ts, d0 = O.extract_events(recs, hdr)
        mode, so, se = O.classify(subtask, ks, d0, d0_none=subtask != 1)
        assert lab["mode"][e] == mode and lab["n_events"][e] == len(ks), e
    assert n_ok > 10 and n_err > 10, (n_ok, n_err)


def test_env_idle_and_hold_semantics():
    """IDLE steps change nothing; splitting a rollout over launches of any
    size gives the same records."""
    import paper_2412_13211_b200 as P
    n = 96
    seeds = np.arange(n) + 5
    a = P.BatchedSubtaskEnv(n)
    b = P.BatchedSubtaskEnv(n)
    ra = a.reset(seeds=seeds, subtask=P.SubtaskKind.Pick, config=P.FuzzConfig(max_gap=8))
    rb = b.reset(seeds=seeds, subtask=P.SubtaskKind.Pick, config=P.FuzzConfig(max_gap=8))
    assert torch.equal(ra.obs.view(torch.int32), rb.obs.view(torch.int32))  # NaN-exact
    T = int(a.script_lengths().max())
    acts = a.scripted_actions(1, T - 1)
    full = a.step(acts)
    got = []
    idle = torch.full((1, n), P.env.IDLE, dtype=torch.uint8, device="cuda")
    for t in range(T - 1):
        b.step(idle)
        got.append(b.step(acts[t:t + 1]).obs)
    live = (acts != P.env.IDLE).unsqueeze(0).expand_as(full.obs)
    assert torch.equal(torch.cat(got, dim=1).view(torch.int32)[live],
                       full.obs.view(torch.int32)[live])
    la, _ = a.labels()
    lb, _ = b.labels()
    assert la.tobytes() == lb.tobytes()


def test_env_cuda_graph_replay():
    """reset + step captured in a CUDA graph replays to the same episodes
    (the reset writes its header from kernel parameters, not host memory)."""
    import paper_2412_13211_b200 as P
    n, T = 512, 120
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        env = P.BatchedSubtaskEnv(n)
        seeds = torch.arange(n, dtype=torch.int64, device="cuda") + 99
        cfg = P.FuzzConfig(max_gap=32, max_tail=32)
        b0 = env._outputs(1, None)
        bT = env._outputs(T, None)
        env.reset(seeds=seeds, subtask=P.SubtaskKind.Place, config=cfg, out=b0)
        acts = env.scripted_actions(1, T)
        env.step(acts, out=bT)
        want_lab, want_n = env.labels()
        want_obs = bT.obs.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            env.reset(seeds=seeds, subtask=P.SubtaskKind.Place, config=cfg, out=b0)
            env.step(acts, out=bT)
        for _ in range(2):
            bT.obs.zero_()
            g.replay()
            torch.cuda.synchronize()
            lab, nrec = env.labels()
            assert lab.tobytes() == want_lab.tobytes() and np.array_equal(nrec, want_n)
            live = (acts != P.env.IDLE).unsqueeze(0).expand_as(bT.obs)
            assert torch.equal(bT.obs.view(torch.int32)[live], want_obs.view(torch.int32)[live])
