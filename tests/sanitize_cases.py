"""Small invocations of every product entry point, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tests/sanitize_cases.py [case ...]

Cases: fuzz_ev (k_fuzz_reset + k_synth_warp + k_scan_emit, long and short
episode configs), fuzz (tl_fuzz), label (k_label vector + generic bodies, f32 and
f64, k_scan_emit), env (k_env_reset + k_env_step, both lane mappings),
filter (k_filter_*), validate (k_validate), predicates, analytics.
Each case checks its result against the oracle / its own invariants so a
sanitizer run is also a correctness run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_13211_b200 as P  # noqa: E402
from paper_2412_13211_b200 import core, model  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

TH = P.Thresholds()


def lab_np(t):
    from paper_2412_13211_b200 import _lib as L
    return t.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)


def case_fuzz_ev():
    cs = core.synth_csets(TH).to_device(torch.device("cuda"))
    for kind, cfg in ((1, P.FuzzConfig(max_gap=64, max_tail=64)), (2, P.FuzzConfig())):
        n = 96
        sb = core.fuzz_batch(np.arange(n), kind, cfg, TH, cs, events=True)
        torch.cuda.synchronize()
        lab = lab_np(sb.labels)
        want = O.fuzz_label_batch_full(0, n, kind, cfg=O.fuzz_cfg(**vars(cfg)), n_threads=2)
        assert (lab["status"] == 0).all()
        assert np.array_equal(lab["mode"], want["mode"])
        off = sb.label_result.ev_off.cpu().numpy()
        assert np.array_equal(off, want["ev_off"])
        assert np.array_equal(sb.label_result.ev_kind.cpu().numpy()[:off[n]], want["ev_kind"])
        print("fuzz_ev", kind, "ok")


def case_fuzz():
    cs = core.synth_csets(TH).to_device(torch.device("cuda"))
    for kind in range(4):
        sb = core.fuzz_batch(np.arange(64), kind, P.FuzzConfig(), TH, cs, want_scripts=True)
        torch.cuda.synchronize()
        _, modes, nev, nrec = O.fuzz_label_batch(0, 64, kind, n_threads=2)
        lab = lab_np(sb.labels)
        assert np.array_equal(lab["mode"], modes) and np.array_equal(lab["n_events"], nev)
    print("fuzz ok")


def case_label():
    trajs = P.fuzz_many(range(48), P.SubtaskKind.Pick) + P.fuzz_many(range(48), P.SubtaskKind.Open)
    for f64 in (False, True):
        for group in (trajs[:48], trajs[48:]):
            rb, ec, cs, nc = core.pack_trajectories(group, force_f64=f64)
            res = core.label_records(rb, ec, cs, nc)
            core.emit_events(rb, res)
            torch.cuda.synchronize()
            assert (lab_np(res.labels)["status"] == 0).all()
    print("label ok")


def case_env():
    for n in (64, 160 * 148):  # 8-lane and 4-lane k_env_step mappings
        env = P.BatchedSubtaskEnv(n)
        seeds = torch.arange(n, dtype=torch.int64, device="cuda")
        env.reset(seeds=seeds, subtask=P.SubtaskKind.Place, config=P.FuzzConfig())
        acts = env.scripted_actions(1, 12)
        env.step(acts[:4])
        for k in range(4, 12):
            env.step(acts[k:k + 1])
        torch.cuda.synchronize()
    print("env ok")


def case_filter():
    spec = P.FilterSpec([P.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 0.5),
                         P.AllowRule("Pick", frozenset({"pick.f8_drop"}), 0.5)], quota_per_target=40)
    labs = [P.LabelRecord(episode_id=f"e{i:05d}", subtask="Pick",
                          mode_id="pick.s1_straightforward" if i % 3 else "pick.f8_drop",
                          success_once=True, success_at_end=False, target_id=f"t{i % 5}")
            for i in range(3000)]
    man = P.filter_labels(labs, spec)
    assert len(man.entries) == 200
    print("filter ok")


def case_validate():
    trajs = P.fuzz_many(range(40), P.SubtaskKind.Place)
    assert not [f for fs in model.validate_many(trajs) for f in fs if f.is_error]
    rb, _, _, _ = core.pack_trajectories(trajs)
    assert not [f for fs in model.validate_batch(rb, [t.header for t in trajs]) for f in fs if f.is_error]
    print("validate ok")


def case_predicates():
    tr = P.fuzz(3, P.SubtaskKind.Place)
    P.success_step(tr.records[0], tr.header, TH)
    P.j_max(tr.records[0].q_arm, tr.header.rest_arm)
    print("predicates ok")


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
