"""GPU parity at the configurations bench.py ships, checked DIRECTLY against
the CPU oracle (oracle/oracle.c, pinned to the reference by
tests/test_oracle_golden.py) or the reference's own fixtures -- never device
against device.  Every label field the reference produces is compared:
mode, success_once / success_at_end, n_events, n_rec, d0 and the ordered
(kind, t) event lists (events.py:94-193, modes.py:235-253), plus records
bit-exact on a sample.  Reference acceptance loop: pkg/tests/test_acceptance.py:46-67.
Runs on a B200 (-m gpu)."""
import os

import numpy as np
import pytest

from golden_data import fuzz_corpus, from_oracle_records, npz, same_bits_f32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

THREADS = max(1, min(32, os.cpu_count() or 1))
LONG = dict(max_gap=64, max_tail=64)          # bench C2 / headline FuzzConfig


@pytest.fixture(scope="module")
def C():
    from paper_2412_13211_b200 import core
    return core


@pytest.fixture(scope="module")
def TH():
    from paper_2412_13211_b200.thresholds import Thresholds
    return Thresholds


def _labels(t):
    from paper_2412_13211_b200 import _lib as L
    return t.cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)


def _oracle(seed0, n, kind, cfg_kw):
    from oracle import oracle as O
    return O.fuzz_label_batch_full(seed0, n, kind, O.fuzz_cfg(**cfg_kw), n_threads=THREADS)


def _check_vs_oracle(lab, n_rec, ev_off, ev_kind, ev_t, want):
    """every label field + the CSR event lists, exact"""
    assert np.all(lab["status"] == 0), np.unique(lab["status"])
    assert np.array_equal(lab["mode"], want["mode"])
    assert np.array_equal(lab["flags"] & 3, want["flags"])
    assert np.array_equal(lab["n_events"], want["n_events"])
    assert np.array_equal(n_rec.astype(np.int64), want["n_rec"])
    d0 = lab["d0"]
    both_nan = np.isnan(d0) & np.isnan(want["d0"])
    assert np.all(both_nan | (d0 == want["d0"]))
    if ev_off is not None:
        assert np.array_equal(ev_off, want["ev_off"])
        tot = int(want["ev_off"][-1])
        assert np.array_equal(ev_kind[:tot], want["ev_kind"])
        assert np.array_equal(ev_t[:tot], want["ev_t"])


def _fuzz_ev(C, TH, seeds, kind, cfg):
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    sb = C.fuzz_batch(np.asarray(seeds, np.int64), kind, cfg, TH(), cs, events=True)
    r = sb.label_result
    return (sb, _labels(sb.labels), sb.records.n_rec.cpu().numpy(), r.ev_off.cpu().numpy(),
            r.ev_kind.cpu().numpy(), r.ev_t.cpu().numpy())


@pytest.mark.parametrize("kind", range(4))
def test_fuzz_ev_lists_vs_reference_fixtures(C, TH, kind):
    """tl_fuzz_ev (the bench's fused path: reset + realize + labels + ordered
    event lists in one launch pair) over the 406 fixture seeds of each
    subtask (incl. seeds >= 2^32) == the reference's own fuzz + extract_events
    + classify output (tests/golden/fuzz.npz)."""
    from paper_2412_13211_b200.synth import FuzzConfig
    c = fuzz_corpus(kind)
    seeds = npz("fuzz")["seeds"]
    _, lab, nrec, off, ek, et = _fuzz_ev(C, TH, seeds, kind, FuzzConfig())
    assert np.array_equal(nrec, np.diff(c.rec_off))
    assert np.array_equal(off, c.ev_off - c.ev_off[0])
    tot = int(off[-1])
    assert np.array_equal(ek[:tot], c.ev_kind)
    assert np.array_equal(et[:tot], c.ev_t)
    assert np.array_equal(lab["mode"], c.mode)
    assert np.array_equal(lab["flags"] & 1, c.success_once)
    assert np.array_equal((lab["flags"] >> 1) & 1, c.success_at_end)


@pytest.mark.parametrize("kind", range(4))
@pytest.mark.parametrize("cfg_name", ["default", "long"])
@pytest.mark.parametrize("n", [1000, 4096, 12000])
def test_shipped_fuzz_configs_vs_oracle(C, TH, kind, cfg_name, n):
    """The bench's workloads (headline: Place, max_gap=max_tail=64, 4096
    envs; C2 at 1024; C3 Open/Close default FuzzConfig at 4096) and the
    batch sizes that select every product launch shape of the reset
    (1 / 4 / 8 episodes per warp: <= 8, <= 64, > 64 episodes per SM) and of
    the realize kernel (2-warp CTAs when an episode fits 64 records
    [default config], 3-warp otherwise [long]) -- all label fields and the
    event lists against the oracle, records bit-exact on every 61st seed."""
    from oracle import oracle as O
    from paper_2412_13211_b200.synth import FuzzConfig
    kw = LONG if cfg_name == "long" else {}
    seed0 = 1_000_003 * (kind + 1) + n
    sb, lab, nrec, off, ek, et = _fuzz_ev(C, TH, np.arange(seed0, seed0 + n), kind, FuzzConfig(**kw))
    want = _oracle(seed0, n, kind, kw)
    _check_vs_oracle(lab, nrec, off, ek, et, want)
    planes = sb.records.planes.cpu().numpy()
    rs = sb.records.rec_start.cpu().numpy()
    for i in range(0, n, 61):
        _, recs = O.fuzz(seed0 + i, kind, O.fuzz_cfg(**kw))
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(planes[:, rs[i]:rs[i] + len(recs)], p), i


@pytest.mark.parametrize("kind", range(4))
def test_fuzz_10k_events_vs_oracle(C, TH, kind):
    """acceptance criterion 2 scale (seeds 0..9999, default FuzzConfig)
    including the event lists (kinds and times), not only modes / counts."""
    from paper_2412_13211_b200.synth import FuzzConfig
    n = 10000
    _, lab, nrec, off, ek, et = _fuzz_ev(C, TH, np.arange(n), kind, FuzzConfig())
    _check_vs_oracle(lab, nrec, off, ek, et, _oracle(0, n, kind, {}))


def test_label_kernel_grid_stride_2e20_vs_oracle(C, TH):
    """k_label's grid-stride loop (engaged above 148 x 128 x 8 = 151,552
    episodes) over 2^20 fuzz episodes of every subtask: tl_label_records on
    the generated records == the oracle's modes / flags / event counts."""
    from paper_2412_13211_b200.synth import FuzzConfig
    from paper_2412_13211_b200 import _lib as L
    n = 1 << 20
    cfg = FuzzConfig()
    cs = C.synth_csets(TH()).to_device(torch.device("cuda"))
    assert n > L.lib().tl_device_sm_count() * 128 * 8
    for kind in range(4):
        seed0 = 7 * 10 ** 7 * (kind + 1)
        sb = C.fuzz_batch(np.arange(seed0, seed0 + n), kind, cfg, TH(), cs, want_scripts=True)
        art = sb.scripts.cpu().numpy().reshape(-1).view(L.SCRIPT_DTYPE)["art_kind"]
        env = torch.from_numpy((3 * kind + art).astype(np.int32)).to("cuda")
        res = C.label_records(sb.records, env, cs, 12, want_events=False)
        lab = res.labels_np()
        want = _oracle(seed0, n, kind, {})
        assert np.all(lab["status"] == 0)
        assert np.array_equal(lab["mode"], want["mode"])
        assert np.array_equal(lab["flags"] & 3, want["flags"])
        assert np.array_equal(lab["n_events"], want["n_events"])
        del sb, res
        torch.cuda.empty_cache()


@pytest.mark.parametrize("kind", range(4))
def test_env_step_4lane_20480_vs_oracle(kind):
    """BatchedSubtaskEnv at 20,480 envs (k_env_step<7,4>: the 4-lanes-per-env
    form selected above 18,944 envs) replaying fuzz action streams: labels,
    record counts and every record bit-exact against the oracle's fuzz;
    step-mask events equal the oracle's event lists."""
    import paper_2412_13211_b200 as P
    from oracle import oracle as O
    from paper_2412_13211_b200 import _lib as L
    n = 20480
    assert n * 8 > L.lib().tl_device_sm_count() * 1024   # the 4-lane form
    seed0 = 555_000 + kind * n
    env = P.BatchedSubtaskEnv(n)
    cfg = P.FuzzConfig()
    r0 = env.reset(seeds=np.arange(seed0, seed0 + n), subtask=P.SubtaskKind(("Pick", "Place", "Open", "Close")[kind]),
                   config=cfg)
    T = int(env.script_lengths().max())
    st = env.step(env.scripted_actions(1, T - 1))
    lab, nrec = env.labels()
    want = _oracle(seed0, n, kind, {})
    _check_vs_oracle(lab, nrec, None, None, None, want)
    obs = torch.cat([r0.obs, st.obs], dim=1)                  # [F, T, N]
    masks = torch.cat([r0.step_mask, st.step_mask], dim=0)    # [T, N]
    from paper_2412_13211_b200.events import EVENT_KINDS, EVENT_ORDER
    from paper_2412_13211_b200.model import SUBTASK_ORDER
    alpha = np.array([EVENT_KINDS.index(k) for k in EVENT_ORDER[SUBTASK_ORDER[kind]]])
    m = masks.cpu().numpy()
    for e in range(0, n, 37):
        k = int(nrec[e])
        a, b = want["ev_off"][e], want["ev_off"][e + 1]
        ts, bits = np.nonzero(((m[:k, e, None].astype(np.int32) >> np.arange(7)) & 1))
        assert np.array_equal(ts, want["ev_t"][a:b]), e
        assert np.array_equal(alpha[bits], want["ev_kind"][a:b]), e
    o = obs[:, :, ::97].cpu().numpy()
    for j, e in enumerate(range(0, n, 97)):
        _, recs = O.fuzz(seed0 + e, kind)
        p, _ = from_oracle_records(O, recs)
        assert same_bits_f32(o[:, :len(recs), j], p), e


def test_c5_bench_scale_filter_vs_oracle():
    """C5 exactly as bench.py runs it: 4 x 250k fuzz episodes (default
    FuzzConfig) -> labels -> filter_labels with the A.6.1 recipe, quota 1000
    per target_id = seed % 9 -- the selected episode set, per-pool counts and
    shortfalls against the oracle's labels fed through the oracle's
    restatement of the selection loop (pipeline.py:276-338)."""
    import paper_2412_13211_b200 as P
    from oracle import oracle as O
    from paper_2412_13211_b200 import dist as D
    from paper_2412_13211_b200.modes import MODE_LIST
    n = 250_000
    spec = P.FilterSpec(allow=[
        P.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0),
        P.AllowRule("Place", frozenset({"place.s1_place_in_goal"}), 0.5),
        P.AllowRule("Place", frozenset({"place.s2_drop_to_goal"}), 0.5),
        P.AllowRule("Open", frozenset({"open.s1_open"}), 1.0),
        P.AllowRule("Close", frozenset({"close.s1_close"}), 1.0)], quota_per_target=1000)
    labels, man, names = D.fuzz_label_filter_sharded(n, spec)
    got = man.selected_rows()
    subs = ("Pick", "Place", "Open", "Close")
    rules_by = {}
    for r in spec.allow:
        rules_by.setdefault(r.subtask, []).append(r)
    pools = sorted((names[k], s) for k in range(9) for s in rules_by)
    pidx = {p: j for j, p in enumerate(pools)}
    pool, sub, rule = [], [], []
    rule_w = np.zeros(64)
    n_rules = np.zeros(4, np.int32)
    for s, name in enumerate(subs):
        n_rules[s] = len(rules_by[name])
        for p, r in enumerate(rules_by[name]):
            rule_w[s * 16 + p] = r.weight
    for s, name in enumerate(subs):
        want = O.fuzz_label_batch(0, n, s, n_threads=THREADS)[1]
        dev_modes = labels.view(-1, 24)[s * n:(s + 1) * n].cpu().numpy().reshape(-1).view(
            np.dtype([("status", "<i4"), ("n_events", "<i4"), ("err", "<i4"), ("sub", "u1"),
                      ("mode", "u1"), ("flags", "u1"), ("pad", "u1"), ("d0", "<f8")]))["mode"]
        assert np.array_equal(dev_modes, want), name
        for seed in range(n):   # seeds in episode_id order within the subtask
            m = MODE_LIST[want[seed]]
            pos = next((p for p, r in enumerate(rules_by[name]) if m in r.modes), -1)
            pool.append(pidx[(names[seed % 9], name)] if pos >= 0 else 0)
            sub.append(s)
            rule.append(pos)
    sel, ps = O.filter_select(pool, sub, rule, len(pools), rule_w, n_rules, spec.quota_per_target)
    assert np.array_equal(got, np.nonzero(sel)[0])
    want_pools = [(p, int(c)) for p, c in zip(pools, ps) if c > 0]
    assert want_pools == list(zip(man.pools, man.pool_selected))
    assert man.shortfalls == [{"quota_key": k, "subtask": s, "requested": 1000, "selected": c,
                               "shortfall": 1000 - c} for (k, s), c in want_pools if c < 1000]
    assert int(sel.sum()) == sum(man.pool_selected)
