"""Structural validation on the GPU (k_validate / tl_validate_records) against
the reference's validate() and check_valid() (model.py:232-288): findings and
messages of 500 crafted broken trajectories (tests/golden/validate.json.gz,
made by make_validate_golden.py from the reference), through the host
object path (f64 planes), the device batch path (f32 planes), and the
generator self-check of the reference's tests (test_synth.py:50-53, :127-131)
over device fuzz batches at the bench size."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from golden_data import js  # noqa: E402

import paper_2412_13211_b200 as P  # noqa: E402
from paper_2412_13211_b200 import core, model  # noqa: E402


@pytest.fixture(scope="module")
def cases():
    return js("validate")


def _traj(c):
    h = P.TrajectoryHeader.from_dict(c["header"])
    recs = [P.TimestepRecord(**dict(r, q_arm=tuple(r["q_arm"]), qd_arm=tuple(r["qd_arm"])))
            for r in c["records"]]
    return P.Trajectory(h, recs)


def _pairs(findings):
    return [[f.severity, f.message] for f in findings]


def test_validate_host_objects_vs_reference(cases):
    for k, c in enumerate(cases):
        tr = _traj(c)
        assert _pairs(P.validate(tr)) == c["findings"], k
        if c["check_valid"] is None:
            P.check_valid(tr)
        else:
            with pytest.raises(P.InvariantViolation) as ei:
                P.check_valid(tr)
            assert str(ei.value) == c["check_valid"], k


def test_validate_many_one_launch_vs_reference(cases):
    got = model.validate_many([_traj(c) for c in cases])
    assert [_pairs(g) for g in got] == [c["findings"] for c in cases]


def test_validate_batch_f32_planes_vs_reference(cases):
    """The f32 family through device planes (pack_trajectories picks f32:
    every value is binary32), grouped by arm_dof; SoA step indices are
    implicit, so cases with a stored-t mismatch are left to the host path."""
    by_dof = {}
    for k, c in enumerate(cases):
        if c["family"] != "f32" or any("has step index" in m for _, m in c["findings"]):
            continue
        tr = _traj(c)
        if len(tr.header.rest_arm) != tr.header.arm_dof:
            continue
        by_dof.setdefault(tr.header.arm_dof, []).append((k, tr))
    n = 0
    for dof, items in by_dof.items():
        trajs = [t for _, t in items]
        rb, _, _, _ = core.pack_trajectories(trajs)
        assert rb.planes.dtype == torch.float32
        got = model.validate_batch(rb, [t.header for t in trajs])
        for (k, _), g in zip(items, got):
            assert _pairs(g) == cases[k]["findings"], k
            n += 1
    assert n >= 200


@pytest.mark.parametrize("kind", list(P.SubtaskKind))
def test_generator_self_check_device_batch(kind):
    """Every fuzz trajectory passes validate (reference test_synth.py:127-131),
    checked on the device batch the generator wrote (4096 episodes, the
    bench size), and the device batch findings equal the host-object path's."""
    from paper_2412_13211_b200 import synth as SY
    seeds = list(range(4096))
    k, cfg, sb = SY._fuzz_device(seeds, kind, P.FuzzConfig(max_gap=64, max_tail=64), None, True)
    scripts = SY._scripts_from_device(k, cfg, sb, seeds)
    headers = [SY._synth_header(s.episode_id, k, s.articulation_kind, 7) for s in scripts]
    found = model.validate_batch(sb.records, headers)
    assert not [f for fs in found for f in fs if f.is_error]
    host = model.validate_many(SY._to_trajectories(sb, headers)[:256])
    assert [_pairs(f) for f in host] == [_pairs(f) for f in found[:256]]


def test_validate_batch_detects_corruption_at_bench_scale():
    """Corrupt chosen records of a 4096-episode Place batch in place on the
    device: exactly those records are reported, with the reference's
    messages (cum decrease, NaN cum, negative dist_obj_goal)."""
    from paper_2412_13211_b200 import synth as SY
    seeds = list(range(10_000, 14_096))
    k, cfg, sb = SY._fuzz_device(seeds, P.SubtaskKind.Place, P.FuzzConfig(max_gap=64, max_tail=64), None, True)
    scripts = SY._scripts_from_device(k, cfg, sb, seeds)
    headers = [SY._synth_header(s.episode_id, k, s.articulation_kind, 7) for s in scripts]
    rb = sb.records
    rs = rb.rec_start.cpu().numpy()
    nr = rb.n_rec.cpu().numpy()
    F_CUM, F_DOG = 2 * 7 + 7, 2 * 7 + 5
    rng = np.random.default_rng(5)
    eps = rng.choice(4096, 40, replace=False)
    want = {}
    for j, e in enumerate(eps.tolist()):
        i = int(rng.integers(1, nr[e]))
        r = int(rs[e]) + i
        if j % 3 == 0:
            prev = float(rb.planes[F_CUM, r - 1])
            rb.planes[F_CUM, r] = prev - 1.0 if prev >= 1.0 else -0.5
            v = float(rb.planes[F_CUM, r])
            want[e] = (f"cumulative force decreased at t={i}" if v >= 0
                       else f"cumulative force invalid at t={i}: {v}")
        elif j % 3 == 1:
            rb.planes[F_CUM, r] = float("nan")
            want[e] = f"cumulative force invalid at t={i}: nan"
        else:
            rb.planes[F_DOG, r] = -0.25
            want[e] = f"dist_obj_goal negative at t={i}: -0.25"
    found = model.validate_batch(rb, headers)
    bad = {e: [f.message for f in fs if f.is_error] for e, fs in enumerate(found)}
    assert {e for e, m in bad.items() if m} == set(want)
    for e, msg in want.items():
        assert bad[e][0] == msg, e
