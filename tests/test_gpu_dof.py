"""arm_dof != 7 (1, 3, 8, 12, 16): realize / env replay bit-exact and labels
(incl. nonzero rest postures) against the reference (tests/golden/dof.json.gz,
make_dof_golden.py).  Exercises the DOFMAX=16 kernel instantiations and the
runtime-dof paths of the DOFMAX=7 ones.  Runs on a B200 (-m gpu)."""
import numpy as np
import pytest

from golden_data import js, same_bits_f32

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _script(P, d):
    return P.EventScript(
        subtask_kind=P.SubtaskKind(d["subtask"]),
        steps=[P.ScriptStep(P.EventKind(k), int(g)) for k, g in d["steps"]],
        tail=d["tail"], initial_grasped=d["initial_grasped"],
        initial_contact=d["initial_contact"], initial_dist_obj_goal=d["initial_dist_obj_goal"],
        initial_art_level=d["initial_art_level"],
        articulation_kind=P.ArticulationKind(d["articulation_kind"]), arm_dof=d["arm_dof"])


def _flat(tr):
    vals = []
    for r in tr.records:
        vals.extend(r.q_arm)
        vals.extend(r.qd_arm)
        vals.extend([r.q_tor, r.v_base_x, r.v_base_y, r.omega_base, r.dist_ee_rest,
                     r.dist_obj_goal, r.force_ee_target, r.cum_robot_force, r.art_q,
                     1.0 if r.grasped else 0.0])
    return np.asarray(vals, np.float32)


def _by_dof():
    out = {}
    for c in js("dof")["cases"]:
        out.setdefault(c["script"]["arm_dof"], []).append(c)
    return out


@pytest.mark.parametrize("dof", [1, 3, 8, 12, 16])
def test_realize_and_labels_other_dof(dof):
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200.pipeline import label_trajectories
    cases = _by_dof()[dof]
    scripts = [_script(P, c["script"]) for c in cases]
    trajs = P.realize_many(scripts, [c["script"]["seed"] for c in cases])
    for c, tr in zip(cases, trajs):
        assert len(tr.records) == c["n_records"]
        want = np.frombuffer(bytes.fromhex(c["records_f32_hex"]), np.float32)
        assert same_bits_f32(_flat(tr), want), c["script"]
    labs = label_trajectories(trajs)
    for c, lab in zip(cases, labs):
        assert [[e["kind"], e["t"]] for e in lab.events] == c["events"]
        assert lab.mode_id == c["mode"]
    # nonzero rest posture (the f64 j_max / torso path)
    for c, tr in zip(cases, trajs):
        tr.header.rest_arm = tuple(c["rest"]["rest_arm"])
        tr.header.rest_tor = c["rest"]["rest_tor"]
    labs = label_trajectories(trajs)
    for c, lab in zip(cases, labs):
        if "error" in c["rest"]:
            assert isinstance(lab, BaseException)
            assert f"{type(lab).__name__}: {lab}" == c["rest"]["error"]
            continue
        assert [[e["kind"], e["t"]] for e in lab.events] == c["rest"]["events"]
        assert lab.mode_id == c["rest"]["mode"]


@pytest.mark.parametrize("dof", [3, 16])
def test_env_replay_other_dof(dof):
    import paper_2412_13211_b200 as P
    cases = _by_dof()[dof]
    scripts = [_script(P, c["script"]) for c in cases]
    env = P.BatchedSubtaskEnv(len(scripts), dof=dof)
    r0 = env.reset(scripts=scripts, seeds=[c["script"]["seed"] for c in cases])
    T = int(env.script_lengths().max())
    st = env.step(env.scripted_actions(1, T - 1))
    obs = torch.cat([r0.obs, st.obs], dim=1).cpu().numpy()
    gr = torch.cat([r0.grasped, st.grasped], dim=0).cpu().numpy().astype(np.float32)
    lab, nrec = env.labels()
    F = 2 * dof + 9
    for i, c in enumerate(cases):
        n = c["n_records"]
        assert nrec[i] == n
        got = np.concatenate([np.concatenate([obs[:, t, i], [gr[t, i]]]) for t in range(n)])
        want = np.frombuffer(bytes.fromhex(c["records_f32_hex"]), np.float32)
        assert got.shape[0] == n * (F + 1)
        assert same_bits_f32(got, want), i
        from paper_2412_13211_b200.modes import MODE_LIST
        assert MODE_LIST[lab["mode"][i]] == c["mode"], i
