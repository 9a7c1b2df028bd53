"""Per-call latency of the scalar drop-in predicates (one record per call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_13211_b200 as T
th = T.Thresholds()
rec = T.TimestepRecord(t=0, q_arm=(0.0,) * 7, qd_arm=(0.01,) * 7, q_tor=0.0, v_base_x=0.0,
                       v_base_y=0.0, omega_base=0.0, dist_ee_rest=0.1, dist_obj_goal=0.1,
                       force_ee_target=0.0, cum_robot_force=0.0, art_q=0.2, grasped=False)
hdr = T.TrajectoryHeader(episode_id="x", subtask_kind=T.SubtaskKind.Open, articulation_kind="Fridge",
                         art_qmin=0.0, art_qmax=1.6)
for f, args in (("is_static", (rec, th)), ("is_open", (0.2, hdr, th)), ("success_step", (rec, hdr, th))):
    fn = getattr(T, f)
    for _ in range(20):
        fn(*args)
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        fn(*args)
    print(f"{f}: {1e6 * (time.perf_counter() - t0) / n:.1f} us/call")

# the previous per-call path (trajectory pack: six H2D copies, three blocking reads)
from paper_2412_13211_b200 import core, predicates as PR  # noqa: E402


def _eval_pack(rec, hdr, th, subtask=None, a0=None):
    h = hdr
    t = T.Trajectory(header=T.TrajectoryHeader(
        episode_id="", subtask_kind=h.subtask_kind, articulation_kind=h.articulation_kind,
        art_qmin=h.art_qmin, art_qmax=h.art_qmax, arm_dof=h.arm_dof,
        rest_arm=h.rest_arm, rest_tor=h.rest_tor, thresholds_override=th), records=[rec])
    rb, env, cs, _ = core.pack_trajectories([t], th, force_f64=True)
    bits, errs, jmax = core.eval_predicates(rb, env, cs, None if a0 is None else [a0])
    return int(bits[0].item()), int(errs[0].item()), float(jmax[0].item())


PR._eval = _eval_pack
n = 200
t0 = time.perf_counter()
for _ in range(n):
    T.success_step(rec, hdr, th)
print(f"success_step via trajectory pack (previous path): {1e6 * (time.perf_counter() - t0) / n:.1f} us/call")
