"""Golden validate() / check_valid() fixtures from the REFERENCE
(model.py:232-288):

    python tests/golden/make_validate_golden.py

validate.json.gz: crafted trajectories (header dict + records) broken in
every way model.validate checks -- negative / NaN / decreasing
cum_robot_force, negative or NaN dist_ee_rest, negative dist_obj_goal and
force_ee_target, art_q outside its bounds, wrong step indices, short arm
vectors, bad headers -- and the reference's findings (severity, message)
plus its check_valid message.  Case family "f32": every value is binary32
(so the same case also runs through f32 device planes); "f64": arbitrary
doubles (-0.0, subnormals, 1e-300).
"""
import gzip
import json
import math
import os
import random
import struct
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import trajlab as T  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "validate.json.gz")
NAN = float("nan")


def f32(x):
    return struct.unpack("<f", struct.pack("<f", x))[0]


def make_case(rng, family):
    q = (lambda x: f32(x)) if family == "f32" else (lambda x: x)
    kind = rng.choice(list(T.SubtaskKind))
    art = rng.choice(["None", "Fridge", "Drawer"])
    dof = rng.choice([7, 7, 7, 3])
    qmin, qmax = (0.0, 1.6) if art == "Fridge" else (0.0, 0.5)
    hkw = dict(episode_id=f"v{rng.randrange(10**6)}", subtask_kind=kind.value,
               articulation_kind=art, arm_dof=dof)
    if art != "None":
        hkw.update(art_qmin=qmin, art_qmax=qmax)
        if rng.random() < 0.05:
            hkw.update(art_qmin=qmax, art_qmax=qmin)   # bounds invalid
    if rng.random() < 0.03:
        hkw["rest_arm"] = tuple([0.0] * (dof + 1))   # rest_arm length
    hdr = T.TrajectoryHeader(**hkw)
    n = rng.choice([0, 1, 2, 5, 31, 32, 33, 64, 65, 97, 130])
    cum = 0.0
    recs = []
    p_bad = rng.choice([0.0, 0.01, 0.05, 0.2])
    for t in range(n):
        cum += q(abs(rng.gauss(0, 1)))
        cum = q(cum)
        # (arm vectors and base velocities are not checked by validate)
        r = dict(t=t, q_arm=(0.0,) * dof, qd_arm=(0.0,) * dof,
                 q_tor=0.0, v_base_x=0.0, v_base_y=0.0, omega_base=0.0,
                 dist_ee_rest=q(rng.uniform(0, 1)),
                 dist_obj_goal=q(rng.uniform(0, 2)) if kind == T.SubtaskKind.Place else NAN,
                 force_ee_target=q(rng.uniform(0, 5)) if kind != T.SubtaskKind.Place else NAN,
                 cum_robot_force=cum,
                 art_q=q(rng.uniform(qmin, qmax)) if art != "None" else NAN,
                 grasped=rng.random() < 0.5)
        if rng.random() < p_bad:
            what = rng.choice(["cum_neg", "cum_nan", "cum_dec", "dee_neg", "dee_nan", "dog_neg",
                               "fet_neg", "art_out", "art_nan_bounds", "t", "arm", "zero"])
            if what == "cum_neg":
                r["cum_robot_force"] = q(-rng.uniform(0, 1))
            elif what == "cum_nan":
                r["cum_robot_force"] = NAN
            elif what == "cum_dec":
                r["cum_robot_force"] = q(cum * rng.uniform(0.1, 0.99))
            elif what == "dee_neg":
                r["dist_ee_rest"] = q(-rng.uniform(0, 1))
            elif what == "dee_nan":
                r["dist_ee_rest"] = NAN
            elif what == "dog_neg":
                r["dist_obj_goal"] = q(-rng.uniform(0, 1))
            elif what == "fet_neg":
                r["force_ee_target"] = q(-rng.uniform(0, 1))
            elif what == "art_out":
                r["art_q"] = q(rng.choice([qmin - 0.01, qmax + 0.01, -5.0]))
            elif what == "art_nan_bounds":
                r["art_q"] = NAN
            elif what == "t":
                r["t"] = t + rng.choice([-1, 1, 5])
            elif what == "arm" and family == "f64":
                r["q_arm"] = r["q_arm"][:-1]
            elif what == "zero":
                # exact boundaries: -0.0 is not < 0; the same cum is not a decrease
                r["dist_ee_rest"] = -0.0
                r["cum_robot_force"] = recs[-1]["cum_robot_force"] if recs else 0.0
                cum = r["cum_robot_force"]
        if family == "f64" and rng.random() < 0.02:
            r["cum_robot_force"] = rng.choice([-1e-300, -5e-324, 1e-300, cum + 1e-12])
        cum = r["cum_robot_force"] if not math.isnan(r["cum_robot_force"]) else cum
        if cum < 0:
            cum = 0.0
        recs.append(r)
    traj = T.Trajectory(hdr, [T.TimestepRecord(**r) for r in recs])
    findings = [[f.severity, f.message] for f in T.validate(traj)]
    try:
        T.check_valid(traj)
        cv = None
    except T.InvariantViolation as e:
        cv = str(e)
    return {"family": family, "header": hdr.to_dict(),
            "records": [dict(r, q_arm=list(r["q_arm"]), qd_arm=list(r["qd_arm"])) for r in recs],
            "findings": findings, "check_valid": cv}


def main():
    rng = random.Random(2412)
    cases = [make_case(rng, fam) for fam in ["f32"] * 300 + ["f64"] * 200]
    with gzip.GzipFile(OUT, "wb", mtime=0) as f:  # byte-reproducible
        f.write(json.dumps(cases).encode())
    n_f = sum(len(c["findings"]) for c in cases)
    print(f"wrote {len(cases)} cases, {n_f} findings")


if __name__ == "__main__":
    main()
