"""Golden realize() + labels for arm_dof != 7 from the REFERENCE
(synth.py:166-190 draws 2*dof+5 uniforms per moving record; predicates.py
j_max / is_static over dof joints):

    python tests/golden/make_dof_golden.py

dof.json.gz: for arm_dof in (1, 3, 8, 12, 16): random_script-like scripts
(all subtasks, defining scripts + fuzz scripts re-stamped with the dof),
the realize seed, the reference's records (f32 hex), events and mode, and a
nonzero-rest-posture variant labelled by the reference.
"""
import gzip
import json
import math
import os
import random
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import trajlab as T  # noqa: E402
from trajlab import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dof.json.gz")


def script_dict(s, seed):
    return {"subtask": s.subtask_kind.value, "steps": [[st.kind.value, st.gap] for st in s.steps],
            "tail": s.tail, "initial_grasped": s.initial_grasped,
            "initial_contact": s.initial_contact, "initial_dist_obj_goal": s.initial_dist_obj_goal,
            "initial_art_level": s.initial_art_level,
            "articulation_kind": s.articulation_kind.value, "arm_dof": s.arm_dof, "seed": seed}


def rec_hex(tr):
    vals = []
    for r in tr.records:
        vals.extend(r.q_arm)
        vals.extend(r.qd_arm)
        vals.extend([r.q_tor, r.v_base_x, r.v_base_y, r.omega_base, r.dist_ee_rest,
                     r.dist_obj_goal, r.force_ee_target, r.cum_robot_force, r.art_q,
                     1.0 if r.grasped else 0.0])
    return np.asarray(vals, np.float32).tobytes().hex()


cases = []
rng = random.Random(77)
for dof in (1, 3, 8, 12, 16):
    scripts = []
    for mode_id, s in synth.defining_scripts().items():
        s.arm_dof = dof
        scripts.append(s)
    for kind in T.SubtaskKind:
        for k in range(6):
            s = T.random_script(rng.randrange(10**6), kind, T.FuzzConfig(max_gap=12, max_tail=12))
            s.arm_dof = dof
            scripts.append(s)
    for s in scripts:
        seed = rng.randrange(2**31)
        tr = T.realize(s, seed)
        ev = T.extract_events(tr, T.Thresholds())
        lab = T.classify(ev)
        # nonzero rest posture: same records, header rest offsets
        tr.header.rest_arm = tuple(rng.uniform(-0.25, 0.25) for _ in range(dof))
        tr.header.rest_tor = rng.uniform(-0.05, 0.05)
        try:
            ev2 = T.extract_events(tr, T.Thresholds())
            lab2 = T.classify(ev2)
            rest = {"rest_arm": list(tr.header.rest_arm), "rest_tor": tr.header.rest_tor,
                    "events": [[e.kind.value, e.t] for e in ev2.events], "mode": lab2.mode_id}
        except T.TrajlabError as e:
            rest = {"rest_arm": list(tr.header.rest_arm), "rest_tor": tr.header.rest_tor,
                    "error": f"{type(e).__name__}: {e}"}
        cases.append({"script": script_dict(s, seed), "n_records": len(tr.records),
                      "records_f32_hex": rec_hex(tr),
                      "events": [[e.kind.value, e.t] for e in ev.events], "mode": lab.mode_id,
                      "rest": rest})
with gzip.open(OUT, "wt") as f:
    json.dump({"cases": cases}, f)
print("wrote", OUT, os.path.getsize(OUT), len(cases), "cases")
