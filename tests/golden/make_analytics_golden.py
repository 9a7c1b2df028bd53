"""Golden fixtures for the analytics rows, made by
running the REFERENCE trajlab.analytics (/root/reference/pkg/src, read-only):

    python tests/golden/make_analytics_golden.py

analytics.json.gz holds, per case, the label set (as compact tuples), the
reference's mode_table(...).to_dict() / to_markdown() / to_csv() for
several group_by / grouping choices, ratio_report texts, and
progressive_completion / independence_upper_bound curves.
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import trajlab as T  # noqa: E402
from trajlab import analytics as A  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "analytics.json.gz")
SUB = ("Pick", "Place", "Open", "Close")


def labels_case(rng, n, subtasks, n_targets=3):
    recs = []
    for i in range(n):
        sub = rng.choice(subtasks)
        kind = T.SubtaskKind(sub)
        modes = T.MODE_IDS[kind]
        # skewed mode mix so some modes are absent
        m = modes[min(int(rng.expovariate(0.6)), len(modes) - 1)]
        recs.append((f"e{i:06d}", sub, m, m in T.SUCCESS_MODE_IDS[kind],
                     m in T.SUCCESS_AT_END_MODES[kind], f"t{rng.randrange(n_targets)}",
                     rng.choice(["TidyHouse", "PrepareGroceries", "SetTable"]),
                     rng.choice(["train", "val"]), rng.choice(["rl", "il"])))
    return recs


def to_records(tuples):
    return [T.LabelRecord(episode_id=e, subtask=s, mode_id=m, success_once=so,
                          success_at_end=se, target_id=t, task=task, split=sp,
                          policy_tag=pt)
            for e, s, m, so, se, t, task, sp, pt in tuples]


def main():
    rng = random.Random(20241213)
    cases = []
    for ci in range(12):
        subtasks = SUB if ci % 3 else ("Pick",)
        tuples = labels_case(rng, rng.choice([1, 7, 50, 333, 2000]), subtasks)
        recs = to_records(tuples)
        tables = []
        for gb in (("subtask",), ("subtask", "target_id"), ("task", "split"),
                   ("policy_tag", "subtask", "split")):
            t = A.mode_table(recs, group_by=gb)
            tables.append({"group_by": list(gb), "grouping": None, "dict": t.to_dict(),
                           "markdown": t.to_markdown(), "csv": t.to_csv()})
        if subtasks == ("Pick",):
            t = A.mode_table(recs, grouping=T.PICK_COARSE)
            tables.append({"group_by": ["subtask"], "grouping": "pick-coarse",
                           "dict": t.to_dict(), "markdown": t.to_markdown(), "csv": t.to_csv()})
        ratios = []
        for _ in range(4):
            sub = T.SubtaskKind(rng.choice(subtasks))
            a, b = rng.sample(T.MODE_IDS[sub], 2)
            try:
                ratios.append([a, b, A.ratio_report(recs, a, b).to_dict()])
            except (T.BothZero, ZeroDivisionError) as e:   # a == 0 < b divides by a
                ratios.append([a, b, type(e).__name__])
        cases.append({"labels": tuples, "tables": tables, "ratios": ratios})
    chains = []
    for pname, plan in A.BUILTIN_PLANS.items():
        for n in (1, 10, 997):
            p_ok = rng.choice([0.3, 0.7, 0.95])
            eps = [[rng.random() < p_ok for _ in range(len(plan))] for _ in range(n)]
            curve = A.progressive_completion(
                [A.ChainEpisode(f"c{i}", s) for i, s in enumerate(eps)], plan)
            chains.append({"plan": pname, "slot_success": eps, "curve": curve})
    bounds = []
    for pname, plan in A.BUILTIN_PLANS.items():
        sor = {s: rng.random() for s in SUB}
        bounds.append({"plan": pname, "sor": sor,
                       "bound": A.independence_upper_bound(sor, plan)})
    rounding = [[x, d, A.round_half_away(x, d)] for x, d in
                [(2.675, 2), (0.005, 2), (1.0, 2), (70.635, 2), (0.125, 2), (99.995, 2),
                 (12.3456, 3), (0.5, 0), (1.5, 0), (2.5, 0), (-2.675, 2), (82.345, 2)]]
    with gzip.open(OUT, "wt") as f:
        json.dump({"cases": cases, "chains": chains, "bounds": bounds,
                   "rounding": rounding}, f)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
