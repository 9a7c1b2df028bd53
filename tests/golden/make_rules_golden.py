"""Fixture: classify() with custom rule tables (modes.py:235-253 accepts any
(mode_id, predicate) table) -- relabelled / reordered builtin predicates
mixed with host callables, dropped catch-alls, empty tables.  Runs the
reference from /root/reference; writes rules.json.gz.
Usage: python tests/golden/make_rules_golden.py"""
import gzip
import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import trajlab as T  # noqa: E402
from trajlab.events import EVENT_ORDER  # noqa: E402
from trajlab.modes import MODE_RULES  # noqa: E402

from rule_recipes import build_table  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
KINDS = list(T.SubtaskKind)


def host_entry(rng, alpha):
    op = rng.choice(["size_ge", "has", "last_lt", "d0_none", "true", "false"])
    lab = f"custom.{op}.{rng.randrange(100)}"
    if op == "size_ge":
        return [op, rng.randrange(6), lab]
    if op == "has":
        return [op, rng.choice(alpha).value, lab]
    if op == "last_lt":
        return [op, rng.choice(alpha).value, rng.choice(alpha).value, lab]
    return [op, lab]


def recipe_for(rng, kind):
    alpha = list(EVENT_ORDER[kind])
    out = {}
    for br in ("success", "failure"):
        rows = [["b", m, m if rng.random() < 0.6 else "relabel." + m]
                for m, _ in MODE_RULES[kind][br]]
        if rng.random() < 0.3:
            rng.shuffle(rows)
        if br == "failure" and rng.random() < 0.2:
            rows = rows[:-1]  # no catch-all
        for _ in range(rng.choice([0, 0, 1, 2, 3])):
            rows.insert(rng.randrange(len(rows) + 1), host_entry(rng, alpha))
        if rng.random() < 0.1:  # a builtin predicate twice (first position wins)
            rows.append(list(rows[0])) if rows and rows[0][0] == "b" else None
        out[br] = rows
    return out


def main():
    rng = random.Random(23)
    cases = []
    for i in range(600):
        kind = KINDS[i % 4]
        alpha = list(EVENT_ORDER[kind])
        n = rng.choice([0, 1, 2, 3, 4, 5, 6, 8])
        kinds = [rng.choice(alpha) for _ in range(n)]
        d0 = rng.choice([None, 0.1, 0.5]) if kind == T.SubtaskKind.Place else None
        shape = rng.random()
        if shape < 0.05:
            recipe = {}  # `rules or MODE_RULES`: the builtin table
        elif shape < 0.08:
            other = KINDS[(i + 1) % 4]
            recipe = {other.value: recipe_for(rng, other)}  # KeyError
        else:
            recipe = {kind.value: recipe_for(rng, kind)}
        table = build_table(recipe, MODE_RULES, T.SubtaskKind, T.EventKind)
        evl = T.EventList(subtask_kind=kind, events=[T.Event(k, t + 1) for t, k in enumerate(kinds)],
                          initial_dist_obj_goal=d0)
        case = {"subtask": kind.value, "kinds": [k.value for k in kinds], "d0": d0, "recipe": recipe}
        try:
            lab = T.classify(evl, rules=table)
            case["result"] = [lab.mode_id, lab.success_once, lab.success_at_end]
        except (T.TrajlabError, TypeError, KeyError) as e:
            case["error"] = [type(e).__name__, str(e)]
        cases.append(case)
    with gzip.open(os.path.join(OUT, "rules.json.gz"), "wt") as f:
        json.dump(cases, f, indent=0)
    print(len(cases), "cases;", sum("error" in c for c in cases), "errors")


if __name__ == "__main__":
    main()
