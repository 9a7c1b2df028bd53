"""Analytics rows: mode_table / ratio_report /
progressive_completion / independence_upper_bound against the reference's
own outputs (tests/golden/analytics.json.gz, make_analytics_golden.py) and
the reference unit-test KATs (tests/test_analytics.py,
tests/test_acceptance.py:84-186).  Host counting runs on CPU; the device
counting kernels (tl_group_mode_counts, tl_chain_progress) are -m gpu."""
import random

import numpy as np
import pytest

from golden_data import js

import paper_2412_13211_b200 as P
from paper_2412_13211_b200 import analytics as A
from paper_2412_13211_b200.modes import MODE_LIST


def _records(tuples):
    return [P.LabelRecord(episode_id=e, subtask=s, mode_id=m, success_once=so,
                          success_at_end=se, target_id=t, task=task, split=sp, policy_tag=pt)
            for e, s, m, so, se, t, task, sp, pt in tuples]


def _labels_from_counts(counts, subtask="Pick"):
    kind = P.SubtaskKind(subtask)
    out = []
    for m, n in counts.items():
        for _ in range(n):
            out.append(P.LabelRecord(episode_id=f"e{len(out):06d}", subtask=subtask,
                                     mode_id=m, success_once=m in P.SUCCESS_MODE_IDS[kind],
                                     success_at_end=m in P.SUCCESS_AT_END_MODES[kind]))
    return out


def test_round_half_away_matches_reference():
    for x, d, want in js("analytics")["rounding"]:
        assert A.round_half_away(x, d) == want, (x, d)


def test_mode_tables_match_reference():
    g = js("analytics")
    n_tables = 0
    for case in g["cases"]:
        recs = _records(case["labels"])
        for t in case["tables"]:
            grouping = P.PICK_COARSE if t["grouping"] == "pick-coarse" else None
            tab = A.mode_table(recs, group_by=tuple(t["group_by"]), grouping=grouping)
            assert tab.to_dict() == t["dict"]
            assert tab.to_markdown() == t["markdown"]
            assert tab.to_csv() == t["csv"]
            n_tables += 1
        for a, b, want in case["ratios"]:
            if isinstance(want, str):
                exc = {"BothZero": P.BothZero, "ZeroDivisionError": ZeroDivisionError}[want]
                with pytest.raises(exc):
                    A.ratio_report(recs, a, b)
            else:
                assert A.ratio_report(recs, a, b).to_dict() == want
    assert n_tables > 40


def test_chain_curves_match_reference():
    g = js("analytics")
    for c in g["chains"]:
        plan = A.BUILTIN_PLANS[c["plan"]]
        eps = [A.ChainEpisode(f"c{i}", s) for i, s in enumerate(c["slot_success"])]
        assert A.progressive_completion(eps, plan) == c["curve"]
    for b in g["bounds"]:
        assert A.independence_upper_bound(b["sor"], A.BUILTIN_PLANS[b["plan"]]) == b["bound"]


def test_reference_table_arithmetic_kats():
    """tests/test_acceptance.py:84-135 (criterion 3)."""
    counts = {"pick.s1_straightforward": 7063, "pick.s2_winding": 188,
              "pick.s3_success_then_drop": 0, "pick.s4_success_then_excessive_collisions": 982,
              "pick.f5_excessive_collisions": 1379, "pick.f6_mobility": 337,
              "pick.f7_cant_grasp": 40, "pick.f8_drop": 10, "pick.f9_too_slow": 0}
    row = A.mode_table(_labels_from_counts(counts)).to_dict()["rows"][0]
    assert abs(row["sor"] - 82.34) <= 0.02 and abs(row["saer"] - 72.52) <= 0.02
    assert abs(row["fr"] - 17.66) <= 0.02
    coarse = {"pick.s1_straightforward": 2946, "pick.f5_excessive_collisions": 3452,
              "pick.f7_cant_grasp": 2817, "pick.f6_mobility": 785}
    row3 = A.mode_table(_labels_from_counts(coarse), grouping=P.PICK_COARSE).to_dict()["rows"][0]
    assert (row3["modes"]["S-Once"], row3["modes"]["F-Col"], row3["modes"]["F-Grasp"],
            row3["modes"]["F-Other"]) == (29.46, 34.52, 28.17, 7.85)

    def ratio(a, b):
        labels = _labels_from_counts({"pick.s1_straightforward": a, "pick.s2_winding": b})
        return A.ratio_report(labels, "pick.s1_straightforward", "pick.s2_winding").text
    assert ratio(317, 100) == "3.17 : 1" and ratio(100, 222) == "1 : 2.22"


def test_reference_chaining_kats():
    """tests/test_acceptance.py:159-186 (criterion 5) and test_analytics.py."""
    plan = A.ChainPlan("p", [A.ChainSlot("Nav", auto_success=True), A.ChainSlot("Pick", "Pick"),
                             A.ChainSlot("Nav", auto_success=True), A.ChainSlot("Place", "Place")])
    assert A.independence_upper_bound({"Pick": 0.8, "Place": 0.5}, plan) == [100.0, 80.0, 80.0, 40.0]
    rng = random.Random(42)
    n = 100_000
    eps = [A.ChainEpisode(f"e{i}", [True, rng.random() < 0.8, True, rng.random() < 0.5])
           for i in range(n)]
    curve = A.progressive_completion(eps, plan)
    assert all(a >= b for a, b in zip(curve, curve[1:]))
    assert abs(curve[-1] - 40.0) <= 3 * 100.0 * (0.4 * 0.6 / n) ** 0.5
    assert [len(A.BUILTIN_PLANS[k]) for k in ("tidyhouse", "preparegroceries", "settable")] == [20, 12, 16]
    with pytest.raises(P.MissingRate):
        A.independence_upper_bound({"Pick": 0.5}, plan)
    with pytest.raises(P.EmptyInput):
        A.progressive_completion([], plan)
    with pytest.raises(ValueError):
        A.progressive_completion([A.ChainEpisode("x", [True])], plan)
    with pytest.raises(ValueError):
        A.ChainPlan("bad", [A.ChainSlot("Nav", "Pick", auto_success=True)])


def test_mode_table_errors():
    with pytest.raises(P.EmptyInput):
        A.mode_table([])
    with pytest.raises(ValueError):
        A.mode_table(_labels_from_counts({"pick.f6_mobility": 1}), group_by=("bogus",))
    with pytest.raises(P.BothZero):
        A.ratio_report(_labels_from_counts({"place.f7_didnt_grasp": 3}, "Place"),
                       "place.s1_place_in_goal", "place.s2_drop_to_goal")


# -- device counting --------------------------------------------------------------

def _device_labels(tuples):
    import torch
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.model import SUBTASK_ORDER
    lab = np.zeros(len(tuples), L.LABEL_DTYPE)
    for i, (e, s, m, so, se, *_rest) in enumerate(tuples):
        lab[i]["subtask"] = [k.value for k in SUBTASK_ORDER].index(s)
        lab[i]["mode"] = MODE_LIST.index(m)
        lab[i]["flags"] = (1 if so else 0) | (2 if se else 0)
        lab[i]["err_index"] = -1
    return torch.from_numpy(lab.view(np.uint8).reshape(-1, 24).copy()).cuda()


@pytest.mark.gpu
def test_device_mode_tables_match_reference():
    g = js("analytics")
    cols = {"target_id": 5, "task": 6, "split": 7, "policy_tag": 8}
    for case in g["cases"]:
        tuples = case["labels"]
        lab = _device_labels(tuples)
        keys = {}
        for k, j in cols.items():
            names = sorted({t[j] for t in tuples})
            keys[k] = (np.array([names.index(t[j]) for t in tuples], np.int32), names)
        batch = A.LabelBatch(lab, keys)
        for t in case["tables"]:
            grouping = P.PICK_COARSE if t["grouping"] == "pick-coarse" else None
            tab = A.mode_table(batch, group_by=tuple(t["group_by"]), grouping=grouping)
            assert tab.to_dict() == t["dict"]
            assert tab.to_csv() == t["csv"]
        for a, b, want in case["ratios"]:
            if not isinstance(want, str):
                assert A.ratio_report(batch, a, b).to_dict() == want


@pytest.mark.gpu
def test_device_chain_progress_matches_reference():
    import torch
    g = js("analytics")
    for c in g["chains"]:
        plan = A.BUILTIN_PLANS[c["plan"]]
        ss = np.array(c["slot_success"], bool)
        n, k = ss.shape
        # one label per (chain, bound slot); auto slots get -1 (their value is ignored)
        auto = np.array([s.auto_success for s in plan.slots])
        tuples, idx = [], np.full((n, k), -1, np.int64)
        for i in range(n):
            for j in range(k):
                if not auto[j]:
                    idx[i, j] = len(tuples)
                    m = "pick.s1_straightforward" if ss[i, j] else "pick.f6_mobility"
                    tuples.append((f"x{len(tuples)}", "Pick", m, bool(ss[i, j]), bool(ss[i, j])))
        lab = _device_labels(tuples)
        assert A.progressive_completion_labels(lab, torch.from_numpy(idx), plan) == c["curve"]
