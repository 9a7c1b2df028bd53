"""Host-side mirrors that need no GPU: exception messages per status code
(byte-identical to the reference's, because label_batch prints them), the
filter's bucket encoding, data-model round trips, and TRJL I/O."""
import io
import json
import math

import numpy as np
import pytest

from golden_data import SUBTASKS, Corpus, js, npz, to_oracle_records
from oracle import oracle as O


def test_infeasible_messages_match_reference():
    from paper_2412_13211_b200.errors import infeasible_error
    LV = {"low": 0, "slight": 1, "open": 2, "high": 3, "closed": 4}
    n = 0
    for case in js("scripts"):
        if case["error"] is None or case["error"][0] != "InfeasibleScript":
            continue
        k = SUBTASKS.index(case["subtask"])
        sc = dict(subtask=k, kinds=[O.EVENT_KINDS.index(s[0]) for s in case["steps"]],
                  gaps=[s[1] for s in case["steps"]], tail=case["tail"],
                  initial_grasped=int(case["initial_grasped"]),
                  initial_contact=int(case["initial_contact"]),
                  initial_dist_obj_goal=case["initial_dist_obj_goal"],
                  initial_level=LV[case["initial_art_level"]],
                  art_kind=O.ART_KINDS.index(case["articulation_kind"]), arm_dof=7)
        with pytest.raises(O.OracleError) as ei:
            O.realize(sc, case["seed"], case["thresholds"])
        step = ei.value.step
        ev = case["steps"][step][0] if step >= 0 else None
        exc = infeasible_error(ei.value.code, case["subtask"], ev, case["initial_art_level"])
        assert [type(exc).__name__, str(exc)] == case["error"]
        n += 1
    assert n > 50


def test_label_error_messages_match_reference():
    from paper_2412_13211_b200.errors import label_error
    d = npz("crafted")
    for tag in ("f32_", "f64_"):
        c = Corpus(d, tag)
        fields = list(d["threshold_fields"])
        for i in range(c.n):
            if not d[tag + "err_type"][i]:
                continue
            th = dict(zip(fields, d[tag + "override"][i])) if d[tag + "has_override"][i] else None
            planes, g = c.records_np(i)
            recs = to_oracle_records(O, planes.astype(np.float64), g)
            h = O.header(int(c.subtask[i]), int(c.art_kind[i]), float(c.art_qmin[i]),
                         float(c.art_qmax[i]), 7, list(c.rest_arm[i]), float(c.rest_tor[i]))
            with pytest.raises(O.OracleError) as ei:
                O.extract_events(recs, h, th)
            exc = label_error(ei.value.code, SUBTASKS[int(c.subtask[i])])
            assert type(exc).__name__ == d[tag + "err_type"][i]
            assert str(exc) == d[tag + "err_msg"][i]


def test_filter_bucket_encoding_matches_reference_grouping():
    from paper_2412_13211_b200.pipeline import AllowRule, FilterSpec, LabelRecord, filter_buckets
    for case in js("filter")[:40]:
        spec = FilterSpec.from_dict(case["spec"])
        labels = [LabelRecord(episode_id=e, subtask=s, mode_id=m, success_once=False,
                              success_at_end=False, target_id=t, task=k, source=src)
                  for e, s, m, t, k, src in case["labels"]]
        order, bucket, pools, b0, w = filter_buckets(labels, spec)
        assert [labels[i].episode_id for i in order] == sorted(l.episode_id for l in labels)
        # oracle restatement of the greedy loop on the same encoding
        sub = [SUBTASKS.index(labels[i].subtask) for i in order]
        pool = np.zeros(len(order), np.int32)
        rule = np.full(len(order), -1, np.int32)
        for j, b in enumerate(bucket):
            if b >= 0:
                p = int(np.searchsorted(b0, b, side="right") - 1)
                pool[j], rule[j] = p, b - b0[p]
        rw = np.zeros(64)
        nr = np.zeros(4, np.int32)
        for p, (key, s) in enumerate(pools):
            si = SUBTASKS.index(s)
            nr[si] = b0[p + 1] - b0[p]
            rw[si * 16: si * 16 + nr[si]] = w[b0[p]:b0[p + 1]]
        sel, ps = O.filter_select(pool, sub, rule, len(pools), rw, nr, spec.quota_per_target)
        got = sorted(labels[order[j]].episode_id for j in range(len(order)) if sel[j])
        assert got == case["selected"]


def test_labelrecord_json_is_sort_keys_canonical():
    from paper_2412_13211_b200.pipeline import LabelRecord
    r = LabelRecord("e1", "Pick", "pick.s1_straightforward", True, True,
                    [{"kind": "Contact", "t": 3}], "obj", "Custom", "Other", "", "/x")
    d = json.loads(r.to_json())
    assert list(d) == sorted(d)
    assert LabelRecord.from_dict(d) == r


@pytest.mark.gpu  # the writers run check_valid, i.e. k_validate
def test_trjl_roundtrip_bit_exact():
    from paper_2412_13211_b200 import io_binary as B
    from paper_2412_13211_b200.model import TimestepRecord, Trajectory, TrajectoryHeader
    c = Corpus(npz("defining"))
    planes, g = c.records_np(0)
    recs = [TimestepRecord(t, tuple(map(float, planes[0:7, t])), tuple(map(float, planes[7:14, t])),
                           *map(float, planes[14:23, t]), bool(g[t])) for t in range(planes.shape[1])]
    traj = Trajectory(TrajectoryHeader(episode_id="x", subtask_kind="Pick"), recs)
    buf = io.BytesIO()
    n = B.write_binary(traj, buf)
    assert B.record_size(7) == 100
    again = B.read_binary(io.BytesIO(buf.getvalue()))
    assert again.records == traj.records and again.header == traj.header
    buf2 = io.BytesIO()
    B.write_binary(again, buf2)
    assert buf.getvalue() == buf2.getvalue() and n == len(buf.getvalue())
    from paper_2412_13211_b200.errors import BadMagic, TruncatedFile
    with pytest.raises(TruncatedFile):
        B.read_binary(io.BytesIO(buf.getvalue()[:60]))
    with pytest.raises(BadMagic):
        B.read_binary(io.BytesIO(b"XXXX" + buf.getvalue()[4:]))
