"""Line-delimited text interchange (format of trajlab.io_text, io_text.py):
line 1 {"header": {...}}, then one flat JSON object per record."""
from __future__ import annotations

import json

from .errors import ParseError
from .model import RECORD_FIELDS, TimestepRecord, Trajectory, TrajectoryHeader, check_valid


def write_text(traj: Trajectory) -> list:
    check_valid(traj)
    return ([json.dumps({"header": traj.header.to_dict()}, sort_keys=True)] +
            [json.dumps(r.to_dict(), sort_keys=True) for r in traj.records])


def _record(obj, line_no):
    missing = [f for f in RECORD_FIELDS if f not in obj]
    if missing:
        raise ParseError(f"record missing field(s) {missing}", line_no)
    try:
        fl = {f: float(obj[f]) for f in ("q_tor", "v_base_x", "v_base_y", "omega_base",
                                         "dist_ee_rest", "dist_obj_goal",
                                         "force_ee_target", "cum_robot_force", "art_q")}
        return TimestepRecord(t=int(obj["t"]),
                              q_arm=tuple(float(v) for v in obj["q_arm"]),
                              qd_arm=tuple(float(v) for v in obj["qd_arm"]),
                              grasped=bool(obj["grasped"]), **fl)
    except (TypeError, ValueError) as e:
        raise ParseError(f"bad record value: {e}", line_no) from e


def read_text(source) -> Trajectory:
    header, records, line_no = None, [], 0
    for raw in source:
        line_no += 1
        line = raw.strip()
        if not line:
            continue
        try:
            obj = json.loads(line)
        except ValueError as e:
            raise ParseError(f"invalid JSON: {e}", line_no) from e
        if header is None:
            if "header" not in obj:
                raise ParseError('first line must be {"header": {...}}', line_no)
            try:
                header = TrajectoryHeader.from_dict(obj["header"])
            except (KeyError, ValueError) as e:
                raise ParseError(f"bad header: {e}", line_no) from e
            continue
        records.append(_record(obj, line_no))
    if header is None:
        raise ParseError("empty stream, no header line", line_no or 1)
    return Trajectory(header=header, records=records)


def write_text_file(traj: Trajectory, path) -> None:
    with open(path, "w", encoding="utf-8") as f:
        for line in write_text(traj):
            f.write(line + "\n")


def read_text_file(path) -> Trajectory:
    with open(path, "r", encoding="utf-8") as f:
        return read_text(f)
