"""Randomised labelling parity: record streams drawn around every predicate
boundary (directed-rounding neighbours of each threshold, NaNs, rest
offsets, missing articulations, 0/1/2-record episodes) labelled on the GPU
(both label paths, f32 and f64 planes) against the CPU oracle's
extract_events + classify, which is pinned to the reference's fixtures.
Runs on a B200 (-m gpu)."""
import math

import numpy as np
import pytest

from golden_data import DOF, to_oracle_records

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

F32 = np.float32


def _around(x, rng):
    """x, or one of its binary32 neighbours, or a nearby random value"""
    f = F32(x)
    c = rng.integers(0, 6)
    if c == 0:
        return float(f)
    if c == 1:
        return float(np.nextafter(f, F32(np.inf)))
    if c == 2:
        return float(np.nextafter(f, F32(-np.inf)))
    if c == 3:
        return float(x)
    return float(x * (1 + rng.uniform(-0.3, 0.3)))


def _episode(rng, sub, art, qmin, qmax, rest, rest_tor, n):
    lim = (5000.0, 7500.0, 10000.0, 10000.0)[sub]
    span = (qmax - qmin) if art else 1.0
    cuts = [0.75 * span + qmin, 0.9 * span + qmin, 0.01 * span + qmin, 0.1 * span + qmin,
            qmin, qmax, 0.3 * span + qmin] if art else [0.5]
    P = np.zeros((2 * DOF + 9, n))
    g = np.zeros(n, np.uint8)
    cum = 0.0
    prev = None
    for t in range(n):
        if prev is not None and rng.random() < 0.6:
            col = prev.copy()
            cum = col[2 * DOF + 7]
            if rng.random() < 0.3:   # cum keeps drifting (non-decreasing)
                cum = _around(min(cum + rng.uniform(0, lim * 0.05), lim * 1.1), rng)
                col[2 * DOF + 7] = cum
        else:
            col = np.zeros(2 * DOF + 9)
            still = rng.random() < 0.5
            for i in range(DOF):
                col[i] = rest[i] + (_around(rng.choice([0.2, 0.6, -0.2, -0.6]), rng)
                                    if rng.random() < 0.3 else rng.uniform(-0.1, 0.1))
                col[DOF + i] = 0.0 if still else _around(rng.choice([0.2, -0.2, 0.1]), rng)
            col[2 * DOF] = rest_tor + (_around(rng.choice([0.01, -0.01]), rng)
                                       if rng.random() < 0.5 else 0.0)
            for j in (1, 2):
                col[2 * DOF + j] = 0.0 if still else _around(rng.choice([0.05, -0.05]), rng)
            col[2 * DOF + 3] = 0.0 if still else _around(rng.choice([0.05, -0.05]), rng)
            col[2 * DOF + 4] = _around(rng.choice([0.05, 0.0, 0.5]), rng)
            col[2 * DOF + 5] = (_around(rng.choice([0.15, 0.3, 0.05]), rng) if sub == 1
                                else (math.nan if rng.random() < 0.9 else 0.2))
            col[2 * DOF + 6] = (math.nan if sub == 1 and rng.random() < 0.9 else
                                _around(rng.choice([1e-6, 0.0, 1.2]), rng))
            if rng.random() < 0.3:
                cum = _around(rng.choice([lim, lim * 0.9, lim * 1.05]), rng)
            else:
                cum = cum + rng.uniform(0, lim * 0.02)
            col[2 * DOF + 7] = cum
            col[2 * DOF + 8] = _around(float(rng.choice(cuts)), rng) if art else math.nan
            if rng.random() < 0.004:  # a NaN in a required channel
                col[2 * DOF + int(rng.choice([5, 6, 8]))] = math.nan
            g_t = rng.random() < 0.5
            prev = col
            g[t] = g_t
        if prev is not None and t > 0 and rng.random() < 0.6:
            g[t] = g[t - 1]
        P[:, t] = col
        prev = col
    return P, g


def _make(rng, n_ep):
    eps = []
    for _ in range(n_ep):
        sub = int(rng.integers(0, 4))
        art = 0
        qmin = qmax = math.nan
        if sub >= 2:
            art = int(rng.choice([1, 2, 1, 2, 0]))   # occasionally missing
            if art:
                qmin, qmax = (0.0, 1.6) if art == 1 else (0.0, 0.5)
        rest = [0.0] * DOF if rng.random() < 0.8 else list(rng.uniform(-0.2, 0.2, DOF))
        rest_tor = 0.0 if rng.random() < 0.8 else float(rng.uniform(-0.1, 0.1))
        n = int(rng.choice([0, 1, 2, 3, 5, 33, 64, 65, 127, 128, 129, 200]))
        P, g = _episode(rng, sub, art, qmin, qmax, rest, rest_tor, n)
        eps.append((sub, art, qmin, qmax, rest, rest_tor, P, g))
    return eps


def _oracle(eps, f32):
    from oracle import oracle as O
    out = []
    for sub, art, qmin, qmax, rest, rest_tor, P, g in eps:
        Pv = P.astype(F32).astype(np.float64) if f32 else P
        recs = to_oracle_records(O, Pv, g)
        hdr = O.header(sub, art, qmin, qmax, DOF, rest, rest_tor)
        try:
            ks, ts, d0 = O.extract_events(recs, hdr)
        except O.OracleError as e:
            out.append(("err", e.code, None, None))
            continue
        try:
            mode, so, se = O.classify(sub, ks, d0, d0_none=(sub != 1))
        except O.OracleError as e:
            out.append(("cls", e.code, list(ks), list(ts)))
            continue
        out.append(("ok", (mode, so, se), list(ks), list(ts)))
    return out


@pytest.mark.parametrize("f32,align", [(True, False), (True, True), (False, False)])
def test_random_boundary_records_match_oracle(f32, align):
    from paper_2412_13211_b200 import core as C
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.thresholds import Thresholds
    rng = np.random.default_rng(20241213 + 7 * f32 + align)
    eps = _make(rng, 1500)
    want = _oracle(eps, f32)
    dt = F32 if f32 else np.float64
    n = [P.shape[1] for *_, P, g in eps]
    slot = [((k + 3) & ~3) if align else k for k in n]
    starts = np.concatenate([[0], np.cumsum(slot)[:-1]]).astype(np.int64)
    R = max(int(sum(slot)), 4)
    planes = np.zeros((2 * DOF + 9, R), dt)
    gr = np.zeros(R, np.uint8)
    tab = C.CsetTable()
    env = np.zeros(len(eps), np.int32)
    for i, (sub, art, qmin, qmax, rest, rest_tor, P, g) in enumerate(eps):
        planes[:, starts[i]:starts[i] + n[i]] = P.astype(dt)
        gr[starts[i]:starts[i] + n[i]] = g
        env[i] = tab.add(sub, art, qmin, qmax, DOF, rest, rest_tor, Thresholds())
    dev = torch.device("cuda")
    rb = C.RecordBatch(torch.from_numpy(planes).to(dev), torch.from_numpy(gr).to(dev),
                       torch.from_numpy(starts).to(dev),
                       torch.from_numpy(np.asarray(n, np.int32)).to(dev), DOF)
    res = C.label_records(rb, torch.from_numpy(env).to(dev), tab.to_device(dev), len(tab))
    lab = res.labels_np()
    off = res.ev_off.cpu().numpy()
    ek, et = res.ev_kind.cpu().numpy(), res.ev_t.cpu().numpy()
    n_checked = {"ok": 0, "err": 0, "cls": 0}
    for i, w in enumerate(want):
        st = int(lab["status"][i])
        n_checked[w[0]] += 1
        if w[0] == "err":
            assert st == w[1], (i, st, w[1], eps[i][0], n[i])
            continue
        assert list(ek[off[i]:off[i + 1]]) == w[2], i
        assert list(et[off[i]:off[i + 1]]) == w[3], i
        if w[0] == "cls":
            assert st == w[1], (i, st, w[1])
            continue
        mode, so, se = w[1]
        assert st == 0 and lab["mode"][i] == mode, (i, st, lab["mode"][i], mode)
        assert bool(lab["flags"][i] & 1) == so and bool(lab["flags"][i] & 2) == se, i
    assert n_checked["ok"] > 300 and n_checked["err"] > 30, n_checked
