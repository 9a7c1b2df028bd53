"""Benchmark of the B200 hot path: batched env reset/step (random_script +
realize) fused with event labelling and mode classification, plus event
list emission (and, for N>1, the NCCL label all-gather + mode-histogram
all-reduce).

Workload (BASELINE.json configs[1], "C2"): Place skill, 1024 parallel envs
per GPU; each env runs one random-action rollout = fuzz(seed, Place,
FuzzConfig(max_gap=64, max_tail=64)) (~200 env steps); every bench step
uses fresh seeds.  Metric: env samples/sec (records generated + labelled
per second, whole job), with labelled trajectories/sec alongside.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ENV = 1024
KIND = 1  # Place
CFG = dict(max_events=8, max_gap=64, max_tail=64, edge_density=1.0, success_prob=0.5)
RECORD_BYTES = 93  # 23 f32 planes + 1 u8 grasped (dof 7), SURVEY 8(d)
LABEL_BYTES = 24
WORKLOAD = ("C2: Place, 1024 envs/GPU, random-action rollout per env = "
            "fuzz(seed, Place, FuzzConfig(max_gap=64, max_tail=64)) (~200 steps), "
            "fresh seeds every step; generation + events + modes (+ event lists)")
METRIC = "env samples/sec (SPS)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profile_traffic():
    """dram bytes/launch of k_synth from the committed ncu capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("k_synth_dram_bytes_per_launch"), d.get("k_synth_records_per_launch")
    except Exception:
        return None, None


def host_info():
    """The host the CPU baseline ran on (core count, CPU model, Python)."""
    import platform
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model, "python": platform.python_version()}


def cpu_baseline(seconds, n_threads=1):
    """CPU oracle (C restatement of the reference path) on a bounded sample."""
    from oracle import oracle as O
    cfg = O.fuzz_cfg(**{k: CFG[k] for k in ("max_events", "max_gap", "max_tail", "edge_density",
                                            "success_prob")})
    n, recs, t = 64, 0, 0.0
    seed = 10 ** 9
    while t < seconds:
        t0 = time.perf_counter()
        r, *_ = O.fuzz_label_batch(seed, n, KIND, cfg, n_threads=n_threads, want_outputs=False)
        t += time.perf_counter() - t0
        recs += r
        seed += n
        n = min(n * 2, 1 << 16)
    eps = seed - 10 ** 9
    return recs / t, eps / t, f"{eps} episodes ({recs} env steps) of the bench workload, {t:.1f} s"


def run_reference(args, rank, world):
    """--impl reference: the reference path's CPU implementation (the C
    oracle port, all host threads) on the same workload."""
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    cfg = O.fuzz_cfg(**{k: CFG[k] for k in ("max_events", "max_gap", "max_tail", "edge_density",
                                            "success_prob")})
    n_env = N_ENV * world
    for k in range(args.warmup):
        O.fuzz_label_batch(-(k + 1) * n_env - 10 ** 8, n_env, KIND, cfg, n_threads=cores, want_outputs=False)
    recs, t0 = 0, time.perf_counter()
    for k in range(args.steps):
        r, *_ = O.fuzz_label_batch(k * n_env, n_env, KIND, cfg, n_threads=cores, want_outputs=False)
        recs += r
    dt = time.perf_counter() - t0
    sps = recs / dt
    out = {"impl": "reference", "metric": METRIC, "value": sps, "unit": "env-steps/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "trajectories_per_sec": n_env * args.steps / dt,
           "config": {"workload": WORKLOAD, "envs_per_step": n_env},
           "cpu_baseline": {"value": sps, "unit": "env-steps/s", "cores": cores, "kind": "port",
                            "sample": f"{args.steps} steps x {n_env} episodes, oracle/oracle.c "
                                      "(C restatement of trajlab fuzz+extract_events+classify), "
                                      f"{cores} threads", "host": host_info()},
           "e2e": {"value": sps, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


LABEL_READ_BYTES = {"pick": 81.0, "place": 85.0, "open": 88.0, "close": 88.0}


def label_sizing_run(L, core, lib, dev, stream, flush, n_env=1 << 20, reps=5, subtask="pick"):
    """HBM roofline of the labelling kernel (SURVEY 8(d) sizing run): 2^20
    episodes x 200 steps (2.1e8 env steps, 19.3 GB of f32 planes), records
    resident in HBM (far larger than L2).  One 4096-episode tile of the
    subtask's success script respaced to 200 records (C1/C3 shapes: Pick /
    Place 3 events gap 60, Open / Close 4 events gap 45, tail 19; fridge and
    drawer alternate) is realized on the GPU and replicated; K1 reads only the
    fields the subtask's predicates need."""
    import ctypes
    import torch
    from paper_2412_13211_b200 import synth as SY
    from paper_2412_13211_b200.events import EventKind as E
    from paper_2412_13211_b200.model import ArticulationKind as A, SubtaskKind as SK
    from paper_2412_13211_b200.thresholds import Thresholds
    from paper_2412_13211_b200 import _lib
    tile = 4096
    T = 200
    plan = {"pick": (SK.Pick, [E.Contact, E.Grasped, E.Success], 60, {}),
            "place": (SK.Place, [E.ObjAtGoal, E.ReleasedAtGoal, E.Success], 60,
                      {"initial_grasped": True}),
            "open": (SK.Open, [E.Contact, E.SlightlyOpened, E.Opened, E.Success], 45, {}),
            "close": (SK.Close, [E.Contact, E.SlightlyClosed, E.Closed, E.Success], 45,
                      {"initial_art_level": "high"})}[subtask]
    kind, evs, gap, kw = plan
    scripts = []
    for i in range(tile):
        art = A.Fridge if i % 2 == 0 else A.Drawer
        scripts.append(SY.EventScript(subtask_kind=kind, steps=[SY.ScriptStep(k, gap) for k in evs],
                                      tail=19, articulation_kind=art, **kw))
    arr, kinds, gaps = SY._script_array(scripts, np.arange(tile))
    cs12 = core.synth_csets(Thresholds()).to_device(dev)
    sb = core.realize_batch(arr, kinds, gaps, Thresholds(), cs12)
    assert int(sb.records.n_rec.min()) == T and int(sb.records.n_rec.max()) == T
    R = n_env * T
    planes = torch.empty((23, R), dtype=torch.float32, device=dev)
    grasped = torch.empty(R, dtype=torch.uint8, device=dev)
    reps_n = n_env // tile
    planes.view(23, reps_n, tile * T).copy_(sb.records.planes[:, :tile * T].unsqueeze(1).expand(23, reps_n, tile * T))
    grasped.view(reps_n, tile * T).copy_(sb.records.grasped[:tile * T].unsqueeze(0).expand(reps_n, tile * T))
    s_idx = int(arr["subtask"][0])
    art_idx = torch.from_numpy(np.where(np.arange(tile) % 2 == 0, 1, 2).astype(np.int32))
    env_tile = s_idx * 3 + (art_idx if s_idx >= 2 else torch.zeros(tile, dtype=torch.int32))
    rec_start = torch.arange(n_env, dtype=torch.int64, device=dev) * T
    n_rec = torch.full((n_env,), T, dtype=torch.int32, device=dev)
    rb = core.RecordBatch(planes, grasped, rec_start, n_rec, 7)
    env = env_tile.to(dev).repeat(reps_n)                        # synth_csets index
    labels = torch.empty((n_env, 24), dtype=torch.uint8, device=dev)
    mask = torch.empty(R, dtype=torch.uint8, device=dev)
    rbc = rb.c()
    sp = ctypes.c_void_p(stream.cuda_stream)
    ms = []
    for k in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        L.check(lib.tl_label_records(ctypes.byref(rbc), n_env, L.ptr(env), L.ptr(cs12), 12, None,
                                     L.ptr(mask), None, L.ptr(labels), sp), "label")
        b.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(a.elapsed_time(b))
    lab = labels.cpu().numpy().reshape(-1).view(_lib.LABEL_DTYPE)
    want = {"pick": 0, "place": 9, "open": 21, "close": 30}[subtask]  # the s1 mode everywhere
    assert (lab["status"] == 0).all() and (lab["mode"] == want).all(), np.unique(lab["mode"])
    t = sum(ms) / len(ms) / 1e3
    # Pick: q 28 + qd 28 + v 8 + w 4 + dist_ee_rest 4 + cum 4 + force 4 + grasped 1
    read_b = LABEL_READ_BYTES[subtask] * R
    write_b = 1.0 * R + 24.0 * n_env
    hbm, _ = peaks()
    del planes, grasped, mask
    return {"kernel": "k_label<float,7> (tl_label_records)", "subtask": subtask, "episodes": n_env,
            "env_steps": R, "avg_launch_ms": 1e3 * t,
            "env_steps_per_s": R / t, "trajectories_per_s": n_env / t,
            "algorithmic_bytes_per_launch": read_b + write_b,
            "achieved_GBps": (read_b + write_b) / t / 1e9, "peak_GBps": hbm,
            "frac": (read_b + write_b) / t / 1e9 / hbm,
            "note": f"{LABEL_READ_BYTES[subtask]:.0f} B/env-step read ({subtask} fields) + 1 B step mask + 24 B/episode label"}


def env_api_run(dev, stream, n_env=4096, T=200, reps=10):
    """North-star env API: BatchedSubtaskEnv.reset(fuzz seeds,
    Place) + T scripted random-action steps per env, (a) one tl_env_step
    launch for all T steps, (b) T single-step launches (CUDA graph).
    Inputs resident; records + step masks written to HBM (93 + 1 B/env-step)."""
    import torch
    import paper_2412_13211_b200 as P
    kind = P.SubtaskKind.Place
    cfg = P.FuzzConfig(max_gap=64, max_tail=64)
    env = P.BatchedSubtaskEnv(n_env)
    seeds = torch.arange(n_env, dtype=torch.int64, device=dev) + 10_000_000
    buf0 = env._outputs(1, None)
    bufT = env._outputs(T, None)
    buf1 = [env._outputs(1, None) for _ in range(T)]
    env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
    acts = env.scripted_actions(1, T)
    records = int((acts != P.env.IDLE).sum()) + n_env

    def block():
        env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
        env.step(acts, out=bufT)

    def single():
        env.reset(seeds=seeds, subtask=kind, config=cfg, out=buf0)
        for k in range(T):
            env.step(acts[k:k + 1], out=buf1[k])

    res = {"api": "BatchedSubtaskEnv.reset(seeds, Place) + step(actions[K, N])",
           "kernels": "k_fuzz_reset + k_env_reset + k_env_step", "n_env": n_env,
           "steps": T, "env_steps": records}
    hbm, _ = peaks()
    for name, fn in (("one_launch", block), ("per_step_launch", single)):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps / 1e3
        res[name] = {"ms": 1e3 * t, "env_steps_per_s": records / t,
                     "achieved_GBps": records * 94.0 / t / 1e9, "frac_hbm": records * 94.0 / t / 1e9 / hbm}
    lab, nrec = env.labels()
    if not ((lab["status"] == 0).all() and int(nrec.sum()) == records):
        raise RuntimeError(f"env rollout check failed: statuses {np.unique(lab['status'])}, "
                           f"records {int(nrec.sum())} != {records}")
    res["note"] = ("records = env steps actually emitted (scripts end before T -> IDLE); "
                   "94 B/env-step written (93 B record + 1 B event mask)")
    return res


def c5_run(dev, stream, world, n_per_subtask=250_000, reps=3):
    """C5: 1M synthetic episodes (fuzz, 250k per subtask, default
    FuzzConfig) labelled, all-gathered in episode order (N>1) and filtered
    with the A.6.1 recipe, quota 1000 per target_id = seed % 9.
    Whole pipeline timed on the device (max over ranks); labels/s is the
    BASELINE 'labelled trajectories/sec'."""
    import torch
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200 import dist as D
    spec = P.FilterSpec(allow=[
        P.AllowRule("Pick", frozenset({"pick.s1_straightforward"}), 1.0),
        P.AllowRule("Place", frozenset({"place.s1_place_in_goal"}), 0.5),
        P.AllowRule("Place", frozenset({"place.s2_drop_to_goal"}), 0.5),
        P.AllowRule("Open", frozenset({"open.s1_open"}), 1.0),
        P.AllowRule("Close", frozenset({"close.s1_close"}), 1.0)], quota_per_target=1000)
    ms = []
    man = None
    for k in range(reps + 1):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        labels, man, _ = D.fuzz_label_filter_sharded(n_per_subtask, spec)
        b.record(stream)
        torch.cuda.synchronize()
        if k:
            ms.append(a.elapsed_time(b))
    t = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    t = float(t.item()) / 1e3
    n_total = 4 * n_per_subtask
    return {"workload": "C5: fuzz 4 x 250k episodes (default FuzzConfig) -> label -> "
                        "all-gather -> filter_labels (A.6.1 recipe, quota 1000/target)",
            "episodes": n_total, "n_gpus": world, "ms": 1e3 * t,
            "labelled_trajectories_per_s": n_total / t,
            "selected": int(sum(man.pool_selected)), "pools": len(man.pools),
            "timing": "CUDA events around the whole pipeline (incl. host glue), max over ranks"}


def fuzz_step_graph(dev, stream, n_env, kind, cfg):
    """One fused fuzz step (tl_fuzz_ev: reset + realize + labels + ordered
    event lists) on preallocated buffers, captured as a CUDA graph.  Returns
    (graph, seeds_buf, workspace)."""
    import ctypes
    import torch
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200 import core
    from paper_2412_13211_b200.thresholds import Thresholds
    lib = L.lib()
    cap = core.fuzz_capacity(cfg)
    ws = core.SynthWorkspace(n_env, cap)
    cs = core.synth_csets(Thresholds()).to_device(dev)
    th_c = core.thresholds_c(Thresholds())
    cfg_c = L.FuzzCfg_c(cfg.max_events, cfg.max_gap, cfg.max_tail, 0, cfg.edge_density,
                        cfg.success_prob)
    seeds_buf = torch.zeros(n_env, dtype=torch.int64, device=dev)
    ev_cap = 4 * n_env * cap
    bufs = dict(ev_off=torch.empty(n_env + 1, dtype=torch.int64, device=dev),
                ev_kind=torch.empty(ev_cap, dtype=torch.uint8, device=dev),
                ev_t=torch.empty(ev_cap, dtype=torch.int32, device=dev))
    rb_c = ws.records().c()

    def body(s):
        L.check(lib.tl_fuzz_ev(L.ptr(seeds_buf), n_env, kind, ctypes.byref(cfg_c),
                               ctypes.byref(th_c), L.ptr(cs), None, ctypes.byref(rb_c), cap,
                               None, None, None, L.ptr(ws.step_mask), L.ptr(ws.labels),
                               L.ptr(bufs["ev_off"]), L.ptr(bufs["ev_kind"]), L.ptr(bufs["ev_t"]),
                               ev_cap, L.ptr(ws.scratch), ctypes.c_void_p(s.cuda_stream)),
                "tl_fuzz_ev")
    body(stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        body(torch.cuda.current_stream())
    ws._keep = (cs, th_c, cfg_c, bufs, rb_c, seeds_buf)  # the graph reads these
    return g, seeds_buf, ws


def c3_run(dev, stream, world, flush, n_env=4096, reps=20):
    """C3: Open and Close (fridge / drawer 50/50 via choice,
    synth.py:374-376), 4096 envs per GPU each, fuzz(seed, kind) with fresh
    rank-disjoint seeds every batch, default FuzzConfig; generation + labels +
    ordered event lists (tl_fuzz_ev, one CUDA graph per batch), device-timed
    per batch with L2 flushed between batches, max over ranks."""
    import torch
    import paper_2412_13211_b200 as P
    rank = torch.distributed.get_rank() if world > 1 else 0
    cfg = P.FuzzConfig()
    out = {}
    for name, kind in (("open", 2), ("close", 3)):
        g, seeds_buf, ws = fuzz_step_graph(dev, stream, n_env, kind, cfg)
        ms, recs = [], 0
        for k in range(reps + 2):
            seeds_buf.copy_(torch.arange(n_env, dtype=torch.int64, device=dev)
                            + (k * world + rank) * n_env)
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            if k >= 2:
                ms.append(a.elapsed_time(b))
                recs += int(ws.n_rec.sum())
        t = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t = float(t.item()) / 1e3
        recs /= reps
        lab = ws.labels.cpu().numpy().reshape(-1).view(L_LABEL_DTYPE())
        out[name] = {"ms": 1e3 * t, "env_steps_per_s": recs * world / t,
                     "labelled_trajectories_per_s": n_env * world / t,
                     "mean_steps": recs / n_env, "failed": int((lab["status"] != 0).sum())}
        del g, ws
    out["workload"] = ("C3: fuzz(seed, Open|Close), 4096 envs/GPU each, default FuzzConfig, "
                       "fresh seeds per batch, generation + labels + ordered event lists "
                       "(tl_fuzz_ev, CUDA graph), L2 flushed between batches")
    return out


def L_LABEL_DTYPE():
    from paper_2412_13211_b200 import _lib
    return _lib.LABEL_DTYPE


def label_batch_files_run(n_files=1000):
    """File-level API (tests/test_acceptance.py C8 shape):
    label_batch over 1000 TRJL1 files of 200 Pick records each -- host
    ingestion (one numpy view per file) + one GPU labelling batch + LabelRecords.
    Wall clock (host work included), best of 3."""
    import tempfile
    import paper_2412_13211_b200 as P
    script = P.EventScript(P.SubtaskKind.Pick, [P.ScriptStep(P.EventKind.Contact, 60),
                                                P.ScriptStep(P.EventKind.Grasped, 60),
                                                P.ScriptStep(P.EventKind.Success, 60)], tail=19)
    trajs = P.realize_many([script] * n_files, list(range(n_files)))
    with tempfile.TemporaryDirectory() as d:
        paths = []
        for i, t in enumerate(trajs):
            t.header.episode_id = f"ep-{i:06d}"
            pth = os.path.join(d, f"{i:06d}.trjl")
            P.write_binary_file(t, pth)
            paths.append(pth)
        P.label_batch(paths[:16])
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            res = P.label_batch(paths)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
    assert len(res.labels) == n_files and not res.errors
    return {"workload": f"label_batch over {n_files} TRJL1 files x 200 records (Pick, C8 shape)",
            "seconds": best, "files_per_s": n_files / best,
            "env_steps_per_s": n_files * 200 / best,
            "reference_note": "the reference takes 0.83 s for this (BASELINE.md C8, 1 worker)"}


def c4_run(dev, stream, world, flush=None, n_chain=4096, reps=5):
    """C4: SetTable chains, 4096 per GPU; chain c runs Open,
    Pick, Place, Close twice with seeds 8c + k (k = 0..7); slot success =
    success_once; progressive_completion over the 16-slot settable plan
    (alive counts all-reduced over ranks).  One fused fuzz graph per subtask
    (both repetitions, 8192 episodes), then tl_chain_progress."""
    import torch
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.analytics import BUILTIN_PLANS
    rank = torch.distributed.get_rank() if world > 1 else 0
    plan = BUILTIN_PLANS["settable"]
    c0 = rank * n_chain
    cfg = P.FuzzConfig()
    order = {"Open": 0, "Pick": 1, "Place": 2, "Close": 3}   # k within a repetition
    sub_idx = {"Pick": 0, "Place": 1, "Open": 2, "Close": 3}
    chains = torch.arange(c0, c0 + n_chain, dtype=torch.int64, device=dev)
    subs = ["Open", "Pick", "Place", "Close"]
    graphs = []
    for si, sub in enumerate(subs):   # label rows [2n*si, 2n*(si+1)): rep 0 then rep 1
        g, seeds_buf, ws = fuzz_step_graph(dev, stream, 2 * n_chain, sub_idx[sub], cfg)
        seeds_buf.copy_(torch.cat([8 * chains + 4 * rep + order[sub] for rep in (0, 1)]))
        graphs.append((g, ws))
    slot_label = torch.full((n_chain, len(plan)), -1, dtype=torch.int64, device=dev)
    for j, slot in enumerate(plan.slots):
        if slot.auto_success:
            continue
        rep = 0 if j < 8 else 1
        slot_label[:, j] = (2 * subs.index(slot.subtask) + rep) * n_chain + \
            torch.arange(n_chain, device=dev)
    lab = torch.empty((4 * 2 * n_chain, 24), dtype=torch.uint8, device=dev)
    alive = torch.empty(len(plan), dtype=torch.int64, device=dev)
    ms = []
    for k in range(reps + 1):
        if flush is not None:
            flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for si, (g, ws) in enumerate(graphs):
            g.replay()
            lab[2 * n_chain * si:2 * n_chain * (si + 1)].copy_(ws.labels)
        L.check(L.lib().tl_chain_progress(L.ptr(lab), L.ptr(slot_label), n_chain, len(plan),
                                          L.ptr(alive), L.stream_ptr()), "chain")
        if world > 1:
            torch.distributed.all_reduce(alive)
        b.record(stream)
        torch.cuda.synchronize()
        if k:
            ms.append(a.elapsed_time(b))
    t = sum(ms) / len(ms) / 1e3
    curve = [100.0 * int(x) / (n_chain * world) for x in alive.cpu().tolist()]
    return {"workload": "C4: SetTable chains (settable plan, 16 slots), 4096 chains/GPU, "
                        "8 fuzz episodes per chain (seeds 8c+k), one fused fuzz graph per "
                        "subtask, progressive_completion",
            "chains_per_gpu": n_chain, "n_gpus": world, "ms": 1e3 * t,
            "chains_per_s": n_chain * world / t,
            "labelled_trajectories_per_s": 8 * n_chain * world / t,
            "progressive_completion": curve}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import ctypes
    import torch
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200 import core
    from paper_2412_13211_b200.synth import FuzzConfig
    from paper_2412_13211_b200.thresholds import Thresholds

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    lib = L.lib()
    cfg = FuzzConfig(**CFG)
    cap = core.fuzz_capacity(cfg)
    ws = core.SynthWorkspace(N_ENV, cap)
    cs = core.synth_csets(Thresholds()).to_device(dev)
    th_c = core.thresholds_c(Thresholds())
    cfg_c = L.FuzzCfg_c(cfg.max_events, cfg.max_gap, cfg.max_tail, 0, cfg.edge_density,
                        cfg.success_prob)
    K, W = args.steps, args.warmup
    # inputs resident in HBM: seeds of every step, rank-disjoint ranges
    all_seeds = (torch.arange(K + W, device=dev, dtype=torch.int64)[:, None] * world + rank) * N_ENV \
        + torch.arange(N_ENV, device=dev, dtype=torch.int64)[None, :]
    seeds_buf = torch.empty(N_ENV, dtype=torch.int64, device=dev)
    ev_cap = 4 * N_ENV * cap   # tl_fuzz_ev bound: <= 4 events per record
    ev_off = torch.empty(N_ENV + 1, dtype=torch.int64, device=dev)
    ev_kind = torch.empty(ev_cap, dtype=torch.uint8, device=dev)
    ev_t = torch.empty(ev_cap, dtype=torch.int32, device=dev)
    scan_scratch = torch.empty(max(16, lib.tl_scan_scratch_bytes(N_ENV)), dtype=torch.uint8, device=dev)
    hist = torch.zeros(L.N_MODES, dtype=torch.int64, device=dev)
    gathered = torch.empty((world, N_ENV, 24), dtype=torch.uint8, device=dev) if world > 1 else None
    rb = ws.records()
    rb_c = rb.c()
    stream = torch.cuda.Stream(device=dev)  # graphs need a non-default stream
    torch.cuda.set_stream(stream)

    def synth_only(s):
        # reset kernel + realize kernel; the realize kernel also builds the
        # ordered event lists (decoupled look-back over episodes)
        sp = ctypes.c_void_p(s.cuda_stream)
        L.check(lib.tl_fuzz_ev(L.ptr(seeds_buf), N_ENV, KIND, ctypes.byref(cfg_c),
                               ctypes.byref(th_c), L.ptr(cs), None, ctypes.byref(rb_c), cap,
                               None, None, None, L.ptr(ws.step_mask), L.ptr(ws.labels),
                               L.ptr(ev_off), L.ptr(ev_kind), L.ptr(ev_t), ev_cap,
                               L.ptr(ws.scratch), sp), "tl_fuzz_ev")

    def step_body(s):
        synth_only(s)

    launches_per_step = 2 + (1 if world > 1 else 0)  # reset, realize(+events) [, histogram]

    # warm-up (also sets kernel attributes before graph capture)
    seeds_buf.copy_(all_seeds[0])
    step_body(stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step_body(torch.cuda.current_stream())

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def collectives():
        # the one exchange step: all-gather the 24-byte labels
        # over NCCL; every rank then builds the global mode histogram from the
        # gathered labels itself (no second collective)
        if world > 1:
            dist.all_gather_into_tensor(gathered.view(-1), ws.labels.view(-1))
            L.check(lib.tl_mode_histogram(L.ptr(gathered), world * N_ENV, L.ptr(hist),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                    "hist")

    for k in range(W):
        seeds_buf.copy_(all_seeds[K + k])
        graph.replay()
        collectives()
    torch.cuda.synchronize()

    # ---- device-timed steps: inputs in HBM, L2 flushed between steps -------
    nrec_log = torch.empty((K, N_ENV), dtype=torch.int32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    gpu_id = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) if \
        os.environ.get("CUDA_VISIBLE_DEVICES") else local
    with ClockSampler(gpu_id) as clocks:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(K):
            ev[k][0].record(stream)
            seeds_buf.copy_(all_seeds[k])
            graph.replay()
            collectives()
            ev[k][1].record(stream)
            nrec_log[k].copy_(ws.n_rec)
            flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        step_ms = [a.elapsed_time(b) for a, b in ev]

        # ---- k_synth alone (roofline of the dominant kernel) ---------------
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            seeds_buf.copy_(all_seeds[k])
            kev[k][0].record(stream)
            synth_only(stream)
            kev[k][1].record(stream)
            flush.zero_()
        torch.cuda.synchronize()
        synth_ms = [a.elapsed_time(b) for a, b in kev]

        # ---- end to end through the C ABI with host buffers ---------------
        # E (headline): pinned host seeds -> GPU -> labels + event lists back
        # to pinned host memory; records stay in HBM (the rollout buffer).
        # E_records: additionally compacts the records and copies them back.
        host_seeds = all_seeds.cpu().pin_memory()
        comp_planes = torch.empty((23, N_ENV * cap), dtype=torch.float32, device=dev)
        comp_g = torch.empty(N_ENV * cap, dtype=torch.uint8, device=dev)
        comp_start = torch.empty(N_ENV + 1, dtype=torch.int64, device=dev)
        comp_nrec = torch.empty(N_ENV, dtype=torch.int32, device=dev)
        comp_c = L.Records_c(comp_planes.data_ptr(), comp_g.data_ptr(), comp_start.data_ptr(),
                             comp_nrec.data_ptr(), N_ENV * cap, 0, 7)
        h_planes = torch.empty((23, N_ENV * cap), dtype=torch.float32).pin_memory()
        h_g = torch.empty(N_ENV * cap, dtype=torch.uint8).pin_memory()
        h_labels = torch.empty((N_ENV, 24), dtype=torch.uint8).pin_memory()
        h_evoff = torch.empty(N_ENV + 1, dtype=torch.int64).pin_memory()
        h_evk = torch.empty(ev_cap, dtype=torch.uint8).pin_memory()
        h_evt = torch.empty(ev_cap, dtype=torch.int32).pin_memory()
        h_tot = torch.empty(2, dtype=torch.int64).pin_memory()
        K2 = max(1, min(K, 50))
        # single GPU: the realize kernel writes labels and ordered event lists
        # straight into pinned host memory (zero-copy over PCIe; UVA makes the
        # pinned buffers device-addressable), so a step needs one sync, not a
        # sync + sized copies.  N > 1 keeps device labels for the NCCL gather.
        graph_zc = None
        if world == 1:
            def synth_zc(s):
                sp = ctypes.c_void_p(s.cuda_stream)
                L.check(lib.tl_fuzz_ev(L.ptr(seeds_buf), N_ENV, KIND, ctypes.byref(cfg_c),
                                       ctypes.byref(th_c), L.ptr(cs), None, ctypes.byref(rb_c),
                                       cap, None, None, None, L.ptr(ws.step_mask),
                                       L.ptr(h_labels), L.ptr(h_evoff), L.ptr(h_evk),
                                       L.ptr(h_evt), ev_cap, L.ptr(ws.scratch), sp), "tl_fuzz_ev")
            synth_zc(stream)
            torch.cuda.synchronize()
            graph_zc = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_zc, stream=stream):
                synth_zc(torch.cuda.current_stream())

        def e2e_loop(with_records):
            ms, recs, h2d, d2h = [], 0, 0, 0
            for k in range(K2):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                seeds_buf.copy_(host_seeds[k], non_blocking=True)
                if graph_zc is not None and not with_records:
                    graph_zc.replay()   # labels + event lists land in pinned host memory
                    b.record(stream)
                    stream.synchronize()
                    ms.append(a.elapsed_time(b))
                    recs += int(nrec_log[k].sum())
                    NE = int(h_evoff[N_ENV])
                    h2d = N_ENV * 8
                    d2h = N_ENV * 24 + (N_ENV + 1) * 8 + NE * 5
                    flush.zero_()
                    continue
                graph.replay()
                collectives()
                sp = ctypes.c_void_p(stream.cuda_stream)
                h_labels.copy_(ws.labels, non_blocking=True)
                h_evoff.copy_(ev_off, non_blocking=True)
                if with_records:
                    L.check(lib.tl_scan_counts(L.ptr(ws.n_rec), N_ENV, L.ptr(comp_start),
                                               L.ptr(scan_scratch), sp), "scan")
                    L.check(lib.tl_compact_records(ctypes.byref(rb_c), N_ENV, L.ptr(comp_start),
                                                   ctypes.byref(comp_c), sp), "compact")
                    h_tot[0:1].copy_(comp_start[N_ENV:N_ENV + 1], non_blocking=True)
                stream.synchronize()  # sizes of the variable-length outputs
                NE = int(h_evoff[N_ENV])
                R = int(h_tot[0]) if with_records else 0
                h_evk[:NE].copy_(ev_kind[:NE], non_blocking=True)
                h_evt[:NE].copy_(ev_t[:NE], non_blocking=True)
                if with_records:
                    for p_ in range(23):
                        h_planes[p_, :R].copy_(comp_planes[p_, :R], non_blocking=True)
                    h_g[:R].copy_(comp_g[:R], non_blocking=True)
                b.record(stream)
                stream.synchronize()
                ms.append(a.elapsed_time(b))
                recs += int(nrec_log[k].sum())
                h2d = N_ENV * 8
                d2h = N_ENV * 24 + (N_ENV + 1) * 8 + NE * 5 + (R * RECORD_BYTES + 8 if with_records else 0)
                flush.zero_()
            return sum(ms) / 1e3, recs, h2d, d2h

        t_e2e, e2e_recs, h2d_b, d2h_b = e2e_loop(False)
        t_e2r, e2r_recs, _, d2h_rb = e2e_loop(True)
        # ---- sizing run: k_label over 2^19 x 200-step episodes
        sizing = label_sizing_run(L, core, lib, dev, stream, flush)
        env_api = env_api_run(dev, stream)
        c3 = c3_run(dev, stream, world, flush)
        c5 = c5_run(dev, stream, world)
        c4 = c4_run(dev, stream, world, flush)
        lbf = label_batch_files_run() if rank == 0 else None
    clk = clocks.summary()

    recs_per_step = nrec_log.sum(dim=1).to(torch.float64)
    total_recs = float(recs_per_step.sum().item())
    t_dev = sum(step_ms) / 1e3
    t_syn = sum(synth_ms) / 1e3
    tt = torch.tensor([t_dev, t_syn, t_e2e, t_e2r, total_recs, float(e2e_recs), float(e2r_recs)],
                      dtype=torch.float64, device=dev)
    if world > 1:
        mx = tt[:4].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tt[4:].clone()
        dist.all_reduce(sm)
        t_dev, t_syn, t_e2e, t_e2r = mx.tolist()
        total_recs, e2e_recs_all, e2r_recs_all = sm.tolist()
    else:
        e2e_recs_all, e2r_recs_all = float(e2e_recs), float(e2r_recs)
    if rank != 0:
        dist.destroy_process_group()
        return
    hbm_peak, peak_src = peaks()
    recs_per_launch = total_recs / world / K
    alg_bytes = recs_per_launch * RECORD_BYTES + N_ENV * LABEL_BYTES
    achieved = alg_bytes / (t_syn / K) / 1e9
    traffic_b, traffic_recs = profile_traffic()
    traffic = None
    if traffic_b and traffic_recs:
        traffic = traffic_b / traffic_recs * recs_per_launch
    cb_sps, cb_eps, cb_sample = cpu_baseline(args.cpu_seconds)
    sps = total_recs / t_dev
    out = {
        "metric": METRIC, "value": sps, "unit": "env-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * t_dev / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "storage": "f32 records",
        "data": "synthetic",
        "trajectories_per_sec": N_ENV * world * K / t_dev,
        "config": {"workload": WORKLOAD, "envs_per_gpu": N_ENV, "subtask": "Place",
                   "fuzz_config": CFG, "mean_steps_per_episode": recs_per_launch / N_ENV,
                   "parallelism": f"episodes sharded over {world} GPU(s), NCCL label all-gather",
                   "l2": "flushed between timed steps (256 MiB write, excluded from timing)",
                   "timing": "CUDA events per step on the launch stream, max over ranks",
                   "step": "1 CUDA graph: tl_fuzz_ev (reset kernel + realize kernel that also emits the ordered event lists)"
                           + (", then NCCL all_gather of labels + tl_mode_histogram of the gathered labels" if world > 1 else "")},
        "gpu_launches": launches_per_step * K,
        "roofline": {"kernel": "k_fuzz_reset + k_synth_cta (tl_fuzz_ev)", "bound": "hbm", "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": 1e3 * t_syn / K,
                     "note": "93 B/record + 24 B/episode written; MT19937 + f64 generation is "
                             "ALU/latency-bound, not HBM-bound (SURVEY 8(d))"},
        "e2e": {"value": e2e_recs_all / t_e2e, "unit": "env-steps/s",
                "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                "steps": K2, "note": "C-ABI calls with host buffers: pinned host seeds -> GPU "
                                      "(H2D copy), labels + ordered event lists written by the "
                                      "kernels into pinned host memory (zero-copy D2H) every "
                                      "step, one stream sync (records stay in HBM)",
                "with_records": {"value": e2r_recs_all / t_e2r, "unit": "env-steps/s",
                                 "d2h_bytes_per_step": d2h_rb,
                                 "note": "same, plus tl_compact_records + D2H of every "
                                         "generated record (93 B/env-step)"}},
        "label_sizing": sizing,
        "env_api": env_api,
        "c3": c3,
        "c5": c5,
        "c4": c4,
        "label_batch_files": lbf,
        "cpu_baseline": {"value": cb_sps, "unit": "env-steps/s", "cores": 1, "kind": "port",
                         "sample": cb_sample, "trajectories_per_sec": cb_eps,
                         "host": host_info()},
        "clocks": clk,
    }
    print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
