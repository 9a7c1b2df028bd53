"""Benchmark of the B200 hot path: batched env reset/step (random_script +
realize) fused with event labelling, mode classification and ordered event
list emission (and, for N>1, the NCCL label all-gather + global mode
histogram).

Headline workload (BASELINE.json configs[1] "C2" rollouts at the north-star
size): Place skill, 4096 parallel envs PER GPU; each env runs one
random-action rollout = fuzz(seed, Place, FuzzConfig(max_gap=64,
max_tail=64)) (~175 env steps); every bench step uses fresh, rank-disjoint
seeds.  Metric: env samples/sec (records generated + labelled per second,
whole job), with labelled trajectories/sec alongside.  C2 at 1024 envs, C3
(Open/Close, 4096 envs/GPU), C4, C5, the env API and the label sizing run are
extra keys.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (one process per GPU, NCCL, 127.0.0.1).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ENV = 4096                 # envs per GPU (north star: >= 4096 per GPU)
KIND = 1                     # Place
CFG = dict(max_events=8, max_gap=64, max_tail=64, edge_density=1.0, success_prob=0.5)
RECORD_BYTES = 93            # 23 f32 planes + 1 u8 grasped (dof 7), SURVEY 8(d)
LABEL_BYTES = 24
METRIC = "env samples/sec (SPS)"
WORKLOAD = ("Place random-action rollouts, 4096 envs per GPU: every env runs "
            "fuzz(seed, Place, FuzzConfig(max_gap=64, max_tail=64)) (~175 env steps; the "
            "BASELINE C2 rollout at the north-star per-GPU size), fresh rank-disjoint seeds "
            "every step; generation + events + modes + ordered event lists")


def bench_config(world):
    """The config dict BOTH arms print (the driver compares them)."""
    return {"workload": WORKLOAD, "envs_per_gpu": N_ENV, "subtask": "Place",
            "fuzz_config": dict(CFG),
            "seeds": "step k, rank r: [(k*N + r)*4096, (k*N + r + 1)*4096)",
            "parallelism": f"episodes (seeds) sharded over {world} GPU(s); labels all-gathered "
                           "over NCCL when N > 1",
            "l2": "flushed between timed steps (256 MiB write, excluded from timing)"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-extras", action="store_true",
                    help="headline only (skip C2/C3/C4/C5/env/sizing side runs)")
    return ap.parse_args(argv)


# ---- multi-GPU plumbing (covered on CPU by tests/test_bench_dist.py) ----------
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_argv(n, argv, port):
    """torchrun command that re-runs this script with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__), *argv]


def maybe_self_launch(args, argv):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run.
    NCCL's init log (nranks) goes to stderr."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(launch_argv(args.gpus, argv, free_port()), env=env)


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def step_seeds(k, rank, world, n_env=N_ENV):
    """seeds of bench step k on rank r: contiguous, rank-disjoint, fresh per step"""
    return (k * world + rank) * n_env + np.arange(n_env, dtype=np.int64)


def max_over_ranks(values, world, device=None):
    """element-wise max over ranks (the timing rule: the slowest rank)"""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values, world, device=None):
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        torch.distributed.all_reduce(t)
    return t.tolist()


def gather_labels(local, out, world):
    """the one exchange step: rank-ordered all-gather of the
    24-byte labels (rank order = episode_id order)"""
    import torch
    if world == 1:
        out.copy_(local.view(out.shape))
        return out
    torch.distributed.all_gather_into_tensor(out.view(-1), local.reshape(-1))
    return out


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


def profile_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def latency_constants():
    """critical-path cycle costs measured by scripts/floor_probe.cu on a B200
    (profiles/r2_floor_probe.json)"""
    d = profile_json("r2_floor_probe.json")
    if d:
        return float(d["cycles_per_seed_step"]), float(d["cum_cycles_per_record"]), \
            "profiles/r2_floor_probe.json (scripts/floor_probe.cu)"
    return 20.0, 72.0, "round-1 estimates (DESIGN.md section 9)"


def host_info():
    """The host the CPU baselines ran on (core count, CPU model, Python)."""
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


def oracle_cfg():
    from oracle import oracle as O
    return O.fuzz_cfg(**{k: CFG[k] for k in ("max_events", "max_gap", "max_tail", "edge_density",
                                             "success_prob")})


def cpu_baseline(seconds, n_threads=1):
    """CPU oracle (C restatement of the reference path) on a bounded sample."""
    from oracle import oracle as O
    cfg = oracle_cfg()
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


# ---- the reference's own Python implementation (baseline/_ref) ----------------
def reference_path():
    """where the unmodified reference package is importable from: the offline
    install baseline/_ref (travels to the GPU box), else the source tree"""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isfile(os.path.join(p, "trajlab", "__init__.py")):
            return p
    return None


def _pyref_chunk(job):
    """Pool worker: the reference's fuzz -> extract_events -> classify over a
    seed chunk (what label_batch's workers do per trajectory,
    pipeline.py:75-94, 134-138)."""
    path, s0, s1 = job
    if path not in sys.path:
        sys.path.insert(0, path)
    import trajlab as T
    cfg = T.FuzzConfig(**{k: CFG[k] for k in ("max_events", "max_gap", "max_tail")})
    th = T.Thresholds()
    recs = 0
    for s in range(s0, s1):
        tr = T.fuzz(s, T.SubtaskKind.Place, cfg)
        T.classify(T.extract_events(tr, th))
        recs += len(tr.records)
    return recs


def python_reference_baseline(seconds=4.0):
    """SURVEY 8(d) CPU reference timing with the REAL reference (pure Python,
    baseline/_ref): (i) one core, generation (fuzz) and labelling
    (classify(extract_events(.))) timed separately; (ii) all cores,
    multiprocessing.Pool over contiguous seed chunks; (iii) the file path
    label_batch(paths, workers=os.cpu_count()) over TRJL1 files."""
    import multiprocessing
    import tempfile
    path = reference_path()
    if path is None:
        return {"unavailable": "reference package not installed in baseline/_ref"}
    if path not in sys.path:
        sys.path.insert(0, path)
    import trajlab as T
    cores = os.cpu_count() or 1
    cfg = T.FuzzConfig(**{k: CFG[k] for k in ("max_events", "max_gap", "max_tail")})
    th = T.Thresholds()
    # (i) single core, generation and labelling separately
    seed, recs, t_gen, t_lab, trajs = 2 * 10 ** 9, 0, 0.0, 0.0, []
    while t_gen + t_lab < seconds:
        t0 = time.perf_counter()
        tr = T.fuzz(seed, T.SubtaskKind.Place, cfg)
        t1 = time.perf_counter()
        T.classify(T.extract_events(tr, th))
        t2 = time.perf_counter()
        t_gen += t1 - t0
        t_lab += t2 - t1
        recs += len(tr.records)
        if len(trajs) < 1000:
            trajs.append(tr)
        seed += 1
    n1 = seed - 2 * 10 ** 9
    one = {"generate_sps": recs / t_gen, "label_sps": recs / t_lab,
           "fuzz_and_label_sps": recs / (t_gen + t_lab),
           "sample": f"{n1} episodes ({recs} env steps), one core, {t_gen + t_lab:.1f} s"}
    # (ii) all cores: Pool over contiguous seed chunks (label_batch's pattern)
    per_ep = (t_gen + t_lab) / n1
    chunk = max(1, int(seconds / per_ep / 4))
    jobs = [(path, 3 * 10 ** 9 + i * chunk, 3 * 10 ** 9 + (i + 1) * chunk) for i in range(4 * cores)]
    ctx = multiprocessing.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_pyref_chunk, [(path, 0, 1)] * cores)       # workers imported
        t0 = time.perf_counter()
        r = sum(pool.map(_pyref_chunk, jobs, chunksize=1))
        t_pool = time.perf_counter() - t0
    pool_d = {"fuzz_and_label_sps": r / t_pool, "workers": cores,
              "sample": f"{len(jobs) * chunk} episodes ({r} env steps), Pool({cores}), {t_pool:.1f} s"}
    # (iii) label_batch over TRJL1 files, all cores
    with tempfile.TemporaryDirectory() as d:
        paths = []
        frecs = 0
        for i, tr in enumerate(trajs):
            p = os.path.join(d, f"{i:06d}.trjl")
            T.write_binary_file(tr, p)
            paths.append(p)
            frecs += len(tr.records)
        t0 = time.perf_counter()
        res = T.label_batch(paths, workers=cores)
        t_lb = time.perf_counter() - t0
    lb = {"label_sps": frecs / t_lb, "workers": cores, "ok": res.ok,
          "sample": f"label_batch over {len(paths)} TRJL1 files ({frecs} env steps), {t_lb:.2f} s"}
    import platform
    return {"kind": "reference-python", "package": os.path.relpath(path, ROOT) if path.startswith(ROOT) else path,
            "single_core": one, "pool": pool_d, "label_batch": lb, "cores": cores,
            "python": platform.python_version(), "workload": "fuzz(seed, Place, FuzzConfig(max_gap=64, "
            "max_tail=64)) -> extract_events -> classify, seeds from 2e9 / 3e9"}


def run_reference(args, rank, world):
    """--impl reference: the reference path's CPU implementation (the C
    restatement oracle/oracle.c, all host threads) on the same workload, the
    same config and seeds as the GPU arm; plus the real Python reference timed
    beside it (python_reference)."""
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    cfg = oracle_cfg()
    n_env = N_ENV * world   # the whole job's episodes per step (weak scaling)
    for k in range(args.warmup):
        O.fuzz_label_batch(-(k + 1) * n_env - 10 ** 8, n_env, KIND, cfg, n_threads=cores, want_outputs=False)
    recs, t0 = 0, time.perf_counter()
    for k in range(args.steps):
        r, *_ = O.fuzz_label_batch(k * n_env, n_env, KIND, cfg, n_threads=cores, want_outputs=False)
        recs += r
    dt = time.perf_counter() - t0
    sps = recs / dt
    pyref = python_reference_baseline()
    out = {"impl": "reference", "metric": METRIC, "value": sps, "unit": "env-steps/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "trajectories_per_sec": n_env * args.steps / dt,
           "config": bench_config(world),
           "cpu_baseline": {"value": sps, "unit": "env-steps/s", "cores": cores, "kind": "port",
                            "sample": f"{args.steps} steps x {n_env} episodes, oracle/oracle.c "
                                      "(C restatement of trajlab fuzz+extract_events+classify), "
                                      f"{cores} threads", "host": host_info()},
           "python_reference": pyref,
           "e2e": {"value": sps, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


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
    t = max_over_ranks([sum(ms) / len(ms)], world, dev)[0] / 1e3
    n_total = 4 * n_per_subtask
    return {"workload": "C5: fuzz 4 x 250k episodes (default FuzzConfig) -> label -> "
                        "all-gather -> filter_labels (A.6.1 recipe, quota 1000/target)",
            "episodes": n_total, "n_gpus": world, "ms": 1e3 * t,
            "labelled_trajectories_per_s": n_total / t,
            "selected": int(sum(man.pool_selected)), "pools": len(man.pools),
            "timing": "CUDA events around the whole pipeline (incl. host glue), max over ranks",
            "parity": "tests/test_gpu_shipped.py::test_c5_bench_scale_filter_vs_oracle"}


def fuzz_step_graph(dev, stream, n_env, kind, cfg, host_out=None, io=None, seeds_host=None,
                    subtasks=None):
    """One fused fuzz step (tl_fuzz_ev: reset + realize + labels + ordered
    event lists) on preallocated buffers, captured as a CUDA graph.  host_out
    (pinned host tensors ev_off / ev_kind / ev_t, optionally labels): the
    kernel writes those outputs straight into host memory (zero-copy).
    io (pinned host tensors seeds [n] int64, labels [n, 24] u8): the graph
    also copies the seeds in (H2D) and the labels out (D2H), so one graph
    launch is the whole host-to-host step.
    seeds_host (pinned host int64 [n]): the reset kernel reads the seeds
    straight from host memory (zero-copy H2D inside the step).
    subtasks (device u8 [n]): a subtask per episode (tl_fuzz_ev_mixed; kind
    is then ignored).
    Returns (graph, seeds_buf, workspace, device event buffers)."""
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
    out = dict(bufs)
    out["labels"] = ws.labels
    if host_out:
        out.update(host_out)
    rb_c = ws.records().c()

    def body(s):
        if io is not None:
            seeds_buf.copy_(io["seeds"], non_blocking=True)
        sp = L.ptr(seeds_buf if seeds_host is None else seeds_host)
        head = (sp, L.ptr(subtasks), n_env) if subtasks is not None else (sp, n_env, kind)
        fn = lib.tl_fuzz_ev_mixed if subtasks is not None else lib.tl_fuzz_ev
        L.check(fn(*head, ctypes.byref(cfg_c),
                               ctypes.byref(th_c), L.ptr(cs), None, ctypes.byref(rb_c), cap,
                               None, None, None, L.ptr(ws.step_mask), L.ptr(out["labels"]),
                               L.ptr(out["ev_off"]), L.ptr(out["ev_kind"]), L.ptr(out["ev_t"]),
                               ev_cap, L.ptr(ws.scratch), ctypes.c_void_p(s.cuda_stream)),
                "tl_fuzz_ev")
        if io is not None:
            io["labels"].copy_(out["labels"], non_blocking=True)
    body(stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        body(torch.cuda.current_stream())
    ws._keep = (cs, th_c, cfg_c, bufs, rb_c, seeds_buf, out, seeds_host, subtasks)  # the graph reads these
    return g, seeds_buf, ws, bufs


def fuzz_batch_timed(dev, stream, world, flush, n_env, kind, cfg, reps):
    """device time per fuzz batch (graph replay, L2 flushed), max over ranks"""
    import torch
    rank = torch.distributed.get_rank() if world > 1 else 0
    g, seeds_buf, ws, _ = fuzz_step_graph(dev, stream, n_env, kind, cfg)
    ms, recs = [], 0
    for k in range(reps + 2):
        seeds_buf.copy_(torch.from_numpy(step_seeds(k + 7919, rank, world, n_env)).to(dev))
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(a.elapsed_time(b))
            recs += int(ws.n_rec.sum())
    t = max_over_ranks([sum(ms) / len(ms)], world, dev)[0] / 1e3
    recs = sum_over_ranks([recs / reps], world, dev)[0]
    lab = ws.labels.cpu().numpy().reshape(-1).view(L_LABEL_DTYPE())
    return {"ms": 1e3 * t, "env_steps_per_s": recs / t,
            "labelled_trajectories_per_s": n_env * world / t,
            "mean_steps": recs / (n_env * world), "failed": int((lab["status"] != 0).sum())}


def c3_run(dev, stream, world, flush, n_env=4096, reps=20):
    """C3: Open and Close (fridge / drawer 50/50 via choice,
    synth.py:374-376), 4096 envs per GPU each, fuzz(seed, kind) with fresh
    rank-disjoint seeds every batch, default FuzzConfig; generation + labels +
    ordered event lists (tl_fuzz_ev, one CUDA graph per batch), device-timed
    per batch with L2 flushed between batches, max over ranks."""
    import paper_2412_13211_b200 as P
    out = {name: fuzz_batch_timed(dev, stream, world, flush, n_env, kind, P.FuzzConfig(), reps)
           for name, kind in (("open", 2), ("close", 3))}
    out["workload"] = ("C3: fuzz(seed, Open|Close), 4096 envs/GPU each, default FuzzConfig, "
                       "fresh seeds per batch, generation + labels + ordered event lists "
                       "(tl_fuzz_ev, CUDA graph), L2 flushed between batches")
    return out


def c2_run(dev, stream, world, flush, reps=20):
    """BASELINE C2 exactly: Place, 1024 envs per GPU, max_gap = max_tail = 64"""
    import paper_2412_13211_b200 as P
    r = fuzz_batch_timed(dev, stream, world, flush, 1024, KIND, P.FuzzConfig(**CFG), reps)
    r["workload"] = ("C2: Place, 1024 envs/GPU, fuzz(seed, Place, FuzzConfig(max_gap=64, "
                     "max_tail=64)), tl_fuzz_ev CUDA graph, L2 flushed between batches")
    return r


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
    (alive counts all-reduced over ranks).  One fused fuzz graph over all
    8 episodes of every chain (tl_fuzz_ev_mixed: a subtask per episode,
    episode 8c + k), then tl_chain_progress."""
    import torch
    import paper_2412_13211_b200 as P
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200.analytics import BUILTIN_PLANS
    rank = torch.distributed.get_rank() if world > 1 else 0
    plan = BUILTIN_PLANS["settable"]
    c0 = rank * n_chain
    cfg = P.FuzzConfig()
    order = ["Open", "Pick", "Place", "Close"]   # k % 4 within a repetition (k // 4)
    sub_idx = {"Pick": 0, "Place": 1, "Open": 2, "Close": 3}
    ks = torch.arange(8, device=dev)
    subtasks = torch.tensor([sub_idx[order[k % 4]] for k in range(8)], dtype=torch.uint8,
                            device=dev).repeat(n_chain)
    g, seeds_buf, ws, _ = fuzz_step_graph(dev, stream, 8 * n_chain, 0, cfg, subtasks=subtasks)
    chains = torch.arange(c0, c0 + n_chain, dtype=torch.int64, device=dev)
    seeds_buf.copy_((8 * chains[:, None] + ks[None, :]).reshape(-1))
    slot_label = torch.full((n_chain, len(plan)), -1, dtype=torch.int64, device=dev)
    for j, slot in enumerate(plan.slots):
        if slot.auto_success:
            continue
        rep = 0 if j < 8 else 1
        slot_label[:, j] = 8 * torch.arange(n_chain, device=dev) + 4 * rep + order.index(slot.subtask)
    alive = torch.empty(len(plan), dtype=torch.int64, device=dev)
    ms = []
    for k in range(reps + 1):
        if flush is not None:
            flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        L.check(L.lib().tl_chain_progress(L.ptr(ws.labels), L.ptr(slot_label), n_chain, len(plan),
                                          L.ptr(alive), L.stream_ptr()), "chain")
        if world > 1:
            torch.distributed.all_reduce(alive)
        b.record(stream)
        torch.cuda.synchronize()
        if k:
            ms.append(a.elapsed_time(b))
    t = max_over_ranks([sum(ms) / len(ms)], world, dev)[0] / 1e3
    curve = [100.0 * int(x) / (n_chain * world) for x in alive.cpu().tolist()]
    return {"workload": "C4: SetTable chains (settable plan, 16 slots), 4096 chains/GPU, "
                        "8 fuzz episodes per chain (seeds 8c+k), one fused mixed-subtask fuzz "
                        "graph, progressive_completion",
            "chains_per_gpu": n_chain, "n_gpus": world, "ms": 1e3 * t,
            "chains_per_s": n_chain * world / t,
            "labelled_trajectories_per_s": 8 * n_chain * world / t,
            "progressive_completion": curve}


def self_check(ws, ev_host, seeds, labels=None):
    """the timed kernels' last outputs against the CPU oracle (oracle/, test
    infrastructure): every label field and the ordered event lists"""
    from oracle import oracle as O
    from paper_2412_13211_b200 import _lib as L
    lab = (ws.labels if labels is None else labels).cpu().numpy().reshape(-1).view(L.LABEL_DTYPE)
    nrec = ws.n_rec.cpu().numpy()
    want = O.fuzz_label_batch_full(int(seeds[0]), len(seeds), KIND, oracle_cfg(),
                                   n_threads=os.cpu_count() or 1)
    off = ev_host["ev_off"].numpy()
    tot = int(off[-1])
    ok = (bool(np.all(lab["status"] == 0)) and np.array_equal(lab["mode"], want["mode"])
          and np.array_equal(lab["flags"] & 3, want["flags"])
          and np.array_equal(lab["n_events"], want["n_events"])
          and np.array_equal(nrec.astype(np.int64), want["n_rec"])
          and np.array_equal(off, want["ev_off"])
          and np.array_equal(ev_host["ev_kind"].numpy()[:tot], want["ev_kind"])
          and np.array_equal(ev_host["ev_t"].numpy()[:tot], want["ev_t"]))
    if not ok:
        raise RuntimeError("bench self-check: GPU labels / event lists differ from the oracle")
    return {"episodes": len(seeds), "events": tot, "vs": "oracle/oracle.c fuzz -> extract_events "
            "-> classify on the same seeds", "fields": "status, mode, flags, n_events, n_rec, "
            "ev_off, ev_kind, ev_t", "ok": True}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    rc = maybe_self_launch(args, argv)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = rank_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import ctypes
    import torch
    from paper_2412_13211_b200 import _lib as L
    from paper_2412_13211_b200 import core
    from paper_2412_13211_b200.synth import FuzzConfig

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    lib = L.lib()
    cfg = FuzzConfig(**CFG)
    cap = core.fuzz_capacity(cfg)
    K, W = args.steps, args.warmup
    stream = torch.cuda.Stream(device=dev)  # graphs need a non-default stream
    torch.cuda.set_stream(stream)
    ev_cap = 4 * N_ENV * cap   # tl_fuzz_ev bound: <= 4 events per record
    # pinned host outputs the e2e path writes into (zero-copy event lists)
    ev_host = dict(ev_off=torch.empty(N_ENV + 1, dtype=torch.int64).pin_memory(),
                   ev_kind=torch.empty(ev_cap, dtype=torch.uint8).pin_memory(),
                   ev_t=torch.empty(ev_cap, dtype=torch.int32).pin_memory())
    graph, seeds_buf, ws, ev_dev = fuzz_step_graph(dev, stream, N_ENV, KIND, cfg)
    graph_h, seeds_h, ws_h, _ = fuzz_step_graph(dev, stream, N_ENV, KIND, cfg, host_out=ev_host)
    # one GPU: zero-copy both ways -- the reset kernel reads the seeds from the
    # pinned staging buffer, the realize kernel writes the labels and
    # k_scan_emit the event lists into pinned memory (scripts/e2e_variants.py:
    # 135 us per step vs 147-152 us with copy_ H2D + D2H around the graph; the
    # copies captured into the graph measured slower still).  N > 1 keeps the
    # labels on the device for the NCCL all-gather and copies them back.
    zc = None
    if world == 1:
        zc_seeds = torch.empty(N_ENV, dtype=torch.int64).pin_memory()
        zc_labels = torch.empty((N_ENV, 24), dtype=torch.uint8).pin_memory()
        graph_zc, _, ws_zc, _ = fuzz_step_graph(dev, stream, N_ENV, KIND, cfg,
                                                host_out=dict(ev_host, labels=zc_labels),
                                                seeds_host=zc_seeds)
        zc = (graph_zc, ws_zc, zc_seeds.numpy(), zc_labels)
    hist = torch.zeros(L.N_MODES, dtype=torch.int64, device=dev)
    gathered = torch.empty((world * N_ENV, 24), dtype=torch.uint8, device=dev)
    # inputs resident in HBM: seeds of every step, rank-disjoint ranges
    all_seeds = torch.from_numpy(np.stack([step_seeds(k, rank, world) for k in range(K + W)])).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def exchange(labels):
        # the one exchange step: all-gather the 24-byte labels
        # over NCCL; every rank builds the global mode histogram itself
        if world > 1:
            gather_labels(labels, gathered, world)
            L.check(lib.tl_mode_histogram(L.ptr(gathered), world * N_ENV, L.ptr(hist),
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                    "hist")

    launches_per_step = 3 + (1 if world > 1 else 0)  # reset, realize, event lists [, histogram]
    for k in range(W):
        seeds_buf.copy_(all_seeds[K + k])
        graph.replay()
        exchange(ws.labels)
    torch.cuda.synchronize()

    gpu_id = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) if \
        os.environ.get("CUDA_VISIBLE_DEVICES") else local
    nrec_log = torch.empty((K, N_ENV), dtype=torch.int32, device=dev)
    with ClockSampler(gpu_id) as clocks:
        # ---- device-timed steps: inputs in HBM, L2 flushed between steps -------
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(K):
            ev[k][0].record(stream)
            seeds_buf.copy_(all_seeds[k])
            graph.replay()
            exchange(ws.labels)
            ev[k][1].record(stream)
            nrec_log[k].copy_(ws.n_rec)
            flush.zero_()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        step_ms = [a.elapsed_time(b) for a, b in ev]

        # ---- the two generator kernels alone (roofline of the dominant work)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for k in range(K):
            seeds_buf.copy_(all_seeds[k])
            kev[k][0].record(stream)
            graph.replay()
            kev[k][1].record(stream)
            flush.zero_()
        torch.cuda.synchronize()
        synth_ms = [a.elapsed_time(b) for a, b in kev]

        # ---- end to end through the C ABI with host buffers (wall clock) ---
        # E: pinned host seeds -> GPU (H2D), k_scan_emit writes the event
        # lists into pinned host memory (zero-copy), labels come back by a D2H
        # copy (N>1: after the NCCL all-gather + histogram, which also comes
        # back); perf_counter around call + synchronize, per step.
        # E_records: additionally tl_scan_counts + tl_compact_records into one
        # contiguous staging buffer [23 planes x R f32 | R grasped u8] and ONE
        # D2H copy of it (+ the record offsets).
        host_seeds = all_seeds.cpu().pin_memory()
        hs_np = host_seeds.numpy()
        h_labels = torch.empty((N_ENV, 24), dtype=torch.uint8).pin_memory()
        h_hist = torch.empty(L.N_MODES, dtype=torch.int64).pin_memory()
        h_tot = torch.empty(1, dtype=torch.int64).pin_memory()
        staging = torch.empty(N_ENV * cap * RECORD_BYTES + 64, dtype=torch.uint8, device=dev)
        h_staging = torch.empty(staging.numel(), dtype=torch.uint8).pin_memory()
        comp_start = torch.empty(N_ENV + 1, dtype=torch.int64, device=dev)
        comp_nrec = torch.empty(N_ENV, dtype=torch.int32, device=dev)
        h_start = torch.empty(N_ENV + 1, dtype=torch.int64).pin_memory()
        scan_scratch = torch.empty(max(16, lib.tl_scan_scratch_bytes(N_ENV)), dtype=torch.uint8, device=dev)
        rb_c = ws_h.records().c()
        K2 = max(1, min(K, 50))

        def e2e_loop(with_records):
            wall, recs, h2d, d2h = 0.0, 0, 0, 0
            for k in range(K2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if zc is not None and not with_records:
                    np.copyto(zc[2], hs_np[k])  # this step's inputs into the staging the kernel reads
                    zc[0].replay()              # seeds over PCIe, labels + event lists back
                    stream.synchronize()
                    wall += time.perf_counter() - t0
                    NE = int(ev_host["ev_off"][N_ENV])
                    recs += int(nrec_log[k].sum())
                    h2d = N_ENV * 8
                    d2h = max(d2h, N_ENV * 24 + (N_ENV + 1) * 8 + NE * 5)
                    flush.zero_()
                    continue
                seeds_h.copy_(host_seeds[k], non_blocking=True)
                graph_h.replay()                          # event lists -> pinned host
                exchange(ws_h.labels)
                h_labels.copy_(ws_h.labels, non_blocking=True)
                d2h_k = N_ENV * 24
                if world > 1:
                    h_hist.copy_(hist, non_blocking=True)
                    d2h_k += L.N_MODES * 8
                sp = ctypes.c_void_p(stream.cuda_stream)
                R = 0
                if with_records:
                    L.check(lib.tl_scan_counts(L.ptr(ws_h.n_rec), N_ENV, L.ptr(comp_start),
                                               L.ptr(scan_scratch), sp), "scan")
                    h_tot.copy_(comp_start[N_ENV:N_ENV + 1], non_blocking=True)
                stream.synchronize()
                if with_records:
                    R = int(h_tot[0])
                    base = staging.data_ptr()
                    dst = L.Records_c(base, base + 23 * 4 * R, comp_start.data_ptr(),
                                      comp_nrec.data_ptr(), R, 0, 7)
                    L.check(lib.tl_compact_records(ctypes.byref(rb_c), N_ENV, L.ptr(comp_start),
                                                   ctypes.byref(dst), sp), "compact")
                    h_staging[:RECORD_BYTES * R].copy_(staging[:RECORD_BYTES * R], non_blocking=True)
                    h_start.copy_(comp_start, non_blocking=True)
                    stream.synchronize()
                    d2h_k += RECORD_BYTES * R + (N_ENV + 1) * 8 + 8
                wall += time.perf_counter() - t0
                NE = int(ev_host["ev_off"][N_ENV])
                recs += int(nrec_log[k].sum())
                h2d = N_ENV * 8
                d2h = max(d2h, d2h_k + (N_ENV + 1) * 8 + NE * 5)
                flush.zero_()
            return wall, recs, h2d, d2h

        t_e2e, e2e_recs, h2d_b, d2h_b = e2e_loop(False)
        check = self_check(zc[1] if zc else ws_h, ev_host, hs_np[K2 - 1],
                           labels=zc[3] if zc else None)
        t_e2r, e2r_recs, _, d2h_rb = e2e_loop(True)
        extras = {}
        if not args.no_extras:
            extras["c2_1024"] = c2_run(dev, stream, world, flush)
            extras["c3"] = c3_run(dev, stream, world, flush)
            extras["env_api"] = env_api_run(dev, stream)
            extras["label_sizing"] = label_sizing_run(L, core, lib, dev, stream, flush)
            extras["c5"] = c5_run(dev, stream, world)
            extras["c4"] = c4_run(dev, stream, world, flush)
            if rank == 0:
                extras["label_batch_files"] = label_batch_files_run()
    clk = clocks.summary()

    recs_k = nrec_log.sum(dim=1).to(torch.float64).cpu().numpy()
    max_rec = float(nrec_log.max().item())
    t_dev, t_syn, t_e2e, t_e2r, max_rec = max_over_ranks(
        [sum(step_ms) / 1e3, sum(synth_ms) / 1e3, t_e2e, t_e2r, max_rec], world, dev)
    total_recs, e2e_recs_all, e2r_recs_all = sum_over_ranks(
        [float(recs_k.sum()), float(e2e_recs), float(e2r_recs)], world, dev)
    if rank != 0:
        dist.destroy_process_group()
        return
    hbm_peak, peak_src = peaks()
    recs_per_launch = total_recs / world / K
    alg_bytes = recs_per_launch * RECORD_BYTES + N_ENV * LABEL_BYTES
    step_s = t_syn / K
    # latency roofline of the generator: the step cannot finish
    # before the serial CPython seeding chain of the reset (1247 dependent
    # steps, synth.py:103 -> init_by_array) plus the serial f64
    # cum_robot_force recurrence of the longest episode (synth.py:192-196)
    c_seed, c_cum, c_src = latency_constants()
    sm_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
    crit_cycles = 1247 * c_seed + max_rec * c_cum
    floor_s = crit_cycles / (sm_ghz * 1e9)
    prof = profile_json("r2_ncu_headline.json") or {}
    # dependency + issue floor: the realize kernel cannot start before the
    # reset's seeding chains end (longest-first claims need every script), and
    # the realize + event-list kernels cannot finish before every SM scheduler
    # has issued their warp instructions at one per cycle (ncu counts, same config)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    inst_after = sum(k["warp_instructions"] for k in prof.get("kernels", [])
                     if "k_synth_warp" in k["kernel"] or "k_scan_emit" in k["kernel"])
    issue_floor_s = (1247 * c_seed / (sm_ghz * 1e9) + inst_after / (4 * n_sm * sm_ghz * 1e9)) \
        if inst_after else None
    sps = total_recs / t_dev
    cb_sps, cb_eps, cb_sample = cpu_baseline(args.cpu_seconds)
    pyref = python_reference_baseline()
    e2e_sps = e2e_recs_all / t_e2e
    out = {
        "metric": METRIC, "value": sps, "unit": "env-steps/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * t_dev / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "storage": "f32 records",
        "data": "synthetic",
        "trajectories_per_sec": N_ENV * world * K / t_dev,
        "config": bench_config(world),
        "mean_steps_per_episode": recs_per_launch / N_ENV,
        "step": "1 CUDA graph: tl_fuzz_ev (k_fuzz_reset, k_synth_warp: realize + labels, "
                "k_scan_emit: ordered event lists)" + (", NCCL all_gather of the labels + tl_mode_histogram of the "
                                  "gathered labels" if world > 1 else ""),
        "timing": "CUDA events per step on the launch stream, max over ranks",
        "gpu_launches": launches_per_step * K,
        "roofline": {
            "kernel": "k_fuzz_reset + k_synth_warp + k_scan_emit (tl_fuzz_ev)", "bound": "latency",
            "achieved": crit_cycles / step_s / 1e9, "peak": sm_ghz,
            "unit": "GHz (critical-path cycles retired per second vs the SM clock)",
            "frac": floor_s / step_s,
            "floor_ms": 1e3 * floor_s, "avg_launch_ms": 1e3 * step_s,
            "floor_model": (f"1247 seeding steps x {c_seed:.1f} cycles + longest episode "
                            f"({int(max_rec)} records) x {c_cum:.1f} cycles of the f64 cum chain, at "
                            f"the sampled SM clock; constants: {c_src}"),
            "issue_active": prof.get("issue_active"), "warps_active": prof.get("warps_active"),
            "traffic": prof.get("dram_bytes_per_launch"),
            "profile": "profiles/r2_ncu_headline.json" if prof else None,
            "realize_kernel": prof.get("realize_kernel"),
            "note": ("floor = one episode's serial chains; the batch is also issue-bound: the "
                     "realize kernel's issue_active (ncu, same config) says how full the SMs are"),
            "issue_floor": None if issue_floor_s is None else {
                "floor_ms": 1e3 * issue_floor_s, "frac": issue_floor_s / step_s,
                "warp_instructions": inst_after, "schedulers": 4 * n_sm,
                "model": ("1247 seeding steps (the reset's chain: the realize kernel needs every "
                          "script) + the realize and event-list kernels' warp instructions "
                          "(profiles/r2_ncu_headline.json) issued at 1 per scheduler per cycle")},
            "hbm": {"achieved": alg_bytes / step_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                    "frac": alg_bytes / step_s / 1e9 / hbm_peak, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "note": "93 B/record + 24 B/episode written; not the bound (MT19937 + f64 "
                            "generation is latency-bound, SURVEY 8(d))"}},
        "e2e": {"value": e2e_sps, "unit": "env-steps/s",
                "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b, "steps": K2,
                "timing": "time.perf_counter around the calls + stream synchronize, per step, "
                          "max over ranks",
                "note": "C-ABI tl_fuzz_ev with host buffers: the step's seeds copied into a "
                        "pinned staging buffer that the reset kernel reads over PCIe, labels "
                        "(realize kernel) and ordered event lists (k_scan_emit) written into "
                        "pinned host memory (zero-copy); N>1: seeds H2D, labels on the device "
                        "for the NCCL all-gather, then labels + histogram D2H",
                "with_records": {"value": e2r_recs_all / t_e2r, "unit": "env-steps/s",
                                 "d2h_bytes_per_step": d2h_rb,
                                 "note": "same, plus tl_scan_counts + tl_compact_records into one "
                                         "contiguous staging buffer and ONE D2H copy of every "
                                         "generated record (93 B/env-step)"}},
        "self_check": check,
        "cpu_baseline": {"value": cb_sps, "unit": "env-steps/s", "cores": 1, "kind": "port",
                         "sample": cb_sample, "trajectories_per_sec": cb_eps,
                         "host": host_info()},
        "python_reference": pyref,
        "clocks": clk,
    }
    pool = (pyref.get("pool") or {}).get("fuzz_and_label_sps") if isinstance(pyref, dict) else None
    if pool:
        out["vs_python_reference"] = {"e2e_ratio": e2e_sps / pool, "ratio": sps / pool,
                                      "against": "python_reference.pool (all host cores)"}
    out.update(extras)
    print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
