"""bench.py's multi-GPU plumbing on CPU (gloo, world size 2), with the CPU
oracle standing in for the kernels: rank-disjoint seed shards, the rank-ordered
label all-gather (the one exchange step), max-over-ranks timing,
and the --gpus N self-launch command."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

N = 64


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _labels_standin(seeds):
    """24-byte label rows from the oracle (status 0, n_events, mode) -- the
    stand-in for tl_fuzz_ev's output on this rank's shard"""
    from oracle import oracle as O
    w = O.fuzz_label_batch_full(int(seeds[0]), len(seeds), bench.KIND, bench.oracle_cfg())
    rows = np.zeros((len(seeds), 24), np.uint8)
    rows[:, 4:8] = w["n_events"].astype("<i4").view(np.uint8).reshape(-1, 4)
    rows[:, 13] = w["mode"]
    rows[:, 14] = w["flags"]
    return torch.from_numpy(rows)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k = 3
        seeds = bench.step_seeds(k, rank, world, N)
        local = _labels_standin(seeds)
        out = torch.empty((world * N, 24), dtype=torch.uint8)
        bench.gather_labels(local, out, world)
        t = bench.max_over_ranks([1.0 + rank, 5.0 - rank], world)
        s = bench.sum_over_ranks([float(rank + 1)], world)
        q.put((rank, seeds, out.numpy().copy(), t, s))
    finally:
        dist.destroy_process_group()


def test_bench_dist_plumbing_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    seeds = np.concatenate([r[1] for r in res])
    # shards: contiguous, rank-disjoint, rank order = seed (= episode_id) order
    assert np.array_equal(seeds, np.arange(seeds[0], seeds[0] + world * N))
    assert seeds[0] == 3 * world * N
    # every rank holds the same rank-ordered gathered labels == the oracle
    # over the whole step's seeds
    want = _labels_standin(seeds).numpy()
    for r in res:
        assert np.array_equal(r[2], want)
        assert r[3] == [2.0, 5.0]          # element-wise max over ranks
        assert r[4] == [3.0]               # sum over ranks


def test_step_seeds_fresh_and_disjoint():
    seen = set()
    for k in range(4):
        for r in range(8):
            s = bench.step_seeds(k, r, 8, 16)
            assert len(s) == 16 and not (seen & set(s.tolist()))
            seen |= set(s.tolist())
    assert seen == set(range(4 * 8 * 16))


def test_self_launch_argv(monkeypatch):
    argv = ["--gpus", "4", "--steps", "7"]
    cmd = bench.launch_argv(4, argv, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == argv and cmd[-5].endswith("bench.py")
    # inside a torchrun rank (WORLD_SIZE set) or for one GPU: no re-launch
    monkeypatch.setenv("WORLD_SIZE", "4")
    assert bench.maybe_self_launch(bench.parse(argv), argv) is None
    monkeypatch.delenv("WORLD_SIZE")
    assert bench.maybe_self_launch(bench.parse(["--gpus", "1"]), []) is None


def test_bench_config_identical_across_arms():
    """both arms print bench_config(world): the driver's same_config check"""
    assert bench.bench_config(2) == bench.bench_config(2)
    assert bench.bench_config(1)["envs_per_gpu"] == bench.N_ENV == 4096
