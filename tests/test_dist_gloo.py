"""World-size-2 gloo tests of the multi-GPU host path (CPU only).

Each rank produces the tl_label bytes of its seed shard (here with the CPU
oracle standing in for the device kernels, since there is no GPU in CI),
then runs the same collective code the GPU path runs: rank-ordered label
all-gather and mode-histogram all-reduce.  The merged result must equal a
single-process run over all seeds."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_labels(lo, hi, kind):
    from oracle import oracle as O
    from paper_2412_13211_b200._lib import LABEL_DTYPE
    total, modes, nev, nrec = O.fuzz_label_batch(lo, hi - lo, kind, n_threads=1)
    lab = np.zeros(hi - lo, LABEL_DTYPE)
    lab["mode"] = modes
    lab["n_events"] = nev
    lab["subtask"] = kind
    return lab


def _worker(rank, world, port, n, kind, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2412_13211_b200 import dist as D
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = D.shard_range(n, rank, world)
    lab = _oracle_labels(lo, hi, kind)
    local = torch.from_numpy(lab.view(np.uint8).reshape(-1, 24).copy())
    gathered = D.allgather_labels(local)
    hist = torch.from_numpy(np.bincount(lab["mode"], minlength=39).astype(np.int64))
    D.allreduce_hist(hist)
    if rank == 0:
        out.put((gathered.numpy().tobytes(), hist.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [101, 640])
def test_gloo_label_allgather_and_histogram(n):
    from paper_2412_13211_b200._lib import LABEL_DTYPE
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 1, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, hist = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    want = _oracle_labels(0, n, 1)
    got = np.frombuffer(got, LABEL_DTYPE)
    assert len(got) == n
    assert np.array_equal(got["mode"], want["mode"])
    assert np.array_equal(got["n_events"], want["n_events"])
    assert hist == np.bincount(want["mode"], minlength=39).tolist()


def test_shard_ranges_cover_exactly():
    from paper_2412_13211_b200.dist import shard_range
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
