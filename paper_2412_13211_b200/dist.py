"""Multi-GPU execution: episodes shard with no data-path exchange; NCCL is
used only to all-gather the per-episode labels and all-reduce the mode
histogram.

Partition: rank r owns the contiguous seed range [r*N/W, (r+1)*N/W).  With
the zero-padded fuzz ids (synth.py:373) rank-order concatenation is
episode_id order within a subtask, so the gathered label array is already
in the order filter_labels sorts by (pipeline.py:290).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

LABEL_BYTES = 24


def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) share of n items for a rank."""
    return n * rank // world, n * (rank + 1) // world


def init_from_env(backend=None):
    """torch.distributed init from RANK/WORLD_SIZE/MASTER_* (127.0.0.1)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world == 1 or dist.is_initialized():
        return dist if dist.is_initialized() else None
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    kw = {}
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        kw["device_id"] = torch.device("cuda", local)
    dist.init_process_group(backend, **kw)
    return dist


def allgather_labels(local_labels, group=None):
    """Concatenate every rank's [n_r, 24] tl_label bytes in rank order.
    Shards may differ in size by one (shard_range), so sizes are exchanged
    first and the payload is padded to the largest shard."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([local_labels.shape[0]], dtype=torch.int64, device=local_labels.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    buf = torch.zeros((m, LABEL_BYTES), dtype=torch.uint8, device=local_labels.device)
    buf[:local_labels.shape[0]] = local_labels
    out = torch.empty((world * m, LABEL_BYTES), dtype=torch.uint8, device=local_labels.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[r * m:r * m + sizes[r]] for r in range(world)])


def allreduce_hist(hist, group=None):
    import torch.distributed as dist
    dist.all_reduce(hist, group=group)
    return hist


@dataclass
class ShardResult:
    labels: object          # local tl_label bytes [n_local, 24] (device)
    all_labels: object      # gathered [n_total, 24]
    hist: object            # global mode histogram [39] int64
    lo: int
    hi: int


def fuzz_label_sharded(n_total: int, subtask: int, cfg, th=None, group=None, seed0=0):
    """Each rank fuzzes + labels its seed shard on its GPU (one fused launch
    pair), then labels are all-gathered; every rank histograms the gathered set."""
    import torch
    import torch.distributed as dist
    from . import core
    from .thresholds import Thresholds
    from . import _lib as L
    th = th or Thresholds()
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lo, hi = shard_range(n_total, rank, world)
    dev = L.device()
    seeds = torch.arange(seed0 + lo, seed0 + hi, dtype=torch.int64, device=dev)
    cs = core.synth_csets(th).to_device(dev)
    sb = core.fuzz_batch(seeds, subtask, cfg, th, cs)
    if world > 1:
        all_labels = allgather_labels(sb.labels[:hi - lo], group)
    else:
        all_labels = sb.labels[:hi - lo]
    # global histogram from the gathered labels: no second collective
    hist = core.mode_histogram(all_labels, int(all_labels.shape[0]))
    return ShardResult(sb.labels[:hi - lo], all_labels, hist, lo, hi)


def fuzz_label_filter_sharded(n_per_subtask: int, spec, cfg=None, n_targets: int = 9,
                              th=None, group=None):
    """C5: fuzz(seed, kind) for seeds [0, n) of every subtask,
    seed-sharded over the ranks, labels all-gathered in rank (= episode_id)
    order, target_id = f"{seed % n_targets:03d}", then filter_labels on every
    rank's GPU (identical, deterministic manifests).  Returns (labels
    [4n, 24] in SUBTASK_ORDER blocks, DeviceManifest, key names)."""
    import torch
    from . import _lib as L
    from .pipeline import filter_labels_device
    from .synth import FuzzConfig
    cfg = cfg or FuzzConfig()
    dev = L.device()
    parts = [fuzz_label_sharded(n_per_subtask, s, cfg, th, group).all_labels for s in range(4)]
    labels = torch.cat(parts)
    keys = (torch.arange(n_per_subtask, dtype=torch.int32, device=dev) % n_targets).repeat(4)
    names = [f"{t:03d}" for t in range(n_targets)]
    return labels, filter_labels_device(labels, keys, names, spec), names
