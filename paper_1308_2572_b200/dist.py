"""Trial sharding across the GPUs of one node.

Trials are independent (one thread per trial), so the scan shards with no
data-path communication: rank r of R takes the r-th of R contiguous trial ranges
whose sizes differ by at most one, the larger ones first (10 trials on 4
workers -> 3, 3, 2, 2) and generates or receives only that
slice of the YET.  The two collectives are:
  1. once per portfolio: broadcast of the raw ELT records, financial terms and layer terms from
     the source rank (``broadcast_inputs``), after which every rank builds its own device store;
  2. per run, before PML/TVaR: all-gather of the YLT slices (``gather_ylt``), so every rank holds
     the full YLT and the metrics are identical on every rank and for every R.
With the NCCL backend the tensors live on the rank's GPU (NVLink / NVSwitch); with gloo (the CPU
tests) they are CPU tensors.  This module only moves data: every step of the method runs in
libara's kernels.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def partition_trials(n_trials: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, disjoint ranges covering [0, n), sizes differing by at most 1; ranks with
    nothing to do get empty ranges."""
    if world < 1:
        raise ValueError("world must be >= 1")
    q, rem = divmod(n_trials, world)
    starts = [r * q + min(r, rem) for r in range(world + 1)]
    return [(starts[r], starts[r + 1]) for r in range(world)]


def shard_range(n_trials: int, rank: int, world: int) -> Tuple[int, int]:
    return partition_trials(n_trials, world)[rank]


def partition_rank0_offload(n_trials: int, world: int, mu: float) -> List[Tuple[int, int]]:
    """Contiguous trial ranges when rank 0 alone computes PML/TVaR after the all-gather, which
    costs it as much time as scanning ``mu`` trials: rank 0 takes n0 = (n + mu) / R - mu trials
    (never more than the balanced share, never fewer than 0) and the other ranks split the rest
    as partition_trials does, so every rank's step (scan, plus the metrics on rank 0) takes the
    same time.  mu <= 0 or R = 1 gives partition_trials."""
    if world <= 1 or not mu or mu <= 0:
        return partition_trials(n_trials, world)
    n0 = int(round((n_trials + mu) / world - mu))
    n0 = min(max(n0, 0), n_trials // world)
    rest = partition_trials(n_trials - n0, world - 1)
    return [(0, n0)] + [(n0 + a, n0 + b) for a, b in rest]


def _dev_for(dist, like=None):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _host_staged(dist) -> bool:
    return dist.get_backend() != "nccl"


def broadcast_inputs(ds, src: int = 0):
    """Broadcast the raw ELT records, terms and layer membership of ``ds`` from ``src`` to every
    rank (in place on the non-source ranks' arrays, which must have the same shapes; use
    ``broadcast_shapes`` first when they do not)."""
    import torch
    import torch.distributed as dist
    dev = _dev_for(dist)
    fields = [("rec_offsets", np.uint64), ("rec_event_ids", np.uint32), ("rec_losses", np.float64),
              ("fin", np.float64), ("layer_terms", np.float64), ("elt_offsets", np.uint32),
              ("elt_index", np.uint32)]
    for name, dt in fields:
        a = np.ascontiguousarray(getattr(ds, name), dtype=dt)
        raw = a.view(np.uint8).reshape(-1)
        t = torch.from_numpy(raw.copy()).to(dev)
        dist.broadcast(t, src=src)
        setattr(ds, name, t.cpu().numpy().view(dt).reshape(a.shape).copy())
    cat = torch.tensor([int(ds.catalogue_size)], dtype=torch.int64, device=dev)
    dist.broadcast(cat, src=src)
    ds.catalogue_size = int(cat.item())
    return ds


def gather_ylt(ylt_local, n_trials: int, out=None, parts=None):
    """All-gather the [L, n_local] YLT slices of every rank into the full [L, n_trials] YLT
    (layer-major rows, trials in rank order).  ``ylt_local`` / ``out`` are tensors on the
    backend's device; ``parts`` = every rank's trial range (default partition_trials)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    L = ylt_local.shape[0]
    if out is None:
        out = torch.empty((L, n_trials), dtype=ylt_local.dtype, device=ylt_local.device)
    if parts is None:
        parts = partition_trials(n_trials, world)
    assert len(parts) == world and parts[-1][1] == n_trials
    m = max(b - a for a, b in parts)
    equal = all(b - a == m for a, b in parts)
    nccl = dist.get_backend() == "nccl"
    if not nccl and ylt_local.is_cuda:  # gloo: stage through host memory
        host = gather_ylt(ylt_local.cpu(), n_trials, parts=parts)
        out.copy_(host)
        return out
    for l in range(L):
        row = ylt_local[l].contiguous()
        if equal and nccl:
            dist.all_gather_into_tensor(out[l], row)
            continue
        # unequal slices (n not divisible by R): pad every slice to the largest one
        padded = torch.zeros(m, dtype=row.dtype, device=row.device)
        padded[: row.numel()] = row
        if nccl:
            buf = torch.empty(world * m, dtype=row.dtype, device=row.device)
            dist.all_gather_into_tensor(buf, padded)
            tmp = [buf[r * m:(r + 1) * m] for r in range(world)]
        else:
            tmp = [torch.empty(m, dtype=row.dtype, device=row.device) for _ in range(world)]
            dist.all_gather(tmp, padded)
        for (a, b), t in zip(parts, tmp):
            out[l, a:b].copy_(t[: b - a])
    return out


def max_over_ranks(values: Sequence[float]):
    """Element-wise max over ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=_dev_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()


def sum_over_ranks(values: Sequence[float]):
    """Element-wise sum over ranks (event counts of the rank slices)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=_dev_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().tolist()


def sharded_metrics(ctx, ylt_slice, n_global: int, p):
    """PML / TVaR of the YLT row whose slices the ranks hold, without gathering it
    (``ara_metrics_sharded``: the radix-select histograms and tail sums are summed across ranks
    pass by pass -- NCCL all-reduce on the context's stream; gloo stages through the host)."""
    import torch.distributed as dist

    def allreduce(t):
        if dist.get_backend() == "nccl":
            dist.all_reduce(t)
        else:
            h = t.cpu()
            dist.all_reduce(h)
            t.copy_(h)

    return ctx.ara_metrics_sharded(ylt_slice, n_global, p, allreduce)
