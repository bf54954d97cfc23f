"""Multi-rank host logic on CPU (gloo, world size 2 and 3): trial partition, input broadcast,
YLT all-gather, max-over-ranks.  Each rank computes its slice with the oracle (the per-rank CUDA
scan is covered by the GPU sharding-invariance test); the gathered YLT and the metrics must equal
the single-process run bit for bit (strong scaling does not change results)."""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import datagen
import oracle
from paper_1308_2572_b200.dist import partition_rank0_offload, partition_trials, shard_range

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
P = [0.9, 0.96, 0.98, 0.99, 0.996, 0.998, 0.999]


@pytest.mark.parametrize("case", GOLD["partition_trials"], ids=lambda c: c["cite"])
def test_partition_spec_examples(case):
    assert [list(r) for r in partition_trials(case["n"], case["workers"])] == case["expected"]


def test_partition_properties():
    for n in (0, 1, 7, 1000, 1_000_000):
        for R in (1, 2, 3, 4, 8):
            parts = partition_trials(n, R)
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a <= b for a, b in parts)
            assert all(parts[i][1] == parts[i + 1][0] for i in range(R - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
            assert shard_range(n, R - 1, R) == parts[-1]


def test_partition_rank0_offload():
    """Rank 0 computes the metrics alone and takes mu fewer trial-equivalents: ranges stay
    contiguous and cover [0, n); rank 0 never exceeds the balanced share; the other ranks split
    the rest as partition_trials does; rank 0's share + mu balances the others' shares."""
    for n in (0, 7, 1000, 1_000_000, 1_000_003):
        for R in (1, 2, 3, 8):
            for mu in (0, 0.0, 5.5, 137, 11_160.4, 10 ** 9):
                parts = partition_rank0_offload(n, R, mu)
                assert len(parts) == R and parts[0][0] == 0 and parts[-1][1] == n
                assert all(parts[i][1] == parts[i + 1][0] for i in range(R - 1))
                sizes = [b - a for a, b in parts]
                assert all(x >= 0 for x in sizes)
                if R == 1 or mu <= 0:
                    assert parts == partition_trials(n, R)
                    continue
                assert sizes[0] <= n // R
                assert parts[1:] == [(parts[0][1] + a, parts[0][1] + b)
                                     for a, b in partition_trials(n - sizes[0], R - 1)]
                if 0 < sizes[0] < n // R:  # not clamped: rank 0's share + mu ~ the others'
                    assert abs(sizes[0] + mu - (n - sizes[0]) / (R - 1)) <= 1 + 1 / (R - 1)


def _worker_parts(rank, world, port, spec, outdir):
    """gather_ylt with the uneven ranges of partition_rank0_offload (bench.py's default split)."""
    import torch
    import torch.distributed as dist

    from paper_1308_2572_b200 import dist as adist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ds = datagen.generate(spec, with_yet=False)
    parts = adist.partition_rank0_offload(spec.n_trials, world, 137.0)
    a, b = parts[rank]
    off, ev = datagen.generate_yet(spec, ds.pool, a, b - a)
    ylt_loc = oracle.run_analysis(ds, trial_offsets=off, events=ev)
    full = adist.gather_ylt(torch.from_numpy(ylt_loc), spec.n_trials, parts=parts).numpy()
    np.savez(os.path.join(outdir, f"p{rank}.npz"), full=full, sizes=np.array([y - x for x, y in parts]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_uneven_ranges_gather(tmp_path, world):
    spec = datagen.PRESETS["tiny"].replace(n_trials=1001, k_min=3, k_max=25)
    mp.spawn(_worker_parts, args=(world, _free_port(), spec, str(tmp_path)), nprocs=world,
             join=True)
    want = oracle.run_analysis(datagen.generate(spec))
    for r in range(world):
        z = np.load(tmp_path / f"p{r}.npz")
        assert z["sizes"][0] < z["sizes"][1]                  # rank 0 scans fewer trials
        assert np.array_equal(z["full"], want)                # gathered YLT == single process


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, outdir):
    import torch
    import torch.distributed as dist

    from paper_1308_2572_b200 import dist as adist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank 0 owns the portfolio; the others start from a different (wrong) one of equal shape
    ds = datagen.generate(spec if rank == 0 else spec.replace(seed=spec.seed + 17),
                          with_yet=False)
    adist.broadcast_inputs(ds, src=0)
    a, b = adist.shard_range(spec.n_trials, rank, world)
    off, ev = datagen.generate_yet(spec, datagen.generate(spec, with_yet=False).pool, a, b - a)
    ylt_loc = oracle.run_analysis(ds, trial_offsets=off, events=ev)
    full = adist.gather_ylt(torch.from_numpy(ylt_loc), spec.n_trials).numpy()
    pml, tvar = oracle.metrics(full[0], P)
    t = adist.max_over_ranks([float(rank), -float(rank)])
    np.savez(os.path.join(outdir, f"r{rank}.npz"), full=full, pml=pml, tvar=tvar, t=np.array(t),
             rec=ds.rec_losses, lt=ds.layer_terms)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_run_equals_single_process(tmp_path, world):
    spec = datagen.PRESETS["tiny"].replace(n_trials=1001, k_min=3, k_max=25)
    mp.spawn(_worker, args=(world, _free_port(), spec, str(tmp_path)), nprocs=world, join=True)
    ds = datagen.generate(spec)
    want = oracle.run_analysis(ds)
    wpml, wtvar = oracle.metrics(want[0], P)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["rec"], ds.rec_losses)        # broadcast reached every rank
        assert np.array_equal(z["lt"], ds.layer_terms)
        assert np.array_equal(z["full"], want)                # gathered YLT == single process
        assert np.array_equal(z["pml"], wpml) and np.array_equal(z["tvar"], wtvar)
        assert z["t"].tolist() == [world - 1.0, 0.0]          # max over ranks
