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
from paper_1308_2572_b200.dist import partition_trials, shard_range

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
