"""One rank of the multi-GPU path over NCCL (run by tests/test_parity_full_gpu.py under torchrun;
not collected by pytest).  Every collective of paper_1308_2572_b200/dist.py runs on the NCCL
backend: broadcast_inputs (ELTs and terms from rank 0), the rank's trial slice scanned through
libara, gather_ylt (all_gather_into_tensor; with world size > 1 the odd trial count also takes
the padded branch), sharded_metrics (all-reduce of the radix-select histograms) and
max_over_ranks.
The gathered YLT must equal the single-process oracle's entry for entry and the metrics its
PML / TVaR (the workload decomposed over the GPUs).  Prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402

P = [1 - 1 / rp for rp in (10, 25, 50, 100, 250, 500, 1000)]


def main():
    import torch
    import torch.distributed as dist

    from paper_1308_2572_b200 import ara
    from paper_1308_2572_b200 import dist as adist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    assert dist.get_backend() == "nccl"
    rank, world = dist.get_rank(), dist.get_world_size()
    out = {"backend": dist.get_backend(), "world": world}
    for n_trials in (20_000, 20_001):
        spec = datagen.PRESETS["medium"].replace(n_trials=n_trials)
        ds = datagen.generate(spec)
        adist.broadcast_inputs(ds, src=0)
        t0, t1 = adist.shard_range(ds.n_trials, rank, world)
        off = ds.trial_offsets[t0:t1 + 1]
        ids = ds.events[int(off[0]):int(off[-1])]
        stream = torch.cuda.current_stream(dev)
        ctx = ara.Context(local, stream)
        ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses,
                          ds.fin)
        ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
        d_off = torch.from_numpy(off.astype(np.uint64).view(np.int64)).to(dev).view(torch.uint64)
        d_ids = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.uint32).view(np.int32)).to(
            dev).view(torch.uint32)
        ylt = torch.empty((ds.n_layers, t1 - t0), dtype=torch.float64, device=dev)
        ctx.ara_run(d_off, d_ids, ylt, flags=ara.ARA_RUN_SYNC)
        full = adist.gather_ylt(ylt, ds.n_trials)
        want = oracle.run_analysis(ds)
        got = full.cpu().numpy()
        assert got.shape == want.shape
        bad = int(np.count_nonzero(got != want))
        assert bad == 0, f"{bad} YLT entries differ (n = {n_trials})"
        pml, tvar = ctx.ara_metrics(full[0], P)
        spml, stvar = adist.sharded_metrics(ctx, ylt[0], ds.n_trials, P)
        opml, otvar = oracle.metrics(want[0], P)
        assert np.array_equal(pml, opml) and np.array_equal(spml, opml), (pml, spml, opml)
        assert np.allclose(tvar, otvar, rtol=1e-9, atol=0)
        assert np.allclose(stvar, otvar, rtol=1e-9, atol=0)
        mx = adist.max_over_ranks([float(rank)])
        assert mx == [float(world - 1)]
        ctx.close()
        out[str(n_trials)] = {"ylt_entries": int(got.size), "mismatches": bad}
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
