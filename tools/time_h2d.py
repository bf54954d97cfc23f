"""PCIe ceiling for the end-to-end line: pinned host -> device copy of the headline YET
(4.0 GB) as one copy and in 64 MiB chunks, CUDA-event timed (median of 5).

    python tools/time_h2d.py > gpurun_out/time_h2d.json
"""
import json
import statistics

import torch


def main():
    n = 1_000_000_000  # u32 ids of 1M trials x 1000 events
    h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.int32, device="cuda:0")
    chunk = 16 << 20
    for mode in ("whole", "chunks_64MiB"):
        ts = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            if mode == "whole":
                d.copy_(h, non_blocking=True)
            else:
                for i in range(0, n, chunk):
                    d[i:i + chunk].copy_(h[i:i + chunk], non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts[1:])
        print(json.dumps({"mode": mode, "bytes": n * 4, "ms": ms, "GBps": n * 4 / ms / 1e6}))


if __name__ == "__main__":
    main()
