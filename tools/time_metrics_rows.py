import sys, json, numpy as np, torch, time
sys.path.insert(0, '.')
from paper_1308_2572_b200 import ara
ctx = ara.Context(0, torch.cuda.current_stream())
P = [1 - 1/r for r in (10, 25, 50, 100, 250, 500, 1000)]
rng = np.random.default_rng(1)
for R in (1, 9):
    rows = rng.lognormal(13, 0.6, (R, 1_000_000)); rows[rng.random(rows.shape) < 0.3] = 0
    d = torch.from_numpy(rows).cuda()
    for _ in range(3): ctx.ara_metrics_rows(d, P)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): ctx.ara_metrics_rows(d, P)
    torch.cuda.synchronize(); tb = (time.perf_counter() - t) * 100
    t = time.perf_counter()
    for _ in range(10):
        for r in range(R): ctx.ara_metrics(d[r], P)
    torch.cuda.synchronize(); ts = (time.perf_counter() - t) * 100
    print(json.dumps({"rows": R, "batched_ms": tb, "separate_ms": ts}))
