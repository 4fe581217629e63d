"""Per-GPU step time of head-sharded HY at 1/2/4/8 GPUs, measured on one GPU (a rank's share
of the heads; head sharding has no collective on the data path), and the implied strong-
scaling efficiency t(24 heads) / (P * t(24/P heads)).

    python tools/shard_sim.py [HY] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_23445_b200 as dfs  # noqa: E402
from bench import WORKLOADS, smooth_fields  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "HY"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dims, H, d, B, Bs, g = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
times = {}
for P in (1, 2, 4, 8):
    h = H // P
    q, k, v = smooth_fields(dims, h, d, 1000, torch.device("cuda"))
    params = dfs.ScoringParams(B, Bs)
    sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(g,), phase_fraction=1.0,
                                 update_interval=1)
    cache = dfs.MaskCache()
    out = torch.empty_like(q)
    f = lambda: dfs.run_step(q, k, v, dims, params, sched, cache, layer=0, step=0, out=out)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        f()
    b.record()
    torch.cuda.synchronize()
    times[P] = a.elapsed_time(b) / steps
    print(f"P={P}: {h} heads per GPU, {times[P]:.3f} ms per call, strong-scaling efficiency "
          f"{times[1] / (P * times[P]):.3f}", flush=True)
    del q, k, v, out, cache
    torch.cuda.empty_cache()
