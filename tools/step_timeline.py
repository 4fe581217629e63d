"""Kernel timeline of run_step at a config shape (torch.profiler / CUPTI): per-kernel
durations and the idle gaps between consecutive kernels inside one update-step call.

    python tools/step_timeline.py [HY|W7|W4|C]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_23445_b200 as dfs  # noqa: E402
from bench import WORKLOADS, smooth_fields  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "HY"
cfg = WORKLOADS[wl]
dims, H, d, B, Bs, gamma = cfg["dims"], cfg["heads"], cfg["d"], cfg["block"], cfg["sub"], cfg["gamma"]
q, k, v = smooth_fields(dims, H, d, 1000, torch.device("cuda"))
params = dfs.ScoringParams(B, Bs)
sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gamma,), phase_fraction=1.0,
                             update_interval=1)
cache = dfs.MaskCache()
out = torch.empty_like(q)
step = lambda: dfs.run_step(q, k, v, dims, params, sched, cache, layer=0, step=0, out=out)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
busy = 0.0
for e in ev:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0.0
    busy += t - s
    print(f"{(s - t0) / 1e3:9.3f} ms  gap {gap:8.1f} us  dur {(t - s) / 1e3:8.3f} ms  {e.name[:70]}")
    prev_end = t
span = ev[-1].time_range.end - t0
print(f"span {span / 1e3:.3f} ms for 3 calls, kernels busy {busy / 1e3:.3f} ms ({100 * busy / span:.1f} %)")
