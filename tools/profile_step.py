"""One warm HunyuanVideo update-step call (decomposed into its kernels) for ncu captures."""
import sys, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
from bench import smooth_fields, WORKLOADS
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "HY"]
dims, H, d, B, Bs, g = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
n = dims[0] * dims[1] * dims[2]
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
sched = m.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(g,), phase_fraction=1.0, update_interval=1)
cache = m.MaskCache()
out = torch.empty_like(q)
for _ in range(3):  # warm-up launches (skip these in ncu with -s)
    m.run_step(q, k, v, dims, m.ScoringParams(B, Bs), sched, cache, layer=0, step=0, out=out)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled_step")
m.run_step(q, k, v, dims, m.ScoringParams(B, Bs), sched, cache, layer=0, step=0, out=out)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
