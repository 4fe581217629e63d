import os, sys, torch
sys.path.insert(0, '.')
os.environ['DFS_HOST_TIMING'] = '1'
import paper_2605_23445_b200 as dfs
from bench import WORKLOADS, smooth_fields
wl = WORKLOADS['HY']
dims, H, d, B, Bs, g = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(g,), phase_fraction=1.0, update_interval=1)
cache = dfs.MaskCache(); out = torch.empty_like(q)
for i in range(4):
    print("STEP", i, file=sys.stderr, flush=True)
    dfs.run_step(q, k, v, dims, dfs.ScoringParams(B, Bs), sched, cache, layer=0, step=0, out=out)
torch.cuda.synchronize()
