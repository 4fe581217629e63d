"""Small launches of every hot-path kernel for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize.py. Config T (B = 64, tcgen05 union tiles), a B = 128,
d = 128 and a d = 64 step (K2, K3 tcgen05 pairs, K4, K5), the fused-exchange Ulysses
step over two simulated ranks, the fp32 compatibility step, the streamed recall and dense
(warmup) steps through the multicast cluster kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_23445_b200 as dfs  # noqa: E402
from paper_2605_23445_b200 import ulysses  # noqa: E402


def step(dims, h, d, b, dtype=torch.bfloat16, recall=False):
    n = dims[0] * dims[1] * dims[2]
    g = torch.Generator().manual_seed(n + d)
    q, k, v = (torch.randn(n, h, d, generator=g).to(dtype).cuda() for _ in range(3))
    sched = dfs.SparsitySchedule(total_steps=2, warmup_fraction=0.0, phase_budgets=(0.25,), phase_fraction=1.0,
                                 update_interval=2)
    cache = dfs.MaskCache()
    for s in (0, 1):  # update step, then mask-reuse step
        dfs.run_step(q, k, v, dims, dfs.ScoringParams(b, 16), sched, cache, layer=0, step=s, record_recall=recall)
    torch.cuda.synchronize()
    return q, k, v


def dense(dims, h, d):
    """A dense (warmup) step: K5 over the full key list in 2-CTA clusters with multicast K/V."""
    n = dims[0] * dims[1] * dims[2]
    g = torch.Generator().manual_seed(n + 7 * d)
    q, k, v = (torch.randn(n, h, d, generator=g).to(torch.bfloat16).cuda() for _ in range(3))
    sched = dfs.SparsitySchedule(total_steps=4, warmup_fraction=0.5, phase_budgets=(0.25,), phase_fraction=0.5,
                                 update_interval=1)  # steps 0 and 1 are dense
    dfs.run_step(q, k, v, dims, dfs.ScoringParams(128, 16), sched, dfs.MaskCache(), layer=0, step=0)
    torch.cuda.synchronize()


if __name__ == "__main__":
    dense((4, 16, 32), 2, 128)  # 16 query blocks per head
    dense((3, 16, 45), 3, 64)  # 17 per head: the odd CTA's phantom tile
    step((4, 8, 8), 2, 64, 64)
    step((4, 16, 32), 2, 128, 128, recall=True)
    step((3, 16, 45), 2, 64, 128)
    step((4, 16, 16), 2, 32, 32, dtype=torch.float32)
    q, k, v = step((4, 16, 32), 4, 128, 128)
    nl = q.shape[0] // 2
    shards = {key: [t[r * nl:(r + 1) * nl].contiguous() for r in range(2)] for key, t in (("q", q), ("k", k), ("v", v))}
    shards["o"] = [torch.zeros_like(shards["q"][0]) for _ in range(2)]
    sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(0.25,), phase_fraction=1.0,
                                 update_interval=1)
    for r in range(2):
        ulysses.alltoall_step_local(shards, (4, 16, 32), dfs.ScoringParams(128, 16), sched, dfs.MaskCache(), 0, 0, r)
    torch.cuda.synchronize()
    print("sanitize workload done")
