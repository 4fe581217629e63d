"""K3-only timing (pooled fp16x3 scorer) at a config shape; prints ms and executed TFLOP/s.

    python tools/score_bench.py [HY|W7|W4|C] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_23445_b200 as dfs  # noqa: E402
from paper_2605_23445_b200 import ops  # noqa: E402
from bench import WORKLOADS, smooth_fields  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "HY"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = WORKLOADS[wl]
dims, H, d, B, Bs = cfg["dims"], cfg["heads"], cfg["d"], cfg["block"], cfg["sub"]
n = dims[0] * dims[1] * dims[2]
q, k, _ = smooth_fields(dims, H, d, 1, torch.device("cuda"))
perm = dfs.hilbert3d_order(dims)
_, pq = ops.permute_to_hnd(q, perm, Bs)
_, pk = ops.permute_to_hnd(k, perm, Bs)
f = lambda: ops.score_pooled(pq, pk, n, dfs.ScoringParams(B, Bs))  # noqa: E731
for _ in range(3):
    f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    f()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
P = -(-n // Bs)
print(f"{wl} K3 scorer {ms:.3f} ms  executed {3 * 2 * P * P * d * H / ms / 1e9:.1f} TFLOP/s (fp16x3)")
