"""K2-only timing at a config shape: the three passes run_step makes (q pooled read-only,
k permute + pool, v permute), with the finite check on; prints ms and GB/s per pass.

    python tools/permute_bench.py [HY|W7|W4|C] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_23445_b200 as dfs  # noqa: E402
from paper_2605_23445_b200 import ops  # noqa: E402
from bench import WORKLOADS, smooth_fields  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "HY"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = WORKLOADS[wl]
dims, H, d, Bs = cfg["dims"], cfg["heads"], cfg["d"], cfg["sub"]
n = dims[0] * dims[1] * dims[2]
q, k, v = smooth_fields(dims, H, d, 1, torch.device("cuda"))
perm = dfs.hilbert3d_order(dims)
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
x_bytes = n * H * d * 2
p_bytes = H * (-(-n // Bs)) * d * 4
passes = [
    ("q pool (read-only)", lambda: ops.pool_gathered(q, perm, Bs, flag), x_bytes + p_bytes),
    ("k permute + pool", lambda: ops.permute_to_hnd(k, perm, Bs, flag), 2 * x_bytes + p_bytes),
    ("v permute", lambda: ops.permute_to_hnd(v, perm, 0, flag), 2 * x_bytes),
]
for name, f, nbytes in passes:
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
    print(f"{wl} {name:20s} {ms:.3f} ms  {nbytes / ms / 1e6:.0f} GB/s")
