"""Head-dim ceiling probe: K5 in dense mode (no key-block list) against cuDNN's SDPA (a
library kernel, two query tiles per CTA) on the same dense problem, at d = 64 and d = 128.
Both do 4*N^2*d FLOP per head; the ratio of the two is how far K5's d = 64 shortfall
(config C) is the head dim's and how far it is K5's.

    python tools/d64_ceiling.py [N] [H]
Under `ncu --metrics sm__cycles_elapsed.max` (tools/d64_cycles.sh) the per-cycle rates follow.
"""
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, ".")
import paper_2605_23445_b200 as m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
h = int(sys.argv[2]) if len(sys.argv) > 2 else 24


def timed(f, reps=5):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for d in (64, 128):
    g = torch.Generator(device="cuda").manual_seed(d)
    q, k, v = (torch.randn(h, n, d, generator=g, device="cuda").bfloat16() for _ in range(3))
    fl = 4.0 * n * n * d * h
    ms_k5 = timed(lambda: m.sparse_attention_csr(q, k, v, None, None, 128))
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        q4, k4, v4 = q[None], k[None], v[None]
        ms_cd = timed(lambda: F.scaled_dot_product_attention(q4, k4, v4))
        ref = F.scaled_dot_product_attention(q4[:, :1], k4[:, :1], v4[:, :1])[0, 0].float()
    out = m.sparse_attention_csr(q[:1], k[:1], v[:1], None, None, 128).float()
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    print(f"d={d:3d} N={n} H={h}: K5 dense {ms_k5:8.3f} ms {fl / ms_k5 / 1e9:6.0f} TFLOP/s | "
          f"cuDNN SDPA {ms_cd:8.3f} ms {fl / ms_cd / 1e9:6.0f} TFLOP/s | K5/cuDNN time {ms_k5 / ms_cd:.3f} "
          f"| head-0 max rel diff {err:.2e}")
