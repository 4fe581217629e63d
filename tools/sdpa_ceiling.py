"""Dense attention ceiling on this B200: torch SDPA (cuDNN / flash backends, library kernels)
at the HY head shape, for comparison with K5's dense mode (same FLOP count, 4*N^2*d per head).

    python tools/sdpa_ceiling.py [N] [H]
"""
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
h = int(sys.argv[2]) if len(sys.argv) > 2 else 24
d = 128
q, k, v = (torch.randn(1, h, n, d, device="cuda", dtype=torch.bfloat16) for _ in range(3))
fl = 4.0 * n * n * d * h
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel([be]):
            f = lambda: F.scaled_dot_product_attention(q, k, v)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            print(f"sdpa {name:9s} N={n} H={h} d={d}: {ms:8.3f} ms  {fl / ms / 1e9:7.0f} TFLOP/s")
    except Exception as e:  # backend unavailable for this shape / build
        print(f"sdpa {name}: unavailable ({type(e).__name__}: {str(e)[:80]})")
