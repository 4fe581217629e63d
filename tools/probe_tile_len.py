import sys, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
H, n, d = 48, 17550, 64
M = -(-n // 128)
g = torch.Generator(device='cuda').manual_seed(0)
q, k, v = (torch.randn(H, n, d, generator=g, device='cuda').bfloat16() for _ in range(3))
sizes = torch.full((M,), 128.0, device='cuda'); sizes[-1] = n - (M - 1) * 128
def run(K, label):
    gen = torch.Generator().manual_seed(1)
    lut = torch.stack([torch.randperm(M, generator=gen)[:K].sort().values for _ in range(H * M)]).to(torch.int32).cuda()
    ptr = ops.lut_row_ptr(H, M, K)
    f = lambda: m.sparse_attention_csr(q, k, v, ptr, lut.reshape(-1), 128)
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    fl = float(4.0 * d * (sizes[lut.long()].sum(-1) * sizes.repeat(H)).sum())
    print(f"{label:20s} K={K:4d} {ms:7.3f} ms {fl / ms / 1e9:6.0f} TFLOP/s")
for K in (28, 69, 138):
    run(K, "C d=64")
