"""K5 probe: where does sparse lose against dense? Same kernel, HY length, 3 heads.
dense (no list) | full list (K=M) | contiguous 93 blocks (sparse tile count, sequential K/V)
| 93 random blocks per query block | 93 blocks in a sliding window around the diagonal."""
import sys, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
H, n, d = 3, 118800, 128
M = -(-n // 128)
g = torch.Generator(device='cuda').manual_seed(0)
q, k, v = (torch.randn(H, n, d, generator=g, device='cuda').bfloat16() for _ in range(3))
sizes = torch.full((M,), 128.0, device='cuda'); sizes[-1] = n - (M - 1) * 128


def run(ptr, idx, label, kk):
    f = lambda: m.sparse_attention_csr(q, k, v, ptr, idx, 128)
    for _ in range(2): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    if idx is None:
        fl = 4.0 * d * n * n * H
    else:
        lut = idx.view(H, M, kk).long()
        fl = float(4.0 * d * (sizes[lut].sum(-1) * sizes[None, :]).sum())
    print(f"{label:34s} {ms:8.2f} ms  {fl / ms / 1e9:7.0f} TFLOP/s executed")


run(None, None, "dense (blk_ptr NULL)", M)
full = torch.arange(M, device='cuda', dtype=torch.int32).repeat(H * M)
run(ops.lut_row_ptr(H, M, M), full, "full list K=M", M)
K = 93
contig = torch.arange(K, device='cuda', dtype=torch.int32).repeat(H * M)
run(ops.lut_row_ptr(H, M, K), contig, "contiguous 93 (same for all u)", K)
u = torch.arange(M, device='cuda')
start = (u - K // 2).clamp(0, M - K)
win = (start[:, None] + torch.arange(K, device='cuda')[None]).to(torch.int32).repeat(H, 1).reshape(-1)
run(ops.lut_row_ptr(H, M, K), win, "sliding window 93 around u", K)
gen = torch.Generator().manual_seed(1)
rnd = torch.stack([torch.randperm(M, generator=gen)[:K].sort().values for _ in range(H * M)]).to(torch.int32).cuda()
run(ops.lut_row_ptr(H, M, K), rnd.reshape(-1), "random 93 per query block", K)
