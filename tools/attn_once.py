import sys, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
H, n, d, k = 24, 118800, 128, 93
g = torch.Generator().manual_seed(0)
q, kk, v = (torch.randn(H, n, d, generator=g).bfloat16().cuda() for _ in range(3))
mq = -(-n // 128)
lut = torch.stack([torch.stack([torch.randperm(mq, generator=g)[:k].sort().values for _ in range(mq)]) for _ in range(H)]).int().cuda()
ptr = ops.lut_row_ptr(H, mq, k)
for _ in range(2): o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128)
torch.cuda.synchronize()
