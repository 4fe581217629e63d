import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['DFS_ATTN_TRACE'] = 'gpurun_out/attn_trace.bin'
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
H, n, d, k = 24, 118800, 128, 93
g = torch.Generator().manual_seed(0)
q, kk, v = (torch.randn(H, n, d, generator=g).bfloat16().cuda() for _ in range(3))
mq = -(-n // 128)
lut = torch.stack([torch.stack([torch.randperm(mq, generator=g)[:k].sort().values for _ in range(mq)]) for _ in range(H)]).int().cuda()
ptr = ops.lut_row_ptr(H, mq, k)
os.makedirs('gpurun_out', exist_ok=True)
o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128); torch.cuda.synchronize()
t = np.fromfile('gpurun_out/attn_trace.bin', dtype=np.uint64).reshape(16, 256).astype(np.int64)
t0 = t[0, 100]
# ring index r: even = K (QK), odd = V (PV) roughly; print a window
print('ring r: kv_wait_start, +wait, next event delta')
for r in range(100, 112):
    print(r, t[0, r] - t0, t[1, r] - t[0, r], t[0, r + 1] - t[1, r])
print('pv i: p_wait_start, p_wait')
for i in range(50, 56):
    print(i, t[2, i] - t0, t[3, i] - t[2, i])
per = np.diff(t[0, 100:200:2])
print('period per 2 ring entries (1 block):', per.mean(), 'kv wait mean', (t[1, 100:200] - t[0, 100:200]).mean(), 'p wait mean', (t[3, 50:100] - t[2, 50:100]).mean())
