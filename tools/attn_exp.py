import os, subprocess, sys
code = r'''
import sys, time, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
H, n, d, k = 24, 118800, 128, 93
g = torch.Generator().manual_seed(0)
q, kk, v = (torch.randn(H, n, d, generator=g).bfloat16().cuda() for _ in range(3))
mq = -(-n // 128)
lut = torch.stack([torch.stack([torch.randperm(mq, generator=g)[:k].sort().values for _ in range(mq)]) for _ in range(H)]).int().cuda()
ptr = ops.lut_row_ptr(H, mq, k)
for i in range(2): o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(5): o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128)
b.record(); torch.cuda.synchronize()
print(a.elapsed_time(b) / 5)
'''
for mode in [0, 4, 1 | 4, 2 | 4, 1 | 2 | 4, 1, 2]:
    env = dict(os.environ, DFS_ATTN_EXP=str(mode))
    r = subprocess.run([sys.executable, '-c', code], env=env, capture_output=True, text=True, timeout=120)
    print('mode', mode, 'skip:', ['QK' if mode & 1 else '', 'PV' if mode & 2 else '', 'softmax' if mode & 4 else ''], 'ms', r.stdout.strip()[-20:], r.stderr[-200:])
