import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['DFS_ATTN_TRACE'] = 'gpurun_out/attn_trace.bin'
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
from bench import smooth_fields
dims, H, d = (33, 45, 80), 24, 128
n = 33*45*80
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
perm = m.hilbert3d_order(dims)
qh, pq = ops.permute_to_hnd(q, perm, 16); kh, pk = ops.permute_to_hnd(k, perm, 16); vh, _ = ops.permute_to_hnd(v, perm, 0)
S = ops.score_pooled(pq, pk, n, m.ScoringParams(128, 16)); lut = m.topk_lut(S, 0.1); ptr = ops.lut_row_ptr(H, 929, 93)
os.makedirs('gpurun_out', exist_ok=True)
o = m.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), 128); torch.cuda.synchronize()
t = np.fromfile('gpurun_out/attn_trace.bin', dtype=np.uint64).reshape(16, 256).astype(np.int64)
t0 = t[t > 0].min()
names = ['kv_wait_start', 'kv_wait_done', 'p_wait_start', 'p_wait_done', 'wg0_s_wait', 'wg0_s_ready', 'wg0_barrier', 'wg0_arrive', 'wg1_s_wait', 'wg1_s_ready', 'wg1_barrier', 'wg1_arrive']
for i, nm in enumerate(names):
    row = t[i] - t0
    print(f"{nm:14s}", ' '.join(f"{x:7d}" for x in row[100:112]))
sr = t[5, 100:200] - t[4, 100:200]; ar = t[7, 100:200] - t[5, 100:200]; pw = t[3, 100:200] - t[2, 100:200]
print('per-block period wg0 arrive', np.diff(t[7, 100:200]).mean(), 'softmax busy', ar.mean(), 's_full wait', sr.mean(), 'MMA p_full wait', pw.mean())
print('kv wait', (t[1, 100:200] - t[0, 100:200]).mean())
