"""MMA-warp timeline of one CTA of K5 at HY (needs a -DDFS_ATTN_TRACE_BUILD library via DFS_B200_LIB).
Events: 0/1 = kv_full wait start/done per ring entry, 2/3 = p_full wait start/done per PV."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['DFS_ATTN_TRACE'] = 'gpurun_out/attn_trace.bin'
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
from bench import smooth_fields
dims, H, d = (33, 45, 80), 24, 128
n = 33 * 45 * 80
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
perm = m.hilbert3d_order(dims)
qh, pq = ops.permute_to_hnd(q, perm, 16); kh, pk = ops.permute_to_hnd(k, perm, 16); vh, _ = ops.permute_to_hnd(v, perm, 0)
S = ops.score_pooled(pq, pk, n, m.ScoringParams(128, 16)); lut = m.topk_lut(S, 0.1); ptr = ops.lut_row_ptr(H, 929, 93)
os.makedirs('gpurun_out', exist_ok=True)
o = m.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), 128); torch.cuda.synchronize()
t = np.fromfile('gpurun_out/attn_trace.bin', dtype=np.uint64).reshape(16, 256).astype(np.int64)
r0, r1 = 100, 200  # ring entries (2 per block)
kvw = t[1, r0:r1] - t[0, r0:r1]
gap = t[0, r0 + 1:r1 + 1] - t[1, r0:r1]  # kv wait done -> next kv wait start (issue work + p wait)
print("ring period", np.diff(t[0, r0:r1]).mean(), "kv wait", kvw.mean(), "done->next", gap.mean())
p0, p1 = 50, 100
print("PV: p wait", (t[3, p0:p1] - t[2, p0:p1]).mean(), "PV period", np.diff(t[2, p0:p1]).mean())
print("ring entries:", [(int(t[0, i] - t[0, r0]), int(t[1, i] - t[0, i])) for i in range(r0, r0 + 12)])
