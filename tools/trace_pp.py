"""Per-block timeline of CTA 0 of the two-tile ping-pong K5 (attn_pp.cu) at HY
(needs a -DDFS_ATTN_TRACE_BUILD library via DFS_B200_LIB and DFS_ATTN_PP=1)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['DFS_ATTN_TRACE'] = 'gpurun_out/attn_pp_trace.bin'
os.environ['DFS_ATTN_PP'] = '1'
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
t = np.fromfile('gpurun_out/attn_pp_trace.bin', dtype=np.uint64).reshape(16, 256).astype(np.int64)
names = {0: "P seen A", 1: "P seen B", 2: "PV iss A", 3: "PV iss B", 4: "QK iss A", 5: "QK iss B", 6: "P wait A",
         7: "P wait B", 8: "S wait A", 9: "S wait B", 10: "S seen A", 11: "S seen B", 12: "exps A", 13: "exps B",
         14: "P arr A", 15: "P arr B"}
lo = 40
t0 = t[10, lo]
for ev in (10, 12, 14, 6, 0, 2, 4, 11, 13, 15, 7, 1, 3, 5):
    print(f"{names[ev]:9s}", " ".join(f"{x - t0:7d}" for x in t[ev, lo:lo + 8]))
print("period per stream block A:", np.diff(t[10, lo:lo + 60]).mean(), "B:", np.diff(t[11, lo:lo + 60]).mean())
