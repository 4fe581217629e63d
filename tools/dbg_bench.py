import sys, time, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
from paper_2605_23445_b200 import ops
from bench import smooth_fields
dims, H, d = (33, 45, 80), int(sys.argv[1]) if len(sys.argv) > 1 else 24, 128
n = 33*45*80
q, k, v = smooth_fields(dims, H, d, 1, torch.device('cuda'))
perm = m.hilbert3d_order(dims)
t = time.time(); qh, pq = ops.permute_to_hnd(q, perm, 16); kh, pk = ops.permute_to_hnd(k, perm, 16); vh, _ = ops.permute_to_hnd(v, perm, 0); torch.cuda.synchronize(); print('perm', time.time()-t, flush=True)
t = time.time(); S = ops.score_pooled(pq, pk, n, m.ScoringParams(128, 16)); torch.cuda.synchronize(); print('score', time.time()-t, flush=True)
t = time.time(); lut = m.topk_lut(S, 0.1); torch.cuda.synchronize(); print('topk', time.time()-t, lut.shape, flush=True)
ptr = ops.lut_row_ptr(H, 929, 93)
for it in range(3):
    t = time.time(); o = m.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), 128); torch.cuda.synchronize(); print('attn', time.time()-t, flush=True)
og = m.sparse_attention_csr(qh[:2], kh[:2], vh[:2], ops.lut_row_ptr(2, 929, 93), lut[:2].reshape(-1), 128, force_generic=True)
print('rel vs generic (2 heads)', float((o[:2].float()-og.float()).abs().max()/og.float().abs().max()), flush=True)
