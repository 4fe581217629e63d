import sys, time, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as m
torch.manual_seed(0)
def rel(a, b): return float((a.float()-b.float()).abs().max()/b.float().abs().max())
for d in (64, 128):
    for h in (1, 2):
        for nq, nk in ((256, 256), (777, 1500)):
            q = torch.randn(h, nq, d).bfloat16().cuda(); k = torch.randn(h, nk, d).bfloat16().cuda(); v = torch.randn(h, nk, d).bfloat16().cuda()
            o_h = m.sparse_attention_csr(q, k, v, None, None, 128)              # HND dense
            o_g = m.sparse_attention_csr(q, k, v, None, None, 128, force_generic=True)
            qn, kn, vn = (x.transpose(0, 1).contiguous() for x in (q, k, v))
            o_n = m.sparse_attention_csr(qn, kn, vn, None, None, 128, layout=0)  # NHD dense
            o_n2 = m.sparse_attention_csr(qn, kn, vn, None, None, 128, layout=0, out_layout=1)
            torch.cuda.synchronize()
            print(d, h, nq, nk, 'hnd', rel(o_h, o_g), 'nhd', rel(o_n.transpose(0, 1), o_g), 'nhd->hnd', rel(o_n2, o_g), flush=True)
