"""Per-block timeline of one CTA of K5 at HY (needs a -DDFS_ATTN_TRACE_BUILD library via DFS_B200_LIB)."""
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
t = np.fromfile('gpurun_out/attn_trace.bin', dtype=np.uint64).reshape(24, 256).astype(np.int64)
names = ['kv_wait_start', 'kv_wait_done', 'p_wait_start', 'p_wait_done', 'A_s_wait', 'A_s_ready', 'A_barrier',
         'A_arrive', 'B_s_wait', 'B_s_ready', 'B_barrier', 'B_arrive']
lo, hi = 60, 120
t0 = t[0, lo * 2]
for i, nm in enumerate(names):
    print(f"{nm:14s}", ' '.join(f"{x - t0:7d}" for x in t[i, lo:lo + 12]))
for s, base in (("A", 4), ("B", 8)):
    w = (t[base + 1, lo:hi] - t[base, lo:hi]).mean()
    busy = (t[base + 3, lo:hi] - t[base + 1, lo:hi]).mean()
    pre = (t[base + 2, lo:hi] - t[base + 1, lo:hi]).mean()
    per = np.diff(t[base + 3, lo:hi]).mean()
    print(f"stream {s}: period/block {per:.0f} (2 blocks of the tile), S wait {w:.0f}, busy {busy:.0f} (to barrier {pre:.0f})")
# warpgroup 0's phases per block (events 4 s_wait, 5 s_ready, 12 ld done, 13 max done,
# 6 row-max exchange done, 14 exponentials done, 7 P stored + arrived)
ph = [(4, 5, "S wait"), (5, 12, "TMEM ld"), (12, 13, "max"), (13, 6, "exchange"), (6, 14, "exp loop"),
      (14, 7, "P store"), (7, 4, "to next")]
for a_, b_, nm in ph:
    if nm == "to next":
        dt = (t[4, lo + 1:hi + 1] - t[7, lo:hi]).mean()
    else:
        dt = (t[b_, lo:hi] - t[a_, lo:hi]).mean()
    print(f"  A {nm:10s} {dt:7.0f} cycles/block")
pw = (t[3, lo:hi] - t[2, lo:hi]).mean()
kvw = (t[1, 2 * lo:2 * hi] - t[0, 2 * lo:2 * hi]).mean()
print(f"MMA: p_full wait/PV {pw:.0f}, kv wait/ring entry {kvw:.0f}, PV period {np.diff(t[2, lo:hi]).mean():.0f}")
