"""Time the streaming recall (dfs_block_recall) at a config shape (all heads, the step's masks)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2605_23445_b200 as dfs
from paper_2605_23445_b200 import ops
from bench import WORKLOADS, smooth_fields
wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "HY"]
dims, H, d, B, Bs, g = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
n = dims[0] * dims[1] * dims[2]
m = -(-n // B)
q, k, v = smooth_fields(dims, H, d, 1, torch.device("cuda"))
perm = dfs.hilbert3d_order(dims)
kh, pk = ops.permute_to_hnd(k, perm, Bs)
pq = ops.pool_gathered(q, perm, Bs)
lut = dfs.topk_lut(ops.score_pooled(pq, pk, n, dfs.ScoringParams(B, Bs)), g)
ptr = ops.lut_row_ptr(H, m, lut.shape[-1])
f = lambda: dfs.block_recall(q, kh, ptr, lut.reshape(-1), q_rows=perm.forward)
f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
rec = f()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'HY'} recall of {H} heads: {ms:.1f} ms, dense QK {2 * d * n * n * H / ms / 1e9:.0f} TFLOP/s, "
      f"recall mean {sum(rec) / len(rec):.4f} min {min(rec):.4f} max {max(rec):.4f}")
