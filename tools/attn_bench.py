"""K5-only timing at a config shape with the real (scored) masks; prints executed TFLOP/s.

    python tools/attn_bench.py [HY|W7|W4|C] [reps]

Each DFS_ATTN_POLY variant runs in a fresh subprocess (the setting is read once per process).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, torch
sys.path.insert(0, ROOT)
import paper_2605_23445_b200 as dfs
from paper_2605_23445_b200 import ops
from bench import WORKLOADS, smooth_fields, executed_flops
wl = WORKLOADS[WL]
dims, H, d, B, Bs, g = wl["dims"], wl["heads"], wl["d"], wl["block"], wl["sub"], wl["gamma"]
n = dims[0] * dims[1] * dims[2]
m = -(-n // B)
q, k, v = smooth_fields(dims, H, d, 1, torch.device("cuda"))
perm = dfs.hilbert3d_order(dims)
qh, pq = ops.permute_to_hnd(q, perm, Bs)
kh, pk = ops.permute_to_hnd(k, perm, Bs)
vh, _ = ops.permute_to_hnd(v, perm, 0)
S = ops.score_pooled(pq, pk, n, dfs.ScoringParams(B, Bs))
lut = dfs.topk_lut(S, g)
K = lut.shape[-1]
ptr = ops.lut_row_ptr(H, m, K)
out = torch.empty_like(q)
f = lambda: dfs.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), B, out_layout=1, out_rows=perm.forward, out=out)
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(REPS): f()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / REPS
fl = executed_flops(lut, n, B, d)
print(f"{WL} poly={POLY} K5 {ms:.3f} ms  executed {fl/ms/1e9:.1f} TFLOP/s  dense-equiv {4*d*n*n*H/ms/1e9:.1f}")
'''

if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "HY"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    polys = os.environ.get("POLYS", "4").split(",")
    for poly in polys:
        env = dict(os.environ, DFS_ATTN_POLY=poly)
        code = CODE.replace("ROOT", repr(ROOT)).replace("WL", repr(wl)).replace("REPS", str(reps)).replace(
            "POLY}", poly + "}")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        print(r.stdout.strip() or r.stderr[-800:], flush=True)
