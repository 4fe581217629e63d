"""K5 alone in a sustained loop (~4 s) at a config shape: CUDA-event ms per call, median SM
clock and board power (NVML) — the power-capped view of a K5 variant (select it with
DFS_B200_LIB). python tools/k5_power.py [HY|C] [seconds]"""
import statistics
import sys
import threading
import time

import torch

sys.path.insert(0, '.')
import paper_2605_23445_b200 as dfs  # noqa: E402
from paper_2605_23445_b200 import ops  # noqa: E402
from bench import WORKLOADS, smooth_fields  # noqa: E402

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else 'HY']
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
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


def call():
    dfs.sparse_attention_csr(q, kh, vh, ptr, lut.reshape(-1), B, layout=1, out_layout=0, in_rows=perm.forward,
                             out_rows=perm.forward, out=out)


for _ in range(3):
    call()
torch.cuda.synchronize()
import pynvml as nv  # noqa: E402

nv.nvmlInit()
hdl = nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
pw, clk, stop = [], [], threading.Event()


def sample():
    while not stop.is_set():
        pw.append(nv.nvmlDeviceGetPowerUsage(hdl) / 1000.0)
        clk.append(nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM))
        time.sleep(0.01)


th = threading.Thread(target=sample, daemon=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
calls = 0
t_end = time.time() + secs
th.start()
e0.record()
while time.time() < t_end:
    for _ in range(10):
        call()
    calls += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
stop.set()
th.join()
half = len(pw) // 2  # the second half: the power loop has settled
print(f"ms/call {e0.elapsed_time(e1) / calls:.3f}  sm_mhz {statistics.median(clk[half:]):.0f}  "
      f"power_w {statistics.median(pw[half:]):.1f}  calls {calls}")
