"""PCIe probe: pinned host<->device copy bandwidth on this box (the bound of bench.py's e2e
number): H2D alone, D2H alone, both directions concurrently, one vs three copy streams."""
import time

import torch

n = 730 * 1024 * 1024 // 2  # one HY q/k/v tensor (bf16 elements)
hs = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
ho = torch.empty(n, dtype=torch.bfloat16).pin_memory()
ds = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
do = torch.empty(n, dtype=torch.bfloat16, device="cuda")
st = [torch.cuda.Stream() for _ in range(4)]


def run(h2d_streams, d2h, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for i in range(3):
            with torch.cuda.stream(st[i % h2d_streams]):
                ds[i].copy_(hs[i], non_blocking=True)
        if d2h:
            with torch.cuda.stream(st[3]):
                ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / reps
    return dt


for _ in range(2):
    run(1, False)
gb_in, gb_out = 3 * n * 2 / 1e9, n * 2 / 1e9
for h, d in ((1, False), (3, False), (1, True), (3, True)):
    dt = run(h, d)
    print(f"h2d streams {h}, d2h {'on ' if d else 'off'}: {dt * 1e3:7.2f} ms per call-equivalent "
          f"(H2D {gb_in:.2f} GB -> {gb_in / dt:5.1f} GB/s{', D2H %.2f GB' % gb_out if d else ''})")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    ho.copy_(do, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"d2h alone: {gb_out / dt:5.1f} GB/s")
