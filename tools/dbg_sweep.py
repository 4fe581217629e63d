import sys, time, subprocess
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import torch
    import paper_2605_23445_b200 as m
    n, k, h, d = (int(x) for x in sys.argv[1:5])
    g = torch.Generator().manual_seed(0)
    q, kk, v = (torch.randn(h, n, d, generator=g).bfloat16().cuda() for _ in range(3))
    mq = -(-n // 128)
    lut = torch.stack([torch.stack([torch.randperm(mq, generator=g)[:k].sort().values for _ in range(mq)]) for _ in range(h)]).int().cuda()
    ptr = m.ops.lut_row_ptr(h, mq, k)
    torch.cuda.synchronize()
    t = time.time()
    o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128)
    torch.cuda.synchronize()
    print(f"n={n} k={k} h={h} d={d} tiles={mq*h} ok {time.time()-t:.3f}s", flush=True)
else:
    for args in [(17550, 28, 3, 128), (17550, 93, 3, 128), (17550, 28, 24, 128), (118800, 8, 1, 128), (118800, 93, 1, 128),
                 (118800, 8, 4, 128), (118800, 93, 4, 64), (118800, 93, 24, 128)]:
        try:
            r = subprocess.run([sys.executable, __file__] + [str(a) for a in args], timeout=25, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
        except subprocess.TimeoutExpired:
            print("TIMEOUT", args, flush=True)
