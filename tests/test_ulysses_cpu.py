"""Ulysses sequence<->head exchange (paper_2605_23445_b200/ulysses.py) on CPU:
world_size 2 and 4 over gloo, 127.0.0.1 rendezvous. The per-head step is a
plain torch fp32 softmax attention here (the exchange is what is under test;
the device step itself is covered by the -m gpu suites), so the sharded result
must equal the single-process computation exactly."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_23445_b200 import ulysses


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dense(q, k, v):
    # [N, H, d] per-head softmax attention, fp32
    s = torch.einsum("nhd,mhd->hnm", q, k) / q.shape[-1] ** 0.5
    return torch.einsum("hnm,mhd->nhd", torch.softmax(s, -1), v)


def _worker(rank, world, port, n, h, d, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        q, k, v = (torch.randn(n, h, d, generator=g) for _ in range(3))
        nl = n // world
        sl = slice(rank * nl, (rank + 1) * nl)
        seen = {}

        def step(qh, kh, vh, head0):
            seen["shape"] = tuple(qh.shape)
            seen["head0"] = head0
            # the exchanged head group must be the full-sequence slice of those heads
            hl = h // world
            assert torch.equal(qh, q[:, head0:head0 + hl]) and torch.equal(vh, v[:, head0:head0 + hl])
            return _dense(qh, kh, vh)

        o = ulysses.ulysses_attention(q[sl], k[sl], v[sl], step)
        ref = _dense(q, k, v)[sl]
        out_q.put((rank, seen["shape"], seen["head0"], float((o - ref).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,h,d", [(2, 64, 4, 8), (4, 96, 8, 16)])
def test_ulysses_exchange_matches_single_process(world, n, h, d):
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, h, d, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(out_q.get(timeout=10) for _ in range(world))
    for rank, shape, head0, err in res:
        assert shape == (n, h // world, d)
        assert head0 == rank * (h // world)
        assert err == 0.0


def test_ulysses_rejects_indivisible_heads():
    with pytest.raises(ValueError):
        ulysses._check(10, 6, 4)
