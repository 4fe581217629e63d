"""Multi-rank paths on one B200 (the round's GPU boxes have one GPU):

* head sharding: ranks own heads [r*H/P, (r+1)*H/P) of the same call and run
  dfs.run_step on them with no collective — outputs and masks must be
  bit-identical to the single-rank run over all heads (every stage is per head);
* Ulysses with the all-to-all fused into K2 / K5 (dfs_alltoall_run_step): ranks
  hold sequence shards [N/P, H, d]; rank r's K2 pulls its heads' rows from every
  shard and its K5 stores each output row into the shard owning the token.
  Simulated in one process (P sets of shard pointers) for P = 2, 4 and across two
  real processes sharing the GPU through CUDA IPC (dfs_alltoall_export/import,
  gloo for the handle exchange) — outputs bit-identical to the single-rank step.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

DIMS, H, D, B, BS = (4, 16, 32), 8, 128, 128, 16


def _inputs(seed=3):
    g = torch.Generator().manual_seed(seed)
    n = DIMS[0] * DIMS[1] * DIMS[2]
    return [torch.randn(n, H, D, generator=g).to(torch.bfloat16).cuda() for _ in range(3)]


def _sched(m, gamma=0.25, steps=1):
    return m.SparsitySchedule(total_steps=steps, warmup_fraction=0.0, phase_budgets=(gamma,), phase_fraction=1.0,
                              update_interval=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reference(m, q, k, v, steps=(0,), force_dense=False):
    cache = m.MaskCache()
    sched = _sched(m, steps=max(steps) + 1)
    outs = []
    for st in steps:
        o, _ = m.run_step(q, k, v, DIMS, m.ScoringParams(B, BS), sched, cache, layer=0, step=st,
                          force_dense=force_dense)
        outs.append(o.clone())
    masks = [cache.find(0, h)[0].bits.cpu() for h in range(H)] if not force_dense else None
    return outs, masks


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("force_dense", [False, True])
def test_fused_alltoall_simulated_ranks(world, force_dense):
    import paper_2605_23445_b200 as m
    from paper_2605_23445_b200 import ulysses

    q, k, v = _inputs()
    n = q.shape[0]
    nl, hl = n // world, H // world
    (want,), want_masks = _reference(m, q, k, v, force_dense=force_dense)
    shards = {key: [t[r * nl:(r + 1) * nl].contiguous() for r in range(world)] for key, t in
              (("q", q), ("k", k), ("v", v))}
    shards["o"] = [torch.full((nl, H, D), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    sched = _sched(m)
    caches = [m.MaskCache() for _ in range(world)]
    for r in range(world):  # every rank's step writes its heads into ALL shards
        st = ulysses.alltoall_step_local(shards, DIMS, m.ScoringParams(B, BS), sched, caches[r], 0, 0, r,
                                         force_dense=force_dense)
        assert st.dense == force_dense and len(st.sparsity) == hl
    torch.cuda.synchronize()
    got = torch.cat(shards["o"], 0)
    assert torch.equal(got, want)
    if not force_dense:
        for r in range(world):
            for hh in range(hl):
                assert torch.equal(caches[r].find(0, hh)[0].bits.cpu(), want_masks[r * hl + hh])


def test_fused_alltoall_mask_reuse_step():
    """Update step then reuse step (cached masks, fresh outputs) through the fused path."""
    import paper_2605_23445_b200 as m
    from paper_2605_23445_b200 import ulysses

    q, k, v = _inputs(seed=4)
    world, n = 2, q.shape[0]
    nl = n // world
    want, _ = _reference(m, q, k, v, steps=(0, 1))
    shards = {key: [t[r * nl:(r + 1) * nl].contiguous() for r in range(world)] for key, t in
              (("q", q), ("k", k), ("v", v))}
    shards["o"] = [torch.zeros((nl, H, D), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    sched = _sched(m, steps=2)
    caches = [m.MaskCache() for _ in range(world)]
    for step in (0, 1):
        for r in range(world):
            st = ulysses.alltoall_step_local(shards, DIMS, m.ScoringParams(B, BS), sched, caches[r], 0, step, r)
            assert all(st.mask_updated) == (step == 0)
        torch.cuda.synchronize()
        assert torch.equal(torch.cat(shards["o"], 0), want[step])


def _ipc_worker(rank, world, port, mode, res_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2605_23445_b200 as m
    from paper_2605_23445_b200 import ulysses

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, k, v = _inputs()
        n = q.shape[0]
        sched = _sched(m)
        params = m.ScoringParams(B, BS)
        cache = m.MaskCache()
        if mode == "heads":
            hl = H // world
            sl = slice(rank * hl, (rank + 1) * hl)
            o, _ = m.run_step(q[:, sl].contiguous(), k[:, sl].contiguous(), v[:, sl].contiguous(), DIMS, params,
                              sched, cache, layer=0, step=0)
            masks = torch.stack([cache.find(0, h)[0].bits for h in range(hl)]).cpu()
            outs = [None] * world
            dist.all_gather_object(outs, (o.cpu(), masks))
            if rank == 0:
                torch.save(outs, res_path)
        else:
            nl = n // world
            sl = slice(rank * nl, (rank + 1) * nl)
            mine = [t[sl].contiguous() for t in (q, k, v)]
            o = torch.zeros_like(mine[0])
            ex = ulysses.PeerExchange(*mine, o)
            ex.fused_run_step(DIMS, params, sched, cache, layer=0, step=0)
            outs = [None] * world
            dist.all_gather_object(outs, o.cpu())
            ex.close()
            if rank == 0:
                torch.save(outs, res_path)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["heads", "ulysses_ipc"])
def test_two_processes_on_one_gpu(mode, tmp_path):
    import torch.multiprocessing as mp

    import paper_2605_23445_b200 as m

    res = str(tmp_path / "res.pt")
    mp.spawn(_ipc_worker, args=(2, _free_port(), mode, res), nprocs=2, join=True)
    q, k, v = _inputs()
    (want,), want_masks = _reference(m, q, k, v)
    outs = torch.load(res)
    if mode == "heads":
        got = torch.cat([o for o, _ in outs], 1)
        masks = torch.cat([mk for _, mk in outs], 0)
        assert torch.equal(got, want.cpu())
        assert torch.equal(masks, torch.stack(want_masks))
    else:
        assert torch.equal(torch.cat(outs, 0), want.cpu())


def test_bench_two_ranks_on_one_gpu():
    """bench.py's multi-rank path as the driver's scaling run uses it (`bench.py --gpus N`
    relaunching itself under torch.distributed.run), here with two ranks sharing one B200
    (DFS_BENCH_RANKS_PER_GPU=2, gloo): one JSON line from rank 0 with n_gpus = 2, each rank
    holding half of the heads, a positive whole-job value, e2e and the CUPTI stage split."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DFS_BENCH_RANKS_PER_GPU="2")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--workload", "C", "--steps",
                        "3", "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                       env=env, cwd=root)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["heads_per_gpu"] == 24, d["config"]
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["step_kernel_ms_cupti"] and "failed" not in d["step_kernel_ms_cupti"], d["step_kernel_ms_cupti"]
