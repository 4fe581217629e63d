"""Ulysses sequence <-> head layout swap around the DFSAttn step (multi-GPU).

The reference has no distributed code (its only parallelism is a
std::thread fan-out over (layer, head) pairs, scheduler.cpp:153). The B200 build
shards the path over the GPUs of one node by attention head: every stage of
run_step (scheduler.cpp:91-135) is per head, so a rank that holds all tokens of
its heads needs no communication at all (bench.py's head-sharded scaling run).

A DiT that keeps its activations sequence-sharded ([N/P, H, d] per rank, token
shards contiguous in raster order) needs one all-to-all before the step and one
after it:

    [N/P, H, d] --all_to_all--> [N, H/P, d]   (q, k, v in one exchange)
    run_step on the rank's H/P heads (reorder, score, top-K, sparse attention)
    [N, H/P, d] --all_to_all--> [N/P, H, d]   (o)

torch.distributed carries the exchange (NCCL over NVLink/NVSwitch on the GPU
box, gloo in the CPU tests); the exchange is wrapped so its layout logic is
testable without a GPU (`ulysses_attention(..., step_fn=...)`).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _check(n_local: int, heads: int, world: int):
    if heads % world:
        raise ValueError(f"ulysses: {heads} heads do not split over {world} ranks")
    if n_local < 1:
        raise ValueError("ulysses: empty token shard")


def seq_to_head(x_local: list[torch.Tensor], group=None) -> list[torch.Tensor]:
    """Sequence-sharded [N/P, H, d] tensors -> head-sharded [N, H/P, d] (raster order).

    All tensors travel in one all_to_all: the send buffer is [P, T, N/P, H/P, d]
    (destination rank major), the receive buffer [P, T, N/P, H/P, d] (source
    rank = token shard major), so concatenating the sources gives raster order."""
    world = dist.get_world_size(group)
    t = len(x_local)
    nl, h, d = x_local[0].shape
    _check(nl, h, world)
    hl = h // world
    send = torch.stack(x_local, 0).view(t, nl, world, hl, d).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    full = recv.permute(1, 0, 2, 3, 4).reshape(t, world * nl, hl, d)
    return [full[i].contiguous() for i in range(t)]


def head_to_seq(o_heads: torch.Tensor, group=None) -> torch.Tensor:
    """Head-sharded [N, H/P, d] -> sequence-sharded [N/P, H, d] (inverse of seq_to_head)."""
    world = dist.get_world_size(group)
    n, hl, d = o_heads.shape
    if n % world:
        raise ValueError("ulysses: token count does not split over the ranks")
    nl = n // world
    send = o_heads.contiguous().view(world, nl, hl, d)  # destination = token shard owner
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    # recv[src] holds head group src of my token shard
    return recv.permute(1, 0, 2, 3).reshape(nl, world * hl, d)


def ulysses_attention(q_local, k_local, v_local, step_fn, group=None):
    """Exchange, run `step_fn(q, k, v, head_offset) -> o` on the rank's heads, exchange back."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    q, k, v = seq_to_head([q_local, k_local, v_local], group)
    o = step_fn(q, k, v, rank * (q_local.shape[1] // world))
    return head_to_seq(o, group)


def ulysses_run_step(q_local, k_local, v_local, dims, params, schedule, cache, layer: int, step: int,
                     group=None, force_dense: bool = False):
    """DFSAttn step (paper_2605_23445_b200.run_step) on sequence-sharded bf16 activations.

    q/k/v_local: [N/P, H, d] CUDA bf16, the rank's contiguous raster token shard.
    Returns the rank's [N/P, H, d] output shard; per-head stats refer to the
    rank's heads [rank*H/P, (rank+1)*H/P) (the mask cache is keyed by local head)."""
    from .ops import run_step

    stats_box = {}

    def step_fn(q, k, v, head0):
        out, stats = run_step(q, k, v, dims, params, schedule, cache, layer=layer, step=step,
                              force_dense=force_dense)
        stats_box["stats"] = stats
        stats_box["head0"] = head0
        return out

    o = ulysses_attention(q_local, k_local, v_local, step_fn, group)
    return o, stats_box["stats"]
