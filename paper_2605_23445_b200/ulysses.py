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


# --------------------------------------------------------------------------- #
# the all-to-all fused into K2 / K5 over peer memory (dfs_alltoall_*)          #
# --------------------------------------------------------------------------- #


def alltoall_step_local(shards, dims, params, schedule, cache, layer: int, step: int, rank: int,
                        force_dense: bool = False):
    """dfs_alltoall_run_step for `rank` given every rank's shard pointers as seen by this process.

    shards: dict with lists "q", "k", "v", "o" of per-rank [N/P, H, d] bf16 CUDA tensors or raw
    device pointers (ints). The rank's head group [rank*H/P, (rank+1)*H/P) is computed: K2 pulls its
    heads' token rows from every shard, K5 stores each output row into the shard owning the token.
    Returns StepStats for the rank's heads. Callers synchronise the ranks around the call."""
    import ctypes as C

    from . import _capi as capi
    from .ops import StepStats, _dims, _stream

    world = len(shards["q"])
    if world > capi.MAX_PEERS:
        raise ValueError(f"ulysses: at most {capi.MAX_PEERS} ranks")
    ref = shards["q"][rank]
    nl, h, d = ref.shape
    if h % world:
        raise ValueError(f"ulysses: {h} heads do not split over {world} ranks")
    for key in ("q", "k", "v", "o"):
        for t in shards[key]:
            if isinstance(t, torch.Tensor) and (t.shape != ref.shape or t.dtype != torch.bfloat16 or
                                                not t.is_contiguous()):
                raise ValueError("ulysses: shards must be contiguous bf16 [N/P, H, d] tensors of one shape")
    dims = _dims(dims)
    hl = h // world

    def ptrs(key):
        arr = (C.c_void_p * capi.MAX_PEERS)()
        for r, t in enumerate(shards[key]):
            arr[r] = t.data_ptr() if isinstance(t, torch.Tensor) else int(t)
        return arr

    dense, budget = C.c_int(), C.c_double()
    upd = (C.c_int * hl)()
    spars = (C.c_double * hl)()
    a = capi.AlltoallStepArgs(ptrs("q"), ptrs("k"), ptrs("v"), ptrs("o"), world, rank, nl, h, d, dims.frames,
                              dims.height, dims.width, params.block_size, params.sub_block_size, layer, step,
                              int(force_dense), C.pointer(dense), C.pointer(budget),
                              C.cast(upd, C.POINTER(C.c_int)), C.cast(spars, C.POINTER(C.c_double)))
    with cache.lock:
        capi.call("dfs_alltoall_run_step", cache.handle.ptr, C.byref(schedule._s), C.byref(a), _stream())
    return StepStats(bool(dense.value), budget.value, [bool(x) for x in upd], list(spars))


class PeerExchange:
    """One rank's view of every rank's sequence shards, mapped with CUDA IPC (dfs_alltoall_export /
    import): the data path of fused_run_step never goes through NCCL or a staging copy.

    q, k, v, o: this rank's [N/P, H, d] bf16 CUDA shards (o is written by the ranks' K5s)."""

    def __init__(self, q, k, v, o, group=None):
        import ctypes as C

        from . import _capi as capi

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.local = {"q": q, "k": k, "v": v, "o": o}
        mine = {}
        for key, t in self.local.items():
            hd = capi.PeerHandle()
            capi.call("dfs_alltoall_export", C.c_void_p(t.data_ptr()), C.byref(hd))
            mine[key] = (bytes(hd.bytes), int(hd.offset))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.shards = {key: [] for key in self.local}
        self._opened = []
        for r in range(self.world):
            for key in self.local:
                if r == self.rank:
                    self.shards[key].append(self.local[key])
                    continue
                raw, off = everyone[r][key]
                hd = capi.PeerHandle()
                C.memmove(hd.bytes, raw, 64)
                hd.offset = off
                p = C.c_void_p()
                capi.call("dfs_alltoall_import", C.byref(hd), C.byref(p))
                self._opened.append(p.value)
                self.shards[key].append(p.value)

    def close(self):
        import ctypes as C

        from . import _capi as capi

        for p in self._opened:
            capi.call("dfs_alltoall_close", C.c_void_p(p))
        self._opened = []

    def fused_run_step(self, dims, params, schedule, cache, layer: int, step: int, force_dense: bool = False):
        """Alg. 1 step on the sequence-sharded activations: every rank's K2 reads its heads from
        all shards, every rank's K5 writes its heads' rows into all shards; barriers on both
        sides make the peers' inputs and outputs visible. Returns the rank's head-group stats."""
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
        stats = alltoall_step_local(self.shards, dims, params, schedule, cache, layer, step, self.rank,
                                    force_dense)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)
        return stats
